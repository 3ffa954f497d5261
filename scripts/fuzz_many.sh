#!/bin/bash
# scripts/fuzz_stress.py in 16 processes: N cases from seed S (16 x N/16), merged into OUT.
# usage: bash scripts/fuzz_many.sh N S OUT.json
N=${1:-2000}; S=${2:-50000}; OUT=${3:-gpurun_out/fuzz.json}
D=$(mktemp -d); P=$((N / 16))
for p in $(seq 0 15); do python scripts/fuzz_stress.py $P $((S + p * P)) $D/fz_$p.json > $D/log_$p.txt 2>&1 & done
wait
python - "$D" "$OUT" "$N" "$S" <<'PY'
import glob, json, sys
d, out, n, s = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
tot, bad, st, secs = 0, [], {}, 0.0
for f in sorted(glob.glob(d + "/fz_*.json")):
    r = json.load(open(f)); tot += r["cases"]; bad += r["mismatches"]; secs = max(secs, r.get("seconds", 0))
    for k, v in r["final_status_counts"].items(): st[k] = st.get(k, 0) + v
json.dump({"cases": tot, "mismatches": bad, "final_status_counts": st, "wall_seconds": secs,
           "what": f"scripts/fuzz_stress.py, 16 processes, seeds {s}-{s + n - 1}, one B200"}, open(out, "w"))
print(tot, len(bad), st)
PY
