#!/bin/bash
# per-kernel time / FP64 / issue / DRAM snapshot of a config (ncu, a few launches of each)
CFG=${CFG:-C4}
python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread --clock-control none -k regex:"kc_|ke_|kl_|kr_|kn_" -s ${SKIP:-14} -c ${COUNT:-7} --csv python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ll_$CFG.csv 2>&1
python - <<'PY'
import csv, collections, os
cfg = os.environ.get("CFG", "C4")
rows = list(csv.reader([l for l in open(f"gpurun_out/ll_{cfg}.csv") if l.startswith('"')]))
h = rows[0]; iK = h.index('Kernel Name'); iM = h.index('Metric Name'); iV = h.index('Metric Value')
d = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    d[r[iK].split('(')[0].replace('void ', '')][r[iM]].append(float(r[iV].replace(',', '')))
for k, v in d.items():
    g = {m.split('__')[1].split('.')[0]: sum(x) / len(x) for m, x in v.items()}
    print("%-24s ms=%.3f fp64=%.1f%% issue=%.1f%% dram=%.1f%% regs=%d" % (k[:24], g['time_duration'] / 1e6, g['pipe_fp64_cycles_active'], g['issue_active'], g['throughput'], g['registers_per_thread']))
PY
