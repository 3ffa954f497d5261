"""Average DRAM bytes (read + write) per launch of every kernel in an ncu report
-> profiles/traffic_<cfg>.json (read by bench.py for roofline.traffic).
usage: python scripts/traffic_from_ncu.py REPORT CFG OUT_JSON"""
import collections, csv, json, subprocess, sys
rep, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
iK, iR, iW, iT = (h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"),
                  h.index("gpu__time_duration.sum"))
iF = h.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
acc = collections.defaultdict(list)
for r in rows[2:]:
    name = r[iK].split("(")[0].replace("void ", "").replace("sale::", "").strip()
    acc[name].append((float(r[iR]) + float(r[iW]), float(r[iT]), float(r[iF])))
per = {k: sum(x[0] for x in v) / len(v) for k, v in acc.items()}
dur = {k: sum(x[1] for x in v) / len(v) for k, v in acc.items()}
fp = {k: sum(x[2] for x in v) / len(v) for k, v in acc.items()}
json.dump({"config": cfg, "source": f"ncu --set full ({rep.split('/')[-1]}), dram__bytes_read.sum + dram__bytes_write.sum",
           "dram_bytes_per_launch": per, "gpu_time_ns_per_launch": dur,
           "fp64_pipe_pct_of_active": fp}, open(out, "w"), indent=1)
print(json.dumps(per, indent=1))
