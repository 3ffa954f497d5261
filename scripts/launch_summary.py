"""Summarise an ncu launch list (gpu__time_duration.sum per launch) per kernel.
usage: python scripts/launch_summary.py launches.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iK, iV, iM = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
acc = collections.defaultdict(list)
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum": continue
    acc[r[iK].split("(")[0].replace("void ", "").replace("sale::", "")].append(float(r[iV].replace(",", "")))
nmax = max(len(v) for v in acc.values())
cyc = {k: v for k, v in acc.items() if len(v) >= nmax}  # the kernels every cycle launches
tot = sum(sum(v) for v in cyc.values())
print("kernel | launches | avg us | share of the per-cycle kernels")
for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    share = 100 * sum(v) / tot if k in cyc else 0.0
    print("%s | %d | %.1f | %.1f%%" % (k, len(v), sum(v) / len(v) / 1e3, share))
