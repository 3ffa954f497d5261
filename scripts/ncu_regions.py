"""Split one kernel's SASS (ncu source page) into regions between BAR.SYNC
instructions and sum warp-stall samples / executed instructions per region.
usage: python scripts/ncu_regions.py REPORT KERNEL_REGEX"""
import csv, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
iA, iS, iN, iI = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
regions, cur = [], None
def new(addr):
    return {"start": addr, "samples": 0.0, "inst": 0.0, "fp64": 0.0, "lds": 0.0, "stalls": collections.Counter(), "n": 0}
cur = new("begin")
for r in rows[hi + 1:]:
    if len(r) <= iI: continue
    src = r[iS].strip()
    try: n = float(r[iN] or 0); ins = float(r[iI] or 0)
    except ValueError: continue
    cur["samples"] += n; cur["inst"] += ins; cur["n"] += 1
    op = src.split()[0] if src else ""
    if op.startswith("@"): op = src.split()[1]
    if op.split(".")[0] in ("DADD", "DMUL", "DFMA"): cur["fp64"] += ins
    if op.startswith("LDS"): cur["lds"] += ins
    for i, c in stall_cols:
        try: cur["stalls"][c] += float(r[i] or 0)
        except ValueError: pass
    if op.startswith("BAR.SYNC") or op.startswith("EXIT"):
        cur["end"] = r[iA]; regions.append(cur); cur = new(r[iA])
regions.append(cur)
tot = sum(x["samples"] for x in regions) or 1
for k, x in enumerate(regions):
    if x["samples"] < 0.005 * tot: continue
    top = ", ".join("%s %.0f%%" % (c, 100 * v / max(x["samples"], 1)) for c, v in x["stalls"].most_common(5))
    print("region %2d  %5.1f%% samples  sass=%4d  inst=%10.0f  fp64=%4.1f%%  lds=%4.1f%%  | %s" % (
        k, 100 * x["samples"] / tot, x["n"], x["inst"], 100 * x["fp64"] / max(x["inst"], 1), 100 * x["lds"] / max(x["inst"], 1), top))
