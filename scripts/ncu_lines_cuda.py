"""Warp-stall samples per CUDA source line of one kernel (ncu source page, cuda+sass view).
usage: python scripts/ncu_lines_cuda.py REPORT KERNEL_REGEX [N]"""
import csv, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iN = h.index("Warp Stall Sampling (All Samples)")
stall = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_")]
src = {}
try:
    path = rows[0][1]
    src = {k + 1: l.rstrip() for k, l in enumerate(open(path))}
except Exception:
    pass
recs, tot = [], 0.0
for r in rows[hi + 1:]:
    if not r or not r[0]:
        continue
    try:
        ln, n = int(r[0]), float(r[iN] or 0)
    except ValueError:
        continue
    st = collections.Counter()
    for i, c in stall:
        try: st[c] += float(r[i] or 0)
        except (ValueError, IndexError): pass
    tot += n
    recs.append((n, ln, st))
print("total samples %d" % tot)
for n, ln, st in sorted(recs, reverse=True)[:N]:
    top = ", ".join("%s %d%%" % (k, 100 * v / max(n, 1)) for k, v in st.most_common(3))
    print("%5.1f%%  L%-5d %-60s | %s" % (100 * n / tot, ln, src.get(ln, "").strip()[:60], top))
