"""Top SASS instructions of one kernel by a stall reason (ncu source page).
usage: python scripts/ncu_top_sass.py REPORT KERNEL_REGEX [stall=long_sb] [N]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
st = sys.argv[3] if len(sys.argv) > 3 else "long_sb"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
iS, iA, iI, iX = h.index("Source"), h.index("Address"), h.index("Instructions Executed"), h.index("stall_" + st)
recs = []
for k, r in enumerate(rows[hi + 1:]):
    try: recs.append((float(r[iX] or 0), k, r[iS].strip(), float(r[iI] or 0)))
    except (ValueError, IndexError): pass
tot = sum(x[0] for x in recs)
print("total %s samples: %d" % (st, tot))
for v, k, src, ins in sorted(recs, reverse=True)[:N]:
    print("%6d  #%-5d %-70s inst=%d" % (v, k, src[:70], ins))
