"""Per-CUDA-source-line stall samples of one kernel in an ncu report (needs -lineinfo).
usage: python scripts/ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import csv, os, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
recs, tot, fname, h = [], 0.0, "", None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = os.path.basename(r[1]); continue
    if r[0] == "Line No": h = r; continue
    if h is None or not r[0]: continue
    iN = 4  # Warp Stall Sampling (All Samples)
    try: n = float(r[iN] or 0); ins = float(r[7] or 0)
    except (ValueError, IndexError): continue
    if n == 0 and ins == 0: continue
    tot += n
    cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    st = sorted(((float(r[i] or 0), c[6:]) for i, c in cols if i < len(r) and r[i] not in ("", "-")), reverse=True)[:3]
    recs.append((n, "%s:%s" % (fname, r[0]), r[1].strip()[:80], ins, st))
recs.sort(reverse=True)
print("total samples", tot)
for n, ln, src, ins, st in recs[:top]:
    print("%5.1f%% %-22s inst=%9.0f %-80s %s" % (100 * n / tot, ln, ins, src, " ".join("%s:%d" % (b, a) for a, b in st)))
