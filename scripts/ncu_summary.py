"""Summarise an ncu report: per kernel time, pipe utilisation, stalls, opcode mix."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
regex = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ['gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum', 'launch__registers_per_thread',
        'smsp__sass_inst_executed_op_shared_ld.sum', 'smsp__inst_executed_op_branch.sum']
stall = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')]
    if regex and regex not in name: continue
    print('=====', name[:60])
    for w in want:
        if w in hdr: print('   %-62s %s' % (w, r[hdr.index(w)]))
    st = sorted(((float(r[hdr.index(h)] or 0), h.replace('smsp__pcsamp_warps_issue_stalled_', '')) for h in stall), reverse=True)[:7]
    print('   stalls:', ', '.join('%s %d' % (n, v) for v, n in st))
if len(sys.argv) > 3:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + sys.argv[3]],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(src.splitlines()))
    h = rr[1]; iS = h.index('Source'); iE = h.index('Instructions Executed')
    by = collections.Counter(); tot = 0
    for r in rr[2:]:
        if len(r) <= iE: continue
        t = r[iS].split()
        if not t: continue
        op = (t[1] if t[0].startswith('@') and len(t) > 1 else t[0]).split('.')[0]
        try: n = int(float(r[iE] or 0))
        except ValueError: continue
        by[op] += n; tot += n
    print('   opcode mix:', ', '.join('%s %.1f%%' % (o, 100 * n / tot) for o, n in by.most_common(16)))
