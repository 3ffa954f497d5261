"""Static SASS statistics per kernel of an object/.so: instruction count, FP64,
MUFU, CALL, LDS/STS, local memory.  usage: python scripts/sass_stats.py FILE [name-regex]"""
import collections, re, subprocess, sys
f = sys.argv[1]
rx = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["cuobjdump", "-sass", f], capture_output=True, text=True).stdout
cur, stats = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1); stats[cur] = collections.Counter(); continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(2)
        if op == "NOP": continue
        c = stats[cur]; c["all"] += 1
        if op in ("DADD", "DMUL", "DFMA"): c["fp64"] += 1
        elif op.startswith("MUFU"): c["mufu"] += 1
        elif op == "CALL": c["call"] += 1
        elif op in ("LDS", "STS"): c[op.lower()] += 1
        elif op in ("LDL", "STL"): c["local"] += 1
        elif op in ("BSSY", "BSYNC", "BRA"): c["ctl"] += 1
for k, c in stats.items():
    if rx and not rx.search(k): continue
    print("%-60s %s" % (k[:60], " ".join("%s=%d" % kv for kv in sorted(c.items()))))
