"""C3 (Lagrange 320^3) on one GPU split into 1/2/4/8 emulated slabs (device-copy halo
exchange), with and without the boundary-first overlap (SALE_OVERLAP), ms per cycle.
Each setting in its own process (the switch is read once).  python scripts/overlap_bench.py"""
import json
import os
import subprocess
import sys

CODE = r"""
import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale
cfg, _ = config('C3')
g = Sale(cfg, impl='fused', local_slabs=%d)
g.step(3); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
a.record(g.stream); g.step_async(K); b.record(g.stream); torch.cuda.synchronize()
rc, done = g.sync(); assert rc == 0 and done == K
print(json.dumps(a.elapsed_time(b) / K))
"""
out = []
for slabs in (1, 2, 4, 8):
    for ov in ("1", "0"):
        if slabs == 1 and ov == "0":
            continue
        r = subprocess.run([sys.executable, "-c", CODE % slabs], env=dict(os.environ, SALE_OVERLAP=ov),
                           capture_output=True, text=True)
        ms = float(r.stdout.strip().splitlines()[-1])
        line = {"workload": "C3", "local_slabs": slabs, "overlap": ov == "1", "ms_per_cycle": ms}
        print(json.dumps(line), flush=True)
        out.append(line)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        for l in out:
            f.write(json.dumps(l) + "\n")
