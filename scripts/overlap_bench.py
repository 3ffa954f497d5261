"""Boundary-first cycles (sale_params.overlap) on emulated slabs: C3 / C4 on 1, 2, 4, 8
slabs of one GPU, overlap off vs on (CUDA events, 20 timed cycles).  On one GPU the
exchange is a set of device copies; the numbers show the cost of the split launches,
not the hidden NCCL time.  python scripts/overlap_bench.py [out.json]"""
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2209_01983_b200.configs import config  # noqa: E402
from paper_2209_01983_b200.sale import Sale  # noqa: E402

lines = []
for name in ("C4", "C3"):
    cfg, _ = config(name)
    for slabs in (1, 2, 4, 8):
        for ov in ((-1, 1) if slabs > 1 else (-1,)):
            g = Sale(dict(cfg, overlap=ov), local_slabs=slabs)
            g.step(3)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(g.stream)
            g.step_async(20)
            b.record(g.stream)
            rc = g.sync()
            torch.cuda.synchronize()
            line = {"workload": name, "slabs": slabs, "overlap": ov, "ms_per_cycle": a.elapsed_time(b) / 20,
                    "rc": rc}
            print(json.dumps(line), flush=True)
            lines.append(line)
            g.close()
            del g
            torch.cuda.empty_cache()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        for ln in lines:
            f.write(json.dumps(ln) + "\n")
