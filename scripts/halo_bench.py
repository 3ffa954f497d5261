"""Halo modes on emulated slabs of one GPU: C3 / C4 on 1, 2, 4, 8 slabs with the copy
exchange (device copies after the cycle's kernels), boundary-first cycles (the copies on
a side stream), and the peer-store halo (sale_params.halo = SALE_HALO_PEER: the
producing kernels store the ghost planes into the neighbouring slab; no copies).  CUDA
events, 20 timed cycles after 3.  On one GPU this measures what each mode costs the
kernels (the extra stores, the split launches), not the NVLink transfer time they hide.
python scripts/halo_bench.py [out.json]"""
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2209_01983_b200.configs import config  # noqa: E402
from paper_2209_01983_b200.sale import HALO_COPY, HALO_PEER, Sale  # noqa: E402

MODES = {"copy": dict(overlap=-1, halo=HALO_COPY), "copy+boundary-first": dict(overlap=1, halo=HALO_COPY),
         "peer": dict(overlap=-1, halo=HALO_PEER)}
lines = []
for name in ("C4", "C3"):
    cfg, _ = config(name)
    for slabs in (1, 2, 4, 8):
        for mode, kw in MODES.items():
            if slabs == 1 and mode != "copy":
                continue
            g = Sale(dict(cfg, **kw), local_slabs=slabs)
            g.step(3)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(g.stream)
            g.step_async(20)
            b.record(g.stream)
            rc = g.sync()
            torch.cuda.synchronize()
            line = {"workload": name, "slabs": slabs, "halo": mode, "ms_per_cycle": a.elapsed_time(b) / 20,
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
