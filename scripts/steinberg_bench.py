"""Throughput of sale_steinberg (the paper's Fig. 6b cell kernel) on the C4 and C3
states: cells/s and achieved GB/s of the algorithmic bytes against the measured HBM
copy bandwidth.  python scripts/steinberg_bench.py [out.json]"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale

peak = json.load(open('/root/repo/MEASURED_PEAKS.json'))['hbm_gbs'] if os.path.exists('/root/repo/MEASURED_PEAKS.json') else 6650.0
prm = dict(G0=0.43, GP=1.7, GT=0.3, Y0=0.2, Ymax=0.9, beta=3.0, n=0.5, cv=0.8, rho0=1.1, T0=0.05)
lines = []
for name, algo in (("C4", 48.0), ("C3", 64.0)):
    cfg, _ = config(name)
    g = Sale(cfg)
    g.step(3)
    cells = cfg["nx"] * cfg["ny"] * cfg["nz"]
    eps_field = torch.rand(g.cell_shape, dtype=torch.float64, device=g.torch_device)
    for eps, nbytes in ((eps_field, algo), (None, algo - 8.0)):  # with / without a plastic strain field
        out = g.steinberg(prm, eps)
        for _ in range(3):
            g.steinberg(prm, eps, out=out)
        torch.cuda.synchronize()
        n = 50
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(g.stream)
        for _ in range(n):
            g.steinberg(prm, eps, out=out)
        b.record(g.stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        gbs = nbytes * cells / (ms * 1e-3) / 1e9
        line = {"workload": name, "eps": "field" if eps is not None else "none", "cells": cells, "ms_per_call": ms,
                "cells_per_s": cells / (ms * 1e-3), "algo_bytes_per_cell": nbytes, "achieved_gbs": gbs,
                "peak_gbs": peak, "frac": gbs / peak, "bound": "hbm"}
        print(json.dumps(line), flush=True)
        lines.append(line)
        del out
    del g, eps_field
    torch.cuda.empty_cache()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        for l in lines:
            f.write(json.dumps(l) + "\n")
