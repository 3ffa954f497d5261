"""Throughput of the multi-material cycle on the C4 and C3
meshes: zone-cycles/s with nmat = 1, 2, 4 materials mixed in every cell (equal
fractions 1/nmat, material densities and energies of the Sedov state, gammas
1.4 / 5/3 / 1.2 / 2.0), beside the single-material kernels on the same mesh.  CUDA events on the context's stream, W warm-up cycles, K timed cycles, the
per-class split from sale_profile.  python scripts/materials_bench.py [out.json]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2209_01983_b200.configs import config  # noqa: E402
from paper_2209_01983_b200.sale import Sale  # noqa: E402

GAMMAS = [1.4, 5.0 / 3.0, 1.2, 2.0]
W, K = 3, 20


def timed(ctx, cells):
    rc, done = ctx.step(W)
    assert rc == 0, ctx.last_error()
    torch.cuda.synchronize()
    ctx.profile(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream)
    ctx.step_async(K)
    b.record(ctx.stream)
    torch.cuda.synchronize()
    rc, done = ctx.sync()
    assert rc == 0 and done == K, ctx.last_error()
    ms = a.elapsed_time(b) / K
    prof = {k: v[0] / K for k, v in ctx.profile_read().items()}
    ctx.profile(False)
    return ms, cells / (ms * 1e-3), prof


lines = []
for name in ("C4", "C3"):
    cfg, _ = config(name)
    cells = cfg["nx"] * cfg["ny"] * cfg["nz"]
    for nmat in (0, 1, 2, 4):
        c = dict(cfg, nmat=nmat, mat_gamma=GAMMAS[:nmat]) if nmat else cfg
        g = Sale(c)
        if nmat > 1:
            m, e = g.get("MAT_M0"), g.get("MAT_E0")
            for k in range(nmat):
                g.set(f"MAT_F{k}", np.full(g.cell_shape, 1.0 / nmat))
                g.set(f"MAT_M{k}", m / nmat)
                g.set(f"MAT_E{k}", e)
        ms, rate, prof = timed(g, cells)
        line = {"workload": name, "nmat": nmat,
                "cells": cells, "ms_per_cycle": ms, "zone_cycles_per_s": rate,
                "class_ms_per_cycle": prof, "steps": K, "warmup": W}
        print(json.dumps(line), flush=True)
        lines.append(line)
        g.close()
        del g
        torch.cuda.empty_cache()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        for ln in lines:
            f.write(json.dumps(ln) + "\n")
