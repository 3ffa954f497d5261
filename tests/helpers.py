"""Shared test helpers: running the CUDA path and the oracle on the same seeded
inputs and comparing them (bitwise target; BASELINE north_star bar: <= 1e-9
relative with reading Q19's denominator)."""
from __future__ import annotations

import numpy as np

from paper_2209_01983_b200 import inputs

STATE_FIELDS_L = ("X", "Y", "Z", "UX", "UY", "UZ", "MASS", "E")
STATE_FIELDS_E = ("UX", "UY", "UZ", "MASS", "E")
DERIVED = ("NODE_MASS", "RHO", "VOL", "P", "Q", "CS")
ALL_FIELDS = ("X", "Y", "Z", "UX", "UY", "UZ", "NODE_MASS", "MASS", "E", "RHO", "VOL", "P", "Q", "CS")


def rel_err(g: np.ndarray, o: np.ndarray) -> float:
    """Q19: |g-o| / max(|o|, 1e-12 * max|o|)."""
    scale = np.maximum(np.abs(o), 1e-12 * max(np.abs(o).max(), 1e-300))
    return float(np.max(np.abs(g - o) / scale)) if o.size else 0.0


def compare(gpu, orc, fields=ALL_FIELDS, bitwise=True, tol=1e-9):
    report = {}
    for f in fields:
        g, o = gpu.get(f), orc.get(f)
        assert g.shape == o.shape, (f, g.shape, o.shape)
        mism = int(np.count_nonzero(g.view(np.int64) != o.view(np.int64)))
        err = rel_err(g, o)
        report[f] = (mism, err)
    bad = {f: r for f, r in report.items() if (r[0] if bitwise else r[1] > tol)}
    assert not bad, f"mismatches (count, max rel err): {bad}"
    return report


def apply_perturbation(ctxs, cfg, seed, lagrange=True, **kw):
    """Load seeded input P<seed> into every context in ctxs."""
    pert = inputs.perturbation(cfg, seed, **kw)
    base = ctxs[0]
    if lagrange:
        xs = {f: base.get(f) + pert[d] for f, d in (("X", "dx"), ("Y", "dy"), ("Z", "dz"))}
    us = {f: pert[f.lower()] for f in ("UX", "UY", "UZ")}
    e = base.get("E") * pert["e_factor"]
    for c in ctxs:
        if lagrange:
            for f, v in xs.items():
                c.set(f, v)
        for f, v in us.items():
            c.set(f, v)
        c.set("E", e)
