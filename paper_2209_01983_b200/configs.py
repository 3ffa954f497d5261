"""The five workloads of BASELINE.json (C0..C4) as plain parameter dicts.

Parameter values only -- no arithmetic of the method lives here.  Readings
(DESIGN.md §3): viscosity c1 = 0.25, c2 = 2.0 (Q3, SPEC S:378 fixes them, which
BASELINE.json config 0 defers to); Sedov octant with reflecting planes
x = y = z = 0 (reflect_mask 0x15) and free outer faces (Fig. 2b; SPEC
S:480-488); C4 grows lz with the GPU count so that every GPU holds 256^3 cubic
cells of side 1/256 (Q15).
"""
from __future__ import annotations

LAGRANGE, EULER = 0, 1
SEDOV_REFLECT = 0x15  # -x, -y, -z reflect; +x, +y, +z free

_SEDOV = dict(lx=1.0, ly=1.0, lz=1.0, gamma=1.4, q_lin=0.25, q_quad=2.0, cfl=0.3,
              dt_growth=1.1, t_end=0.0, reflect_mask=SEDOV_REFLECT, rho0=1.0,
              e_background=1e-10, e_deposit=1.0)


def sedov(n: tuple[int, int, int], rezone: int, **over) -> dict:
    cfg = dict(_SEDOV, nx=n[0], ny=n[1], nz=n[2], rezone=rezone)
    cfg.update(over)
    return cfg


def config(name: str, n_gpus: int = 1) -> tuple[dict, int]:
    """Return (params, cycles) for C0..C4.  cycles = -1 means 'until t_end'."""
    if name == "C0":
        return sedov((16, 16, 16), LAGRANGE), 100
    if name == "C1":
        return sedov((64, 64, 64), LAGRANGE, t_end=0.5), -1
    if name == "C2":
        return sedov((64, 64, 64), EULER), 300
    if name == "C3":
        return sedov((320, 320, 320), LAGRANGE), 200
    if name == "C4":
        return sedov((256, 256, 256 * n_gpus), EULER, lz=float(n_gpus)), 100
    raise KeyError(name)


CONFIG_NAMES = ("C0", "C1", "C2", "C3", "C4")
