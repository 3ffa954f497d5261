"""The five workloads of BASELINE.json (C0..C4) as plain parameter dicts.

Parameter values only -- no arithmetic of the method lives here.  Readings
(DESIGN.md §3): viscosity c1 = 0.25, c2 = 2.0 (Q3, SPEC S:378 fixes them, which
BASELINE.json config 0 defers to); hourglass viscosity hg = 0.5 (reading HG); Sedov octant with reflecting planes
x = y = z = 0 (reflect_mask 0x15) and free outer faces (Fig. 2b; SPEC
S:480-488); C4 grows lz with the GPU count so that every GPU holds 256^3 cubic
cells of side 1/256 (Q15).
"""
from __future__ import annotations

LAGRANGE, EULER = 0, 1
SEDOV_REFLECT = 0x15  # -x, -y, -z reflect; +x, +y, +z free

_SEDOV = dict(lx=1.0, ly=1.0, lz=1.0, gamma=1.4, q_lin=0.25, q_quad=2.0, cfl=0.3,
              dt_growth=1.1, t_end=0.0, reflect_mask=SEDOV_REFLECT, rho0=1.0,
              e_background=1e-10, e_deposit=1.0, hg=0.5)


def sedov(n: tuple[int, int, int], rezone: int, **over) -> dict:
    cfg = dict(_SEDOV, nx=n[0], ny=n[1], nz=n[2], rezone=rezone)
    cfg.update(over)
    return cfg


def config(name: str, n_gpus: int = 1) -> tuple[dict, int]:
    """Return (params, cycles) for C0..C4.  cycles = -1 means 'until t_end'.
    C0M2 / C2M2: the C0 / C2 runs with two materials (gammas 1.4 and 5/3; the initial
    layout is inputs.material_halves) -- the multi-material cells of SURVEY §8(f) NEXT-2."""
    if name in ("C0M2", "C2M2"):
        cfg, cycles = config(name[:2], n_gpus)
        return dict(cfg, nmat=2, mat_gamma=[1.4, 5.0 / 3.0]), cycles
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


# ---- further workloads on the same path -----------------
# One-dimensional problems as degenerate 3D meshes: n cubic cells along x, one
# cell across, every y/z face reflecting so the flow stays planar.  Their initial
# states are loaded through set_field (inputs.shock_tube_state / noh_state).

def shock_tube(n: int, rezone: int, **over) -> dict:
    """Sod's shock tube on [0,1]: walls at both ends,
    diaphragm at x = 0.5, gamma = 1.4, run to t = 0.2."""
    cfg = dict(_SEDOV, nx=n, ny=1, nz=1, ly=1.0 / n, lz=1.0 / n, rezone=rezone, gamma=1.4, t_end=0.2,
               reflect_mask=0x3F)
    cfg.update(over)
    return cfg


def noh_planar(n: int, **over) -> dict:
    """Planar Noh implosion on [0,1]: cold gas at u = -1
    onto a wall at x = 0, free face at x = 1, gamma = 5/3, run to t = 0.6.
    Lagrangian mode (the Eulerian remap has no inflow boundary: Q18)."""
    cfg = dict(_SEDOV, nx=n, ny=1, nz=1, ly=1.0 / n, lz=1.0 / n, rezone=LAGRANGE, gamma=5.0 / 3.0,
               t_end=0.6, reflect_mask=0x3D)
    cfg.update(over)
    return cfg


def noh_spherical(n: int, **over) -> dict:
    """Noh's spherical implosion in the octant [0,1]^3 ("spherical divergent shocks
    (Noh)"): cold gas at u = -r_hat, gamma = 5/3, reflecting planes
    x = y = z = 0, free outer faces, Lagrangian mode, run to t = 0.6 (the shock at
    r = 0.2).  The state comes from inputs.noh_spherical_state."""
    cfg = dict(_SEDOV, nx=n, ny=n, nz=n, rezone=LAGRANGE, gamma=5.0 / 3.0, t_end=0.6, e_deposit=0.0,
               e_background=0.0)
    cfg.update(over)
    return cfg


def sod_2d(n: int, rezone: int, **over) -> dict:
    """Sod's problem in 2D (Fig. 2a "2D Lagrangian Sod simulation"): n x n x 1
    cubic cells on [0,1]^2 (one cell across z), every face reflecting, gamma = 1.4, run
    to t = 0.2.  The diaphragm runs along the diagonal x + y = 1, oblique to the mesh,
    so the grid is tested off its axes (inputs.sod_oblique_state; SPEC S:526 reads the
    paper's 2D Sod as planar)."""
    cfg = dict(_SEDOV, nx=n, ny=n, nz=1, lz=1.0 / n, rezone=rezone, gamma=1.4, t_end=0.2, reflect_mask=0x3F,
               e_deposit=0.0, e_background=0.0)
    cfg.update(over)
    return cfg
