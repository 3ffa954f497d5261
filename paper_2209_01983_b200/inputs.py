"""Seeded synthetic input generators shared by the tests of the oracle and of
the CUDA path (inputs P0-P2).

This module holds NONE of the method's arithmetic: it only draws random
numbers (numpy ``Generator(PCG64(seed))``) and masks.  The caller adds the
returned jitter to node coordinates it read back through ``get_field`` and
multiplies the energy factor into ``e``, then loads the same bits into both the
oracle and the GPU context with ``set_field``.

Recipe: interior node coordinates jittered by U(-0.05h, 0.05h)
per axis (boundary nodes are left on their planes); node velocity
U(-1e-3, 1e-3) per component, with the normal component zeroed on reflecting
planes; specific energy multiplied by U(0.5, 1.5).
"""
from __future__ import annotations

import numpy as np


def perturbation(cfg: dict, seed: int, u_scale: float = 1e-3, x_frac: float = 0.05,
                 e_lo: float = 0.5, e_hi: float = 1.5):
    """Return dict(dx, dy, dz, ux, uy, uz [node arrays (nz+1, ny+1, nx+1)],
    e_factor [cell array (nz, ny, nx)])."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    hs = (cfg["lx"] / nx, cfg["ly"] / ny, cfg["lz"] / nz)
    rng = np.random.Generator(np.random.PCG64(seed))
    nshape = (nz + 1, ny + 1, nx + 1)
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1),
                          indexing="ij")
    interior = (i > 0) & (i < nx) & (j > 0) & (j < ny) & (k > 0) & (k < nz)
    out = {}
    for name, h in zip(("dx", "dy", "dz"), hs):
        d = rng.uniform(-x_frac * h, x_frac * h, size=nshape)
        out[name] = np.where(interior, d, 0.0)
    mask = int(cfg["reflect_mask"])
    planes = (((i == 0), (i == nx)), ((j == 0), (j == ny)), ((k == 0), (k == nz)))
    for ax, name in enumerate(("ux", "uy", "uz")):
        u = rng.uniform(-u_scale, u_scale, size=nshape)
        lo, hi = planes[ax]
        zero = np.zeros(nshape, dtype=bool)
        if mask & (1 << (2 * ax)):
            zero |= lo
        if mask & (1 << (2 * ax + 1)):
            zero |= hi
        out[name] = np.where(zero, 0.0, u)
    out["e_factor"] = rng.uniform(e_lo, e_hi, size=(nz, ny, nx))
    return out


def uniform_velocity(cfg: dict, u: tuple[float, float, float]):
    """Constant node velocity arrays (no randomness)."""
    nshape = (cfg["nz"] + 1, cfg["ny"] + 1, cfg["nx"] + 1)
    return {n: np.full(nshape, float(v)) for n, v in zip(("ux", "uy", "uz"), u)}


# ---- initial states of the further workloads (configs.shock_tube / noh_planar) ----
# Problem data, not method arithmetic: the caller passes the MASS a fresh context
# holds (the Sedov init with rho0 = 1 sets m = V, the cell volume), and loads the
# returned fields into the oracle and the GPU context alike with set_field.

def shock_tube_state(cfg: dict, volume: np.ndarray, x0: float = 0.5, left=(1.0, 1.0), right=(0.125, 0.1)):
    """Sod: (rho, p) = (1, 1) for cell centres x < x0, (0.125, 0.1) beyond, at rest.
    volume: the cells' V (cell array).  Returns {"MASS", "E"}; specific energy
    e = p / ((gamma - 1) rho)."""
    nx = cfg["nx"]
    xc = (np.arange(nx) + 0.5) * (cfg["lx"] / nx)
    lft = (xc < x0)[None, None, :]
    rho = np.where(lft, left[0], right[0])
    p = np.where(lft, left[1], right[1])
    g = cfg["gamma"]
    return {"MASS": rho * volume, "E": np.broadcast_to(p / ((g - 1.0) * rho), volume.shape).copy()}


def noh_state(cfg: dict, u0: float = -1.0, p0: float = 1e-6):
    """Planar Noh: rho = 1 (the Sedov init's m with rho0 = 1), u_x = u0
    on every node except the wall plane x = 0 (reflecting, u_x = 0), and a pressure
    floor p0 = 1e-6 of the dynamic pressure rho u0^2, i.e. e = p0 / ((gamma-1) rho).
    Returns {"UX", "E"}."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    ux = np.full((nz + 1, ny + 1, nx + 1), u0)
    ux[:, :, 0] = 0.0
    e = p0 * u0 * u0 / (cfg["gamma"] - 1.0)
    return {"UX": ux, "E": np.full((nz, ny, nx), e)}


def two_material_tube_state(cfg: dict, volume: np.ndarray, x0: float = 0.5, left=(1.0, 1.0),
                            right=(0.125, 0.1)):
    """Sod's tube with two materials: material 0 (gamma
    cfg["mat_gamma"][0]) fills the cells with centre x < x0 at (rho, p) = left, material
    1 (mat_gamma[1]) the others at right; every cell is pure (f = 1 or 0).  volume: the
    cells' V.  Returns the material fields {"MAT_F0", "MAT_M0", "MAT_E0", "MAT_F1", ...};
    e_m = p / ((gamma_m - 1) rho)."""
    nx = cfg["nx"]
    xc = (np.arange(nx) + 0.5) * (cfg["lx"] / nx)
    lft = np.broadcast_to((xc < x0)[None, None, :], volume.shape)
    out = {}
    for m, (side, (rho, p)) in enumerate(((lft, left), (~lft, right))):
        g = cfg["mat_gamma"][m]
        out[f"MAT_F{m}"] = np.where(side, 1.0, 0.0)
        out[f"MAT_M{m}"] = np.where(side, rho * volume, 0.0)
        out[f"MAT_E{m}"] = np.where(side, p / ((g - 1.0) * rho), 0.0)
    return out


def material_mix(cfg: dict, seed: int, mass: np.ndarray, energy: np.ndarray, pure_frac: float = 0.3):
    """Seeded mixed cells for nmat = cfg["nmat"] materials: in a
    random pure_frac of the cells material 0 alone (f = 1, the others absent); elsewhere
    fractions w_k / sum w (w ~ U(0.1, 1)), masses f_k * mass * U(0.5, 2), energies
    energy * U(0.5, 1.5).  Returns {"MAT_F<k>", "MAT_M<k>", "MAT_E<k>"} (cell arrays)."""
    n = int(cfg["nmat"])
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = mass.shape
    w = rng.uniform(0.1, 1.0, size=(n,) + shape)
    pure = rng.uniform(size=shape) < pure_frac
    out = {}
    for k in range(n):
        f = w[k] / w.sum(axis=0)
        f = np.where(pure, 1.0 if k == 0 else 0.0, f)
        out[f"MAT_F{k}"] = f
        out[f"MAT_M{k}"] = f * mass * rng.uniform(0.5, 2.0, size=shape)
        out[f"MAT_E{k}"] = np.where(f > 0, energy * rng.uniform(0.5, 1.5, size=shape), 0.0)
    return out


def material_halves(cfg: dict, mass: np.ndarray, energy: np.ndarray, x0: float = 0.125):
    """The C0M2 / C2M2 layout (configs.config): cells whose centre lies at x > x0 (the
    blast crosses that plane within the run) hold
    material 1 (same mass and specific energy as the Sedov state there), the others
    material 0; every cell pure.  Returns the MAT_* fields."""
    nx = cfg["nx"]
    xc = (np.arange(nx) + 0.5) * (cfg["lx"] / nx)
    right = np.broadcast_to((xc > x0)[None, None, :], mass.shape)
    return {"MAT_F0": np.where(right, 0.0, 1.0), "MAT_M0": np.where(right, 0.0, mass),
            "MAT_E0": np.where(right, 0.0, energy), "MAT_F1": np.where(right, 1.0, 0.0),
            "MAT_M1": np.where(right, mass, 0.0), "MAT_E1": np.where(right, energy, 0.0)}


def noh_spherical_state(cfg: dict, X: np.ndarray, Y: np.ndarray, Z: np.ndarray, u0: float = -1.0,
                        p0: float = 1e-6):
    """Spherical Noh: node velocity u0 * (x, y, z) / r (zero at the origin) from the node
    coordinates the context holds, and the pressure floor p0 of planar Noh (e = p0 u0^2 /
    (gamma - 1) at rho = 1).  Returns {"UX", "UY", "UZ", "E"}."""
    r = np.sqrt(X * X + Y * Y + Z * Z)
    rs = np.where(r > 0.0, r, 1.0)
    out = {f: np.where(r > 0.0, u0 * (A / rs), 0.0) for f, A in (("UX", X), ("UY", Y), ("UZ", Z))}
    out["E"] = np.full((cfg["nz"], cfg["ny"], cfg["nx"]), p0 * u0 * u0 / (cfg["gamma"] - 1.0))
    return out


def sod_oblique_state(cfg: dict, volume: np.ndarray, left=(1.0, 1.0), right=(0.125, 0.1)):
    """2D Sod with the diaphragm along x + y = 1: (rho, p) = left for cell centres with
    x + y < 1, right beyond, at rest.  volume: the cells' V.  Returns {"MASS", "E"}."""
    nx, ny = cfg["nx"], cfg["ny"]
    xc = (np.arange(nx) + 0.5) * (cfg["lx"] / nx)
    yc = (np.arange(ny) + 0.5) * (cfg["ly"] / ny)
    lft = (yc[:, None] + xc[None, :] < 1.0)[None, :, :]
    rho = np.where(lft, left[0], right[0])
    p = np.where(lft, left[1], right[1])
    g = cfg["gamma"]
    return {"MASS": rho * volume, "E": np.broadcast_to(p / ((g - 1.0) * rho), volume.shape).copy()}
