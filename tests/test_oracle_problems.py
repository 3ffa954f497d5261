"""The further workloads of SURVEY §8(f) NEXT-3 on the oracle, pinned by exact
solutions (tests/exact.py): Sod's shock tube (Table I; SPEC
S:489-497) against the exact Riemann solution, the planar Noh implosion (
SPEC S:499-503) against its closed form.  The exact solver itself is
pinned first, by the published star state of the Sod problem and by symmetry."""
import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200 import inputs
from paper_2209_01983_b200.configs import EULER, LAGRANGE, noh_planar, noh_spherical, shock_tube, sod_2d
from tests import exact


def test_exact_riemann_pins():
    # Sod, gamma = 1.4: p* = 0.30313, u* = 0.92745 (Toro, Table 4.3, test 1)
    ps, us = exact.star_state((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), 1.4)
    assert abs(ps - 0.30313) < 5e-5 and abs(us - 0.92745) < 5e-5
    # equal states: no waves
    W = exact.exact_riemann(np.linspace(0, 1, 11), 0.1, (0.7, 0.2, 0.9), (0.7, 0.2, 0.9), 1.4)
    assert np.allclose(W, np.array([[0.7], [0.2], [0.9]]))
    # mirror-symmetric colliding flows: u* = 0
    ps2, us2 = exact.star_state((1.0, 1.0, 1.0), (1.0, -1.0, 1.0), 1.4)
    assert abs(us2) < 1e-12 and ps2 > 1.0
    # the two strong shocks of the 123-like expansion are rarefactions: p* < both
    ps3, _ = exact.star_state((1.0, -2.0, 0.4), (1.0, 2.0, 0.4), 1.4)
    assert ps3 < 0.4


def test_exact_noh_pins():
    xs, rho2, p2, e2 = exact.noh_planar(0.6, 5.0 / 3.0)
    assert abs(xs - 0.2) < 1e-15 and abs(rho2 - 4.0) < 1e-15 and abs(p2 - 4.0 / 3.0) < 1e-15
    # Rankine-Hugoniot across the shock (frame of the wall): mass, momentum, energy
    D, u0, g = 1.0 / 3.0, -1.0, 5.0 / 3.0
    assert abs(1.0 * (D - u0) - rho2 * D) < 1e-14
    assert abs(p2 - 1.0 * (D - u0) * (0.0 - u0)) < 1e-14
    assert abs(p2 / ((g - 1.0) * rho2) - e2) < 1e-14


def run_oracle_problem(cfg, state):
    o = O.Oracle(cfg)
    vol = o.get("MASS")  # rho0 = 1: m = V
    for f, v in state(cfg, vol).items():
        o.set(f, v)
    rc, done = o.step(10 ** 6)
    assert rc == 0 and o.clock()["finished"] == 1 and o.clock()["t"] == cfg["t_end"]
    return o


def centres(o, cfg):
    if cfg["rezone"] == LAGRANGE:
        X = o.get("X")[0, 0, :]
    else:
        X = np.linspace(0.0, cfg["lx"], cfg["nx"] + 1)
    return 0.5 * (X[:-1] + X[1:]), np.diff(X)


def sod_errors(n, rezone):
    cfg = shock_tube(n, rezone)
    o = run_oracle_problem(cfg, lambda c, v: inputs.shock_tube_state(c, v))
    xc, dx = centres(o, cfg)
    ex = exact.exact_riemann(xc, cfg["t_end"])
    rho, p = o.get("RHO")[0, 0], o.get("P")[0, 0]
    l1 = lambda a, b: float(np.sum(np.abs(a - b) * dx))
    plateau = (xc > 0.55) & (xc < 0.65)  # between the contact (0.685) and the rarefaction tail
    return l1(rho, ex[0]), l1(p, ex[2]), float(np.median(p[plateau])), o


@pytest.mark.parametrize("rezone,tol", [(LAGRANGE, 0.004), (EULER, 0.011)])
def test_sod_against_exact(rezone, tol):
    e_rho, e_p, p_star, o = sod_errors(200, rezone)
    assert e_rho < tol and e_p < tol
    assert abs(p_star - 0.30313) < 3e-3
    # mass conserved to round-off (walls at both ends)
    m = o.get("MASS")
    assert abs(np.sum(m) - (0.5 * 1.0 + 0.5 * 0.125) / 200 ** 2) < 1e-15


def test_sod_first_order_convergence():
    e100 = sod_errors(100, LAGRANGE)[0]
    e200 = sod_errors(200, LAGRANGE)[0]
    e400 = sod_errors(400, LAGRANGE)[0]
    # L1 error of a first-order shock-capturing scheme halves with h (discontinuities)
    assert e200 < 0.7 * e100 and e400 < 0.7 * e200


def test_noh_planar_against_exact():
    cfg = noh_planar(200)
    o = run_oracle_problem(cfg, lambda c, v: inputs.noh_state(c))
    xc, _ = centres(o, cfg)
    xs, rho2, p2, _ = exact.noh_planar(cfg["t_end"], cfg["gamma"])
    rho, p = o.get("RHO")[0, 0], o.get("P")[0, 0]
    inner = (xc > 0.03) & (xc < xs - 0.03)  # away from the wall-heating cells and the shock
    assert abs(np.median(rho[inner]) - rho2) < 0.01 * rho2
    assert abs(np.median(p[inner]) - p2) < 0.01 * p2
    ahead = (xc > xs + 0.03) & (np.arange(len(xc)) < len(xc) - 4)  # the free face's p0 rarefies its last cells
    assert np.max(np.abs(rho[ahead] - 1.0)) < 1e-6
    # shock position: the last cell compressed past half the jump
    shock = xc[np.nonzero(rho > 0.5 * (1.0 + rho2))[0].max()]
    assert abs(shock - xs) < 3.0 / 200


# ---------------------------------------------------------------- spherical Noh
def test_exact_noh_spherical_pins():
    """Rankine-Hugoniot across the spherical shock (frame of the centre, gamma = 5/3):
    the gas arriving from ahead (rho = (1 + t/r_s)^2 = 16 at r_s = t/3) fills the
    shocked sphere (rho2 = 64) behind a shock moving out at D = 1/3: mass, momentum,
    energy."""
    g, t = 5.0 / 3.0, 0.6
    rs, rho = exact.noh_spherical(np.array([0.0, 0.1, 0.2 + 1e-12]), t, g)
    assert abs(rs - 0.2) < 1e-15 and rho[0] == rho[1] == 64.0
    ra = (1.0 + t / rs) ** 2
    assert abs(ra - 16.0) < 1e-12 and abs(rho[2] - ra) < 1e-9
    D, u0 = 1.0 / 3.0, 1.0
    p2, e2 = (g - 1.0) * 64.0 * 0.5, 0.5
    assert abs(ra * (D + u0) - 64.0 * D) < 1e-12                  # mass
    assert abs(p2 - ra * (D + u0) * u0) < 1e-12                    # momentum (upstream cold)
    # energy, [rho (u - D)(e + u^2/2) + p u] = 0: ahead u = -1, e = p = 0; behind u = 0
    assert abs(ra * (-u0 - D) * (0.5 * u0 * u0) - 64.0 * (0.0 - D) * e2) < 1e-12


def _noh_spherical_run(n):
    cfg = noh_spherical(n)
    o = O.Oracle(cfg)
    for f, v in inputs.noh_spherical_state(cfg, o.get("X"), o.get("Y"), o.get("Z")).items():
        o.set(f, v)
    E0 = _total_energy(o)
    rc, _ = o.step(10 ** 6)
    assert rc == 0 and o.clock()["t"] == cfg["t_end"] and o.clock()["finished"] == 1
    return cfg, o, E0


def _total_energy(o):
    import math
    u2 = o.get("UX") ** 2 + o.get("UY") ** 2 + o.get("UZ") ** 2
    return math.fsum((o.get("MASS") * o.get("E")).ravel()) + math.fsum((0.5 * o.get("NODE_MASS") * u2).ravel())


def _cell_radius(o):
    def cc(A):
        return 0.125 * (A[:-1, :-1, :-1] + A[1:, :-1, :-1] + A[:-1, 1:, :-1] + A[1:, 1:, :-1]
                        + A[:-1, :-1, 1:] + A[1:, :-1, 1:] + A[:-1, 1:, 1:] + A[1:, 1:, 1:])
    return np.sqrt(cc(o.get("X")) ** 2 + cc(o.get("Y")) ** 2 + cc(o.get("Z")) ** 2)


def test_noh_spherical_against_exact():
    """Spherical Noh in the octant at 24^3 to t = 0.6: total energy conserved
    and the octant symmetry kept to round-off (the compatible Lagrangian scheme with
    HG); the cold gas ahead of the shock compressed by convergence as (1 + t/r)^2
    within 12% where it came from inside the unit sphere (r + t < 1); the shocked
    sphere's peak density within 20% of 64 and its shell mean (0.1 < r < 0.2) above
    0.4 x 64 -- at this resolution the plateau is not reached (wall heating at the
    centre, smearing at the shock: DESIGN.md §10; SPEC S:514 calls 3D Noh no
    acceptance target)."""
    cfg, o, E0 = _noh_spherical_run(24)
    assert abs(_total_energy(o) - E0) <= 1e-12 * E0
    e = o.get("E")
    for perm in ((0, 2, 1), (2, 1, 0), (1, 0, 2)):
        assert np.max(np.abs(e - e.transpose(perm))) <= 1e-10 * np.abs(e).max()
    rho, r = o.get("RHO"), _cell_radius(o)
    rs, ex = exact.noh_spherical(r, cfg["t_end"], cfg["gamma"])
    ahead = (r > 0.32) & (r < 0.40)
    assert abs(rho[ahead].mean() / ex[ahead].mean() - 1.0) < 0.12
    assert abs(rho.max() / 64.0 - 1.0) < 0.20
    shell = (r > 0.1) & (r < 0.2)
    assert rho[shell].mean() > 0.4 * 64.0


# ----------------------------------------------------------------- 2D Sod
@pytest.mark.parametrize("rezone,tol", [(LAGRANGE, 0.025), (EULER, 0.03)])
def test_sod_2d_oblique_against_exact(rezone, tol):
    """2D Sod (Fig. 2a) on 64 x 64 x 1 with the diaphragm along x + y = 1,
    oblique to the mesh: along the diagonal i = j, normal to the diaphragm, the density
    is the exact 1D Riemann solution in xi = (x + y - 1)/sqrt(2) (the walls' disturbances
    have not reached |xi| < 0.4 by t = 0.2): mean |error| within tol; the problem's
    mirror symmetry x <-> y kept to round-off; mass conserved."""
    cfg = sod_2d(64, rezone)
    o = run_oracle_problem(cfg, lambda c, v: inputs.sod_oblique_state(c, v))
    rho = o.get("RHO")[0]
    n = cfg["nx"]
    if rezone == LAGRANGE:
        def cx(A):
            return 0.25 * (A[0, :-1, :-1] + A[0, 1:, :-1] + A[0, :-1, 1:] + A[0, 1:, 1:])
        Xc, Yc = cx(o.get("X")), cx(o.get("Y"))
    else:
        xc = (np.arange(n) + 0.5) / n
        Xc, Yc = np.meshgrid(xc, xc, indexing="xy")
    d = np.arange(n)
    xi = (Xc[d, d] + Yc[d, d] - 1.0) / np.sqrt(2.0)
    ex = exact.exact_riemann(xi + 0.5, cfg["t_end"])[0]
    sel = np.abs(xi) < 0.4
    assert np.mean(np.abs(rho[d, d][sel] - ex[sel])) < tol
    assert np.max(np.abs(rho - rho.T)) <= 1e-9 * rho.max()
    m = o.get("MASS")
    m0 = O.Oracle(cfg)
    st = inputs.sod_oblique_state(cfg, m0.get("MASS"))
    assert abs(np.sum(m) - np.sum(st["MASS"])) <= 1e-13 * np.sum(st["MASS"])
