"""The further workloads of SURVEY §8(f) NEXT-3 on the oracle, pinned by exact
solutions (tests/exact.py): Sod's shock tube (Table I; SPEC
S:489-497) against the exact Riemann solution, the planar Noh implosion (
SPEC S:499-503) against its closed form.  The exact solver itself is
pinned first, by the published star state of the Sod problem and by symmetry."""
import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200 import inputs
from paper_2209_01983_b200.configs import EULER, LAGRANGE, noh_planar, shock_tube
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
