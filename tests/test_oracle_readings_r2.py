"""Pins of the oracle parts added in round 2 (DESIGN.md §3 readings HG, DT-Q, DT-C)
and of the dt growth cap (c.5), against things other than the
oracle itself: SPEC's printed example, closed forms that follow from the algebra of
the hourglass base vectors (orthogonality to affine fields, |Gamma_m|^2 = 8), the
exact one-cycle decay of an hourglass mode on a single free box, energy
conservation, and the growth-cap inequality on the Sedov trajectory.

A mutation of any of these parts -- the cap dropped, a Gamma sign or index wrong, the
hourglass work missing from the energy, the cap on nu dropped, the viscous speed
with the wrong sign -- fails at least one test below (checked when written).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200.configs import LAGRANGE, config, sedov

# hex corner h = (c*2+b)*2+a; xi = 2a-1, eta = 2b-1, zeta = 2c-1 (DESIGN.md §3 HG)
CORNERS = [(h & 1, (h >> 1) & 1, h >> 2) for h in range(8)]


def gamma(m, h):
    a, b, c = CORNERS[h]
    xi, eta, zeta = 2 * a - 1, 2 * b - 1, 2 * c - 1
    return [xi * eta, eta * zeta, zeta * xi, xi * eta * zeta][m]


# ------------------------------------------------------------ c.5 growth cap
def test_growth_cap_spec_example():
    """dt_prev = 1e-3 and an unconstrained candidate of order 1 give
    dt = 1.1e-3 (the cap); with no previous dt (cycle 0, Q10) no cap applies."""
    cfg = sedov((2, 2, 2), LAGRANGE, e_deposit=0.0, e_background=1e-12)
    o = O.Oracle(cfg)
    rc, dt0 = o.next_dt()
    assert rc == 0 and dt0 > 1.0           # c ~ 1e-6: the CFL candidate is huge
    o.set_clock(0.0, 1e-3, 1)
    rc, dt = o.next_dt()
    assert rc == 0 and dt == pytest.approx(1.1e-3, rel=1e-15)


def test_growth_cap_binds_on_the_sedov_trajectory():
    """C0 cycle by cycle: dt_n <= 1.1 dt_{n-1} always, with equality in the cycles
    where the CFL candidate grows faster (the hot cell expanding)."""
    cfg, _ = config("C0")
    o = O.Oracle(cfg)
    prev, binds = None, 0
    for _ in range(100):
        assert o.step(1) == (0, 1)
        dt = o.clock()["dt_last"]
        if prev is not None:
            assert dt <= 1.1 * prev
            binds += dt == 1.1 * prev
        prev = dt
    assert binds >= 1


# ------------------------------------------------------- DT-C collapse rule
def test_collapse_without_end_time():
    """DT-C: with t_end <= 0, dt_u < 1e-14 * t is a collapse (the t_end rule of S:318
    scaled by the time reached); at t = 0 only !(dt_u > 0) is."""
    cfg = sedov((4, 4, 4), LAGRANGE)
    o = O.Oracle(cfg)
    assert o.next_dt()[0] == 0
    rc, dt = o.next_dt()
    o.set_clock(2e-14 * 1e14 * dt * 0.99, -1.0, 0)   # dt just above 1e-14 t
    assert o.next_dt()[0] == 0
    o.set_clock(dt / 1e-14 * 1.01, -1.0, 0)          # dt just below 1e-14 t
    assert o.next_dt()[0] == O.EDTCOLLAPSE


# ------------------------------------------------------- DT-Q signal speed
def test_viscous_signal_speed_reduces_to_spec_without_compression():
    """DT-Q adds the viscous speed only for a compressing cell: du >= 0 reproduces
    S:320's 0.0025 bit for bit; compression only shortens the candidate, and the
    more so the stronger it is (a monotone added speed)."""
    base = O.dt_cell(0.25, 1e-4, 0.0, 1.0, 0.0)
    assert base == pytest.approx(0.0025, rel=1e-15)
    assert O.dt_cell(0.25, 1e-4, 0.0, 1.0, 0.7) == base
    d = [O.dt_cell(0.25, 1e-4, 0.0, 1.0, -x) for x in (1e-9, 1e-3, 0.1, 1.0, 10.0)]
    assert all(a > b for a, b in zip([base] + d, d))


# ------------------------------------------------------ HG hourglass modes
def test_hourglass_modes_vanish_on_affine_fields():
    """The four base vectors are orthogonal to 1, xi, eta, zeta, so any affine
    velocity field on a parallelepiped has zero hourglass amplitudes (dyadic inputs:
    exact)."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        Amap = rng.integers(-8, 9, (3, 3)) / 8.0 + np.eye(3)
        x0 = rng.integers(-8, 9, 3) / 4.0
        N = np.array([x0 + Amap @ np.array(CORNERS[h], float) for h in range(8)])
        G = rng.integers(-8, 9, (3, 3)) / 8.0
        a = rng.integers(-8, 9, 3) / 8.0
        U = np.array([a + G @ N[h] for h in range(8)])
        assert np.array_equal(O.hg_modes(U), np.zeros((4, 3)))


@pytest.mark.parametrize("m", range(4))
def test_hourglass_modes_of_pure_patterns(m):
    """u_h = Gamma_m(h) v: g_m = 8 v (|Gamma_m|^2 = 8) and the other three modes 0."""
    v = np.array([0.375, -1.25, 2.0])
    U = np.array([gamma(m, h) * v for h in range(8)])
    g = O.hg_modes(U)
    for k in range(4):
        assert np.array_equal(g[k], 8 * v if k == m else np.zeros(3))


def test_hourglass_corner_forces_conserve_momentum_and_dissipate():
    """sum_h f_h = 0 (each Gamma sums to zero: no net force, momentum conserved) and
    sum_h f_h . u_h = -nu sum_m |g_m|^2 <= 0 (orthogonality: a pure damping)."""
    rng = np.random.default_rng(9)
    for _ in range(10):
        U = rng.normal(size=(8, 3))
        g = O.hg_modes(U)
        nu = rng.uniform(0.1, 3.0)
        f = np.array([O.hg_corner(g, nu, h) for h in range(8)])
        assert np.max(np.abs(f.sum(axis=0))) <= 1e-13 * np.abs(f).max()
        P = float(np.sum(f * U))
        assert P == pytest.approx(-nu * float(np.sum(g * g)), rel=1e-12)
        assert P <= 0.0


def test_cell_energy_hourglass_heat_closed_form():
    """Reading HG in the compatible energy (the per-cell entry point): on the unit cube
    with a pure xi*eta*zeta mode u_h = Gamma_3(h) v (u' = u, dyadic values, so every
    operation is exact), the pressure work W = sum_h C_h . ubar_h is 0 (C_h = (xi, eta,
    zeta), orthogonal to the mode), g_3 = 8 v, f_h = -8 nu Gamma_3(h) v, and the
    hourglass work W_hg = sum_h f_h . ubar_h = -64 nu |v|^2: the cell heats by
    64 nu |v|^2 dt / m.  (scripts/oracle_mutations.py found the entry point's W_hg
    otherwise unpinned.)"""
    N0 = np.array([[float(a), float(b), float(c)] for (a, b, c) in CORNERS])
    v = np.array([0.25, -0.5, 0.75])
    U = np.array([gamma(3, h) * v for h in range(8)])
    nu, sigma, m, e, dt = 0.375, 0.7, 2.0, 1.0, 0.125
    e1 = O.cell_energy(N0, U, U, sigma, m, e, dt, nu=nu)
    assert e1 == e + 64.0 * nu * float(v @ v) * dt / m == 2.3125
    assert O.cell_energy(N0, U, U, sigma, m, e, dt, nu=0.0) == e  # no damping: W = 0, no heat


def _box_cycle(hg, eps=1e-3, dims=(2.0, 1.0, 0.5), e0=2.5, gam=1.4):
    """One free box cell with pressure and an xi*eta*zeta hourglass mode of amplitude
    eps in u_z: returns (g3_z before, after, nu, dt, m, energies before/after)."""
    cfg = sedov((1, 1, 1), LAGRANGE, reflect_mask=0, lx=dims[0], ly=dims[1], lz=dims[2],
                e_deposit=e0 * dims[0] * dims[1] * dims[2], e_background=e0, gamma=gam, hg=hg)
    o = O.Oracle(cfg)
    o.set("E", np.full(o.cell_shape, e0))
    uz = np.zeros(o.node_shape)
    for h, (a, b, c) in enumerate(CORNERS):
        uz[c, b, a] = eps * gamma(3, h)
    o.set("UZ", uz)

    def g3(o):
        U = np.zeros((8, 3))
        for h, (a, b, c) in enumerate(CORNERS):
            U[h] = [o.get(f)[c, b, a] for f in ("UX", "UY", "UZ")]
        return O.hg_modes(U)[3][2]

    def energy(o):
        M = o.get("NODE_MASS")
        ke = math.fsum((0.5 * M * (o.get("UX") ** 2 + o.get("UY") ** 2 + o.get("UZ") ** 2)).ravel())
        return math.fsum((o.get("MASS") * o.get("E")).ravel()) + ke

    m = float(o.get("MASS")[0, 0, 0])
    b3, E0 = g3(o), energy(o)
    assert o.step(1) == (0, 1)
    dt = o.clock()["dt_last"]
    rho = m / (dims[0] * dims[1] * dims[2])
    c = math.sqrt(gam * ((gam - 1.0) * rho * e0) / rho)
    # c.5 on the box: shortest edge min(dims), speed eps, no compression at t^n
    assert dt == pytest.approx(0.3 * min(dims) / (c + eps), rel=1e-14)
    lbar = sum(dims) / 3.0      # the face-centroid separations are the box sides
    nu = min(hg * m * c / lbar, m / 64.0 / dt)
    return b3, g3(o), nu, dt, m, E0, energy(o)


@pytest.mark.parametrize("hg", [0.0, 0.05, 0.1])
def test_single_box_hourglass_decay_closed_form(hg):
    """One cycle on a free box: the pressure forces have no xi*eta*zeta component, so
    the mode's amplitude scales by exactly 1 - 64 nu dt / m (node mass m/8, |Gamma|^2 =
    8), nu = hg m c / lbar below the cap; total energy is conserved (the damped kinetic
    energy heats the cell)."""
    b3, a3, nu, dt, m, E0, E1 = _box_cycle(hg)
    assert b3 == pytest.approx(8e-3, rel=1e-15)
    assert nu < m / 64.0 / dt                      # the cap does not bind here
    assert a3 == pytest.approx(b3 * (1.0 - 64.0 * nu * dt / m), rel=1e-10, abs=1e-15)
    assert abs(E1 - E0) <= 1e-14 * E0


def test_single_box_hourglass_cap_kills_the_mode():
    """With the cap binding, nu = (m/64)/dt removes the whole mode in one cycle."""
    b3, a3, nu, dt, m, E0, E1 = _box_cycle(1e3)
    assert nu == pytest.approx(m / 64.0 / dt, rel=1e-15)
    assert abs(a3) <= 1e-10 * abs(b3)
    assert abs(E1 - E0) <= 1e-14 * E0


@pytest.mark.parametrize("rezone,hg", [(LAGRANGE, 0.5), (LAGRANGE, 3.0)])
def test_energy_and_momentum_with_hourglass_on_perturbed_state(rezone, hg):
    """Compatible hourglass work: Lagrange IE + KE conserved to round-off over 20
    cycles of a perturbed free state; momentum of a free body conserved."""
    from tests.helpers import apply_perturbation
    cfg = sedov((9, 8, 7), rezone, reflect_mask=0 if rezone == LAGRANGE else 0x3F, e_background=0.5, hg=hg)
    o = O.Oracle(cfg)
    apply_perturbation([o], cfg, 4, lagrange=(rezone == LAGRANGE), u_scale=0.05)

    def totals(o):
        M = o.get("NODE_MASS")
        ke = math.fsum((0.5 * M * (o.get("UX") ** 2 + o.get("UY") ** 2 + o.get("UZ") ** 2)).ravel())
        mom = [math.fsum((M * o.get(f)).ravel()) for f in ("UX", "UY", "UZ")]
        return math.fsum((o.get("MASS") * o.get("E")).ravel()) + ke, mom, math.fsum((M * 0.05).ravel())

    E0, P0, scale = totals(o)
    assert o.step(20) == (0, 20)
    E1, P1, _ = totals(o)
    assert abs(E1 - E0) <= 1e-12 * E0
    for a, b in zip(P0, P1):
        assert abs(a - b) <= 1e-12 * scale
