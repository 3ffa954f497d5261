"""Pins of the oracle's multi-material cells (the Data4d material
axis, per-material EoS, mixed-cell closure, per-material remap; P:133, P:183, P:403;
SPEC S:195-288; readings MM1-MM7 in DESIGN.md §10d).

What pins the material path to something other than itself:
* the SPEC's worked closure examples and exact algebraic special cases;
* reduction: one material reproduces the single-material scheme bit for bit, and two
  identical materials splitting every cell reproduce it to round-off;
* conservation: per-material mass (bitwise in Lagrange mode, round-off in Euler mode),
  total energy in Lagrange mode with two different gammas in every cell (compatible
  per-material work sums to the cell's work);
* pressure equilibrium: a contact between two gases at equal pressure and velocity is
  advected by the remap without disturbing p or u, mixed cells included;
* the two-gamma Riemann problem solved exactly (tests/exact.py, itself pinned by the
  conservation of its own solution), first-order convergence of the contact position.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200 import inputs
from paper_2209_01983_b200.configs import EULER, LAGRANGE, sedov, shock_tube
from tests import exact


def mm(cfg, gammas, **over):
    c = dict(cfg, nmat=len(gammas), mat_gamma=list(gammas))
    c.update(over)
    return c


# ------------------------------------------------------------ the exact solver
def test_two_gamma_riemann_solution_conserves():
    """The exact solution with gamma_L != gamma_R conserves mass, momentum and energy
    over [0, 1] (ends undisturbed, so momentum grows by (p_L - p_R) t); gamma_L = gamma_R
    gives the one-gas solver's star state."""
    WL, WR, g, t = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1), (1.4, 5.0 / 3.0), 0.2
    ps, us = exact.star_state(WL, WR, g)
    xc = 0.5 + us * t
    n = 400000
    x = (np.arange(n) + 0.5) / n
    r, u, p = exact.exact_riemann(x, t, WL, WR, g)
    gam = np.where(x < xc, g[0], g[1])
    M = np.mean(r)
    P = np.mean(r * u)
    E = np.mean(p / (gam - 1.0) + 0.5 * r * u * u)
    assert abs(M - 0.5 * (WL[0] + WR[0])) < 1e-5
    assert abs(P - (WL[2] - WR[2]) * t) < 1e-5
    assert abs(E - 0.5 * (WL[2] / (g[0] - 1.0) + WR[2] / (g[1] - 1.0))) < 1e-5
    assert exact.star_state(WL, WR, (1.4, 1.4)) == exact.star_state(WL, WR, 1.4)


# ------------------------------------------------------------ MM1 closure
def test_mix_eos_spec_examples():
    g = 1.4
    # f = (1, 0): identical to the pure-material EoS, bit for bit
    for rho_in, e in ((1.0, 2.5), (0.125, 2.0), (3.7, 0.01), (0.5, -1.0)):
        V = 0.3
        m = rho_in * V
        rho = m / V
        assert O.mix_eos([g, 1.7], [1.0, 0.0], [m, 0.0], [e, 5.0], V, rho) == O.eos(g, rho, e)
    # two identical materials at f = (0.5, 0.5) with the same (rho, e): the pure cell
    V, rho_in, e = 0.8, 1.3, 2.1
    m = rho_in * V
    rho = m / V
    p, pf, cs = O.eos(g, rho, e)
    assert O.mix_eos([g, g], [0.5, 0.5], [0.5 * m, 0.5 * m], [e, e], V, rho) == (p, pf, cs)
    # f = (0.25, 0.75), p_0 = 4, p_1 = 0 -> p = 1; c^2 = 0.25 gamma_0 p_0 / rho
    p, P, cs = O.mix_eos([1.5, 1.4], [0.25, 0.75], [0.25, 0.75], [8.0, 0.0], 1.0, 1.0)
    assert (p, P) == (1.0, 1.0) and cs == math.sqrt(1.5)
    # a negative material pressure counts in p, is floored in P and c
    p, P, cs = O.mix_eos([1.5, 1.5], [0.5, 0.5], [0.5, 0.5], [8.0, -4.0], 1.0, 1.0)
    assert (p, P) == (1.0, 2.0) and cs == math.sqrt(3.0)
    # an absent material (f = 0, m = 0) contributes nothing (no 0/0)
    assert O.mix_eos([1.5, 2.0, 1.2], [0.5, 0.0, 0.5], [1.0, 0.0, 1.0], [2.0, 0.0, 2.0], 2.0, 1.0) == \
        O.mix_eos([1.5, 1.2], [0.5, 0.5], [1.0, 1.0], [2.0, 2.0], 2.0, 1.0)


def test_material_parameter_and_field_checks():
    cfg = sedov((3, 3, 3), EULER)
    for bad in (mm(cfg, [1.4] * 5), mm(cfg, [1.4, 1.0]), mm(cfg, [1.4], nmat=-1)):
        with pytest.raises(ValueError):
            O.Oracle(bad)
    o = O.Oracle(mm(cfg, [1.4, 1.6]))
    assert np.array_equal(o.get("MAT_F0"), np.ones(o.cell_shape))  # MM7: Sedov = material 0
    assert np.array_equal(o.get("MAT_M0"), o.get("MASS"))
    assert not o.get("MAT_F1").any() and not o.get("MAT_M1").any()
    for f in ("MASS", "E"):
        with pytest.raises(ValueError):
            o.set(f, np.ones(o.cell_shape))
    with pytest.raises(ValueError):
        o.get("MAT_F2")
    o.set("MAT_M1", np.full(o.cell_shape, 0.5))
    assert np.array_equal(o.get("MASS"), o.get("MAT_M0") + 0.5)  # the cell mass is the sum


# ------------------------------------------------------------ reductions
def perturbed_pair(cfg, gammas_split, seed, lagrange):
    """(single-material oracle, material oracle) on the same perturbed Sedov state;
    gammas_split: list of (gamma, fraction) -- every cell split in those fractions."""
    a = O.Oracle(cfg)
    b = O.Oracle(mm(cfg, [g for g, _ in gammas_split]))
    pert = inputs.perturbation(cfg, seed)
    if lagrange:
        for f, d in (("X", "dx"), ("Y", "dy"), ("Z", "dz")):
            v = a.get(f) + pert[d]
            a.set(f, v)
            b.set(f, v)
    for f in ("UX", "UY", "UZ"):
        a.set(f, pert[f.lower()])
        b.set(f, pert[f.lower()])
    e = a.get("E") * pert["e_factor"]
    a.set("E", e)
    m = a.get("MASS")
    for k, (_, frac) in enumerate(gammas_split):
        b.set(f"MAT_F{k}", np.full(a.cell_shape, frac))
        b.set(f"MAT_M{k}", frac * m if len(gammas_split) > 1 else m)
        b.set(f"MAT_E{k}", e)
    return a, b


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_one_material_reduces_bitwise(rezone):
    """a single-material configuration takes the material path and the
    scalar path to the same bits (every state and derived field, the clock)."""
    cfg = sedov((6, 5, 7), rezone)
    a, b = perturbed_pair(cfg, [(cfg["gamma"], 1.0)], seed=3, lagrange=rezone == LAGRANGE)
    for _ in range(3):
        assert a.step(5) == (0, 5) and b.step(5) == (0, 5)
        for f in ("X", "Y", "Z", "UX", "UY", "UZ", "NODE_MASS", "MASS", "RHO", "VOL", "P", "Q", "CS"):
            assert np.array_equal(a.get(f), b.get(f)), f
        assert np.array_equal(a.get("E"), b.get("MAT_E0"))
        assert np.array_equal(b.get("MAT_F0"), np.ones(a.cell_shape))
        assert np.array_equal(b.get("MAT_M0"), a.get("MASS"))
        assert a.clock() == b.clock()


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_identical_materials_split_matches_single(rezone):
    """Two copies of the same gas sharing every cell (f = 1/4, 3/4) evolve as one gas:
    each material keeps the cell's density and energy, the mixture matches the scalar
    scheme to round-off."""
    cfg = sedov((6, 6, 5), rezone)
    g = cfg["gamma"]
    a, b = perturbed_pair(cfg, [(g, 0.25), (g, 0.75)], seed=5, lagrange=rezone == LAGRANGE)
    assert a.step(12) == (0, 12) and b.step(12) == (0, 12)
    rel = lambda x, y: float(np.max(np.abs(x - y)) / np.max(np.abs(y)))
    for f in ("UX", "UY", "UZ", "MASS", "P", "CS", "Q"):
        assert rel(b.get(f), a.get(f)) < 1e-11, f
    for k in (0, 1):
        assert rel(b.get(f"MAT_E{k}"), a.get("E")) < 1e-11
    assert rel(b.get("MAT_F0"), np.full(a.cell_shape, 0.25)) < 1e-12
    assert rel(b.get("MAT_M0"), 0.25 * a.get("MASS")) < 1e-11


# ------------------------------------------------------------ conservation
def test_lagrange_two_gamma_energy_conservation():
    """Lagrange mode, all faces free, two gases (gamma 1.4 / 1.8) in every cell with
    fractions from {1/8, ..., 7/8} (sums exactly 1): material masses never change and
    internal + kinetic energy is conserved to round-off (MM4 is compatible: the
    materials' work sum_m f_m sigma_m W dt is the cell's sigma W dt)."""
    cfg = sedov((5, 6, 4), LAGRANGE, reflect_mask=0, e_background=1.0, e_deposit=3.0)
    o = O.Oracle(mm(cfg, [1.4, 1.8]))
    pert = inputs.perturbation(cfg, 7, u_scale=0.05)
    for a, f in (("dx", "X"), ("dy", "Y"), ("dz", "Z")):
        o.set(f, o.get(f) + pert[a])
    for f in ("UX", "UY", "UZ"):
        o.set(f, pert[f.lower()])
    rng = np.random.Generator(np.random.PCG64(11))
    f0 = rng.integers(1, 8, size=o.cell_shape) / 8.0
    m = o.get("MASS")
    o.set("MAT_F0", f0)
    o.set("MAT_F1", 1.0 - f0)
    o.set("MAT_M0", m * f0 * 0.7)
    o.set("MAT_M1", m * (1.0 - f0) * 1.3)
    o.set("MAT_E0", rng.uniform(0.5, 2.0, size=o.cell_shape))
    o.set("MAT_E1", rng.uniform(0.5, 2.0, size=o.cell_shape))

    def total_energy():
        ie = math.fsum((o.get("MAT_M0") * o.get("MAT_E0")).ravel()) + \
            math.fsum((o.get("MAT_M1") * o.get("MAT_E1")).ravel())
        M = o.get("NODE_MASS")
        ke = math.fsum((0.5 * M * ((o.get("UX") ** 2 + o.get("UY") ** 2) + o.get("UZ") ** 2)).ravel())
        return ie, ke

    m0, m1 = o.get("MAT_M0"), o.get("MAT_M1")
    ie0, ke0 = total_energy()
    assert o.step(25) == (0, 25)
    ie, ke = total_energy()
    assert ke > ke0 * 1.5  # the gas expanded and moved
    assert abs((ie + ke) - (ie0 + ke0)) <= 1e-13 * (ie0 + ke0)
    assert np.array_equal(o.get("MAT_M0"), m0) and np.array_equal(o.get("MAT_M1"), m1)
    assert np.array_equal(o.get("MAT_F0"), f0)


def test_euler_contact_in_pressure_equilibrium_advects_cleanly():
    """Two gases (same gamma, densities 1 and 0.25, equal pressure 1) move at u = 0.5
    through the fixed mesh: in every interior cell, mixed ones included, p stays 1 and u
    stays 0.5 to round-off, each material keeps its density, and material 1 enters
    cells that held only material 0."""
    n = 64
    cfg = mm(shock_tube(n, EULER, reflect_mask=0x3C), [1.4, 1.4])
    o = O.Oracle(cfg)
    st = inputs.two_material_tube_state(cfg, o.get("MASS"), x0=0.5, left=(0.25, 1.0), right=(1.0, 1.0))
    for f, v in st.items():
        o.set(f, v)
    o.set("UX", np.full(o.node_shape, 0.5))
    cycles = 8
    assert o.step(cycles) == (0, cycles)
    inner = slice(3 * cycles, n - 3 * cycles)
    p = o.get("P")[0, 0, inner]
    ux = o.get("UX")[0, 0, inner]
    assert np.max(np.abs(p - 1.0)) < 1e-12
    assert np.max(np.abs(ux - 0.5)) < 1e-12
    f0 = o.get("MAT_F0")[0, 0, inner]
    assert np.count_nonzero((f0 > 1e-9) & (f0 < 1.0 - 1e-9)) >= 1  # a mixed cell exists
    V = o.get("VOL")[0, 0, inner]
    for k, rho_k in ((0, 0.25), (1, 1.0)):
        fk, mk = o.get(f"MAT_F{k}")[0, 0, inner], o.get(f"MAT_M{k}")[0, 0, inner]
        present = fk > 1e-9
        assert np.max(np.abs(mk[present] / (fk[present] * V[present]) - rho_k)) < 1e-12


# ------------------------------------------------------------ two-gamma Sod
def run_two_material_sod(n, rezone):
    cfg = shock_tube(n, rezone, nmat=2, mat_gamma=[1.4, 5.0 / 3.0])
    o = O.Oracle(cfg)
    for f, v in inputs.two_material_tube_state(cfg, o.get("MASS")).items():
        o.set(f, v)
    masses = [math.fsum(o.get(f"MAT_M{k}").ravel()) for k in (0, 1)]
    rc, _ = o.step(10 ** 6)
    assert rc == 0 and o.clock()["t"] == cfg["t_end"]
    return cfg, o, masses


@pytest.mark.parametrize("rezone,tol", [(LAGRANGE, 0.0035), (EULER, 0.011)])
def test_two_material_sod_against_exact(rezone, tol):
    n = 200
    cfg, o, masses = run_two_material_sod(n, rezone)
    X = o.get("X")[0, 0, :] if rezone == LAGRANGE else np.linspace(0.0, 1.0, n + 1)
    xc, dx = 0.5 * (X[:-1] + X[1:]), np.diff(X)
    g = (1.4, 5.0 / 3.0)
    ex = exact.exact_riemann(xc, cfg["t_end"], g=g)
    l1 = lambda a, b: float(np.sum(np.abs(a - b) * dx))
    assert l1(o.get("RHO")[0, 0], ex[0]) < tol and l1(o.get("P")[0, 0], ex[2]) < tol
    for k in (0, 1):  # per-material mass: bitwise in Lagrange mode, round-off in Euler mode
        assert math.fsum(o.get(f"MAT_M{k}").ravel()) == pytest.approx(masses[k], rel=1e-14, abs=0)
    # material 0's volume is the gas left of the contact x_c = 0.5 + u* t
    ps, us = exact.star_state((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), g)
    vol0 = float(np.sum(o.get("MAT_F0") * o.get("VOL"))) * n * n
    xc_exact = 0.5 + us * cfg["t_end"]
    assert abs(vol0 - xc_exact) < (1e-4 if rezone == LAGRANGE else 1.0 / n)


def test_two_material_contact_converges_first_order():
    errs = []
    for n in (100, 200, 400):
        cfg, o, _ = run_two_material_sod(n, EULER)
        _, us = exact.star_state((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), (1.4, 5.0 / 3.0))
        vol0 = float(np.sum(o.get("MAT_F0") * o.get("VOL"))) * n * n
        errs.append(abs(vol0 - (0.5 + us * cfg["t_end"])))
    assert errs[1] < 0.6 * errs[0] and errs[2] < 0.6 * errs[1]
