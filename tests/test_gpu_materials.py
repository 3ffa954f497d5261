"""GPU parity of the multi-material cells (readings MM0-MM7,
DESIGN.md §10d): the material kernels (kernels_mat.cu) against the oracle's material
path, bit for bit, on seeded mixed states (inputs.material_mix: random fractions,
material densities and energies, a third of the cells pure) in both rezone modes, with
one to four materials, emulated slabs, several sale_step chunks; one material against
the single-material kernels; the two-gas shock tube; the argument checks."""
import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200 import inputs
from paper_2209_01983_b200.configs import EULER, LAGRANGE, sedov, shock_tube
from tests.helpers import ALL_FIELDS, apply_perturbation, compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GAMMAS = [1.4, 5.0 / 3.0, 1.2, 2.0]


def mat_fields(n):
    return tuple(f"MAT_{q}{k}" for k in range(n) for q in "FME")


def _pair(cfg, seed, local_slabs=1):
    from paper_2209_01983_b200.sale import Sale
    g, o = Sale(cfg, local_slabs=local_slabs), O.Oracle(cfg)
    apply_perturbation_mm((g, o), cfg, seed)
    return g, o


def apply_perturbation_mm(ctxs, cfg, seed):
    """P<seed> positions / velocities and a seeded material mix."""
    lag = cfg["rezone"] == LAGRANGE
    pert = inputs.perturbation(cfg, seed)
    base = ctxs[1]  # the oracle supplies the read-back geometry and Sedov state
    if lag:
        xs = {f: base.get(f) + pert[d] for f, d in (("X", "dx"), ("Y", "dy"), ("Z", "dz"))}
    mix = inputs.material_mix(cfg, seed, base.get("MASS"), base.get("MAT_E0") * pert["e_factor"])
    for c in ctxs:
        if lag:
            for f, v in xs.items():
                c.set(f, v)
        for f in ("UX", "UY", "UZ"):
            c.set(f, pert[f.lower()])
        for f, v in mix.items():
            c.set(f, v)


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
@pytest.mark.parametrize("nmat", [1, 2, 3, 4])
def test_materials_bitwise(rezone, nmat):
    cfg = sedov((13, 9, 11), rezone, nmat=nmat, mat_gamma=GAMMAS[:nmat])
    g, o = _pair(cfg, seed=nmat)
    compare(g, o, ALL_FIELDS + mat_fields(nmat))
    for n in (1, 4, 7):
        assert g.step(n) == o.step(n) == (0, n)
        compare(g, o, ALL_FIELDS + mat_fields(nmat))
    assert g.clock() == o.clock()


@pytest.mark.parametrize("rezone,slabs", [(LAGRANGE, 3), (EULER, 2), (EULER, 3)])
def test_materials_slabs_bitwise(rezone, slabs):
    cfg = sedov((10, 7, 12), rezone, nmat=2, mat_gamma=GAMMAS[:2])
    g, o = _pair(cfg, seed=9, local_slabs=slabs)
    for n in (3, 6):
        assert g.step(n) == o.step(n) == (0, n)
    compare(g, o, ALL_FIELDS + mat_fields(2))


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_one_material_equals_single_material_kernels(rezone):
    """nmat = 1 through the material kernels == nmat = 0 through the fused kernels."""
    from paper_2209_01983_b200.sale import Sale
    cfg = sedov((12, 10, 9), rezone)
    a = Sale(cfg)
    b = Sale(dict(cfg, nmat=1, mat_gamma=[cfg["gamma"]]))
    o = O.Oracle(cfg)
    apply_perturbation([o, a], cfg, seed=4, lagrange=rezone == LAGRANGE)
    for f in ("X", "Y", "Z") if rezone == LAGRANGE else ():
        b.set(f, o.get(f))
    for f in ("UX", "UY", "UZ"):
        b.set(f, o.get(f))
    b.set("MAT_E0", o.get("E"))
    assert a.step(9) == b.step(9) == (0, 9)
    for f in ("X", "Y", "Z", "UX", "UY", "UZ", "MASS", "RHO", "P", "CS", "Q"):
        assert np.array_equal(a.get(f), b.get(f)), f
    assert np.array_equal(a.get("E"), b.get("MAT_E0"))


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_two_gas_shock_tube_bitwise(rezone):
    from paper_2209_01983_b200.sale import Sale
    cfg = shock_tube(150, rezone, nmat=2, mat_gamma=[1.4, 5.0 / 3.0])
    g, o = Sale(cfg), O.Oracle(cfg)
    for f, v in inputs.two_material_tube_state(cfg, o.get("MASS")).items():
        g.set(f, v)
        o.set(f, v)
    for n in (3, 50, 10 ** 6):
        assert g.step(n) == o.step(n)
    assert g.clock() == o.clock() and g.clock()["finished"] == 1
    compare(g, o, ALL_FIELDS + mat_fields(2))


def test_material_argument_checks():
    from paper_2209_01983_b200.sale import Sale, SaleError, workspace_bytes
    cfg = sedov((6, 6, 6), EULER)
    assert workspace_bytes(dict(cfg, nmat=5, mat_gamma=[1.4] * 4)) == 0
    assert workspace_bytes(dict(cfg, nmat=2, mat_gamma=[1.4, 1.0])) == 0
    assert workspace_bytes(dict(cfg, nmat=2, mat_gamma=[1.4, 1.5])) > workspace_bytes(cfg)
    g = Sale(dict(cfg, nmat=2, mat_gamma=[1.4, 1.5]))
    for f in ("MASS", "E"):
        with pytest.raises(SaleError):
            g.set(f, np.ones(g.cell_shape))
    with pytest.raises(SaleError):
        g.get("MAT_F2")
    with pytest.raises(ValueError):  # one Steinberg parameter set per material
        g.steinberg(dict(G0=1.0, GP=0.0, GT=0.0, Y0=1.0, Ymax=2.0, beta=0.0, n=1.0, cv=1.0, rho0=1.0, T0=0.0))
    g.set("MAT_M1", np.full(g.cell_shape, 0.25))
    assert np.array_equal(g.get("MASS"), g.get("MAT_M0") + 0.25)


@pytest.mark.parametrize("name", ["C4", "C3"])
def test_full_size_material_properties(name):
    """At the benchmark sizes (the launch configuration materials_bench times): one
    material through the material kernels equals the single-material kernels bit for
    bit, and two copies of the gas splitting every cell (1/4, 3/4) conserve each
    material's mass and track the single gas to round-off."""
    from paper_2209_01983_b200.configs import config
    from paper_2209_01983_b200.sale import Sale
    cfg, _ = config(name)
    cycles = 6
    a = Sale(cfg)
    assert a.step(cycles) == (0, cycles)
    ref = {f: a.get(f) for f in ("UX", "MASS", "E", "P")}
    a.close()
    del a
    torch.cuda.empty_cache()
    b = Sale(dict(cfg, nmat=1, mat_gamma=[cfg["gamma"]]))
    assert b.step(cycles) == (0, cycles)
    for f in ("UX", "MASS", "P"):
        assert np.array_equal(b.get(f), ref[f]), f
    assert np.array_equal(b.get("MAT_E0"), ref["E"])
    b.close()
    del b
    torch.cuda.empty_cache()
    c = Sale(dict(cfg, nmat=2, mat_gamma=[cfg["gamma"]] * 2))
    m, e = c.get("MAT_M0"), c.get("MAT_E0")
    c.set("MAT_F0", np.full(c.cell_shape, 0.25))
    c.set("MAT_F1", np.full(c.cell_shape, 0.75))
    c.set("MAT_M0", 0.25 * m)
    c.set("MAT_M1", 0.75 * m)
    c.set("MAT_E1", e)
    m0 = [float(np.sum(c.get(f"MAT_M{k}"), dtype=np.float64)) for k in (0, 1)]
    assert c.step(cycles) == (0, cycles)
    for k in (0, 1):
        assert abs(float(np.sum(c.get(f"MAT_M{k}"), dtype=np.float64)) - m0[k]) <= 1e-12 * m0[k]
    ux = c.get("UX")
    assert np.max(np.abs(ux - ref["UX"])) <= 1e-10 * max(np.max(np.abs(ref["UX"])), 1e-300)
    assert np.max(np.abs(c.get("MASS") - ref["MASS"])) <= 1e-12 * np.max(ref["MASS"])


def test_material_error_paths_same_cycle_and_cell():
    """The material path reports the oracle's status, cycle and cell: a tangled cell in
    Lagrange mode, and ENEGMASS in Euler mode when a CFL number above 1 lets the faces
    sweep more than a cell's volume out of it."""
    from paper_2209_01983_b200.sale import Sale
    cfg = sedov((4, 4, 4), LAGRANGE, nmat=2, mat_gamma=[1.4, 1.6])
    g, o = Sale(cfg), O.Oracle(cfg)
    X = o.get("X")
    X[2, 2, 2] += 2.0
    for c in (g, o):
        c.set("X", X)
    assert g.step(3) == o.step(3) == (O.ETANGLED, 0)
    assert o.last_error().split()[-1] in g.last_error()
    # a uniform translation at CFL 1.5 sweeps 1.5 cell volumes through every face
    # (no deformation, so no tangle); alternating densities leave cells with m'' < 0
    cfg = sedov((7, 6, 5), EULER, nmat=2, mat_gamma=[1.4, 1.6], cfl=1.5, reflect_mask=0, e_deposit=0.0,
                e_background=1e-6)
    g, o = Sale(cfg), O.Oracle(cfg)
    m = o.get("MAT_M0") * np.where((np.arange(7) % 2) == 0, 1.0, 0.05)[None, None, :]
    for c in (g, o):
        c.set("UX", np.ones(o.node_shape))
        c.set("MAT_M0", m)
    rg, ro = g.step(20), o.step(20)
    assert rg == ro == (O.ENEGMASS, 0), (rg, ro)
    assert o.last_error().split()[-1] in g.last_error()
    assert g.clock() == o.clock()
