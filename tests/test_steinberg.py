"""Steinberg shear modulus / yield stress (the paper's
extension example, Fig. 6b).  CPU: the oracle's formula pinned by the
SPEC's hand-evaluated examples and by its limits.  GPU: libsale's
kernel against the oracle on evolved Sedov states of both modes (pow is not
correctly rounded on either side: agreement to a few ulp, not bitwise)."""
import numpy as np
import pytest

import oracle as O

BASE = dict(G0=1.0, GP=0.0, GT=0.0, Y0=1.0, Ymax=10.0, beta=1.0, n=2.0, cv=1.0, rho0=1.0, T0=0.0)


def P(**kw):
    return dict(BASE, **kw)


def test_shear_pins():
    # p = 0, T = T_init -> shear = G0
    sh, _ = O.steinberg_point(P(G0=3.5, GP=2.0, GT=0.7, T0=2.0), 0.0, 1.0, 2.0)
    assert sh == 3.5
    # G0=1, GP=2, GT=0, p=1, rho0/rho=8 -> 1 + 2*8^(1/3) = 5
    sh, _ = O.steinberg_point(P(GP=2.0, rho0=8.0), 1.0, 1.0, 0.0)
    assert abs(sh - 5.0) < 4e-15
    # G0=1, GP=0, GT=0.5, T - T_init = 2 -> 2, T = e / cv
    sh, _ = O.steinberg_point(P(GT=0.5, cv=2.0), 0.0, 1.0, 4.0)
    assert sh == 2.0


def test_yield_pins():
    # eps_p = 0, shear = G0 -> Y0
    assert O.steinberg_point(P(Y0=0.3), 0.0, 1.0, 0.0, 0.0)[1] == 0.3
    # Y0=1, beta=1, N=2, eps=1, Ymax=10 -> min(4, 10) = 4
    assert O.steinberg_point(P(), 0.0, 1.0, 0.0, 1.0)[1] == 4.0
    # eps = 9 -> (1+9)^2 = 100 capped at 10
    assert O.steinberg_point(P(), 0.0, 1.0, 0.0, 9.0)[1] == 10.0
    # yield scales with shear / G0
    sh, y = O.steinberg_point(P(G0=2.0, GP=1.0, rho0=1.0), 2.0, 1.0, 0.0, 0.0)
    assert sh == 4.0 and y == 1.0 * (4.0 / 2.0)


def test_oracle_field_matches_points():
    from paper_2209_01983_b200.configs import LAGRANGE, sedov
    cfg = sedov((6, 5, 4), LAGRANGE)
    o = O.Oracle(cfg)
    o.step(10)
    prm = P(GP=1.7, GT=0.3, cv=0.8, rho0=1.1, T0=0.05, Y0=0.2, Ymax=0.9, beta=3.0, n=0.5)
    eps = np.linspace(0.0, 2.0, 120).reshape(4, 5, 6)
    sh, y = o.steinberg(prm, eps)
    rho, p, e = o.get("RHO"), o.get("P"), o.get("E")
    for K in np.ndindex(rho.shape):
        assert (sh[K], y[K]) == O.steinberg_point(prm, p[K], rho[K], e[K], eps[K])


@pytest.mark.gpu
@pytest.mark.parametrize("rezone", [0, 1])
def test_gpu_steinberg_vs_oracle(rezone):
    torch = pytest.importorskip("torch")
    from paper_2209_01983_b200.configs import sedov
    from paper_2209_01983_b200.sale import Sale
    cfg = sedov((37, 11, 14), rezone)
    g, o = Sale(cfg, local_slabs=2), O.Oracle(cfg)
    assert g.step(12) == o.step(12)
    prm = P(G0=0.43, GP=1.7, GT=0.3, cv=0.8, rho0=1.1, T0=0.05, Y0=0.2, Ymax=0.9, beta=3.0, n=0.5)
    eps = np.random.Generator(np.random.PCG64(7)).uniform(0.0, 2.0, size=g.cell_shape)
    gs, gy = (t.cpu().numpy() for t in g.steinberg(prm, eps))
    os_, oy = o.steinberg(prm, eps)
    for a, b in ((gs, os_), (gy, oy)):
        rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
        assert rel.max() < 1e-14, rel.max()


MATS = [P(G0=0.43, GP=1.7, GT=0.3, cv=0.8, rho0=1.1, T0=0.05, Y0=0.2, Ymax=0.9, beta=3.0, n=0.5),
        P(G0=0.8, GP=0.9, GT=0.1, cv=1.3, rho0=0.9, T0=0.0, Y0=0.5, Ymax=1.5, beta=1.0, n=0.3),
        P(G0=0.43, GP=1.7, GT=0.3, cv=0.8, rho0=1.1, T0=0.05, Y0=0.2, Ymax=0.9, beta=3.0, n=0.5)]


def _mixed_oracle(rezone):
    from paper_2209_01983_b200 import inputs
    from paper_2209_01983_b200.configs import sedov
    cfg = sedov((6, 5, 4), rezone, nmat=3, mat_gamma=[1.4, 5.0 / 3.0, 1.2])
    o = O.Oracle(cfg)
    for f, v in inputs.material_mix(cfg, 3, o.get("MASS"), o.get("MAT_E0")).items():
        o.set(f, v)
    assert o.step(6) == (0, 6)
    return cfg, o


@pytest.mark.parametrize("rezone", [0, 1])
def test_oracle_material_steinberg(rezone):
    """Fig. 6b loops over materials: material m's shear / yield are the point formula
    with m's constants at the cell's rho, p and mixture energy (RHO / P / E); two
    materials with the same constants give the same bits."""
    cfg, o = _mixed_oracle(rezone)
    eps = np.linspace(0.0, 2.0, 120).reshape(4, 5, 6)
    sh, y = o.steinberg(MATS, eps)
    assert sh.shape == (3, 4, 5, 6)
    rho, p, e = o.get("RHO"), o.get("P"), o.get("E")
    for m in range(3):
        for K in list(np.ndindex(rho.shape))[::7]:
            assert (sh[(m,) + K], y[(m,) + K]) == O.steinberg_point(MATS[m], p[K], rho[K], e[K], eps[K])
    assert np.array_equal(sh[0], sh[2]) and np.array_equal(y[0], y[2])
    assert not np.array_equal(sh[0], sh[1])


@pytest.mark.gpu
@pytest.mark.parametrize("rezone", [0, 1])
def test_gpu_material_steinberg_vs_oracle(rezone):
    torch = pytest.importorskip("torch")
    from paper_2209_01983_b200 import inputs
    from paper_2209_01983_b200.configs import sedov
    from paper_2209_01983_b200.sale import Sale
    cfg = sedov((23, 9, 14), rezone, nmat=3, mat_gamma=[1.4, 5.0 / 3.0, 1.2])
    g, o = Sale(cfg, local_slabs=2), O.Oracle(cfg)
    for f, v in inputs.material_mix(cfg, 8, o.get("MASS"), o.get("MAT_E0")).items():
        g.set(f, v)
        o.set(f, v)
    assert g.step(9) == o.step(9)
    eps = np.random.Generator(np.random.PCG64(3)).uniform(0.0, 2.0, size=g.cell_shape)
    gs, gy = (t.cpu().numpy() for t in g.steinberg(MATS, eps))
    os_, oy = o.steinberg(MATS, eps)
    assert gs.shape == os_.shape == (3,) + g.cell_shape
    for a, b in ((gs, os_), (gy, oy)):
        rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
        assert rel.max() < 1e-14, rel.max()
