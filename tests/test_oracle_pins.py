"""Pins of the oracle's primitives against things other than the oracle itself:
values SPEC.md prints for worked examples (cited S:n), closed forms, and
independent brute-force computations (Gauss quadrature of the trilinear map).

The paper (arXiv 2209.01983) prints no discrete formula for the scheme
(SURVEY §0), so the pins are the SPEC examples and mathematics; the oracle
follows SURVEY §8(c).
"""
import math

import numpy as np
import pytest

import oracle as O


# ---------------------------------------------------------------- EoS (c.3 s1)
def test_eos_spec_pressure_examples():
    # gamma=1.4, rho=1, e=2.5 -> p = 1.0 ; rho=0.125, e=2.0 -> p = 0.1
    p, pf, _ = O.eos(1.4, 1.0, 2.5)
    assert p == pytest.approx(1.0, rel=1e-15) and pf == p
    p, _, _ = O.eos(1.4, 0.125, 2.0)
    assert p == pytest.approx(0.1, rel=1e-15)
    # S:216 trivial: e = 0 -> p = 0, c = 0
    assert O.eos(1.4, 1.0, 0.0) == (0.0, 0.0, 0.0)


def test_eos_spec_sound_speed_examples():
    # gamma=1.4, rho=1, p=1 -> c = sqrt(1.4); gamma=5/3, rho=1, p=5/3 -> c = 5/3
    _, _, c = O.eos(1.4, 1.0, 2.5)
    assert c == pytest.approx(math.sqrt(1.4), rel=1e-15)
    g = 5.0 / 3.0
    _, _, c = O.eos(g, 1.0, 2.5)  # p = (2/3)*2.5 = 5/3
    assert c == pytest.approx(5.0 / 3.0, rel=1e-15)


def test_eos_pressure_floor_reading_q8():
    # Q8 / S:272: p stays negative, the floored pf and c use max(p, 0)
    p, pf, c = O.eos(1.4, 2.0, -1.0)
    assert p < 0 and pf == 0.0 and c == 0.0


# --------------------------------------------------------------- q (c.3 s2)
def test_q_spec_example():
    # rho=1, c=1, du=-0.1, c_q=2, c_l=0.25 -> q = 2*0.01 + 0.25*0.1 = 0.045
    assert O.q_of_du(1.0, 1.0, -0.1, 0.25, 2.0) == pytest.approx(0.045, rel=1e-14)


def test_q_zero_in_expansion_and_uniform_flow():
    # expansion and uniform flow give q = 0 exactly
    assert O.q_of_du(1.0, 1.0, 0.3, 0.25, 2.0) == 0.0
    assert O.q_of_du(1.0, 1.0, 0.0, 0.25, 2.0) == 0.0


# ---------------------------------------------------------------- dt (c.5)
def test_dt_spec_example():
    # u=0, c=1, dx=0.01, cfl=0.25 -> dt = 0.0025
    assert O.dt_cell(0.25, 0.01 * 0.01, 0.0, 1.0) == pytest.approx(0.0025, rel=1e-15)


def test_dt_max_speed_adds_to_sound_speed():
    # c.5 / S:315: signal speed c + |u|
    assert O.dt_cell(0.5, 4.0, 9.0, 1.0) == pytest.approx(0.5 * 2.0 / (1.0 + 3.0), rel=1e-15)


# ---------------------------------------------------------- geometry (c.2)
def _unit_cube_nodes(scale=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    N = np.zeros((8, 3))
    for c in range(2):
        for b in range(2):
            for a in range(2):
                N[(c * 2 + b) * 2 + a] = [origin[0] + a * scale[0], origin[1] + b * scale[1],
                                          origin[2] + c * scale[2]]
    return N


def test_face_orientation_unit_cube():
    # c.2: the canonical face orderings give +axis unit normals on the unit cube
    X = [[0, 0, 0], [0, 1, 0], [0, 1, 1], [0, 0, 1]]
    Y = [[0, 0, 0], [0, 0, 1], [1, 0, 1], [1, 0, 0]]
    Z = [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]]
    for P, n in ((X, [1, 0, 0]), (Y, [0, 1, 0]), (Z, [0, 0, 1])):
        A, Xb, s = O.face(P)
        assert np.array_equal(A, np.array(n, float))
        assert s == float(np.dot(Xb, A))


def _gauss_volume(N):
    """Independent brute force: integral of det J of the trilinear map over
    [0,1]^3 with 3-point Gauss-Legendre per axis (exact: det J has degree <= 2
    in each variable)."""
    g, w = np.polynomial.legendre.leggauss(3)
    g = 0.5 * (g + 1.0)
    w = 0.5 * w
    X = N.reshape(2, 2, 2, 3)  # [c][b][a]
    vol = 0.0
    for xi, wx in zip(g, w):
        for eta, wy in zip(g, w):
            for zeta, wz in zip(g, w):
                lx = np.array([1 - xi, xi]); ly = np.array([1 - eta, eta]); lz = np.array([1 - zeta, zeta])
                dlx = np.array([-1.0, 1.0])
                dxi = np.einsum("c,b,a,cbaq->q", lz, ly, dlx, X)
                deta = np.einsum("c,b,a,cbaq->q", lz, dlx, lx, X)
                dzeta = np.einsum("c,b,a,cbaq->q", dlx, ly, lx, X)
                vol += wx * wy * wz * np.linalg.det(np.stack([dxi, deta, dzeta]))
    return vol


def test_hex_volume_unit_and_box():
    assert O.hex_volume(_unit_cube_nodes()) == 1.0
    assert O.hex_volume(_unit_cube_nodes((0.5, 0.25, 2.0), (3, -1, 7))) == pytest.approx(0.25, rel=1e-15)


@pytest.mark.parametrize("seed", range(8))
def test_hex_volume_equals_trilinear_gauss_volume(seed):
    # SURVEY c.2: the face formula is the exact volume of the trilinear hex
    rng = np.random.default_rng(seed)
    N = _unit_cube_nodes() + rng.uniform(-0.3, 0.3, size=(8, 3))
    assert O.hex_volume(N) == pytest.approx(_gauss_volume(N), rel=1e-13, abs=1e-14)


def test_hex_volume_affine_map():
    rng = np.random.default_rng(11)
    A = np.eye(3) + rng.uniform(-0.3, 0.3, (3, 3))
    N = _unit_cube_nodes() @ A.T + rng.uniform(-2, 2, 3)
    assert O.hex_volume(N) == pytest.approx(np.linalg.det(A), rel=1e-13)


# --------------------------------------------------------- remap (c.4 s1)
def test_swept_volume_translation_closed_form():
    # a flat unit face moved by d along its normal sweeps A.d; zero motion sweeps 0 exactly
    PT = np.array([[0, 0, 0], [0, 1, 0], [0, 1, 1], [0, 0, 1]], float)   # X-face, A = (1,0,0)
    assert O.swept_volume(PT, PT) == 0.0
    d = np.array([0.01, 0.3, -0.2])
    assert O.swept_volume(PT, PT + d) == pytest.approx(0.01, rel=1e-13)
    assert O.swept_volume(PT, PT - d) == pytest.approx(-0.01, rel=1e-13)


@pytest.mark.parametrize("seed", range(6))
def test_swept_volume_identity(seed):
    # SURVEY c.4 s1: V_L - sum(signed dV) = V_T for any node motion
    rng = np.random.default_rng(100 + seed)
    NT = _unit_cube_nodes() + rng.uniform(-0.2, 0.2, (8, 3))
    NL = NT + rng.uniform(-0.1, 0.1, (8, 3))
    faces = {"X0": [0, 2, 6, 4], "X1": [1, 3, 7, 5], "Y0": [0, 4, 5, 1], "Y1": [2, 6, 7, 3],
             "Z0": [0, 1, 3, 2], "Z1": [4, 5, 7, 6]}
    dV = {k: O.swept_volume(NT[v], NL[v]) for k, v in faces.items()}
    VT, VL = O.hex_volume(NT), O.hex_volume(NL)
    # a +face moving outward enlarges the Lagrangian cell, a -face moving +a shrinks it
    recon = VL - dV["X1"] + dV["X0"] - dV["Y1"] + dV["Y0"] - dV["Z1"] + dV["Z0"]
    assert recon == pytest.approx(VT, abs=1e-14)


# ------------------------------------------------------ energy (c.3 s7)
def test_energy_spec_uniaxial_compression():
    # single cell compressed 1% at p+q = 1, m = 1, V0 = 1 -> de = +0.01
    N0 = _unit_cube_nodes()
    dt = 0.5
    U = np.zeros((8, 3))
    U[[1, 3, 5, 7], 0] = -0.01 / dt       # +x face moves in by 0.01
    e1 = O.cell_energy(N0, U, U, 0.25 * 1.0, 1.0, 3.0, dt)   # sigma = (p+q)/4
    assert e1 - 3.0 == pytest.approx(0.01, rel=1e-12)


def test_energy_no_motion_unchanged_bitwise():
    # no vertex motion -> e unchanged bitwise
    N0 = _unit_cube_nodes()
    Z = np.zeros((8, 3))
    assert O.cell_energy(N0, Z, Z, 0.7, 1.3, 2.25, 0.1) == 2.25
