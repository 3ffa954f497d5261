"""The alternative kernel schedules kept behind environment switches (read once per
process, so each runs in a subprocess) must stay bit-identical to the oracle:
SALE_ESWEEP=1 (kf_energy_e + kr_sweep fused), SALE_REMAP=6 (pipelined kr_cells_p),
SALE_REMAP=0 (three-barrier kr_cells), SALE_FORCE_E=1 (one-kernel kf_force_e with
the remap's kn_dt pass), SALE_RNODES=0 (z-march kr_nodes), SALE_GRAPHS=0 (no CUDA-graph
replay of the cycle pairs)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import oracle as O
from paper_2209_01983_b200.configs import sedov, EULER
from paper_2209_01983_b200.sale import Sale
from tests.helpers import apply_perturbation, compare
for shape, seed in (((13, 7, 9), None), ((40, 11, 37), 1), ((1, 1, 6), None)):
    cfg = sedov(shape, EULER)
    g, o = Sale(cfg, impl="fused"), O.Oracle(cfg)
    if seed is not None:
        apply_perturbation([g, o], cfg, seed, lagrange=False)
    for chunk in (1, 7, 12):  # several sale_step calls (prologue paths) of different lengths
        rg, ro = g.step(chunk), o.step(chunk)
        assert rg == ro, (shape, rg, ro)
    compare(g, o)
    assert g.clock() == o.clock()
print("ok")
"""


@pytest.mark.parametrize("env", [{"SALE_ESWEEP": "1"}, {"SALE_REMAP": "6"}, {"SALE_REMAP": "0"},
                                 {"SALE_FORCE_E": "1"}, {"SALE_FORCE_E": "1", "SALE_RNODES": "0"},
                                 {"SALE_GRAPHS": "0"}])
def test_variant_bitwise(env):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=e, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


MAT_SCRIPT = r"""
import sys
sys.path.insert(0, %r)
import oracle as O
from paper_2209_01983_b200 import inputs
from paper_2209_01983_b200.configs import sedov, EULER, LAGRANGE
from paper_2209_01983_b200.sale import Sale
from tests.helpers import ALL_FIELDS, compare
from tests.test_gpu_materials import apply_perturbation_mm, mat_fields
for rezone in (EULER, LAGRANGE):
    for shape, nmat in (((13, 7, 9), 2), ((21, 5, 8), 3), ((1, 1, 6), 1)):
        cfg = sedov(shape, rezone, nmat=nmat, mat_gamma=[1.4, 5.0 / 3.0, 1.2][:nmat])
        g, o = Sale(cfg, impl="fused"), O.Oracle(cfg)
        apply_perturbation_mm((g, o), cfg, 6)
        for chunk in (1, 7, 12):
            rg, ro = g.step(chunk), o.step(chunk)
            assert rg == ro, (shape, rg, ro)
        compare(g, o, ALL_FIELDS + mat_fields(nmat))
        assert g.clock() == o.clock()
print("ok")
"""


@pytest.mark.parametrize("env", [{"SALE_MAT_V0": "1"}, {"SALE_GRAPHS": "0"}])
def test_material_variant_bitwise(env):
    """The material path's one-thread-per-cell Euler kernels (SALE_MAT_V0=1, the
    cross-check of the z-march kernels with the material axis), and the material path
    without CUDA-graph replay."""
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", MAT_SCRIPT % ROOT], env=e, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


SLAB_SCRIPT = r"""
import sys
sys.path.insert(0, %r)
import oracle as O
from paper_2209_01983_b200.configs import sedov, LAGRANGE
from paper_2209_01983_b200.sale import Sale
from tests.helpers import apply_perturbation, compare
for shape, slabs, seed in (((13, 7, 9), 2, 1), ((20, 9, 23), 3, 2), ((8, 8, 5), 5, 3), ((5, 6, 17), 4, None)):
    cfg = sedov(shape, LAGRANGE)
    g, o = Sale(cfg, impl="fused", local_slabs=slabs), O.Oracle(cfg)
    if seed is not None:
        apply_perturbation([g, o], cfg, seed, lagrange=True)
    for chunk in (1, 7, 12):
        rg, ro = g.step(chunk), o.step(chunk)
        assert rg == ro, (shape, rg, ro)
    compare(g, o)
    assert g.clock() == o.clock()
print("ok")
"""


@pytest.mark.parametrize("env", [{"SALE_OVERLAP": "1"}, {"SALE_OVERLAP": "1", "SALE_GRAPHS": "0"}, {}])
def test_lagrange_slabs_overlap_bitwise(env):
    """Lagrange with emulated slabs: boundary planes first and the halo exchange on a
    side stream overlapping the interior (SALE_OVERLAP=1, with and without graph replay),
    and the default single-stream cycle; thin slabs (< 2g+2 planes) take the whole-slab
    path."""
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", SLAB_SCRIPT % ROOT], env=e, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
