"""The cycle without CUDA-graph replay (SALE_GRAPHS=0, read once per process, so each
case runs in a subprocess) must stay bit-identical to the oracle, as the default
(graph-replayed) schedule does: single material (Euler), the material axis (both
modes), emulated Lagrange slabs (the ghost cell-state pass inside the graphs)."""
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
    g, o = Sale(cfg), O.Oracle(cfg)
    if seed is not None:
        apply_perturbation([g, o], cfg, seed, lagrange=False)
    for chunk in (1, 7, 12):  # several sale_step calls (prologue paths) of different lengths
        rg, ro = g.step(chunk), o.step(chunk)
        assert rg == ro, (shape, rg, ro)
    compare(g, o)
    assert g.clock() == o.clock()
print("ok")
"""


@pytest.mark.parametrize("env", [{"SALE_GRAPHS": "0"}, {}])
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
        g, o = Sale(cfg), O.Oracle(cfg)
        apply_perturbation_mm((g, o), cfg, 6)
        for chunk in (1, 7, 12):
            rg, ro = g.step(chunk), o.step(chunk)
            assert rg == ro, (shape, rg, ro)
        compare(g, o, ALL_FIELDS + mat_fields(nmat))
        assert g.clock() == o.clock()
print("ok")
"""


@pytest.mark.parametrize("env", [{"SALE_GRAPHS": "0"}])
def test_material_variant_bitwise(env):
    """The material path without CUDA-graph replay."""
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
    g, o = Sale(cfg, local_slabs=slabs), O.Oracle(cfg)
    if seed is not None:
        apply_perturbation([g, o], cfg, seed, lagrange=True)
    for chunk in (1, 7, 12):
        rg, ro = g.step(chunk), o.step(chunk)
        assert rg == ro, (shape, rg, ro)
    compare(g, o)
    assert g.clock() == o.clock()
print("ok")
"""


@pytest.mark.parametrize("env", [{"SALE_GRAPHS": "0"}, {}])
def test_lagrange_slabs_bitwise(env):
    """Lagrange with emulated slabs (the ghost cell-state pass after each exchange), with
    and without graph replay; slabs of one plane included."""
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", SLAB_SCRIPT % ROOT], env=e, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
