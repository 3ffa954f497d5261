"""Randomised parity sweep: seeded random mesh shapes (1..41 cells per axis), both
rezone modes, a random perturbed state, one to three emulated slabs and random
sale_step chunkings, bit for bit against the oracle.  Varying tile raggedness,
z-chunk lengths and slab boundaries this way is also this repository's race
detector on the GPU (compute-sanitizer is closed on this pool): a shared-memory
race shows up as a bitwise mismatch on some shape."""
import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200.configs import EULER, LAGRANGE, sedov
from tests.helpers import apply_perturbation, compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", range(48))
def test_random_shapes_bitwise(case):
    from paper_2209_01983_b200.sale import Sale
    rng = np.random.Generator(np.random.PCG64(1000 + case))
    shape = tuple(int(x) for x in rng.integers(1, 42, size=3))
    rezone = (LAGRANGE, EULER)[case % 2]
    g_depth = 1 if rezone == LAGRANGE else 3  # every slab must own >= g planes
    slabs = max(1, min(int(rng.integers(1, 4)), shape[2] // g_depth))
    cfg = sedov(shape, rezone)
    g = Sale(dict(cfg, halo=(case // 2) % 2), local_slabs=slabs)  # copy / peer-store halo
    o = O.Oracle(cfg)
    apply_perturbation([g, o], cfg, int(rng.integers(0, 1000)), lagrange=(rezone == LAGRANGE))
    for n in rng.integers(1, 9, size=3):
        rg, ro = g.step(int(n)), o.step(int(n))
        assert rg == ro, (shape, rezone, slabs, rg, ro)
    compare(g, o)
    assert g.clock() == o.clock()


@pytest.mark.parametrize("case", range(24))
def test_random_shapes_materials_bitwise(case):
    """The same sweep through the material kernels: 1-4 materials, a seeded mixed state
    (inputs.material_mix), random gammas."""
    from paper_2209_01983_b200.sale import Sale
    from tests.test_gpu_materials import apply_perturbation_mm, mat_fields
    from tests.helpers import ALL_FIELDS
    rng = np.random.Generator(np.random.PCG64(5000 + case))
    shape = tuple(int(x) for x in rng.integers(1, 34, size=3))
    rezone = (LAGRANGE, EULER)[case % 2]
    g_depth = 1 if rezone == LAGRANGE else 3
    slabs = max(1, min(int(rng.integers(1, 4)), shape[2] // g_depth))
    nmat = int(rng.integers(1, 5))
    cfg = sedov(shape, rezone, nmat=nmat, mat_gamma=[float(x) for x in rng.uniform(1.1, 3.0, size=nmat)])
    g = Sale(dict(cfg, halo=(case // 2) % 2), local_slabs=slabs)  # copy / peer-store halo
    o = O.Oracle(cfg)
    apply_perturbation_mm((g, o), cfg, int(rng.integers(0, 1000)))
    for n in rng.integers(1, 9, size=3):
        rg, ro = g.step(int(n)), o.step(int(n))
        assert rg == ro, (shape, rezone, slabs, nmat, rg, ro)
    compare(g, o, ALL_FIELDS + mat_fields(nmat))
    assert g.clock() == o.clock()
