"""GPU parity: libsale (through its C ABI) vs the CPU oracle on the same seeded
inputs, element by element.  Target bitwise (both sides are correctly rounded
fp64 in the SURVEY §8(c) order); the hard bar is BASELINE's 1e-9 relative and
bit-exact dt-selection cycle counts."""
import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200.configs import EULER, LAGRANGE, config, sedov
from tests.helpers import ALL_FIELDS, apply_perturbation, compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

def _sale(cfg, **kw):
    from paper_2209_01983_b200.sale import Sale
    return Sale(cfg, **kw)


def run_pair(cfg, cycles, **kw):
    g = _sale(cfg, **kw)
    o = O.Oracle(cfg)
    rg, dg = g.step(cycles)
    ro, do = o.step(cycles)
    return g, o, (rg, dg), (ro, do)


def test_C0_full_bitwise():
    cfg, cycles = config("C0")
    g, o, rg, ro = run_pair(cfg, cycles)
    assert rg == ro == (0, cycles)
    compare(g, o)
    assert g.clock() == o.clock()


@pytest.mark.parametrize("shape", [(13, 7, 9), (5, 11, 4), (1, 1, 6)])
@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_ragged_sedov_bitwise(shape, rezone):
    cfg = sedov(shape, rezone)
    g, o, rg, ro = run_pair(cfg, 25)
    assert rg == ro
    compare(g, o)
    assert g.clock() == o.clock()


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_perturbed_states_bitwise(seed, rezone):
    cfg = sedov((16, 12, 10), rezone, reflect_mask=[0x15, 0x3F, 0x00][seed], e_background=0.5)
    g, o = _sale(cfg), O.Oracle(cfg)
    apply_perturbation([o, g], cfg, seed, lagrange=(rezone == LAGRANGE))
    compare(g, o)
    assert g.step(20) == o.step(20)
    compare(g, o)
    assert g.clock() == o.clock()


def test_euler_sedov_bitwise():
    cfg = sedov((24, 24, 24), EULER)
    g, o, rg, ro = run_pair(cfg, 60)
    assert rg == ro == (0, 60)
    compare(g, o)


@pytest.mark.parametrize("rezone,slabs", [(LAGRANGE, 2), (LAGRANGE, 5), (EULER, 2), (EULER, 4)])
def test_local_slabs_bitwise(rezone, slabs):
    """Emulated ranks on one GPU: z-slabs with ghost planes exchanged by device
    copies give the same bits as one slab and as the oracle."""
    cfg = sedov((12, 10, 17), rezone)
    g1 = _sale(cfg)
    gs = _sale(cfg, local_slabs=slabs)
    o = O.Oracle(cfg)
    for c in (g1, gs, o):
        assert c.step(30) == (0, 30)
    compare(gs, g1)
    compare(gs, o)


def test_tangle_same_cycle_and_cell():
    cfg = sedov((4, 4, 4), LAGRANGE)
    g, o = _sale(cfg), O.Oracle(cfg)
    X = o.get("X")
    X[2, 2, 2] += 2.0
    for c in (g, o):
        c.set("X", X)
    rg, ro = g.step(3), o.step(3)
    assert rg == ro == (O.ETANGLED, 0)
    assert "cycle=0 cell=2,1,1" in g.last_error()
    assert g.step(1)[0] == 8  # poisoned


def test_t_end_landing_and_collapse():
    cfg = sedov((6, 6, 6), EULER, t_end=2e-3)
    g, o = _sale(cfg), O.Oracle(cfg)
    assert g.step(100000) == o.step(100000)
    assert g.clock() == o.clock()
    assert g.clock()["t"] == 2e-3 and g.clock()["finished"] == 1
    compare(g, o)
    cfg = sedov((4, 4, 4), LAGRANGE, t_end=1e20)
    g, o = _sale(cfg), O.Oracle(cfg)
    assert g.step(2) == o.step(2) == (O.EDTCOLLAPSE, 0)


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_checkpoint_resume_bitwise(rezone):
    cfg = sedov((8, 8, 8), rezone)
    a = _sale(cfg)
    a.step(12)
    b = _sale(cfg)
    b.step(6)
    fields = ["UX", "UY", "UZ", "MASS", "E"] + (["X", "Y", "Z"] if rezone == LAGRANGE else [])
    snap = {f: b.get(f) for f in fields}
    clk = b.clock()
    c = _sale(cfg)
    for f, v in snap.items():
        c.set(f, v)
    c.set_clock(clk["t"], clk["dt_last"], clk["cycle"])
    c.step(6)
    compare(c, a)
    assert c.clock() == a.clock()


def test_device_field_io_and_async():
    cfg = sedov((8, 8, 8), LAGRANGE)
    g = _sale(cfg)
    g.step_async(3)
    g.step_async(2)
    assert g.sync() == (0, 5)
    o = O.Oracle(cfg)
    o.step(5)
    out = torch.empty(g.node_shape, dtype=torch.float64, device="cuda")
    g.get("UX", out=out)
    assert np.array_equal(out.cpu().numpy(), o.get("UX"))
    g.set("E", torch.from_numpy(o.get("E")).cuda())
    assert np.array_equal(g.get("E"), o.get("E"))


@pytest.mark.parametrize("name,cycles", [("C3", 3), ("C4", 3)])
def test_full_size_slab_split_bitwise(name, cycles):
    """Full-size meshes in the bench launch configuration (one slab) against the same
    mesh as two emulated z-slabs exchanging ghost planes: every state field and the
    clock agree bitwise (the oracle vouches for both at full size through the golden
    digests of tests/golden/, and element by element at smaller sizes above)."""
    cfg, _ = config(name)
    a = _sale(cfg)
    assert a.step(cycles) == (0, cycles)
    fields = ("UX", "UY", "UZ", "E", "MASS") + (("X", "Y", "Z") if cfg["rezone"] == LAGRANGE else ())
    ref = {f: a.get(f) for f in fields}
    clk = a.clock()
    a.close()
    del a
    torch.cuda.empty_cache()
    b = _sale(cfg, local_slabs=2)
    assert b.step(cycles) == (0, cycles)
    for f in fields:
        g = b.get(f)
        assert np.array_equal(g.view(np.int64), ref[f].view(np.int64)), f
    assert b.clock() == clk


@pytest.mark.parametrize("hg", [0.0, 2.0])
@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_hourglass_coefficient_bitwise(hg, rezone):
    """Reading HG off (hg = 0) and strong (the cap binds in most cells): bitwise."""
    cfg = sedov((11, 9, 13), rezone, hg=hg, e_background=0.2)
    g, o = _sale(cfg), O.Oracle(cfg)
    apply_perturbation([o, g], cfg, 3, lagrange=(rezone == LAGRANGE), u_scale=0.05)
    assert g.step(12) == o.step(12) == (0, 12)
    compare(g, o)
    assert g.clock() == o.clock()


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_nccl_one_rank_communicator(rezone):
    """The NCCL plumbing on one GPU: a 1-rank communicator (ncclCommInitRank from
    a unique id, the per-cycle 16-byte ncclAllReduce(min) on the stream, async
    error polling, ncclCommDestroy) gives the same bits as the NCCL-free path."""
    from paper_2209_01983_b200.sale import nccl_unique_id
    cfg = sedov((12, 10, 9), rezone)
    a = _sale(cfg, nccl_id=nccl_unique_id())
    b = _sale(cfg)
    o = O.Oracle(cfg)
    for c in (a, b, o):
        assert c.step(15) == (0, 15)
    compare(a, b)
    compare(a, o)
    a.close()


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
@pytest.mark.parametrize("shape", [(67, 17, 70), (31, 44, 33)])
def test_multi_tile_ragged_bitwise(rezone, shape):
    """Meshes spanning several fused tiles in x (30/31/29-column tiles), y (5-9
    rows) and z (32-plane chunks) with ragged tails, against the oracle."""
    cfg = sedov(shape, rezone, e_background=0.3)
    g, o = _sale(cfg), O.Oracle(cfg)
    apply_perturbation([o, g], cfg, 7, lagrange=(rezone == LAGRANGE))
    assert g.step(6) == o.step(6) == (0, 6)
    compare(g, o)
    assert g.clock() == o.clock()


def test_degenerate_single_free_cube():
    cfg = sedov((1, 1, 1), LAGRANGE, reflect_mask=0, e_deposit=2.5, e_background=2.5)
    g, o = _sale(cfg), O.Oracle(cfg)
    assert g.step(3) == o.step(3) == (0, 3)
    compare(g, o)


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_quiescent_state_gpu(rezone):
    """Uniform state, all faces reflecting: equal to the oracle bit for bit; a
    fixed point to round-off (bitwise only on power-of-two meshes, SURVEY c.9)."""
    cfg = sedov((9, 7, 8), rezone, gamma=1.5, reflect_mask=0x3F)
    g, o = _sale(cfg), O.Oracle(cfg)
    for c in (g, o):
        c.set("E", np.full(g.cell_shape, 2.0))
    assert g.step(5) == o.step(5) == (0, 5)
    compare(g, o)
    for f in ("UX", "UY", "UZ"):
        assert np.max(np.abs(g.get(f))) <= 1e-13
    assert np.max(np.abs(g.get("E") - 2.0)) <= 1e-13


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
@pytest.mark.parametrize("slabs,shape", [(2, (12, 10, 17)), (3, (9, 7, 26)), (4, (7, 6, 13))])
@pytest.mark.parametrize("nmat", [0, 2])
def test_boundary_first_overlap_bitwise(rezone, slabs, shape, nmat):
    """Boundary-first cycles (sale_params.overlap = 1): the tail
    kernel on the exchanged planes first, the halo exchange on a side stream while the
    interior finishes -- bitwise against the plain cycle and the oracle, thin slabs
    (no interior) included, with the CUDA-graph replay of cycle pairs."""
    kw = dict(nmat=nmat, mat_gamma=[1.4, 5.0 / 3.0]) if nmat else {}
    cfg = sedov(shape, rezone, e_background=0.3, **kw)
    a = _sale(dict(cfg, overlap=1), local_slabs=slabs)
    b = _sale(dict(cfg, overlap=-1), local_slabs=slabs)
    o = O.Oracle(cfg)
    if not nmat:
        apply_perturbation([o, a, b], cfg, 5, lagrange=(rezone == LAGRANGE))
    for n in (1, 6, 11):
        ra, rb, ro = a.step(n), b.step(n), o.step(n)
        assert ra == rb == ro, (ra, rb, ro)
    compare(a, b)
    compare(a, o)
    assert a.clock() == o.clock()
