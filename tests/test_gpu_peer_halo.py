"""GPU parity of the peer-store halo (sale_params.halo = SALE_HALO_PEER; SURVEY §8(f)
NEXT-1, the paper's per-cycle exchange P:372-375 fused into the kernels that produce
the planes): on emulated slabs the producer kernels (Lagrange kc_force / kc_energy,
Euler kr_tail, materials k_mat_flux / kn_update) store the ghost planes straight into
the neighbouring slab, no copy exchange runs -- bitwise against the copy exchange and
the oracle, both modes, 0 / 2 mixed materials, thin slabs, CUDA-graph replay on and
off, several sale_step calls.  The rank path (CUDA IPC mappings + the system-scope
arrival counters) needs two GPUs: tests/test_multigpu.py runs it with halo = PEER."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from paper_2209_01983_b200.configs import EULER, LAGRANGE, sedov
from tests.helpers import ALL_FIELDS, apply_perturbation, compare
from tests.test_gpu_materials import GAMMAS, apply_perturbation_mm, mat_fields

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sale(cfg, **kw):
    from paper_2209_01983_b200.sale import Sale
    return Sale(cfg, **kw)


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
@pytest.mark.parametrize("slabs,shape", [(2, (12, 10, 17)), (3, (9, 7, 26)), (4, (7, 6, 13))])
@pytest.mark.parametrize("nmat", [0, 2])
def test_peer_halo_bitwise(rezone, slabs, shape, nmat):
    from paper_2209_01983_b200.sale import HALO_COPY, HALO_PEER
    kw = dict(nmat=nmat, mat_gamma=GAMMAS[:nmat]) if nmat else {}
    cfg = sedov(shape, rezone, e_background=0.3, **kw)
    a = _sale(dict(cfg, halo=HALO_PEER), local_slabs=slabs)
    b = _sale(dict(cfg, halo=HALO_COPY), local_slabs=slabs)
    o = O.Oracle(cfg)
    fields = ALL_FIELDS + (mat_fields(nmat) if nmat else ())
    if nmat:
        apply_perturbation_mm((a, o, b), cfg, 11)  # (the oracle, second, supplies the base state)
    else:
        apply_perturbation([o, a, b], cfg, 5, lagrange=(rezone == LAGRANGE))
    for n in (1, 6, 11):
        ra, rb, ro = a.step(n), b.step(n), o.step(n)
        assert ra == rb == ro, (ra, rb, ro)
    compare(a, b, fields)
    compare(a, o, fields)
    assert a.clock() == o.clock()


@pytest.mark.parametrize("rezone", [LAGRANGE, EULER])
def test_peer_halo_without_graphs(rezone):
    """The same on the plain launch path (SALE_GRAPHS=0: every cycle enqueued
    individually), in a child process (the switch is read once per process)."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import oracle as O\n"
        "from paper_2209_01983_b200.configs import sedov\n"
        "from paper_2209_01983_b200.sale import Sale, HALO_PEER\n"
        "from tests.helpers import apply_perturbation, compare\n"
        "cfg = sedov((11, 9, 20), %d, e_background=0.3)\n"
        "g, o = Sale(dict(cfg, halo=HALO_PEER), local_slabs=3), O.Oracle(cfg)\n"
        "apply_perturbation([o, g], cfg, 3, lagrange=(%d == 0))\n"
        "for n in (2, 5, 7):\n"
        "    assert g.step(n) == o.step(n) == (0, n)\n"
        "compare(g, o)\n"
        "print('ok')\n" % (ROOT, rezone, rezone))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SALE_GRAPHS="0"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_peer_halo_single_slab_and_args():
    """One slab: PEER has no neighbour (the copy path's results); an unknown mode is
    rejected by sale_workspace_bytes / sale_create."""
    from paper_2209_01983_b200 import sale
    cfg = sedov((8, 8, 8), EULER)
    a, b = _sale(dict(cfg, halo=sale.HALO_PEER)), _sale(cfg)
    assert a.step(5) == b.step(5) == (0, 5)
    compare(a, b)
    assert sale.workspace_bytes(dict(cfg, halo=2)) == 0
    assert sale.workspace_bytes(dict(cfg, halo=sale.HALO_PEER)) > sale.workspace_bytes(cfg) - 1


@pytest.mark.parametrize("name,slabs", [("C3", 4), ("C4n2", 2), ("C2M2", 3)])
def test_peer_halo_full_length_digest(name, slabs):
    """The BASELINE runs on emulated slabs with the peer-store halo reproduce the oracle's
    golden digests (tests/golden/, written by scripts/oracle_digests.py from the oracle
    only): C3 on 4 slabs (200 Lagrangian cycles), the 2-GPU weak-scaling problem C4n2 on
    2 slabs (100 Eulerian cycles), and the two-material C2M2 on 3 slabs (300 cycles)."""
    import hashlib
    import json
    from paper_2209_01983_b200 import inputs
    from paper_2209_01983_b200.configs import config
    from paper_2209_01983_b200.sale import HALO_PEER
    path = os.path.join(ROOT, "tests", "golden", f"{name}.json")
    if not os.path.exists(path):
        pytest.skip("no golden")
    g = json.load(open(path))
    cfg, _ = config(name.split("n")[0], int(name.split("n")[1]) if "n" in name else 1)
    ctx = _sale(dict(cfg, halo=HALO_PEER), local_slabs=slabs)
    if cfg.get("nmat"):
        for f, v in inputs.material_halves(cfg, ctx.get("MASS"), ctx.get("MAT_E0")).items():
            ctx.set(f, v)
    done, rc = 0, 0
    while done < g["requested_cycles"]:
        rc, d = ctx.step(min(1000, g["requested_cycles"] - done))
        done += d
        if rc or d == 0:
            break
    assert (rc, done) == (g["status"], g["cycles_done"])
    assert ctx.clock() == g["clock"]
    bad = [f for f, ref in g["fields"].items()
           if hashlib.sha256(ctx.get(f).ravel().tobytes()).hexdigest() != ref["sha256"]]
    assert not bad, bad


def test_peer_halo_error_paths_same_cycle_and_cell():
    """Errors with the peer-store halo on emulated slabs: a tangled cell in the upper slab
    (Lagrange) and ENEGMASS from a CFL-1.5 uniform translation over alternating
    densities (Euler) -- the oracle's status, good-cycle count, cell and clock."""
    from paper_2209_01983_b200.sale import HALO_PEER
    cfg = sedov((4, 4, 8), LAGRANGE)
    g, o = _sale(dict(cfg, halo=HALO_PEER), local_slabs=2), O.Oracle(cfg)
    X = o.get("X")
    X[6, 2, 2] += 2.0  # a node of the upper slab
    for c in (g, o):
        c.set("X", X)
    assert g.step(3) == o.step(3) == (O.ETANGLED, 0)
    assert o.last_error().split()[-1] in g.last_error()
    cfg = sedov((7, 6, 9), EULER, cfl=1.5, reflect_mask=0, e_deposit=0.0, e_background=1e-6)
    g, o = _sale(dict(cfg, halo=HALO_PEER), local_slabs=3), O.Oracle(cfg)
    m = o.get("MASS") * np.where((np.arange(7) % 2) == 0, 1.0, 0.05)[None, None, :]
    for c in (g, o):
        c.set("UX", np.ones(o.node_shape))
        c.set("MASS", m)
    rg, ro = g.step(20), o.step(20)
    assert rg == ro and ro[0] == O.ENEGMASS, (rg, ro)
    assert o.last_error().split()[-1] in g.last_error()
    assert g.clock() == o.clock()
