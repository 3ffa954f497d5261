"""The N>1 path's host logic on CPU: the z-slab layout and the X1 halo plan that
sale_step executes with ncclSend/ncclRecv, run here over torch.distributed gloo
with world_size 2 and 3.  Each rank fills its owned planes from a global array
with unique values, executes its plan, and checks that every ghost plane now
holds the neighbour's bits and nothing else changed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_01983_b200 import build, sale
from paper_2209_01983_b200.configs import EULER, LAGRANGE, sedov

NODE = ("X", "Y", "Z", "UX", "UY", "UZ")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global(cfg, field):
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    shape = (nz + 1, ny + 1, nx + 1) if field in NODE else (nz, ny, nx)
    k, j, i = np.meshgrid(*(np.arange(n) for n in shape), indexing="ij")
    return (sale.FIELDS[field] * 1e7 + k * 1e4 + j * 1e2 + i).astype(np.float64)


def _worker(rank, world, port, cfg, full, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        lay = sale.local_layout(cfg, rank, world)
        plan = sale.halo_plan(cfg, rank, world, full=full)
        k0, k1, g = lay["k0"], lay["k1"], lay["ghost"]
        kb = k0 - g
        fields = sorted({m["field"] for m in plan})
        loc, ref = {}, {}
        for f in fields:
            G = _global(cfg, f)
            nplanes = lay["node_planes"] if f in NODE else lay["cell_planes"]
            L = np.full((nplanes,) + G.shape[1:], np.nan)
            hi = k1 + 1 if f in NODE else k1
            L[k0 - kb:hi - kb] = G[k0:hi]
            loc[f] = torch.from_numpy(L)
            ref[f] = G
        reqs = []
        for m in plan:
            flat = loc[m["field"]].view(-1)
            seg = flat[m["offset"]:m["offset"] + m["count"]]
            # one tag for every message, posted in plan order: a receive matches the
            # peer's sends to this rank in posting order -- the pairing ncclSend /
            # ncclRecv use inside one group (no tags there)
            if m["send"]:
                reqs.append(dist.isend(seg.clone(), m["peer"], tag=0))
            else:
                buf = torch.empty_like(seg)
                reqs.append((dist.irecv(buf, m["peer"], tag=0), seg, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                r[1].copy_(r[2])
            else:
                r.wait()
        bad = []
        for f in fields:
            L, G = loc[f].numpy(), ref[f]
            top = cfg["nz"] if f in NODE else cfg["nz"] - 1
            for l in range(L.shape[0]):
                k = kb + l
                ghost = (k0 - g <= k < k0) or ((k1 + 1 if f in NODE else k1) <= k < (k1 + 1 if f in NODE else k1) + g)
                owned = (k0 <= k <= k1) if f in NODE else (k0 <= k < k1)
                if owned or (ghost and 0 <= k <= top):
                    if not np.array_equal(L[l], G[k]):
                        bad.append((f, k))
                elif not np.all(np.isnan(L[l])):
                    bad.append(("touched", f, k))
        q.put((rank, bad, [(m["peer"], m["send"], m["field"], m["count"]) for m in plan]))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        q.put((rank, ["exception: %r" % ex], []))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("rezone,full,nmat", [(LAGRANGE, False, 0), (LAGRANGE, True, 0), (EULER, False, 0),
                                              (EULER, False, 2), (LAGRANGE, True, 3)])
def test_halo_plan_over_gloo(world, rezone, full, nmat):
    build.build()
    cfg = sedov((5, 4, 13), rezone)
    if nmat:  # the material axis: one cell array per material and quantity joins the plan
        cfg = dict(cfg, nmat=nmat, mat_gamma=[1.4, 1.6, 1.8][:nmat])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, full, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, bad, plan = q.get(timeout=120)
        res[r] = (bad, plan)
    for p in procs:
        p.join(timeout=60)
    for r, (bad, _) in res.items():
        assert not bad, (r, bad[:5])
    # NCCL pairing: the k-th send from a to b is the k-th receive at b from a, with the
    # same field and count (the plans list the fields in the same order on every rank)
    for a, (_, plan_a) in res.items():
        for b in res:
            sends = [(f, c) for peer, send, f, c in plan_a if peer == b and send]
            recvs = [(f, c) for peer, send, f, c in res[b][1] if peer == a and not send]
            assert sends == recvs, (a, b)


def test_layout_remainder_to_lowest_ranks():
    build.build()
    cfg = sedov((4, 4, 10), EULER)
    lays = [sale.local_layout(cfg, r, 3) for r in range(3)]
    assert [(l["k0"], l["k1"]) for l in lays] == [(0, 4), (4, 7), (7, 10)]
    assert all(l["ghost"] == 3 and l["cell_planes"] == (l["k1"] - l["k0"]) + 6 for l in lays)
    cfg = sedov((4, 4, 10), LAGRANGE)
    assert sale.local_layout(cfg, 0, 4)["ghost"] == 1
    with pytest.raises(sale.SaleError):
        sale.local_layout(sedov((4, 4, 5), EULER), 0, 2)  # slabs of 2 planes < g = 3


def test_plan_field_sets():
    build.build()
    cfg = sedov((4, 4, 8), LAGRANGE)
    f = {m["field"] for m in sale.halo_plan(cfg, 0, 2)}
    assert f == {"X", "Y", "Z", "UX", "UY", "UZ", "E"}
    assert "MASS" in {m["field"] for m in sale.halo_plan(cfg, 0, 2, full=True)}
    e = {m["field"] for m in sale.halo_plan(sedov((4, 4, 8), EULER), 1, 2)}
    assert e == {"UX", "UY", "UZ", "MASS", "E"}
    assert sale.halo_plan(cfg, 0, 1) == []
    m = {m["field"] for m in sale.halo_plan(sedov((4, 4, 8), EULER, nmat=2, mat_gamma=[1.4, 1.6]), 1, 2)}
    assert m == e | {"MAT_F0", "MAT_M0", "MAT_E0", "MAT_F1", "MAT_M1", "MAT_E1"}
    lm = sedov((4, 4, 8), LAGRANGE, nmat=2, mat_gamma=[1.4, 1.6])
    assert {m["field"] for m in sale.halo_plan(lm, 0, 2)} == f | {"MAT_E0", "MAT_E1"}  # f_k, m_k constant
    assert {m["field"] for m in sale.halo_plan(lm, 0, 2, full=True)} >= {"MAT_F1", "MAT_M1", "MASS"}
