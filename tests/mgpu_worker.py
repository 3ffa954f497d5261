"""One rank of the multi-GPU parity check (tests/test_multigpu.py), launched as
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port P tests/mgpu_worker.py [--full]

Every rank runs its z-slab through the C ABI on its own GPU (NCCL halo exchange and
dt allreduce); rank 0 assembles the owned slabs (the interface node
plane is replicated: both owners' copies must be bit-equal) and compares:
  - small meshes with the CPU oracle, element by element, bitwise;
  - with --full, BASELINE's C1 / C2 / C3 runs, the 2-GPU C4 problem (C4n2) and the
    two-material C2M2 with the
    oracle's golden SHA-256 digests in tests/golden/ (the same files the 1-GPU
    test_gpu_golden.py reproduces), so the assembled multi-GPU fields must be the
    1-GPU bits.
Prints one JSON line per case on rank 0; exits non-zero on any mismatch.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2209_01983_b200 import inputs, sale as S  # noqa: E402
from paper_2209_01983_b200.configs import EULER, LAGRANGE, config, sedov  # noqa: E402

STATE = ("UX", "UY", "UZ", "MASS", "E")


def assemble(ctx, cfg, field, rank, world):
    """The global field on rank 0 from every rank's owned slab (None elsewhere)."""
    a = ctx.get(field)
    parts = [None] * world if rank == 0 else None
    dist.gather_object((ctx.k0, ctx.k1, a), parts, dst=0)
    if rank != 0:
        return None
    node = field in S.NODE_FIELDS
    nz = cfg["nz"]
    out = np.full(((nz + 1) if node else nz,) + a.shape[1:], np.nan)
    for k0, k1, arr in parts:
        lo = k0
        if node and not np.isnan(out[k0]).all():  # the replicated interface plane
            if not np.array_equal(out[k0].view(np.int64), arr[0].view(np.int64)):
                raise AssertionError(f"{field}: interface plane {k0} differs between its two owners")
        out[lo:lo + arr.shape[0]] = arr
    return out


def fresh_nccl_id(rank):
    """A new NCCL unique id from rank 0 for every context (an id initialises one
    communicator only)."""
    obj = [S.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def run_case(name, cfg, cycles, world, rank, local, mat_halves=False):
    ctx = S.Sale(cfg, device=local, rank=rank, nranks=world, nccl_id=fresh_nccl_id(rank))
    if mat_halves:  # C2M2's initial material layout, from the assembled Sedov state
        m = assemble(ctx, cfg, "MASS", rank, world)
        e0 = assemble(ctx, cfg, "MAT_E0", rank, world)
        halves = inputs.material_halves(cfg, m, e0) if rank == 0 else None
        obj = [halves]
        dist.broadcast_object_list(obj, src=0)
        for f, v in obj[0].items():
            ctx.set(f, np.ascontiguousarray(v[ctx.k0:ctx.k1]))
    done, rc = 0, 0
    target = cycles if cycles > 0 else 10 ** 9
    while done < target:
        rc, d = ctx.step(min(1000, target - done))
        done += d
        if rc or d == 0:
            break
    clk = ctx.clock()
    fields = (("X", "Y", "Z") if cfg["rezone"] == LAGRANGE else ()) + STATE
    if cfg.get("nmat"):
        fields += tuple(f"MAT_{q}{k}" for k in range(cfg["nmat"]) for q in "FME")
    glob = {f: assemble(ctx, cfg, f, rank, world) for f in fields}
    ctx.close()
    return rc, done, clk, glob


def main():
    full = "--full" in sys.argv
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    failures = 0

    # small meshes against the CPU oracle (rank 0 computes it)
    small = [("C0", *config("C0")), ("E24", sedov((24, 20, 4 * world + 9), EULER), 40),
             ("L-warm", sedov((17, 13, 3 * world + 11), LAGRANGE, e_background=0.3), 25)]
    # and the same with the peer-store halo (kernels storing straight into the
    # neighbours' ghost planes over NVLink; sale_params.halo = SALE_HALO_PEER)
    small += [(name + "-peer", dict(cfg, halo=S.HALO_PEER), cycles) for name, cfg, cycles in small]
    for name, cfg, cycles in small:
        rc, done, clk, glob = run_case(name, cfg, cycles, world, rank, local)
        if rank == 0:
            import oracle as O
            o = O.Oracle(cfg)
            ro = o.step(cycles)
            mism = {f: int(np.count_nonzero(v.view(np.int64) != o.get(f).view(np.int64)))
                    for f, v in glob.items()}
            ok = (rc, done) == ro and clk == o.clock() and not any(mism.values())
            failures += not ok
            print(json.dumps({"case": name, "n_gpus": world, "ok": ok, "status": [rc, done],
                              "oracle_status": list(ro), "mismatches": mism}), flush=True)

    if full:  # BASELINE configs against the oracle's golden digests
        gold = os.path.join(ROOT, "tests", "golden")
        # (and C3 / C4n2 once more with the peer-store halo)
        for name in ("C1", "C2", "C2M2", "C3", "C4n2", "C3-peer", "C4n2-peer"):
            base = name.split("-")[0]
            path = os.path.join(gold, f"{base}.json")
            if not os.path.exists(path):
                continue
            g = json.load(open(path))
            cfg, _ = config(base.split("n")[0], int(base.split("n")[1]) if "n" in base else 1)
            if name.endswith("-peer"):
                cfg = dict(cfg, halo=S.HALO_PEER)
            rc, done, clk, glob = run_case(name, cfg, g["requested_cycles"], world, rank, local,
                                           mat_halves=bool(cfg.get("nmat")))
            if rank == 0:
                bad = [f for f, v in glob.items()
                       if hashlib.sha256(np.ascontiguousarray(v).ravel().tobytes()).hexdigest()
                       != g["fields"][f]["sha256"]]
                ok = (rc, done) == (g["status"], g["cycles_done"]) and clk == g["clock"] and not bad
                failures += not ok
                print(json.dumps({"case": name, "n_gpus": world, "ok": ok, "status": [rc, done],
                                  "golden_status": [g["status"], g["cycles_done"]], "digest_mismatch": bad}),
                      flush=True)
    obj = [failures]
    dist.broadcast_object_list(obj, src=0)
    dist.destroy_process_group()
    sys.exit(1 if obj[0] else 0)


if __name__ == "__main__":
    main()
