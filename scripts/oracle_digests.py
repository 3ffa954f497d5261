"""Write golden digests of the CPU oracle for a BASELINE config (calls only oracle/).

    python scripts/oracle_digests.py C2            # full length
    python scripts/oracle_digests.py C3 --cycles 200 --threads 7

Output tests/golden/<name>.json: the clock, the status, and for every state and
derived field the SHA-256 of its float64 bytes (x fastest, then y, then z) plus a
strided sample (every 4099th element) for a tolerance comparison if the bits ever
differ.  The GPU tests recompute the same digests from libsale's fields.
--threads N runs the -fopenmp build of the same oracle source (bit-identical to the
serial build: oracle.c header).  Sedov runs also record, after every chunk, the
shell-averaged radius of the density peak and the total energy (harness side, c.7),
so the similarity law can be checked on the oracle's own trajectory (tests/
test_oracle_physics.py).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2209_01983_b200 import inputs  # noqa: E402
from paper_2209_01983_b200.configs import config  # noqa: E402

FIELDS = ("X", "Y", "Z", "UX", "UY", "UZ", "MASS", "E", "NODE_MASS", "RHO", "VOL", "P", "Q", "CS")
STRIDE = 4099


def snapshot(o, cfg):
    """t, cycle, shell-averaged radius of the density peak (bins of one cell width over
    the cell-centroid radius; centroid = mean of the 8 nodes), total energy IE + KE
    (math.fsum, c.7)."""
    import math
    rho = o.get("RHO")
    X, Y, Z = (o.get(f) for f in ("X", "Y", "Z"))

    def cc(A):
        return 0.125 * (A[:-1, :-1, :-1] + A[1:, :-1, :-1] + A[:-1, 1:, :-1] + A[1:, 1:, :-1]
                        + A[:-1, :-1, 1:] + A[1:, :-1, 1:] + A[:-1, 1:, 1:] + A[1:, 1:, 1:])
    r = np.sqrt(cc(X) ** 2 + cc(Y) ** 2 + cc(Z) ** 2)
    h = cfg["lx"] / cfg["nx"]
    bins = np.arange(0.0, 2.0, h)
    idx = np.digitize(r.ravel(), bins)
    cnt = np.bincount(idx, minlength=len(bins) + 2)
    prof = np.bincount(idx, weights=rho.ravel(), minlength=len(bins) + 2) / np.maximum(cnt, 1)
    R = float(bins[int(np.argmax(prof)) - 1] + 0.5 * h)
    u2 = o.get("UX") ** 2 + o.get("UY") ** 2 + o.get("UZ") ** 2
    E = math.fsum((o.get("MASS") * o.get("E")).ravel()) + math.fsum((0.5 * o.get("NODE_MASS") * u2).ravel())
    clk = o.clock()
    return {"t": clk["t"], "cycle": clk["cycle"], "R": R, "rho_max": float(rho.max()), "E_total": E}


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--cycles", type=int, default=None)
    ap.add_argument("--chunk", type=int, default=10)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--gpus", type=int, default=1, help="C4 only: the n-GPU problem (lz = n), file C4n<n>.json")
    args = ap.parse_args()
    if args.threads > 0:
        os.environ["OMP_NUM_THREADS"] = str(args.threads)
        O.use_openmp()
    cfg, cycles = config(args.name, args.gpus)
    if args.cycles is not None:
        cycles = args.cycles
    o = O.Oracle(cfg)
    fields = FIELDS
    if cfg.get("nmat"):  # the material runs: initial layout, and the material fields too
        for f, v in inputs.material_halves(cfg, o.get("MASS"), o.get("MAT_E0")).items():
            o.set(f, v)
        fields = FIELDS + tuple(f"MAT_{q}{k}" for k in range(cfg["nmat"]) for q in "FME")
    t0 = time.time()
    done, rc = 0, 0
    target = cycles if cycles > 0 else 10 ** 9
    traj = []
    while done < target:
        rc, d = o.step(min(args.chunk, target - done))
        done += d
        print(f"{args.name}: {done} cycles, t={o.clock()['t']:.6g}, {time.time() - t0:.0f}s", flush=True)
        if not rc and d and not cfg.get("nmat"):
            traj.append(snapshot(o, cfg))
        if rc or d == 0:
            break
    out = {"config": args.name, "params": cfg, "requested_cycles": cycles, "cycles_done": done, "status": rc,
           "last_error": o.last_error() if rc else "", "clock": o.clock(), "stride": STRIDE, "fields": {},
           "oracle_seconds": time.time() - t0, "trajectory": traj}
    for f in fields:
        a = o.get(f).ravel()
        out["fields"][f] = {"sha256": digest(a), "n": int(a.size),
                            "sample": [float(v) for v in a[::STRIDE]]}
    tag = args.name + (f"n{args.gpus}" if args.gpus > 1 else "")
    out["config"] = tag
    out["n_gpus"] = args.gpus
    path = os.path.join(ROOT, "tests", "golden", f"{tag}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        json.dump(out, fh)
    print("wrote", path)


if __name__ == "__main__":
    main()
