"""A longer randomised parity sweep than tests/test_gpu_fuzz.py (the race detector while
compute-sanitizer is closed on the pool): N seeded random cases -- mesh shape 1..41 per
axis, rezone mode, 1-3 emulated slabs, 0 or 1-4 materials, a perturbed / mixed state,
hourglass coefficient 0 / 0.5 / 3, boundary-first cycles on or off, the copy or the
peer-store halo, random sale_step chunkings -- each compared bit for bit with the oracle.
python scripts/fuzz_stress.py N [first_seed] [out.json]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import oracle as O  # noqa: E402
from paper_2209_01983_b200.configs import EULER, LAGRANGE, sedov  # noqa: E402
from paper_2209_01983_b200.sale import Sale  # noqa: E402
from tests.helpers import ALL_FIELDS, apply_perturbation  # noqa: E402
from tests.test_gpu_materials import apply_perturbation_mm, mat_fields  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
first = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
t0 = time.time()
bad, statuses = [], {}
for case in range(first, first + n):
    rng = np.random.Generator(np.random.PCG64(case))
    shape = tuple(int(x) for x in rng.integers(1, 42, size=3))
    rezone = (LAGRANGE, EULER)[int(rng.integers(0, 2))]
    g_depth = 1 if rezone == LAGRANGE else 3
    slabs = max(1, min(int(rng.integers(1, 4)), shape[2] // g_depth))
    nmat = int(rng.integers(0, 5)) if rng.uniform() < 0.5 else 0
    extra = {"nmat": nmat, "mat_gamma": [float(x) for x in rng.uniform(1.1, 3.0, size=nmat)]} if nmat else {}
    hg = (0.0, 0.5, 3.0)[int(rng.integers(0, 3))]
    ov = (-1, 1)[int(rng.integers(0, 2))]
    cfg = sedov(shape, rezone, hg=hg, **extra)
    halo = int(np.random.Generator(np.random.PCG64(case + 7919)).integers(0, 2))  # copy / peer-store halo
    g, o = Sale(dict(cfg, overlap=ov, halo=halo), local_slabs=slabs), O.Oracle(cfg)
    seed = int(rng.integers(0, 1000))
    if nmat:
        apply_perturbation_mm((g, o), cfg, seed)
    else:
        apply_perturbation([g, o], cfg, seed, lagrange=(rezone == LAGRANGE))
    ok = True
    for k in rng.integers(1, 9, size=3):
        rg, ro = g.step(int(k)), o.step(int(k))
        ok = ok and rg == ro
    statuses[str(ro[0])] = statuses.get(str(ro[0]), 0) + 1
    fields = ALL_FIELDS + (mat_fields(nmat) if nmat else ())
    for f in fields:
        if not np.array_equal(g.get(f).view(np.int64), o.get(f).view(np.int64)):
            ok = False
    ok = ok and g.clock() == o.clock()
    if not ok:
        bad.append({"case": case, "shape": shape, "rezone": rezone, "slabs": slabs, "nmat": nmat, "hg": hg,
                    "overlap": ov, "halo": halo})
    g.close()
res = {"cases": n, "first_seed": first, "mismatches": bad, "final_status_counts": statuses,
       "seconds": time.time() - t0}
print(json.dumps(res))
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as f:
        json.dump(res, f)
