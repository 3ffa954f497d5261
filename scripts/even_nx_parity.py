import sys, numpy as np
sys.path.insert(0, "/root/repo")
import oracle as O
from paper_2209_01983_b200.configs import sedov, EULER
from paper_2209_01983_b200.sale import Sale
from tests.helpers import compare, apply_perturbation
bad = 0
for case in range(40):
    rng = np.random.Generator(np.random.PCG64(777 + case))
    nx = 2 * int(rng.integers(1, 21)); ny = int(rng.integers(1, 41)); nz = int(rng.integers(3, 41))
    slabs = max(1, min(int(rng.integers(1, 4)), nz // 3))
    cfg = sedov((nx, ny, nz), EULER)
    g, o = Sale(dict(cfg, halo=case % 2), local_slabs=slabs), O.Oracle(cfg)
    apply_perturbation([g, o], cfg, case, lagrange=False)
    ok = True
    for n in rng.integers(1, 9, size=3):
        if g.step(int(n)) != o.step(int(n)): ok = False
    try: compare(g, o)
    except AssertionError as e: ok = False; print(str(e)[:300])
    print("ok" if ok else "FAIL", (nx, ny, nz), slabs, flush=True); bad += not ok
sys.exit(1 if bad else 0)
