"""Tiny workload for compute-sanitizer: every cycle kernel of both modes (fused and v0
schedules, one and two local slabs) on a small ragged mesh, a few cycles each."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import EULER, LAGRANGE, sedov
from paper_2209_01983_b200.sale import Sale
for rezone in (LAGRANGE, EULER):
    for impl in ("fused", "v0"):
        for slabs in (1, 2):
            cfg = sedov((37, 11, 14), rezone)
            g = Sale(cfg, impl=impl, local_slabs=slabs)
            rc = g.step(4)
            assert rc == (0, 4), rc
            for f in ("UX", "E", "RHO", "MASS"):
                g.get(f)
            print("ok", rezone, impl, slabs, flush=True)
            del g
