"""Quick GPU-vs-oracle bitwise check on small meshes (both modes, emulated slabs,
materials) for iteration; the full suite is tests/ -m gpu."""
import sys
sys.path.insert(0, "/root/repo")
import oracle as O
from paper_2209_01983_b200.configs import sedov, LAGRANGE, EULER
from paper_2209_01983_b200.sale import Sale
from tests.helpers import compare, apply_perturbation

bad = 0
for rez in (LAGRANGE, EULER):
    for shape, slabs, nmat in (((12, 10, 9), 1, 0), ((33, 17, 40), 1, 0), ((13, 7, 19), 3, 0), ((11, 9, 8), 1, 2)):
        kw = dict(nmat=nmat, mat_gamma=[1.4, 5.0 / 3.0]) if nmat else {}
        cfg = sedov(shape, rez, **kw)
        g, o = Sale(cfg, local_slabs=slabs), O.Oracle(cfg)
        if not nmat:
            apply_perturbation([o, g], cfg, 1, lagrange=(rez == LAGRANGE))
        ok = True
        for n in (1, 4, 9):
            rg, ro = g.step(n), o.step(n)
            if rg != ro:
                print("STATUS", rez, shape, slabs, nmat, rg, ro, g.last_error()); ok = False; break
            try:
                compare(g, o)
            except AssertionError as ex:
                print("MISMATCH", rez, shape, slabs, nmat, n, str(ex)[:400]); ok = False; break
        print("ok" if ok else "FAIL", rez, shape, slabs, nmat, g.clock()["cycle"])
        bad += not ok
sys.exit(1 if bad else 0)
