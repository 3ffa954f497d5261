import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import sedov, LAGRANGE, EULER
from paper_2209_01983_b200.sale import Sale
for rez in (LAGRANGE, EULER):
    for shape in ((4, 4, 4), (16, 16, 16), (40, 9, 5)):
        cfg = sedov(shape, rez)
        a, b = Sale(cfg, impl="v0"), Sale(cfg, impl="fused")
        for cyc in range(1, 4):
            ra, rb = a.step(1), b.step(1)
            bad = []
            for f in ("X", "Y", "Z", "UX", "UY", "UZ", "E", "MASS"):
                if rez == EULER and f in "XYZ": continue
                x, y = a.get(f), b.get(f)
                if not np.array_equal(x, y):
                    idx = np.argwhere(x != y)
                    bad.append((f, len(idx), idx[:3].tolist(), float(np.max(np.abs(x - y)))))
            print(rez, shape, cyc, ra, rb, a.clock()["dt_last"], b.clock()["dt_last"], bad[:4])
            if bad: break
