import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import sedov, LAGRANGE, EULER
from paper_2209_01983_b200.sale import Sale
for shape in ((4, 4, 4), (16, 16, 16), (40, 9, 5)):
    for n in (2, 3):
        cfg = sedov(shape, LAGRANGE)
        a, b = Sale(cfg, impl="v0"), Sale(cfg, impl="fused")
        ra, rb = a.step(n), b.step(n)
        print(shape, n, ra, rb, a.clock()["dt_last"], b.clock()["dt_last"], b.clock()["dt_last"]/a.clock()["dt_last"])
