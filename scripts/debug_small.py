import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle as O
from paper_2209_01983_b200.configs import sedov, EULER
from paper_2209_01983_b200.sale import Sale
shape = tuple(int(x) for x in sys.argv[1].split(',')) if len(sys.argv) > 1 else (1, 1, 6)
cfg = sedov(shape, EULER)
g, o = Sale(cfg, impl="fused"), O.Oracle(cfg)
for n in range(10):
    rg, ro = g.step(1), o.step(1)
    cg, co = g.clock(), o.clock()
    print(n, "gpu dt %.17g" % cg["dt_last"], "oracle dt %.17g" % co["dt_last"], "ratio to prev", cg["dt_last"])
