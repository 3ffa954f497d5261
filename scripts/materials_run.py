"""A few cycles of C4 with 2 (or argv[1]) mixed materials, for ncu launch lists."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale
nmat = int(sys.argv[1]) if len(sys.argv) > 1 else 2
name = sys.argv[2] if len(sys.argv) > 2 else "C4"
cfg, _ = config(name)
g = Sale(dict(cfg, nmat=nmat, mat_gamma=[1.4, 5.0 / 3.0, 1.2, 2.0][:nmat]))
m, e = g.get("MAT_M0"), g.get("MAT_E0")
for k in range(nmat):
    g.set(f"MAT_F{k}", np.full(g.cell_shape, 1.0 / nmat))
    g.set(f"MAT_M{k}", m / nmat)
    g.set(f"MAT_E{k}", e)
rc, done = g.step(4)
assert rc == 0, g.last_error()
print("ok", done)
