"""Bitwise comparison of sale_steinberg's outputs between two library builds (experiments
only; e.g. the thread-per-cell Lagrange kernel of commit 99c0249 vs k_steinberg_zl): C3 after 3
cycles, a perturbed 2-slab Lagrangian mesh, a 2-material mesh; with and without a strain
field.  usage: python scripts/steinberg_bits_ab.py lib_a.so lib_b.so"""
import os, subprocess, sys, numpy as np
CH = r'''
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2209_01983_b200.configs import config, sedov, LAGRANGE
from paper_2209_01983_b200.sale import Sale
from paper_2209_01983_b200 import inputs
prm = dict(G0=0.43, GP=1.7, GT=0.3, Y0=0.2, Ymax=0.9, beta=3.0, n=0.5, cv=0.8, rho0=1.1, T0=0.05)
out = {}
for name, cfg in (("C3", config("C3")[0]), ("P", sedov((37, 23, 29), LAGRANGE, e_background=0.3)),
                  ("M", sedov((21, 17, 19), LAGRANGE, nmat=2, mat_gamma=[1.4, 1.6]))):
    g = Sale(cfg, local_slabs=2 if name == "P" else 1)
    if name == "P":  # the seeded perturbed state P3 (inputs.perturbation), applied to the GPU state itself
        pert = inputs.perturbation(cfg, 3)
        for f, d in (("X", "dx"), ("Y", "dy"), ("Z", "dz")):
            g.set(f, g.get(f) + pert[d])
        for f in ("UX", "UY", "UZ"):
            g.set(f, pert[f.lower()])
        g.set("E", g.get("E") * pert["e_factor"])
    g.step(3)
    eps = torch.rand(g.cell_shape, dtype=torch.float64, device=g.torch_device, generator=torch.Generator(device="cuda").manual_seed(1))
    for tag, e in (("f", eps), ("n", None)):
        sh, yl = g.steinberg([prm, dict(prm, G0=0.5)] if cfg.get("nmat") else prm, e)
        out[name + tag + "s"] = sh.cpu().numpy() if hasattr(sh, "cpu") else np.asarray(sh)
        out[name + tag + "y"] = yl.cpu().numpy() if hasattr(yl, "cpu") else np.asarray(yl)
    del g; torch.cuda.empty_cache()
np.savez(sys.argv[1], **out)
'''
res = []
for lib in sys.argv[1:]:
    f = "/tmp/" + os.path.basename(lib) + ".npz"
    r = subprocess.run([sys.executable, "-c", CH, f], env=dict(os.environ, SALE_LIB_PATH=os.path.abspath(lib)), capture_output=True, text=True)
    if r.returncode: print(r.stderr[-3000:]); sys.exit(1)
    res.append(np.load(f))
a, b = res
bad = 0
for k in a.files:
    eq = np.array_equal(a[k].view(np.int64), b[k].view(np.int64))
    print(k, a[k].shape, "bitwise" if eq else "DIFF max %g" % np.max(np.abs(a[k] - b[k])))
    bad += not eq
sys.exit(1 if bad else 0)
