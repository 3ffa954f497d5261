import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale
for name in ("C3", "C4"):
    cfg, _ = config(name)
    g = Sale(cfg, impl="v0")
    g.step(2)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.step_async(10); e.record(); print(g.sync())
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    ncell = cfg["nx"]*cfg["ny"]*cfg["nz"]
    print(name, "v0 ms/cycle", ms, "zone-cycles/s %.3e" % (ncell / (ms*1e-3)), g.clock())
    del g; torch.cuda.empty_cache()
