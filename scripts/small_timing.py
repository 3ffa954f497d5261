"""Wall time per cycle of the small configs (launch-bound): python scripts/small_timing.py"""
import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale
for name in ("C0", "C2"):
    cfg, cycles = config(name)
    g = Sale(cfg)
    g.step(5)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 100
    s.record(g.stream); g.step_async(n); e.record(g.stream); rc = g.sync()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    cells = cfg["nx"] * cfg["ny"] * cfg["nz"]
    print(name, "us/cycle %.1f" % (ms * 1e3), "zone-cycles/s %.3e" % (cells / (ms * 1e-3)), rc)
    del g
