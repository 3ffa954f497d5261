"""Cycle time of C4 / C3 from a fully active state (seeded perturbation P0: every node
moving, every cell's energy scaled) next to the Sedov state: the Sedov bulk is
quiescent (zero velocity jumps, forces, swept volumes), where the exact zero-operand
shortcuts of division and square root apply.  python scripts/dense_timing.py"""
import json, sys, torch
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import config, LAGRANGE
from paper_2209_01983_b200.sale import Sale
from tests.helpers import apply_perturbation
for name in ("C4", "C3"):
    for dense in (False, True):
        cfg, _ = config(name)
        g = Sale(cfg)
        if dense:
            apply_perturbation([g], cfg, 0, lagrange=(cfg["rezone"] == LAGRANGE))
        g.step(3)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 30
        a.record(g.stream); g.step_async(n); b.record(g.stream); rc = g.sync()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        cells = cfg["nx"] * cfg["ny"] * cfg["nz"]
        print(json.dumps({"workload": name, "state": "perturbed P0 (all active)" if dense else "Sedov",
                          "ms_per_cycle": ms, "zone_cycles_per_s": cells / (ms * 1e-3), "rc": rc}), flush=True)
        del g
        torch.cuda.empty_cache()
