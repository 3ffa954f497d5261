"""Small fixed workload for ncu captures: N cycles of a config (python scripts/prof_run.py C4 5)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg, _ = config(name)
g = Sale(cfg)
rc = g.step(n)
print(name, rc, g.clock())
assert rc == (0, n)
