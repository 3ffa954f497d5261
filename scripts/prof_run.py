"""Small fixed workload for ncu captures: N cycles of a config with one impl."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
impl = sys.argv[2] if len(sys.argv) > 2 else "fused"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg, _ = config(name)
g = Sale(cfg, impl=impl)
rc = g.step(n)
print(name, impl, rc, g.clock())
assert rc == (0, n)
