import sys
sys.path.insert(0, "/root/repo")
from paper_2209_01983_b200.configs import sedov, EULER
from paper_2209_01983_b200.sale import Sale
g = Sale(sedov((12, 10, 9), EULER))
print(g.step(1), flush=True)
print(g.step(3), flush=True)
