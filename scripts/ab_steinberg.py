"""A/B of sale_steinberg across library builds (experiments only): each library in its own
process (SALE_LIB_PATH), the steinberg_bench lines.  usage: python scripts/ab_steinberg.py lib_a.so lib_b.so ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sys.argv[1:]:
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "steinberg_bench.py")], capture_output=True,
                         text=True, env=dict(os.environ, SALE_LIB_PATH=os.path.abspath(lib)))
    for line in out.stdout.splitlines():
        print(os.path.basename(lib), line[:110], flush=True)
