"""A/B cycle timing of libsale builds (experiments only): each library in its own
process (SALE_LIB_PATH), alternating, R repeats; CUDA events around n cycles of the
Sedov state after warm-up.
usage: python scripts/ab_time.py C4,C3 lib_a.so lib_b.so ...   (R=2 N=40 env)"""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, torch
sys.path.insert(0, %r)
from paper_2209_01983_b200.configs import config
from paper_2209_01983_b200.sale import Sale
for name in %r:
    cfg, _ = config(name)
    g = Sale(cfg)
    g.step(5)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = %d
    a.record(g.stream); g.step_async(n); b.record(g.stream); rc = g.sync()
    torch.cuda.synchronize()
    print(json.dumps({"cfg": name, "ms": a.elapsed_time(b) / n, "rc": list(rc)}), flush=True)
    del g
    torch.cuda.empty_cache()
'''


def main():
    cfgs = sys.argv[1].split(",")
    libs = sys.argv[2:]
    reps, n = int(os.environ.get("R", "2")), int(os.environ.get("N", "40"))
    res = {}
    for r in range(reps):
        for lib in libs:
            env = dict(os.environ, SALE_LIB_PATH=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfgs, n)], env=env, capture_output=True,
                                 text=True)
            if out.returncode:
                print(lib, "FAILED", out.stderr[-2000:], flush=True)
                continue
            for line in out.stdout.splitlines():
                d = json.loads(line)
                res.setdefault((lib, d["cfg"]), []).append(d["ms"])
                print(r, os.path.basename(lib), d["cfg"], "%.4f ms" % d["ms"], d["rc"], flush=True)
    for (lib, cfg), v in sorted(res.items(), key=lambda x: (x[0][1], x[0][0])):
        print("%-40s %s min %.4f mean %.4f" % (os.path.basename(lib), cfg, min(v), sum(v) / len(v)))


if __name__ == "__main__":
    main()
