"""Build libsale.so in-tree with nvcc for sm_100a (B200).

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false.
-fmad=false keeps every a*b+c as a separate DMUL/DADD so results are
bit-identical to the operation order of SURVEY §8(c); div/sqrt stay IEEE
(-prec-div/-prec-sqrt default true); never -use_fast_math.
NCCL comes from the torch-bundled nvidia/nccl package (rpath-linked).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libsale.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in spec.submodule_search_locations:
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl headers not found under the nvidia package")


def flags():
    inc, _ = nccl_dirs()
    fmad = os.environ.get("SALE_FMAD", "false")
    return ARCH + ["-O3", "-lineinfo", f"-fmad={fmad}", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]


def _compile(src: str, obj: str, verbose: bool) -> str:
    cmd = [NVCC, *flags(), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return r.stderr if verbose else ""


STAMP = os.path.join(LIBDIR, "libsale.stamp")


def _stamp() -> str:
    """The compile configuration the library was built with (nvcc, flags, sources): a
    library built under other flags (e.g. SALE_FMAD=true, which breaks the bitwise
    parity with the oracle) is rebuilt, never silently reused."""
    srcs = sorted(os.path.basename(s) for s in glob.glob(os.path.join(CSRC, "*.cu")))
    return "\n".join([NVCC, " ".join(flags()), " ".join(srcs)])


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "sale.h"), __file__]
    newest = max(os.path.getmtime(d) for d in deps)
    stamp = _stamp()
    same = os.path.exists(STAMP) and open(STAMP).read() == stamp
    if not force and same and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    os.makedirs(os.path.join(LIBDIR, "obj"), exist_ok=True)
    objs = [os.path.join(LIBDIR, "obj", os.path.basename(s)[:-3] + ".o") for s in srcs]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        logs = list(ex.map(lambda a: _compile(a[0], a[1], verbose), zip(srcs, objs)))
    if verbose:
        for lg in logs:
            sys.stderr.write(lg)
    _, libdir = nccl_dirs()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{libdir}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(stamp)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
