"""S10 fused into K1 across PROCESSES: two ranks on one GPU exchange their partials through
CUDA-IPC-mapped buffers (smcsd_tp_step, the product TP path; no collective call), with gloo only
for the handle plumbing.  Runs scripts/tp_multiproc.py under torchrun: every rank must get
bit-identical log-weights and ancestors, within 1e-4 of the unsharded smcsd_step, status 0."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tp_step_two_processes_ipc():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561",
           os.path.join(ROOT, "scripts", "tp_multiproc.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert out.count(" OK") == 2, out[-3000:]
    assert "identical across ranks False" not in out
