"""Multi-rank runs of the sharded axes through tests/mgpu_worker.py under
torchrun: DP bit-identity against a single-device run, fused-TP cross-rank identity and oracle
parity, and (one GPU per rank) the NCCL all-gather form.

* test_multigpu_ranks_own_devices: min(8, device_count) ranks, one GPU each (real NVLink P2P
  between the ranks' exchange buffers); skipped on a box with fewer than 2 GPUs.
* test_two_ranks_share_one_gpu: 2 ranks on cuda:0 (CUDA IPC between processes, time-sliced);
  runs on any GPU box, so the worker itself is exercised every round."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(nproc, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={**os.environ, **(env or {})})
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(" OK (device") == nproc, out[-4000:]
    return out


def test_multigpu_ranks_own_devices():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip(f"{n} GPU on this box: the one-device-per-rank run needs >= 2")
    out = _launch(min(8, n))
    for r in range(min(8, n)):
        assert f"device cuda:{r}" in out


def test_two_ranks_share_one_gpu():
    out = _launch(2, env={"CUDA_VISIBLE_DEVICES": os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]})
    assert out.count("device cuda:0") == 2
