"""The NCCL code path of the row bands (process group, grouped send/recv,
overlapped interior/edge launches, miss all-reduce, all-gather) under
torchrun on the GPUs present (N = 1 here: no peer, but every collective
and launch path runs), bitwise equal to the whole-frame session."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_nccl_band_path(cuda_dev):
    n = torch.cuda.device_count()
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(root, "tests", "helpers", "nccl_band_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
