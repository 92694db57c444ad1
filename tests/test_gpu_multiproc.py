"""Cross-process pipeline (torchrun, two ranks, CUDA-IPC mailboxes, shm flags,
latency gate, cross-process delegated host ring) vs the oracle's full-batch
gradients.  With two GPUs the ranks sit on different GPUs (NVLink) and the
NCCL baseline arms (N1) run too; with one GPU both ranks share cuda:0, which
still exercises every cross-process path of the transport."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", [0, 1])
def test_two_rank_pipeline_matches_oracle(mode):
    n = torch.cuda.device_count()
    env = dict(os.environ, S="4", N="8", MODE=str(mode))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + mode), os.path.join(ROOT, "scripts/mp_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert "FAIL" not in r.stdout
    assert r.stdout.count("OK") == (18 if n >= 2 else 8)
