"""Row-sharded checkpoint on 2+ GPUs (NCCL) vs the single-process oracle payload.

Skipped on a one-GPU box; run with `gpurun --gpus 2 -- python -m pytest
tests/test_multi_gpu.py -m gpu`.
"""
import os
import subprocess
import sys

import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ("peer", "nccl"))
@pytest.mark.parametrize("bitwidth", ("8", "4", "fp32"))
def test_row_sharded_payload_matches_oracle(bitwidth, exchange):
    """Three checkpoint intervals (one staged) per run; the count exchange over
    NVLink peer memory (default) and the NCCL all_gather."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    env = dict(os.environ, DS_COUNTS_EXCHANGE=exchange)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 4)}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + int(os.getpid()) % 1000),
           os.path.join(HERE, "multi_gpu_worker.py"), bitwidth]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
