"""Multi-GPU parity (distributed placements over NVLink): runs
tests/gpu_multi_parity.py under torchrun on every visible GPU (needs >= 2)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_multi_gpu_placements():
    import torch
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(root, "tests", "gpu_multi_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "MULTI-GPU PARITY OK" in r.stdout
