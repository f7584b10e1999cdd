"""Multi-rank GPU parity: launches tests/mp_gpu_parity.py with torchrun on P GPUs (NCCL)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_multirank_parity(P):
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", "--master-port=29611", os.path.join(HERE, "mp_gpu_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    sys.stdout.write(r.stdout[-6000:])
    sys.stderr.write(r.stderr[-6000:])
    assert r.returncode == 0
    assert f"MULTIRANK P={P} failures=0" in r.stdout
