"""Multi-rank GPU parity: launches tests/mp_gpu_parity.py with torchrun on P GPUs (NCCL
bootstrap), once per halo transport (device-initiated NVLink stores, and NCCL send/recv);
P = 3 exercises uneven z-slabs (the low ranks take the remainder planes)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("halo", ["peer", "nccl"])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_multirank_parity(P, halo):
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    env = dict(os.environ)
    env["SPMAT_HALO"] = halo
    port = 29611 + P + (0 if halo == "peer" else 20)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(HERE, "mp_gpu_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    sys.stdout.write(r.stdout[-6000:])
    sys.stderr.write(r.stderr[-6000:])
    assert r.returncode == 0
    assert f"MULTIRANK P={P} failures=0" in r.stdout
    want = 2 if halo == "peer" else 1
    assert f"halo_mode={want}" in r.stdout


@pytest.mark.parametrize("ro_w,fuse", [("1", "1"), ("32", "1"), ("1", "0"), ("8", "0")])
def test_multirank_offdiag_lanes(ro_w, fuse):
    """The off-diagonal SpMV-add with forced lanes per row (1: plain row sums, 32: one warp per
    row), fused into the SpMV kernel's comm warps or (SPMAT_FUSE_TAIL=0) as the standalone
    NVLink kernel."""
    P = 2
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    env = dict(os.environ)
    env["SPMAT_RO_W"] = ro_w
    env["SPMAT_FUSE_TAIL"] = fuse
    env["SPMAT_SPMV_KERNEL"] = "tma"  # the small cases would take the one-launch direct kernel
    port = 29661 + int(ro_w) + 40 * int(fuse)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(HERE, "mp_gpu_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    sys.stdout.write(r.stdout[-6000:])
    sys.stderr.write(r.stderr[-6000:])
    assert r.returncode == 0
    assert f"MULTIRANK P={P} failures=0" in r.stdout


ENV3 = [{"SPMAT_BSR_FUSE": "1"}, {"SPMAT_BSR_FUSE": "0", "SPMAT_OB_W": "1"},
        {"SPMAT_BSR_FUSE": "0", "SPMAT_OB_W": "8"}, {"SPMAT_BSR_OFFDIAG": "0"}, {"SPMAT_HALO": "nccl"},
        {"SPMAT_BSR_FMA": "0"}]


@pytest.mark.parametrize("k", range(len(ENV3)))
def test_multirank_offdiag_3x3(k):
    """3x3 off-diagonal blocks: by the block SpMV's comm warps (default), by its consumers
    (SPMAT_BSR_FUSE=1), by the standalone kernel (SPMAT_BSR_FUSE=0) with forced lanes per block
    row, switched off (CSR off-diagonal kernels), on the NCCL ghost vector, and with separately
    rounded products in the block SpMV -- elasticity cases (real and integer) and full-size C5."""
    env = ENV3[k]
    P = 2
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    e = dict(os.environ)
    e.update(env)
    e["MP_CASES"] = "elasticity,full-c5"
    port = 29721 + k
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(HERE, "mp_gpu_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=e)
    sys.stdout.write(r.stdout[-6000:])
    sys.stderr.write(r.stderr[-6000:])
    assert r.returncode == 0
    assert f"MULTIRANK P={P} failures=0" in r.stdout
    assert "PASS full-c5" in r.stdout


@pytest.mark.parametrize("split", ["1", "0"])
def test_multirank_tma_tails(split):
    """The bulk-copy SpMV with its fused off-diagonal tail on every small case (they default to
    the one-launch direct kernel): the split tail (sums during the sweep, add pass after; the
    default for box partitions) forced on, and the boundary-first tail forced on."""
    P = 2
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    env = dict(os.environ)
    env["SPMAT_SPMV_KERNEL"] = "tma"
    env["SPMAT_SPLIT_TAIL"] = split
    env["MP_CASES"] = "stencil,q1,elasticity,random,box"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={29731 + int(split)}", os.path.join(HERE, "mp_gpu_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    sys.stdout.write(r.stdout[-6000:])
    sys.stderr.write(r.stderr[-6000:])
    assert r.returncode == 0
    assert f"MULTIRANK P={P} failures=0" in r.stdout


def test_multirank_nccl_board():
    """CG and the device dots with the cross-rank scalar sum over ncclAllReduce instead of the
    NVLink scalar board (SPMAT_BOARD=nccl)."""
    P = 2
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    env = dict(os.environ)
    env["SPMAT_BOARD"] = "nccl"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", "--master-port=29651", os.path.join(HERE, "mp_gpu_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    sys.stdout.write(r.stdout[-6000:])
    sys.stderr.write(r.stderr[-6000:])
    assert r.returncode == 0
    assert f"MULTIRANK P={P} failures=0" in r.stdout


def test_multirank_sf_bulk_protocol():
    """Star-forest segments of >= 4 values take the bulk protocol (plain doubles + per-chunk
    release flags) instead of flagged lines (SPMAT_SF_BULK_MIN=4; the default is 2^21)."""
    P = 2
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    env = dict(os.environ)
    env["SPMAT_SF_BULK_MIN"] = "4"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", "--master-port=29652", os.path.join(HERE, "mp_gpu_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    sys.stdout.write(r.stdout[-6000:])
    sys.stderr.write(r.stderr[-6000:])
    assert r.returncode == 0
    assert f"MULTIRANK P={P} failures=0" in r.stdout
