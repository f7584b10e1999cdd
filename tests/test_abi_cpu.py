"""The C-ABI boundary without a GPU: libspmat.so builds, loads, and exports every function
include/spmat.h declares; the binding names match; the product package never touches the
oracle; and without a device the library reports errors instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spmat.h")
PKG = os.path.join(ROOT, "paper_2406_08646_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while")))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_08646_b200 import build
    path = build.build()
    return path


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("spmat_create_coo", "spmat_set_values_coo", "spmat_mult", "sf_bcast_begin",
                 "sf_bcast_end", "sf_create", "spmat_comm_create"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_binding_matches_header(lib):
    import paper_2406_08646_b200 as sp
    assert sorted(sp.ABI_SYMBOLS) == declared_functions()
    L = sp.load()
    for n in sp.ABI_SYMBOLS:
        assert getattr(L, n) is not None
    assert L.spmat_version() >= 100


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2406_08646_b200 as sp
    with pytest.raises(sp.SpmatError) as e:
        sp.comm_create(None, 1, 0, 0)
    assert e.value.status in (sp.SPMAT_ERR_CUDA, sp.SPMAT_ERR_ARG)
    # null-handle calls are argument errors, never crashes
    L = sp.load()
    assert L.spmat_mult(None, None, None, None) == sp.SPMAT_ERR_ARG
    assert L.sf_bcast_end(None, None, None, 0, None) == sp.SPMAT_ERR_ARG


def test_product_path_never_uses_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, flags=re.M), f
                assert "liboracle" not in txt and "oracle.c" not in txt, f
    hdr = open(HEADER).read()
    assert "oracle" not in hdr.lower()


def test_oracle_shares_nothing_with_the_cuda_path():
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    assert "#include \"" not in src  # only system headers
    assert "spmat" not in src
