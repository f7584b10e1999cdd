"""paper_2406_08646_b200 -- B200-native distributed fp64 MatMult on MPIAIJ with COO assembly.

Thin ctypes binding over the C ABI in ``include/spmat.h`` (``libspmat.so``, built in-tree by
``paper_2406_08646_b200.build``).  Every function here only marshals arguments: all of the
method's work runs in the CUDA kernels and NCCL calls of libspmat.  PyTorch provides device
memory (``torch.Tensor.data_ptr()``), streams (``torch.cuda.Stream.cuda_stream``) and the
process group used to broadcast the NCCL unique id.

There is no CPU fallback: importing the binding without a built ``libspmat.so`` raises.

Names follow the C ABI (and through it the paper's MatSetPreallocationCOO /
MatSetValuesCOO / MatMult / PetscSFBcastBegin/End):

    comm_unique_id, comm_create, comm_check, comm_destroy,
    sf_create, sf_bcast_begin, sf_bcast_end, sf_reduce_begin, sf_reduce_end, sf_get_info, sf_export,
    sf_transport, sf_check, sf_destroy,
    spmat_create_coo, spmat_set_values_coo, spmat_mult, spmat_mult_async, spmat_mult_pipelined,
    spmat_mult_flush, spmat_mult_transpose, spmat_mult_part,
    spmat_get_info, spmat_export, spmat_get_halo_sf, spmat_profile, spmat_profile_read,
    spmat_destroy

plus small RAII wrappers (``Comm``, ``StarForest``, ``Mat``) used by the tests and bench.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPMAT_LIB") or os.path.join(_HERE, "libspmat.so")  # SPMAT_LIB: A/B builds

SPMAT_OK, SPMAT_ERR_ARG, SPMAT_ERR_RANGE, SPMAT_ERR_STATE = 0, 1, 2, 3
SPMAT_ERR_MISMATCH, SPMAT_ERR_OOM, SPMAT_ERR_CUDA, SPMAT_ERR_NCCL = 4, 5, 6, 7
STATUS_NAMES = {0: "OK", 1: "ERR_ARG", 2: "ERR_RANGE", 3: "ERR_STATE", 4: "ERR_MISMATCH",
                5: "ERR_OOM", 6: "ERR_CUDA", 7: "ERR_NCCL"}
INSERT, ADD = 0, 1
REPLACE, SUM = 0, 1
PART_DIAG, PART_HALO, PART_OFFDIAG = 1, 2, 4

EXPORT = dict(rowptr_d=0, col_d=1, val_d=2, rowptr_o=3, col_o=4, val_o=5, colmap=6, jmap=7,
              csrc=8, cpos=9, send_count=10, send_k=11, recv_count=12, rows_o=13)
INFO_KEYS = ("rstart", "rend", "cstart", "cend", "nnz_d", "nnz_o", "n_ghost", "n_offdiag_rows",
             "n_contrib", "n_send", "n_recv", "n_mixed", "spmv_kernel_id", "n_rowblocks",
             "max_row_nnz", "plan_builds", "block_size", "offdiag_3x3", "offdiag_lanes", "halo_mode",
             "nccl_bytes_sent", "nccl_bytes_recv", "nvlink_bytes_put", "n_mult", "n_set_values",
             "spmv_grid", "offdiag_grid", "halo_sf_transport")
SF_INFO_KEYS = ("nroots", "nleaves", "n_send_nbr", "n_recv_nbr", "n_send", "n_recv", "n_self",
                "packed")
SF_EXPORT = dict(recv_ranks=0, recv_counts=1, leaf_idx=2, send_ranks=3, send_counts=4,
                 root_idx=5)

# every symbol include/spmat.h declares (checked by the CPU test suite)
ABI_SYMBOLS = (
    "spmat_version", "spmat_last_error", "spmat_comm_unique_id", "spmat_comm_create",
    "spmat_comm_check", "spmat_comm_destroy", "sf_create", "sf_bcast_begin", "sf_bcast_end",
    "sf_reduce_begin", "sf_reduce_end",
    "sf_get_info", "sf_export", "sf_transport", "sf_check", "sf_destroy", "spmat_create_coo", "spmat_set_values_coo",
    "spmat_mult", "spmat_mult_async", "spmat_mult_pipelined", "spmat_mult_flush", "spmat_mult_transpose", "spmat_mult_part", "spmat_get_info", "spmat_export", "spmat_get_halo_sf",
    "spmat_profile", "spmat_profile_read", "spmat_check", "spmat_halo_mode", "spmat_trace_read",
    "spmat_vec_dot", "spmat_cg", "spmat_set_block_size",
    "spmat_destroy")


class SpmatError(RuntimeError):
    def __init__(self, status, fn, message):
        super().__init__(f"{fn}: {STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


_lib = None


def load(path: str = LIB_PATH):
    """Load libspmat.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `python -m paper_2406_08646_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    p, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    P = ctypes.POINTER
    sig = {
        "spmat_version": ([], i32),
        "spmat_last_error": ([], ctypes.c_char_p),
        "spmat_comm_unique_id": ([p], i32),
        "spmat_comm_create": ([p, i32, i32, i32, P(p)], i32),
        "spmat_comm_check": ([p], i32),
        "spmat_comm_destroy": ([p], i32),
        "sf_create": ([p, i64, i64, p, p, p, P(p)], i32),
        "sf_bcast_begin": ([p, p, p, i32, p], i32),
        "sf_bcast_end": ([p, p, p, i32, p], i32),
        "sf_reduce_begin": ([p, p, p, i32, p], i32),
        "sf_reduce_end": ([p, p, p, i32, p], i32),
        "sf_get_info": ([p, p], i32),
        "sf_export": ([p, i32, p, i64, P(i64)], i32),
        "sf_destroy": ([p], i32),
        "sf_transport": ([p], i32),
        "sf_check": ([p], i32),
        "spmat_create_coo": ([p, i64, i64, i64, i64, i64, p, p, P(p)], i32),
        "spmat_set_values_coo": ([p, p, i32, p], i32),
        "spmat_mult": ([p, p, p, p], i32),
        "spmat_mult_async": ([p, p, p, p], i32),
        "spmat_mult_pipelined": ([p, p, p, p], i32),
        "spmat_mult_flush": ([p, p], i32),
        "spmat_mult_transpose": ([p, p, p, p], i32),
        "spmat_mult_part": ([p, p, p, i32, p], i32),
        "spmat_get_info": ([p, p], i32),
        "spmat_export": ([p, i32, p, i64, P(i64)], i32),
        "spmat_get_halo_sf": ([p, P(p)], i32),
        "spmat_profile": ([p, i32], i32),
        "spmat_profile_read": ([p, p, p], i32),
        "spmat_check": ([p], i32),
        "spmat_halo_mode": ([p], i32),
        "spmat_trace_read": ([p, p, i64, P(i64)], i32),
        "spmat_vec_dot": ([p, p, p, p, p], i32),
        "spmat_cg": ([p, p, p, i32, p, p], i32),
        "spmat_set_block_size": ([p, i32], i32),
        "spmat_destroy": ([p], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status, fn):
    if status != SPMAT_OK:
        msg = load().spmat_last_error()
        raise SpmatError(status, fn, msg.decode() if msg else "")


def _ptr(t):
    """Device or host pointer of a torch tensor / numpy array / int (None -> NULL)."""
    if t is None:
        return ctypes.c_void_p(0)
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    if isinstance(t, np.ndarray):
        return ctypes.c_void_p(t.ctypes.data if t.size else 0)
    return ctypes.c_void_p(t.data_ptr() if t.numel() else 0)


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


# ---------------------------------------------------------------- raw ABI names
def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().spmat_comm_unique_id(buf), "spmat_comm_unique_id")
    return buf.raw


def comm_create(uid, nranks: int, rank: int, device: int):
    h = ctypes.c_void_p()
    idp = ctypes.c_char_p(uid) if uid is not None else None
    _check(load().spmat_comm_create(idp, nranks, rank, device, ctypes.byref(h)), "spmat_comm_create")
    return h


def comm_check(h):
    _check(load().spmat_comm_check(h), "spmat_comm_check")


def comm_destroy(h):
    _check(load().spmat_comm_destroy(h), "spmat_comm_destroy")


def sf_create(comm_h, nroots, nleaves, ilocal, remote_rank, remote_offset):
    h = ctypes.c_void_p()
    _check(load().sf_create(comm_h, int(nroots), int(nleaves), _ptr(ilocal), _ptr(remote_rank),
                            _ptr(remote_offset), ctypes.byref(h)), "sf_create")
    return h


def sf_bcast_begin(sf_h, rootdata, leafdata, op=REPLACE, stream=None):
    _check(load().sf_bcast_begin(sf_h, _ptr(rootdata), _ptr(leafdata), op, _stream(stream)),
           "sf_bcast_begin")


def sf_bcast_end(sf_h, rootdata, leafdata, op=REPLACE, stream=None):
    _check(load().sf_bcast_end(sf_h, _ptr(rootdata), _ptr(leafdata), op, _stream(stream)),
           "sf_bcast_end")


def sf_reduce_begin(sf_h, leafdata, rootdata, op=SUM, stream=None):
    _check(load().sf_reduce_begin(sf_h, _ptr(leafdata), _ptr(rootdata), op, _stream(stream)),
           "sf_reduce_begin")


def sf_reduce_end(sf_h, leafdata, rootdata, op=SUM, stream=None):
    _check(load().sf_reduce_end(sf_h, _ptr(leafdata), _ptr(rootdata), op, _stream(stream)),
           "sf_reduce_end")


def sf_get_info(sf_h) -> dict:
    a = np.zeros(8, dtype=np.int64)
    _check(load().sf_get_info(sf_h, _ptr(a)), "sf_get_info")
    return dict(zip(SF_INFO_KEYS, (int(v) for v in a)))


def sf_export(sf_h, key) -> np.ndarray:
    n = ctypes.c_int64()
    what = SF_EXPORT[key]
    _check(load().sf_export(sf_h, what, None, 0, ctypes.byref(n)), "sf_export")
    out = np.zeros(n.value, dtype=np.int64)
    _check(load().sf_export(sf_h, what, _ptr(out), n.value, ctypes.byref(n)), "sf_export")
    return out


def sf_transport(sf_h) -> int:
    """2: flagged lines over NVLink peer memory, 1: NCCL, 0: single rank."""
    return int(load().sf_transport(sf_h))


def sf_check(sf_h):
    _check(load().sf_check(sf_h), "sf_check")


def sf_destroy(sf_h):
    _check(load().sf_destroy(sf_h), "sf_destroy")


def spmat_create_coo(comm_h, m_local, n_local, M, N, coo_i, coo_j):
    h = ctypes.c_void_p()
    n = int(coo_i.numel() if hasattr(coo_i, "numel") else len(coo_i))
    _check(load().spmat_create_coo(comm_h, int(m_local), int(n_local), int(M), int(N), n,
                                   _ptr(coo_i), _ptr(coo_j), ctypes.byref(h)), "spmat_create_coo")
    return h


def spmat_set_values_coo(A_h, v, mode=INSERT, stream=None):
    _check(load().spmat_set_values_coo(A_h, _ptr(v), mode, _stream(stream)), "spmat_set_values_coo")


def spmat_mult(A_h, x, y, stream=None):
    _check(load().spmat_mult(A_h, _ptr(x), _ptr(y), _stream(stream)), "spmat_mult")


def spmat_mult_async(A_h, x, y, stream=None):
    _check(load().spmat_mult_async(A_h, _ptr(x), _ptr(y), _stream(stream)), "spmat_mult_async")


def spmat_mult_pipelined(A_h, x, y, stream=None):
    _check(load().spmat_mult_pipelined(A_h, _ptr(x), _ptr(y), _stream(stream)), "spmat_mult_pipelined")


def spmat_mult_flush(A_h, stream=None):
    _check(load().spmat_mult_flush(A_h, _stream(stream)), "spmat_mult_flush")


def spmat_mult_transpose(A_h, x, y, stream=None):
    _check(load().spmat_mult_transpose(A_h, _ptr(x), _ptr(y), _stream(stream)), "spmat_mult_transpose")


def spmat_mult_part(A_h, x, y, part, stream=None):
    _check(load().spmat_mult_part(A_h, _ptr(x), _ptr(y), int(part), _stream(stream)),
           "spmat_mult_part")


def spmat_get_info(A_h) -> dict:
    a = np.zeros(32, dtype=np.int64)
    _check(load().spmat_get_info(A_h, _ptr(a)), "spmat_get_info")
    return dict(zip(INFO_KEYS, (int(v) for v in a)))


def spmat_export(A_h, key) -> np.ndarray:
    what = EXPORT[key]
    n = ctypes.c_int64()
    _check(load().spmat_export(A_h, what, None, 0, ctypes.byref(n)), "spmat_export")
    dt = np.float64 if key in ("val_d", "val_o") else np.int64
    out = np.zeros(n.value, dtype=dt)
    _check(load().spmat_export(A_h, what, _ptr(out), n.value, ctypes.byref(n)), "spmat_export")
    return out


def spmat_get_halo_sf(A_h):
    h = ctypes.c_void_p()
    _check(load().spmat_get_halo_sf(A_h, ctypes.byref(h)), "spmat_get_halo_sf")
    return h


def spmat_profile(A_h, enable=True):
    _check(load().spmat_profile(A_h, 1 if enable else 0), "spmat_profile")


def spmat_profile_read(A_h):
    ms = np.zeros(4, dtype=np.float64)
    n = np.zeros(4, dtype=np.int64)
    _check(load().spmat_profile_read(A_h, _ptr(ms), _ptr(n)), "spmat_profile_read")
    return ms, n


def spmat_check(A_h):
    _check(load().spmat_check(A_h), "spmat_check")


def spmat_halo_mode(A_h) -> int:
    return int(load().spmat_halo_mode(A_h))


def spmat_trace_read(A_h) -> np.ndarray:
    n = ctypes.c_int64()
    _check(load().spmat_trace_read(A_h, None, 0, ctypes.byref(n)), "spmat_trace_read")
    out = np.zeros(n.value, dtype=np.int64)
    _check(load().spmat_trace_read(A_h, _ptr(out), n.value, ctypes.byref(n)), "spmat_trace_read")
    return out


def spmat_vec_dot(A_h, a, b, result, stream=None):
    _check(load().spmat_vec_dot(A_h, _ptr(a), _ptr(b), _ptr(result), _stream(stream)),
           "spmat_vec_dot")


def spmat_cg(A_h, b, x, maxit, rr_hist=None, stream=None):
    _check(load().spmat_cg(A_h, _ptr(b), _ptr(x), int(maxit), _ptr(rr_hist), _stream(stream)),
           "spmat_cg")


def spmat_destroy(A_h):
    _check(load().spmat_destroy(A_h), "spmat_destroy")


# ---------------------------------------------------------------- RAII wrappers
class Comm:
    """One rank's communicator.  With torch.distributed initialised and world size > 1,
    rank 0 draws the NCCL unique id and broadcasts it over the default process group."""

    def __init__(self, device: int | None = None, nranks: int | None = None, rank: int | None = None,
                 uid: bytes | None = None):
        import torch
        import torch.distributed as dist
        if nranks is None:
            if dist.is_available() and dist.is_initialized():
                nranks, rank = dist.get_world_size(), dist.get_rank()
            else:
                nranks, rank = 1, 0
        if device is None:
            device = torch.cuda.current_device()
        if nranks > 1 and uid is None:
            from . import dist as _d
            uid = _d.share_unique_id(comm_unique_id)
        self.nranks, self.rank, self.device = nranks, rank, device
        self.h = comm_create(uid, nranks, rank, device)

    def check(self):
        comm_check(self.h)

    def close(self):
        if getattr(self, "h", None) is not None:
            comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StarForest:
    def __init__(self, comm: Comm, nroots, ilocal, remote_rank, remote_offset, nleaves=None):
        rr = np.ascontiguousarray(np.asarray(remote_rank, dtype=np.int32))
        ro = np.ascontiguousarray(np.asarray(remote_offset, dtype=np.int64))
        il = None if ilocal is None else np.ascontiguousarray(np.asarray(ilocal, dtype=np.int64))
        self.comm = comm
        self.h = sf_create(comm.h, nroots, len(rr) if nleaves is None else nleaves, il, rr, ro)

    def bcast_begin(self, root, leaf, op=REPLACE, stream=None):
        sf_bcast_begin(self.h, root, leaf, op, stream)

    def bcast_end(self, root, leaf, op=REPLACE, stream=None):
        sf_bcast_end(self.h, root, leaf, op, stream)

    def reduce_begin(self, leaf, root, op=SUM, stream=None):
        sf_reduce_begin(self.h, leaf, root, op, stream)

    def reduce_end(self, leaf, root, op=SUM, stream=None):
        sf_reduce_end(self.h, leaf, root, op, stream)

    def info(self):
        return sf_get_info(self.h)

    def export(self, key):
        return sf_export(self.h, key)

    def transport(self):
        return sf_transport(self.h)

    def check(self):
        sf_check(self.h)

    def close(self):
        if getattr(self, "h", None) is not None:
            sf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Mat:
    """MPIAIJ matrix assembled by COO on the device (MatSetPreallocationCOO)."""

    def __init__(self, comm: Comm, m_local, n_local, M, N, coo_i, coo_j):
        self.comm = comm
        self.m, self.n, self.M, self.N = int(m_local), int(n_local), int(M), int(N)
        self.h = spmat_create_coo(comm.h, m_local, n_local, M, N, coo_i, coo_j)

    def set_values(self, v, mode=INSERT, stream=None):
        spmat_set_values_coo(self.h, v, mode, stream)

    def mult(self, x, y, stream=None):
        spmat_mult(self.h, x, y, stream)

    def mult_async(self, x, y, stream=None):
        """spmat_mult_async: enqueue only, also for (pinned) host x / y."""
        spmat_mult_async(self.h, x, y, stream)

    def mult_pipelined(self, x, y, stream=None):
        """spmat_mult_pipelined: enqueue only; y complete after the next call or flush()."""
        spmat_mult_pipelined(self.h, x, y, stream)

    def flush(self, stream=None):
        spmat_mult_flush(self.h, stream)

    def mult_transpose(self, x, y, stream=None):
        spmat_mult_transpose(self.h, x, y, stream)

    def mult_part(self, x, y, part, stream=None):
        spmat_mult_part(self.h, x, y, part, stream)

    def info(self):
        return spmat_get_info(self.h)

    def export(self, key):
        return spmat_export(self.h, key)

    def halo_sf(self):
        return spmat_get_halo_sf(self.h)

    def check(self):
        spmat_check(self.h)

    def set_block_size(self, bs):
        _check(load().spmat_set_block_size(self.h, int(bs)), "spmat_set_block_size")

    def dot(self, a, b, result, stream=None):
        spmat_vec_dot(self.h, a, b, result, stream)

    def cg(self, b, x, maxit, rr_hist=None, stream=None):
        spmat_cg(self.h, b, x, maxit, rr_hist, stream)

    def halo_mode(self):
        return spmat_halo_mode(self.h)

    def profile(self, enable=True):
        spmat_profile(self.h, enable)

    def profile_read(self):
        return spmat_profile_read(self.h)

    def close(self):
        if getattr(self, "h", None) is not None:
            spmat_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
