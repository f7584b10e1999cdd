"""Serial CPU oracle for the distributed COO-assembled MatMult (arXiv 2406.08646).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs, never by the product package
``paper_2406_08646_b200``.  It shares no code with the CUDA path; the only common module is
``synth`` (seeded inputs, no method arithmetic).

The arithmetic lives in ``oracle.c`` (plain C, ``gcc -O2 -ffp-contract=off``); this file is
ctypes marshalling plus numpy containers.  See the header of oracle.c for the paper
passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

INSERT, ADD = 0, 1
REPLACE, SUM = 0, 1

ORC_OK, ORC_ERR_ARG, ORC_ERR_RANGE, ORC_ERR_STATE = 0, 1, 2, 3

EXPORT = dict(rowptr_d=0, col_d=1, val_d=2, rowptr_o=3, col_o=4, val_o=5, colmap=6, jmap=7,
              csrc=8, ck=9, send_count=10, send_k=11, recv_count=12, leaf_owner=13,
              leaf_offset=14, root_count=15, root_offsets=16)
INFO = dict(rstart=0, rend=1, cstart=2, cend=3, nnz_d=4, nnz_o=5, n_ghost=6, ncontrib=7,
            nsend=8, nroot_offsets=9, n_offdiag_rows=10)


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-pthread",
                               "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            p = ctypes.c_void_p
            i64 = ctypes.c_int64
            L.orc_create_coo.argtypes = [ctypes.c_int, i64, i64, p, p, p, p, p,
                                         ctypes.POINTER(p), ctypes.POINTER(i64),
                                         ctypes.POINTER(i64)]
            L.orc_set_values_coo.argtypes = [p, p, p, ctypes.c_int]
            L.orc_mult.argtypes = [p, p, p]
            L.orc_mult_transpose.argtypes = [p, p, p]
            L.orc_info.argtypes = [p, ctypes.c_int, ctypes.c_int]
            L.orc_info.restype = i64
            L.orc_export.argtypes = [p, ctypes.c_int, ctypes.c_int, p]
            L.orc_export.restype = i64
            L.orc_destroy.argtypes = [p]
            L.orc_sf_bcast.argtypes = [ctypes.c_int, p, p, p, p, p, p, p, p, ctypes.c_int]
            L.orc_sf_reduce.argtypes = [ctypes.c_int, p, p, p, p, p, p, p, p, ctypes.c_int]
            L.orc_sample_rows.argtypes = [i64, p, p, p, i64, p, p, p]
            L.orc_cg.argtypes = [p, p, p, ctypes.c_int, p]
            L.orc_csr_direct.argtypes = [i64, i64, i64, p, p, p, p, p, p, ctypes.POINTER(i64)]
            L.orc_csr_mult.argtypes = [i64, p, p, p, p, p, ctypes.c_int]
            _lib = L
    return _lib


def _np(a, dtype):
    """torch tensor / list / ndarray -> contiguous numpy array of dtype (host)."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


class OracleRangeError(ValueError):
    def __init__(self, rank, k):
        super().__init__(f"COO index out of range on rank {rank} at k={k}")
        self.rank, self.k = rank, k


class OracleMat:
    """P simulated ranks of an MPIAIJ matrix assembled by COO."""

    def __init__(self, M, N, row_sizes, col_sizes, coo_i, coo_j):
        """coo_i/coo_j: list (one per rank) of int64 arrays (negatives = ignored)."""
        self.P = len(row_sizes)
        self.M, self.N = int(M), int(N)
        self.roff = _np(np.concatenate([[0], np.cumsum(row_sizes)]), np.int64)
        self.coff = _np(np.concatenate([[0], np.cumsum(col_sizes)]), np.int64)
        ii = [_np(a, np.int64) for a in coo_i]
        jj = [_np(a, np.int64) for a in coo_j]
        self.cooff = _np(np.concatenate([[0], np.cumsum([a.size for a in ii])]), np.int64)
        gi = _np(np.concatenate(ii) if ii else np.zeros(0), np.int64)
        gj = _np(np.concatenate(jj) if jj else np.zeros(0), np.int64)
        h = ctypes.c_void_p()
        br, bk = ctypes.c_int64(-1), ctypes.c_int64(-1)
        st = lib().orc_create_coo(self.P, self.M, self.N, _ptr(self.roff), _ptr(self.coff),
                                  _ptr(self.cooff), _ptr(gi), _ptr(gj), ctypes.byref(h),
                                  ctypes.byref(br), ctypes.byref(bk))
        if st == ORC_ERR_RANGE:
            raise OracleRangeError(br.value, bk.value)
        if st != ORC_OK:
            raise ValueError(f"oracle create failed: {st}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.orc_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def set_values(self, coo_v, mode=INSERT):
        gv = _np(np.concatenate([_np(a, np.float64) for a in coo_v]) if coo_v else np.zeros(0),
                 np.float64)
        st = lib().orc_set_values_coo(self._h, _ptr(self.cooff), _ptr(gv), int(mode))
        if st != ORC_OK:
            raise ValueError(f"oracle set_values failed: {st}")

    def mult(self, x_global):
        x = _np(x_global, np.float64)
        assert x.size == self.N
        y = np.zeros(self.M, dtype=np.float64)
        st = lib().orc_mult(self._h, _ptr(x), _ptr(y))
        if st != ORC_OK:
            raise ValueError(f"oracle mult failed: {st}")
        return y

    def mult_transpose(self, x_global):
        """y = A^T x (oracle.c orc_mult_transpose): x in the row layout (M), y in the column
        layout (N)."""
        x = _np(x_global, np.float64)
        assert x.size == self.M
        y = np.zeros(self.N, dtype=np.float64)
        st = lib().orc_mult_transpose(self._h, _ptr(x), _ptr(y))
        if st != ORC_OK:
            raise ValueError(f"oracle mult_transpose failed: {st}")
        return y

    def cg(self, b_global, x0_global, maxit):
        """Unpreconditioned CG (oracle.c orc_cg); returns (x, rr_hist)."""
        b = _np(b_global, np.float64)
        x = _np(x0_global, np.float64).copy()
        hist = np.zeros(maxit + 1)
        st = lib().orc_cg(self._h, _ptr(b), _ptr(x), int(maxit), _ptr(hist))
        if st != ORC_OK:
            raise ValueError(f"oracle cg failed: {st}")
        return x, hist

    def info(self, r, key):
        return int(lib().orc_info(self._h, r, INFO[key]))

    def export(self, r, key):
        what = EXPORT[key]
        n = lib().orc_export(self._h, r, what, None)
        dt = np.float64 if key in ("val_d", "val_o") else np.int64
        out = np.zeros(n, dtype=dt)
        if n:
            lib().orc_export(self._h, r, what, _ptr(out))
        return out

    def dense(self):
        """Dense global matrix assembled from the rank blocks (tiny sizes only)."""
        A = np.zeros((self.M, self.N))
        for r in range(self.P):
            rs, cs = self.info(r, "rstart"), self.info(r, "cstart")
            rpd, cd, vd = self.export(r, "rowptr_d"), self.export(r, "col_d"), self.export(r, "val_d")
            rpo, co, vo = self.export(r, "rowptr_o"), self.export(r, "col_o"), self.export(r, "val_o")
            cm = self.export(r, "colmap")
            for q in range(len(rpd) - 1):
                for t in range(rpd[q], rpd[q + 1]):
                    A[rs + q, cs + cd[t]] = vd[t]
                for t in range(rpo[q], rpo[q + 1]):
                    A[rs + q, cm[co[t]]] = vo[t]
        return A


def sf_bcast(nroots, leaves, rootdata, leafdata, op=REPLACE):
    """Graph-walk SF broadcast over P simulated ranks.

    nroots[p]: roots on rank p; leaves[p]: (ilocal or None, remote_rank, remote_offset);
    rootdata[p], leafdata[p]: per-rank arrays.  Returns the new leafdata list."""
    P = len(nroots)
    lv = [len(l[1]) for l in leaves]
    lvoff = _np(np.concatenate([[0], np.cumsum(lv)]), np.int64)
    il = None
    if any(l[0] is not None for l in leaves):
        il = _np(np.concatenate([_np(l[0] if l[0] is not None else np.arange(len(l[1])),
                                     np.int64) for l in leaves]), np.int64)
    rr = _np(np.concatenate([_np(l[1], np.int64) for l in leaves]), np.int64)
    ro = _np(np.concatenate([_np(l[2], np.int64) for l in leaves]), np.int64)
    rd = [_np(a, np.float64) for a in rootdata]
    ld = [_np(a, np.float64).copy() for a in leafdata]
    rdoff = _np(np.concatenate([[0], np.cumsum([a.size for a in rd])]), np.int64)
    ldoff = _np(np.concatenate([[0], np.cumsum([a.size for a in ld])]), np.int64)
    for p in range(P):
        assert rd[p].size >= nroots[p]
    # the oracle validates offsets against the owner's nroots
    rdoff_n = _np(np.concatenate([[0], np.cumsum(nroots)]), np.int64)
    R = _np(np.concatenate(rd) if rd else np.zeros(0), np.float64)
    R2 = np.zeros(int(rdoff_n[-1]))
    for p in range(P):
        R2[rdoff_n[p]:rdoff_n[p + 1]] = rd[p][:nroots[p]]
    Lg = _np(np.concatenate(ld) if ld else np.zeros(0), np.float64)
    st = lib().orc_sf_bcast(P, _ptr(lvoff), _ptr(il) if il is not None else ctypes.c_void_p(0),
                            _ptr(rr), _ptr(ro), _ptr(rdoff_n), _ptr(ldoff), _ptr(R2), _ptr(Lg),
                            int(op))
    del R
    if st != ORC_OK:
        raise ValueError(f"oracle sf_bcast failed: {st}")
    return [Lg[ldoff[p]:ldoff[p + 1]].copy() for p in range(P)]


def sf_reduce(nroots, leaves, leafdata, rootdata, op=SUM):
    """Graph-walk SF reduce (leaf -> root) over P simulated ranks; returns new rootdata.
    leaves[p] = (ilocal or None, remote_rank, remote_offset)."""
    P = len(nroots)
    lv = [len(l[1]) for l in leaves]
    lvoff = _np(np.concatenate([[0], np.cumsum(lv)]), np.int64)
    il = None
    if any(l[0] is not None for l in leaves):
        il = _np(np.concatenate([_np(l[0] if l[0] is not None else np.arange(len(l[1])),
                                     np.int64) for l in leaves]), np.int64)
    rr = _np(np.concatenate([_np(l[1], np.int64) for l in leaves]), np.int64)
    ro = _np(np.concatenate([_np(l[2], np.int64) for l in leaves]), np.int64)
    ld = [_np(a, np.float64) for a in leafdata]
    rd = [_np(a, np.float64).copy() for a in rootdata]
    ldoff = _np(np.concatenate([[0], np.cumsum([a.size for a in ld])]), np.int64)
    rdoff = _np(np.concatenate([[0], np.cumsum(nroots)]), np.int64)
    L = _np(np.concatenate(ld) if ld else np.zeros(0), np.float64)
    R = np.zeros(int(rdoff[-1]))
    for p in range(P):
        R[rdoff[p]:rdoff[p + 1]] = rd[p][:nroots[p]]
    st = lib().orc_sf_reduce(P, _ptr(lvoff), _ptr(il) if il is not None else ctypes.c_void_p(0),
                             _ptr(rr), _ptr(ro), _ptr(rdoff), _ptr(ldoff), _ptr(L), _ptr(R), int(op))
    if st != ORC_OK:
        raise ValueError(f"oracle sf_reduce failed: {st}")
    out = []
    for p in range(P):
        a = rd[p].copy()
        a[:nroots[p]] = R[rdoff[p]:rdoff[p + 1]]
        out.append(a)
    return out


def sample_rows(coo_i, coo_j, coo_v, rows, x_global):
    """y_i for sorted unique sampled rows straight from the COO definition (P=1 order)."""
    gi, gj, gv = _np(coo_i, np.int64), _np(coo_j, np.int64), _np(coo_v, np.float64)
    rows = _np(rows, np.int64)
    x = _np(x_global, np.float64)
    y = np.zeros(rows.size)
    lib().orc_sample_rows(gi.size, _ptr(gi), _ptr(gj), _ptr(gv), rows.size, _ptr(rows),
                          _ptr(x), _ptr(y))
    return y


class OracleCsr:
    """One rank's CSR built directly from a row-sorted, duplicate-free COO (oracle.c
    orc_csr_direct) -- full-size matrices for timing the oracle beside the GPU."""

    def __init__(self, M, N, coo_i, coo_j, coo_v):
        gi, gj, gv = _np(coo_i, np.int64), _np(coo_j, np.int64), _np(coo_v, np.float64)
        self.M, self.N = int(M), int(N)
        nvalid = int(np.count_nonzero((gi >= 0) & (gj >= 0)))
        self.rowptr = np.zeros(self.M + 1, dtype=np.int64)
        self.col = np.zeros(max(nvalid, 1), dtype=np.int64)
        self.val = np.zeros(max(nvalid, 1), dtype=np.float64)
        nnz = ctypes.c_int64(0)
        st = lib().orc_csr_direct(self.M, self.N, gi.size, _ptr(gi), _ptr(gj), _ptr(gv),
                                  _ptr(self.rowptr), _ptr(self.col), _ptr(self.val),
                                  ctypes.byref(nnz))
        if st == ORC_ERR_RANGE:
            raise ValueError("orc_csr_direct: index out of range")
        if st != ORC_OK:
            raise ValueError("orc_csr_direct: COO not in CSR order without duplicates")
        self.nnz = nnz.value

    @classmethod
    def from_oracle(cls, O, r=0):
        """Rank r's diagonal-block CSR of an OracleMat with no off-diagonal block (P=1)."""
        assert O.info(r, "nnz_o") == 0
        C = cls.__new__(cls)
        C.M = O.info(r, "rend") - O.info(r, "rstart")
        C.N = O.info(r, "cend") - O.info(r, "cstart")
        C.rowptr = O.export(r, "rowptr_d")
        C.col = O.export(r, "col_d")
        C.val = O.export(r, "val_d")
        C.nnz = int(C.col.size)
        return C

    def mult(self, x, nthreads=1, out=None):
        x = _np(x, np.float64)
        assert x.size == self.N
        y = out if out is not None else np.zeros(self.M, dtype=np.float64)
        st = lib().orc_csr_mult(self.M, _ptr(self.rowptr), _ptr(self.col), _ptr(self.val),
                                _ptr(x), _ptr(y), int(nthreads))
        if st != ORC_OK:
            raise ValueError(f"orc_csr_mult failed: {st}")
        return y
