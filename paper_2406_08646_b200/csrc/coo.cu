// coo.cu -- device COO assembly: MatSetPreallocationCOO / MatSetValuesCOO.
//
// Symbolic (spmat_create_coo), all on the device except the tiny per-rank
// count vectors:
//   1. classify every entry k: ignored (i<0 or j<0), range error, or owner rank
//   2. stable radix sort of (owner, k) -> per-destination k lists; the off-rank ones are the
//      COO send plan ("destined for ... a send buffer")
//   3. NCCL exchange of the (i, j) of off-rank entries ("exchanges information about remote
//      entries")
//   4. contributions in canonical (src rank, k) order -> 64-bit key (i - rstart) * N + j;
//      stable LSD radix sort by key keeps (src, k) order inside equal keys (reading Z1)
//   5. run-length heads -> nonzeros; diag / offdiag split by column ownership;
//      CSR row pointers; colmap = sorted unique ghost columns; jmap/perm per block
//   6. the halo SF from colmap
// Numeric (spmat_set_values_coo): gather the send buffer, start the NCCL value
// exchange on the comm stream, then one thread per nonzero sums its contribution segment
// ("each thread accumulates into a single nonzero entry", no atomics).  Nonzeros
// whose segment contains received values are finished after the exchange, still in
// canonical order, so the result is bit-identical to a serial sum in (src, k) order.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <memory>

#include "internal.h"

namespace spmat {

// ------------------------------------------------------------------ helpers
struct Tmp {
  DevBuf<char> buf;
  int ensure(size_t bytes) {
    if (bytes <= buf.n) return SPMAT_OK;
    return buf.alloc(bytes);
  }
};

#define CUB_CALL(tmp, stream, call_with_tmp)                                       \
  do {                                                                             \
    size_t _bytes = 0;                                                             \
    void *d_temp_storage = nullptr;                                                \
    size_t &temp_storage_bytes = _bytes;                                           \
    SP_CUDA(call_with_tmp);                                                        \
    SP_TRY((tmp).ensure(_bytes));                                                  \
    d_temp_storage = (tmp).buf.get();                                              \
    SP_CUDA(call_with_tmp);                                                        \
  } while (0)

static inline unsigned nblk(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)1 << 30));
}

static inline int bits_for(uint64_t maxval) {  // bits needed to represent 0..maxval
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return std::max(b, 1);
}

#define GRID_STRIDE(t, n) \
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (n); t += (int64_t)gridDim.x * blockDim.x)

// ------------------------------------------------------------------ symbolic kernels
__global__ void k_classify(const int64_t *__restrict__ ci, const int64_t *__restrict__ cj,
                           int64_t n, int64_t M, int64_t N, const int64_t *__restrict__ roff,
                           int P, uint32_t *__restrict__ dest,
                           unsigned long long *__restrict__ bad_k) {
  GRID_STRIDE(k, n) {
    int64_t i = ci[k], j = cj[k];
    uint32_t d = (uint32_t)P;  // P = dropped
    if (i >= 0 && j >= 0) {
      if (i >= M || j >= N) {
        atomicMin(bad_k, (unsigned long long)k);
      } else {  // owner: largest r with roff[r] <= i (upper bound - 1)
        int lo = 0, hi = P;  // invariant: roff[lo] <= i < roff[hi]
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (roff[mid] <= i) lo = mid; else hi = mid;
        }
        d = (uint32_t)lo;
      }
    }
    dest[k] = d;
  }
}

__global__ void k_iota(uint32_t *__restrict__ out, int64_t n) {
  GRID_STRIDE(t, n) out[t] = (uint32_t)t;
}

// dofs[d] = lower_bound(sorted, d) for d = 0..P+1
__global__ void k_bounds(const uint32_t *__restrict__ sorted, int64_t n, int P,
                         int64_t *__restrict__ dofs) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d > P + 1) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < (uint32_t)d) lo = mid + 1; else hi = mid;
  }
  dofs[d] = lo;
}

__global__ void k_gather_ij(const int64_t *__restrict__ ci, const int64_t *__restrict__ cj,
                            const uint32_t *__restrict__ ks, int64_t n,
                            longlong2 *__restrict__ out) {
  GRID_STRIDE(t, n) {
    uint32_t k = ks[t];
    out[t] = make_longlong2(ci[k], cj[k]);
  }
}

// received entries: recv position t -> canonical position; value index = ncoo + t
__global__ void k_keys_recv(const longlong2 *__restrict__ rij, int64_t nrecv, int64_t before,
                            int64_t nlocal, int64_t rstart, int64_t N, uint64_t ncoo,
                            uint64_t *__restrict__ key, uint32_t *__restrict__ val) {
  GRID_STRIDE(t, nrecv) {
    longlong2 e = rij[t];
    int64_t pos = t < before ? t : t + nlocal;
    key[pos] = (uint64_t)(e.x - rstart) * (uint64_t)N + (uint64_t)e.y;
    val[pos] = (uint32_t)(ncoo + (uint64_t)t);
  }
}

__global__ void k_keys_local(const int64_t *__restrict__ ci, const int64_t *__restrict__ cj,
                             const uint32_t *__restrict__ ks, int64_t nlocal, int64_t before,
                             int64_t rstart, int64_t N, uint64_t *__restrict__ key,
                             uint32_t *__restrict__ val) {
  GRID_STRIDE(u, nlocal) {
    uint32_t k = ks[u];
    key[before + u] = (uint64_t)(ci[k] - rstart) * (uint64_t)N + (uint64_t)cj[k];
    val[before + u] = k;
  }
}

__global__ void k_heads(const uint64_t *__restrict__ key, int64_t n, uint32_t *__restrict__ head) {
  GRID_STRIDE(t, n) head[t] = (t == 0 || key[t] != key[t - 1]) ? 1u : 0u;
}

// per nonzero z (segment start s = segstart[z]): row, column, block, row counts
__global__ void k_nz_classify(const uint64_t *__restrict__ key, const uint32_t *__restrict__ segstart,
                              int64_t nnz, int64_t N, int64_t cstart, int64_t cend,
                              uint32_t *__restrict__ isdiag, int32_t *__restrict__ cnt_d,
                              int32_t *__restrict__ cnt_o) {
  GRID_STRIDE(z, nnz) {
    uint64_t kk = key[segstart[z]];
    int64_t row = (int64_t)(kk / (uint64_t)N), col = (int64_t)(kk % (uint64_t)N);
    bool d = col >= cstart && col < cend;
    isdiag[z] = d ? 1u : 0u;
    atomicAdd(d ? &cnt_d[row] : &cnt_o[row], 1);
  }
}

__global__ void k_nz_cols(const uint64_t *__restrict__ key, const uint32_t *__restrict__ segstart,
                          const uint32_t *__restrict__ isdiag, const uint32_t *__restrict__ pos_d,
                          int64_t nnz, int64_t N, int64_t cstart, int32_t *__restrict__ col_d,
                          int64_t *__restrict__ ocol) {
  GRID_STRIDE(z, nnz) {
    uint64_t kk = key[segstart[z]];
    int64_t col = (int64_t)(kk % (uint64_t)N);
    if (isdiag[z]) col_d[pos_d[z]] = (int32_t)(col - cstart);
    else ocol[z - pos_d[z]] = col;
  }
}

__global__ void k_ghost_index(const int64_t *__restrict__ ocol, int64_t nnz_o,
                              const int64_t *__restrict__ colmap, int64_t ng,
                              int32_t *__restrict__ col_o) {
  GRID_STRIDE(t, nnz_o) {
    int64_t c = ocol[t], lo = 0, hi = ng;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (colmap[mid] < c) lo = mid + 1; else hi = mid;
    }
    col_o[t] = (int32_t)lo;
  }
}

// contribution t belongs to nonzero zid1[t] - 1 (zid1 = inclusive scan of run heads);
// flag whether that nonzero is diagonal
__global__ void k_cflag(const uint32_t *__restrict__ zid1, const uint32_t *__restrict__ isdiag,
                        int64_t n, uint32_t *__restrict__ cflag) {
  GRID_STRIDE(t, n) cflag[t] = isdiag[zid1[t] - 1];
}

__global__ void k_perm(const uint32_t *__restrict__ val, const uint32_t *__restrict__ cflag,
                       const uint32_t *__restrict__ cpos_d, int64_t n, int64_t total_d,
                       uint32_t *__restrict__ perm) {
  GRID_STRIDE(t, n) {
    int64_t at = cflag[t] ? (int64_t)cpos_d[t] : total_d + (t - (int64_t)cpos_d[t]);
    perm[at] = val[t];
  }
}

__global__ void k_jmap(const uint32_t *__restrict__ segstart, const uint32_t *__restrict__ isdiag,
                       const uint32_t *__restrict__ pos_d, const uint32_t *__restrict__ cpos_d,
                       int64_t nnz, int64_t nnz_d, int64_t total_d, int64_t nt,
                       uint32_t *__restrict__ jmap) {
  GRID_STRIDE(z, nnz) {
    int64_t s = segstart[z];
    if (isdiag[z]) jmap[pos_d[z]] = cpos_d[s];
    else jmap[nnz_d + (z - pos_d[z])] = (uint32_t)(total_d + (s - (int64_t)cpos_d[s]));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) jmap[nnz] = (uint32_t)nt;
}

__global__ void k_mixed_flag(const uint32_t *__restrict__ jmap, const uint32_t *__restrict__ perm,
                             int64_t nnz, uint64_t ncoo, uint32_t *__restrict__ flag) {
  GRID_STRIDE(z, nnz) {
    uint32_t f = 0;
    for (uint32_t t = jmap[z]; t < jmap[z + 1]; ++t)
      if (perm[t] >= ncoo) { f = 1; break; }
    flag[z] = f;
  }
}

__global__ void k_nonempty(const int32_t *__restrict__ cnt, int64_t m, uint32_t *__restrict__ f) {
  GRID_STRIDE(r, m) f[r] = cnt[r] > 0 ? 1u : 0u;
}

__global__ void k_gather_i32(const int32_t *__restrict__ src, const int32_t *__restrict__ idx,
                             int64_t n, int32_t *__restrict__ dst) {
  GRID_STRIDE(t, n) dst[t] = src[idx[t]];
}

// ------------------------------------------------------------------ numeric kernels
__global__ void k_send_gather(const double *__restrict__ v, const uint32_t *__restrict__ sp,
                              int64_t n, double *__restrict__ out) {
  GRID_STRIDE(t, n) out[t] = v[sp[t]];
}

// Nonzeros whose contributions are all local: s = +0.0; s = s + v[k] in canonical order.
// A nonzero that meets a received contribution is left for k_numeric_mixed.
__global__ void k_numeric_local(const uint32_t *__restrict__ jmap, const uint32_t *__restrict__ perm,
                                const double *__restrict__ v, uint64_t ncoo, int64_t nnz_d,
                                int64_t nnz, double *__restrict__ val_d,
                                double *__restrict__ val_o, int mode) {
  GRID_STRIDE(z, nnz) {
    uint32_t t0 = jmap[z], t1 = jmap[z + 1];
    double s = 0.0;
    bool local = true;
    for (uint32_t t = t0; t < t1; ++t) {
      uint32_t p = perm[t];
      if (p >= ncoo) { local = false; break; }
      s = __dadd_rn(s, v[p]);
    }
    if (local) {
      double *a = z < nnz_d ? val_d + z : val_o + (z - nnz_d);
      *a = mode == SPMAT_INSERT ? __dadd_rn(0.0, s) : __dadd_rn(*a, s);
    }
  }
}

// Element COO (several contributions per nonzero, C3: 1..8): one nonzero per thread, its
// contribution segment read kSeg at a time -- the kSeg perm loads, then the kSeg v gathers, are
// each issued together before any is used, so a segment costs one jmap -> perm -> v chain of
// latencies instead of one per contribution -- then summed in canonical order.
template <int kSeg>
__global__ void __launch_bounds__(256) k_numeric_seg(
    const uint32_t *__restrict__ jmap, const uint32_t *__restrict__ perm, const double *__restrict__ v,
    uint64_t ncoo, int64_t nnz_d, int64_t nnz, double *__restrict__ val_d, double *__restrict__ val_o,
    int mode) {
  GRID_STRIDE(z, nnz) {
    const uint32_t t0 = __ldg(jmap + z), t1 = __ldg(jmap + z + 1);
    double s = 0.0;
    bool local = true;
    for (uint32_t a = t0; a < t1; a += kSeg) {
      uint32_t q[kSeg];
#pragma unroll
      for (int k = 0; k < kSeg; ++k) q[k] = a + k < t1 ? __ldg(perm + a + k) : 0u;
      double w[kSeg];
#pragma unroll
      for (int k = 0; k < kSeg; ++k) w[k] = (a + k < t1 && q[k] < ncoo) ? __ldg(v + q[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < kSeg; ++k) {
        if (a + k < t1) {
          if (q[k] >= ncoo) local = false;  // received contribution: k_numeric_mixed finishes it
          s = __dadd_rn(s, w[k]);
        }
      }
    }
    if (local) {
      double *dst = z < nnz_d ? val_d + z : val_o + (z - nnz_d);
      *dst = mode == SPMAT_INSERT ? __dadd_rn(0.0, s) : __dadd_rn(*dst, s);
    }
  }
}

template <int S, int T>
struct PipeCfg {
  static constexpr int first = S, second = T;
};

// The same sums, software-pipelined over a grid-stride loop: while the v gathers of nonzero z
// are in flight, the perm loads of z + stride and the jmap loads of z + 2 stride are too, so
// each thread keeps three dependent stages of different nonzeros outstanding.
template <int kSeg, int kTail, bool kInsert, bool kMixed>
__global__ void __launch_bounds__(256) k_numeric_seg_pipe(
    const uint32_t *__restrict__ jmap, const uint32_t *__restrict__ perm, const double *__restrict__ v,
    uint32_t ncoo, int64_t nnz_d, int64_t nnz, double *__restrict__ val_d, double *__restrict__ val_o) {
  // perm entries >= ncoo are received contributions (several ranks): such a nonzero is left for
  // k_numeric_mixed, as in k_numeric_seg
  const int64_t stride = (int64_t)gridDim.x * 256;
  int64_t z = (int64_t)blockIdx.x * 256 + threadIdx.x;
  uint32_t a0 = 0u, n0 = 0u, a1 = 0u, n1 = 0u;
  if (z < nnz) {
    a0 = __ldg(jmap + z);
    n0 = __ldg(jmap + z + 1) - a0;
  }
  if (z + stride < nnz) {
    a1 = __ldg(jmap + z + stride);
    n1 = __ldg(jmap + z + stride + 1) - a1;
  }
  uint32_t q[kSeg];
#pragma unroll
  for (int k = 0; k < kSeg; ++k) q[k] = (uint32_t)k < n0 ? __ldg(perm + a0 + k) : 0u;
  for (; z < nnz; z += stride) {
    double w[kSeg];
    bool local = true;
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
      const bool in = (uint32_t)k < n0, mine = !kMixed || q[k] < ncoo;
      w[k] = 0.0;
      if (in && mine) w[k] = __ldg(v + q[k]);
      if (kMixed) local = local && (!in || mine);
    }
#pragma unroll
    for (int k = 0; k < kSeg; ++k) q[k] = (uint32_t)k < n1 ? __ldg(perm + a1 + k) : 0u;
    uint32_t a2 = 0u, n2 = 0u;
    if (z + 2 * stride < nnz) {
      a2 = __ldg(jmap + z + 2 * stride);
      n2 = __ldg(jmap + z + 2 * stride + 1) - a2;
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kSeg; ++k) s = __dadd_rn(s, w[k]);
    for (uint32_t a = kSeg; a < n0; a += kTail) {  // longer segments: kTail at a time
      double u[kTail];
#pragma unroll
      for (int k = 0; k < kTail; ++k) {
        u[k] = 0.0;
        if (a + k < n0) {
          const uint32_t p = __ldg(perm + a0 + a + k);
          const bool mine = !kMixed || p < ncoo;
          if (mine) u[k] = __ldg(v + p);
          if (kMixed) local = local && mine;
        }
      }
#pragma unroll
      for (int k = 0; k < kTail; ++k) s = __dadd_rn(s, u[k]);
    }
    if (local) {
      double *dst = z < nnz_d ? val_d + z : val_o + (z - nnz_d);
      *dst = kInsert ? __dadd_rn(0.0, s) : __dadd_rn(*dst, s);
    }
    a0 = a1;
    n0 = n1;
    a1 = a2;
    n1 = n2;
  }
}

// Element COO, warp-cooperative: a warp takes 32 consecutive nonzeros, whose contribution
// segments are one contiguous range of perm (<= kWSpan entries): the lanes load that range
// coalesced (8 perm loads, then their 8 v gathers, per lane in flight) into shared memory, then
// each lane sums its own nonzero's segment from shared memory in canonical order.  No per-lane
// predication over a fixed segment width.  A range longer than kWSpan falls back to each lane
// summing its segment from global memory.
constexpr int kWSpan = 256;
__global__ void __launch_bounds__(256) k_numeric_warp(
    const uint32_t *__restrict__ jmap, const uint32_t *__restrict__ perm, const double *__restrict__ v,
    uint64_t ncoo, int64_t nnz_d, int64_t nnz, double *__restrict__ val_d, double *__restrict__ val_o,
    int mode) {
  __shared__ double sw[8][kWSpan];
  __shared__ uint32_t sq[8][kWSpan];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t z0 = ((int64_t)blockIdx.x * 8 + wib) * 32; z0 < nnz; z0 += nwarps * 32) {
    const int64_t z = z0 + lane;
    const bool valid = z < nnz;
    const uint32_t a = valid ? __ldg(jmap + z) : 0u, b = valid ? __ldg(jmap + z + 1) : 0u;
    const int last = (int)(nnz - 1 - z0 < 31 ? nnz - 1 - z0 : 31);
    const uint32_t base = __shfl_sync(0xffffffffu, a, 0), end = __shfl_sync(0xffffffffu, b, last);
    const uint32_t span = end - base;
    double s = 0.0;
    bool local = true;
    if (span <= (uint32_t)kWSpan) {
      uint32_t q[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t t = lane + 32 * k;
        q[k] = t < span ? __ldg(perm + base + t) : 0u;
      }
      double w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = (lane + 32 * k < span && q[k] < ncoo) ? __ldg(v + q[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t t = lane + 32 * k;
        if (t < span) {
          sq[wib][t] = q[k];
          sw[wib][t] = w[k];
        }
      }
      __syncwarp();
      for (uint32_t t = a - base; t < b - base; ++t) {
        if (sq[wib][t] >= ncoo) local = false;  // received contribution: k_numeric_mixed finishes it
        s = __dadd_rn(s, sw[wib][t]);
      }
      __syncwarp();
    } else {
      for (uint32_t t = a; t < b; ++t) {
        const uint32_t p = __ldg(perm + t);
        if (p >= ncoo) {
          local = false;
          break;
        }
        s = __dadd_rn(s, __ldg(v + p));
      }
    }
    if (valid && local) {
      double *dst = z < nnz_d ? val_d + z : val_o + (z - nnz_d);
      *dst = mode == SPMAT_INSERT ? __dadd_rn(0.0, s) : __dadd_rn(*dst, s);
    }
  }
}

// 3x3 blocks (spmat_set_block_size(A, 3)), no received contributions: the numeric step writes
// the block copy bval directly (the CSR val_d is then stale until spmat_sync_csr_values) -- one
// pass over the compulsory bytes instead of val_d plus a val_d -> bval copy.  A warp walks a
// block row's 9*nb values in bval order (v = 9q + 3i + j is nonzero rowptr[3br+i] + 3q + j),
// kNumU values per lane in flight, each summed in canonical order.  ONE: every nonzero has
// exactly one contribution (ncontrib == nnz, e.g. node-block COO without duplicates), so
// jmap[z] == z -- the jmap reads and one level of the load chain disappear.
template <bool ONE>
__global__ void __launch_bounds__(256) k_numeric_bsr3(
    const int32_t *__restrict__ rowptr, const int32_t *__restrict__ browptr, const uint32_t *__restrict__ jmap,
    const uint32_t *__restrict__ perm, const double *__restrict__ v, int64_t mb, double *__restrict__ bval,
    int mode) {
  constexpr int U = ONE ? 8 : 4;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t br = warp; br < mb; br += nwarps) {
    const int bp0 = browptr[br], n9 = 9 * (browptr[br + 1] - bp0);
    const int r0 = rowptr[3 * br], r1 = rowptr[3 * br + 1], r2 = rowptr[3 * br + 2];
    for (int v0 = lane; v0 < n9; v0 += 32 * U) {
      uint32_t a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int vv = v0 + 32 * u;
        const int q = vv / 9, i = (vv % 9) / 3, j = vv % 3;
        const int z = (i == 0 ? r0 : (i == 1 ? r1 : r2)) + 3 * q + j;
        a[u] = vv < n9 ? (ONE ? (uint32_t)z : __ldg(jmap + z)) : 0u;
        b[u] = vv < n9 ? (ONE ? (uint32_t)z + 1u : __ldg(jmap + z + 1)) : 0u;
      }
      double s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] = 0.0;
      for (;;) {  // one contribution of every unfinished value per round (canonical order)
        bool any = false;
        uint32_t q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          q[u] = a[u] < b[u] ? __ldg(perm + a[u]) : 0u;
          any |= a[u] < b[u];
        }
        if (!any) break;
        double w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) w[u] = a[u] < b[u] ? __ldg(v + q[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (a[u] < b[u]) {
            s[u] = __dadd_rn(s[u], w[u]);
            ++a[u];
          }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int vv = v0 + 32 * u;
        if (vv < n9) {
          double *dst = bval + 9 * (int64_t)bp0 + vv;
          *dst = mode == SPMAT_INSERT ? __dadd_rn(0.0, s[u]) : __dadd_rn(*dst, s[u]);
        }
      }
    }
  }
}

// k_numeric_bsr3 for one contribution per nonzero (node-block COO, C5): straight-line
// perm -> v -> store per value, 8 values per lane in flight, and the next block row's
// (browptr, rowptr) prefetched while the current one is gathered -- per block row one chain of
// two dependent loads instead of three (the index loads were the first link).
__global__ void __launch_bounds__(256) k_numeric_bsr3_one(
    const int32_t *__restrict__ rowptr, const int32_t *__restrict__ browptr, const uint32_t *__restrict__ perm,
    const double *__restrict__ v, int64_t mb, double *__restrict__ bval, int mode) {
  constexpr int U = 8;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t br = warp;
  if (br >= mb) return;
  int bp0 = browptr[br], bp1 = browptr[br + 1];
  int r0 = rowptr[3 * br], r1 = rowptr[3 * br + 1], r2 = rowptr[3 * br + 2];
  for (;;) {
    const int64_t nb = br + nwarps;
    int nbp0 = 0, nbp1 = 0, nr0 = 0, nr1 = 0, nr2 = 0;
    if (nb < mb) {  // prefetch: independent of the gathers below
      nbp0 = browptr[nb];
      nbp1 = browptr[nb + 1];
      nr0 = rowptr[3 * nb];
      nr1 = rowptr[3 * nb + 1];
      nr2 = rowptr[3 * nb + 2];
    }
    const int n9 = 9 * (bp1 - bp0);
    for (int v0 = lane; v0 < n9; v0 += 32 * U) {
      uint32_t q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int vv = v0 + 32 * u;
        const int qq = vv / 9, i = (vv % 9) / 3, j = vv % 3;
        const int z = (i == 0 ? r0 : (i == 1 ? r1 : r2)) + 3 * qq + j;
        q[u] = vv < n9 ? __ldg(perm + z) : 0u;
      }
      double w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = v0 + 32 * u < n9 ? __ldg(v + q[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int vv = v0 + 32 * u;
        if (vv < n9) {
          const double s = __dadd_rn(0.0, w[u]);  // the one-term canonical sum
          double *dst = bval + 9 * (int64_t)bp0 + vv;
          *dst = mode == SPMAT_INSERT ? __dadd_rn(0.0, s) : __dadd_rn(*dst, s);
        }
      }
    }
    if (nb >= mb) break;
    br = nb;
    bp0 = nbp0;
    bp1 = nbp1;
    r0 = nr0;
    r1 = nr1;
    r2 = nr2;
  }
}

// One contribution per nonzero (jmap[z] == z: stencil and node-block COO), no loop: each thread
// loads U perm entries (coalesced), then their U v values (nearly coalesced: perm permutes only
// within a row), then stores val -- s = +0.0 + v, INSERT val = +0.0 + s, ADD val = val + s, the
// canonical sums of a one-term segment.  kMixed: perm entries >= lim are received
// contributions (several ranks), left for k_numeric_mixed.
template <int U, bool kInsert, bool kMixed>
__global__ void __launch_bounds__(256) k_numeric_one(const uint32_t *__restrict__ perm, const double *__restrict__ v,
                                                     uint32_t lim, int64_t z0, int64_t nnz_d, int64_t nnz,
                                                     double *__restrict__ val_d, double *__restrict__ val_o) {
  const int64_t zb = z0 + (int64_t)blockIdx.x * (256 * U) + threadIdx.x;
  uint32_t q[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t z = zb + 256 * u;
    q[u] = z < nnz ? __ldg(perm + z) : 0u;
  }
  double w[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t z = zb + 256 * u;
    w[u] = 0.0;
    if (z < nnz && (!kMixed || q[u] < lim)) w[u] = __ldg(v + q[u]);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t z = zb + 256 * u;
    if (z < nnz && (!kMixed || q[u] < lim)) {
      double *dst = z < nnz_d ? val_d + z : val_o + (z - nnz_d);
      const double sum = __dadd_rn(0.0, w[u]);
      *dst = kInsert ? __dadd_rn(0.0, sum) : __dadd_rn(*dst, sum);
    }
  }
}

// Default numeric kernel (ONE: jmap[z] == z, as in k_numeric_bsr3): each thread finishes kNumU nonzeros z = base + u*blockDim + tid
// (coalesced across the warp), advancing all of them one contribution per round so every
// level of the jmap -> perm -> v chain has kNumU loads in flight.  Each nonzero is still
// summed in canonical order by one thread; a nonzero meeting a received contribution is left
// for k_numeric_mixed.
constexpr int kNumU = 4;
template <bool ONE>
__global__ void __launch_bounds__(256) k_numeric_ilp(
    const uint32_t *__restrict__ jmap, const uint32_t *__restrict__ perm, const double *__restrict__ v,
    uint64_t ncoo, int64_t nnz_d, int64_t nnz, double *__restrict__ val_d, double *__restrict__ val_o,
    int mode, int64_t z0) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * kNumU;
  for (int64_t base = z0 + (int64_t)blockIdx.x * blockDim.x * kNumU + threadIdx.x; base < nnz; base += stride) {
    uint32_t a[kNumU], b[kNumU];
    double s[kNumU];
    bool ok[kNumU];
#pragma unroll
    for (int u = 0; u < kNumU; ++u) {
      const int64_t z = base + (int64_t)u * blockDim.x;
      a[u] = z < nnz ? (ONE ? (uint32_t)z : __ldg(jmap + z)) : 0u;
      b[u] = z < nnz ? (ONE ? (uint32_t)z + 1u : __ldg(jmap + z + 1)) : 0u;
      s[u] = 0.0;
      ok[u] = z < nnz;
    }
    for (;;) {  // one contribution of every unfinished nonzero per round
      uint32_t q[kNumU];
      bool any = false;
#pragma unroll
      for (int u = 0; u < kNumU; ++u) {
        const bool live = ok[u] && a[u] < b[u];
        q[u] = live ? __ldg(perm + a[u]) : 0u;
        any |= live;
      }
      if (!any) break;
      double vv[kNumU];
#pragma unroll
      for (int u = 0; u < kNumU; ++u) {
        const bool live = ok[u] && a[u] < b[u];
        if (live && q[u] >= ncoo) ok[u] = false;  // received contribution: mixed nonzero
        vv[u] = (live && q[u] < ncoo) ? __ldg(v + q[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kNumU; ++u) {
        if (ok[u] && a[u] < b[u]) {
          s[u] = __dadd_rn(s[u], vv[u]);
          ++a[u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kNumU; ++u) {
      const int64_t z = base + (int64_t)u * blockDim.x;
      if (ok[u]) {
        double *dst = z < nnz_d ? val_d + z : val_o + (z - nnz_d);
        *dst = mode == SPMAT_INSERT ? __dadd_rn(0.0, s[u]) : __dadd_rn(*dst, s[u]);
      }
    }
  }
}

__global__ void k_numeric_mixed(const uint32_t *__restrict__ mixed, int64_t nmixed,
                                const uint32_t *__restrict__ jmap, const uint32_t *__restrict__ perm,
                                const double *__restrict__ v, const double *__restrict__ recv,
                                uint64_t ncoo, int64_t nnz_d, double *__restrict__ val_d,
                                double *__restrict__ val_o, int mode) {
  GRID_STRIDE(q, nmixed) {
    int64_t z = mixed[q];
    double s = 0.0;
    for (uint32_t t = jmap[z]; t < jmap[z + 1]; ++t) {
      uint32_t p = perm[t];
      s = __dadd_rn(s, p < ncoo ? v[p] : recv[p - ncoo]);
    }
    double *a = z < nnz_d ? val_d + z : val_o + (z - nnz_d);
    *a = mode == SPMAT_INSERT ? __dadd_rn(0.0, s) : __dadd_rn(*a, s);
  }
}

// ------------------------------------------------------------------ symbolic driver
static int create_impl(spmat_comm_s *c, int64_t m_local, int64_t n_local, int64_t M, int64_t N,
                       int64_t ncoo, const int64_t *coo_i, const int64_t *coo_j, spmat_s **out) {
  const int P = c->nranks, me = c->rank;
  cudaStream_t st = c->setup_stream;
  // ---- layout agreement (a1): allgather (m, n, M, N, ncoo-ok)
  int64_t mine[4] = {m_local, n_local, M, N};
  std::vector<int64_t> all(4 * (size_t)P);
  SP_TRY(c->allgather_i64(mine, 4, all.data()));
  std::vector<int64_t> roff(P + 1, 0), coff(P + 1, 0);
  bool mismatch = false;
  for (int r = 0; r < P; ++r) {
    if (all[4 * r + 2] != M || all[4 * r + 3] != N) mismatch = true;
    if (all[4 * r] < 0 || all[4 * r + 1] < 0) mismatch = true;
    roff[r + 1] = roff[r] + all[4 * r];
    coff[r + 1] = coff[r] + all[4 * r + 1];
  }
  if (roff[P] != M || coff[P] != N) mismatch = true;
  if (mismatch)
    return fail(SPMAT_ERR_MISMATCH,
                "spmat_create_coo: ranks disagree on M,N or local sizes do not sum (M=%lld N=%lld)",
                (long long)M, (long long)N);
  const int64_t rstart = roff[me], cstart = coff[me], cend = coff[me + 1];
  // Errors found on one rank only are agreed on (Comm::agree) before the next collective, so
  // every rank returns an error instead of the others blocking in NCCL.
  const char *who = "spmat_create_coo";

  Tmp tmp;
  // ---- inputs on the device (memtype detection); not retained
  DevBuf<int64_t> di, dj;
  const int64_t *ci = coo_i, *cj = coo_j;
  SP_TRY(c->agree([&]() -> int {
    if (m_local > INT32_MAX - 1) return fail(SPMAT_ERR_ARG, "m_local must be < 2^31");
    if ((uint64_t)ncoo >= (1ull << 32)) return fail(SPMAT_ERR_ARG, "ncoo must be < 2^32");
    // device COO arrays may still be being written by the caller's kernels on any stream, and
    // this (host-synchronising) call reads them on the library's setup stream: wait for the
    // device first
    SP_CUDA(cudaDeviceSynchronize());
    if (ncoo > 0) {
      if (!coo_i || !coo_j) return fail(SPMAT_ERR_ARG, "spmat_create_coo: null coo_i/coo_j");
      if (!is_device_ptr(coo_i)) {
        SP_TRY(di.alloc(ncoo));
        SP_CUDA(cudaMemcpyAsync(di.get(), coo_i, ncoo * 8, cudaMemcpyHostToDevice, st));
        ci = di.get();
      }
      if (!is_device_ptr(coo_j)) {
        SP_TRY(dj.alloc(ncoo));
        SP_CUDA(cudaMemcpyAsync(dj.get(), coo_j, ncoo * 8, cudaMemcpyHostToDevice, st));
        cj = dj.get();
      }
    }
    return SPMAT_OK;
  }(), who));

  // ---- 1. classify
  DevBuf<int64_t> droff;
  DevBuf<unsigned long long> dbad;
  DevBuf<uint32_t> dest, dest2, kk, kk2;
  unsigned long long bad = ~0ull;
  const int sB = [&]() -> int {
    SP_TRY(droff.alloc(P + 1));
    SP_CUDA(cudaMemcpyAsync(droff.get(), roff.data(), (P + 1) * 8, cudaMemcpyHostToDevice, st));
    SP_TRY(dbad.alloc(1));
    SP_CUDA(cudaMemsetAsync(dbad.get(), 0xff, 8, st));
    SP_TRY(dest.alloc(ncoo));
    if (ncoo > 0) {
      k_classify<<<nblk(ncoo), 256, 0, st>>>(ci, cj, ncoo, M, N, droff.get(), P, dest.get(), dbad.get());
      SP_LAUNCH();
    }
    SP_CUDA(cudaMemcpyAsync(&bad, dbad.get(), 8, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    return SPMAT_OK;
  }();
  {  // the range-error exchange also carries the local status (-2 - status)
    int64_t b = sB != SPMAT_OK ? -2 - (int64_t)sB : (bad == ~0ull ? -1 : (int64_t)bad);
    std::vector<int64_t> allbad(P);
    SP_TRY(c->allgather_i64(&b, 1, allbad.data()));
    for (int r = 0; r < P; ++r)
      if (allbad[r] <= -2)
        return sB != SPMAT_OK ? sB : fail((int)(-2 - allbad[r]), "%s: failed on rank %d", who, r);
    for (int r = 0; r < P; ++r)
      if (allbad[r] >= 0)
        return fail(SPMAT_ERR_RANGE, "spmat_create_coo: COO index out of range on rank %d at k=%lld",
                    r, (long long)allbad[r]);
  }

  // ---- 2. stable sort (dest, k) -> per-destination k lists
  std::vector<int64_t> dofs(P + 2, 0);
  int64_t nlocal = 0;
  spmat_s *A = new spmat_s();
  std::unique_ptr<spmat_s, int (*)(spmat_s *)> guard(A, [](spmat_s *a) { return spmat_destroy(a); });
  A->comm = c;
  const int sC = [&]() -> int {
  SP_TRY(kk.alloc(ncoo));
  SP_TRY(kk2.alloc(ncoo));
  SP_TRY(dest2.alloc(ncoo));
  if (ncoo > 0) {
    k_iota<<<nblk(ncoo), 256, 0, st>>>(kk.get(), ncoo);
    SP_LAUNCH();
    cub::DoubleBuffer<uint32_t> dk(dest.get(), dest2.get()), dv(kk.get(), kk2.get());
    int eb = bits_for((uint64_t)P);
    CUB_CALL(tmp, st, cub::DeviceRadixSort::SortPairs(d_temp_storage, temp_storage_bytes, dk, dv,
                                                      ncoo, 0, eb, st));
    DevBuf<int64_t> ddofs;
    SP_TRY(ddofs.alloc(P + 2));
    k_bounds<<<1, 64 * ((P + 2 + 63) / 64), 0, st>>>(dk.Current(), ncoo, P, ddofs.get());
    SP_LAUNCH();
    SP_CUDA(cudaMemcpyAsync(dofs.data(), ddofs.get(), (P + 2) * 8, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    if (dv.Current() != kk.get()) std::swap(kk.p, kk2.p);
  }
  kk2.release();
  dest.release();
  dest2.release();
  A->M = M; A->N = N; A->m = m_local; A->n = n_local;
  A->rstart = rstart; A->rend = roff[me + 1]; A->cstart = cstart; A->cend = cend;
  A->roff = roff; A->coff = coff;
  A->ncoo = ncoo;
  nlocal = dofs[me + 1] - dofs[me];
  A->send_count.assign(P, 0);
  A->send_off.assign(P + 1, 0);
  for (int d = 0; d < P; ++d) A->send_count[d] = d == me ? 0 : dofs[d + 1] - dofs[d];
  for (int d = 0; d < P; ++d) A->send_off[d + 1] = A->send_off[d] + A->send_count[d];
  A->nsend = A->send_off[P];
  SP_TRY(A->sendperm.alloc(A->nsend));
  if (dofs[me] > 0)
    SP_CUDA(cudaMemcpyAsync(A->sendperm.get(), kk.get(), dofs[me] * 4, cudaMemcpyDeviceToDevice, st));
  if (dofs[P] - dofs[me + 1] > 0)
    SP_CUDA(cudaMemcpyAsync(A->sendperm.get() + dofs[me], kk.get() + dofs[me + 1],
                            (dofs[P] - dofs[me + 1]) * 4, cudaMemcpyDeviceToDevice, st));
  return SPMAT_OK;
  }();

  // ---- 3. exchange (i, j) of off-rank entries
  {  // the count exchange also carries the local status (last element)
    std::vector<int64_t> mine(P + 1, 0), allc((size_t)P * (P + 1));
    if (sC == SPMAT_OK)
      for (int d = 0; d < P; ++d) mine[d] = A->send_count[d];
    mine[P] = sC;
    SP_TRY(c->allgather_i64(mine.data(), P + 1, allc.data()));
    for (int r = 0; r < P; ++r)
      if (allc[(size_t)r * (P + 1) + P] != SPMAT_OK)
        return sC != SPMAT_OK ? sC : fail((int)allc[(size_t)r * (P + 1) + P], "%s: failed on rank %d", who, r);
    A->recv_count.assign(P, 0);
    A->recv_off.assign(P + 1, 0);
    for (int s = 0; s < P; ++s) A->recv_count[s] = s == me ? 0 : allc[(size_t)s * (P + 1) + me];
    for (int s = 0; s < P; ++s) A->recv_off[s + 1] = A->recv_off[s] + A->recv_count[s];
    A->nrecv = A->recv_off[P];
  }
  DevBuf<longlong2> sij, rij;
  SP_TRY(c->agree([&]() -> int {
    if ((uint64_t)ncoo + (uint64_t)A->nrecv >= (1ull << 32))
      return fail(SPMAT_ERR_ARG, "ncoo + received entries must be < 2^32");
    SP_TRY(sij.alloc(A->nsend));
    SP_TRY(rij.alloc(A->nrecv));
    if (A->nsend > 0) {
      k_gather_ij<<<nblk(A->nsend), 256, 0, st>>>(ci, cj, A->sendperm.get(), A->nsend, sij.get());
      SP_LAUNCH();
    }
    return SPMAT_OK;
  }(), who));
  SP_TRY(c->exchange_dev(sij.get(), A->send_off.data(), A->send_count.data(), rij.get(),
                         A->recv_off.data(), A->recv_count.data(), sizeof(longlong2), st));
  sij.release();

  // ---- 4. canonical contributions, keyed (row, col), stable radix sort
  const int64_t nt = nlocal + A->nrecv;
  std::vector<int64_t> cm, off;
  std::vector<int32_t> own;
  SP_TRY(c->agree([&]() -> int {
  if (nt >= INT32_MAX) return fail(SPMAT_ERR_ARG, "more than 2^31 contributions on one rank");
  A->ncontrib = nt;
  DevBuf<uint64_t> key, key2;
  DevBuf<uint32_t> val, val2;
  SP_TRY(key.alloc(nt));
  SP_TRY(val.alloc(nt));
  const int64_t before = A->recv_off[me];  // received from src < me
  if (A->nrecv > 0) {
    k_keys_recv<<<nblk(A->nrecv), 256, 0, st>>>(rij.get(), A->nrecv, before, nlocal, rstart, N,
                                                (uint64_t)ncoo, key.get(), val.get());
    SP_LAUNCH();
  }
  if (nlocal > 0) {
    k_keys_local<<<nblk(nlocal), 256, 0, st>>>(ci, cj, kk.get() + dofs[me], nlocal, before,
                                               rstart, N, key.get(), val.get());
    SP_LAUNCH();
  }
  rij.release();
  kk.release();
  di.release();
  dj.release();
  if (nt > 0) {
    SP_TRY(key2.alloc(nt));
    SP_TRY(val2.alloc(nt));
    cub::DoubleBuffer<uint64_t> dk(key.get(), key2.get());
    cub::DoubleBuffer<uint32_t> dv(val.get(), val2.get());
    uint64_t maxkey = (uint64_t)std::max<int64_t>(m_local, 1) * (uint64_t)std::max<int64_t>(N, 1) - 1;
    CUB_CALL(tmp, st, cub::DeviceRadixSort::SortPairs(d_temp_storage, temp_storage_bytes, dk, dv,
                                                      (int)nt, 0, bits_for(maxkey), st));
    if (dk.Current() != key.get()) std::swap(key.p, key2.p);
    if (dv.Current() != val.get()) std::swap(val.p, val2.p);
    key2.release();
    val2.release();
  }

  // ---- 5. nonzeros
  DevBuf<uint32_t> head, zid, segstart;
  SP_TRY(head.alloc(nt));
  SP_TRY(zid.alloc(nt));
  SP_TRY(segstart.alloc(nt));
  int64_t nnz = 0;
  if (nt > 0) {
    k_heads<<<nblk(nt), 256, 0, st>>>(key.get(), nt, head.get());
    SP_LAUNCH();
    CUB_CALL(tmp, st, cub::DeviceScan::InclusiveSum(d_temp_storage, temp_storage_bytes, head.get(),
                                                    zid.get(), (int)nt, st));
    DevBuf<int> dn;
    SP_TRY(dn.alloc(1));
    CUB_CALL(tmp, st, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes,
                                                 thrust::counting_iterator<uint32_t>(0), head.get(),
                                                 segstart.get(), dn.get(), (int)nt, st));
    int hn = 0;
    SP_CUDA(cudaMemcpyAsync(&hn, dn.get(), 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    nnz = hn;
  }
  head.release();
  DevBuf<uint32_t> isdiag, pos_d;
  DevBuf<int32_t> cnt_d, cnt_o;
  SP_TRY(isdiag.alloc(nnz));
  SP_TRY(pos_d.alloc(nnz));
  SP_TRY(cnt_d.alloc(m_local + 1));
  SP_TRY(cnt_o.alloc(m_local + 1));
  SP_CUDA(cudaMemsetAsync(cnt_d.get(), 0, (m_local + 1) * 4, st));
  SP_CUDA(cudaMemsetAsync(cnt_o.get(), 0, (m_local + 1) * 4, st));
  int64_t nnz_d = 0;
  if (nnz > 0) {
    k_nz_classify<<<nblk(nnz), 256, 0, st>>>(key.get(), segstart.get(), nnz, N, cstart, cend,
                                             isdiag.get(), cnt_d.get(), cnt_o.get());
    SP_LAUNCH();
    CUB_CALL(tmp, st, cub::DeviceScan::ExclusiveSum(d_temp_storage, temp_storage_bytes,
                                                    isdiag.get(), pos_d.get(), (int)nnz, st));
    uint32_t last[2];
    SP_CUDA(cudaMemcpyAsync(&last[0], pos_d.get() + nnz - 1, 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaMemcpyAsync(&last[1], isdiag.get() + nnz - 1, 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    nnz_d = (int64_t)last[0] + last[1];
  }
  const int64_t nnz_o = nnz - nnz_d;
  A->nnz_d = nnz_d;
  A->nnz_o = nnz_o;
  // diag CSR
  // +8 padding: the bulk-copy SpMV rounds tile bounds out to 16-byte multiples
  SP_TRY(A->rowptr_d.alloc(m_local + 1 + 8));
  CUB_CALL(tmp, st, cub::DeviceScan::ExclusiveSum(d_temp_storage, temp_storage_bytes, cnt_d.get(),
                                                  A->rowptr_d.get(), (int)(m_local + 1), st));
  SP_TRY(A->col_d.alloc(nnz_d + 8));
  SP_TRY(A->val_d.alloc(nnz_d + 8));
  DevBuf<int64_t> ocol;
  SP_TRY(ocol.alloc(nnz_o));
  if (nnz > 0) {
    k_nz_cols<<<nblk(nnz), 256, 0, st>>>(key.get(), segstart.get(), isdiag.get(), pos_d.get(), nnz,
                                         N, cstart, A->col_d.get(), ocol.get());
    SP_LAUNCH();
  }
  key.release();
  // colmap = sorted unique ghost columns
  if (nnz_o > 0) {
    DevBuf<int64_t> sorted;
    SP_TRY(sorted.alloc(nnz_o));
    CUB_CALL(tmp, st, cub::DeviceRadixSort::SortKeys(d_temp_storage, temp_storage_bytes,
                                                     (const uint64_t *)ocol.get(),
                                                     (uint64_t *)sorted.get(), (int)nnz_o, 0,
                                                     bits_for((uint64_t)N), st));
    DevBuf<int64_t> uniq;
    SP_TRY(uniq.alloc(nnz_o));
    DevBuf<int> dn;
    SP_TRY(dn.alloc(1));
    CUB_CALL(tmp, st, cub::DeviceSelect::Unique(d_temp_storage, temp_storage_bytes, sorted.get(),
                                                uniq.get(), dn.get(), (int)nnz_o, st));
    int ng = 0;
    SP_CUDA(cudaMemcpyAsync(&ng, dn.get(), 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    A->n_ghost = ng;
    SP_TRY(A->colmap.alloc(ng));
    SP_CUDA(cudaMemcpyAsync(A->colmap.get(), uniq.get(), (size_t)ng * 8, cudaMemcpyDeviceToDevice, st));
    SP_TRY(A->col_o.alloc(nnz_o));
    k_ghost_index<<<nblk(nnz_o), 256, 0, st>>>(ocol.get(), nnz_o, A->colmap.get(), ng, A->col_o.get());
    SP_LAUNCH();
  }
  ocol.release();
  // compressed offdiag rows
  {
    DevBuf<uint32_t> ne;
    SP_TRY(ne.alloc(m_local));
    DevBuf<int32_t> rows;
    SP_TRY(rows.alloc(m_local));
    DevBuf<int> dn;
    SP_TRY(dn.alloc(1));
    int nro = 0;
    if (m_local > 0 && nnz_o > 0) {
      k_nonempty<<<nblk(m_local), 256, 0, st>>>(cnt_o.get(), m_local, ne.get());
      SP_LAUNCH();
      CUB_CALL(tmp, st, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes,
                                                   thrust::counting_iterator<int32_t>(0), ne.get(),
                                                   rows.get(), dn.get(), (int)m_local, st));
      SP_CUDA(cudaMemcpyAsync(&nro, dn.get(), 4, cudaMemcpyDeviceToHost, st));
      SP_CUDA(cudaStreamSynchronize(st));
    }
    A->n_ro = nro;
    SP_TRY(A->rows_o.alloc(nro));
    SP_TRY(A->rowptr_o.alloc(nro + 1));
    if (nro > 0) {
      SP_CUDA(cudaMemcpyAsync(A->rows_o.get(), rows.get(), (size_t)nro * 4, cudaMemcpyDeviceToDevice, st));
      DevBuf<int32_t> cc;
      SP_TRY(cc.alloc(nro + 1));
      SP_CUDA(cudaMemsetAsync(cc.get() + nro, 0, 4, st));
      k_gather_i32<<<nblk(nro), 256, 0, st>>>(cnt_o.get(), A->rows_o.get(), nro, cc.get());
      SP_LAUNCH();
      CUB_CALL(tmp, st, cub::DeviceScan::ExclusiveSum(d_temp_storage, temp_storage_bytes, cc.get(),
                                                      A->rowptr_o.get(), nro + 1, st));
    }
    SP_TRY(A->val_o.alloc(nnz_o));
  }
  // ---- jmap / perm in block order (diag nonzeros, then offdiag nonzeros)
  SP_TRY(A->jmap.alloc(nnz + 1));
  SP_TRY(A->perm.alloc(nt));
  if (nt > 0) {
    // zid holds inclusive sums of the run heads (1-based nonzero ids)
    DevBuf<uint32_t> cflag, cpos;
    SP_TRY(cflag.alloc(nt));
    SP_TRY(cpos.alloc(nt));
    k_cflag<<<nblk(nt), 256, 0, st>>>(zid.get(), isdiag.get(), nt, cflag.get());
    SP_LAUNCH();
    CUB_CALL(tmp, st, cub::DeviceScan::ExclusiveSum(d_temp_storage, temp_storage_bytes, cflag.get(),
                                                    cpos.get(), (int)nt, st));
    uint32_t last[2];
    SP_CUDA(cudaMemcpyAsync(&last[0], cpos.get() + nt - 1, 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaMemcpyAsync(&last[1], cflag.get() + nt - 1, 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    int64_t total_d = (int64_t)last[0] + last[1];
    k_perm<<<nblk(nt), 256, 0, st>>>(val.get(), cflag.get(), cpos.get(), nt, total_d, A->perm.get());
    SP_LAUNCH();
    k_jmap<<<nblk(nnz), 256, 0, st>>>(segstart.get(), isdiag.get(), pos_d.get(), cpos.get(), nnz,
                                      nnz_d, total_d, nt, A->jmap.get());
    SP_LAUNCH();
  } else {
    SP_CUDA(cudaMemsetAsync(A->jmap.get(), 0, 4, st));
  }
  val.release();
  zid.release();
  segstart.release();
  isdiag.release();
  pos_d.release();
  // ---- mixed nonzeros (with received contributions)
  if (A->nrecv > 0 && nnz > 0) {
    DevBuf<uint32_t> flag, ids;
    SP_TRY(flag.alloc(nnz));
    SP_TRY(ids.alloc(nnz));
    k_mixed_flag<<<nblk(nnz), 256, 0, st>>>(A->jmap.get(), A->perm.get(), nnz, (uint64_t)ncoo, flag.get());
    SP_LAUNCH();
    DevBuf<int> dn;
    SP_TRY(dn.alloc(1));
    CUB_CALL(tmp, st, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes,
                                                 thrust::counting_iterator<uint32_t>(0), flag.get(),
                                                 ids.get(), dn.get(), (int)nnz, st));
    int nm = 0;
    SP_CUDA(cudaMemcpyAsync(&nm, dn.get(), 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    A->n_mixed = nm;
    SP_TRY(A->mixed.alloc(nm));
    if (nm) SP_CUDA(cudaMemcpyAsync(A->mixed.get(), ids.get(), (size_t)nm * 4, cudaMemcpyDeviceToDevice, st));
  }
  SP_TRY(A->sendbuf.alloc(A->nsend));
  SP_TRY(A->recvbuf.alloc(A->nrecv));
  SP_TRY(A->lvec.alloc(A->n_ghost));
  SP_CUDA(cudaEventCreateWithFlags(&A->ev_send_ready, cudaEventDisableTiming));
  SP_CUDA(cudaEventCreateWithFlags(&A->ev_recv_done, cudaEventDisableTiming));

  // ---- 6. halo SF from colmap: leaf g -> (owner(colmap[g]), colmap[g] - cstart_owner)
  {
    cm.resize(A->n_ghost);
    off.resize(A->n_ghost);
    own.resize(A->n_ghost);
    if (A->n_ghost)
      SP_CUDA(cudaMemcpyAsync(cm.data(), A->colmap.get(), A->n_ghost * 8, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    for (int64_t g = 0; g < A->n_ghost; ++g) {
      int q = (int)(std::upper_bound(coff.begin(), coff.end(), cm[g]) - coff.begin()) - 1;
      own[g] = q;
      off[g] = cm[g] - coff[q];
    }
  }
  return SPMAT_OK;
  }(), who));
  SP_TRY(sf_build(c, n_local, A->n_ghost, nullptr, own.data(), off.data(), &A->halo, true));
  SP_TRY(c->agree(spmv_prepare(A, st), who));
  SP_TRY(halo_peer_setup(A));
  if (!A->peer) SP_TRY(sf_ensure_peer(A->halo));  // the MatMult halo goes through the SF (A->peer is agreed)
  SP_CUDA(cudaStreamSynchronize(st));
  A->plan_builds = 1;
  *out = guard.release();
  return SPMAT_OK;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_create_coo(spmat_comm_t comm, int64_t m_local, int64_t n_local, int64_t M, int64_t N,
                     int64_t ncoo, const int64_t *coo_i, const int64_t *coo_j, spmat_t *out) {
  SP_NVTX("spmat_create_coo");
  if (!comm || !out) return fail(SPMAT_ERR_ARG, "spmat_create_coo: null argument");
  *out = nullptr;
  if (ncoo < 0) return fail(SPMAT_ERR_ARG, "spmat_create_coo: negative ncoo");
  DeviceGuard g(comm->device);
  return create_impl(comm, m_local, n_local, M, N, ncoo, coo_i, coo_j, out);
}

int spmat_set_values_coo(spmat_t A, const double *v, int mode, void *stream) {
  SP_NVTX("spmat_set_values_coo");
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_set_values_coo: null matrix");
  if (mode != SPMAT_INSERT && mode != SPMAT_ADD)
    return fail(SPMAT_ERR_ARG, "spmat_set_values_coo: bad mode %d", mode);
  if (A->ncoo > 0 && !v) return fail(SPMAT_ERR_ARG, "spmat_set_values_coo: null v");
  if (mode == SPMAT_ADD && !A->values_set)
    return fail(SPMAT_ERR_STATE, "spmat_set_values_coo: ADD before any INSERT");
  ++A->val_version;  // transposed values (transpose.cu) are re-gathered on next use
  spmat_comm_s *c = A->comm;
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nnz = A->nnz_d + A->nnz_o;
  const bool exchange = c->nranks > 1;
  if (exchange) {
    if (A->nsend > 0) {
      k_send_gather<<<nblk(A->nsend), 256, 0, s>>>(v, A->sendperm.get(), A->nsend, A->sendbuf.get());
      SP_LAUNCH();
    }
    SP_CUDA(cudaEventRecord(A->ev_send_ready, s));
    SP_CUDA(cudaStreamWaitEvent(c->comm_stream, A->ev_send_ready, 0));
    SP_TRY(c->exchange_dev(A->sendbuf.get(), A->send_off.data(), A->send_count.data(),
                           A->recvbuf.get(), A->recv_off.data(), A->recv_count.data(),
                           sizeof(double), c->comm_stream));
    SP_CUDA(cudaEventRecord(A->ev_recv_done, c->comm_stream));
    A->stat_nccl_sent += 8 * A->nsend;
    A->stat_nccl_recv += 8 * A->nrecv;
  }
  ++A->stat_setvals;
  // 3x3 blocks and no received contributions: the diagonal values go straight into bval
  const bool direct_bsr = A->bs == 3 && A->n_mixed == 0 && A->mb > 0 && !A->env_numeric_csr;
  if (nnz > 0) {
    // one contribution per nonzero: k_numeric_one; several of varying count (element COO):
    // k_numeric_seg_pipe<2, 2>.  SPMAT_NUMERIC_KERNEL selects the measured alternatives:
    // ilp, plain, seg (k_numeric_seg), warp, pipe4 (k_numeric_seg_pipe<4, 1>), pipe8 (<8, 8>)
    const char *nk = getenv("SPMAT_NUMERIC_KERNEL");
    int kind = (double)A->ncontrib > 1.5 * (double)nnz ? 9 : 0;  // 0 one/ilp, 9 pipe
    if (nk)
      kind = !strcmp(nk, "plain") ? 1 : !strcmp(nk, "seg") ? 2 : !strcmp(nk, "warp") ? 3
           : !strcmp(nk, "pipe8") ? 7 : !strcmp(nk, "pipe4") ? 8 : !strcmp(nk, "pipe") ? 9 : 0;
    const int64_t z0 = direct_bsr ? A->nnz_d : 0;  // direct_bsr: off-diagonal nonzeros only
    // one contribution per nonzero (every nonzero has at least one): jmap is the identity
    const bool one = A->ncontrib == nnz && !A->env_numeric_jmap;
    if (direct_bsr) {
      const int64_t blocks = std::min<int64_t>((A->mb + 7) / 8, (int64_t)A->comm->num_sms * 64);
      if (one)
        k_numeric_bsr3_one<<<(unsigned)blocks, 256, 0, s>>>(A->rowptr_d.get(), A->browptr.get(), A->perm.get(), v,
                                                            A->mb, A->bval.get(), mode);
      else
        k_numeric_bsr3<false><<<(unsigned)blocks, 256, 0, s>>>(A->rowptr_d.get(), A->browptr.get(), A->jmap.get(),
                                                               A->perm.get(), v, A->mb, A->bval.get(), mode);
      SP_LAUNCH();
    }
    if (nnz > z0) {
      if (kind == 3 && z0 == 0) {
        const int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)A->comm->num_sms * 64);
        k_numeric_warp<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(
            A->jmap.get(), A->perm.get(), v, (uint64_t)A->ncoo, A->nnz_d, nnz, A->val_d.get(), A->val_o.get(), mode);
      } else if (kind == 1) {
        k_numeric_local<<<nblk(nnz), 256, 0, s>>>(A->jmap.get(), A->perm.get(), v, (uint64_t)A->ncoo,
                                                  A->nnz_d, nnz, A->val_d.get(), A->val_o.get(), mode);
      } else if (kind >= 7 && z0 == 0) {
        const bool ins = mode == SPMAT_INSERT;
        const uint32_t *jm = A->jmap.get(), *pm = A->perm.get();
        double *vd = A->val_d.get(), *vo = A->val_o.get();
        // (kSeg, kTail): 7 (8,8)  8 (4,1)  9 (2,2).  C3, one box (ms): (8,8) 0.934, (4,1) 0.821,
        // (3,1) 0.821, (2,1) 0.805, (1,1) 0.85, (2,2) 0.755-0.767
        const bool mixed = A->n_mixed > 0;
        auto pick = [&](auto tag) -> const void * {
          constexpr int S = decltype(tag)::first, T = decltype(tag)::second;
          return mixed ? (ins ? (const void *)k_numeric_seg_pipe<S, T, true, true>
                              : (const void *)k_numeric_seg_pipe<S, T, false, true>)
                       : (ins ? (const void *)k_numeric_seg_pipe<S, T, true, false>
                              : (const void *)k_numeric_seg_pipe<S, T, false, false>);
        };
        const void *fn = kind == 7 ? pick(PipeCfg<8, 8>{}) : kind == 8 ? pick(PipeCfg<4, 1>{}) : pick(PipeCfg<2, 2>{});
        int per_sm = 0;
        SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
        const unsigned g = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((nnz + 255) / 256, (int64_t)A->comm->num_sms * std::max(per_sm, 1)));
        const int64_t nd = A->nnz_d;
        const uint32_t lim = A->n_mixed > 0 ? (uint32_t)A->ncoo : 0xffffffffu;
        void *args[] = {(void *)&jm, (void *)&pm, (void *)&v, (void *)&lim, (void *)&nd, (void *)&nnz, (void *)&vd, (void *)&vo};
        SP_CUDA(cudaLaunchKernel(fn, dim3(g), dim3(256), args, 0, s));
      } else if (kind == 2 && z0 == 0) {
        // contributions read 8 at a time (C3, same box: 1.149 ms vs 1.200 ms 4 at a time,
        // 1.206 ms for the plain serial loop)
        if (A->env_numeric_seg != 4)
          k_numeric_seg<8><<<nblk(nnz), 256, 0, s>>>(A->jmap.get(), A->perm.get(), v, (uint64_t)A->ncoo,
                                                     A->nnz_d, nnz, A->val_d.get(), A->val_o.get(), mode);
        else
          k_numeric_seg<4><<<nblk(nnz), 256, 0, s>>>(A->jmap.get(), A->perm.get(), v, (uint64_t)A->ncoo,
                                                     A->nnz_d, nnz, A->val_d.get(), A->val_o.get(), mode);
      } else if (one && !(nk && !strcmp(nk, "ilp"))) {
        constexpr int U = 8;
        const unsigned g = (unsigned)std::max<int64_t>(1, (nnz - z0 + 256 * U - 1) / (256 * U));
        const bool ins = mode == SPMAT_INSERT, mixed = A->n_mixed > 0;
        const uint32_t lim = (uint32_t)A->ncoo;
        const uint32_t *pm = A->perm.get();
        double *vd = A->val_d.get(), *vo = A->val_o.get();
        const int64_t nd = A->nnz_d;
        if (ins)
          mixed ? k_numeric_one<U, true, true><<<g, 256, 0, s>>>(pm, v, lim, z0, nd, nnz, vd, vo)
                : k_numeric_one<U, true, false><<<g, 256, 0, s>>>(pm, v, lim, z0, nd, nnz, vd, vo);
        else
          mixed ? k_numeric_one<U, false, true><<<g, 256, 0, s>>>(pm, v, lim, z0, nd, nnz, vd, vo)
                : k_numeric_one<U, false, false><<<g, 256, 0, s>>>(pm, v, lim, z0, nd, nnz, vd, vo);
      } else {
        const int64_t blocks = std::min<int64_t>((nnz - z0 + 256 * kNumU - 1) / (256 * kNumU),
                                                 (int64_t)A->comm->num_sms * 32);
        if (one)
          k_numeric_ilp<true><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(
              A->jmap.get(), A->perm.get(), v, (uint64_t)A->ncoo, A->nnz_d, nnz, A->val_d.get(), A->val_o.get(),
              mode, z0);
        else
          k_numeric_ilp<false><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(
              A->jmap.get(), A->perm.get(), v, (uint64_t)A->ncoo, A->nnz_d, nnz, A->val_d.get(), A->val_o.get(),
              mode, z0);
      }
      SP_LAUNCH();
    }
  }
  A->val_d_stale = direct_bsr;
  if (exchange) {
    SP_CUDA(cudaStreamWaitEvent(s, A->ev_recv_done, 0));
    if (A->n_mixed > 0) {
      k_numeric_mixed<<<nblk(A->n_mixed), 256, 0, s>>>(A->mixed.get(), A->n_mixed, A->jmap.get(),
                                                      A->perm.get(), v, A->recvbuf.get(),
                                                      (uint64_t)A->ncoo, A->nnz_d, A->val_d.get(),
                                                      A->val_o.get(), mode);
      SP_LAUNCH();
    }
  }
  SP_TRY(bsr_refresh(A, s, !direct_bsr));  // block copies of the values, if any
  A->values_set = true;
  return SPMAT_OK;
}

int spmat_get_info(spmat_t A, int64_t info[32]) {
  if (!A || !info) return fail(SPMAT_ERR_ARG, "spmat_get_info: null argument");
  const int64_t mode = A->comm->nranks == 1 ? 0 : (A->peer ? 2 : 1);
  int64_t v[32] = {A->rstart, A->rend, A->cstart, A->cend, A->nnz_d, A->nnz_o, A->n_ghost,
                   A->n_ro, A->ncontrib, A->nsend, A->nrecv, A->n_mixed, A->kernel_id,
                   A->n_rowblocks, A->max_row_nnz, A->plan_builds,
                   A->bs, A->ob_ok ? 1 : 0, A->ob_ok ? A->ob_w : A->ro_w, mode,
                   A->stat_nccl_sent, A->stat_nccl_recv, A->stat_nvlink_put, A->stat_mults,
                   A->stat_setvals, A->bs == 3 ? A->bsr_grid : A->tma_grid,
                   A->bs == 3 ? A->bsr_grid : A->tma_grid_tail,
                   A->halo ? (A->halo->peer_deferred ? 0 : (A->halo->peer ? 2 : 1)) : 0, 0};
  memcpy(info, v, sizeof v);
  return SPMAT_OK;
}

int spmat_check(spmat_t A) {
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_check: null matrix");
  DeviceGuard g(A->comm->device);
  SP_CUDA(cudaDeviceSynchronize());
  if (A->peer && A->halo_err.get()) {
    int e = 0;
    SP_CUDA(cudaMemcpy(&e, A->halo_err.get(), 4, cudaMemcpyDeviceToHost));
    if (e) return fail(SPMAT_ERR_NCCL, "device-initiated halo: a peer did not answer (timeout)");
  }
  return spmat_comm_check(A->comm);
}

int spmat_trace_read(spmat_t A, int64_t *host_buf, int64_t cap, int64_t *len) {
  if (!A || !len) return fail(SPMAT_ERR_ARG, "spmat_trace_read: null argument");
  DeviceGuard g(A->comm->device);
  SP_CUDA(cudaDeviceSynchronize());
  *len = (int64_t)A->trace.n;
  if (host_buf && cap > 0 && A->trace.n)
    SP_CUDA(cudaMemcpy(host_buf, A->trace.get(), 8 * std::min<int64_t>(cap, *len), cudaMemcpyDeviceToHost));
  return SPMAT_OK;
}

int spmat_halo_mode(spmat_t A) {
  if (!A) return -1;
  return A->comm->nranks == 1 ? 0 : (A->peer ? 2 : 1);
}

int spmat_get_halo_sf(spmat_t A, sf_t *borrowed) {
  if (!A || !borrowed) return fail(SPMAT_ERR_ARG, "spmat_get_halo_sf: null argument");
  DeviceGuard g(A->comm->device);
  SP_TRY(sf_ensure_peer(A->halo));  // collective on first call
  *borrowed = A->halo;
  return SPMAT_OK;
}

int spmat_export(spmat_t A, int what, void *host_buf, int64_t cap, int64_t *len) {
  if (!A || !len) return fail(SPMAT_ERR_ARG, "spmat_export: null argument");
  DeviceGuard g(A->comm->device);
  SP_CUDA(cudaDeviceSynchronize());
  if (what == 2 && A->val_d_stale) {  // values written straight into the 3x3 block copy
    SP_TRY(csr_sync(A, A->comm->setup_stream));
    SP_CUDA(cudaStreamSynchronize(A->comm->setup_stream));
  }
  const int P = A->comm->nranks;
  std::vector<int64_t> out;
  std::vector<double> outd;
  bool is_double = false;
  auto pull32 = [&](const int32_t *d, int64_t n) -> int {
    std::vector<int32_t> h(n);
    if (n) SP_CUDA(cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost));
    out.assign(h.begin(), h.end());
    return SPMAT_OK;
  };
  auto pullu32 = [&](const uint32_t *d, int64_t n) -> int {
    std::vector<uint32_t> h(n);
    if (n) SP_CUDA(cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost));
    out.assign(h.begin(), h.end());
    return SPMAT_OK;
  };
  auto pulld = [&](const double *d, int64_t n) -> int {
    outd.resize(n);
    if (n) SP_CUDA(cudaMemcpy(outd.data(), d, n * 8, cudaMemcpyDeviceToHost));
    is_double = true;
    return SPMAT_OK;
  };
  switch (what) {
    case 0: SP_TRY(pull32(A->rowptr_d.get(), A->m + 1)); break;
    case 1: SP_TRY(pull32(A->col_d.get(), A->nnz_d)); break;
    case 2: SP_TRY(pulld(A->val_d.get(), A->nnz_d)); break;
    case 3: {  // full-length offdiag row pointer from the compressed form
      std::vector<int64_t> rows, rp;
      SP_TRY(pull32(A->rows_o.get(), A->n_ro));
      rows = out;
      if (A->n_ro) {
        SP_TRY(pull32(A->rowptr_o.get(), A->n_ro + 1));
        rp = out;
      } else {
        rp.assign(1, 0);
      }
      out.assign(A->m + 1, 0);
      for (int64_t q = 0; q < A->n_ro; ++q) out[rows[q] + 1] = rp[q + 1] - rp[q];
      for (int64_t r = 0; r < A->m; ++r) out[r + 1] += out[r];
      break;
    }
    case 4: SP_TRY(pull32(A->col_o.get(), A->nnz_o)); break;
    case 5: SP_TRY(pulld(A->val_o.get(), A->nnz_o)); break;
    case 6:
      out.resize(A->n_ghost);
      if (A->n_ghost) SP_CUDA(cudaMemcpy(out.data(), A->colmap.get(), A->n_ghost * 8, cudaMemcpyDeviceToHost));
      break;
    case 7: SP_TRY(pullu32(A->jmap.get(), A->nnz_d + A->nnz_o + 1)); break;
    case 8:
    case 9: {
      SP_TRY(pullu32(A->perm.get(), A->ncontrib));
      std::vector<int64_t> perm = out;
      out.resize(perm.size());
      for (size_t t = 0; t < perm.size(); ++t) {
        int64_t p = perm[t];
        if (p < A->ncoo) {
          out[t] = what == 8 ? A->comm->rank : p;
        } else {
          int64_t q = p - A->ncoo;
          int s = (int)(std::upper_bound(A->recv_off.begin(), A->recv_off.end(), q) - A->recv_off.begin()) - 1;
          out[t] = what == 8 ? s : q - A->recv_off[s];
        }
      }
      break;
    }
    case 10: out = A->send_count; break;
    case 11: SP_TRY(pullu32(A->sendperm.get(), A->nsend)); break;
    case 12: out = A->recv_count; break;
    case 13: SP_TRY(pull32(A->rows_o.get(), A->n_ro)); break;
    default: return fail(SPMAT_ERR_ARG, "spmat_export: unknown what=%d", what);
  }
  (void)P;
  if (is_double) {
    *len = (int64_t)outd.size();
    if (host_buf && cap > 0) memcpy(host_buf, outd.data(), 8 * std::min<int64_t>(cap, *len));
  } else {
    *len = (int64_t)out.size();
    if (host_buf && cap > 0) memcpy(host_buf, out.data(), 8 * std::min<int64_t>(cap, *len));
  }
  return SPMAT_OK;
}

int spmat_destroy(spmat_t A) {
  if (!A) return SPMAT_OK;
  {
    DeviceGuard g(A->comm->device);
    cudaDeviceSynchronize();
    cg_graph_release(A);
    halo_peer_release(A);
    if (A->halo) sf_free(A->halo);
    for (cudaEvent_t e : A->pipe_ev) cudaEventDestroy(e);
    if (A->pipe_in) cudaStreamDestroy(A->pipe_in);
    if (A->pipe_out) cudaStreamDestroy(A->pipe_out);
    if (A->pipe_comp) cudaStreamDestroy(A->pipe_comp);
    if (A->pipe_comm) cudaStreamDestroy(A->pipe_comm);
    if (A->ev_send_ready) cudaEventDestroy(A->ev_send_ready);
    if (A->ev_recv_done) cudaEventDestroy(A->ev_recv_done);
    for (auto &v : A->prof_ev)
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    // DevBuf members free themselves in ~spmat_s (device still selected here)
    A->rowptr_d.release(); A->col_d.release(); A->val_d.release();
    A->rows_o.release(); A->rowptr_o.release(); A->col_o.release(); A->val_o.release();
    A->colmap.release(); A->lvec.release(); A->jmap.release(); A->perm.release();
    A->mixed.release(); A->sendperm.release(); A->sendbuf.release(); A->recvbuf.release();
    A->rbp.release(); A->sched.release(); A->block_order.release(); A->blocks4.release(); A->tail_ctr.release(); A->trace.release(); A->halo_flags.release(); A->ghost.release(); A->halo_puts.release(); A->halo_waits.release(); A->halo_counter.release(); A->halo_err.release(); A->longrows.release(); A->xstage.release(); A->ystage.release(); A->pipe_blocks4.release(); A->cg_r.release(); A->cg_p.release(); A->cg_q.release(); A->cg_partial.release(); A->cg_scalars.release(); A->cg_reduced.release();
  }
  delete A;
  return SPMAT_OK;
}

}  // extern "C"
