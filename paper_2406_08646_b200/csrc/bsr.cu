// bsr.cu -- 3x3 block-CSR diagonal block for multi-dof matrices (the paper's planned
// "block-CSR on GPU").
//
// spmat_set_block_size(A, 3) checks that the assembled diagonal CSR block is made of dense,
// aligned 3x3 blocks (true for node-block COO such as the 3-dof elasticity config C5) and keeps
// a block copy: browptr (block rows), bcol (one column index per block), bval (9 values per
// block, row-major).  Bytes per nonzero drop from 12 (8 value + 4 column) to 8.44 (8 value +
// 4/9 column), so the HBM-bound SpMV moves ~30 % fewer bytes.  bval is refreshed from the CSR
// values after every spmat_set_values_coo (the assembly plan stays the CSR one).
//
// k_spmv_bsr3 mirrors k_spmv_tma: persistent warp-specialised CTAs, a producer warp staging
// (bval, bcol, browptr) slices of a "row block" of block rows through cp.async.bulk into a
// 2-stage mbarrier ring, 8 consumer warps computing W lanes per block row.  A lane walks its
// blocks in ascending column order and adds v_i0*x_0, v_i1*x_1, v_i2*x_2 for each block row i,
// which with W = 1 is exactly the CSR row's left-to-right order.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstring>

#include "halo_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace spmat {

namespace {

constexpr int kT = 256;                    // consumer threads
constexpr int kCtaT = kT + 32;             // + producer warp
constexpr int kBudgetD = 2880;             // doubles per row block (9*blocks + 6*block rows): ~24 KB
constexpr int kCapD = kBudgetD + 576;      // stage capacity in doubles (a 64-block row fits)
constexpr int kMaxBR = kBudgetD / 6;       // block rows per row block
constexpr int kStagesB = 2;

struct __align__(16) BsrStage {
  double val[kCapD + 2];
  int col[(kCapD / 9 + 11) & ~3];  // multiples of 4 ints keep every array 16-byte aligned
  int rp[(kMaxBR + 11) & ~3];
  int4 hdr;  // br0, br1, bp0, bp1
  int4 ext;  // .x, .y: off-diagonal block rows [t0, t1) of this row block (fused MatMult)
};
constexpr size_t kBsrSmem = kStagesB * sizeof(BsrStage) + 2 * kStagesB * sizeof(unsigned long long);

#define GSTRIDE(t, n) \
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (n); t += (int64_t)gridDim.x * blockDim.x)

inline unsigned nb(int64_t n, int t = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, (int64_t)1 << 30));
}

// warp per block row: rows 3br..3br+2 share one column list made of aligned triples
__global__ void k_bsr_check(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                            int64_t mb, int *__restrict__ bad) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= mb) return;
  const int64_t r = 3 * warp;
  const int a0 = rowptr[r], a1 = rowptr[r + 1], a2 = rowptr[r + 2], a3 = rowptr[r + 3];
  const int len = a1 - a0;
  if (a2 - a1 != len || a3 - a2 != len || len % 3) {
    if (lane == 0) atomicOr(bad, 1);
    return;
  }
  for (int p = lane; p < len; p += 32) {
    const int c0 = col[a0 + p];
    bool ok = c0 == col[a1 + p] && c0 == col[a2 + p];
    ok = ok && ((p % 3 == 0) ? (c0 % 3 == 0) : (c0 == col[a0 + p - 1] + 1));
    if (!ok) atomicOr(bad, 1);
  }
}

__global__ void k_bsr_build(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                            int64_t mb, int32_t *__restrict__ browptr, int32_t *__restrict__ bcol) {
  GSTRIDE(br, mb + 1) {
    const int a = rowptr[3 * br];
    browptr[br] = a / 9;
    if (br < mb) {
      const int nblk_row = (rowptr[3 * br + 1] - a) / 3;
      for (int q = 0; q < nblk_row; ++q) bcol[a / 9 + q] = col[a + 3 * q] / 3;
    }
  }
}

// the inverse: val[rowptr[3br+i] + 3q + j] = bval[9*(bp0+q) + 3i + j]
__global__ void k_bsr_unrefresh(const int32_t *__restrict__ rowptr, const double *__restrict__ bval,
                                const int32_t *__restrict__ browptr, int64_t mb, double *__restrict__ val) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t br = warp; br < mb; br += nwarps) {
    const int bp0 = browptr[br], nbr = browptr[br + 1] - bp0;
    const int r0 = rowptr[3 * br], r1 = rowptr[3 * br + 1], r2 = rowptr[3 * br + 2];
    for (int v = lane; v < 9 * nbr; v += 32) {
      const int q = v / 9, i = (v % 9) / 3, j = v % 3;
      const int base = i == 0 ? r0 : (i == 1 ? r1 : r2);
      val[base + 3 * q + j] = bval[9 * (int64_t)bp0 + v];
    }
  }
}

// warp per block row: bval[9*(bp0+q) + 3i + j] = val[rowptr[3br+i] + 3q + j]
__global__ void k_bsr_refresh(const int32_t *__restrict__ rowptr, const double *__restrict__ val,
                              const int32_t *__restrict__ browptr, int64_t mb, double *__restrict__ bval) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t br = warp; br < mb; br += nwarps) {
    const int bp0 = browptr[br], nbr = browptr[br + 1] - bp0;
    const int r0 = rowptr[3 * br], r1 = rowptr[3 * br + 1], r2 = rowptr[3 * br + 2];
    for (int v = lane; v < 9 * nbr; v += 32) {
      const int q = v / 9, i = (v % 9) / 3, j = v % 3;
      const int base = i == 0 ? r0 : (i == 1 ? r1 : r2);
      bval[9 * (int64_t)bp0 + v] = val[base + 3 * q + j];
    }
  }
}

// row-block boundaries over block rows: cost(br) = 9*browptr[br] + 6*br
__global__ void k_bsr_candidates(const int32_t *__restrict__ browptr, int64_t mb, int64_t ncost,
                                 int32_t *__restrict__ cand) {
  GSTRIDE(t, ncost) {
    const int64_t target = t * (int64_t)kBudgetD;
    int64_t lo = 0, hi = mb;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (9 * (int64_t)browptr[mid] + 6 * mid < target) lo = mid + 1; else hi = mid;
    }
    cand[t] = (int32_t)lo;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cand[ncost] = (int32_t)mb;
}

__global__ void k_bsr_blocks4(const int32_t *__restrict__ bounds, const int32_t *__restrict__ browptr,
                              int64_t n, int4 *__restrict__ out) {
  GSTRIDE(t, n) {
    const int a = bounds[t], b = bounds[t + 1];
    out[t] = make_int4(a, b, browptr[a], browptr[b]);
  }
}

// FMA: each block row's 9 products accumulated with fused multiply-adds (half the fp64 pipe
// instructions; a different rounding, still within the 1e-12 bar and exact for integer data)
template <int W, bool FMA, int NT>
__device__ __forceinline__ void brows_w(int br0, int br1, int bp0, const int *__restrict__ rp,
                                        const int *__restrict__ sc, const double *__restrict__ sv,
                                        const double *__restrict__ x, double *__restrict__ y, int tid) {
  constexpr int U = 4;  // blocks per lane in flight
  const int lane = tid & (W - 1);
  for (int br = br0 + tid / W; br < br1; br += NT / W) {
    const int a = rp[br] - bp0, z = rp[br + 1] - bp0;
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    for (int e0 = a + lane; e0 < z; e0 += U * W) {
      double xv[U][3];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * W;
        const int c = e < z ? sc[e] : 0;
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) xv[u][jj] = __ldg(x + 3 * c + jj);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * W;
        if (e < z) {
          const double *v = sv + 9 * e;
#pragma unroll
          for (int jj = 0; jj < 3; ++jj) {
            if (FMA) {
              y0 = __fma_rn(v[jj], xv[u][jj], y0);
              y1 = __fma_rn(v[3 + jj], xv[u][jj], y1);
              y2 = __fma_rn(v[6 + jj], xv[u][jj], y2);
            } else {
              y0 = __dadd_rn(y0, __dmul_rn(v[jj], xv[u][jj]));
              y1 = __dadd_rn(y1, __dmul_rn(v[3 + jj], xv[u][jj]));
              y2 = __dadd_rn(y2, __dmul_rn(v[6 + jj], xv[u][jj]));
            }
          }
        }
      }
    }
    if (W > 1) {
      const unsigned mask = __activemask();
#pragma unroll
      for (int o = W >> 1; o > 0; o >>= 1) {
        y0 = __dadd_rn(y0, __shfl_down_sync(mask, y0, o, W));
        y1 = __dadd_rn(y1, __shfl_down_sync(mask, y1, o, W));
        y2 = __dadd_rn(y2, __shfl_down_sync(mask, y2, o, W));
      }
    }
    if (lane == 0) {
      y[3 * (int64_t)br] = y0;
      y[3 * (int64_t)br + 1] = y1;
      y[3 * (int64_t)br + 2] = y2;
    }
  }
}

// Fused off-diagonal blocks (NVLink halo): row blocks holding block rows with off-diagonal
// blocks are claimed LAST (by then the neighbours' ghost lines, stored at the start of their
// MatMult, have long landed); once the consumer warps have written such a block's diagonal
// y (named barrier), they add its off-diagonal block rows y[3br+i] += sum_b A_o(br,b) g(b):
// the off-diagonal product streams with the diagonal one instead of running as a separate
// latency-bound kernel.  The last CTA to finish releases the ghost buffer and ends the epoch.
struct BsrOff {
  const int2 *range;                    // per claim index: [t0, t1); nullptr: not fused
  const int32_t *rows, *rowptr, *col;   // ob_rows, ob_rowptr, ob_col
  const double *val;                    // ob_val
  const uint4 *ghost;                   // flagged ghost lines, buffer (epoch & 1) at ghost_stride
  int64_t ghost_stride;
  unsigned long long *epoch_ctr;
  const HaloWait *waits;
  int nwaits;
  unsigned int *done;                   // CTAs whose consumers finished (epoch end)
  int *err;
  // comm-warp mode: this epoch's puts, boundary row blocks claimed first, tail counters
  const HaloPut *puts;
  int nputs, put_chunks;
  int n_bblocks;                        // row blocks with off-diagonal block rows (claimed first)
  int64_t nobr;
  unsigned int *ctr;                    // [0] boundary-block warps done, [1] chunk claims, [2] comm warps done
  int wmax;                             // cap on the lanes per block row of the diagonal product
};

// W = 4 lanes per off-diagonal block row, every consumer thread of the CTA takes part
// (uniform loop bound: all lanes reach the shuffles).  Not inlined: the hot diagonal loop keeps
// its register budget.
static __device__ __noinline__ void bsr_off_rows(const BsrOff off, int t0, int t1, double *y, int tid,
                                                 unsigned long long epoch) {
  constexpr int W = 4, U = 2;
  const uint32_t flag = ll_flag(epoch);
  const uint4 *gl = off.ghost + (int64_t)(epoch & 1) * off.ghost_stride;
  const int sub = tid & (W - 1);
  for (int base = t0; base < t1; base += kT / W) {
    const int t = base + tid / W;
    const bool valid = t < t1;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (valid) {
      const int a = off.rowptr[t], z = off.rowptr[t + 1];
      for (int e0 = a + sub; e0 < z; e0 += U * W) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = e0 + u * W < z ? off.col[e0 + u * W] : -1;
        uint4 raw[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (c[u] >= 0) raw[u][j] = ll_load_raw(gl + 3 * (int64_t)c[u] + j);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (c[u] < 0) continue;
          const double *v = off.val + 9 * (int64_t)(e0 + u * W);
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double g = ll_value(gl + 3 * (int64_t)c[u] + j, raw[u][j], flag, off.err);
            s0 = __dadd_rn(s0, __dmul_rn(__ldg(v + j), g));
            s1 = __dadd_rn(s1, __dmul_rn(__ldg(v + 3 + j), g));
            s2 = __dadd_rn(s2, __dmul_rn(__ldg(v + 6 + j), g));
          }
        }
      }
    }
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) {
      s0 = __dadd_rn(s0, __shfl_down_sync(0xffffffffu, s0, o, W));
      s1 = __dadd_rn(s1, __shfl_down_sync(0xffffffffu, s1, o, W));
      s2 = __dadd_rn(s2, __shfl_down_sync(0xffffffffu, s2, o, W));
    }
    if (valid && sub == 0) {
      const int64_t r = 3 * (int64_t)off.rows[t];
      y[r] = __dadd_rn(y[r], s0);
      y[r + 1] = __dadd_rn(y[r + 1], s1);
      y[r + 2] = __dadd_rn(y[r + 2], s2);
    }
  }
}

// Comm-warp mode (NVLink halo, the default with 3x3 off-diagonal blocks): one warp of every
// CTA stores this rank's boundary x into the neighbours' ghost lines at kernel start, waits
// until the boundary row blocks (claimed first) are written, then adds the 3x3 off-diagonal
// block rows in chunks of 8 (4 lanes each) beside the consumers' streaming -- the k_spmv_tma
// design on 3x3 blocks.  The consumers lose one warp (7 instead of 8): a C5 row block holds
// ~11 block rows, which 7 warps still cover in one pass.  The last comm warp releases the
// ghost buffer and ends the epoch.
static __device__ __noinline__ void bsr_comm_tail(const BsrOff off, unsigned long long epoch, double *y,
                                                  int consumer_warps) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    const unsigned target = (unsigned)(consumer_warps * off.n_bblocks);
    const long long t0 = clock64();
    unsigned ns = 64;
    while (ld_acquire_gpu(off.ctr) < target) {
      if (clock64() - t0 > kSpinLimit) {
        atomicExch(off.err, 2);
        break;
      }
      __nanosleep(ns);
      ns = ns < 256 ? 2 * ns : ns;
    }
  }
  __syncwarp();
  constexpr int W = 4, U = 2;
  const uint32_t flag = ll_flag(epoch);
  const uint4 *gl = off.ghost + (int64_t)(epoch & 1) * off.ghost_stride;
  const int sub = lane & (W - 1);
  const int64_t n_chunks = (off.nobr + 32 / W - 1) / (32 / W);
  for (;;) {
    int64_t c = 0;
    if (lane == 0) c = atomicAdd(off.ctr + 1, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= n_chunks) break;
    const int64_t t = c * (32 / W) + lane / W;
    const bool valid = t < off.nobr;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (valid) {
      const int a = off.rowptr[t], z = off.rowptr[t + 1];
      for (int e0 = a + sub; e0 < z; e0 += U * W) {
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cc[u] = e0 + u * W < z ? off.col[e0 + u * W] : -1;
        uint4 raw[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (cc[u] >= 0) raw[u][j] = ll_load_raw(gl + 3 * (int64_t)cc[u] + j);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (cc[u] < 0) continue;
          const double *v = off.val + 9 * (int64_t)(e0 + u * W);
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double g = ll_value(gl + 3 * (int64_t)cc[u] + j, raw[u][j], flag, off.err);
            s0 = __dadd_rn(s0, __dmul_rn(__ldg(v + j), g));
            s1 = __dadd_rn(s1, __dmul_rn(__ldg(v + 3 + j), g));
            s2 = __dadd_rn(s2, __dmul_rn(__ldg(v + 6 + j), g));
          }
        }
      }
    }
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) {
      s0 = __dadd_rn(s0, __shfl_down_sync(0xffffffffu, s0, o, W));
      s1 = __dadd_rn(s1, __shfl_down_sync(0xffffffffu, s1, o, W));
      s2 = __dadd_rn(s2, __shfl_down_sync(0xffffffffu, s2, o, W));
    }
    if (valid && sub == 0) {
      const int64_t r = 3 * (int64_t)off.rows[t];
      y[r] = __dadd_rn(__ldcg(y + r), s0);
      y[r + 1] = __dadd_rn(__ldcg(y + r + 1), s1);
      y[r + 2] = __dadd_rn(__ldcg(y + r + 2), s2);
    }
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(off.ctr + 2, 1u) == gridDim.x - 1) {
      atomicExch(off.ctr, 0u);
      atomicExch(off.ctr + 1, 0u);
      atomicExch(off.ctr + 2, 0u);
      __threadfence();
      for (int q = 0; q < off.nwaits; ++q) st_release_sys(off.waits[q].peer_done, epoch);
      *off.epoch_ctr = epoch;  // this MatMult is done
    }
  }
}

// MODE 0: diagonal only; 1: off-diagonal blocks added by the consumers (claimed last);
// 2: comm warp (puts + off-diagonal tail, boundary row blocks claimed first)
template <bool FMA, int MODE>
__global__ void __launch_bounds__(kCtaT, 3)
    k_spmv_bsr3(const int4 *__restrict__ blocks, int n_blocks, const int32_t *__restrict__ browptr,
                const int32_t *__restrict__ bcol, const double *__restrict__ bval,
                const double *__restrict__ x, double *__restrict__ y, unsigned int *__restrict__ sched,
                const BsrOff off) {
  extern __shared__ __align__(128) unsigned char smem[];
  BsrStage *st = reinterpret_cast<BsrStage *>(smem);
  // this MatMult's halo epoch (fused off-diagonal blocks): read by every CTA before its
  // consumers finish, so before the last CTA stores it back
  constexpr bool FUSE = MODE == 1;
  constexpr int NT = MODE == 2 ? kT - 32 : kT;  // consumer threads
  const unsigned long long epoch = MODE ? *off.epoch_ctr + 1ull : 0ull;
  unsigned long long *full = reinterpret_cast<unsigned long long *>(smem + kStagesB * sizeof(BsrStage));
  unsigned long long *empty = full + kStagesB;
  const int tid = threadIdx.x, warp = tid >> 5, lane32 = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStagesB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (MODE == 2 && warp == NT / 32 + 1) {  // comm warp: puts, then the off-diagonal tail
    for (int c = blockIdx.x; c < off.put_chunks; c += gridDim.x)
      halo_put_warp(off.puts, off.nputs, c, x, epoch, off.err);
    bsr_comm_tail(off, epoch, y, NT / 32);
    return;
  }
  if (warp == NT / 32) {  // producer
    if (lane32 != 0) return;
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int b = (int)atomicAdd(sched, 1u);
    int b_next = (int)atomicAdd(sched, 1u);
    int4 H = b < n_blocks ? blocks[b] : make_int4(0, 0, 0, 0);
    for (int it = 0;; ++it) {
      const int s = it % kStagesB;
      if (it >= kStagesB) mbar_wait(&empty[s], (uint32_t)(((it / kStagesB) - 1) & 1));
      if (b >= n_blocks) {
        st[s].hdr = make_int4(-1, 0, 0, 0);
        mbar_arrive_tx(&full[s], 0);
        __threadfence();
        if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
          atomicExch(sched, 0u);
          atomicExch(sched + 1, 0u);
        }
        return;
      }
      st[s].hdr = H;
      if (FUSE) {
        const int2 rg = off.range[b];
        st[s].ext = make_int4(rg.x, rg.y, 0, 0);
      } else if (MODE == 2) {
        st[s].ext = make_int4(0, 0, b < off.n_bblocks ? 1 : 0, 0);
      }
      const int64_t v0 = 9 * (int64_t)H.z, v1 = 9 * (int64_t)H.w;
      const int64_t va = v0 & ~1ll, ve = (v1 + 1) & ~1ll;
      const int ca = H.z & ~3, ce = (H.w + 3) & ~3;
      const int ra = H.x & ~3, re = (H.y + 4) & ~3;
      mbar_arrive_tx(&full[s], (uint32_t)((ve - va) * 8 + (ce - ca) * 4 + (re - ra) * 4));
      if (ve > va) bulk_g2s(st[s].val, bval + va, (uint32_t)((ve - va) * 8), &full[s], policy);
      if (ce > ca) bulk_g2s(st[s].col, bcol + ca, (ce - ca) * 4, &full[s], policy);
      bulk_g2s(st[s].rp, browptr + ra, (re - ra) * 4, &full[s], policy);
      b = b_next;
      if (b < n_blocks) {
        b_next = (int)atomicAdd(sched, 1u);
        H = blocks[b];
      }
    }
  }
  // comm-warp mode: boundary row blocks are claimed first, so a warp publishes how many it wrote
  // (one fence + one atomic per warp) when it meets its first other claim
  unsigned bdone = 0;
  bool published = MODE != 2;
  for (int it = 0;; ++it) {  // consumers
    const int s = it % kStagesB;
    mbar_wait(&full[s], (uint32_t)((it / kStagesB) & 1));
    const int4 h = st[s].hdr;
    const int bnd = MODE == 2 ? st[s].ext.z : 0;
    if (!published && (h.x < 0 || !bnd)) {
      published = true;
      __syncwarp();
      if (lane32 == 0 && bdone) {
        __threadfence();
        atomicAdd(off.ctr, bdone);
      }
    }
    if (h.x < 0) break;
    const int br0 = h.x, br1 = h.y, bp0 = h.z;
    const int t0 = FUSE ? st[s].ext.x : 0, t1 = FUSE ? st[s].ext.y : 0;
    const double *sv = st[s].val + ((9 * (int64_t)bp0) & 1);
    const int *sc = st[s].col + (bp0 & 3);
    const int *rp = st[s].rp - (br0 & ~3);
    const int nbr = br1 - br0, wm = off.wmax;
    if (nbr * 2 > NT || wm <= 1) brows_w<1, FMA, NT>(br0, br1, bp0, rp, sc, sv, x, y, tid);
    else if (nbr * 4 > NT || wm <= 2) brows_w<2, FMA, NT>(br0, br1, bp0, rp, sc, sv, x, y, tid);
    else if (nbr * 8 > NT || wm <= 4) brows_w<4, FMA, NT>(br0, br1, bp0, rp, sc, sv, x, y, tid);
    else if (nbr * 16 > NT || wm <= 8) brows_w<8, FMA, NT>(br0, br1, bp0, rp, sc, sv, x, y, tid);
    else if (nbr * 32 > NT || wm <= 16) brows_w<16, FMA, NT>(br0, br1, bp0, rp, sc, sv, x, y, tid);
    else brows_w<32, FMA, NT>(br0, br1, bp0, rp, sc, sv, x, y, tid);
    __syncwarp();
    if (lane32 == 0) mbar_arrive(&empty[s]);
    bdone += bnd;
    if (FUSE && t1 > t0) {  // this block's diagonal y is written by all consumer warps: add A_o g
      asm volatile("bar.sync 1, %0;" ::"r"(kT) : "memory");
      bsr_off_rows(off, t0, t1, y, tid, epoch);
    }
  }
  if (FUSE) {  // the last CTA whose consumers are done ends the MatMult's halo epoch
    asm volatile("bar.sync 2, %0;" ::"r"(kT) : "memory");
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(off.done, 1u) == gridDim.x - 1) {
        atomicExch(off.done, 0u);
        __threadfence();
        for (int w = 0; w < off.nwaits; ++w) st_release_sys(off.waits[w].peer_done, epoch);
        *off.epoch_ctr = epoch;
      }
    }
  }
}

// ------------------------------------------------------------------ off-diagonal 3x3 blocks
// warp per row triple t of the compressed off-diagonal rows: rows 3br..3br+2, equal column
// lists made of aligned ghost triples (3 dofs of one ghost node)
__global__ void k_bsr_o_check(const int32_t *__restrict__ rows, const int32_t *__restrict__ rowptr,
                              const int32_t *__restrict__ col, int64_t nobr, int *__restrict__ bad) {
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nobr) return;
  const int r0 = rows[3 * t];
  const int a0 = rowptr[3 * t], a1 = rowptr[3 * t + 1], a2 = rowptr[3 * t + 2], a3 = rowptr[3 * t + 3];
  const int len = a1 - a0;
  if (r0 % 3 || rows[3 * t + 1] != r0 + 1 || rows[3 * t + 2] != r0 + 2 || a2 - a1 != len || a3 - a2 != len ||
      len % 3) {
    if (lane == 0) atomicOr(bad, 1);
    return;
  }
  for (int p = lane; p < len; p += 32) {
    const int c0 = col[a0 + p];
    bool ok = c0 == col[a1 + p] && c0 == col[a2 + p];
    ok = ok && ((p % 3 == 0) ? (c0 % 3 == 0) : (c0 == col[a0 + p - 1] + 1));
    if (!ok) atomicOr(bad, 1);
  }
}

__global__ void k_bsr_o_build(const int32_t *__restrict__ rows, const int32_t *__restrict__ rowptr,
                              const int32_t *__restrict__ col, int64_t nobr, int32_t *__restrict__ ob_rows,
                              int32_t *__restrict__ ob_rowptr, int32_t *__restrict__ ob_col) {
  GSTRIDE(t, nobr + 1) {
    const int a = rowptr[3 * t];
    ob_rowptr[t] = a / 9;
    if (t < nobr) {
      ob_rows[t] = rows[3 * t] / 3;
      const int nb_row = (rowptr[3 * t + 1] - a) / 3;
      for (int q = 0; q < nb_row; ++q) ob_col[a / 9 + q] = col[a + 3 * q] / 3;
    }
  }
}

// warp per block row: ob_val[9*(b0+q) + 3i + j] = val_o[rowptr_o[3t+i] + 3q + j]
__global__ void k_bsr_o_refresh(const int32_t *__restrict__ rowptr, const double *__restrict__ val,
                                const int32_t *__restrict__ ob_rowptr, int64_t nobr, double *__restrict__ ob_val) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < nobr; t += nwarps) {
    const int b0 = ob_rowptr[t], n = ob_rowptr[t + 1] - b0;
    const int r0 = rowptr[3 * t], r1 = rowptr[3 * t + 1], r2 = rowptr[3 * t + 2];
    for (int v = lane; v < 9 * n; v += 32) {
      const int q = v / 9, i = (v % 9) / 3, j = v % 3;
      const int base = i == 0 ? r0 : (i == 1 ? r1 : r2);
      ob_val[9 * (int64_t)b0 + v] = val[base + 3 * q + j];
    }
  }
}

// Off-diagonal SpMV-add y += A_o lvec on 3x3 blocks (block CSR L1163).
// W lanes per block row; a lane takes blocks a+lane, a+lane+W, ... (ascending columns), loads
// each block's 3 ghost values (flagged lines of this epoch, or the NCCL ghost vector) once for
// the block's 3 rows, and adds v_i0*g_0, v_i1*g_1, v_i2*g_2 per row i (W = 1: the CSR row's
// left-to-right order); then a shuffle tree over the W lanes.
// Standalone kernel (NCCL ghost vector, isolated parts, SPMAT_BSR_FUSE=0); the full MatMult
// with the NVLink halo adds the off-diagonal blocks inside k_spmv_bsr3 (bsr_off_rows).  The
// last CTA releases the ghost buffer to the senders and advances the epoch (NVLink mode, cur).
// (Measured and dropped: this kernel as a PDL dependent sized to fit beside the block SpMV,
// doing its reads before pdl_wait -- 2 warps per SM starved by the saturated HBM: C5 P=4
// 0.93 ms per MatMult against 0.74 ms sequential.)
constexpr int kObT = 256;
template <int W, bool PEER>
__global__ void __launch_bounds__(kObT)
    k_offdiag_bsr3(const int32_t *__restrict__ ob_rows, const int32_t *__restrict__ ob_rowptr,
                   const int32_t *__restrict__ ob_col, const double *__restrict__ ob_val,
                   const uint4 *ghost_base, int64_t ghost_stride, const double *lvec, double *y,
                   int64_t nobr, const HaloWait *__restrict__ waits, int nwaits,
                   unsigned long long *epoch_ctr, unsigned int *counter, int *err, int cur) {
  // the epoch counter is written only by the MatMult's last kernel, never by the block SpMV
  // this grid overlaps, so it may be read before pdl_wait.  cur = 0: the lines of the last
  // completed epoch (an isolated off-diagonal part, nothing to end)
  pdl_wait();
  const unsigned long long epoch = PEER ? *epoch_ctr + (cur ? 1ull : 0ull) : 0ull;
  const uint32_t flag = ll_flag(epoch);
  const uint4 *gl = PEER ? ghost_base + (int64_t)(epoch & 1) * ghost_stride : nullptr;
  const int sub = threadIdx.x & (W - 1);
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  constexpr int U = 2;  // blocks per lane in flight
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nobr * W; base += step) {
    const int64_t q = (base + threadIdx.x) / W;
    const bool valid = q < nobr;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (valid) {
      const int a = ob_rowptr[q], z = ob_rowptr[q + 1];
      for (int e0 = a + sub; e0 < z; e0 += U * W) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = e0 + u * W < z ? ob_col[e0 + u * W] : -1;
        double g[U][3];
        if (PEER) {
          uint4 raw[U][3];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < 3; ++j)
              if (c[u] >= 0) raw[u][j] = ll_load_raw(gl + 3 * (int64_t)c[u] + j);
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < 3; ++j)
              g[u][j] = c[u] >= 0 ? ll_value(gl + 3 * (int64_t)c[u] + j, raw[u][j], flag, err) : 0.0;
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < 3; ++j) g[u][j] = c[u] >= 0 ? __ldcg(lvec + 3 * (int64_t)c[u] + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (c[u] < 0) continue;
          const double *v = ob_val + 9 * (int64_t)(e0 + u * W);
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            s0 = __dadd_rn(s0, __dmul_rn(__ldg(v + j), g[u][j]));
            s1 = __dadd_rn(s1, __dmul_rn(__ldg(v + 3 + j), g[u][j]));
            s2 = __dadd_rn(s2, __dmul_rn(__ldg(v + 6 + j), g[u][j]));
          }
        }
      }
    }
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) {
      s0 = __dadd_rn(s0, __shfl_down_sync(0xffffffffu, s0, o, W));
      s1 = __dadd_rn(s1, __shfl_down_sync(0xffffffffu, s1, o, W));
      s2 = __dadd_rn(s2, __shfl_down_sync(0xffffffffu, s2, o, W));
    }
    if (valid && sub == 0) {
      const int64_t r = 3 * (int64_t)ob_rows[q];
      y[r] = __dadd_rn(__ldcg(y + r), s0);
      y[r + 1] = __dadd_rn(__ldcg(y + r + 1), s1);
      y[r + 2] = __dadd_rn(__ldcg(y + r + 2), s2);
    }
  }
  if (!PEER || !cur) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      atomicExch(counter, 0u);
      for (int w = 0; w < nwaits; ++w) st_release_sys(waits[w].peer_done, epoch);
      *epoch_ctr = epoch;  // this MatMult is done
    }
  }
}

// per row block (br0, br1): off-diagonal block rows [t0, t1) with br0 <= ob_rows[t] < br1
__global__ void k_bsr_obrange(const int4 *__restrict__ blk, int64_t nbk, const int32_t *__restrict__ ob_rows,
                              int64_t nobr, int2 *__restrict__ rng, uint32_t *__restrict__ f_in,
                              uint32_t *__restrict__ f_out) {
  GSTRIDE(b, nbk) {
    int64_t lo = 0, hi = nobr;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ob_rows[mid] < blk[b].x) lo = mid + 1; else hi = mid;
    }
    const int64_t t0 = lo;
    hi = nobr;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ob_rows[mid] < blk[b].y) lo = mid + 1; else hi = mid;
    }
    rng[b] = make_int2((int)t0, (int)lo);
    f_in[b] = lo > t0 ? 1u : 0u;
    f_out[b] = lo > t0 ? 0u : 1u;
  }
}

__global__ void k_bsr_permute(const int4 *__restrict__ nat, const int2 *__restrict__ rng,
                              const int32_t *__restrict__ order, int64_t nbk, int4 *__restrict__ blk,
                              int2 *__restrict__ out_rng) {
  GSTRIDE(c, nbk) {
    blk[c] = nat[order[c]];
    out_rng[c] = rng[order[c]];
  }
}

#define CUB_CALL2(tmp, call_with_tmp)                                          \
  do {                                                                         \
    size_t temp_storage_bytes = 0;                                             \
    void *d_temp_storage = nullptr;                                            \
    SP_CUDA(call_with_tmp);                                                    \
    if (temp_storage_bytes > (tmp).n) SP_TRY((tmp).alloc(temp_storage_bytes)); \
    d_temp_storage = (tmp).get();                                              \
    SP_CUDA(call_with_tmp);                                                    \
  } while (0)

}  // namespace

int bsr_refresh(spmat_s *A, cudaStream_t s, bool diag) {
  if (A->bs != 3) return SPMAT_OK;
  if (diag && A->mb > 0) {
    k_bsr_refresh<<<nb(A->mb * 32), 256, 0, s>>>(A->rowptr_d.get(), A->val_d.get(), A->browptr.get(),
                                                  A->mb, A->bval.get());
    SP_LAUNCH();
  }
  if (A->ob_ok && A->obr > 0) {
    k_bsr_o_refresh<<<nb(A->obr * 32), 256, 0, s>>>(A->rowptr_o.get(), A->val_o.get(), A->ob_rowptr.get(),
                                                     A->obr, A->ob_val.get());
    SP_LAUNCH();
  }
  return SPMAT_OK;
}

int csr_sync(spmat_s *A, cudaStream_t s) {
  if (!A->val_d_stale) return SPMAT_OK;
  if (A->mb > 0) {
    k_bsr_unrefresh<<<nb(A->mb * 32), 256, 0, s>>>(A->rowptr_d.get(), A->bval.get(), A->browptr.get(), A->mb,
                                                    A->val_d.get());
    SP_LAUNCH();
  }
  A->val_d_stale = false;
  return SPMAT_OK;
}

int bsr_spmv(spmat_s *A, const double *x, double *y, cudaStream_t s, int mode) {
  BsrOff off{};
  off.wmax = A->env_bsr_wmax;
  if (mode) {  // NVLink halo: off-diagonal blocks inside the kernel, which ends the epoch
    off.range = A->ob_range.get();
    off.rows = A->ob_rows.get();
    off.rowptr = A->ob_rowptr.get();
    off.col = A->ob_col.get();
    off.val = A->ob_val.get();
    off.ghost = A->ghost.get();
    off.ghost_stride = A->ghost_stride;
    off.epoch_ctr = A->d_epoch.get();
    off.waits = A->halo_waits.get();
    off.nwaits = A->n_waits;
    off.done = A->ob_done.get();
    off.err = A->halo_err.get();
  }
  if (mode == 2) {  // comm warps: this epoch's puts and the off-diagonal tail
    off.puts = A->halo_puts.get();
    off.nputs = A->n_puts;
    off.put_chunks = A->put_chunks_total;
    off.n_bblocks = (int)A->ob_nbblocks;
    off.nobr = A->obr;
    off.ctr = A->ob_ctr.get();
  }
  auto kern = mode == 1 ? (A->env_bsr_fma ? k_spmv_bsr3<true, 1> : k_spmv_bsr3<false, 1>)
            : mode == 2 ? (A->env_bsr_fma ? k_spmv_bsr3<true, 2> : k_spmv_bsr3<false, 2>)
                        : (A->env_bsr_fma ? k_spmv_bsr3<true, 0> : k_spmv_bsr3<false, 0>);
  if (mode == 2) {  // comm warps spin on the peers' lines: every CTA co-resident
    SP_CUDA(launch_coop(kern, (unsigned)A->bsr_grid, kCtaT, kBsrSmem, s, (const int4 *)A->bblocks4.get(),
                        (int)A->n_brblocks, (const int32_t *)A->browptr.get(), (const int32_t *)A->bcol.get(),
                        (const double *)A->bval.get(), x, y, A->bsched.get(), off));
    return SPMAT_OK;
  }
  kern<<<(unsigned)A->bsr_grid, kCtaT, kBsrSmem, s>>>(A->bblocks4.get(), (int)A->n_brblocks, A->browptr.get(),
                                                    A->bcol.get(), A->bval.get(), x, y, A->bsched.get(), off);
  SP_LAUNCH();
  return SPMAT_OK;
}

// y += A_o lvec on the 3x3 block copy (standalone kernel)
template <int W>
static cudaError_t launch_ob(spmat_s *A, double *y, const double *lvec, cudaStream_t s, unsigned grid,
                             int cur) {
  const bool peer = lvec == nullptr;
  return launch_pdl(peer ? k_offdiag_bsr3<W, true> : k_offdiag_bsr3<W, false>, grid, kObT, 0, s, (const int32_t *)A->ob_rows.get(),
                    (const int32_t *)A->ob_rowptr.get(), (const int32_t *)A->ob_col.get(),
                    (const double *)A->ob_val.get(), peer ? (const uint4 *)A->ghost.get() : nullptr,
                    A->ghost_stride, lvec, y, A->obr,
                    peer ? (const HaloWait *)A->halo_waits.get() : nullptr, peer ? A->n_waits : 0,
                    peer ? A->d_epoch.get() : nullptr, peer ? A->halo_counter.get() : nullptr,
                    peer ? A->halo_err.get() : nullptr, cur);
}

int bsr_offdiag(spmat_s *A, double *y, const double *lvec, cudaStream_t s, bool cur) {
  const int64_t work = A->obr * A->ob_w;
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + kObT - 1) / kObT, 16L * A->comm->num_sms));
  cudaError_t e;
  switch (A->ob_w) {
    case 1: e = launch_ob<1>(A, y, lvec, s, grid, cur ? 1 : 0); break;
    case 2: e = launch_ob<2>(A, y, lvec, s, grid, cur ? 1 : 0); break;
    case 8: e = launch_ob<8>(A, y, lvec, s, grid, cur ? 1 : 0); break;
    default: e = launch_ob<4>(A, y, lvec, s, grid, cur ? 1 : 0); break;
  }
  SP_CUDA(e);
  return SPMAT_OK;
}

// 3x3 block copy of the off-diagonal block, when it is made of aligned blocks (else the CSR
// off-diagonal kernels stay in use)
static int bsr_o_setup(spmat_s *A, cudaStream_t st) {
  A->ob_ok = false;
  if (A->n_ro == 0 || A->n_ro % 3) return SPMAT_OK;
  const int64_t nobr = A->n_ro / 3;
  DevBuf<int> bad;
  SP_TRY(bad.alloc(1));
  SP_CUDA(cudaMemsetAsync(bad.get(), 0, 4, st));
  k_bsr_o_check<<<nb(nobr * 32), 256, 0, st>>>(A->rows_o.get(), A->rowptr_o.get(), A->col_o.get(), nobr, bad.get());
  SP_LAUNCH();
  int hbad = 0;
  SP_CUDA(cudaMemcpyAsync(&hbad, bad.get(), 4, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  if (hbad) return SPMAT_OK;
  A->obr = nobr;
  A->onnzb = A->nnz_o / 9;
  SP_TRY(A->ob_rows.alloc(nobr));
  SP_TRY(A->ob_rowptr.alloc(nobr + 1));
  SP_TRY(A->ob_col.alloc(A->onnzb));
  SP_TRY(A->ob_val.alloc(9 * A->onnzb));
  k_bsr_o_build<<<nb(nobr + 1), 256, 0, st>>>(A->rows_o.get(), A->rowptr_o.get(), A->col_o.get(), nobr,
                                              A->ob_rows.get(), A->ob_rowptr.get(), A->ob_col.get());
  SP_LAUNCH();
  // lanes per block row: the largest power of two <= 8 with >= 2 blocks per lane on average
  A->ob_w = 1;
  while (A->ob_w < 8 && 4 * A->ob_w * nobr <= A->onnzb) A->ob_w *= 2;
  if (const char *w = getenv("SPMAT_OB_W")) {
    const int v = atoi(w);
    if (v == 1 || v == 2 || v == 4 || v == 8) A->ob_w = v;
  }
  A->ob_ok = true;
  if (const char *e = getenv("SPMAT_BSR_OFFDIAG")) A->ob_ok = atoi(e) != 0;
  return SPMAT_OK;
}

static int bsr_o_env(spmat_s *A) {
  const char *e = getenv("SPMAT_NUMERIC_BSR");
  A->env_numeric_csr = e && atoi(e) == 0;
  // fused multiply-adds in the block SpMV by default: half the fp64 instructions, and C5 runs at
  // the 1 kW power cap -- measured 0.8-1.4 % faster on one box (2.760 / 2.752 vs 2.782 / 2.791 ms)
  e = getenv("SPMAT_BSR_FMA");
  A->env_bsr_fma = !(e && atoi(e) == 0);
  // lanes per block row of the diagonal product: at most 8 (C5: ~11 block rows of 27 blocks
  // per row block; 16 lanes fill more threads but spend ~40 % of the instructions on the
  // shuffle reductions -- 8 lanes: 1.086 G -> 0.770 G instructions, 2.79 -> 2.62 ms at P=1 under
  // the power cap, 0.641 -> 0.629 ms at P=4; 4 lanes: 2.92 ms).  SPMAT_BSR_WMAX overrides.
  e = getenv("SPMAT_BSR_WMAX");
  A->env_bsr_wmax = e ? std::max(1, atoi(e)) : 8;
  // off-diagonal blocks with the NVLink halo: 2 = comm warps of the block SpMV (puts + tail,
  // default), 1 = added by the consumers themselves (measured slower: each boundary row block
  // stalls its CTA's stage ring for a ghost-read latency chain, 0.859 vs 0.836 ms at P=4),
  // 0 = standalone put kernel + block SpMV + standalone off-diagonal kernel
  // Default per rank: comm warps when the off-diagonal block rows are >= 2.5 % of the rank's
  // block rows (C5 interior ranks at P=4: 0.635 vs 0.650 ms), else the standalone kernels (one
  // neighbour, C5 P=2: 1.280 vs 1.295 ms -- the 8th consumer warp is worth more there).  Ranks
  // may differ: both modes store the same flagged lines into the same peer buffers.
  e = getenv("SPMAT_BSR_FUSE");
  A->bsr_fuse_mode = e ? atoi(e) : (A->obr * 40 >= A->mb ? 2 : 0);
  if (A->bsr_fuse_mode < 0 || A->bsr_fuse_mode > 2) A->bsr_fuse_mode = 0;
  return SPMAT_OK;
}

// Claim order of the block SpMV with off-diagonal blocks, and per claim index the range
// [t0, t1) of off-diagonal block rows inside the row block.  Comm-warp mode: row blocks with
// off-diagonal block rows FIRST (the comm warps add them while the rest streams); in-kernel
// mode: LAST (by then every neighbour's ghost lines have landed).
static int bsr_claim_order(spmat_s *A, cudaStream_t st) {
  const bool boundary_first = A->bsr_fuse_mode != 1;
  const int64_t nbk = A->n_brblocks;
  DevBuf<int4> nat;
  DevBuf<int2> rng;
  DevBuf<uint32_t> f_in, f_out;
  DevBuf<int32_t> order;
  DevBuf<int> dn;
  DevBuf<char> tmp;
  SP_TRY(nat.alloc(nbk));
  SP_TRY(rng.alloc(nbk));
  SP_TRY(f_in.alloc(nbk));
  SP_TRY(f_out.alloc(nbk));
  SP_TRY(order.alloc(nbk));
  SP_TRY(dn.alloc(2));
  SP_CUDA(cudaMemcpyAsync(nat.get(), A->bblocks4.get(), nbk * sizeof(int4), cudaMemcpyDeviceToDevice, st));
  k_bsr_obrange<<<nb(nbk), 256, 0, st>>>(nat.get(), nbk, A->ob_rows.get(), A->obr, rng.get(), f_in.get(), f_out.get());
  SP_LAUNCH();
  uint32_t *fa = boundary_first ? f_in.get() : f_out.get(), *fb = boundary_first ? f_out.get() : f_in.get();
  CUB_CALL2(tmp, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes, thrust::counting_iterator<int32_t>(0),
                                            fa, order.get(), dn.get(), (int)nbk, st));
  int nfirst = 0;
  SP_CUDA(cudaMemcpyAsync(&nfirst, dn.get(), 4, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  CUB_CALL2(tmp, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes, thrust::counting_iterator<int32_t>(0),
                                            fb, order.get() + nfirst, dn.get() + 1, (int)nbk, st));
  A->ob_nbblocks = boundary_first ? nfirst : (int64_t)nbk - nfirst;
  SP_TRY(A->ob_range.alloc(nbk));
  k_bsr_permute<<<nb(nbk), 256, 0, st>>>(nat.get(), rng.get(), order.get(), nbk, A->bblocks4.get(), A->ob_range.get());
  SP_LAUNCH();
  SP_TRY(A->ob_done.alloc(1));
  SP_CUDA(cudaMemsetAsync(A->ob_done.get(), 0, 4, st));
  SP_TRY(A->ob_ctr.alloc(3));
  SP_CUDA(cudaMemsetAsync(A->ob_ctr.get(), 0, 12, st));
  SP_CUDA(cudaStreamSynchronize(st));
  return SPMAT_OK;
}

static int bsr_setup(spmat_s *A) {
  cudaStream_t st = A->comm->setup_stream;
  // the caller's spmat_set_values_coo may still be writing val_d on its own stream, and this
  // (host-synchronising) call reads the CSR on the setup stream: wait for the device first
  SP_CUDA(cudaDeviceSynchronize());
  const int64_t mb = A->m / 3;
  DevBuf<int> bad;
  SP_TRY(bad.alloc(1));
  SP_CUDA(cudaMemsetAsync(bad.get(), 0, 4, st));
  if (mb > 0) {
    k_bsr_check<<<nb(mb * 32), 256, 0, st>>>(A->rowptr_d.get(), A->col_d.get(), mb, bad.get());
    SP_LAUNCH();
  }
  int hbad = 0;
  SP_CUDA(cudaMemcpyAsync(&hbad, bad.get(), 4, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  if (hbad) return fail(SPMAT_ERR_ARG, "spmat_set_block_size: the diagonal block is not made of aligned 3x3 blocks");
  const int64_t nnzb = A->nnz_d / 9;
  A->mb = mb;
  A->nnzb = nnzb;
  SP_TRY(A->browptr.alloc(mb + 1 + 8));
  SP_TRY(A->bcol.alloc(nnzb + 8));
  SP_TRY(A->bval.alloc(9 * nnzb + 8));
  k_bsr_build<<<nb(mb + 1), 256, 0, st>>>(A->rowptr_d.get(), A->col_d.get(), mb, A->browptr.get(), A->bcol.get());
  SP_LAUNCH();
  // longest block row must fit one stage
  std::vector<int32_t> h(mb + 1);
  SP_CUDA(cudaMemcpyAsync(h.data(), A->browptr.get(), (mb + 1) * 4, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  for (int64_t br = 0; br < mb; ++br)
    if (9 * (int64_t)(h[br + 1] - h[br]) > kCapD - kBudgetD)
      return fail(SPMAT_ERR_ARG, "spmat_set_block_size: a block row has more than %d blocks", (kCapD - kBudgetD) / 9);
  // row blocks over block rows
  const int64_t total = 9 * nnzb + 6 * mb;
  const int64_t ncost = (total + kBudgetD - 1) / kBudgetD;
  DevBuf<int32_t> cand, uniq;
  DevBuf<int> dn;
  DevBuf<char> tmp;
  SP_TRY(cand.alloc(ncost + 1));
  SP_TRY(uniq.alloc(ncost + 1));
  SP_TRY(dn.alloc(1));
  k_bsr_candidates<<<nb(ncost), 256, 0, st>>>(A->browptr.get(), mb, ncost, cand.get());
  SP_LAUNCH();
  CUB_CALL2(tmp, cub::DeviceSelect::Unique(d_temp_storage, temp_storage_bytes, cand.get(), uniq.get(),
                                           dn.get(), (int)(ncost + 1), st));
  int nu = 0;
  SP_CUDA(cudaMemcpyAsync(&nu, dn.get(), 4, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  A->n_brblocks = nu - 1;
  SP_TRY(A->bblocks4.alloc(std::max(nu - 1, 1)));
  if (nu > 1) {
    k_bsr_blocks4<<<nb(nu - 1), 256, 0, st>>>(uniq.get(), A->browptr.get(), nu - 1, A->bblocks4.get());
    SP_LAUNCH();
  }
  SP_TRY(A->bsched.alloc(2));
  SP_CUDA(cudaMemsetAsync(A->bsched.get(), 0, 8, st));
  SP_CUDA(cudaFuncSetAttribute(k_spmv_bsr3<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsrSmem));
  SP_CUDA(cudaFuncSetAttribute(k_spmv_bsr3<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsrSmem));
  SP_CUDA(cudaFuncSetAttribute(k_spmv_bsr3<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsrSmem));
  SP_CUDA(cudaFuncSetAttribute(k_spmv_bsr3<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsrSmem));
  SP_CUDA(cudaFuncSetAttribute(k_spmv_bsr3<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsrSmem));
  SP_CUDA(cudaFuncSetAttribute(k_spmv_bsr3<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsrSmem));
  int per_sm = 0;
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_bsr3<false, 0>, kCtaT, kBsrSmem));
  A->bsr_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(per_sm, 1) * A->comm->num_sms,
                                                           std::max<int64_t>(A->n_brblocks, 1)));
  SP_TRY(bsr_o_setup(A, st));
  SP_TRY(bsr_o_env(A));
  if (A->ob_ok && A->n_brblocks > 0) SP_TRY(bsr_claim_order(A, st));
  A->bs = 3;
  A->kernel_id = 4;
  if (A->values_set) SP_TRY(bsr_refresh(A, st));
  SP_CUDA(cudaStreamSynchronize(st));
  return SPMAT_OK;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_set_block_size(spmat_t A, int bs) {
  SP_NVTX("spmat_set_block_size");
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_set_block_size: null matrix");
  DeviceGuard g(A->comm->device);
  cg_graph_release(A);  // a captured CG iteration would still launch the old kernel
  if (bs == 1) {
    if (A->val_d_stale) {  // the values live in bval: bring the CSR copy up to date first
      SP_CUDA(cudaDeviceSynchronize());
      SP_TRY(csr_sync(A, A->comm->setup_stream));
      SP_CUDA(cudaStreamSynchronize(A->comm->setup_stream));
    }
    A->bs = 1;
    A->kernel_id = A->kernel_id_csr;
    return SPMAT_OK;
  }
  if (bs != 3) return fail(SPMAT_ERR_ARG, "spmat_set_block_size: only 1 and 3 are supported");
  if (A->m % 3 || A->n % 3) return fail(SPMAT_ERR_ARG, "spmat_set_block_size: local sizes not multiples of 3");
  if (A->bs == 3) return SPMAT_OK;
  return bsr_setup(A);
}

}  // extern "C"
