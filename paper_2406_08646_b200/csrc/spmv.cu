// spmv.cu -- CSR SpMV kernels for sm_100a (diagonal and off-diagonal blocks of MPIAIJ).
//
// MatMult on MPIAIJ: y = A_d x_local + A_o lvec.  The paper's runs
// used the vendor csrMV (cuSPARSE); here every kernel is hand-written.
//
// SpMV is HBM-bound (2 flops per >= 12 bytes of val+col, AI ~0.15 flop/B): no tensor cores.
// Default diagonal kernel (KERNEL_TMA): persistent CTAs stream "row blocks" of the CSR --
// the val, col and row-pointer slices of a block land in a shared-memory stage through
// cp.async.bulk (the TMA engine's 1-D copy) tracked by an mbarrier, kStages blocks in
// flight per CTA, so DRAM requests never wait for the arithmetic.  The arithmetic then walks
// rows straight out of shared memory with W lanes per row (W per row block from its row count
// -- the row-statistics selector -- so every block is done in one pass): with W = 1 (3D
// 7-point stencils) lane l owns row r0 + l, so a
// warp's x gathers hit consecutive x entries (coalesced), and each row is summed left to
// right from +0.0 with separately rounded products -- bit-identical to a serial CSR loop.
//
// Row blocks: boundaries where the running cost rowptr[r] + kAlpha * r crosses a multiple of
// the budget (kBudget, or less when a smaller budget lets the consumers finish every block in
// one round of x gathers -- spmv_prepare), plus a block of its own for every row longer than
// kLong; so a block has at most kBudget / kAlpha rows and at most kBudget + kLong nonzeros
// (fits one stage).
//
// Alternatives kept for A/B measurement (SPMAT_SPMV_KERNEL=stream|vector): a non-persistent
// CTA-per-row-block kernel that stages products in shared memory, and a plain sub-warp
// vector CSR kernel.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "halo_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace spmat {

constexpr int kThreads = 256;                 // CTA size
constexpr int kBudget = 2048;                 // row-block cost budget (nonzeros + kAlpha*rows)
constexpr int kAlpha = 2;
constexpr int kMaxRows = kBudget / kAlpha;    // max rows per row block
constexpr int kLong = 512;                    // rows longer than this get their own block
constexpr int kCap = kBudget + kLong;         // max nonzeros of a staged row block
constexpr int kStages = 2;                    // row blocks in flight per CTA

enum { KERNEL_STREAM = 1, KERNEL_VECTOR = 2, KERNEL_TMA = 3, KERNEL_DIRECT = 5 };
constexpr int64_t kSmallBytes = 16ll << 20;  // below this the direct kernel (latency-bound sizes)

// one shared-memory stage; every array starts 16-byte aligned (bulk-copy requirement)
struct __align__(16) TmaStage {
  double val[kCap + 2];    // p0 rounded down to even
  int col[kCap + 4];       // p0 rounded down to a multiple of 4
  int rp[kMaxRows + 8];    // r0 rounded down to a multiple of 4, through r1
  int4 hdr;                // r0, r1, p0, p1 of the block in this stage
  int4 flags;              // .x = 1: a boundary block (rows with off-diagonal entries)
};
constexpr size_t kTmaSmem = kStages * sizeof(TmaStage) + 2 * kStages * sizeof(unsigned long long);

#define GRID_STRIDE(t, n) \
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (n); t += (int64_t)gridDim.x * blockDim.x)

static inline unsigned nblk(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)1 << 30));
}

// ------------------------------------------------------------------ row-block schedule
// candidate t < n_cost: first row r with rowptr[r] + kAlpha * r >= t * kBudget
__global__ void k_rb_candidates(const int32_t *__restrict__ rowptr, int64_t m, int64_t n_cost,
                                int32_t *__restrict__ cand, int budget) {
  GRID_STRIDE(t, n_cost) {
    const int64_t target = t * (int64_t)budget;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)rowptr[mid] + kAlpha * mid < target) lo = mid + 1; else hi = mid;
    }
    cand[t] = (int32_t)lo;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cand[n_cost] = (int32_t)m;
}

__global__ void k_long_rows(const int32_t *__restrict__ rowptr, int64_t m,
                            uint32_t *__restrict__ flag, int32_t *__restrict__ maxlen) {
  GRID_STRIDE(r, m) {
    const int32_t len = rowptr[r + 1] - rowptr[r];
    flag[r] = len > kLong ? 1u : 0u;
    atomicMax(maxlen, len);
  }
}

__global__ void k_long_bounds(const int32_t *__restrict__ rows, int64_t n,
                              int32_t *__restrict__ cand) {
  GRID_STRIDE(t, n) {
    cand[2 * t] = rows[t];
    cand[2 * t + 1] = rows[t] + 1;
  }
}

// flag[b] = 1 if row block b holds a row with off-diagonal entries (rows_o sorted)
__global__ void k_boundary_blocks(const int2 *__restrict__ rb, int64_t nb, const int32_t *__restrict__ rows_o,
                                  int64_t nro, uint32_t *__restrict__ flag, uint32_t *__restrict__ nflag) {
  GRID_STRIDE(b, nb) {
    const int r0 = rb[b].x, r1 = rb[b + 1].x;
    int64_t lo = 0, hi = nro;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rows_o[mid] < r0) lo = mid + 1; else hi = mid;
    }
    const uint32_t f = (lo < nro && rows_o[lo] < r1) ? 1u : 0u;
    flag[b] = f;
    nflag[b] = 1u - f;
  }
}

__global__ void k_scatter_ro(const int32_t *__restrict__ rows_o, int64_t nro, int32_t *__restrict__ ro_of_row) {
  GRID_STRIDE(q, nro) ro_of_row[rows_o[q]] = (int32_t)q;
}

// blocks4[c] = (r0, r1, p0, p1) of the row block claimed c-th (order == nullptr: identity)
__global__ void k_blocks4(const int2 *__restrict__ rb, const int32_t *__restrict__ order, int64_t nb,
                          int4 *__restrict__ out) {
  GRID_STRIDE(c, nb) {
    const int b = order ? order[c] : (int)c;
    const int2 A = rb[b], B = rb[b + 1];
    out[c] = make_int4(A.x, B.x, A.y, B.y);
  }
}

__global__ void k_rb_pairs(const int32_t *__restrict__ rows, const int32_t *__restrict__ rowptr,
                           int64_t n, int2 *__restrict__ out) {
  GRID_STRIDE(t, n) out[t] = make_int2(rows[t], rowptr[rows[t]]);
}

// W lanes per row: lane l of a row's group sums elements a+l, a+l+W, ... (8 in flight), then
// a shuffle reduction; W = 1 is a plain left-to-right sum (the serial CSR order)
template <int W>
__device__ __forceinline__ void rows_w(int r0, int r1, int p0, const int *__restrict__ rp,
                                       const int *__restrict__ sc, const double *__restrict__ sv,
                                       const double *__restrict__ x, double *__restrict__ y, int tid) {
  constexpr int U = 8;
  const int lane = tid & (W - 1);
  for (int r = r0 + tid / W; r < r1; r += kThreads / W) {
    const int a = rp[r] - p0, z = rp[r + 1] - p0;
    double acc = 0.0;
    for (int e0 = a + lane; e0 < z; e0 += U * W) {
      int cc[U];
      double vv[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * W;
        cc[u] = e < z ? sc[e] : 0;
        vv[u] = e < z ? sv[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + cc[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (e0 + u * W < z) acc = __dadd_rn(acc, __dmul_rn(vv[u], xv[u]));
    }
    if (W > 1) {
      const unsigned mask = __activemask();
#pragma unroll
      for (int o = W >> 1; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(mask, acc, o, W));
    }
    if (lane == 0) y[r] = acc;
  }
}

constexpr int kConsumerWarps = kThreads / 32;
// SPMAT_TRACE=1 record per CTA (globaltimer ns): consumer start, puts out, last block done,
// consumer end, comm warp saw the boundary blocks, comm warp tail done
constexpr int kTraceCta = 6;
constexpr int kCtaThreads = kThreads + 64;  // + producer warp + comm warp

__global__ void __launch_bounds__(kCtaThreads, 3)
    k_spmv_tma(const int4 *__restrict__ blocks, int n_blocks, const int32_t *__restrict__ rowptr,
               const int32_t *__restrict__ col, const double *__restrict__ val,
               const double *__restrict__ x, double *__restrict__ y,
               unsigned int *__restrict__ sched, const SpmvHalo halo, const SpmvTail tail) {
  extern __shared__ __align__(128) unsigned char smem[];
  TmaStage *st = reinterpret_cast<TmaStage *>(smem);
  unsigned long long *full = reinterpret_cast<unsigned long long *>(smem + kStages * sizeof(TmaStage));
  unsigned long long *empty = full + kStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane32 = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // (launch_pdl) the barrier set-up above may overlap the previous kernel
  // this MatMult's halo epoch: read by every CTA before any claim, so before the last CTA
  // (which only exists once every CTA has claimed) stores it back
  const unsigned long long epoch = halo.epoch_ctr ? *halo.epoch_ctr + 1ull : 0ull;
  __syncthreads();
  unsigned long long *trc = tail.trace ? tail.trace + kTraceCta * (size_t)blockIdx.x : nullptr;
  if (warp == kConsumerWarps + 1) {  // ---------------- comm warp: halo puts, then the tail
    for (int c = blockIdx.x; c < halo.put_chunks; c += gridDim.x)
      halo_put_warp(halo.puts, halo.nputs, c, x, epoch, halo.err);
    if (trc && lane32 == 0) trc[1] = gtimer();  // this CTA's puts are out
    if (tail.enabled) tail_warp(tail, epoch, halo.err, y, trc, kConsumerWarps);
    return;
  }
  if (warp == kConsumerWarps) {  // ---------------- producer warp
    if (lane32 != 0) return;
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    // claims run two ahead: the atomic for block it+2 is in flight while block it is issued,
    // so only the (order, bounds) loads of the next block sit on the producer's path.
    // Claim index c is row block c of the claim order (boundary blocks first when the tail is
    // fused).
    const int n_total = n_blocks;
    auto bounds = [&](int c, int4 &H) { H = blocks[c]; };  // one 16-byte load: (r0, r1, p0, p1)
    int b = (int)atomicAdd(sched, 1u);
    int b_next = (int)atomicAdd(sched, 1u);
    int4 H = make_int4(0, 0, 0, 0);
    if (b < n_total) bounds(b, H);
    for (int it = 0;; ++it) {
      const int s = it % kStages;
      if (it >= kStages) mbar_wait(&empty[s], (uint32_t)(((it / kStages) - 1) & 1));
      if (b >= n_total) {  // out of work: terminal header, then hand the counter back
        st[s].hdr = make_int4(-1, 0, 0, 0);
        mbar_arrive_tx(&full[s], 0);
        __threadfence();
        if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
          atomicExch(sched, 0u);
          atomicExch(sched + 1, 0u);
          if (halo.bump && halo.epoch_ctr) *halo.epoch_ctr = epoch;  // this MatMult is done
        }
        return;
      }
      {
        const int r0 = H.x, r1 = H.y, p0 = H.z, p1 = H.w;
        st[s].hdr = H;
        st[s].flags.x = (tail.enabled && b < tail.n_bblocks) ? 1 : 0;
        if (p1 - p0 > kCap) {  // a single long row: k_spmv_long computes it
          mbar_arrive_tx(&full[s], 0);
        } else {
          const int va = p0 & ~1, ve = (p1 + 1) & ~1;
          const int ca = p0 & ~3, ce = (p1 + 3) & ~3;
          const int ra = r0 & ~3, re = (r1 + 4) & ~3;
          mbar_arrive_tx(&full[s], (uint32_t)((ve - va) * 8 + (ce - ca) * 4 + (re - ra) * 4));
          if (ve > va) bulk_g2s(st[s].val, val + va, (ve - va) * 8, &full[s], policy);
          if (ce > ca) bulk_g2s(st[s].col, col + ca, (ce - ca) * 4, &full[s], policy);
          bulk_g2s(st[s].rp, rowptr + ra, (re - ra) * 4, &full[s], policy);
        }
      }
      b = b_next;
      if (b < n_total) {
        b_next = (int)atomicAdd(sched, 1u);
        bounds(b, H);
      }
    }
  }
  // ---------------- consumer warps
  if (trc && tid == 0) trc[0] = gtimer();
  // boundary blocks are claimed before everything else, so a warp publishes how many it
  // wrote (one fence + one atomic per warp) when it meets its first other claim
  unsigned bdone = 0;
  bool published = !tail.enabled;
  auto publish = [&]() {
    if (published) return;
    published = true;
    __syncwarp();
    if (lane32 == 0 && bdone) {
      __threadfence();
      atomicAdd(tail.ctr, bdone);
    }
  };
  for (int it = 0;; ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (uint32_t)((it / kStages) & 1));
    const int4 h = st[s].hdr;
    const int r0 = h.x, r1 = h.y, p0 = h.z, p1 = h.w;
    if (r0 < 0 || !st[s].flags.x) publish();
    if (r0 == -1) {
      if (trc && tid == 0) trc[2] = gtimer();
      break;
    }
    const int boundary = st[s].flags.x;
    if (p1 - p0 <= kCap) {
      const double *sv = st[s].val + (p0 & 1);  // sv[e - p0] = val[e]
      const int *sc = st[s].col + (p0 & 3);
      const int *rp = st[s].rp - (r0 & ~3);     // rp[r] = rowptr[r]
      // lanes per row, per block: the largest power of two that still covers every row of
      // the block in one pass (W = 1 for stencil-like blocks: left-to-right row sums)
      const int nrows = r1 - r0;
      if (nrows * 2 > kThreads) rows_w<1>(r0, r1, p0, rp, sc, sv, x, y, tid);
      else if (nrows * 4 > kThreads) rows_w<2>(r0, r1, p0, rp, sc, sv, x, y, tid);
      else if (nrows * 8 > kThreads) rows_w<4>(r0, r1, p0, rp, sc, sv, x, y, tid);
      else if (nrows * 16 > kThreads) rows_w<8>(r0, r1, p0, rp, sc, sv, x, y, tid);
      else if (nrows * 32 > kThreads) rows_w<16>(r0, r1, p0, rp, sc, sv, x, y, tid);
      else rows_w<32>(r0, r1, p0, rp, sc, sv, x, y, tid);
    }
    __syncwarp();
    if (lane32 == 0) mbar_arrive(&empty[s]);
    bdone += boundary ? 1u : 0u;
  }
  if (trc) {
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    if (tid == 0) trc[3] = gtimer();
  }
}

// one CTA per row longer than kCap nonzeros (rows the staged kernels skip)
__global__ void __launch_bounds__(kThreads) k_spmv_long(const int32_t *__restrict__ rows,
                                                        const int32_t *__restrict__ rowptr,
                                                        const int32_t *__restrict__ col,
                                                        const double *__restrict__ val,
                                                        const double *__restrict__ x,
                                                        double *__restrict__ y) {
  __shared__ double red[kThreads / 32];
  const int r = rows[blockIdx.x];
  const int a = rowptr[r], z = rowptr[r + 1];
  if (z - a <= kCap) return;
  double s = 0.0;
  for (int e = a + threadIdx.x; e < z; e += kThreads)
    s = __dadd_rn(s, __dmul_rn(ld_stream(val + e), __ldg(x + ld_stream(col + e))));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t = __dadd_rn(t, red[w]);
    y[r] = t;
  }
}

// ------------------------------------------------------------------ alternative: stream
// One CTA per row block: coalesced val/col loads, products parked in shared memory, then
// one thread per row sums them left to right.
__global__ void __launch_bounds__(kThreads) k_spmv_stream(
    const int2 *__restrict__ rb, const int32_t *__restrict__ rowptr,
    const int32_t *__restrict__ col, const double *__restrict__ val,
    const double *__restrict__ x, double *__restrict__ y) {
  __shared__ double prod[kCap];
  const int2 A = rb[blockIdx.x], B = rb[blockIdx.x + 1];
  const int r0 = A.x, r1 = B.x, p0 = A.y, n = B.y - A.y;
  if (n > kCap) return;  // long row: k_spmv_long
  const int tid = threadIdx.x;
  constexpr int U = 8;
  for (int base = 0; base < n; base += kThreads * U) {
    int c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * kThreads + tid;
      c[u] = e < n ? ld_stream(col + p0 + e) : 0;
      v[u] = e < n ? ld_stream(val + p0 + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * kThreads + tid;
      if (e < n) prod[e] = __dmul_rn(v[u], __ldg(x + c[u]));
    }
  }
  __syncthreads();
  for (int r = r0 + tid; r < r1; r += kThreads) {
    const int a = rowptr[r] - p0, z = rowptr[r + 1] - p0;
    double s = 0.0;
    for (int e = a; e < z; ++e) s = __dadd_rn(s, prod[e]);
    y[r] = s;
  }
}

// ------------------------------------------------------------------ small matrices: direct
// Latency-bound sizes (a few MB, L2-resident: C1, Kuu-sized): no persistent grid, no
// mbarrier ring, no claim counter -- W lanes per row straight from global memory, each lane
// issuing 8 (col, val) loads, then their 8 x gathers, before it sums; one launch-to-store
// chain of rowptr -> col/val -> x -> y.  W = 1 sums each row left to right (serial order).
template <int W>
__global__ void __launch_bounds__(128) k_spmv_direct(const int32_t *__restrict__ rowptr,
                                                     const int32_t *__restrict__ col,
                                                     const double *__restrict__ val,
                                                     const double *__restrict__ x,
                                                     double *__restrict__ y, int64_t m) {
  pdl_wait();
  constexpr int U = 8;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / W;
  const int lane = threadIdx.x & (W - 1);
  const bool valid = row < m;
  const int a = valid ? __ldg(rowptr + row) : 0, z = valid ? __ldg(rowptr + row + 1) : 0;
  double s = 0.0;
  for (int e0 = a + lane; e0 < z; e0 += U * W) {
    int c[U];
    double v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * W;
      c[u] = e < z ? __ldg(col + e) : 0;
      v[u] = e < z ? __ldg(val + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * W < z) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
  }
#pragma unroll
  for (int o = W >> 1; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o, W));
  if (valid && lane == 0) y[row] = s;
}

// Small matrices with the NVLink halo (Kuu-sized systems on several GPUs): ONE cooperative
// launch per MatMult -- warps of the first CTAs store this rank's boundary x as flagged lines into
// the neighbours' ghost buffers (halo_put_warp) at kernel start, every row group computes its
// diagonal sum as in k_spmv_direct, and a row with off-diagonal entries (ro_of_row[r] = q >= 0)
// adds them from the ghost lines once they carry this epoch: y = S_d + S_o, written once.  The
// last CTA releases the ghost buffer to the senders and ends the epoch.  Cooperative, because
// rows spin on data the peers' CTAs store.
template <int W>
__global__ void __launch_bounds__(128) k_spmv_direct_halo(
    const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col, const double *__restrict__ val,
    const double *__restrict__ x, double *__restrict__ y, int64_t m, const int32_t *__restrict__ ro_of_row,
    const int32_t *__restrict__ rowptr_o, const int32_t *__restrict__ col_o, const double *__restrict__ val_o,
    const SpmvHalo halo, const uint4 *ghost, int64_t ghost_stride, const HaloWait *__restrict__ waits, int nwaits,
    unsigned int *counter) {
  constexpr int U = 8;
  const unsigned long long epoch = *halo.epoch_ctr + 1ull;
  const int warp_g = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (warp_g < halo.put_chunks) halo_put_warp(halo.puts, halo.nputs, warp_g, x, epoch, halo.err);
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / W;
  const int lane = threadIdx.x & (W - 1);
  const bool valid = row < m;
  int a = valid ? __ldg(rowptr + row) : 0, z = valid ? __ldg(rowptr + row + 1) : 0;
  double s = 0.0;
  for (int e0 = a + lane; e0 < z; e0 += U * W) {
    int c[U];
    double v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * W;
      c[u] = e < z ? __ldg(col + e) : 0;
      v[u] = e < z ? __ldg(val + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * W < z) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
  }
#pragma unroll
  for (int o = W >> 1; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o, W));
  // off-diagonal part of the row (ghost lines of this epoch), reduced over the same W lanes
  const int q = valid ? __ldg(ro_of_row + row) : -1;
  double so = 0.0;
  if (q >= 0) {
    const uint4 *gl = ghost + (int64_t)(epoch & 1) * ghost_stride;
    const uint32_t flag = ll_flag(epoch);
    a = __ldg(rowptr_o + q);
    z = __ldg(rowptr_o + q + 1);
    for (int e = a + lane; e < z; e += W)
      so = __dadd_rn(so, __dmul_rn(__ldg(val_o + e), ll_load(gl + __ldg(col_o + e), flag, halo.err)));
  }
  const unsigned qmask = __ballot_sync(0xffffffffu, q >= 0);
  if (qmask) {
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) so = __dadd_rn(so, __shfl_down_sync(0xffffffffu, so, o, W));
  }
  if (valid && lane == 0) y[row] = q >= 0 ? __dadd_rn(s, so) : s;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      atomicExch(counter, 0u);
      __threadfence();
      for (int w = 0; w < nwaits; ++w) st_release_sys(waits[w].peer_done, epoch);
      *halo.epoch_ctr = epoch;  // this MatMult is done
    }
  }
}

// ------------------------------------------------------------------ alternative: vector
template <int W>
__global__ void __launch_bounds__(256) k_spmv_vector(const int32_t *__restrict__ rowptr,
                                                     const int32_t *__restrict__ col,
                                                     const double *__restrict__ val,
                                                     const double *__restrict__ x,
                                                     double *__restrict__ y, int64_t m) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / W;
  const int lane = threadIdx.x % W;
  if (row >= m) return;
  const int a = rowptr[row], z = rowptr[row + 1];
  double s = 0.0;
  for (int e = a + lane; e < z; e += W)
    s = __dadd_rn(s, __dmul_rn(ld_stream(val + e), __ldg(x + ld_stream(col + e))));
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o, W));
  if (lane == 0) y[row] = s;
}

// ------------------------------------------------------------------ off-diagonal block
// y[rows_o[q]] = y[rows_o[q]] + (left-to-right sum over the compressed off-diagonal row)
__global__ void __launch_bounds__(256) k_spmv_offdiag(const int32_t *__restrict__ rows,
                                                      const int32_t *__restrict__ rowptr,
                                                      const int32_t *__restrict__ col,
                                                      const double *__restrict__ val,
                                                      const double *__restrict__ lvec,
                                                      const uint4 *__restrict__ ghost,
                                                      int64_t ghost_stride,
                                                      const unsigned long long *__restrict__ epoch_ctr,
                                                      double *__restrict__ y, int64_t nro, int W,
                                                      int *err) {
  pdl_wait();
  // NCCL mode: lvec.  NVLink mode: the ghost lines of the last completed epoch (already landed).
  const unsigned long long epoch = ghost ? *epoch_ctr : 0ull;
  const uint4 *gl = ghost ? ghost + (int64_t)(epoch & 1) * ghost_stride : nullptr;
  if (W == 1) {
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x * kRowsU; t0 < nro; t0 += (int64_t)gridDim.x * blockDim.x * kRowsU)
      offdiag_rows_u<kRowsU>(t0 + threadIdx.x, blockDim.x, nro, rows, rowptr, col, val, gl, lvec,
                             ll_flag(epoch), err, y);
    return;
  }
  // block-uniform loop bound: every lane reaches the shuffles in offdiag_row_w
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < nro * W; t0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = (t0 + threadIdx.x) / W;
    offdiag_row_w(q, q < nro, W, rows, rowptr, col, val, gl, lvec, ll_flag(epoch), err, y);
  }
}

// ------------------------------------------------------------------ host side
#define CUB_CALL(tmp, call_with_tmp)                                           \
  do {                                                                         \
    size_t temp_storage_bytes = 0;                                             \
    void *d_temp_storage = nullptr;                                            \
    SP_CUDA(call_with_tmp);                                                    \
    if (temp_storage_bytes > (tmp).n) SP_TRY((tmp).alloc(temp_storage_bytes)); \
    d_temp_storage = (tmp).get();                                              \
    SP_CUDA(call_with_tmp);                                                    \
  } while (0)

static int lanes_for(double mean) {  // W lanes per row from the mean row length
  if (mean <= 12) return 1;
  if (mean <= 24) return 2;
  if (mean <= 48) return 4;
  if (mean <= 96) return 8;
  if (mean <= 192) return 16;
  return 32;
}

static int tma_setup(spmat_s *A) {
  // per device (the attribute belongs to the current device's context): set at every setup
  SP_CUDA(cudaFuncSetAttribute(k_spmv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
  int per_sm = 0;
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_tma, kCtaThreads, kTmaSmem));
  // SPMAT_RESERVE_SMS leaves SMs free for concurrently running kernels (e.g. NCCL's)
  int reserve = 0;
  if (const char *e = getenv("SPMAT_RESERVE_SMS")) reserve = std::max(0, atoi(e));
  const int64_t sms = std::max<int64_t>(1, A->comm->num_sms - reserve);
  const int64_t full = (int64_t)std::max(per_sm, 1) * sms;
  A->tma_grid = (int)std::max<int64_t>(1, std::min<int64_t>(full, A->n_rowblocks));
  // with the fused off-diagonal add every CTA's comm warp takes chunks of off-diagonal rows:
  // small matrices (fewer row blocks than chunks) get extra CTAs that only do that
  const int64_t per = A->ro_w == 1 ? 32 * kRowsU : 32 / A->ro_w;
  const int64_t chunks = (A->n_ro + per - 1) / per;
  A->tma_grid_tail = (int)std::max<int64_t>(A->tma_grid, std::min<int64_t>(full, chunks));
  return SPMAT_OK;
}

int spmv_prepare(spmat_s *A, cudaStream_t st) {
  const int64_t m = A->m, nnz = A->nnz_d;
  {
    const char *e = getenv("SPMAT_FUSE");
    A->env_no_fuse = e && !strcmp(e, "0");
    e = getenv("SPMAT_FUSE_TAIL");
    A->env_no_tail = e && !strcmp(e, "0");
    e = getenv("SPMAT_NUMERIC_SEG");
    A->env_numeric_seg = (e && atoi(e) == 4) ? 4 : 8;
    e = getenv("SPMAT_NUMERIC_JMAP");
    A->env_numeric_jmap = e && atoi(e) != 0;
    e = getenv("SPMAT_PIPE_CHUNKS");
    const int c = e ? atoi(e) : 0;
    A->env_pipe_chunks = c >= 2 && c <= 256 ? c : 16;
    e = getenv("SPMAT_PIPE_CHUNKS_ASYNC");
    const int ca = e ? atoi(e) : 0;
    A->env_pipe_chunks_async = ca >= 1 && ca <= 256 ? ca : 1;
  }
  A->kernel_id = KERNEL_TMA;
  // small matrices on one rank (or with the NCCL halo): the direct kernel; the NVLink halo
  // needs the comm warps of the bulk-copy kernel
  // (several ranks with the NVLink halo: k_spmv_direct_halo, the halo fused into the direct kernel)
  const bool small = 12 * nnz + 20 * m < kSmallBytes;
  if (small) A->kernel_id = KERNEL_DIRECT;
  const char *env = getenv("SPMAT_SPMV_KERNEL");
  if (env && !strcmp(env, "tma")) A->kernel_id = KERNEL_TMA;
  if (env && !strcmp(env, "direct")) A->kernel_id = KERNEL_DIRECT;
  if (env && !strcmp(env, "vector")) A->kernel_id = KERNEL_VECTOR;
  if (env && !strcmp(env, "stream")) A->kernel_id = KERNEL_STREAM;
  A->kernel_id_csr = A->kernel_id;
  A->max_row_nnz = 0;
  A->n_rowblocks = 0;
  A->lanes = lanes_for(m ? (double)nnz / (double)m : 0.0);
  // off-diagonal rows: the largest power of two w <= 32 with >= 2 entries per lane on average
  // (stencil slabs: 1 entry per row -> w = 1, the plain row sum).  The SpMV-add is latency-
  // bound (a dependent ghost read per entry), so short lane loops matter more than lanes.
  A->ro_w = 1;
  if (A->n_ro > 0)
    while (A->ro_w < 32 && 4 * A->ro_w * A->n_ro <= A->nnz_o) A->ro_w *= 2;
  if (const char *w = getenv("SPMAT_RO_W")) {
    const int v = atoi(w);
    if (v >= 1 && v <= 32 && (v & (v - 1)) == 0) A->ro_w = v;
  }
  if (m == 0) return SPMAT_OK;
  DevBuf<char> tmp;
  DevBuf<uint32_t> flag;
  DevBuf<int32_t> longrows, maxlen;
  SP_TRY(flag.alloc(m));
  SP_TRY(longrows.alloc(m));
  SP_TRY(maxlen.alloc(2));
  SP_CUDA(cudaMemsetAsync(maxlen.get(), 0, 8, st));
  k_long_rows<<<nblk(m), 256, 0, st>>>(A->rowptr_d.get(), m, flag.get(), maxlen.get());
  SP_LAUNCH();
  CUB_CALL(tmp, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes,
                                           thrust::counting_iterator<int32_t>(0), flag.get(),
                                           longrows.get(), maxlen.get() + 1, (int)m, st));
  int32_t h[2];
  SP_CUDA(cudaMemcpyAsync(h, maxlen.get(), 8, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  A->max_row_nnz = h[0];
  const int64_t nlong = h[1];
  // Row-block budget.  The consumers cover a block's rows with W lanes per row (the largest
  // power of two with rows * W <= 256); with more than 256 / W rows, or more than 8 entries per
  // lane, a block costs them two rounds of dependent x gathers.  When kBudget gives two rounds
  // and a budget sized for ONE (256 / W' rows, W' the smallest power of two with <= 8 entries
  // per lane, 2 % slack for shorter boundary rows) keeps >= 85 % of kBudget, use it: C3 (27-point,
  // 70 rows at W = 2 -> ~63 at W = 4): 0.2225 -> 0.2068 ms.  Smaller blocks cost more than the
  // second round saves (Bump 45-point at 1442: 0.2486 -> 0.2744 ms; Q2 with the slack: +2 %), so
  // C4, Q2 and Bump keep kBudget.  SPMAT_RB_BUDGET overrides (0: kBudget).
  A->rb_budget = kBudget;
  if (m > 0) {
    const double L = (double)nnz / (double)m;
    const double rows = std::floor(kBudget / (L + kAlpha));  // rows of a typical block
    int w0 = 1;
    while (w0 < 32 && rows * 2 * w0 <= kThreads) w0 *= 2;
    const bool two_rounds = rows > kThreads / w0 || L > 8.0 * w0;
    int w1 = 1;
    while (w1 < 32 && L > 8.0 * w1) w1 *= 2;
    const double b1 = 0.98 * (kThreads / w1) * (L + kAlpha);
    if (two_rounds && b1 >= 0.85 * kBudget && b1 < kBudget) A->rb_budget = (int)b1;
  }
  if (const char *e = getenv("SPMAT_RB_BUDGET")) {
    const int b = atoi(e);
    A->rb_budget = b <= 0 ? kBudget : std::max(64, std::min(kBudget, b));
  }
  const int64_t total_cost = nnz + kAlpha * m;
  const int64_t n_cost = (total_cost + A->rb_budget - 1) / A->rb_budget;  // t = 0 .. n_cost-1, plus m
  const int64_t ncand = n_cost + 1 + 2 * nlong;
  DevBuf<int32_t> cand, sorted, uniq;
  DevBuf<int> dn;
  SP_TRY(cand.alloc(ncand));
  SP_TRY(sorted.alloc(ncand));
  SP_TRY(uniq.alloc(ncand));
  SP_TRY(dn.alloc(1));
  k_rb_candidates<<<nblk(n_cost), 256, 0, st>>>(A->rowptr_d.get(), m, n_cost, cand.get(), A->rb_budget);
  SP_LAUNCH();
  if (nlong > 0) {
    k_long_bounds<<<nblk(nlong), 256, 0, st>>>(longrows.get(), nlong, cand.get() + n_cost + 1);
    SP_LAUNCH();
  }
  CUB_CALL(tmp, cub::DeviceRadixSort::SortKeys(d_temp_storage, temp_storage_bytes, cand.get(),
                                               sorted.get(), (int)ncand, 0, 32, st));
  CUB_CALL(tmp, cub::DeviceSelect::Unique(d_temp_storage, temp_storage_bytes, sorted.get(),
                                          uniq.get(), dn.get(), (int)ncand, st));
  int nu = 0;
  SP_CUDA(cudaMemcpyAsync(&nu, dn.get(), 4, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  // uniq = 0 = r_0 < r_1 < ... < r_last = m
  A->n_rowblocks = nu - 1;
  SP_TRY(A->rbp.alloc(nu));
  k_rb_pairs<<<nblk(nu), 256, 0, st>>>(uniq.get(), A->rowptr_d.get(), nu, A->rbp.get());
  SP_LAUNCH();
  A->n_long = nlong;
  SP_TRY(A->longrows.alloc(nlong));
  if (nlong)
    SP_CUDA(cudaMemcpyAsync(A->longrows.get(), longrows.get(), (size_t)nlong * 4, cudaMemcpyDeviceToDevice, st));
  SP_TRY(A->sched.alloc(2));
  SP_CUDA(cudaMemsetAsync(A->sched.get(), 0, 8, st));
  SP_TRY(A->tail_ctr.alloc(5));
  SP_CUDA(cudaMemsetAsync(A->tail_ctr.get(), 0, 20, st));

  A->n_bblocks = 0;
  A->tail_split = false;
  if (A->n_ro > 0) {  // claim order for the fused off-diagonal tail: boundary blocks first
    const int64_t nbk = A->n_rowblocks;
    DevBuf<uint32_t> f1, f0;
    DevBuf<int> dn2;
    SP_TRY(f1.alloc(nbk));
    SP_TRY(f0.alloc(nbk));
    SP_TRY(dn2.alloc(2));
    SP_TRY(A->block_order.alloc(nbk));
    k_boundary_blocks<<<nblk(nbk), 256, 0, st>>>(A->rbp.get(), nbk, A->rows_o.get(), A->n_ro, f1.get(), f0.get());
    SP_LAUNCH();
    CUB_CALL(tmp, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes,
                                             thrust::counting_iterator<int32_t>(0), f1.get(),
                                             A->block_order.get(), dn2.get(), (int)nbk, st));
    int nbb = 0;
    SP_CUDA(cudaMemcpyAsync(&nbb, dn2.get(), 4, cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    CUB_CALL(tmp, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes,
                                             thrust::counting_iterator<int32_t>(0), f0.get(),
                                             A->block_order.get() + nbb, dn2.get() + 1, (int)nbk, st));
    A->n_bblocks = nbb;
    // Boundary rows in most row blocks (box partitions): boundary-first would sweep the matrix
    // twice (the diagonal SpMV alone loses ~6 %), and in natural order the latency-bound tail
    // waits for the whole sweep; instead natural order with the split tail -- sums during the
    // sweep, one short add pass after it (halo_dev.cuh split_tail)
    const char *pe = getenv("SPMAT_SPLIT_TAIL");
    A->tail_split = pe ? atoi(pe) != 0 : 2 * nbb > nbk;
    if (A->tail_split) {
      A->block_order.release();
      A->n_bblocks = nbk;  // every block counts: the add pass waits for the whole sweep
      SP_TRY(A->tail_obuf.alloc(A->n_ro));
    }
  }
  SP_TRY(A->blocks4.alloc(A->n_rowblocks));
  k_blocks4<<<nblk(A->n_rowblocks), 256, 0, st>>>(A->rbp.get(), A->block_order.get(),
                                                  A->n_rowblocks, A->blocks4.get());
  SP_LAUNCH();
  SP_TRY(tma_setup(A));
  if (const char *tr = getenv("SPMAT_TRACE")) {  // device trace of the fused MatMult kernel
    if (atoi(tr)) {
      SP_TRY(A->trace.alloc(kTraceCta * (size_t)A->tma_grid_tail + 16));
      SP_CUDA(cudaMemsetAsync(A->trace.get(), 0, A->trace.n * 8, st));
      const unsigned long long hdr[2] = {(unsigned long long)A->tma_grid_tail, (unsigned long long)kTraceCta};
      SP_CUDA(cudaMemcpyAsync(A->trace.get() + A->trace.n - 2, hdr, sizeof hdr, cudaMemcpyHostToDevice, st));
    }
  }
  SP_CUDA(cudaStreamSynchronize(st));
  return SPMAT_OK;
}

static cudaError_t launch_tma(spmat_s *A, const double *x, double *y, cudaStream_t s, bool fuse_put,
                              bool fuse_tail) {
  // the kernel ends the MatMult (bumps the device epoch) when it also runs the off-diagonal
  // add; otherwise k_spmv_offdiag_peer does
  SpmvHalo h{A->halo_puts.get(), A->n_puts, fuse_put ? A->put_chunks_total : 0,
             A->peer ? A->d_epoch.get() : nullptr, (fuse_put && fuse_tail) ? 1 : 0, A->halo_err.get()};
  SpmvTail t{};
  t.trace = A->trace.get();
  if (fuse_tail) {  // the comm warps add A_o lvec once the boundary blocks (claimed first) are written
    t.n_bblocks = (int)A->n_bblocks;
    t.enabled = 1;
    t.w = A->ro_w;
    t.rows = A->rows_o.get();
    t.rowptr = A->rowptr_o.get();
    t.col = A->col_o.get();
    t.val = A->val_o.get();
    t.ghost = A->ghost.get();
    t.ghost_stride = A->ghost_stride;
    t.n_ro = A->n_ro;
    t.waits = A->halo_waits.get();
    t.nwaits = A->n_waits;
    t.ctr = A->tail_ctr.get();
    if (A->tail_split) t.obuf = A->tail_obuf.get();
  }
  const unsigned grid = (unsigned)(fuse_tail ? A->tma_grid_tail : A->tma_grid);
  if (fuse_tail)  // comm warps spin on lines written by the peers' CTAs: all CTAs co-resident
    return launch_coop(k_spmv_tma, grid, kCtaThreads, kTmaSmem, s, (const int4 *)A->blocks4.get(),
                       (int)A->n_rowblocks, (const int32_t *)A->rowptr_d.get(), (const int32_t *)A->col_d.get(),
                       (const double *)A->val_d.get(), x, y, A->sched.get(), h, t);
  return launch_pdl(k_spmv_tma, grid, kCtaThreads, kTmaSmem, s, (const int4 *)A->blocks4.get(),
                    (int)A->n_rowblocks, (const int32_t *)A->rowptr_d.get(), (const int32_t *)A->col_d.get(),
                    (const double *)A->val_d.get(), x, y, A->sched.get(), h, t);
}

template <int W>
static cudaError_t launch_direct(spmat_s *A, const double *x, double *y, cudaStream_t s) {
  const int64_t threads = A->m * W;
  const unsigned grid = (unsigned)std::max<int64_t>(1, (threads + 127) / 128);
  return launch_pdl(k_spmv_direct<W>, grid, 128, 0, s, (const int32_t *)A->rowptr_d.get(),
                    (const int32_t *)A->col_d.get(), (const double *)A->val_d.get(), x, y, A->m);
}

template <int W>
static int64_t direct_halo_grid(spmat_s *A) {
  const int64_t threads = std::max<int64_t>(A->m * W, 32LL * A->put_chunks_total);
  return std::max<int64_t>(1, (threads + 127) / 128);
}

// 1 if the one-launch small MatMult fits a cooperative launch (every CTA resident)
template <int W>
static int direct_halo_fits(spmat_s *A) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_direct_halo<W>, 128, 0) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return direct_halo_grid<W>(A) <= (int64_t)per_sm * A->comm->num_sms ? 1 : 0;
}

int direct_halo_ok(spmat_s *A) {
  if (A->direct_halo_ok < 0) {
    switch (A->lanes) {
      case 1: A->direct_halo_ok = direct_halo_fits<1>(A); break;
      case 2: A->direct_halo_ok = direct_halo_fits<2>(A); break;
      case 4: A->direct_halo_ok = direct_halo_fits<4>(A); break;
      case 8: A->direct_halo_ok = direct_halo_fits<8>(A); break;
      case 16: A->direct_halo_ok = direct_halo_fits<16>(A); break;
      default: A->direct_halo_ok = direct_halo_fits<32>(A); break;
    }
  }
  return A->direct_halo_ok;
}

template <int W>
static cudaError_t launch_direct_halo(spmat_s *A, const double *x, double *y, cudaStream_t s) {
  const unsigned grid = (unsigned)direct_halo_grid<W>(A);
  SpmvHalo h{A->halo_puts.get(), A->n_puts, A->put_chunks_total, A->d_epoch.get(), 1, A->halo_err.get()};
  return launch_coop(k_spmv_direct_halo<W>, grid, 128, 0, s, (const int32_t *)A->rowptr_d.get(),
                     (const int32_t *)A->col_d.get(), (const double *)A->val_d.get(), x, y, A->m,
                     (const int32_t *)A->ro_of_row.get(), (const int32_t *)A->rowptr_o.get(),
                     (const int32_t *)A->col_o.get(), (const double *)A->val_o.get(), h,
                     (const uint4 *)A->ghost.get(), A->ghost_stride, (const HaloWait *)A->halo_waits.get(),
                     A->n_waits, A->halo_counter.get());
}

// the whole MatMult of a small matrix with the NVLink halo in one launch (k_spmv_direct_halo)
int spmv_direct_halo(spmat_s *A, const double *x, double *y, cudaStream_t s) {
  if (!A->ro_of_row.get()) {  // row -> compressed off-diagonal row (or -1), built on first use
    SP_TRY(A->ro_of_row.alloc(std::max<int64_t>(A->m, 1)));
    SP_CUDA(cudaMemsetAsync(A->ro_of_row.get(), 0xff, std::max<int64_t>(A->m, 1) * 4, s));
    if (A->n_ro > 0) {
      k_scatter_ro<<<nblk(A->n_ro), 256, 0, s>>>(A->rows_o.get(), A->n_ro, A->ro_of_row.get());
      SP_LAUNCH();
    }
  }
  cudaError_t e;
  switch (A->lanes) {
    case 1: e = launch_direct_halo<1>(A, x, y, s); break;
    case 2: e = launch_direct_halo<2>(A, x, y, s); break;
    case 4: e = launch_direct_halo<4>(A, x, y, s); break;
    case 8: e = launch_direct_halo<8>(A, x, y, s); break;
    case 16: e = launch_direct_halo<16>(A, x, y, s); break;
    default: e = launch_direct_halo<32>(A, x, y, s); break;
  }
  SP_CUDA(e);
  return SPMAT_OK;
}

template <int W>
static void launch_vector(spmat_s *A, const double *x, double *y, cudaStream_t s) {
  k_spmv_vector<W><<<nblk(A->m * W), 256, 0, s>>>(A->rowptr_d.get(), A->col_d.get(), A->val_d.get(),
                                                  x, y, A->m);
}

int spmv_diag(spmat_s *A, const double *x, double *y, cudaStream_t s, bool fuse_put, bool fuse_tail) {
  if (A->m == 0) return SPMAT_OK;
  if (A->bs == 3) return bsr_spmv(A, x, y, s);
  if (A->kernel_id == KERNEL_DIRECT) {
    cudaError_t e;
    switch (A->lanes) {
      case 1: e = launch_direct<1>(A, x, y, s); break;
      case 2: e = launch_direct<2>(A, x, y, s); break;
      case 4: e = launch_direct<4>(A, x, y, s); break;
      case 8: e = launch_direct<8>(A, x, y, s); break;
      case 16: e = launch_direct<16>(A, x, y, s); break;
      default: e = launch_direct<32>(A, x, y, s); break;
    }
    SP_CUDA(e);
    return SPMAT_OK;
  }
  if (A->kernel_id == KERNEL_VECTOR) {
    switch (std::max(A->lanes, 4)) {
      case 4: launch_vector<4>(A, x, y, s); break;
      case 8: launch_vector<8>(A, x, y, s); break;
      case 16: launch_vector<16>(A, x, y, s); break;
      default: launch_vector<32>(A, x, y, s); break;
    }
    SP_LAUNCH();
    return SPMAT_OK;
  }
  if (A->kernel_id == KERNEL_TMA) {
    SP_CUDA(launch_tma(A, x, y, s, fuse_put, fuse_tail));
  } else {
    k_spmv_stream<<<(unsigned)A->n_rowblocks, kThreads, 0, s>>>(A->rbp.get(), A->rowptr_d.get(),
                                                               A->col_d.get(), A->val_d.get(), x, y);
  }
  SP_LAUNCH();
  if (A->n_long > 0) {
    k_spmv_long<<<(unsigned)A->n_long, kThreads, 0, s>>>(A->longrows.get(), A->rowptr_d.get(),
                                                         A->col_d.get(), A->val_d.get(), x, y);
    SP_LAUNCH();
  }
  return SPMAT_OK;
}

int spmv_offdiag(spmat_s *A, double *y, cudaStream_t s) {
  if (A->n_ro == 0) return SPMAT_OK;
  if (A->bs == 3 && A->ob_ok)  // NCCL ghost vector, or (isolated part) the landed lines
    return A->peer ? bsr_offdiag(A, y, nullptr, s, false) : bsr_offdiag(A, y, A->lvec.get(), s);
  k_spmv_offdiag<<<nblk(A->ro_w == 1 ? (A->n_ro + kRowsU - 1) / kRowsU : A->n_ro * A->ro_w), 256, 0, s>>>(
      A->rows_o.get(), A->rowptr_o.get(), A->col_o.get(), A->val_o.get(), A->lvec.get(),
      A->peer ? A->ghost.get() : nullptr, A->ghost_stride, A->peer ? A->d_epoch.get() : nullptr, y,
      A->n_ro, A->ro_w, A->peer ? A->halo_err.get() : nullptr);
  SP_LAUNCH();
  return SPMAT_OK;
}

}  // namespace spmat

namespace spmat {

// ------------------------------------------------------------------ host-buffer pipeline
// first and last column read by each chunk of rows (columns ascend within a row)
__global__ void k_chunk_cols(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                             int64_t r0, int64_t r1, int *__restrict__ lo, int *__restrict__ hi) {
  int a_min = INT_MAX, b_max = -1;
  for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int a = rowptr[r], z = rowptr[r + 1];
    if (z > a) {
      a_min = min(a_min, col[a]);
      b_max = max(b_max, col[z - 1]);
    }
  }
  atomicMin(lo, a_min);
  atomicMax(hi, b_max);
}

// Row chunks of the host-buffer pipeline (mult.cu): `chunks` ranges of whole row blocks in row
// order, the x rows each reads, its compressed off-diagonal rows, and the chunks the NVLink
// halo puts read (uploaded first).
int spmv_pipe_prepare(spmat_s *A, int chunks) {
  if (A->pipe_chunks == chunks) return SPMAT_OK;
  const int64_t nb = A->n_rowblocks;
  if (nb < chunks) chunks = (int)std::max<int64_t>(1, nb);
  // row-ordered block table (the claim order puts boundary blocks first when multi-rank)
  if (A->block_order.get()) {
    SP_TRY(A->pipe_blocks4.alloc(nb));
    k_blocks4<<<nblk(nb), 256>>>(A->rbp.get(), nullptr, nb, A->pipe_blocks4.get());
    SP_LAUNCH();
  }
  const int4 *rb4 = A->block_order.get() ? A->pipe_blocks4.get() : A->blocks4.get();
  A->pipe_block.assign(chunks + 1, 0);
  A->pipe_row.assign(chunks + 1, 0);
  A->pipe_xmin.assign(chunks, 0);
  A->pipe_xneed.assign(chunks, 0);
  A->pipe_q.assign(chunks + 1, 0);
  std::vector<int4> edge(chunks + 1);
  for (int k = 0; k <= chunks; ++k) A->pipe_block[k] = nb * k / chunks;
  for (int k = 0; k < chunks; ++k)
    SP_CUDA(cudaMemcpy(&edge[k], rb4 + A->pipe_block[k], sizeof(int4), cudaMemcpyDeviceToHost));
  for (int k = 0; k < chunks; ++k) A->pipe_row[k] = edge[k].x;
  A->pipe_row[chunks] = A->m;
  DevBuf<int> mn, mx;
  SP_TRY(mn.alloc(chunks));
  SP_TRY(mx.alloc(chunks));
  SP_CUDA(cudaMemset(mn.get(), 0x7f, chunks * sizeof(int)));
  SP_CUDA(cudaMemset(mx.get(), 0xff, chunks * sizeof(int)));
  for (int k = 0; k < chunks; ++k) {
    k_chunk_cols<<<nblk(A->pipe_row[k + 1] - A->pipe_row[k]), 256>>>(
        A->rowptr_d.get(), A->col_d.get(), A->pipe_row[k], A->pipe_row[k + 1], mn.get() + k, mx.get() + k);
    SP_LAUNCH();
  }
  std::vector<int> h0(chunks), h1(chunks);
  SP_CUDA(cudaMemcpy(h0.data(), mn.get(), chunks * sizeof(int), cudaMemcpyDeviceToHost));
  SP_CUDA(cudaMemcpy(h1.data(), mx.get(), chunks * sizeof(int), cudaMemcpyDeviceToHost));
  for (int k = 0; k < chunks; ++k) {
    A->pipe_xmin[k] = h1[k] < 0 ? A->pipe_row[k] : h0[k];  // empty chunk: nothing to wait for
    A->pipe_xneed[k] = h1[k] < 0 ? A->pipe_row[k] : h1[k];
  }
  // compressed off-diagonal rows of each chunk (rows_o ascending)
  if (A->n_ro > 0) {
    std::vector<int32_t> ro(A->n_ro);
    SP_CUDA(cudaMemcpy(ro.data(), A->rows_o.get(), A->n_ro * 4, cudaMemcpyDeviceToHost));
    for (int k = 0; k <= chunks; ++k)
      A->pipe_q[k] = std::lower_bound(ro.begin(), ro.end(), (int32_t)A->pipe_row[k]) - ro.begin();
  }
  // x rows the NVLink puts read: contiguous root ranges, or everything when a put gathers
  A->pipe_put_chunk.assign(chunks, 0);
  if (A->peer && A->halo) {
    const sf_s *sf = A->halo;
    for (size_t a = 0; a < sf->snbr.size(); ++a) {
      int64_t r0 = 0, r1 = A->n;
      if (sf->root_start[a] >= 0) {
        r0 = sf->root_start[a];
        r1 = r0 + sf->scount[a];
      }
      for (int k = 0; k < chunks; ++k)
        if (A->pipe_row[k] < r1 && A->pipe_row[k + 1] > r0) A->pipe_put_chunk[k] = 1;
    }
  }
  A->pipe_chunks = chunks;
  return SPMAT_OK;
}

// the bulk-copy SpMV over the row blocks [pipe_block[k], pipe_block[k+1]) of row order
int spmv_diag_chunk(spmat_s *A, const double *x, double *y, int k, cudaStream_t s) {
  const int64_t c0 = A->pipe_block[k], c1 = A->pipe_block[k + 1];
  if (c1 <= c0) return SPMAT_OK;
  SpmvHalo h{A->halo_puts.get(), 0, 0, nullptr, 0, A->halo_err.get()};
  SpmvTail t{};
  const int4 *rb4 = A->block_order.get() ? A->pipe_blocks4.get() : A->blocks4.get();
  const unsigned grid = (unsigned)std::min<int64_t>(A->tma_grid, c1 - c0);
  k_spmv_tma<<<grid, kCtaThreads, kTmaSmem, s>>>(rb4 + c0, (int)(c1 - c0), A->rowptr_d.get(),
                                                A->col_d.get(), A->val_d.get(), x, y, A->sched.get(), h, t);
  SP_LAUNCH();
  return SPMAT_OK;
}

}  // namespace spmat
