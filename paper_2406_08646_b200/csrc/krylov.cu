// krylov.cu -- host-synchronisation-free CG on top of MatMult (the paper's CGAsync).
//
// CG "does all its computation and communication on device, and does not need any
// synchronization on host": dot products land in DEVICE scalars (VecDotAsync,
// P:715-724), AXPYs read their coefficient from device memory (VecAXPYAsync),
// scalar arithmetic runs in tiny device kernels, and the loop runs a user-given
// number of iterations without a host-side convergence test.  The paper reduced
// the partial dots with NVSHMEM; here the cross-rank reduction goes through a "scalar board":
// each rank's small device array is IPC-mapped into every other rank (NVLink), a rank stores
// its partial into every board as a line flagged with the reduction's epoch (halo_dev.cuh),
// then sums the P partials of its own board in rank order once they carry the epoch -- the
// same bit-identical value on every rank, no NCCL kernel, no host, no fence.
//
// Local dot products use a fixed decomposition (a function of m only: CTAs x 256 threads, fixed strides,
// fixed reduction trees), so results are deterministic run to run.
//
// Every epoch (halo, board) and the residual-history index live in device memory, so one CG
// iteration is captured once as a CUDA graph and replayed maxit times (SPMAT_GRAPH=0 turns the
// graph off): the launch cost of the iteration's kernels becomes one graph launch.  Each dot is
// one kernel: the last CTA to finish sums the partials and does the cross-rank step.
#include <algorithm>
#include <cstring>

#include <cooperative_groups.h>

#include "halo_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace spmat {

constexpr int kDotThreads = 256;

// ------------------------------------------------------------------ scalar board
int board_setup(Comm *c) {
  const int P = c->nranks, me = c->rank;
  c->board_ok = false;
  if (P == 1) return SPMAT_OK;
  SP_TRY(c->board_line.alloc(2 * (size_t)P));
  SP_TRY(c->board_err.alloc(1));
  SP_TRY(c->d_board_epoch.alloc(1));
  SP_CUDA(cudaMemset(c->board_line.get(), 0, 2 * P * sizeof(uint4)));  // flag 0: no epoch
  SP_CUDA(cudaMemset(c->board_err.get(), 0, sizeof(int)));
  SP_CUDA(cudaMemset(c->d_board_epoch.get(), 0, sizeof(unsigned long long)));
  cudaIpcMemHandle_t hv;
  memset(&hv, 0, sizeof hv);
  int64_t fail = 0;
  if (getenv("SPMAT_BOARD") && !strcmp(getenv("SPMAT_BOARD"), "nccl")) fail = 1;
  if (!fail && cudaIpcGetMemHandle(&hv, c->board_line.get()) != cudaSuccess) {
    cudaGetLastError();
    fail = 1;
  }
  std::vector<int64_t> mine(8), all(8 * (size_t)P);
  memcpy(mine.data(), &hv, 64);
  SP_TRY(c->allgather_i64(mine.data(), 8, all.data()));
  std::vector<uint4 *> pl(P, nullptr);
  pl[me] = c->board_line.get();
  for (int q = 0; q < P && !fail; ++q) {
    if (q == me) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, all.data() + 8 * (size_t)q, 64);
    void *a = nullptr;
    if (cudaIpcOpenMemHandle(&a, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      fail = 1;
      break;
    }
    c->board_peer_mem.push_back(a);
    pl[q] = (uint4 *)a;
  }
  int64_t vote[1] = {fail};
  SP_TRY(c->allreduce_max_i64(vote, 1));
  if (vote[0]) {
    if (!(getenv("SPMAT_BOARD") && !strcmp(getenv("SPMAT_BOARD"), "nccl")))
      note_fallback(c, "the cross-rank dot sums", "CUDA IPC of the scalar board failed on some rank");
    board_release(c);
    return SPMAT_OK;  // reductions fall back to ncclAllReduce
  }
  SP_TRY(c->d_peer_line.alloc(P));
  SP_CUDA(cudaMemcpy(c->d_peer_line.get(), pl.data(), P * sizeof(uint4 *), cudaMemcpyHostToDevice));
  c->board_ok = true;
  return SPMAT_OK;
}

void board_release(Comm *c) {
  for (void *p : c->board_peer_mem) cudaIpcCloseMemHandle(p);
  c->board_peer_mem.clear();
  c->board_ok = false;
}

// ------------------------------------------------------------------ kernels
// fixed-shape CTA reduction: warp shuffle tree, then warp 0 over the 8 warp sums
__device__ __forceinline__ double block_sum(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < kDotThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  }
  __syncthreads();  // red may be reused
  return s;  // valid in thread 0
}

struct CgScalars {
  double rr, pq, alpha, beta;
  int stopped, iter;  // iter: index of the last residual-history entry written
};

enum { OP_DOT = 0, OP_CG_INIT = 1, OP_CG_ALPHA = 2, OP_CG_BETA = 3 };

// What the CTA that finishes a dot does with the partial sums.
struct FinArgs {
  double *partial;  // one partial per CTA of the dot kernel
  int op;
  CgScalars *sc;
  double *result, *hist;
  uint4 *const *peer_line;  // scalar board (nullptr: single rank, or NCCL path)
  int P, me;
  unsigned long long *board_epoch;
  int *err;
  const double *preduced;  // NCCL path: the value already all-reduced over ranks
  unsigned *count;         // non-null: the last CTA of the dot kernel finalizes in place
};

// One CTA: local sum of the np partials (fixed order), the cross-rank sum through the scalar
// board (or the NCCL-reduced value), then the scalar step of CG.  The board epoch is read from
// and written back to device memory.
// the fixed-order local sum of np partials (valid in thread 0)
__device__ __forceinline__ double fold_partials(const double *partial, int np, double *red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += kDotThreads) s = __dadd_rn(s, __ldcg(partial + i));
  return block_sum(s, red);
}

__device__ void finalize_cta(const FinArgs &f, int np) {
  __shared__ double red[kDotThreads / 32];
  __shared__ double total;
  double s = fold_partials(f.partial, np, red);
  if (threadIdx.x == 0) total = s;
  __syncthreads();
  if (f.preduced) {  // NCCL already summed the local values over ranks
    if (threadIdx.x == 0) total = *f.preduced;
  } else if (f.peer_line) {
    // my partial, flagged with this reduction's epoch, into every rank's board (one 16-byte
    // store each, no fence); then the P lines of my board, summed in rank order once each
    // carries the epoch -- the same value on every rank
    const unsigned long long epoch = *f.board_epoch + 1ull;
    const int par = (int)(epoch & 1);
    const int P = f.P;
    const uint32_t flag = ll_flag(epoch);
    if (threadIdx.x < P) ll_store(f.peer_line[threadIdx.x] + (size_t)par * P + f.me, total, flag);
    if (threadIdx.x == 0) {
      const uint4 *mine = f.peer_line[f.me] + (size_t)par * P;
      double t = 0.0;
      for (int q = 0; q < P; ++q) t = __dadd_rn(t, ll_load(mine + q, flag, f.err));  // rank order
      total = t;
      *f.board_epoch = epoch;
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const double g = total;
  CgScalars *sc = f.sc;
  if (f.op == OP_DOT) {
    *f.result = g;
  } else if (f.op == OP_CG_INIT) {
    sc->rr = g;
    sc->beta = 0.0;  // the small-matrix path forms p_0 = r_0 + 0 * p (p = r after init)
    sc->stopped = g == 0.0 ? 1 : 0;
    sc->iter = 0;
    if (f.hist) f.hist[0] = g;
  } else if (f.op == OP_CG_ALPHA) {
    sc->pq = g;
    if (g == 0.0 || sc->rr == 0.0) sc->stopped = 1;
    sc->alpha = sc->stopped ? 0.0 : sc->rr / g;
  } else {  // OP_CG_BETA
    if (!sc->stopped) {
      sc->beta = g / sc->rr;
      sc->rr = g;
    }
    sc->iter += 1;
    if (f.hist) f.hist[sc->iter] = sc->rr;
  }
}

// Each CTA stores its partial; with f.count the last CTA to arrive finalizes (one kernel per
// dot instead of two).  Called by every thread of the CTA.
__device__ __forceinline__ void partial_done(double s, const FinArgs &f) {
  __shared__ int last;
  if (f.count && gridDim.x == 1) {  // one CTA: no cross-CTA handshake
    if (threadIdx.x == 0) f.partial[0] = s;
    __syncthreads();
    finalize_cta(f, 1);
    return;
  }
  if (threadIdx.x == 0) {
    f.partial[blockIdx.x] = s;
    if (f.count) {
      __threadfence();
      last = atomicAdd(f.count, 1u) == gridDim.x - 1 ? 1 : 0;
    }
  }
  if (!f.count) return;
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) *f.count = 0u;  // ready for the next dot
  __threadfence();
  finalize_cta(f, gridDim.x);
}

__global__ void __launch_bounds__(kDotThreads) k_finalize(FinArgs f, int np) {
  pdl_wait();
  finalize_cta(f, np);
}

constexpr int kU = 4;  // elements per thread in flight in the streaming vector kernels

__device__ __forceinline__ double combine(const double (&acc)[kU]) {
  return __dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3]));
}

// CTA c owns [c*chunk, (c+1)*chunk); partial[c] = sum of a*b there.  VEC (both vectors
// 16-byte aligned): even chunks read as double2, kU pairs of each vector in flight per thread
// (16 B per load, twice the bytes in flight of the scalar loop); the order of the sums is a
// fixed function of n, the grid and VEC.
template <bool VEC>
__global__ void __launch_bounds__(kDotThreads) k_dot_partial(const double *__restrict__ a,
                                                             const double *__restrict__ b, int64_t n,
                                                             FinArgs f) {
  __shared__ double red[kDotThreads / 32];
  pdl_wait();
  double acc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) acc[u] = 0.0;
  if (VEC) {
    const int64_t chunk = ((n + gridDim.x - 1) / gridDim.x + 1) & ~(int64_t)1;
    const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    const int64_t n2 = hi > lo ? (hi - lo) / 2 : 0;
    const double2 *a2 = reinterpret_cast<const double2 *>(a + lo);
    const double2 *b2 = reinterpret_cast<const double2 *>(b + lo);
    int64_t i = threadIdx.x;
    for (; i + (kU - 1) * kDotThreads < n2; i += kU * kDotThreads) {
      double2 av[kU], bv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        av[u] = a2[i + u * kDotThreads];
        bv[u] = b2[i + u * kDotThreads];
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        acc[u] = __dadd_rn(acc[u], __dmul_rn(av[u].x, bv[u].x));
        acc[u] = __dadd_rn(acc[u], __dmul_rn(av[u].y, bv[u].y));
      }
    }
    for (; i < n2; i += kDotThreads) {
      const double2 av = a2[i], bv = b2[i];
      acc[0] = __dadd_rn(acc[0], __dmul_rn(av.x, bv.x));
      acc[0] = __dadd_rn(acc[0], __dmul_rn(av.y, bv.y));
    }
    if (threadIdx.x == 0 && hi > lo && ((hi - lo) & 1)) acc[1] = __dadd_rn(acc[1], __dmul_rn(a[hi - 1], b[hi - 1]));
  } else {
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    // kU independent accumulators (kU loads of each vector in flight per thread)
    int64_t i = lo + threadIdx.x;
    for (; i + (kU - 1) * kDotThreads < hi; i += kU * kDotThreads) {
      double av[kU], bv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        av[u] = a[i + u * kDotThreads];
        bv[u] = b[i + u * kDotThreads];
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(av[u], bv[u]));
    }
    for (; i < hi; i += kDotThreads) acc[0] = __dadd_rn(acc[0], __dmul_rn(a[i], b[i]));
  }
  partial_done(block_sum(combine(acc), red), f);
}

// Small matrices on one rank (the direct SpMV kernel's regime, e.g. Kuu-sized): q = A p and
// the p.q partial in ONE kernel -- W lanes per row as in k_spmv_direct (8 (col, val) loads,
// then 8 x gathers per lane in flight), q[r] stored, q[r]*p[r] summed per CTA by the fixed
// tree, the last CTA finalizes alpha.  One launch and one pass over p and q fewer per iteration.
// With the p update folded in (the small path's 2-kernel iteration): p holds p_{i-1}, and every
// use forms p_i = r + beta p_{i-1} on the fly (the same rounded operations as k_cg_pupdate, so
// the same bits); k_cg_update_p then stores p_i.
template <int W>
__global__ void __launch_bounds__(kDotThreads) k_cg_spmv_dot(const int32_t *__restrict__ rowptr,
                                                             const int32_t *__restrict__ col,
                                                             const double *__restrict__ val,
                                                             const double *__restrict__ p, double *__restrict__ q,
                                                             int64_t m, FinArgs f, const double *__restrict__ r) {
  __shared__ double red[kDotThreads / 32];
  pdl_wait();
  const double beta = f.sc->beta;  // read before this kernel's last CTA rewrites the scalars
  auto pv = [&](int64_t c) { return r ? __dadd_rn(r[c], __dmul_rn(beta, p[c])) : p[c]; };
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
    for (int u = 0; u < U; ++u) xv[u] = pv(c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * W < z) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
  }
#pragma unroll
  for (int o = W >> 1; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o, W));
  double pq = 0.0;
  if (valid && lane == 0) {
    q[row] = s;
    pq = __dmul_rn(pv(row), s);
  }
  partial_done(block_sum(pq, red), f);
}

static inline bool aligned16(const void *p, const void *q) {
  return (((uintptr_t)p | (uintptr_t)q) & 15) == 0;
}

// r = b - q; p = r; partial of r.r
__global__ void __launch_bounds__(kDotThreads) k_cg_init(const double *__restrict__ b,
                                                         const double *__restrict__ q, double *__restrict__ r,
                                                         double *__restrict__ p, int64_t n, FinArgs f) {
  __shared__ double red[kDotThreads / 32];
  pdl_wait();
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kDotThreads) {
    const double ri = __dsub_rn(b[i], q[i]);
    r[i] = ri;
    p[i] = ri;
    s = __dadd_rn(s, __dmul_rn(ri, ri));
  }
  partial_done(block_sum(s, red), f);
}

// x = x + alpha p; r = r - alpha q; partial of r.r (products rounded separately, no FMA)
__global__ void __launch_bounds__(kDotThreads) k_cg_update(double *__restrict__ x, double *__restrict__ r,
                                                           const double *__restrict__ p,
                                                           const double *__restrict__ q, int64_t n,
                                                           FinArgs f) {
  __shared__ double red[kDotThreads / 32];
  pdl_wait();
  const double alpha = f.sc->alpha;
  const bool go = !f.sc->stopped;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double acc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) acc[u] = 0.0;
  int64_t i = lo + threadIdx.x;
  for (; i + (kU - 1) * kDotThreads < hi; i += kU * kDotThreads) {
    double rv[kU], xv[kU], pv[kU], qv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = i + u * kDotThreads;
      rv[u] = r[k];
      if (go) {
        xv[u] = x[k];
        pv[u] = p[k];
        qv[u] = q[k];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = i + u * kDotThreads;
      if (go) {
        x[k] = __dadd_rn(xv[u], __dmul_rn(alpha, pv[u]));
        rv[u] = __dsub_rn(rv[u], __dmul_rn(alpha, qv[u]));
        r[k] = rv[u];
      }
      acc[u] = __dadd_rn(acc[u], __dmul_rn(rv[u], rv[u]));
    }
  }
  for (; i < hi; i += kDotThreads) {
    double ri = r[i];
    if (go) {
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      ri = __dsub_rn(ri, __dmul_rn(alpha, q[i]));
      r[i] = ri;
    }
    acc[0] = __dadd_rn(acc[0], __dmul_rn(ri, ri));
  }
  // every CTA has read sc->alpha/stopped before the last one (which rewrites sc) gets here
  partial_done(block_sum(combine(acc), red), f);
}

// The small path's update of one chunk [lo, hi): p_i = r + beta p_{i-1} formed and stored
// (the p update folded in), x += alpha p_i, r -= alpha q; returns this thread's r.r partial.
// kU elements per thread in flight (kU accumulators, combined in a fixed tree), so a short
// chunk costs ~2 rounds of loads instead of one per element.  Shared by k_cg_update_p and
// k_cg_persist, so both give the same bits.
__device__ __forceinline__ double update_p_chunk(double *__restrict__ x, double *__restrict__ r,
                                                 double *__restrict__ p, const double *__restrict__ q,
                                                 int64_t lo, int64_t hi, double alpha, double beta, bool go) {
  double acc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) acc[u] = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kU * kDotThreads) {
    double rv[kU], pv[kU], xv[kU], qv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = i + u * kDotThreads;
      const bool in = k < hi;
      rv[u] = in ? r[k] : 0.0;
      if (go && in) {
        pv[u] = p[k];
        xv[u] = x[k];
        qv[u] = q[k];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = i + u * kDotThreads;
      if (k >= hi) continue;
      if (go) {
        const double pi = __dadd_rn(rv[u], __dmul_rn(beta, pv[u]));
        p[k] = pi;
        x[k] = __dadd_rn(xv[u], __dmul_rn(alpha, pi));
        rv[u] = __dsub_rn(rv[u], __dmul_rn(alpha, qv[u]));
        r[k] = rv[u];
      }
      acc[u] = __dadd_rn(acc[u], __dmul_rn(rv[u], rv[u]));
    }
  }
  return combine(acc);
}

// The small path's update kernel (one chunk per CTA)
__global__ void __launch_bounds__(kDotThreads) k_cg_update_p(double *__restrict__ x, double *__restrict__ r,
                                                             double *__restrict__ p, const double *__restrict__ q,
                                                             int64_t n, FinArgs f) {
  __shared__ double red[kDotThreads / 32];
  pdl_wait();
  const double alpha = f.sc->alpha, beta = f.sc->beta;
  const bool go = !f.sc->stopped;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  const double acc = update_p_chunk(x, r, p, q, lo, hi, alpha, beta, go);
  // every CTA has read sc->alpha/beta/stopped before the last one (which rewrites sc) gets here
  partial_done(block_sum(acc, red), f);
}

// p = r + beta p
__global__ void k_cg_pupdate(double *__restrict__ p, const double *__restrict__ r, int64_t n,
                             const CgScalars *__restrict__ sc) {
  pdl_wait();
  if (sc->stopped) return;
  const double beta = sc->beta;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + (kU - 1) * stride < n; i += kU * stride) {  // kU loads of each vector in flight
    double rv[kU], pv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      rv[u] = r[i + u * stride];
      pv[u] = p[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) p[i + u * stride] = __dadd_rn(rv[u], __dmul_rn(beta, pv[u]));
  }
  for (; i < n; i += stride) p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

// Small matrices on one rank: ALL maxit iterations in one cooperative launch.  Each iteration
// is the small path's two kernels (k_cg_spmv_dot's q = A p_i with p_i = r + beta p_{i-1} on the
// fly and its p.q partials over the same ga CTAs; k_cg_update_p's p/x/r update and r.r partials
// over the same nb chunks) separated by grid barriers, and instead of a last CTA finalizing each
// dot, EVERY CTA folds the partials itself (fold_partials: the same order, so the same alpha
// and beta in every CTA and the same bits as the two-kernel path); CTA 0 records the residual
// history and leaves the scalars in sc.  Two grid barriers per iteration instead of two kernel
// launches; partials of the two dots go to separate arrays, so a CTA still folding one dot
// never races a CTA already writing the next.
template <int W>
__global__ void __launch_bounds__(kDotThreads) k_cg_persist(const int32_t *__restrict__ rowptr,
                                                            const int32_t *__restrict__ col,
                                                            const double *__restrict__ val, double *x,
                                                            double *r, double *p, double *q, int64_t m, int ga,
                                                            int nb, int maxit, double *partA, double *partB,
                                                            CgScalars *sc, double *hist) {
  __shared__ double red[kDotThreads / 32];
  __shared__ double total;
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  double rr = sc->rr, alpha = sc->alpha, beta = sc->beta;
  int stopped = sc->stopped, iter = sc->iter;
  const int b = blockIdx.x;
  constexpr int U = 8;
  for (int it = 0; it < maxit; ++it) {
    // ---- q = A p_i, partials of p_i . q (k_cg_spmv_dot)
    if (b < ga) {
      auto pv = [&](int64_t c) { return __dadd_rn(r[c], __dmul_rn(beta, p[c])); };
      const int64_t row = (b * (int64_t)kDotThreads + threadIdx.x) / W;
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
        for (int u = 0; u < U; ++u) xv[u] = pv(c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (e0 + u * W < z) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
      }
#pragma unroll
      for (int o = W >> 1; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o, W));
      double pq = 0.0;
      if (valid && lane == 0) {
        q[row] = s;
        pq = __dmul_rn(pv(row), s);
      }
      pq = block_sum(pq, red);
      if (threadIdx.x == 0) partA[b] = pq;
    }
    grid.sync();
    {  // alpha (the OP_CG_ALPHA step of finalize_cta)
      const double g = fold_partials(partA, ga, red);
      if (threadIdx.x == 0) total = g;
      __syncthreads();
      const double gg = total;
      if (gg == 0.0 || rr == 0.0) stopped = 1;
      alpha = stopped ? 0.0 : rr / gg;
      if (b == 0 && threadIdx.x == 0) sc->pq = gg;
    }
    // ---- p_i stored, x += alpha p_i, r -= alpha q, partials of r.r (k_cg_update_p)
    if (b < nb) {
      const int64_t chunk = (m + nb - 1) / nb;
      const int64_t lo = b * chunk, hi = min(m, lo + chunk);
      const double acc = block_sum(update_p_chunk(x, r, p, q, lo, hi, alpha, beta, !stopped), red);
      if (threadIdx.x == 0) partB[b] = acc;
    }
    grid.sync();
    {  // beta, rr (the OP_CG_BETA step)
      const double g = fold_partials(partB, nb, red);
      if (threadIdx.x == 0) total = g;
      __syncthreads();
      const double gg = total;
      if (!stopped) {
        beta = gg / rr;
        rr = gg;
      }
      iter += 1;
      if (b == 0 && threadIdx.x == 0 && hist) hist[iter] = rr;
      __syncthreads();  // total is rewritten by the next fold
    }
  }
  if (b == 0 && threadIdx.x == 0) {
    sc->rr = rr;
    sc->alpha = alpha;
    sc->beta = beta;
    sc->stopped = stopped;
    sc->iter = iter;
  }
}

// ------------------------------------------------------------------ host side
static int max_dot_blocks(spmat_s *A) { return A->comm->num_sms * 4; }

// CTAs of the update kernels (x/r update + r.r, CG init): ~2 elements per thread (the update
// keeps kU = 4 in flight, so a chunk is one round of loads; Kuu-sized one-launch CG: 9.0 µs per
// iteration vs 9.0 µs at ~8 per thread), at most 4 CTAs per SM; of a pure dot (p.q,
// spmat_vec_dot): one CTA up to 64 elements per thread (the cross-CTA handshake costs more than
// the loop), else the same.  Functions of m only, so every dot of a matrix reduces in the same
// fixed order.
static int dot_blocks(spmat_s *A) {
  const int64_t want = (A->m + 2 * kDotThreads - 1) / (2 * kDotThreads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, max_dot_blocks(A)));
}
static int pure_dot_blocks(spmat_s *A) { return A->m <= 64 * kDotThreads ? 1 : dot_blocks(A); }

static int ensure_ws(spmat_s *A) {
  if (A->cg_partial.n) return SPMAT_OK;
  SP_TRY(A->cg_partial.alloc(max_dot_blocks(A)));
  SP_TRY(A->cg_scalars.alloc(sizeof(CgScalars) / sizeof(double) + 2));
  SP_TRY(A->cg_reduced.alloc(2));
  SP_TRY(A->cg_count.alloc(1));
  SP_CUDA(cudaMemset(A->cg_count.get(), 0, sizeof(unsigned)));
  return SPMAT_OK;
}

// the NCCL path (several ranks without the scalar board) cannot finalize inside the dot kernel
static bool nccl_reduce(spmat_s *A) { return A->comm->nranks > 1 && !A->comm->board_ok; }

static FinArgs fin_args(spmat_s *A, int op, double *result, double *hist) {
  Comm *c = A->comm;
  FinArgs f{};
  f.partial = A->cg_partial.get();
  f.op = op;
  f.sc = (CgScalars *)A->cg_scalars.get();
  f.result = result;
  f.hist = hist;
  f.P = c->nranks;
  f.me = c->rank;
  if (nccl_reduce(A)) {  // the dot kernel only stores partials; finish_nccl does the rest
    f.op = OP_DOT;
    f.result = A->cg_reduced.get();
    return f;
  }
  f.count = A->cg_count.get();
  if (c->nranks > 1) {
    f.peer_line = c->d_peer_line.get();
    f.board_epoch = c->d_board_epoch.get();
    f.err = c->board_err.get();
  }
  return f;
}

// NCCL path: local sum of the partials, ncclAllReduce of the scalar, then the scalar step
static int finish_nccl(spmat_s *A, int op, double *result, double *hist, int np, cudaStream_t s) {
  if (!nccl_reduce(A)) return SPMAT_OK;
  Comm *c = A->comm;
  FinArgs f = fin_args(A, OP_DOT, nullptr, nullptr);
  k_finalize<<<1, kDotThreads, 0, s>>>(f, np);
  SP_LAUNCH();
  SP_NCCL(c->api, c->api->AllReduce(A->cg_reduced.get(), A->cg_reduced.get() + 1, 1, ncclFloat64,
                                    ncclSum, c->nccl, s));
  FinArgs g{};
  g.partial = A->cg_partial.get();
  g.op = op;
  g.sc = (CgScalars *)A->cg_scalars.get();
  g.result = result;
  g.hist = hist;
  g.P = 1;
  g.preduced = A->cg_reduced.get() + 1;
  k_finalize<<<1, kDotThreads, 0, s>>>(g, 0);
  SP_LAUNCH();
  return SPMAT_OK;
}

// one CG iteration on stream s (captured into a graph, or launched directly)
static int cg_iteration(spmat_s *A, double *x, double *rr_hist, cudaStream_t s) {
  const int64_t m = A->m;
  double *r = A->cg_r.get(), *p = A->cg_p.get(), *q = A->cg_q.get();
  CgScalars *sc = (CgScalars *)A->cg_scalars.get();
  const int nb = dot_blocks(A);
  const unsigned gv = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)A->comm->num_sms * 8));
  const int64_t fused_grid = (m * A->lanes + kDotThreads - 1) / kDotThreads;
  if (A->comm->nranks == 1 && A->kernel_id == 5 && A->bs == 1 && m > 0 && fused_grid <= max_dot_blocks(A)) {
    // q = A p and p.q in one kernel (small matrices, one rank)
    const FinArgs f = fin_args(A, OP_CG_ALPHA, nullptr, nullptr);
    const int32_t *rp = A->rowptr_d.get(), *cl = A->col_d.get();
    const double *vl = A->val_d.get();
    const unsigned g = (unsigned)fused_grid;
    const double *rr = r;  // p_i = r + beta p_{i-1} formed on the fly (the p update folded in)
    cudaError_t e;
    switch (A->lanes) {
      case 1: e = launch_pdl(k_cg_spmv_dot<1>, g, kDotThreads, 0, s, rp, cl, vl, (const double *)p, q, m, f, rr); break;
      case 2: e = launch_pdl(k_cg_spmv_dot<2>, g, kDotThreads, 0, s, rp, cl, vl, (const double *)p, q, m, f, rr); break;
      case 4: e = launch_pdl(k_cg_spmv_dot<4>, g, kDotThreads, 0, s, rp, cl, vl, (const double *)p, q, m, f, rr); break;
      case 8: e = launch_pdl(k_cg_spmv_dot<8>, g, kDotThreads, 0, s, rp, cl, vl, (const double *)p, q, m, f, rr); break;
      case 16: e = launch_pdl(k_cg_spmv_dot<16>, g, kDotThreads, 0, s, rp, cl, vl, (const double *)p, q, m, f, rr); break;
      default: e = launch_pdl(k_cg_spmv_dot<32>, g, kDotThreads, 0, s, rp, cl, vl, (const double *)p, q, m, f, rr); break;
    }
    SP_CUDA(e);
    // x, r update with p_i formed and stored here; no separate p update
    SP_CUDA(launch_pdl(k_cg_update_p, nb, kDotThreads, 0, s, x, r, p, (const double *)q, m,
                       fin_args(A, OP_CG_BETA, nullptr, rr_hist)));
    return SPMAT_OK;
  } else {
    SP_TRY(spmat_mult_part(A, p, q, 7, s));                            // q = A p
    SP_CUDA(launch_pdl(aligned16(p, q) ? k_dot_partial<true> : k_dot_partial<false>, pure_dot_blocks(A),
                       kDotThreads, 0, s, (const double *)p, (const double *)q, m,
                       fin_args(A, OP_CG_ALPHA, nullptr, nullptr)));
    SP_TRY(finish_nccl(A, OP_CG_ALPHA, nullptr, nullptr, pure_dot_blocks(A), s));  // alpha = rr / p.q
  }
  SP_CUDA(launch_pdl(k_cg_update, nb, kDotThreads, 0, s, x, r, (const double *)p, (const double *)q, m,
                     fin_args(A, OP_CG_BETA, nullptr, rr_hist)));
  SP_TRY(finish_nccl(A, OP_CG_BETA, nullptr, rr_hist, nb, s));      // beta, rr = r.r
  SP_CUDA(launch_pdl(k_cg_pupdate, gv, 256, 0, s, p, (const double *)r, m, (const CgScalars *)sc));  // p = r + beta p
  return SPMAT_OK;
}

// the persistent small-matrix CG: one rank, the direct SpMV regime, every CTA resident
static int64_t fused_grid_of(spmat_s *A) { return (A->m * A->lanes + kDotThreads - 1) / kDotThreads; }

static bool persist_ok(spmat_s *A) {
  const char *e = getenv("SPMAT_CG_PERSIST");
  if (e && !strcmp(e, "0")) return false;
  return A->comm->nranks == 1 && A->kernel_id == 5 && A->bs == 1 && A->m > 0 &&
         fused_grid_of(A) <= max_dot_blocks(A) && !A->profile;
}

template <int W>
static cudaError_t launch_persist(spmat_s *A, double *x, double *hist, int maxit, int ga, int nb, int grid,
                                  cudaStream_t s) {
  auto kern = k_cg_persist<W>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDotThreads, 0);
  if (e != cudaSuccess) return e;
  if ((int64_t)per_sm * A->comm->num_sms < grid) return cudaErrorCooperativeLaunchTooLarge;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDotThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  double *partA = A->cg_partial.get(), *partB = A->cg_partial2.get();
  return cudaLaunchKernelEx(&cfg, kern, (const int32_t *)A->rowptr_d.get(), (const int32_t *)A->col_d.get(),
                            (const double *)A->val_d.get(), x, A->cg_r.get(), A->cg_p.get(), A->cg_q.get(), A->m,
                            ga, nb, maxit, partA, partB, (CgScalars *)A->cg_scalars.get(), hist);
}

static int cg_persist(spmat_s *A, double *x, double *hist, int maxit, cudaStream_t s) {
  if (A->cg_partial2.n == 0) SP_TRY(A->cg_partial2.alloc(max_dot_blocks(A)));
  const int ga = (int)fused_grid_of(A), nb = dot_blocks(A), grid = std::max(ga, nb);
  cudaError_t e;
  switch (A->lanes) {
    case 1: e = launch_persist<1>(A, x, hist, maxit, ga, nb, grid, s); break;
    case 2: e = launch_persist<2>(A, x, hist, maxit, ga, nb, grid, s); break;
    case 4: e = launch_persist<4>(A, x, hist, maxit, ga, nb, grid, s); break;
    case 8: e = launch_persist<8>(A, x, hist, maxit, ga, nb, grid, s); break;
    case 16: e = launch_persist<16>(A, x, hist, maxit, ga, nb, grid, s); break;
    default: e = launch_persist<32>(A, x, hist, maxit, ga, nb, grid, s); break;
  }
  SP_CUDA(e);
  return SPMAT_OK;
}

constexpr int kCgBatch = 8;  // CG iterations per graph launch

static bool graph_ok(spmat_s *A) {
  const char *e = getenv("SPMAT_GRAPH");
  if (e && !strcmp(e, "0")) return false;
  if (A->profile) return false;
  if (A->comm->nranks == 1) return true;
  return A->peer && A->comm->board_ok;  // NCCL stays out of captured graphs
}

static void cg_graph_release_execs(spmat_s *A) {
  if (A->cg_exec) cudaGraphExecDestroy(A->cg_exec);
  if (A->cg_exec_batch) cudaGraphExecDestroy(A->cg_exec_batch);
  A->cg_exec = A->cg_exec_batch = nullptr;
}

void cg_graph_release(spmat_s *A) {
  cg_graph_release_execs(A);
  if (A->cg_stream) cudaStreamDestroy(A->cg_stream);
  A->cg_stream = nullptr;
  for (auto &e : A->cg_ev)
    if (e) cudaEventDestroy(e), e = nullptr;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_vec_dot(spmat_t A, const double *a, const double *b, double *result, void *stream) {
  SP_NVTX("spmat_vec_dot");
  if (!A || !result || (A->m > 0 && (!a || !b))) return fail(SPMAT_ERR_ARG, "spmat_vec_dot: null argument");
  DeviceGuard g(A->comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  SP_TRY(ensure_ws(A));
  SP_CUDA(launch_pdl(aligned16(a, b) ? k_dot_partial<true> : k_dot_partial<false>, pure_dot_blocks(A),
                     kDotThreads, 0, s, a, b, A->m, fin_args(A, OP_DOT, result, nullptr)));
  return finish_nccl(A, OP_DOT, result, nullptr, pure_dot_blocks(A), s);
}

int spmat_cg(spmat_t A, const double *b, double *x, int maxit, double *rr_hist, void *stream) {
  SP_NVTX("spmat_cg");
  if (!A || maxit < 0 || (A->m > 0 && (!b || !x)))
    return fail(SPMAT_ERR_ARG, "spmat_cg: bad argument");
  if (A->M != A->N || A->m != A->n) return fail(SPMAT_ERR_ARG, "spmat_cg: matrix must be square");
  if (!A->values_set && A->nnz_d + A->nnz_o > 0)
    return fail(SPMAT_ERR_STATE, "spmat_cg before spmat_set_values_coo");
  DeviceGuard g(A->comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  SP_TRY(ensure_ws(A));
  const int64_t m = A->m;
  if (A->cg_r.n < (size_t)m || A->cg_r.n == 0) {
    SP_TRY(A->cg_r.alloc(std::max<int64_t>(m, 1)));
    SP_TRY(A->cg_p.alloc(std::max<int64_t>(m, 1)));
    SP_TRY(A->cg_q.alloc(std::max<int64_t>(m, 1)));
  }
  double *r = A->cg_r.get(), *p = A->cg_p.get(), *q = A->cg_q.get();
  const int nb = dot_blocks(A);
  const bool use_graph = graph_ok(A) && maxit > 0;
  cudaStream_t cs = s;
  if (use_graph) {  // our own stream (capturable even when the caller uses the legacy stream)
    if (!A->cg_stream) {
      SP_CUDA(cudaStreamCreateWithFlags(&A->cg_stream, cudaStreamNonBlocking));
      SP_CUDA(cudaEventCreateWithFlags(&A->cg_ev[0], cudaEventDisableTiming));
      SP_CUDA(cudaEventCreateWithFlags(&A->cg_ev[1], cudaEventDisableTiming));
    }
    cs = A->cg_stream;
    SP_CUDA(cudaEventRecord(A->cg_ev[0], s));
    SP_CUDA(cudaStreamWaitEvent(cs, A->cg_ev[0], 0));
  }
  // r = b - A x; p = r; rr = r.r
  SP_TRY(spmat_mult_part(A, x, q, 7, cs));
  SP_CUDA(launch_pdl(k_cg_init, nb, kDotThreads, 0, cs, b, (const double *)q, r, p, m,
                     fin_args(A, OP_CG_INIT, nullptr, rr_hist)));
  SP_TRY(finish_nccl(A, OP_CG_INIT, nullptr, rr_hist, nb, cs));
  if (maxit > 0 && persist_ok(A)) {  // every iteration in one cooperative launch
    SP_TRY(cg_persist(A, x, rr_hist, maxit, cs));
    if (use_graph) {
      SP_CUDA(cudaEventRecord(A->cg_ev[1], cs));
      SP_CUDA(cudaStreamWaitEvent(s, A->cg_ev[1], 0));
    }
    return SPMAT_OK;
  }
  if (!use_graph) {
    for (int k = 0; k < maxit; ++k) SP_TRY(cg_iteration(A, x, rr_hist, s));
    return SPMAT_OK;
  }
  // two graphs: one iteration, and kCgBatch iterations (one graph launch per kCgBatch
  // iterations: for small systems the per-launch cost of a graph is a large part of an iteration)
  if (!A->cg_exec || A->cg_key_x != x || A->cg_key_h != rr_hist) {
    cg_graph_release_execs(A);
    for (int w = 0; w < 2; ++w) {
      const int iters = w == 0 ? 1 : kCgBatch;
      cudaGraph_t graph;
      SP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int st = SPMAT_OK;
      for (int k = 0; k < iters && st == SPMAT_OK; ++k) st = cg_iteration(A, x, rr_hist, cs);
      cudaError_t e = cudaStreamEndCapture(cs, &graph);
      if (st != SPMAT_OK) return st;
      if (e != cudaSuccess) return fail(SPMAT_ERR_CUDA, "spmat_cg: graph capture: %s", cudaGetErrorString(e));
      e = cudaGraphInstantiate(w == 0 ? &A->cg_exec : &A->cg_exec_batch, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return fail(SPMAT_ERR_CUDA, "spmat_cg: graph instantiate: %s", cudaGetErrorString(e));
    }
    A->cg_key_x = x;
    A->cg_key_h = rr_hist;
  }
  int k = 0;
  for (; k + kCgBatch <= maxit; k += kCgBatch) SP_CUDA(cudaGraphLaunch(A->cg_exec_batch, cs));
  for (; k < maxit; ++k) SP_CUDA(cudaGraphLaunch(A->cg_exec, cs));
  SP_CUDA(cudaEventRecord(A->cg_ev[1], cs));
  SP_CUDA(cudaStreamWaitEvent(s, A->cg_ev[1], 0));
  return SPMAT_OK;
}

}  // extern "C"
