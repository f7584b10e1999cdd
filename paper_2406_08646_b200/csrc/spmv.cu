// spmv.cu -- CSR SpMV kernels for sm_100a and the MatMult orchestration.
//
// MatMult on MPIAIJ: y = A_d x_local + A_o lvec, where
// lvec holds the ghost x entries fetched by a halo SF broadcast.  The paper's
// GPUs used the vendor csrMV (cuSPARSE); here every step is a hand-written kernel.
//
// SpMV is HBM-bound (2 flops per 12 bytes of val+col, AI ~0.15 flop/B): no tensor cores.
// The diagonal block uses a row-block "stream" kernel: the rows are cut into blocks of at
// most kRows rows and ~kTile nonzeros (boundaries from the row pointer, precomputed once);
// a CTA streams its block's val/col with coalesced loads, many in flight per thread,
// multiplies by the gathered x (read through L1/L2 -- stencil locality keeps the
// +-plane window cache-resident), parks the products in shared memory, then one thread per
// row sums its products left to right.  Rows longer than kLong get a block of their own and
// a CTA-wide reduction.  A sub-warp "vector" kernel is kept for long-row matrices.
//
// The halo exchange is issued first on the high-priority comm stream (NCCL), the
// diagonal SpMV runs on the caller's stream meanwhile, and the off-diagonal SpMV-add waits
// on the halo event on the device -- the host never blocks (contrast P:492-509).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace spmat {

constexpr int kThreads = 256;       // CTA size of the stream kernel
constexpr int kRows = kThreads;     // max rows per row block
constexpr int kTile = 1792;         // target nonzeros per row block (7 * 256)
constexpr int kLong = 256;          // rows longer than this get their own block
constexpr int kCap = kTile + kLong; // shared-memory product buffer (doubles)

enum { KERNEL_STREAM = 1, KERNEL_VECTOR = 2, KERNEL_TMA = 3 };

// bulk-copy (TMA engine) pipeline of the persistent SpMV
constexpr int kStages = 3;
constexpr int kValCap = kCap + 2;   // doubles per stage (16-byte alignment slop)
constexpr int kColCap = kCap + 4;   // ints per stage
constexpr int kRpCap = kRows + 8;   // row-pointer ints per stage
struct __align__(16) TmaStage {
  double val[kValCap];
  int col[kColCap];
  int rp[kRpCap];
  int4 hdr;  // r0, r1, p0, p1 of the row block held by this stage
  int4 pad;
};
constexpr size_t kTmaSmem = kStages * sizeof(TmaStage) + kStages * sizeof(unsigned long long);

#define GRID_STRIDE(t, n) \
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (n); t += (int64_t)gridDim.x * blockDim.x)

static inline unsigned nblk(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)1 << 30));
}

// ------------------------------------------------------------------ row-block schedule
__global__ void k_rb_candidates(const int32_t *__restrict__ rowptr, int64_t m, int64_t nnz,
                                int64_t n_tile, int64_t n_rowc, int32_t *__restrict__ cand) {
  GRID_STRIDE(t, n_tile + n_rowc) {
    int32_t r;
    if (t < n_tile) {  // first row whose start is >= t * kTile
      int64_t target = t * (int64_t)kTile;
      int64_t lo = 0, hi = m;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (rowptr[mid] < target) lo = mid + 1; else hi = mid;
      }
      r = (int32_t)lo;
    } else {
      int64_t b = t - n_tile;
      r = (int32_t)std::min<int64_t>(b * kRows, m);
    }
    cand[t] = r;
  }
}

__global__ void k_long_rows(const int32_t *__restrict__ rowptr, int64_t m,
                            uint32_t *__restrict__ flag, int32_t *__restrict__ maxlen) {
  GRID_STRIDE(r, m) {
    int32_t len = rowptr[r + 1] - rowptr[r];
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

__global__ void k_rb_pairs(const int32_t *__restrict__ rows, const int32_t *__restrict__ rowptr,
                           int64_t n, int2 *__restrict__ out) {
  GRID_STRIDE(t, n) out[t] = make_int2(rows[t], rowptr[rows[t]]);
}

__global__ void k_spmv_tma(const int2 *__restrict__ rb, int n_blocks, const int32_t *__restrict__ rowptr,
                           const int32_t *__restrict__ col, const double *__restrict__ val,
                           const double *__restrict__ x, double *__restrict__ y);

#define CUB_CALL(tmp, call_with_tmp)                     \
  do {                                                   \
    size_t temp_storage_bytes = 0;                       \
    void *d_temp_storage = nullptr;                      \
    SP_CUDA(call_with_tmp);                              \
    if (temp_storage_bytes > (tmp).n) SP_TRY((tmp).alloc(temp_storage_bytes)); \
    d_temp_storage = (tmp).get();                        \
    SP_CUDA(call_with_tmp);                              \
  } while (0)

int spmv_prepare(spmat_s *A, cudaStream_t st) {
  const int64_t m = A->m, nnz = A->nnz_d;
  A->kernel_id = KERNEL_TMA;
  const char *env = getenv("SPMAT_SPMV_KERNEL");
  if (env && !strcmp(env, "vector")) A->kernel_id = KERNEL_VECTOR;
  if (env && !strcmp(env, "stream")) A->kernel_id = KERNEL_STREAM;
  A->max_row_nnz = 0;
  A->n_rowblocks = 0;
  if (m == 0) {
    SP_TRY(A->rowblocks.alloc(1));
    SP_CUDA(cudaMemsetAsync(A->rowblocks.get(), 0, 4, st));
    return SPMAT_OK;
  }
  DevBuf<char> tmp;
  DevBuf<uint32_t> flag;
  DevBuf<int32_t> longrows, maxlen, nlong_d;
  SP_TRY(flag.alloc(m));
  SP_TRY(longrows.alloc(m));
  SP_TRY(maxlen.alloc(2));
  SP_CUDA(cudaMemsetAsync(maxlen.get(), 0, 8, st));
  k_long_rows<<<nblk(m), 256, 0, st>>>(A->rowptr_d.get(), m, flag.get(), maxlen.get());
  SP_LAUNCH();
  CUB_CALL(tmp, cub::DeviceSelect::Flagged(d_temp_storage, temp_storage_bytes,
                                           cub::CountingInputIterator<int32_t>(0), flag.get(),
                                           longrows.get(), maxlen.get() + 1, (int)m, st));
  int32_t h[2];
  SP_CUDA(cudaMemcpyAsync(h, maxlen.get(), 8, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  A->max_row_nnz = h[0];
  const int64_t nlong = h[1];
  const int64_t n_tile = (nnz + kTile - 1) / kTile;
  const int64_t n_rowc = (m + kRows - 1) / kRows + 1;  // includes m itself
  const int64_t ncand = n_tile + n_rowc + 2 * nlong;
  DevBuf<int32_t> cand, sorted, uniq;
  DevBuf<int> dn;
  SP_TRY(cand.alloc(ncand));
  SP_TRY(sorted.alloc(ncand));
  SP_TRY(uniq.alloc(ncand));
  SP_TRY(dn.alloc(1));
  k_rb_candidates<<<nblk(n_tile + n_rowc), 256, 0, st>>>(A->rowptr_d.get(), m, nnz, n_tile, n_rowc,
                                                         cand.get());
  SP_LAUNCH();
  if (nlong > 0) {
    k_long_bounds<<<nblk(nlong), 256, 0, st>>>(longrows.get(), nlong, cand.get() + n_tile + n_rowc);
    SP_LAUNCH();
  }
  CUB_CALL(tmp, cub::DeviceRadixSort::SortKeys(d_temp_storage, temp_storage_bytes, cand.get(),
                                               sorted.get(), (int)ncand, 0, 32, st));
  CUB_CALL(tmp, cub::DeviceSelect::Unique(d_temp_storage, temp_storage_bytes, sorted.get(),
                                          uniq.get(), dn.get(), (int)ncand, st));
  int nu = 0;
  SP_CUDA(cudaMemcpyAsync(&nu, dn.get(), 4, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  // uniq holds 0 = r_0 < r_1 < ... < r_last = m
  A->n_rowblocks = nu - 1;
  SP_TRY(A->rowblocks.alloc(nu));
  SP_CUDA(cudaMemcpyAsync(A->rowblocks.get(), uniq.get(), (size_t)nu * 4, cudaMemcpyDeviceToDevice, st));
  SP_TRY(A->rbp.alloc(nu));
  k_rb_pairs<<<nblk(nu), 256, 0, st>>>(A->rowblocks.get(), A->rowptr_d.get(), nu, A->rbp.get());
  SP_LAUNCH();
  A->n_long = nlong;
  SP_TRY(A->longrows.alloc(nlong));
  if (nlong)
    SP_CUDA(cudaMemcpyAsync(A->longrows.get(), longrows.get(), (size_t)nlong * 4, cudaMemcpyDeviceToDevice, st));
  // persistent grid: as many CTAs as fit (2 per SM at ~80 KB of shared memory each)
  static bool attr_set = false;
  if (!attr_set) {
    SP_CUDA(cudaFuncSetAttribute(k_spmv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
    attr_set = true;
  }
  int per_sm = 0;
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_tma, kThreads, kTmaSmem));
  A->tma_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * A->comm->num_sms, A->n_rowblocks));
  SP_CUDA(cudaStreamSynchronize(st));
  return SPMAT_OK;
}

// ------------------------------------------------------------------ kernels
__device__ __forceinline__ double ld_stream(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// y[r] = sum_e val[e] * x[col[e]] over the row block; products rounded separately and summed
// left to right from +0.0 within each row (same order as a serial CSR loop).
__global__ void __launch_bounds__(kThreads) k_spmv_stream(
    const int32_t *__restrict__ rowblocks, const int32_t *__restrict__ rowptr,
    const int32_t *__restrict__ col, const double *__restrict__ val,
    const double *__restrict__ x, double *__restrict__ y) {
  __shared__ double prod[kCap];
  __shared__ double red[kThreads / 32];
  const int b = blockIdx.x;
  const int r0 = rowblocks[b], r1 = rowblocks[b + 1];
  const int p0 = rowptr[r0], p1 = rowptr[r1];
  const int n = p1 - p0;
  const int tid = threadIdx.x;
  if (n <= kCap) {
    constexpr int U = 8;
    for (int base = 0; base < n; base += kThreads * U) {
      int c[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int e = base + u * kThreads + tid;
        if (e < n) {
          c[u] = ld_stream(col + p0 + e);
          v[u] = ld_stream(val + p0 + e);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int e = base + u * kThreads + tid;
        if (e < n) prod[e] = __dmul_rn(v[u], __ldg(x + c[u]));
      }
    }
    __syncthreads();
    const int r = r0 + tid;
    if (r < r1) {
      const int a = rowptr[r] - p0, z = rowptr[r + 1] - p0;
      double s = 0.0;
      for (int e = a; e < z; ++e) s = __dadd_rn(s, prod[e]);
      y[r] = s;
    }
  } else {  // a single long row: CTA-wide reduction
    double s = 0.0;
    for (int e = tid; e < n; e += kThreads)
      s = __dadd_rn(s, __dmul_rn(ld_stream(val + p0 + e), __ldg(x + ld_stream(col + p0 + e))));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) t = __dadd_rn(t, red[w]);
      y[r0] = t;
    }
  }
}

// W lanes per row; lanes stride the row, shuffle reduction.
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


// ------------------------------------------------------------------ bulk-copy (TMA) SpMV
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
// global -> shared bulk copy on the TMA engine, completion counted on an mbarrier;
// L2 evict_first: val/col/rowptr are streamed once, x should stay resident
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         unsigned long long *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Persistent CTAs, each owning a contiguous range of row blocks.  Thread 0 keeps kStages
// row blocks in flight: val, col and row-pointer slices of a row block land in a shared
// memory stage through cp.async.bulk, tracked by that stage's mbarrier.  All threads then
// (1) gather x and overwrite val with the products in place, (2) sum rows -- one thread per
// row, left to right, when the block has >= kThreads/2 rows (the stencil case, bit-identical
// to a serial CSR loop), otherwise W lanes per row with a shuffle reduction -- and (3) free
// the stage, which thread 0 refills with the row block kStages ahead.
__global__ void __launch_bounds__(kThreads, 2)
    k_spmv_tma(const int2 *__restrict__ rb, int n_blocks, const int32_t *__restrict__ rowptr,
               const int32_t *__restrict__ col, const double *__restrict__ val,
               const double *__restrict__ x, double *__restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  TmaStage *st = reinterpret_cast<TmaStage *>(smem);
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + kStages * sizeof(TmaStage));
  const int tid = threadIdx.x;
  const int G = gridDim.x, c = blockIdx.x;
  const int b0 = (int)((long long)n_blocks * c / G), b1 = (int)((long long)n_blocks * (c + 1) / G);
  const int nb = b1 - b0;
  if (nb <= 0) return;
  uint64_t policy = 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  }
  __syncthreads();
  // thread 0: issue row block `it` (relative to b0) into stage it % kStages
  int2 nA, nB;  // prefetched bounds of the next block to issue
  auto issue = [&](int it, int2 A, int2 B) {
    const int s = it % kStages;
    const int r0 = A.x, r1 = B.x, p0 = A.y, p1 = B.y;
    st[s].hdr = make_int4(r0, r1, p0, p1);
    if (p1 - p0 > kCap) {  // long row: done by k_spmv_long
      mbar_arrive_tx(&bars[s], 0);
      return;
    }
    const int va = p0 & ~1, ve = (p1 + 1) & ~1;
    const int ca = p0 & ~3, ce = (p1 + 3) & ~3;
    const int ra = r0 & ~3, re = (r1 + 4) & ~3;
    const uint32_t bytes = (uint32_t)((ve - va) * 8 + (ce - ca) * 4 + (re - ra) * 4);
    mbar_arrive_tx(&bars[s], bytes);
    if (ve > va) bulk_g2s(st[s].val, val + va, (ve - va) * 8, &bars[s], policy);
    if (ce > ca) bulk_g2s(st[s].col, col + ca, (ce - ca) * 4, &bars[s], policy);
    bulk_g2s(st[s].rp, rowptr + ra, (re - ra) * 4, &bars[s], policy);
  };
  if (tid == 0) {
    const int pre = min(kStages, nb);
    for (int it = 0; it < pre; ++it) issue(it, rb[b0 + it], rb[b0 + it + 1]);
    if (pre < nb) {
      nA = rb[b0 + pre];
      nB = rb[b0 + pre + 1];
    }
  }
  __syncthreads();  // stage headers visible
  for (int it = 0; it < nb; ++it) {
    const int s = it % kStages;
    mbar_wait(&bars[s], (uint32_t)((it / kStages) & 1));
    const int4 h = st[s].hdr;
    const int r0 = h.x, r1 = h.y, p0 = h.z, p1 = h.w, n = p1 - p0;
    if (n <= kCap) {
      double *sv = st[s].val + (p0 - (p0 & ~1));
      const int *sc = st[s].col + (p0 - (p0 & ~3));
      const int *rp = st[s].rp - (r0 & ~3);  // rp[r] = rowptr[r]
      constexpr int U = 8;
      for (int base = 0; base < n; base += kThreads * U) {
        int cc[U];
        double xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = base + u * kThreads + tid;
          cc[u] = e < n ? sc[e] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = cc[u] >= 0 ? __ldg(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = base + u * kThreads + tid;
          if (e < n) sv[e] = __dmul_rn(sv[e], xv[u]);
        }
      }
      __syncthreads();
      const int nrows = r1 - r0;
      if (nrows * 2 >= kThreads) {
        for (int r = r0 + tid; r < r1; r += kThreads) {
          const int a = rp[r] - p0, z = rp[r + 1] - p0;
          double acc = 0.0;
          for (int e = a; e < z; ++e) acc = __dadd_rn(acc, sv[e]);
          y[r] = acc;
        }
      } else {
        int W = 1;
        while (W < 32 && nrows * W * 2 <= kThreads) W <<= 1;
        const int r = r0 + tid / W, lane = tid % W;
        double acc = 0.0;
        if (r < r1) {
          const int a = rp[r] - p0, z = rp[r + 1] - p0;
          for (int e = a + lane; e < z; e += W) acc = __dadd_rn(acc, sv[e]);
        }
        for (int o = W >> 1; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o, W));
        if (r < r1 && lane == 0) y[r] = acc;
      }
    }
    __syncthreads();  // stage s consumed by every thread
    if (tid == 0 && it + kStages < nb) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
      issue(it + kStages, nA, nB);
      if (it + kStages + 1 < nb) {
        nA = nB;
        nB = rb[b0 + it + kStages + 2];
      }
    }
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
  for (int e = a + threadIdx.x; e < z; e += kThreads) s = __dadd_rn(s, __dmul_rn(val[e], __ldg(x + col[e])));
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

// y[rows_o[q]] = y[rows_o[q]] + (sum over the compressed off-diagonal row, left to right)
__global__ void __launch_bounds__(256) k_spmv_offdiag(const int32_t *__restrict__ rows,
                                                      const int32_t *__restrict__ rowptr,
                                                      const int32_t *__restrict__ col,
                                                      const double *__restrict__ val,
                                                      const double *__restrict__ lvec,
                                                      double *__restrict__ y, int64_t nro) {
  GRID_STRIDE(q, nro) {
    double s = 0.0;
    for (int e = rowptr[q]; e < rowptr[q + 1]; ++e)
      s = __dadd_rn(s, __dmul_rn(val[e], lvec[col[e]]));
    const int r = rows[q];
    y[r] = __dadd_rn(y[r], s);
  }
}

int spmv_diag(spmat_s *A, const double *x, double *y, cudaStream_t s) {
  if (A->m == 0) return SPMAT_OK;
  if (A->kernel_id == KERNEL_VECTOR) {
    double mean = A->m ? (double)A->nnz_d / (double)A->m : 0.0;
    if (mean <= 6) {
      k_spmv_vector<4><<<nblk(A->m * 4), 256, 0, s>>>(A->rowptr_d.get(), A->col_d.get(), A->val_d.get(), x, y, A->m);
    } else if (mean <= 12) {
      k_spmv_vector<8><<<nblk(A->m * 8), 256, 0, s>>>(A->rowptr_d.get(), A->col_d.get(), A->val_d.get(), x, y, A->m);
    } else if (mean <= 24) {
      k_spmv_vector<16><<<nblk(A->m * 16), 256, 0, s>>>(A->rowptr_d.get(), A->col_d.get(), A->val_d.get(), x, y, A->m);
    } else {
      k_spmv_vector<32><<<nblk(A->m * 32), 256, 0, s>>>(A->rowptr_d.get(), A->col_d.get(), A->val_d.get(), x, y, A->m);
    }
    SP_LAUNCH();
    return SPMAT_OK;
  }
  if (A->kernel_id == KERNEL_TMA) {
    k_spmv_tma<<<(unsigned)A->tma_grid, kThreads, kTmaSmem, s>>>(A->rbp.get(), (int)A->n_rowblocks,
                                                               A->rowptr_d.get(), A->col_d.get(),
                                                               A->val_d.get(), x, y);
    SP_LAUNCH();
    if (A->n_long > 0) {
      k_spmv_long<<<(unsigned)A->n_long, kThreads, 0, s>>>(A->longrows.get(), A->rowptr_d.get(),
                                                           A->col_d.get(), A->val_d.get(), x, y);
      SP_LAUNCH();
    }
    return SPMAT_OK;
  }
  k_spmv_stream<<<(unsigned)A->n_rowblocks, kThreads, 0, s>>>(A->rowblocks.get(), A->rowptr_d.get(),
                                                             A->col_d.get(), A->val_d.get(), x, y);
  SP_LAUNCH();
  return SPMAT_OK;
}

int spmv_offdiag(spmat_s *A, double *y, cudaStream_t s) {
  if (A->n_ro == 0) return SPMAT_OK;
  k_spmv_offdiag<<<nblk(A->n_ro), 256, 0, s>>>(A->rows_o.get(), A->rowptr_o.get(), A->col_o.get(),
                                              A->val_o.get(), A->lvec.get(), y, A->n_ro);
  SP_LAUNCH();
  return SPMAT_OK;
}

static cudaEvent_t *prof_pair(spmat_s *A, int kind) {
  auto &v = A->prof_ev[kind];
  size_t i = A->prof_n[kind];
  if (2 * i + 2 > v.size()) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return nullptr;
    v.push_back(a);
    v.push_back(b);
  }
  A->prof_n[kind]++;
  return &v[2 * i];
}

static int mult_impl(spmat_s *A, const double *x, double *y, int part, cudaStream_t s) {
  const bool halo = (part & 2) && A->comm->nranks > 1;
  cudaEvent_t *pe;
  if (halo) {
    pe = A->profile ? prof_pair(A, 2) : nullptr;
    SP_TRY(sf_begin(A->halo, x, A->lvec.get(), SF_REPLACE, s, pe));
  }
  if (part & 1) {
    pe = A->profile ? prof_pair(A, 0) : nullptr;
    if (pe) SP_CUDA(cudaEventRecord(pe[0], s));
    SP_TRY(spmv_diag(A, x, y, s));
    if (pe) SP_CUDA(cudaEventRecord(pe[1], s));
  }
  if (halo) SP_TRY(sf_end(A->halo, x, A->lvec.get(), SF_REPLACE, s));
  if ((part & 4) && A->n_ro > 0) {
    pe = A->profile ? prof_pair(A, 1) : nullptr;
    if (pe) SP_CUDA(cudaEventRecord(pe[0], s));
    SP_TRY(spmv_offdiag(A, y, s));
    if (pe) SP_CUDA(cudaEventRecord(pe[1], s));
  }
  return SPMAT_OK;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_mult(spmat_t A, const double *x, double *y, void *stream) {
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_mult: null matrix");
  if ((A->n > 0 && !x) || (A->m > 0 && !y)) return fail(SPMAT_ERR_ARG, "spmat_mult: null x or y");
  if (x && (const void *)x == (const void *)y) return fail(SPMAT_ERR_ARG, "spmat_mult: x and y alias");
  if (!A->values_set && A->nnz_d + A->nnz_o > 0)
    return fail(SPMAT_ERR_STATE, "spmat_mult before spmat_set_values_coo");
  DeviceGuard g(A->comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  const bool hx = A->n > 0 && !is_device_ptr(x);
  const bool hy = A->m > 0 && !is_device_ptr(y);
  if (!hx && !hy) return mult_impl(A, x, y, 7, s);
  // host buffers: stage through device copies inside the stream order
  const double *dx = x;
  double *dy = y;
  if (hx) {
    if (A->xstage.n < (size_t)A->n) SP_TRY(A->xstage.alloc(A->n));
    SP_CUDA(cudaMemcpyAsync(A->xstage.get(), x, A->n * 8, cudaMemcpyHostToDevice, s));
    dx = A->xstage.get();
  }
  if (hy) {
    if (A->ystage.n < (size_t)A->m) SP_TRY(A->ystage.alloc(A->m));
    dy = A->ystage.get();
  }
  SP_TRY(mult_impl(A, dx, dy, 7, s));
  if (hy) SP_CUDA(cudaMemcpyAsync(y, dy, A->m * 8, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  return SPMAT_OK;
}

int spmat_mult_part(spmat_t A, const double *x, double *y, int part, void *stream) {
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_mult_part: null matrix");
  if (part < 1 || part > 7) return fail(SPMAT_ERR_ARG, "spmat_mult_part: bad part %d", part);
  if (x && (const void *)x == (const void *)y) return fail(SPMAT_ERR_ARG, "spmat_mult_part: x and y alias");
  DeviceGuard g(A->comm->device);
  return mult_impl(A, x, y, part, (cudaStream_t)stream);
}

int spmat_profile(spmat_t A, int enable) {
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_profile: null matrix");
  A->profile = enable != 0;
  return SPMAT_OK;
}

int spmat_profile_read(spmat_t A, double ms[4], int64_t n[4]) {
  if (!A || !ms || !n) return fail(SPMAT_ERR_ARG, "spmat_profile_read: null argument");
  DeviceGuard g(A->comm->device);
  SP_CUDA(cudaDeviceSynchronize());
  for (int k = 0; k < 4; ++k) {
    ms[k] = 0.0;
    n[k] = 0;
  }
  for (int k = 0; k < 3; ++k) {
    for (size_t i = 0; i < A->prof_n[k]; ++i) {
      float t = 0.f;
      SP_CUDA(cudaEventElapsedTime(&t, A->prof_ev[k][2 * i], A->prof_ev[k][2 * i + 1]));
      ms[k] += t;
    }
    n[k] = (int64_t)A->prof_n[k];
    A->prof_n[k] = 0;
  }
  return SPMAT_OK;
}

}  // extern "C"
