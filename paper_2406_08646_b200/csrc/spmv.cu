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

enum { KERNEL_STREAM = 1, KERNEL_VECTOR = 2 };

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
  A->kernel_id = KERNEL_STREAM;
  const char *env = getenv("SPMAT_SPMV_KERNEL");
  if (env && !strcmp(env, "vector")) A->kernel_id = KERNEL_VECTOR;
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
