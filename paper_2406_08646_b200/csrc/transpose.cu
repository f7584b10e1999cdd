// transpose.cu -- MatMultTranspose y = A^T x on the row-partitioned MPIAIJ matrix, the
// operation PetscSF's reduce enables.
//
// PETSc's MPIAIJ order, kept here:  lvec = A_o^T x  (one value per ghost column),  y = A_d^T x,
// then the halo SF reduces lvec into the owners' y with SUM (sf_reduce_begin/end: the owner's
// value first, then the contributions in ascending source rank).  The transposed blocks are
// built on the device on the first call (a stable radix sort of the entries by column keeps
// every transposed row in ascending original-row order) and their values re-gathered after
// each spmat_set_values_coo; each y entry is summed left to right from +0.0 with separately
// rounded products -- PETSc's order written out, reproducible bit for bit.
// Not the hot path: plain one-thread-per-row kernels.
#include <cub/cub.cuh>

#include <algorithm>

#include "internal.h"

namespace spmat {

namespace {

#define TGRID(t, n) \
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (n); t += (int64_t)gridDim.x * blockDim.x)

inline unsigned tblocks(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)1 << 20));
}

// row id of every entry of a CSR block with `nrows` rows (row ids mapped through `rows` if given)
__global__ void k_entry_rows(const int32_t *__restrict__ rowptr, int64_t nrows, const int32_t *__restrict__ rows,
                             int32_t *__restrict__ out) {
  TGRID(q, nrows) {
    const int32_t r = rows ? rows[q] : (int32_t)q;
    for (int e = rowptr[q]; e < rowptr[q + 1]; ++e) out[e] = r;
  }
}

__global__ void k_iota32(int32_t *__restrict__ v, int64_t n) { TGRID(t, n) v[t] = (int32_t)t; }

// rowptr_t[c] = first position of key c in the sorted keys (lower bound), c in [0, ncols]
__global__ void k_bounds(const int32_t *__restrict__ skeys, int64_t n, int64_t ncols, int32_t *__restrict__ rowptr_t) {
  TGRID(c, ncols + 1) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (skeys[mid] < c) lo = mid + 1; else hi = mid;
    }
    rowptr_t[c] = (int32_t)lo;
  }
}

__global__ void k_gather_idx(const int32_t *__restrict__ src, const int32_t *__restrict__ perm, int64_t n,
                             int32_t *__restrict__ dst) {
  TGRID(t, n) dst[t] = src[perm[t]];
}

__global__ void k_gather_val(const double *__restrict__ src, const int32_t *__restrict__ perm, int64_t n,
                             double *__restrict__ dst) {
  TGRID(t, n) dst[t] = src[perm[t]];
}

// y[c] = sum over transposed row c, left to right from +0.0
__global__ void k_spmv_t(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
                         const double *__restrict__ val, const double *__restrict__ x, int64_t nrows,
                         double *__restrict__ y) {
  TGRID(c, nrows) {
    double s = 0.0;
    for (int k = rowptr[c]; k < rowptr[c + 1]; ++k) s = __dadd_rn(s, __dmul_rn(val[k], x[col[k]]));
    y[c] = s;
  }
}

struct Tmp {
  DevBuf<char> buf;
  int ensure(size_t n) { return buf.n >= n ? SPMAT_OK : buf.alloc(n); }
};

#define TCUB(tmp, call_with_tmp)                \
  do {                                          \
    size_t temp_storage_bytes = 0;              \
    void *d_temp_storage = nullptr;             \
    SP_CUDA(call_with_tmp);                     \
    SP_TRY((tmp).ensure(temp_storage_bytes));   \
    d_temp_storage = (tmp).buf.get();           \
    SP_CUDA(call_with_tmp);                     \
  } while (0)

// transposed structure of one CSR block: nnz entries with column keys `cols` (in [0, ncols))
// and row ids `erows`; outputs rowptr_t [ncols+1], col_t (original rows) and perm_t (entry ids)
int build_t(const int32_t *cols, const int32_t *erows, int64_t nnz, int64_t ncols, DevBuf<int32_t> &rowptr_t,
            DevBuf<int32_t> &col_t, DevBuf<int32_t> &perm_t, cudaStream_t st) {
  SP_TRY(rowptr_t.alloc(ncols + 1));
  SP_TRY(col_t.alloc(std::max<int64_t>(nnz, 1)));
  SP_TRY(perm_t.alloc(std::max<int64_t>(nnz, 1)));
  if (nnz == 0) {
    SP_CUDA(cudaMemsetAsync(rowptr_t.get(), 0, (ncols + 1) * 4, st));
    return SPMAT_OK;
  }
  DevBuf<int32_t> keys_out, ids;
  Tmp tmp;
  SP_TRY(keys_out.alloc(nnz));
  SP_TRY(ids.alloc(nnz));
  k_iota32<<<tblocks(nnz), 256, 0, st>>>(ids.get(), nnz);
  SP_LAUNCH();
  int bits = 1;
  while (bits < 31 && ((int64_t)1 << bits) <= ncols) ++bits;
  TCUB(tmp, cub::DeviceRadixSort::SortPairs(d_temp_storage, temp_storage_bytes, cols, keys_out.get(), ids.get(),
                                            perm_t.get(), (int)nnz, 0, bits, st));
  k_bounds<<<tblocks(ncols + 1), 256, 0, st>>>(keys_out.get(), nnz, ncols, rowptr_t.get());
  SP_LAUNCH();
  k_gather_idx<<<tblocks(nnz), 256, 0, st>>>(erows, perm_t.get(), nnz, col_t.get());
  SP_LAUNCH();
  SP_CUDA(cudaStreamSynchronize(st));  // the temporaries go out of scope
  return SPMAT_OK;
}

}  // namespace

static int transpose_prepare(spmat_s *A, cudaStream_t s) {
  cudaStream_t st = A->comm->setup_stream;
  if (!A->t_built) {
    DevBuf<int32_t> er;
    SP_TRY(er.alloc(std::max<int64_t>(A->nnz_d, 1)));
    if (A->m > 0) {
      k_entry_rows<<<tblocks(A->m), 256, 0, st>>>(A->rowptr_d.get(), A->m, nullptr, er.get());
      SP_LAUNCH();
    }
    SP_TRY(build_t(A->col_d.get(), er.get(), A->nnz_d, A->n, A->t_rowptr_d, A->t_col_d, A->t_perm_d, st));
    DevBuf<int32_t> ero;
    SP_TRY(ero.alloc(std::max<int64_t>(A->nnz_o, 1)));
    if (A->n_ro > 0) {
      k_entry_rows<<<tblocks(A->n_ro), 256, 0, st>>>(A->rowptr_o.get(), A->n_ro, A->rows_o.get(), ero.get());
      SP_LAUNCH();
    }
    SP_TRY(build_t(A->col_o.get(), ero.get(), A->nnz_o, A->n_ghost, A->t_rowptr_o, A->t_col_o, A->t_perm_o, st));
    SP_TRY(A->t_val_d.alloc(std::max<int64_t>(A->nnz_d, 1)));
    SP_TRY(A->t_val_o.alloc(std::max<int64_t>(A->nnz_o, 1)));
    SP_TRY(A->t_lvec.alloc(std::max<int64_t>(A->n_ghost, 1)));
    SP_CUDA(cudaStreamSynchronize(st));
    A->t_built = true;
    A->t_val_version = -1;
  }
  if (A->t_val_version != A->val_version) {  // values changed since the last gather
    SP_TRY(csr_sync(A, s));  // (stream order: after the set_values that wrote bval)
    if (A->nnz_d > 0) {
      k_gather_val<<<tblocks(A->nnz_d), 256, 0, s>>>(A->val_d.get(), A->t_perm_d.get(), A->nnz_d, A->t_val_d.get());
      SP_LAUNCH();
    }
    if (A->nnz_o > 0) {
      k_gather_val<<<tblocks(A->nnz_o), 256, 0, s>>>(A->val_o.get(), A->t_perm_o.get(), A->nnz_o, A->t_val_o.get());
      SP_LAUNCH();
    }
    A->t_val_version = A->val_version;
  }
  return SPMAT_OK;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_mult_transpose(spmat_t A, const double *x, double *y, void *stream) {
  SP_NVTX("spmat_mult_transpose");
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_mult_transpose: null matrix");
  if ((A->m > 0 && !x) || (A->n > 0 && !y)) return fail(SPMAT_ERR_ARG, "spmat_mult_transpose: null x or y");
  if (x && (const void *)x == (const void *)y) return fail(SPMAT_ERR_ARG, "spmat_mult_transpose: x and y alias");
  if (!A->values_set && A->nnz_d + A->nnz_o > 0)
    return fail(SPMAT_ERR_STATE, "spmat_mult_transpose before spmat_set_values_coo");
  if ((A->m > 0 && !is_device_ptr(x)) || (A->n > 0 && !is_device_ptr(y)))
    return fail(SPMAT_ERR_ARG, "spmat_mult_transpose: x and y must be device arrays");
  DeviceGuard g(A->comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (A->comm->nranks > 1) SP_TRY(sf_ensure_peer(A->halo));  // collective on first call
  SP_TRY(transpose_prepare(A, s));
  const bool multi = A->comm->nranks > 1 && A->halo;
  if (multi && A->n_ghost > 0) {  // lvec = A_o^T x, one value per ghost column
    k_spmv_t<<<tblocks(A->n_ghost), 256, 0, s>>>(A->t_rowptr_o.get(), A->t_col_o.get(), A->t_val_o.get(), x,
                                                 A->n_ghost, A->t_lvec.get());
    SP_LAUNCH();
  }
  if (A->n > 0) {  // y = A_d^T x
    k_spmv_t<<<tblocks(A->n), 256, 0, s>>>(A->t_rowptr_d.get(), A->t_col_d.get(), A->t_val_d.get(), x, A->n, y);
    SP_LAUNCH();
  }
  if (multi) {  // y += the ghosts' sums on their owners (reduce SUM, ascending source rank)
    SP_TRY(sf_reduce_begin_impl(A->halo, A->t_lvec.get(), y, SF_SUM, s));
    SP_TRY(sf_reduce_end_impl(A->halo, A->t_lvec.get(), y, SF_SUM, s));
  }
  return SPMAT_OK;
}

}  // extern "C"
