// halo.cu -- device-initiated halo exchange for MatMult over NVLink peer memory.
//
// The paper's experimental NVSHMEM PetscSF removes the host from the halo
// path: "symmetric send/recv buffers", a kernel "calls nvshmem_putmem_nbi", synchronisation
// on the device.  Its motivation: an MPI/NCCL exchange needs host ordering or,
// as measured here on B200, an NCCL p2p kernel whose handshakes crawl while the SpMV keeps
// HBM saturated (the 17 us transfer then completes only after the SpMV).
//
// B200 design: at create time every rank exports its ghost buffer and a small flag array
// through CUDA IPC; each owner opens the ghost buffer of the ranks that need its rows and
// learns where its values go (the halo SF leaves are contiguous per owner).  Ghost values
// travel as flagged 16-byte lines {value, epoch} (halo_dev.cuh): the flag in the line is the
// readiness signal, so a put is stores only and a reader waits per value.
// Per MatMult (epoch e, kept on the device):
//   put (comm warps of the diagonal SpMV, or k_halo_put): wait until the destination has
//     finished reading epoch e-2 (done flag; two buffers by epoch parity), store the owned x
//     entries as lines flagged e straight into the destination's buffer over NVLink;
//   off-diagonal SpMV-add (the fused kernel's comm warps, or k_spmv_offdiag_peer): read each
//     ghost line until it carries flag e, add A_o lvec into y; the last CTA tells every sender
//     that the buffer may be overwritten (done = e) and advances the epoch.
// The transfer (0.5-2 MB of lines) overlaps the diagonal SpMV; no NCCL kernel, no host
// synchronisation.  Spins are bounded (a stuck peer sets an error word instead of hanging).
#include <algorithm>
#include <cstring>

#include "halo_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace spmat {

constexpr int kPutWarps = 4;  // warps per CTA of the standalone put kernel

static inline int put_chunks(int64_t count) {
  return (int)std::max<int64_t>(1, (count + kPutChunk - 1) / kPutChunk);
}

// standalone put (halo-only MatMult parts, or a diagonal kernel without comm warps)
__global__ void __launch_bounds__(32 * kPutWarps) k_halo_put(const HaloPut *__restrict__ puts, int nputs,
                                                             int total, const double *__restrict__ x,
                                                             const unsigned long long *epoch_ctr, int *err) {
  pdl_wait();
  const int c = blockIdx.x * kPutWarps + (threadIdx.x >> 5);
  if (c < total) halo_put_warp(puts, nputs, c, x, *epoch_ctr + 1ull, err);
}

// y[rows[q]] += A_o lvec with this MatMult's ghost lines (each read waits for its flag); with
// nro == 0 it only waits until all n_ghost lines have landed (halo-only timing).  The last
// CTA releases the buffer to the senders and advances the epoch.
__global__ void __launch_bounds__(256) k_spmv_offdiag_peer(
    const int32_t *__restrict__ rows, const int32_t *__restrict__ rowptr,
    const int32_t *__restrict__ col, const double *__restrict__ val, const uint4 *ghost_base,
    int64_t ghost_stride, int64_t n_ghost, double *__restrict__ y, int64_t nro, int W,
    const HaloWait *__restrict__ waits, int nwaits, unsigned long long *epoch_ctr,
    unsigned int *counter, int *err) {
  pdl_wait();
  // this MatMult's epoch; every CTA reads it before its arrival on `counter`, so before the
  // last CTA stores it back
  const unsigned long long epoch = *epoch_ctr + 1ull;
  const uint32_t flag = ll_flag(epoch);
  const uint4 *gl = ghost_base + (int64_t)(epoch & 1) * ghost_stride;
  if (nro > 0 && W == 1) {
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x * kRowsU; t0 < nro; t0 += (int64_t)gridDim.x * blockDim.x * kRowsU)
      offdiag_rows_u<kRowsU>(t0 + threadIdx.x, blockDim.x, nro, rows, rowptr, col, val, gl, nullptr, flag, err, y);
  } else if (nro > 0) {  // block-uniform loop bound: every lane reaches the shuffles in offdiag_row_w
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < nro * W; t0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t q = (t0 + threadIdx.x) / W;
      offdiag_row_w(q, q < nro, W, rows, rowptr, col, val, gl, nullptr, flag, err, y);
    }
  } else {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_ghost; g += (int64_t)gridDim.x * blockDim.x)
      (void)ll_load(gl + g, flag, err);
  }
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

// Host-buffer pipeline pieces (mult.cu): the off-diagonal SpMV-add of compressed rows [q0, q1)
// with this MatMult's ghost lines (no epoch bookkeeping), and the epoch end: release the
// ghost buffer to the senders and advance the epoch.
__global__ void __launch_bounds__(256) k_offdiag_peer_range(
    const int32_t *__restrict__ rows, const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col,
    const double *__restrict__ val, const uint4 *ghost_base, int64_t ghost_stride, double *__restrict__ y,
    int64_t q0, int64_t q1, int W, const unsigned long long *epoch_ctr, int *err) {
  pdl_wait();
  const unsigned long long epoch = *epoch_ctr + 1ull;
  const uint32_t flag = ll_flag(epoch);
  const uint4 *gl = ghost_base + (int64_t)(epoch & 1) * ghost_stride;
  const int64_t n = q1 - q0;
  if (W == 1) {
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x * kRowsU; t0 < n; t0 += (int64_t)gridDim.x * blockDim.x * kRowsU)
      offdiag_rows_u<kRowsU>(t0 + threadIdx.x, blockDim.x, n, rows + q0, rowptr + q0, col, val, gl, nullptr, flag,
                             err, y);
  } else {
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < n * W; t0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t q = (t0 + threadIdx.x) / W;
      offdiag_row_w(q, q < n, W, rows + q0, rowptr + q0, col, val, gl, nullptr, flag, err, y);
    }
  }
}

__global__ void k_epoch_end(const HaloWait *__restrict__ waits, int nwaits, unsigned long long *epoch_ctr) {
  pdl_wait();
  const unsigned long long epoch = *epoch_ctr + 1ull;
  for (int w = 0; w < nwaits; ++w) st_release_sys(waits[w].peer_done, epoch);
  *epoch_ctr = epoch;
}

int halo_peer_offdiag_range(spmat_s *A, double *y, int64_t q0, int64_t q1, cudaStream_t s) {
  if (q1 <= q0) return SPMAT_OK;
  const int64_t work = A->ro_w == 1 ? (q1 - q0 + kRowsU - 1) / kRowsU : (q1 - q0) * A->ro_w;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 4L * A->comm->num_sms));
  k_offdiag_peer_range<<<grid, 256, 0, s>>>(A->rows_o.get(), A->rowptr_o.get(), A->col_o.get(), A->val_o.get(),
                                            A->ghost.get(), A->ghost_stride, y, q0, q1, A->ro_w, A->d_epoch.get(),
                                            A->halo_err.get());
  SP_LAUNCH();
  return SPMAT_OK;
}

int halo_peer_epoch_end(spmat_s *A, cudaStream_t s) {
  k_epoch_end<<<1, 1, 0, s>>>(A->halo_waits.get(), A->n_waits, A->d_epoch.get());
  SP_LAUNCH();
  return SPMAT_OK;
}

int halo_peer_setup(spmat_s *A) {
  spmat_comm_s *c = A->comm;
  const int P = c->nranks, me = c->rank;
  sf_s *sf = A->halo;
  A->peer = false;
  if (P == 1) return SPMAT_OK;
  const char *env = getenv("SPMAT_HALO");
  int64_t want = (env && !strcmp(env, "nccl")) ? 0 : 1;
  // local feasibility: leaves contiguous per owner; device can reach every peer it talks to
  int64_t fail = 0;
  for (size_t a = 0; a < sf->rnbr.size(); ++a)
    if (sf->leaf_start[a] < 0) fail = 1;
  if (sf->nself) fail = 1;
  {  // agree on feasibility before allocating anything rank-specific
    int64_t vote0[2] = {want ? 0 : 1, fail};
    SP_TRY(c->allreduce_max_i64(vote0, 2));
    if (!vote0[0] && vote0[1])
      note_fallback(c, "the MatMult halo", "ghost leaves not contiguous per owner (or self edges) on some rank");
    if (vote0[0] || vote0[1]) return SPMAT_OK;  // NCCL halo on every rank
  }
  SP_TRY(A->halo_flags.alloc(P));  // [q]: done flag from receiver q
  SP_CUDA(cudaMemset(A->halo_flags.get(), 0, P * sizeof(unsigned long long)));
  // two ghost buffers (epoch parity) so an owner never waits for the previous epoch's reads;
  // zeroed lines carry flag 0, which no epoch (>= 1) matches
  A->ghost_stride = std::max<int64_t>(A->n_ghost, 1);
  SP_TRY(A->ghost.alloc(2 * (size_t)A->ghost_stride));
  SP_CUDA(cudaMemset(A->ghost.get(), 0, A->ghost.n * sizeof(uint4)));
  cudaIpcMemHandle_t hl, hf;
  memset(&hl, 0, sizeof hl);
  memset(&hf, 0, sizeof hf);
  if (want && !fail) {
    if (cudaIpcGetMemHandle(&hl, A->ghost.get()) != cudaSuccess ||
        cudaIpcGetMemHandle(&hf, A->halo_flags.get()) != cudaSuccess) {
      cudaGetLastError();
      fail = 1;
    }
  }
  // agree on the mode before anything else collective
  int64_t vote[2] = {want ? 0 : 1, fail};
  SP_TRY(c->allreduce_max_i64(vote, 2));
  if (!vote[0] && vote[1]) note_fallback(c, "the MatMult halo", "cudaIpcGetMemHandle failed on some rank");
  if (vote[0] || vote[1]) return SPMAT_OK;  // NCCL halo on every rank
  // exchange handles and, per (receiver, sender), the receiver's leaf start for that sender
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::vector<int64_t> mine(17 + P, -1), all((size_t)(17 + P) * P);
  memcpy(mine.data(), &hl, 64);
  memcpy(mine.data() + 8, &hf, 64);
  mine[16] = A->ghost_stride;
  for (size_t a = 0; a < sf->rnbr.size(); ++a) mine[17 + sf->rnbr[a]] = sf->leaf_start[a];
  SP_TRY(c->allgather_i64(mine.data(), 17 + P, all.data()));
  A->peer_ghost.assign(P, nullptr);
  A->peer_flags.assign(P, nullptr);
  int64_t open_fail = 0;
  auto open_rank = [&](int q) {
    if (A->peer_flags[q] || open_fail) return;
    cudaIpcMemHandle_t h1, h2;
    memcpy(&h1, all.data() + (size_t)(17 + P) * q, 64);
    memcpy(&h2, all.data() + (size_t)(17 + P) * q + 8, 64);
    void *p1 = nullptr, *p2 = nullptr;
    if (cudaIpcOpenMemHandle(&p1, h1, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&p2, h2, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      open_fail = 1;
      if (p1) cudaIpcCloseMemHandle(p1);
      return;
    }
    A->peer_ghost[q] = (uint4 *)p1;
    A->peer_flags[q] = (unsigned long long *)p2;
  };
  for (int q : sf->snbr) open_rank(q);
  for (int q : sf->rnbr) open_rank(q);
  int64_t v2[1] = {open_fail};
  SP_TRY(c->allreduce_max_i64(v2, 1));
  if (v2[0]) {
    note_fallback(c, "the MatMult halo", "cudaIpcOpenMemHandle failed on some rank (peers not on one node?)");
    halo_peer_release(A);
    return SPMAT_OK;
  }
  // put descriptors (one per destination) and wait descriptors (one per sender)
  std::vector<HaloPut> puts;
  int total_chunks = 0;
  for (size_t a = 0; a < sf->snbr.size(); ++a) {
    const int q = sf->snbr[a];
    const int64_t lstart = all[(size_t)(17 + P) * q + 17 + me];
    HaloPut p{};
    p.dst = A->peer_ghost[q] + lstart;
    p.dst_stride = all[(size_t)(17 + P) * q + 16];
    p.count = sf->scount[a];
    p.root_start = sf->root_start[a] >= 0 ? sf->root_start[a] : 0;
    p.root_idx = sf->root_start[a] >= 0 ? nullptr : sf->d_root_idx.get() + sf->soff[a];
    p.my_done = A->halo_flags.get() + q;
    p.nchunk = put_chunks(p.count);
    total_chunks += p.nchunk;
    puts.push_back(p);
  }
  std::vector<HaloWait> waits;
  for (size_t a = 0; a < sf->rnbr.size(); ++a) {
    const int q = sf->rnbr[a];
    HaloWait w;
    w.peer_done = A->peer_flags[q] + me;
    waits.push_back(w);
  }
  SP_TRY(A->halo_puts.alloc(puts.size()));
  SP_TRY(A->halo_waits.alloc(waits.size()));
  if (!puts.empty())
    SP_CUDA(cudaMemcpy(A->halo_puts.get(), puts.data(), puts.size() * sizeof(HaloPut), cudaMemcpyHostToDevice));
  if (!waits.empty())
    SP_CUDA(cudaMemcpy(A->halo_waits.get(), waits.data(), waits.size() * sizeof(HaloWait), cudaMemcpyHostToDevice));
  SP_TRY(A->halo_counter.alloc(1));
  SP_CUDA(cudaMemset(A->halo_counter.get(), 0, 4));
  SP_TRY(A->halo_err.alloc(1));
  SP_CUDA(cudaMemset(A->halo_err.get(), 0, 4));
  A->n_puts = (int)puts.size();
  A->n_waits = (int)waits.size();
  A->put_chunks_total = total_chunks;
  SP_TRY(A->d_epoch.alloc(1));
  SP_CUDA(cudaMemset(A->d_epoch.get(), 0, sizeof(unsigned long long)));
  A->peer = true;
  // every rank's flags are zero and every handle is open before the first put
  int64_t sync[1] = {0};
  SP_TRY(c->allreduce_max_i64(sync, 1));
  return SPMAT_OK;
}

void halo_peer_release(spmat_s *A) {
  for (size_t q = 0; q < A->peer_ghost.size(); ++q) {
    if (A->peer_ghost[q]) cudaIpcCloseMemHandle(A->peer_ghost[q]);
    if (A->peer_flags[q]) cudaIpcCloseMemHandle(A->peer_flags[q]);
  }
  A->peer_ghost.clear();
  A->peer_flags.clear();
  A->peer = false;
}

// flagged-line puts described by `puts` (chunks = sum of their nchunk) of epoch *epoch_ctr + 1
int peer_put_launch(const HaloPut *puts, int nputs, int chunks, const double *src,
                    const unsigned long long *epoch_ctr, int *err, cudaStream_t s) {
  if (nputs == 0 || chunks == 0) return SPMAT_OK;
  const int grid = (chunks + kPutWarps - 1) / kPutWarps;
  SP_CUDA(launch_pdl(k_halo_put, grid, 32 * kPutWarps, 0, s, puts, nputs, chunks, src, epoch_ctr, err));
  return SPMAT_OK;
}

int put_chunks_of(int64_t count) { return put_chunks(count); }
// bulk segments: 8 x the values of a flagged-line chunk per warp (16 KB per system fence)
int bulk_chunks_of(int64_t count) {
  return (int)std::max<int64_t>(1, (count + 8 * kPutChunk - 1) / (8 * kPutChunk));
}

// standalone put of the current epoch on stream s
int halo_peer_put(spmat_s *A, const double *x, cudaStream_t s) {
  if (A->n_puts == 0) return SPMAT_OK;
  const int grid = (A->put_chunks_total + kPutWarps - 1) / kPutWarps;
  k_halo_put<<<grid, 32 * kPutWarps, 0, s>>>(A->halo_puts.get(), A->n_puts, A->put_chunks_total, x,
                                            A->d_epoch.get(), A->halo_err.get());
  SP_LAUNCH();
  return SPMAT_OK;
}

// off-diagonal SpMV-add on the epoch's ghost lines; with compute == false it only waits for
// them and releases (halo-only timing).  Always launched: it also ends the MatMult's epoch.
int halo_peer_offdiag(spmat_s *A, double *y, cudaStream_t s, bool compute) {
  const int64_t nro = compute ? A->n_ro : 0;
  const int64_t work = nro > 0 ? (A->ro_w == 1 ? (nro + kRowsU - 1) / kRowsU : nro * A->ro_w) : A->n_ghost;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 4L * A->comm->num_sms));
  SP_CUDA(launch_pdl(k_spmv_offdiag_peer, grid, 256, 0, s, (const int32_t *)A->rows_o.get(),
                     (const int32_t *)A->rowptr_o.get(), (const int32_t *)A->col_o.get(),
                     (const double *)A->val_o.get(), (const uint4 *)A->ghost.get(), A->ghost_stride,
                     A->n_ghost, y, nro, A->ro_w, (const HaloWait *)A->halo_waits.get(), A->n_waits,
                     A->d_epoch.get(), A->halo_counter.get(), A->halo_err.get()));
  return SPMAT_OK;
}

}  // namespace spmat
