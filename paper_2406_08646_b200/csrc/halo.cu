// halo.cu -- device-initiated halo exchange for MatMult over NVLink peer memory.
//
// The paper's experimental NVSHMEM PetscSF removes the host from the halo
// path: "symmetric send/recv buffers", a kernel "calls nvshmem_putmem_nbi", synchronisation
// on the device.  Its motivation: an MPI/NCCL exchange needs host ordering or,
// as measured here on B200, an NCCL p2p kernel whose handshakes crawl while the SpMV keeps
// HBM saturated (the 17 us transfer then completes only after the SpMV).
//
// B200 design: at create time every rank exports its ghost vector (lvec) and a small flag
// array through CUDA IPC; each owner opens the lvec of the ranks that need its rows and
// learns where in their lvec its values go (the halo SF leaves are contiguous per owner).
// Per MatMult (epoch e):
//   k_halo_put (high-priority comm stream, a few CTAs per destination): wait until the
//     destination has finished reading epoch e-1 (done flag), store the owned x entries
//     straight into the destination's lvec over NVLink, fence, then bump the destination's
//     ready counter (release, system scope);
//   k_spmv_offdiag_peer (caller's stream, after the diagonal SpMV): wait until every
//     sender's ready counter shows epoch e (acquire), add A_o lvec into y, and the last CTA
//     tells each sender that lvec may be overwritten (done = e).
// The transfer (0.5-1 MB) overlaps the diagonal SpMV completely; no NCCL kernel, no host
// synchronisation.  Spins are bounded (a stuck peer sets an error word instead of hanging).
#include <algorithm>
#include <cstring>

#include "internal.h"

namespace spmat {

constexpr int kPutThreads = 512;
constexpr int64_t kPutChunk = 16384;  // values per put CTA
constexpr long long kSpinLimit = 20LL * 2000 * 1000 * 1000;  // ~20 s of SM clocks

static inline int put_chunks(int64_t count) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(16, (count + kPutChunk - 1) / kPutChunk));
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// returns false on timeout (and records it)
__device__ bool spin_until_geq(const unsigned long long *flag, unsigned long long target, int *err) {
  const long long t0 = clock64();
  while (ld_acquire_sys(flag) < target) {
    if (clock64() - t0 > kSpinLimit) {
      atomicExch(err, 1);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// one CTA per (destination, chunk)
__global__ void __launch_bounds__(kPutThreads) k_halo_put(const HaloPut *__restrict__ puts, int nputs,
                                                          const double *__restrict__ x,
                                                          unsigned long long epoch, int *err) {
  // locate this CTA's destination and chunk
  int c = blockIdx.x, d = 0;
  while (d < nputs && c >= puts[d].nchunk) c -= puts[d++].nchunk;
  if (d >= nputs) return;
  const HaloPut p = puts[d];
  __shared__ int ok;
  if (threadIdx.x == 0) ok = epoch <= 1 ? 1 : spin_until_geq(p.my_done, epoch - 1, err);
  __syncthreads();
  if (!ok) return;
  const int64_t per = (p.count + p.nchunk - 1) / p.nchunk;
  const int64_t lo = c * per, hi = min(p.count, lo + per);
  if (p.root_idx) {
    for (int64_t t = lo + threadIdx.x; t < hi; t += kPutThreads) p.dst[t] = __ldg(x + p.root_idx[t]);
  } else {
    const double *src = x + p.root_start;
    for (int64_t t = lo + threadIdx.x; t < hi; t += kPutThreads) p.dst[t] = __ldg(src + t);
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) red_release_sys_add(p.peer_ready, 1ull);
}

// y[rows[q]] += A_o lvec, after the senders' epoch-e data has landed; the last CTA releases lvec
__global__ void __launch_bounds__(256) k_spmv_offdiag_peer(
    const int32_t *__restrict__ rows, const int32_t *__restrict__ rowptr,
    const int32_t *__restrict__ col, const double *__restrict__ val, const double *lvec,
    double *__restrict__ y, int64_t nro, const HaloWait *__restrict__ waits, int nwaits,
    unsigned long long epoch, unsigned int *counter, int *err, int signal) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    int good = 1;
    for (int w = 0; w < nwaits && good; ++w)
      good = spin_until_geq(waits[w].my_ready, epoch * (unsigned long long)waits[w].nchunk, err);
    ok = good;
  }
  __syncthreads();
  if (ok) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nro;
         q += (int64_t)gridDim.x * blockDim.x) {
      double s = 0.0;
      for (int e = rowptr[q]; e < rowptr[q + 1]; ++e) s = __dadd_rn(s, __dmul_rn(val[e], __ldcg(lvec + col[e])));
      const int r = rows[q];
      y[r] = __dadd_rn(y[r], s);
    }
  }
  if (!signal) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      atomicExch(counter, 0u);
      for (int w = 0; w < nwaits; ++w) st_release_sys(waits[w].peer_done, epoch);
    }
  }
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
  SP_TRY(A->halo_flags.alloc(2 * (size_t)P));  // [0,P): ready from sender q; [P,2P): done from receiver q
  SP_CUDA(cudaMemset(A->halo_flags.get(), 0, 2 * P * sizeof(unsigned long long)));
  if (A->lvec.n == 0) SP_TRY(A->lvec.alloc(1));
  cudaIpcMemHandle_t hl, hf;
  memset(&hl, 0, sizeof hl);
  memset(&hf, 0, sizeof hf);
  if (want && !fail) {
    if (cudaIpcGetMemHandle(&hl, A->lvec.get()) != cudaSuccess ||
        cudaIpcGetMemHandle(&hf, A->halo_flags.get()) != cudaSuccess) {
      cudaGetLastError();
      fail = 1;
    }
  }
  // agree on the mode before anything else collective
  int64_t vote[2] = {want ? 0 : 1, fail};
  SP_TRY(c->allreduce_max_i64(vote, 2));
  if (vote[0] || vote[1]) return SPMAT_OK;  // NCCL halo on every rank
  // exchange handles and, per (receiver, sender), the receiver's leaf start for that sender
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::vector<int64_t> mine(16 + P, -1), all((size_t)(16 + P) * P);
  memcpy(mine.data(), &hl, 64);
  memcpy(mine.data() + 8, &hf, 64);
  for (size_t a = 0; a < sf->rnbr.size(); ++a) mine[16 + sf->rnbr[a]] = sf->leaf_start[a];
  SP_TRY(c->allgather_i64(mine.data(), 16 + P, all.data()));
  A->peer_lvec.assign(P, nullptr);
  A->peer_flags.assign(P, nullptr);
  int64_t open_fail = 0;
  auto open_rank = [&](int q) {
    if (A->peer_flags[q] || open_fail) return;
    cudaIpcMemHandle_t h1, h2;
    memcpy(&h1, all.data() + (size_t)(16 + P) * q, 64);
    memcpy(&h2, all.data() + (size_t)(16 + P) * q + 8, 64);
    void *p1 = nullptr, *p2 = nullptr;
    if (cudaIpcOpenMemHandle(&p1, h1, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&p2, h2, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      open_fail = 1;
      if (p1) cudaIpcCloseMemHandle(p1);
      return;
    }
    A->peer_lvec[q] = (double *)p1;
    A->peer_flags[q] = (unsigned long long *)p2;
  };
  for (int q : sf->snbr) open_rank(q);
  for (int q : sf->rnbr) open_rank(q);
  int64_t v2[1] = {open_fail};
  SP_TRY(c->allreduce_max_i64(v2, 1));
  if (v2[0]) {
    halo_peer_release(A);
    return SPMAT_OK;
  }
  // put descriptors (one per destination) and wait descriptors (one per sender)
  std::vector<HaloPut> puts;
  int total_chunks = 0;
  for (size_t a = 0; a < sf->snbr.size(); ++a) {
    const int q = sf->snbr[a];
    const int64_t lstart = all[(size_t)(16 + P) * q + 16 + me];
    HaloPut p;
    p.dst = A->peer_lvec[q] + lstart;
    p.count = sf->scount[a];
    p.root_start = sf->root_start[a] >= 0 ? sf->root_start[a] : 0;
    p.root_idx = sf->root_start[a] >= 0 ? nullptr : sf->d_root_idx.get() + sf->soff[a];
    p.peer_ready = A->peer_flags[q] + me;
    p.my_done = A->halo_flags.get() + P + q;
    p.nchunk = put_chunks(p.count);
    total_chunks += p.nchunk;
    puts.push_back(p);
  }
  std::vector<HaloWait> waits;
  for (size_t a = 0; a < sf->rnbr.size(); ++a) {
    const int q = sf->rnbr[a];
    HaloWait w;
    w.my_ready = A->halo_flags.get() + q;
    w.nchunk = put_chunks(sf->rcount[a]);
    w.peer_done = A->peer_flags[q] + P + me;
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
  A->epoch = 0;
  A->peer = true;
  SP_CUDA(cudaEventCreateWithFlags(&A->ev_put_begin, cudaEventDisableTiming));
  SP_CUDA(cudaEventCreateWithFlags(&A->ev_put_done, cudaEventDisableTiming));
  // every rank's flags are zero and every handle is open before the first put
  int64_t sync[1] = {0};
  SP_TRY(c->allreduce_max_i64(sync, 1));
  return SPMAT_OK;
}

void halo_peer_release(spmat_s *A) {
  for (size_t q = 0; q < A->peer_lvec.size(); ++q) {
    if (A->peer_lvec[q]) cudaIpcCloseMemHandle(A->peer_lvec[q]);
    if (A->peer_flags[q]) cudaIpcCloseMemHandle(A->peer_flags[q]);
  }
  A->peer_lvec.clear();
  A->peer_flags.clear();
  if (A->ev_put_begin) cudaEventDestroy(A->ev_put_begin);
  if (A->ev_put_done) cudaEventDestroy(A->ev_put_done);
  A->ev_put_begin = A->ev_put_done = nullptr;
  A->peer = false;
}

// enqueue the puts of epoch e on the comm stream (after the caller's pending work on s)
int halo_peer_begin(spmat_s *A, const double *x, cudaStream_t s, cudaEvent_t *prof) {
  spmat_comm_s *c = A->comm;
  ++A->epoch;
  if (A->n_puts == 0) return SPMAT_OK;
  SP_CUDA(cudaEventRecord(A->ev_put_begin, s));
  SP_CUDA(cudaStreamWaitEvent(c->comm_stream, A->ev_put_begin, 0));
  if (prof) SP_CUDA(cudaEventRecord(prof[0], c->comm_stream));
  k_halo_put<<<A->put_chunks_total, kPutThreads, 0, c->comm_stream>>>(
      A->halo_puts.get(), A->n_puts, x, (unsigned long long)A->epoch, A->halo_err.get());
  SP_LAUNCH();
  if (prof) SP_CUDA(cudaEventRecord(prof[1], c->comm_stream));
  SP_CUDA(cudaEventRecord(A->ev_put_done, c->comm_stream));
  return SPMAT_OK;
}

// the caller may reuse x once the puts have read it
int halo_peer_end(spmat_s *A, cudaStream_t s) {
  if (A->n_puts == 0) return SPMAT_OK;
  SP_CUDA(cudaStreamWaitEvent(s, A->ev_put_done, 0));
  return SPMAT_OK;
}

// off-diagonal SpMV-add gated on the epoch's halo; with compute == false it only waits and
// releases (halo-only timing)
int halo_peer_offdiag(spmat_s *A, double *y, cudaStream_t s, bool compute) {
  if (A->n_waits == 0 && (!compute || A->n_ro == 0)) return SPMAT_OK;
  const int64_t nro = compute ? A->n_ro : 0;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nro + 255) / 256, 4L * A->comm->num_sms));
  k_spmv_offdiag_peer<<<grid, 256, 0, s>>>(A->rows_o.get(), A->rowptr_o.get(), A->col_o.get(),
                                           A->val_o.get(), A->lvec.get(), y, nro,
                                           A->halo_waits.get(), A->n_waits,
                                           (unsigned long long)A->epoch, A->halo_counter.get(),
                                           A->halo_err.get(), 1);
  SP_LAUNCH();
  return SPMAT_OK;
}

}  // namespace spmat
