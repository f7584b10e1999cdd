// mult.cu -- MatMult orchestration: halo SF broadcast on the comm stream overlapped with
// the diagonal SpMV, then the off-diagonal SpMV-add.
//
// The halo exchange is issued first on the high-priority comm stream (NCCL), the diagonal
// SpMV runs on the caller's stream meanwhile, and the off-diagonal SpMV-add waits on the
// halo event on the device: the host never blocks (contrast the MPI path of P:492-509).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace spmat {

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
  const bool multi = A->comm->nranks > 1;
  cudaEvent_t *pe;
  if (part == 7) ++A->stat_mults;
  if (multi && (part & 2) && A->halo) {  // bytes this MatMult's halo moves (one direction each)
    if (A->peer) {
      A->stat_nvlink_put += 16 * A->halo->nsend;
    } else {
      A->stat_nccl_sent += 8 * A->halo->nsend;
      A->stat_nccl_recv += 8 * A->halo->nrecv;
    }
  }
  if (multi && A->peer) {  // device-initiated halo over NVLink (halo.cu)
    if (part == 7 && A->kernel_id == 5 && A->bs == 1 && A->m > 0 && !A->env_no_fuse && direct_halo_ok(A))
      return spmv_direct_halo(A, x, y, s);  // small matrix: puts, SpMV and off-diagonal add in one launch
    bool fused = false;
    if (part & 2) {
      // the epoch lives on the device (A->d_epoch): kernels read it, the MatMult's last kernel
      // advances it -- so MatMults can be captured in CUDA graphs.
      // the bulk-copy SpMV's comm warps do the puts; otherwise a standalone put kernel
      // (only k_spmv_tma has comm warps: a comm-warp variant of the 3x3 block kernel capped it
      // at 64 registers and lost more on the stream than the overlap gained -- C5 P=2 1.43 ms
      // either way, P=1 -2 %)
      fused = !A->env_no_fuse && (part & 1) && A->kernel_id == 3 && A->m > 0 && A->n_rowblocks > 0;
      // 3x3 blocks, comm-warp mode: the block SpMV's comm warps do the puts
      const bool bsr_comm = A->bs == 3 && A->ob_ok && A->bsr_fuse_mode == 2 && part == 7 && A->m > 0 && A->n_ro > 0;
      if (!fused && !bsr_comm) {
        pe = A->profile ? prof_pair(A, 2) : nullptr;
        if (pe) SP_CUDA(cudaEventRecord(pe[0], s));
        SP_TRY(halo_peer_put(A, x, s));
        if (pe) SP_CUDA(cudaEventRecord(pe[1], s));
      }
    }
    // full MatMult, no long rows: the off-diagonal SpMV-add runs in the same kernel's tail
    const bool tail = fused && (part & 4) && A->n_ro > 0 && A->n_long == 0 && !A->env_no_tail;
    // 3x3 blocks: the block SpMV adds the off-diagonal blocks of its boundary row blocks
    // (claimed last) from this epoch's ghost lines and ends the epoch (bsr.cu bsr_off_rows)
    const bool ob = A->bs == 3 && A->ob_ok && (part & 6) == 6 && A->n_ro > 0;
    const int ob_mode =
        (ob && (part & 1) && A->m > 0) ? (A->bsr_fuse_mode == 2 && part == 7 ? 2 : (A->bsr_fuse_mode == 1 ? 1 : 0)) : 0;
    const bool ob_fused = ob_mode != 0;
    if (part & 1) {
      pe = A->profile ? prof_pair(A, 0) : nullptr;
      if (pe) SP_CUDA(cudaEventRecord(pe[0], s));
      if (A->bs == 3 && A->m > 0)
        SP_TRY(bsr_spmv(A, x, y, s, ob_mode));
      else
        SP_TRY(spmv_diag(A, x, y, s, fused, tail));
      if (pe) SP_CUDA(cudaEventRecord(pe[1], s));
    }
    if (tail || ob_fused) return SPMAT_OK;
    if (part & 2) {
      pe = (A->profile && (part & 4) && A->n_ro > 0) ? prof_pair(A, 1) : nullptr;
      if (pe) SP_CUDA(cudaEventRecord(pe[0], s));
      if (ob)
        SP_TRY(bsr_offdiag(A, y, nullptr, s));
      else
        SP_TRY(halo_peer_offdiag(A, y, s, (part & 4) != 0));
      if (pe) SP_CUDA(cudaEventRecord(pe[1], s));
    } else if ((part & 4) && A->n_ro > 0) {
      SP_TRY(spmv_offdiag(A, y, s));
    }
    return SPMAT_OK;
  }
  const bool halo = (part & 2) && multi;
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

// Host x and y: copy x in row chunks on one stream, run the SpMV of row chunk k as soon as
// every x row it reads has arrived, and copy y chunk k back on a third stream -- PCIe is full
// duplex, so the x upload, the SpMV and the y download overlap chunk by chunk.  Several ranks
// (NVLink halo): the chunks holding the x rows the puts read go first, a standalone put kernel
// on a high-priority stream sends them once they have landed, each row chunk's off-diagonal
// rows are added right after its diagonal SpMV (reading the flagged ghost lines), and a last
// one-thread kernel ends the epoch.
static bool pipeline_ok(spmat_s *A) {
  const char *e = getenv("SPMAT_HOST_PIPELINE");
  if (e && !strcmp(e, "0")) return false;
  if (!(A->kernel_id == 3 && A->n_long == 0 && A->m == A->n && A->m >= (1 << 20) && A->n_rowblocks >= 64))
    return false;
  return A->comm->nranks == 1 || A->peer;
}

// Calls alternate between two staging slots (x and y copies on the device), so with
// asynchronous calls call k+1's upload overlaps call k's download -- PCIe is full duplex.  Slot
// reuse is ordered by events: the upload into a slot waits for the SpMV that read it two calls
// ago, the SpMV writing a slot's y for that slot's last download; the put of the next call
// (several ranks) for this call's epoch end.
//   mode 0 (spmat_mult): the call returns after y is on the host.
//   mode 1 (spmat_mult_async): enqueue only; the caller's stream waits for this call's
//     download, so its completion means y is on the host (the next call's SpMV, on that stream,
//     then also waits for it).
//   mode 2 (spmat_mult_pipelined): enqueue only; the SpMV runs on an internal stream and the
//     caller's stream waits for this call's download only at the NEXT call on this matrix (or
//     spmat_mult_flush) -- so call k+1's SpMV overlaps call k's download too.
enum { MULT_SYNC = 0, MULT_ASYNC = 1, MULT_PIPELINED = 2 };

// the caller's stream waits for the download a pipelined call left pending
static int flush_pending(spmat_s *A, cudaStream_t s) {
  if (A->pipe_pending) {
    SP_CUDA(cudaStreamWaitEvent(s, A->pipe_ev_pending, 0));
    A->pipe_pending = false;
  }
  return SPMAT_OK;
}

static int mult_host_pipelined(spmat_s *A, const double *x, double *y, cudaStream_t s, int mode) {
  // asynchronous calls overlap across calls, so few chunks (less per-copy and per-kernel
  // overhead); synchronous calls need the chunks to overlap within the call
  SP_TRY(spmv_pipe_prepare(A, mode != MULT_SYNC ? A->env_pipe_chunks_async : A->env_pipe_chunks));
  const int nc = A->pipe_chunks;
  const bool multi = A->comm->nranks > 1;
  ++A->stat_mults;
  if (multi) A->stat_nvlink_put += 16 * A->halo->nsend;
  if (!A->pipe_in) {
    int lo = 0, hi = 0;
    SP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SP_CUDA(cudaStreamCreateWithFlags(&A->pipe_in, cudaStreamNonBlocking));
    SP_CUDA(cudaStreamCreateWithFlags(&A->pipe_out, cudaStreamNonBlocking));
    SP_CUDA(cudaStreamCreateWithFlags(&A->pipe_comp, cudaStreamNonBlocking));
    SP_CUDA(cudaStreamCreateWithPriority(&A->pipe_comm, cudaStreamNonBlocking, hi));
  }
  // [0,nc) x chunk in, [nc,2nc) y chunk done, 2nc start, 2nc+1 end, 2nc+2 puts done,
  // 2nc+3+slot: slot's x free (its SpMV done), 2nc+5+slot: slot's y downloaded, 2nc+7 epoch end,
  // 2nc+8 this call's compute done
  while (A->pipe_ev.size() < (size_t)(2 * nc + 9)) {
    cudaEvent_t e;
    SP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    A->pipe_ev.push_back(e);
  }
  if (A->xstage.n < 2 * (size_t)A->n) SP_TRY(A->xstage.alloc(2 * (size_t)A->n));
  if (A->ystage.n < 2 * (size_t)A->m) SP_TRY(A->ystage.alloc(2 * (size_t)A->m));
  const int slot = A->pipe_slot;
  A->pipe_slot ^= 1;
  double *dx = A->xstage.get() + (size_t)slot * A->n, *dy = A->ystage.get() + (size_t)slot * A->m;
  cudaEvent_t *ev = A->pipe_ev.data();
  cudaEvent_t ev_xfree = ev[2 * nc + 3 + slot], ev_yfree = ev[2 * nc + 5 + slot], ev_epoch = ev[2 * nc + 7];
  // the compute stream: the caller's, or (pipelined) an internal one that starts after the
  // caller's work so far -- recorded BEFORE the caller's stream waits for the previous download
  cudaStream_t cs = s;
  if (mode == MULT_PIPELINED) {
    cs = A->pipe_comp;
    SP_CUDA(cudaEventRecord(ev[2 * nc], s));
    SP_CUDA(cudaStreamWaitEvent(cs, ev[2 * nc], 0));
    SP_TRY(flush_pending(A, s));
  } else if (mode == MULT_SYNC) {  // earlier work on s (e.g. a device-pointer MatMult using the same buffers)
    SP_CUDA(cudaEventRecord(ev[2 * nc], s));
    SP_CUDA(cudaStreamWaitEvent(A->pipe_in, ev[2 * nc], 0));
    SP_CUDA(cudaStreamWaitEvent(A->pipe_out, ev[2 * nc], 0));
  }
  SP_CUDA(cudaStreamWaitEvent(A->pipe_in, ev_xfree, 0));  // the SpMV of two calls ago read this slot
  SP_CUDA(cudaStreamWaitEvent(cs, ev_yfree, 0));          // this slot's y of two calls ago is downloaded
  std::vector<int> order;
  for (int pass = 0; pass < 2; ++pass)  // chunks the puts read first
    for (int k = 0; k < nc; ++k)
      if ((A->pipe_put_chunk[k] != 0) == (pass == 0)) order.push_back(k);
  for (int k : order) {
    const int64_t r0 = A->pipe_row[k], r1 = A->pipe_row[k + 1];
    SP_CUDA(cudaMemcpyAsync(dx + r0, x + r0, (r1 - r0) * 8, cudaMemcpyHostToDevice, A->pipe_in));
    SP_CUDA(cudaEventRecord(ev[k], A->pipe_in));
  }
  if (multi) {
    if (mode == MULT_SYNC) SP_CUDA(cudaStreamWaitEvent(A->pipe_comm, ev[2 * nc], 0));
    SP_CUDA(cudaStreamWaitEvent(A->pipe_comm, ev_epoch, 0));  // the previous call's epoch is over
    for (int k = 0; k < nc; ++k)
      if (A->pipe_put_chunk[k]) SP_CUDA(cudaStreamWaitEvent(A->pipe_comm, ev[k], 0));
    SP_TRY(halo_peer_put(A, dx, A->pipe_comm));
    SP_CUDA(cudaEventRecord(ev[2 * nc + 2], A->pipe_comm));
  }
  bool put_waited = false;
  for (int k = 0; k < nc; ++k) {
    for (int j = 0; j < nc; ++j)  // every x chunk holding a column this row chunk reads
      if (A->pipe_row[j] <= A->pipe_xneed[k] && A->pipe_row[j + 1] > A->pipe_xmin[k])
        SP_CUDA(cudaStreamWaitEvent(cs, ev[j], 0));
    SP_TRY(spmv_diag_chunk(A, dx, dy, k, cs));
    if (multi && A->pipe_q[k + 1] > A->pipe_q[k]) {
      // my puts are out before this stream spins on the neighbours' lines: no rank can hold
      // every SM waiting while its own puts are still queued
      if (!put_waited) SP_CUDA(cudaStreamWaitEvent(cs, ev[2 * nc + 2], 0));
      put_waited = true;
      SP_TRY(halo_peer_offdiag_range(A, dy, A->pipe_q[k], A->pipe_q[k + 1], cs));
    }
    SP_CUDA(cudaEventRecord(ev[nc + k], cs));
    SP_CUDA(cudaStreamWaitEvent(A->pipe_out, ev[nc + k], 0));
    const int64_t r0 = A->pipe_row[k], r1 = A->pipe_row[k + 1];
    SP_CUDA(cudaMemcpyAsync(y + r0, dy + r0, (r1 - r0) * 8, cudaMemcpyDeviceToHost, A->pipe_out));
  }
  if (multi) {  // the put read this epoch's number: it must be done before the epoch advances
    if (!put_waited) SP_CUDA(cudaStreamWaitEvent(cs, ev[2 * nc + 2], 0));
    SP_TRY(halo_peer_epoch_end(A, cs));
    SP_CUDA(cudaEventRecord(ev_epoch, cs));
  }
  SP_CUDA(cudaEventRecord(ev_xfree, cs));
  SP_CUDA(cudaEventRecord(ev_yfree, A->pipe_out));
  if (mode == MULT_PIPELINED) {
    // the caller's later work (e.g. set_values on this matrix) must follow this call's SpMV;
    // its wait for the download is deferred to the next call / spmat_mult_flush
    SP_CUDA(cudaEventRecord(ev[2 * nc + 8], cs));
    SP_CUDA(cudaStreamWaitEvent(s, ev[2 * nc + 8], 0));
    A->pipe_ev_pending = ev_yfree;
    A->pipe_pending = true;
    return SPMAT_OK;
  }
  SP_CUDA(cudaStreamWaitEvent(s, ev_yfree, 0));
  if (mode == MULT_SYNC) SP_CUDA(cudaStreamSynchronize(s));
  return SPMAT_OK;
}

// spmat_mult / spmat_mult_async body: device pointers enqueue only; host pointers are staged
// (pipelined when large enough), and with async == false the call returns after y is written
static int mult_entry(spmat_t A, const double *x, double *y, void *stream, int mode, const char *who) {
  if (!A) return fail(SPMAT_ERR_ARG, "%s: null matrix", who);
  if ((A->n > 0 && !x) || (A->m > 0 && !y)) return fail(SPMAT_ERR_ARG, "%s: null x or y", who);
  if (x && (const void *)x == (const void *)y) return fail(SPMAT_ERR_ARG, "%s: x and y alias", who);
  if (!A->values_set && A->nnz_d + A->nnz_o > 0)
    return fail(SPMAT_ERR_STATE, "%s before spmat_set_values_coo", who);
  DeviceGuard g(A->comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  const bool hx = A->n > 0 && !is_device_ptr(x);
  const bool hy = A->m > 0 && !is_device_ptr(y);
  const bool pipe = hx && hy && pipeline_ok(A);
  if (!(pipe && mode == MULT_PIPELINED)) SP_TRY(flush_pending(A, s));
  if (!hx && !hy) return mult_impl(A, x, y, 7, s);
  if (pipe) return mult_host_pipelined(A, x, y, s, mode);
  const bool async = mode != MULT_SYNC;
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
  if (!async) SP_CUDA(cudaStreamSynchronize(s));
  return SPMAT_OK;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_mult(spmat_t A, const double *x, double *y, void *stream) {
  SP_NVTX("spmat_mult");
  return mult_entry(A, x, y, stream, MULT_SYNC, "spmat_mult");
}

int spmat_mult_async(spmat_t A, const double *x, double *y, void *stream) {
  SP_NVTX("spmat_mult_async");
  return mult_entry(A, x, y, stream, MULT_ASYNC, "spmat_mult_async");
}

int spmat_mult_pipelined(spmat_t A, const double *x, double *y, void *stream) {
  SP_NVTX("spmat_mult_pipelined");
  return mult_entry(A, x, y, stream, MULT_PIPELINED, "spmat_mult_pipelined");
}

int spmat_mult_flush(spmat_t A, void *stream) {
  if (!A) return fail(SPMAT_ERR_ARG, "spmat_mult_flush: null matrix");
  DeviceGuard g(A->comm->device);
  return flush_pending(A, (cudaStream_t)stream);
}

int spmat_mult_part(spmat_t A, const double *x, double *y, int part, void *stream) {
  SP_NVTX("spmat_mult_part");
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
