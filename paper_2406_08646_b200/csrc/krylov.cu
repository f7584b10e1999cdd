// krylov.cu -- host-synchronisation-free CG on top of MatMult (the paper's CGAsync).
//
// CG "does all its computation and communication on device, and does not need any
// synchronization on host": dot products land in DEVICE scalars (VecDotAsync,
// P:715-724), AXPYs read their coefficient from device memory (VecAXPYAsync),
// scalar arithmetic runs in tiny device kernels, and the loop runs a user-given
// number of iterations without a host-side convergence test.  The paper reduced
// the partial dots with NVSHMEM; here the cross-rank reduction goes through a "scalar board":
// each rank's small device array is IPC-mapped into every other rank (NVLink), a rank stores
// its partial into every board and raises an epoch flag, then sums the P partials of its own
// board in rank order -- the same bit-identical value on every rank, no NCCL kernel, no host.
//
// Local dot products use a fixed decomposition (kDotBlocks CTAs x 256 threads, fixed strides,
// fixed reduction trees), so results are deterministic run to run.
//
// Every epoch (halo, board) and the residual-history index live in device memory, so one CG
// iteration is captured once as a CUDA graph and replayed maxit times (SPMAT_GRAPH=0 turns the
// graph off): the launch cost of ~6 kernels per iteration becomes one graph launch.
#include <algorithm>
#include <cstring>

#include "halo_dev.cuh"
#include "internal.h"

namespace spmat {

constexpr int kDotThreads = 256;

// ------------------------------------------------------------------ scalar board
int board_setup(Comm *c) {
  const int P = c->nranks, me = c->rank;
  c->board_ok = false;
  if (P == 1) return SPMAT_OK;
  const int W = Comm::kBoardWidth;
  SP_TRY(c->board_val.alloc(2 * (size_t)P * W));
  SP_TRY(c->board_flag.alloc(2 * (size_t)P));
  SP_TRY(c->board_err.alloc(1));
  SP_TRY(c->d_board_epoch.alloc(1));
  SP_CUDA(cudaMemset(c->board_val.get(), 0, 2 * P * W * sizeof(double)));
  SP_CUDA(cudaMemset(c->board_flag.get(), 0, 2 * P * sizeof(unsigned long long)));
  SP_CUDA(cudaMemset(c->board_err.get(), 0, sizeof(int)));
  SP_CUDA(cudaMemset(c->d_board_epoch.get(), 0, sizeof(unsigned long long)));
  cudaIpcMemHandle_t hv, hf;
  memset(&hv, 0, sizeof hv);
  memset(&hf, 0, sizeof hf);
  int64_t fail = 0;
  if (getenv("SPMAT_BOARD") && !strcmp(getenv("SPMAT_BOARD"), "nccl")) fail = 1;
  if (!fail && (cudaIpcGetMemHandle(&hv, c->board_val.get()) != cudaSuccess ||
                cudaIpcGetMemHandle(&hf, c->board_flag.get()) != cudaSuccess)) {
    cudaGetLastError();
    fail = 1;
  }
  std::vector<int64_t> mine(16), all(16 * (size_t)P);
  memcpy(mine.data(), &hv, 64);
  memcpy(mine.data() + 8, &hf, 64);
  SP_TRY(c->allgather_i64(mine.data(), 16, all.data()));
  std::vector<double *> pv(P, nullptr);
  std::vector<unsigned long long *> pf(P, nullptr);
  pv[me] = c->board_val.get();
  pf[me] = c->board_flag.get();
  for (int q = 0; q < P && !fail; ++q) {
    if (q == me) continue;
    cudaIpcMemHandle_t h1, h2;
    memcpy(&h1, all.data() + 16 * (size_t)q, 64);
    memcpy(&h2, all.data() + 16 * (size_t)q + 8, 64);
    void *a = nullptr, *b = nullptr;
    if (cudaIpcOpenMemHandle(&a, h1, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&b, h2, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      if (a) cudaIpcCloseMemHandle(a);
      fail = 1;
      break;
    }
    c->board_peer_mem.push_back(a);
    c->board_peer_mem.push_back(b);
    pv[q] = (double *)a;
    pf[q] = (unsigned long long *)b;
  }
  int64_t vote[1] = {fail};
  SP_TRY(c->allreduce_max_i64(vote, 1));
  if (vote[0]) {
    board_release(c);
    return SPMAT_OK;  // reductions fall back to ncclAllReduce
  }
  SP_TRY(c->d_peer_val.alloc(P));
  SP_TRY(c->d_peer_flag.alloc(P));
  SP_CUDA(cudaMemcpy(c->d_peer_val.get(), pv.data(), P * sizeof(double *), cudaMemcpyHostToDevice));
  SP_CUDA(cudaMemcpy(c->d_peer_flag.get(), pf.data(), P * sizeof(void *), cudaMemcpyHostToDevice));
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
  return s;  // valid in thread 0
}

// CTA c owns [c*chunk, (c+1)*chunk); partial[c] = sum of a*b there
__global__ void __launch_bounds__(kDotThreads) k_dot_partial(const double *__restrict__ a,
                                                             const double *__restrict__ b, int64_t n,
                                                             double *__restrict__ partial) {
  __shared__ double red[kDotThreads / 32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kDotThreads) s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// r = b - q; p = r; partial of r.r
__global__ void __launch_bounds__(kDotThreads) k_cg_init(const double *__restrict__ b,
                                                         const double *__restrict__ q, double *__restrict__ r,
                                                         double *__restrict__ p, int64_t n,
                                                         double *__restrict__ partial) {
  __shared__ double red[kDotThreads / 32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kDotThreads) {
    const double ri = __dsub_rn(b[i], q[i]);
    r[i] = ri;
    p[i] = ri;
    s = __dadd_rn(s, __dmul_rn(ri, ri));
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

struct CgScalars {
  double rr, pq, alpha, beta;
  int stopped, iter;  // iter: index of the last residual-history entry written
};

// x = x + alpha p; r = r - alpha q; partial of r.r (products rounded separately, no FMA)
__global__ void __launch_bounds__(kDotThreads) k_cg_update(double *__restrict__ x, double *__restrict__ r,
                                                           const double *__restrict__ p,
                                                           const double *__restrict__ q, int64_t n,
                                                           const CgScalars *__restrict__ sc,
                                                           double *__restrict__ partial) {
  __shared__ double red[kDotThreads / 32];
  const double alpha = sc->alpha;
  const bool go = !sc->stopped;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kDotThreads) {
    double ri = r[i];
    if (go) {
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      ri = __dsub_rn(ri, __dmul_rn(alpha, q[i]));
      r[i] = ri;
    }
    s = __dadd_rn(s, __dmul_rn(ri, ri));
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// p = r + beta p
__global__ void k_cg_pupdate(double *__restrict__ p, const double *__restrict__ r, int64_t n,
                             const CgScalars *__restrict__ sc) {
  if (sc->stopped) return;
  const double beta = sc->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

enum { OP_DOT = 0, OP_CG_INIT = 1, OP_CG_ALPHA = 2, OP_CG_BETA = 3 };

// One CTA: local sum of the partials (fixed order), the cross-rank sum through the scalar
// board (or the value already all-reduced by NCCL when preduced != nullptr), then the scalar
// step of CG.  The board epoch is read from and written back to device memory.
__global__ void __launch_bounds__(kDotThreads) k_finalize(
    const double *__restrict__ partial, int np, int op, CgScalars *sc, double *result,
    double *__restrict__ hist, double *const *peer_val, unsigned long long *const *peer_flag, int P,
    int me, unsigned long long *board_epoch, int *err, const double *preduced) {
  __shared__ double red[kDotThreads / 32];
  __shared__ double total;
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += kDotThreads) s = __dadd_rn(s, partial[i]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) total = s;
  __syncthreads();
  if (preduced) {  // NCCL already summed the local values over ranks
    if (threadIdx.x == 0) total = *preduced;
  } else if (peer_val) {
    const unsigned long long epoch = *board_epoch + 1ull;
    const int par = (int)(epoch & 1);
    const int W = Comm::kBoardWidth;
    if (threadIdx.x < P) {  // my partial into every rank's board, then its flag
      const int q = threadIdx.x;
      peer_val[q][((size_t)par * P + me) * W] = total;
      __threadfence_system();
      st_release_sys(peer_flag[q] + (size_t)par * P + me, epoch);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long *mine = peer_flag[me] + (size_t)par * P;
      bool ok = true;
      for (int q = 0; q < P && ok; ++q) ok = spin_until_geq(mine + q, epoch, err);
      double t = 0.0;
      const double *v = peer_val[me] + (size_t)par * P * W;
      for (int q = 0; q < P; ++q) t = __dadd_rn(t, __ldcg(v + (size_t)q * W));  // rank order
      total = t;
      *board_epoch = epoch;
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const double g = total;
  if (op == OP_DOT) {
    *result = g;
  } else if (op == OP_CG_INIT) {
    sc->rr = g;
    sc->stopped = g == 0.0 ? 1 : 0;
    sc->iter = 0;
    if (hist) hist[0] = g;
  } else if (op == OP_CG_ALPHA) {
    sc->pq = g;
    if (g == 0.0 || sc->rr == 0.0) sc->stopped = 1;
    sc->alpha = sc->stopped ? 0.0 : sc->rr / g;
  } else {  // OP_CG_BETA
    if (!sc->stopped) {
      sc->beta = g / sc->rr;
      sc->rr = g;
    }
    sc->iter += 1;
    if (hist) hist[sc->iter] = sc->rr;
  }
}

// ------------------------------------------------------------------ host side
static int dot_blocks(spmat_s *A) { return A->comm->num_sms * 4; }

static int ensure_ws(spmat_s *A) {
  if (A->cg_partial.n) return SPMAT_OK;
  SP_TRY(A->cg_partial.alloc(dot_blocks(A)));
  SP_TRY(A->cg_scalars.alloc(sizeof(CgScalars) / sizeof(double) + 2));
  SP_TRY(A->cg_reduced.alloc(2));
  return SPMAT_OK;
}

// global sum of partials -> op; cross-rank through the board or ncclAllReduce
static int finalize(spmat_s *A, int op, double *result, double *hist, cudaStream_t s) {
  Comm *c = A->comm;
  const int np = dot_blocks(A);
  CgScalars *sc = (CgScalars *)A->cg_scalars.get();
  if (c->nranks > 1 && !c->board_ok) {
    // local sum first, then NCCL all-reduce of the scalar, then the scalar step
    k_finalize<<<1, kDotThreads, 0, s>>>(A->cg_partial.get(), np, OP_DOT, sc, A->cg_reduced.get(),
                                         nullptr, nullptr, nullptr, 1, 0, nullptr, nullptr, nullptr);
    SP_LAUNCH();
    SP_NCCL(c->api, c->api->AllReduce(A->cg_reduced.get(), A->cg_reduced.get() + 1, 1, ncclFloat64,
                                      ncclSum, c->nccl, s));
    k_finalize<<<1, kDotThreads, 0, s>>>(A->cg_partial.get(), 0, op, sc, result, hist, nullptr, nullptr,
                                         1, 0, nullptr, nullptr, A->cg_reduced.get() + 1);
    SP_LAUNCH();
    return SPMAT_OK;
  }
  const bool board = c->nranks > 1;
  k_finalize<<<1, kDotThreads, 0, s>>>(A->cg_partial.get(), np, op, sc, result, hist,
                                       board ? c->d_peer_val.get() : nullptr,
                                       board ? c->d_peer_flag.get() : nullptr, c->nranks, c->rank,
                                       board ? c->d_board_epoch.get() : nullptr,
                                       board ? c->board_err.get() : nullptr, nullptr);
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
  SP_TRY(spmat_mult_part(A, p, q, 7, s));                            // q = A p
  k_dot_partial<<<nb, kDotThreads, 0, s>>>(p, q, m, A->cg_partial.get());
  SP_LAUNCH();
  SP_TRY(finalize(A, OP_CG_ALPHA, nullptr, nullptr, s));            // alpha = rr / p.q
  k_cg_update<<<nb, kDotThreads, 0, s>>>(x, r, p, q, m, sc, A->cg_partial.get());
  SP_LAUNCH();
  SP_TRY(finalize(A, OP_CG_BETA, nullptr, rr_hist, s));             // beta, rr = r.r
  k_cg_pupdate<<<gv, 256, 0, s>>>(p, r, m, sc);                     // p = r + beta p
  SP_LAUNCH();
  return SPMAT_OK;
}

static bool graph_ok(spmat_s *A) {
  const char *e = getenv("SPMAT_GRAPH");
  if (e && !strcmp(e, "0")) return false;
  if (A->profile) return false;
  if (A->comm->nranks == 1) return true;
  return A->peer && A->comm->board_ok;  // NCCL stays out of captured graphs
}

void cg_graph_release(spmat_s *A) {
  if (A->cg_exec) cudaGraphExecDestroy(A->cg_exec);
  A->cg_exec = nullptr;
  if (A->cg_stream) cudaStreamDestroy(A->cg_stream);
  A->cg_stream = nullptr;
  for (auto &e : A->cg_ev)
    if (e) cudaEventDestroy(e), e = nullptr;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_vec_dot(spmat_t A, const double *a, const double *b, double *result, void *stream) {
  if (!A || !result || (A->m > 0 && (!a || !b))) return fail(SPMAT_ERR_ARG, "spmat_vec_dot: null argument");
  DeviceGuard g(A->comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  SP_TRY(ensure_ws(A));
  k_dot_partial<<<dot_blocks(A), kDotThreads, 0, s>>>(a, b, A->m, A->cg_partial.get());
  SP_LAUNCH();
  return finalize(A, OP_DOT, result, nullptr, s);
}

int spmat_cg(spmat_t A, const double *b, double *x, int maxit, double *rr_hist, void *stream) {
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
  k_cg_init<<<nb, kDotThreads, 0, cs>>>(b, q, r, p, m, A->cg_partial.get());
  SP_LAUNCH();
  SP_TRY(finalize(A, OP_CG_INIT, nullptr, rr_hist, cs));
  if (!use_graph) {
    for (int k = 0; k < maxit; ++k) SP_TRY(cg_iteration(A, x, rr_hist, s));
    return SPMAT_OK;
  }
  if (!A->cg_exec || A->cg_key_x != x || A->cg_key_h != rr_hist) {
    if (A->cg_exec) cudaGraphExecDestroy(A->cg_exec);
    A->cg_exec = nullptr;
    cudaGraph_t graph;
    SP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int st = cg_iteration(A, x, rr_hist, cs);
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (st != SPMAT_OK) return st;
    if (e != cudaSuccess) return fail(SPMAT_ERR_CUDA, "spmat_cg: graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&A->cg_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(SPMAT_ERR_CUDA, "spmat_cg: graph instantiate: %s", cudaGetErrorString(e));
    A->cg_key_x = x;
    A->cg_key_h = rr_hist;
  }
  for (int k = 0; k < maxit; ++k) SP_CUDA(cudaGraphLaunch(A->cg_exec, cs));
  SP_CUDA(cudaEventRecord(A->cg_ev[1], cs));
  SP_CUDA(cudaStreamWaitEvent(s, A->cg_ev[1], 0));
  return SPMAT_OK;
}

}  // extern "C"
