// internal.h -- shared internals of libspmat (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "nccl.h"
#include "spmat.h"

namespace spmat {

// ------------------------------------------------------------------ errors
void set_error(const char *fmt, ...);
int fail(int status, const char *fmt, ...);

#define SP_CUDA(expr)                                                                    \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return ::spmat::fail(_e == cudaErrorMemoryAllocation ? SPMAT_ERR_OOM : SPMAT_ERR_CUDA, \
                           "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
  } while (0)

#define SP_TRY(expr)                    \
  do {                                  \
    int _s = (expr);                    \
    if (_s != SPMAT_OK) return _s;      \
  } while (0)

#define SP_LAUNCH()  SP_CUDA(cudaGetLastError())

// ------------------------------------------------------------------ NCCL (dlopen'ed)
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *);  // may be null
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
  const char *(*GetErrorString)(ncclResult_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t);
};
int nccl_api(NcclApi **out);

#define SP_NCCL(api, expr)                                                               \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess)                                                               \
      return ::spmat::fail(SPMAT_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr,    \
                           (api)->GetErrorString(_r));                                   \
  } while (0)

// ------------------------------------------------------------------ NVTX
// Host-side ranges around every ABI entry point (header-only NVTX v3: a no-op unless a tool
// such as Nsight Systems is attached), so a trace shows create / set_values / mult / SF calls.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define SP_NVTX(name) ::spmat::NvtxRange _nvtx_range_(name)

// ------------------------------------------------------------------ device guard
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------------ device buffers
template <typename T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  int alloc(size_t count) {
    release();
    n = count;
    if (count == 0) return SPMAT_OK;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(SPMAT_ERR_OOM, "cudaMalloc(%zu bytes): %s", count * sizeof(T),
                  cudaGetErrorString(e));
    }
    return SPMAT_OK;
  }
  T *get() const { return p; }
};

// Launch with programmatic stream serialization (PDL, ptx.cuh) unless SPMAT_PDL=0: the
// kernel's CTAs may start while the previous kernel of the stream drains.
bool pdl_on();
int coop_mode();  // SPMAT_COOP: 0 plain launch, 1 cooperative (default), 2 cooperative + PDL
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
// Cooperative launch: every CTA of the grid is resident at once, or the launch fails (instead of
// CTAs that spin on peer data waiting for CTAs that other work keeps off the SMs).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = coop_mode() == 2 && pdl_on() ? 2 : 1;
  if (coop_mode() == 0) {  // SPMAT_COOP=0: plain (PDL) launch, no co-residency guarantee
    cfg.attrs = at + 1;
    cfg.numAttrs = pdl_on() ? 1 : 0;
  }
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// is `p` a device (or managed) pointer?
bool is_device_ptr(const void *p);

// ------------------------------------------------------------------ communicator
struct Comm {
  int nranks = 1, rank = 0, device = 0;
  ncclComm_t nccl = nullptr;
  NcclApi *api = nullptr;
  cudaStream_t comm_stream = nullptr;   // high priority, non-blocking
  cudaStream_t setup_stream = nullptr;  // used by collective setup calls
  int num_sms = 148;
  int nccl_max_ctas = 0;                // ncclConfig_t.maxCTAs used at init (0: NCCL's default)

  // Collectives used by setup (host-synchronising).  All operate on host arrays.
  int allgather_i64(const int64_t *send, int64_t count, int64_t *recv_host);  // recv: count*P
  int allreduce_max_i64(int64_t *v, int64_t count);
  // Agree on a status found locally before the next collective: every rank returns an error
  // (its own, or "failed on another rank") if any rank failed, instead of the others
  // blocking in NCCL.  Collective, host-synchronising.
  int agree(int local_status, const char *what);
  // Exchange variable-size int64 payloads (host-side counts known on both sides):
  // send[d] of scount[d] elements to d, recv from s of rcount[s] elements; device buffers.
  int exchange_dev(const void *d_send, const int64_t *soff, const int64_t *scount,
                   void *d_recv, const int64_t *roff, const int64_t *rcount,
                   size_t elem_bytes, cudaStream_t stream);

  // Scalar board (krylov.cu): every rank's small device array, mapped into every other rank
  // through CUDA IPC, for device-side all-reductions of a scalar over NVLink.
  // line[parity][src]: src's partial as a flagged 16-byte line (halo_dev.cuh).
  bool board_ok = false;
  DevBuf<uint4> board_line;
  std::vector<void *> board_peer_mem;               // opened IPC mappings (to close)
  DevBuf<uint4 *> d_peer_line;                      // per rank: its line array (self included)
  DevBuf<int> board_err;
  DevBuf<unsigned long long> d_board_epoch;  // completed board reductions (device, graph-safe)
};
int board_setup(Comm *c);      // collective; leaves board_ok false when IPC is unavailable
// say plainly (stderr, rank 0) that a transport fell back from NVLink peer memory to NCCL
void note_fallback(const Comm *c, const char *what, const char *why);
void board_release(Comm *c);

}  // namespace spmat

struct spmat_comm_s : spmat::Comm {};

// ------------------------------------------------------------------ device-initiated halo
struct HaloPut {                       // one destination rank of my owned x entries
  uint4 *dst;                          // peer ghost lines + first leaf for me (IPC mapping)
  int64_t dst_stride;                  // peer ghost buffer stride in lines (double-buffered by epoch)
  int64_t count, root_start;           // contiguous x slice, or...
  const int64_t *root_idx;             // ...gather indices (device), nullptr if contiguous
  unsigned long long *my_done;         // destination -> me: "ghost buffer free" epoch (local)
  int nchunk, pad;
  // bulk protocol (large star-forest segments): plain doubles in the first half of the
  // destination's line region, then per chunk a fence and a release of cflag[chunk] = epoch
  unsigned long long *cflag;           // nullptr: flagged lines (the default)
};
struct SfSeg {                         // consumer view of one producer's segment (star forest)
  int64_t start, count;                // range in the staging buffer's order
  const unsigned long long *cflag;     // bulk chunk flags (local), nullptr: flagged lines
  int64_t per;                         // values per bulk chunk
};
struct HaloWait {                      // one sender of my ghost entries
  unsigned long long *peer_done;       // sender's "ghost buffer free" flag for me (IPC mapping)
};

// ------------------------------------------------------------------ star forest
struct sf_s {
  spmat_comm_s *comm = nullptr;
  int64_t nroots = 0, nleaves = 0;
  // receive side (leaves), neighbours ascending, excluding self
  std::vector<int> rnbr;
  std::vector<int64_t> rcount, roff;     // per neighbour, offsets into recv order
  std::vector<int64_t> leaf_start;       // leaf index of first leaf if contiguous, else -1
  spmat::DevBuf<int64_t> d_leaf_idx;     // leaf indices in recv order (all neighbours)
  int64_t nrecv = 0;
  // send side (roots), requesters ascending, excluding self
  std::vector<int> snbr;
  std::vector<int64_t> scount, soff;
  std::vector<int64_t> root_start;       // first root offset if contiguous, else -1
  spmat::DevBuf<int64_t> d_root_idx;     // root offsets in send order
  int64_t nsend = 0;
  // self edges (leaf and root on this rank)
  spmat::DevBuf<int64_t> d_self_leaf, d_self_root;
  int64_t nself = 0;
  // buffers
  spmat::DevBuf<double> d_sendbuf, d_recvbuf;
  bool need_pack = false, need_unpack_any = false;
  // host copies for export
  std::vector<int64_t> h_leaf_idx, h_root_idx;
  // split-phase state
  cudaEvent_t ev_begin = nullptr, ev_done = nullptr;
  cudaEvent_t ev_take = nullptr;         // NVLink transport: the last consuming kernel (epoch advanced)
  bool take_captured = false;            // ev_take was recorded inside a stream capture
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;  // profiling (comm stream)
  bool pending = false;
  bool peer_deferred = false;            // the NVLink transport is set up on first use (sf_ensure_peer)
  const double *p_root = nullptr;
  double *p_leaf = nullptr;
  int p_op = -1;
  int p_kind = 0;                        // pending op: 1 = bcast, 2 = reduce
  // reduce (leaf -> root) plan: touched roots, their contributions in (source rank, leaf)
  // order; code >= 0 -> received value redbuf[code], code < 0 -> own leaf self_leaf[-code-1]
  int64_t n_touched = 0;
  spmat::DevBuf<int64_t> d_red_roots, d_red_ptr, d_red_code;
  spmat::DevBuf<double> d_redbuf;        // received leaf values, requester-major (soff layout)
  // NVLink transport (sf_peer_setup, the default with several ranks): values travel as
  // flagged 16-byte lines (halo_dev.cuh) stored by the producer straight into the consumer's
  // IPC-mapped staging buffer -- bcast: leaf side [2][nrecv] in recv order; reduce: root side
  // [2][nsend] in requester-major order; two buffers by epoch parity, done flags back.
  bool peer = false;
  spmat::DevBuf<uint4> bline, rline;
  int64_t bstride = 0, rstride = 0;
  spmat::DevBuf<unsigned long long> pflags;  // [q] bcast done from receiver q, [P+q] reduce done from owner q,
                                             // then the bulk segments' chunk flags
  spmat::DevBuf<unsigned long long> d_ep;    // [0] completed bcasts, [1] completed reduces
  std::vector<void *> peer_mem;              // opened IPC mappings
  spmat::DevBuf<HaloPut> bputs, rputs;       // bcast: my roots -> leaf owners; reduce: my leaves -> root owners
  int nbputs = 0, nrputs = 0, bchunks = 0, rchunks = 0;
  spmat::DevBuf<HaloWait> bwaits, rwaits;    // producers to release after consuming
  spmat::DevBuf<SfSeg> bsegs, rsegs;         // consumer segment tables (bulk or flagged lines)
  int nbwaits = 0, nrwaits = 0;
  spmat::DevBuf<unsigned int> pcounter;      // last-CTA detection of the consuming kernels
  spmat::DevBuf<int> perr;                   // bounded-spin timeouts
};

namespace spmat {
// build an SF from host leaf arrays (ilocal may be null); collective
int sf_build(spmat_comm_s *comm, int64_t nroots, int64_t nleaves, const int64_t *h_ilocal,
             const int32_t *h_rank, const int64_t *h_offset, sf_s **out, bool defer_peer = false);
int sf_begin(sf_s *sf, const double *root, double *leaf, int op, cudaStream_t stream,
             cudaEvent_t *prof /* optional pair recorded on the comm stream */);
int sf_end(sf_s *sf, const double *root, double *leaf, int op, cudaStream_t stream);
void sf_free(sf_s *sf);
int sf_reduce_begin_impl(sf_s *sf, const double *leaf, double *root, int op, cudaStream_t stream);
int sf_reduce_end_impl(sf_s *sf, const double *leaf, double *root, int op, cudaStream_t stream);
}  // namespace spmat

// kernel-parameter bundles of the bulk-copy SpMV
struct SpmvHalo {                      // fused NVLink halo puts (comm warps)
  const HaloPut *puts;
  int nputs, put_chunks;
  // device epoch counter (NVLink mode, else nullptr): this MatMult is epoch *epoch_ctr + 1;
  // with bump, the kernel's last CTA stores it back (the MatMult ends in this kernel).
  // Device-side so that MatMults can be captured in CUDA graphs and replayed.
  unsigned long long *epoch_ctr;
  int bump;
  int *err;
};
struct SpmvTail {                      // fused off-diagonal SpMV-add (comm warps, halo_dev.cuh tail_warp)
  int n_bblocks, enabled;              // boundary blocks are the first n_bblocks in claim order
  const int32_t *rows, *rowptr, *col;  // compressed off-diagonal block
  const double *val;
  const uint4 *ghost;                  // flagged ghost lines, buffer (epoch & 1) at ghost_stride
  int64_t ghost_stride;
  int64_t n_ro;
  const HaloWait *waits;
  int nwaits, w;                       // w: lanes per off-diagonal row (power of two <= 32)
  unsigned int *ctr;                   // [0] boundary-block warps done, [1] chunk claims, [2] comm warps done,
                                       // [3] split tail: comm warps with sums out, [4] add-pass claims
  unsigned long long *trace;           // SPMAT_TRACE=1: globaltimer stamps (nullptr = off)
  // split tail (boundary rows in most row blocks, e.g. box partitions): natural claim order,
  // every block counts as a boundary block; the off-diagonal sums go to obuf during the sweep
  // and are added into y after it (halo_dev.cuh split_tail)
  double *obuf;                        // nullptr: boundary-blocks-first tail
};

// ------------------------------------------------------------------ matrix
struct spmat_s {
  spmat_comm_s *comm = nullptr;
  int64_t M = 0, N = 0, m = 0, n = 0;
  int64_t rstart = 0, rend = 0, cstart = 0, cend = 0;
  std::vector<int64_t> roff, coff;  // P+1 ownership offsets
  // diagonal block CSR (int32 local)
  int64_t nnz_d = 0;
  spmat::DevBuf<int32_t> rowptr_d, col_d;
  spmat::DevBuf<double> val_d;
  // off-diagonal block: compressed rows
  int64_t nnz_o = 0, n_ro = 0;
  int ro_w = 1;  // lanes per off-diagonal row in the SpMV-add kernels (offdiag_rows_w)
  spmat::DevBuf<int32_t> rows_o, rowptr_o, col_o;
  spmat::DevBuf<double> val_o;
  int64_t n_ghost = 0;
  spmat::DevBuf<int64_t> colmap;
  spmat::DevBuf<double> lvec;
  sf_s *halo = nullptr;
  // COO plan: nonzeros in block order (diag then offdiag)
  int64_t ncoo = 0, ncontrib = 0;
  spmat::DevBuf<uint32_t> jmap;     // nnz_d + nnz_o + 1
  spmat::DevBuf<uint32_t> perm;     // ncontrib: k (< ncoo) or ncoo + recv position
  int64_t n_mixed = 0;
  spmat::DevBuf<uint32_t> mixed;    // nonzero ids (block order) with received contributions
  // COO value exchange plan
  std::vector<int64_t> send_count, recv_count, send_off, recv_off;  // per rank
  int64_t nsend = 0, nrecv = 0;
  spmat::DevBuf<uint32_t> sendperm;  // k's, destination-major
  spmat::DevBuf<double> sendbuf, recvbuf;
  cudaEvent_t ev_send_ready = nullptr, ev_recv_done = nullptr;
  bool values_set = false;
  // SpMV schedule
  int kernel_id = 0;
  int kernel_id_csr = 0;
  spmat::DevBuf<int32_t> ro_of_row;  // row -> compressed off-diagonal row or -1 (k_spmv_direct_halo)
  int direct_halo_ok = -1;           // -1 not yet known             // the CSR kernel chosen at create (restored by set_block_size(A, 1))
  int64_t n_rowblocks = 0, max_row_nnz = 0;
  int lanes = 1;                     // lanes per row of the diagonal SpMV (row statistics)
  spmat::DevBuf<int2> rbp;           // n_rowblocks + 1 (first row, first nonzero) pairs
  spmat::DevBuf<int32_t> longrows;   // rows with more than kLong nonzeros
  int64_t n_long = 0;
  int env_bsr_wmax = 8;              // SPMAT_BSR_WMAX: cap on the lanes per block row (k_spmv_bsr3)
  int rb_budget = 0;                 // row-block cost budget (spmv_prepare; <= kBudget)
  int tma_grid = 0;                  // persistent grid of the bulk-copy SpMV
  int tma_grid_tail = 0;             // its grid with the fused off-diagonal add (>= tma_grid)
  spmat::DevBuf<int32_t> block_order;  // boundary row blocks first (fused off-diagonal tail)
  spmat::DevBuf<int4> blocks4;         // (r0, r1, p0, p1) per row block in claim order
  int64_t n_bblocks = 0;
  bool tail_split = false;             // SpmvTail.obuf mode (boundary rows in most row blocks)
  spmat::DevBuf<double> tail_obuf;
  spmat::DevBuf<unsigned int> tail_ctr;
  spmat::DevBuf<unsigned long long> trace;  // SPMAT_TRACE: [cta][kTraceCta] globaltimer stamps + header
  spmat::DevBuf<unsigned int> sched; // its block counter + finished-CTA counter
  // host staging for host x / y
  spmat::DevBuf<double> xstage, ystage;
  // profiling
  bool profile = false;
  std::vector<cudaEvent_t> prof_ev[3];  // pairs per kind
  size_t prof_n[3] = {0, 0, 0};
  int64_t plan_builds = 0;
  // counters (spmat_get_info): bytes enqueued on NCCL / stored into peers, calls
  int64_t stat_nccl_sent = 0, stat_nccl_recv = 0, stat_nvlink_put = 0, stat_mults = 0, stat_setvals = 0;
  // environment switches, read when the matrix is created (not process-wide statics)
  bool env_no_fuse = false;     // SPMAT_FUSE=0: standalone put kernel instead of the fused puts
  bool env_no_tail = false;     // SPMAT_FUSE_TAIL=0: off-diagonal add as its own kernel
  int env_pipe_chunks = 16;     // SPMAT_PIPE_CHUNKS: row chunks of the host-buffer pipeline
  int env_pipe_chunks_async = 1;  // SPMAT_PIPE_CHUNKS_ASYNC: the same for spmat_mult_async (measured 1: 3.06 ms, 2: 3.24, 8: 3.33 on C4)
  // device-initiated halo over NVLink peer memory (halo.cu)
  bool peer = false;
  spmat::DevBuf<unsigned long long> halo_flags;  // [q]: done flag from receiver q
  spmat::DevBuf<uint4> ghost;    // flagged ghost lines (halo_dev.cuh), two epochs' buffers
  std::vector<uint4 *> peer_ghost;
  std::vector<unsigned long long *> peer_flags;
  spmat::DevBuf<HaloPut> halo_puts;
  spmat::DevBuf<HaloWait> halo_waits;
  spmat::DevBuf<unsigned int> halo_counter;
  spmat::DevBuf<int> halo_err;
  int n_puts = 0, n_waits = 0, put_chunks_total = 0;
  spmat::DevBuf<unsigned long long> d_epoch;  // completed NVLink-halo MatMults (device)
  int64_t ghost_stride = 0;         // lines per epoch buffer of `ghost`
  // CUDA graph of one CG iteration (krylov.cu), keyed by the caller's x / history pointers
  cudaGraphExec_t cg_exec = nullptr, cg_exec_batch = nullptr;  // one iteration / kCgBatch iterations
  const void *cg_key_x = nullptr, *cg_key_h = nullptr;
  cudaStream_t cg_stream = nullptr;
  cudaEvent_t cg_ev[2] = {nullptr, nullptr};
  // 3x3 block-CSR copy of the diagonal block (bsr.cu), after spmat_set_block_size(A, 3)
  int bs = 1;
  int64_t mb = 0, nnzb = 0, n_brblocks = 0;
  int bsr_grid = 0;
  spmat::DevBuf<int32_t> browptr, bcol;
  spmat::DevBuf<double> bval;
  spmat::DevBuf<int4> bblocks4;
  spmat::DevBuf<unsigned int> bsched;
  // 3x3 block copy of the off-diagonal block (when it is made of aligned 3x3 blocks too):
  // block rows ob_rows (block-row ids), ob_rowptr, ob_col (ghost block = 3 consecutive ghost
  // lines), ob_val (9 per block); ob_range: per claim index of the block SpMV, the block rows
  // [t0, t1) of A_o in that row block (row blocks with off-diagonal block rows are claimed
  // last, so the fused kernel adds them after the ghost lines have landed)
  bool ob_ok = false;
  // set_values wrote the diagonal values straight into bval (k_numeric_bsr3): val_d is stale
  // until csr_sync (export, MatMultTranspose, set_block_size(A, 1))
  bool val_d_stale = false;
  bool env_numeric_csr = false;  // SPMAT_NUMERIC_BSR=0: always val_d, then the bval copy
  bool env_numeric_jmap = false; // SPMAT_NUMERIC_JMAP=1: read jmap even when it is the identity
  int env_numeric_seg = 8;       // SPMAT_NUMERIC_SEG=4|8: contributions per step of k_numeric_seg
  int64_t obr = 0, onnzb = 0;
  int ob_w = 4;
  int bsr_fuse_mode = 2;         // SPMAT_BSR_FUSE: 2 comm warps (default), 1 in-kernel add, 0 standalone kernels
  int64_t ob_nbblocks = 0;       // row blocks with off-diagonal block rows
  spmat::DevBuf<unsigned int> ob_ctr;  // comm-warp tail counters
  bool env_bsr_fma = true;       // SPMAT_BSR_FMA=0: separately rounded products in the block SpMV
  spmat::DevBuf<int32_t> ob_rows, ob_rowptr, ob_col;
  spmat::DevBuf<double> ob_val;
  spmat::DevBuf<int2> ob_range;
  spmat::DevBuf<unsigned int> ob_done;
  // host-buffer MatMult pipeline (mult.cu / spmv.cu), built on first use
  int pipe_chunks = 0;
  int pipe_slot = 0;                       // staging slot of the next host-buffer call (double-buffered)
  std::vector<int64_t> pipe_block, pipe_row, pipe_xmin, pipe_xneed;  // row-order block range, row range, x rows read
  std::vector<int64_t> pipe_q;             // [chunks+1] first compressed off-diagonal row of each chunk
  std::vector<char> pipe_put_chunk;        // chunk holds x rows the NVLink puts read
  spmat::DevBuf<int4> pipe_blocks4;        // row-ordered block table (when the claim order differs)
  cudaStream_t pipe_comm = nullptr;        // high-priority stream of the standalone put
  cudaStream_t pipe_in = nullptr, pipe_out = nullptr;
  cudaStream_t pipe_comp = nullptr;        // SpMV chunks of pipelined calls (spmat_mult_pipelined)
  bool pipe_pending = false;               // a pipelined call's download not yet waited for by the caller's stream
  cudaEvent_t pipe_ev_pending = nullptr;
  std::vector<cudaEvent_t> pipe_ev;                        // 2 * chunks + 2
  // CG / dot workspace (krylov.cu), allocated on first use
  spmat::DevBuf<double> cg_r, cg_p, cg_q, cg_partial, cg_partial2, cg_scalars, cg_reduced;
  // MatMultTranspose (transpose.cu): transposed diagonal / off-diagonal blocks, built lazily
  bool t_built = false;
  int64_t val_version = 0, t_val_version = -1;  // set_values count / values gathered for
  spmat::DevBuf<int32_t> t_rowptr_d, t_col_d, t_perm_d, t_rowptr_o, t_col_o, t_perm_o;
  spmat::DevBuf<double> t_val_d, t_val_o, t_lvec;
  spmat::DevBuf<unsigned> cg_count;  // CTA arrival counter of the dot kernels (last CTA finalizes)
};

namespace spmat {
int spmv_prepare(spmat_s *A, cudaStream_t stream);  // row blocks + kernel choice
// fuse_put: the bulk-copy SpMV's comm warps also perform this epoch's halo puts;
// fuse_tail: its consumer warps also add A_o lvec after the last row block
int spmv_diag(spmat_s *A, const double *x, double *y, cudaStream_t stream, bool fuse_put = false,
              bool fuse_tail = false);
int spmv_offdiag(spmat_s *A, double *y, cudaStream_t stream);
int spmv_direct_halo(spmat_s *A, const double *x, double *y, cudaStream_t s);  // small matrix, NVLink halo, one launch
int direct_halo_ok(spmat_s *A);  // its grid fits a cooperative launch
void cg_graph_release(spmat_s *A);            // drop the captured CG iteration
int bsr_refresh(spmat_s *A, cudaStream_t s, bool diag = true);  // bval (diag) and ob_val from the CSR values
int csr_sync(spmat_s *A, cudaStream_t s);  // val_d from bval when set_values wrote bval directly
// mode 1 / 2: also add the 3x3 off-diagonal blocks from this epoch's ghost lines and end the
// epoch (full MatMult, NVLink halo) -- by the consumers (1) or by comm warps that also do the
// puts (2); 0: diagonal only
int bsr_spmv(spmat_s *A, const double *x, double *y, cudaStream_t s, int mode = 0);
// off-diagonal SpMV-add on the 3x3 block copy: NVLink ghost lines of this epoch (ends the
// epoch, like k_spmv_offdiag_peer) or, with lvec != nullptr, the NCCL ghost vector
// cur: this MatMult's epoch (waits for its lines, ends the epoch); else the last completed one
int bsr_offdiag(spmat_s *A, double *y, const double *lvec, cudaStream_t s, bool cur = true);
// host-buffer pipeline (single rank): row chunks of the diagonal SpMV
int spmv_pipe_prepare(spmat_s *A, int chunks);  // chunk rows + the x columns each chunk reads
int spmv_diag_chunk(spmat_s *A, const double *x, double *y, int k, cudaStream_t s);
int peer_put_launch(const HaloPut *puts, int nputs, int chunks, const double *src,
                    const unsigned long long *epoch_ctr, int *err, cudaStream_t s);
int put_chunks_of(int64_t count);   // put warps (chunks) for `count` values (flagged lines)
int bulk_chunks_of(int64_t count);  // put warps of a bulk segment (one fence + flag per chunk)
int sf_peer_setup(sf_s *sf);
int sf_ensure_peer(sf_s *sf);      // collective; the deferred sf_peer_setup of a matrix halo SF       // collective; leaves sf->peer false (NCCL) when unavailable
int halo_peer_setup(spmat_s *A);                  // collective; leaves A->peer false on NCCL
void halo_peer_release(spmat_s *A);
int halo_peer_put(spmat_s *A, const double *x, cudaStream_t s);  // standalone put kernel
int halo_peer_offdiag(spmat_s *A, double *y, cudaStream_t s, bool compute);
int halo_peer_offdiag_range(spmat_s *A, double *y, int64_t q0, int64_t q1, cudaStream_t s);  // no epoch end
int halo_peer_epoch_end(spmat_s *A, cudaStream_t s);   // release the ghost buffer, advance the epoch
}  // namespace spmat
