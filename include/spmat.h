/*
 * spmat.h -- C ABI of libspmat: a B200-native (sm_100a) distributed fp64 MatMult on a
 * row-partitioned MPIAIJ matrix assembled on the device by COO, with a star-forest (SF) halo
 * exchange over NCCL.  The method is the one of arXiv 2406.08646 (PETSc/TAO on GPU-based
 * exascale systems); citations "P:n" are lines of that paper's text.
 *
 * Plain C: no torch or CUDA types in the signatures.  Streams are passed as `void *`
 * holding a cudaStream_t (NULL = the legacy default stream).  Every call returns an
 * spmat_status; a human-readable message for the last failure on the calling thread is
 * available from spmat_last_error().
 *
 * Process model: one process (rank) per GPU.  Collective calls must be made by every rank
 * of the communicator in the same order.
 *
 * Ownership: handles are opaque and caller-owned, freed by the matching *_destroy.  Data
 * pointers are borrowed for the duration of the call (host arrays) or until the work
 * enqueued on `stream` completes (device arrays).
 */
#ifndef SPMAT_H
#define SPMAT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPMAT_OK = 0,
  SPMAT_ERR_ARG = 1,      /* bad argument (null handle, negative size, x == y, bad op) */
  SPMAT_ERR_RANGE = 2,    /* COO index >= M or >= N; SF root offset outside the owner */
  SPMAT_ERR_STATE = 3,    /* call out of order (bcast_end without begin, op mismatch) */
  SPMAT_ERR_MISMATCH = 4, /* ranks disagree on global sizes / local sizes do not sum */
  SPMAT_ERR_OOM = 5,      /* device allocation failed */
  SPMAT_ERR_CUDA = 6,     /* CUDA runtime error (possibly from earlier asynchronous work) */
  SPMAT_ERR_NCCL = 7      /* NCCL missing (nranks > 1) or an NCCL error */
} spmat_status;

/* MatSetValuesCOO(A, v, mode).  Reading (Z2): INSERT sets every
   stored nonzero to +0.0 + (sum of its contributions); ADD adds that sum to the value. */
typedef enum { SPMAT_INSERT = 0, SPMAT_ADD = 1 } spmat_mode;

/* PetscSFBcast op: MPI_REPLACE or MPI_SUM ("add the source values or ... replace the
   destination values"). */
typedef enum { SF_REPLACE = 0, SF_SUM = 1 } sf_op;

typedef struct spmat_comm_s *spmat_comm_t;
typedef struct spmat_s *spmat_t;
typedef struct sf_s *sf_t;

/* Library version (major*10000 + minor*100 + patch). */
int spmat_version(void);

/* Thread-local message describing the last failure (never NULL). */
const char *spmat_last_error(void);

/* ------------------------------------------------------------------ communicator --- */

/* Fill id[128] with a fresh NCCL unique id.  Called on rank 0 only; the caller broadcasts
   the bytes to the other ranks (e.g. with torch.distributed).  Needs NCCL. */
int spmat_comm_unique_id(unsigned char id[128]);

/* Create the per-rank communicator on CUDA device `device`.  Collective when nranks > 1
   (NCCL communicator from `id`); with nranks == 1 `id` may be NULL and NCCL is not used.
   Creates the library's high-priority communication stream on that device. */
int spmat_comm_create(const unsigned char *id, int nranks, int rank, int device,
                      spmat_comm_t *out);

/* Poll asynchronous NCCL errors (ncclCommGetAsyncError) and sticky CUDA errors. */
int spmat_comm_check(spmat_comm_t comm);

int spmat_comm_destroy(spmat_comm_t comm);

/* ------------------------------------------------------------------- star forest --- */

/* PetscSF creation: "created collectively by specifying, for each leaf on the
   current process, the owner rank and an offset of the corresponding root on the owner".
     nroots           number of roots owned by this rank (valid offsets are [0, nroots))
     nleaves          number of leaves on this rank
     ilocal           leaf l's index in leafdata (host or device array of nleaves); NULL
                      means leaf l is leafdata[l]
     remote_rank      owner rank of leaf l's root (host or device, nleaves entries)
     remote_offset    root offset on the owner (host or device, nleaves entries)
   Collective and host-synchronising.  Errors: SPMAT_ERR_ARG (rank outside [0,nranks),
   duplicate ilocal), SPMAT_ERR_RANGE (offset >= owner's nroots; reported on every rank).
   The plan groups leaves by owner rank ascending, then (root offset, leaf index). */
int sf_create(spmat_comm_t comm, int64_t nroots, int64_t nleaves, const int64_t *ilocal,
              const int32_t *remote_rank, const int64_t *remote_offset, sf_t *out);

/* Split-phase broadcast root -> leaf.  rootdata (nroots doubles) and leafdata
   (covering every ilocal) are DEVICE arrays.  It never blocks the host.  Transport (chosen
   collectively at sf_create, see sf_transport):
     NVLink (default with several ranks, the paper's NVSHMEM SF P:533-562 with CUDA IPC):
       begin enqueues on `stream` a put kernel that stores the root values as flagged 16-byte
       lines straight into the leaf owners' staging buffers (it waits only for the owner to
       have released the buffer it used two operations ago); end enqueues on `stream` the
       kernel that reads each line once it has landed and writes leafdata.
     NCCL (SPMAT_SF=nccl or SPMAT_HALO=nccl, or IPC unavailable): begin enqueues pack -> NCCL
       send/recv -> unpack on the communication stream; end makes `stream` wait for it.
   Between begin and end the caller may enqueue independent work on `stream`; it must not
   write rootdata or read leafdata.  Leaf entries not in the SF are untouched.  End must
   name the same buffers and op as begin (else SPMAT_ERR_STATE).  Collective: every rank
   calls begin/end the same number of times. */
int sf_bcast_begin(sf_t sf, const double *rootdata, double *leafdata, int op, void *stream);
int sf_bcast_end(sf_t sf, const double *rootdata, double *leafdata, int op, void *stream);

/* Split-phase reduce leaf -> root ("reduces leaf values into roots").  leafdata
   and rootdata are DEVICE arrays.  Contributions to one root are applied in ascending
   (source rank, leaf index) order (reading of SPEC.md L139-141): SUM adds them one at a time
   to the root's value; REPLACE stores the last one.  Roots nobody references are untouched.
   Same split-phase and stream rules as sf_bcast_*; begin must not be issued while another
   operation of this SF is pending (SPMAT_ERR_STATE). */
int sf_reduce_begin(sf_t sf, const double *leafdata, double *rootdata, int op, void *stream);
int sf_reduce_end(sf_t sf, const double *leafdata, double *rootdata, int op, void *stream);

/* info[0..7] = nroots, nleaves, n_send_neighbours, n_recv_neighbours, n_send_values,
   n_recv_values, n_self_edges, packed (1 if any pack or unpack kernel is needed) */
int sf_get_info(sf_t sf, int64_t info[8]);

/* Test hook: what = 0 recv neighbour ranks, 1 recv counts, 2 leaf indices in receive
   order, 3 send neighbour ranks, 4 send counts, 5 root offsets in send order
   (all int64).  Copies min(cap, len) values into host_buf; *len = full length. */
int sf_export(sf_t sf, int what, void *host_buf, int64_t cap, int64_t *len);

/* 2 if this SF moves data as flagged lines over NVLink peer memory, 1 if over NCCL (0 with
   one rank and no remote edges). */
int sf_transport(sf_t sf);

/* Synchronise the device and report a timed-out NVLink wait (a peer that never delivered
   or released a buffer within ~20 s) as SPMAT_ERR_NCCL; else SPMAT_OK. */
int sf_check(sf_t sf);

int sf_destroy(sf_t sf);

/* ------------------------------------------------------------------------ matrix --- */

/* MatSetPreallocationCOO(A, n, i, j).  Symbolic COO assembly.
     m_local, n_local   rows / columns owned by this rank (contiguous ranges in rank order,
                        P:661-662); they must sum to M / N over ranks
     ncoo               length of coo_i / coo_j on this rank
     coo_i, coo_j       global int64 indices, host or device memory (detected); not
                        retained ("can be freed after this stage")
   Entries with i < 0 or j < 0 are ignored.  Off-rank rows are routed to their
   owners over NCCL; the owner sorts contributions by (i, j, src rank, k), splits the
   diagonal block (columns in [cstart, cend)) from the off-diagonal block, builds colmap
   (sorted unique ghost columns), the per-nonzero contribution plan (jmap/perm), the COO
   send/receive plans and the halo SF.  Collective and host-synchronising: it first waits for
   all work already queued on the device (cudaDeviceSynchronize), so device coo_i/coo_j may
   come from kernels on any stream.
   Errors: SPMAT_ERR_RANGE if i >= M or j >= N (message names the rank and k; reported on
   every rank), SPMAT_ERR_MISMATCH if ranks disagree on M, N or the local sizes,
   SPMAT_ERR_ARG for m_local >= 2^31, ncoo >= 2^32, null coo_i/coo_j with ncoo > 0, or more
   than 2^31 contributions on a rank.  An error found on one rank only (an argument, an
   allocation) is agreed on before the next collective step: every rank returns an error
   (the others "failed on another rank") instead of blocking in NCCL. */
int spmat_create_coo(spmat_comm_t comm, int64_t m_local, int64_t n_local, int64_t M,
                     int64_t N, int64_t ncoo, const int64_t *coo_i, const int64_t *coo_j,
                     spmat_t *out);

/* MatSetValuesCOO(A, v, mode).  v: DEVICE array of this rank's ncoo doubles in
   the order of coo_i/coo_j.  Enqueue-only: send-buffer gather -> NCCL value exchange on
   the comm stream, overlapped with the kernel that finishes every nonzero whose
   contributions are all local; nonzeros with received contributions are finished after the
   exchange.  Each nonzero is summed by one thread in ascending (src rank, k) order: no
   atomics, deterministic.  After spmat_set_block_size(A, 3) (and when no
   contribution is received from another rank) the diagonal values are summed straight into
   the 3x3 block copy; the CSR copy is brought up to date when it is needed (export,
   MatMultTranspose, set_block_size(A, 1)).  Collective. */
int spmat_set_values_coo(spmat_t A, const double *v, int mode, void *stream);

/* MatMult y = A x.  x: n_local doubles, y: m_local doubles, x != y.
   Device pointers: enqueue-only -- halo bcast_begin (x -> ghost vector) on the comm stream,
   diagonal-block SpMV on `stream`, bcast_end, off-diagonal SpMV-add on `stream`.
   Host pointers (pinned or pageable; memtype detected as in P:252-260): x is copied to the
   device and y back inside the call's stream order; the call then returns after y is
   written.  Collective.
   NVLink halo: a peer that never delivers (bounded device spins, ~20 s) makes the affected
   ghost values 0.0 and sets an error word that the call itself cannot report without a
   host synchronisation -- spmat_check() reports it (SPMAT_ERR_NCCL).  The fused kernel
   (comm warps spinning on peer data) is launched cooperatively, so every CTA is resident
   or the launch fails. */
int spmat_mult(spmat_t A, const double *x, double *y, void *stream);

/* spmat_mult that never blocks the host, also for host x / y (which must then be pinned to
   overlap): the copies and the MatMult are only enqueued, y is valid and x may be rewritten
   once the work enqueued on `stream` has completed (synchronise the stream or an event).
   Consecutive calls alternate between two device staging slots, so call k+1's upload of x
   overlaps call k's download of y (PCIe is full duplex).  Device pointers: as spmat_mult.
   Collective. */
int spmat_mult_async(spmat_t A, const double *x, double *y, void *stream);

/* spmat_mult_async for a stream of MatMults on pinned host buffers (a serving loop): the SpMV
   runs on an internal stream and the caller's `stream` is made to wait for this call's download
   of y only at the NEXT call on this matrix (any spmat_mult* call) or at spmat_mult_flush -- so
   call k+1's SpMV also overlaps call k's download.  y of a call is valid once `stream` has
   completed the work enqueued up to the next call or flush.  Work the caller enqueues on
   `stream` after the call is ordered after this call's SpMV (set_values may follow safely).
   Device pointers: as spmat_mult.  Collective. */
int spmat_mult_pipelined(spmat_t A, const double *x, double *y, void *stream);

/* Make `stream` wait for the download of y left pending by the last spmat_mult_pipelined call
   (no-op if none).  Enqueue only. */
int spmat_mult_flush(spmat_t A, void *stream);

/* MatMultTranspose: y = A^T x (collective, enqueue-only).  x: DEVICE array of m_local doubles
   (the row layout), y: DEVICE array of n_local doubles (the column layout).  PETSc's MPIAIJ
   order: lvec = A_o^T x, y = A_d^T x, then the halo star forest reduces lvec into the owners' y
   with SUM (sf_reduce): every y entry is summed from +0.0 over its column's rows in
   ascending order, then the other ranks' sums are added in ascending rank order -- a fixed,
   rank-count-independent order (real-valued results reproducible bit for bit).  The transposed blocks are built on
   the first call (device radix sort, host-synchronising) and their values re-gathered after
   every spmat_set_values_coo; the first call also builds the halo SF's NVLink transport
   (collective, host-synchronising; see spmat_get_halo_sf).  Host x or y: SPMAT_ERR_ARG. */
int spmat_mult_transpose(spmat_t A, const double *x, double *y, void *stream);

/* MatSetBlockSize analogue for the SpMV storage (block-CSR on GPU): bs = 3 checks that
   the assembled diagonal block consists of dense, aligned 3x3 blocks (node-block matrices with
   3 dofs per node) and from then on multiplies it from a 3x3 block-CSR copy (8.44 instead of
   12 bytes per nonzero), refreshed after every spmat_set_values_coo; bs = 1 returns to CSR.
   SPMAT_ERR_ARG if the structure is not blocked (the matrix keeps CSR).  Local, host-
   synchronising.  With several ranks, an off-diagonal block made of aligned 3x3 blocks too
   (node-block COO) is also kept as 3x3 blocks and multiplied by its own kernel
   (SPMAT_BSR_OFFDIAG=0: the CSR off-diagonal kernels; SPMAT_BSR_FUSE=1: added inside the
   block SpMV instead of after it). */
int spmat_set_block_size(spmat_t A, int bs);

/* Parts of MatMult for isolated timing: part bit 1 = diagonal SpMV (y = A_d x), bit 2 =
   halo exchange (x -> ghost vector), bit 4 = off-diagonal SpMV-add (y += A_o ghosts).
   part 7 == spmat_mult on device pointers. */
int spmat_mult_part(spmat_t A, const double *x, double *y, int part, void *stream);

/* info[0..15] = rstart, rend, cstart, cend, nnz_d, nnz_o, n_ghost, n_offdiag_rows,
   n_contrib, n_send (COO entries sent), n_recv (COO entries received), n_mixed (nonzeros
   with received contributions), spmv_kernel_id, n_rowblocks, max_row_nnz, plan_builds;
   info[16..31] = block_size, offdiag_3x3 (1: the off-diagonal block is kept in 3x3 blocks
   too), offdiag_lanes, halo_mode (0 one rank, 1 NCCL, 2 NVLink stores), and cumulative
   counters since create (host-side, counted when work is enqueued): nccl_bytes_sent,
   nccl_bytes_recv (COO value exchange + NCCL-mode halo), nvlink_bytes_put (halo lines stored
   into peers: 16 B per value), n_mult, n_set_values, then spmv_grid, offdiag_grid (the
   grid with the fused off-diagonal add, incl. CTAs that only run it),
   halo_sf_transport (the halo SF's own transport: 0 not built yet / one rank, 1 NCCL,
   2 NVLink), 0...
   The caller provides 32 entries. */
int spmat_get_info(spmat_t A, int64_t info[32]);

/* Test hook: copy a device array to host.  All integer arrays are returned as int64.
     0 rowptr_d[m+1]   1 col_d (local)   2 val_d (f64)   3 rowptr_o[m+1] (full rows)
     4 col_o (ghost index)   5 val_o (f64)   6 colmap (global ghost columns)
     7 jmap[nnz_d+nnz_o+1] (diag nonzeros then offdiag nonzeros)
     8 contribution source rank per jmap entry   9 contribution index per jmap entry: k for
       local entries, position within the message from that source rank for received ones
     10 send_count[nranks]  11 send_k (COO k's sent, destination-major)
     12 recv_count[nranks]  13 rows_o (compressed off-diagonal rows)
   *len = full length; min(cap, len) values are copied. */
int spmat_export(spmat_t A, int what, void *host_buf, int64_t cap, int64_t *len);

/* The halo SF (leaves = ghost columns in colmap order).  Borrowed: do not destroy.
   Collective on the first call with several ranks: the SF's NVLink transport (staging lines
   and peer mappings) is built then, not at create, when the matrix's own MatMult halo has its
   NVLink path -- only MatMultTranspose and borrowed SFs use it.  The first
   spmat_mult_transpose builds it the same way. */
int spmat_get_halo_sf(spmat_t A, sf_t *borrowed);

/* Per-kernel timing with CUDA events recorded on the launching streams.  enable=1 starts
   recording around the diagonal SpMV and off-diagonal SpMV-add of every spmat_mult;
   spmat_profile_read() synchronises, returns the summed milliseconds and launch counts
   (ms[0]/n[0] diagonal SpMV, ms[1]/n[1] off-diagonal, ms[2]/n[2] halo on the comm stream)
   and clears them. */
int spmat_profile(spmat_t A, int enable);
int spmat_profile_read(spmat_t A, double ms[4], int64_t n[4]);

/* ------------------------------------------------------ Krylov (CGAsync) --- */

/* VecDotAsync: *result (DEVICE scalar) = sum over all ranks of a.b, a and b
   DEVICE arrays of m_local doubles in this matrix's row layout.  Enqueue-only, collective.
   Deterministic: fixed per-rank reduction tree, ranks summed in rank order through a scalar
   board in IPC-mapped device memory (NVLink); identical result on every rank. */
int spmat_vec_dot(spmat_t A, const double *a, const double *b, double *result, void *stream);

/* Unpreconditioned conjugate gradients for a square A, maxit iterations, all scalars on the
   device and no host synchronisation (CGAsync; no convergence test inside the
   loop).  Per iteration: q = A p (spmat_mult), alpha = rr / p.q, x += alpha p,
   r -= alpha q, rr' = r.r, beta = rr'/rr, p = r + beta p.  b (in), x (in: initial guess,
   out: iterate) are DEVICE arrays of m_local doubles; rr_hist (DEVICE, maxit+1 doubles, or
   NULL) receives r_k.r_k.  If p.q or rr becomes 0 the iterate stops changing.
   Enqueue-only, collective; workspace is allocated on first use. */
int spmat_cg(spmat_t A, const double *b, double *x, int maxit, double *rr_hist, void *stream);

/* Synchronise the device and report asynchronous failures of this matrix's work: CUDA
   errors, NCCL async errors, and a device-initiated halo whose peer never answered. */
int spmat_check(spmat_t A);

/* Halo transport chosen at create time (collectively): 0 = single rank (none), 1 = NCCL
   send/recv on the comm stream, 2 = device-initiated stores into the peer ghost vectors over
   NVLink (CUDA IPC mappings; the NVSHMEM-SF analogue of P:533-562).  SPMAT_HALO=nccl in the
   environment forces 1. */
int spmat_halo_mode(spmat_t A);

/* Device trace of the last fused MatMult kernel (created with SPMAT_TRACE=1 in the
   environment, else *len = 0): globaltimer nanoseconds, per CTA [start, -, last block done,
   end] then per off-diagonal work item [start, halo ready, done].  Copies min(cap, len). */
int spmat_trace_read(spmat_t A, int64_t *host_buf, int64_t cap, int64_t *len);

int spmat_destroy(spmat_t A);

#ifdef __cplusplus
}
#endif

#endif /* SPMAT_H */
