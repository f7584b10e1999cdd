// sf.cu -- star-forest (PetscSF) plan and split-phase broadcast over NCCL.
//
// P:446-482.  "Leaves are locally indexed with integers, while roots are globally indexed
// via tuples of (owner rank, offset).  A PetscSF is created collectively by specifying, for
// each leaf on the current process, the owner rank and an offset of the corresponding root
// on the owner.  PETSc analyzes the graph and derives the communication pattern."
// Bcast moves root values to leaves with REPLACE or SUM; when roots or leaves are not
// consecutive "PETSc will call its pack or unpack kernels".  With REPLACE and
// consecutive indices the user buffers are the transport buffers directly.
//
// B200 design: the plan (grouping, contiguity detection) is built on the host once; each
// Bcast is fully stream-ordered on the library's high-priority comm stream: pack kernel
// (only for non-consecutive roots) -> grouped ncclSend/ncclRecv -> self-edge copy kernel ->
// unpack kernel (only for non-consecutive leaves or SUM).  No host synchronisation.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "halo_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace spmat {

__global__ void k_gather(const double *__restrict__ src, const int64_t *__restrict__ idx,
                         double *__restrict__ dst, int64_t n) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; t < n; t += stride) dst[t] = src[idx[t]];
}

// leaf[lidx[t]] = src[sidx ? sidx[t] : t]  (REPLACE)  or  += (SUM)
__global__ void k_scatter(const double *__restrict__ src, const int64_t *__restrict__ sidx,
                          double *__restrict__ leaf, const int64_t *__restrict__ lidx, int64_t n,
                          int op) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; t < n; t += stride) {
    double v = src[sidx ? sidx[t] : t];
    int64_t l = lidx[t];
    leaf[l] = op == SF_REPLACE ? v : leaf[l] + v;
  }
}

static inline unsigned grid_for(int64_t n, int threads, int sms) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sms * 8;
  return (unsigned)std::max<int64_t>(1, std::min(b, cap));
}

void sf_free(sf_s *sf) {
  if (!sf) return;
  for (void *p : sf->peer_mem) cudaIpcCloseMemHandle(p);
  sf->peer_mem.clear();
  if (sf->ev_begin) cudaEventDestroy(sf->ev_begin);
  if (sf->ev_done) cudaEventDestroy(sf->ev_done);
  if (sf->ev_take) cudaEventDestroy(sf->ev_take);
  delete sf;
}

int sf_build(spmat_comm_s *comm, int64_t nroots, int64_t nleaves, const int64_t *h_ilocal,
             const int32_t *h_rank, const int64_t *h_offset, sf_s **out, bool defer_peer) {
  *out = nullptr;
  const int P = comm->nranks, me = comm->rank;
  // ---- local validation, agreed collectively so that no rank is left in a collective
  int64_t st[2] = {SPMAT_OK, 0};
  std::string msg;
  if (nroots < 0 || nleaves < 0) {
    st[0] = SPMAT_ERR_ARG;
    msg = "negative nroots/nleaves";
  }
  for (int64_t l = 0; l < nleaves && st[0] == SPMAT_OK; ++l) {
    if (h_rank[l] < 0 || h_rank[l] >= P) {
      st[0] = SPMAT_ERR_ARG;
      char b[128];
      snprintf(b, sizeof b, "leaf %lld: remote rank %d outside [0,%d)", (long long)l,
               h_rank[l], P);
      msg = b;
    } else if (h_offset[l] < 0) {
      st[0] = SPMAT_ERR_RANGE;
      char b[128];
      snprintf(b, sizeof b, "leaf %lld: negative root offset", (long long)l);
      msg = b;
    } else if (h_ilocal && h_ilocal[l] < 0) {
      st[0] = SPMAT_ERR_ARG;
      msg = "negative ilocal";
    }
  }
  if (st[0] == SPMAT_OK && h_ilocal) {
    std::vector<int64_t> s(h_ilocal, h_ilocal + nleaves);
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end()) {
      st[0] = SPMAT_ERR_ARG;
      msg = "duplicate ilocal entries";
    }
  }
  SP_TRY(comm->allreduce_max_i64(st, 1));
  if (st[0] != SPMAT_OK)
    return fail((int)st[0], "sf_create: %s", msg.empty() ? "error on another rank" : msg.c_str());

  // ---- order leaves by (owner rank, root offset, leaf index)
  auto leaf_of = [&](int64_t l) { return h_ilocal ? h_ilocal[l] : l; };
  std::vector<int64_t> ord(nleaves);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
    if (h_rank[a] != h_rank[b]) return h_rank[a] < h_rank[b];
    if (h_offset[a] != h_offset[b]) return h_offset[a] < h_offset[b];
    return leaf_of(a) < leaf_of(b);
  });
  sf_s *sf = new sf_s();
  sf->comm = comm;
  sf->nroots = nroots;
  sf->nleaves = nleaves;
  std::vector<int64_t> cnt(P, 0);
  for (int64_t l = 0; l < nleaves; ++l) cnt[h_rank[l]]++;
  std::vector<int64_t> self_leaf, self_root, req_off;  // req_off: offsets requested, by owner
  std::vector<int64_t> req_start(P + 1, 0);
  for (int q = 0; q < P; ++q) req_start[q + 1] = req_start[q] + (q == me ? 0 : cnt[q]);
  req_off.resize(req_start[P]);
  sf->h_leaf_idx.resize(req_start[P]);
  {
    std::vector<int64_t> fill(P, 0);
    for (int64_t t = 0; t < nleaves; ++t) {
      int64_t l = ord[t];
      int q = h_rank[l];
      if (q == me) {
        self_leaf.push_back(leaf_of(l));
        self_root.push_back(h_offset[l]);
      } else {
        int64_t at = req_start[q] + fill[q]++;
        req_off[at] = h_offset[l];
        sf->h_leaf_idx[at] = leaf_of(l);
      }
    }
  }
  for (int q = 0; q < P; ++q) {
    if (q == me || cnt[q] == 0) continue;
    sf->rnbr.push_back(q);
    sf->rcount.push_back(cnt[q]);
    sf->roff.push_back(req_start[q]);
    bool contig = true;
    for (int64_t t = 1; t < cnt[q] && contig; ++t)
      contig = sf->h_leaf_idx[req_start[q] + t] == sf->h_leaf_idx[req_start[q]] + t;
    sf->leaf_start.push_back(contig ? sf->h_leaf_idx[req_start[q]] : -1);
    if (!contig) sf->need_unpack_any = true;
  }
  sf->nrecv = req_start[P];
  sf->nself = (int64_t)self_leaf.size();
  // self-edge offsets are validated locally
  int64_t bad = -1;
  for (size_t t = 0; t < self_root.size(); ++t)
    if (self_root[t] >= nroots) bad = self_root[t];

  // ---- exchange request counts and offsets
  std::vector<int64_t> mine(P, 0), all((size_t)P * P, 0);
  for (int q = 0; q < P; ++q) mine[q] = q == me ? 0 : cnt[q];
  int s = comm->allgather_i64(mine.data(), P, all.data());
  if (s != SPMAT_OK) {
    sf_free(sf);
    return s;
  }
  std::vector<int64_t> scount(P), sstart(P + 1, 0);
  for (int p = 0; p < P; ++p) scount[p] = all[(size_t)p * P + me];
  for (int p = 0; p < P; ++p) sstart[p + 1] = sstart[p] + scount[p];
  sf->nsend = sstart[P];
  sf->h_root_idx.resize(sf->nsend);
  if (P > 1) {
    DevBuf<int64_t> dreq, dgot;
    std::vector<int64_t> rc(P);
    for (int q = 0; q < P; ++q) rc[q] = req_start[q + 1] - req_start[q];
    if ((s = dreq.alloc(req_off.size())) || (s = dgot.alloc(sf->nsend))) {
      sf_free(sf);
      return s;
    }
    cudaError_t e = cudaSuccess;
    if (!req_off.empty())
      e = cudaMemcpyAsync(dreq.get(), req_off.data(), req_off.size() * 8, cudaMemcpyHostToDevice,
                          comm->setup_stream);
    if (e == cudaSuccess) {
      s = comm->exchange_dev(dreq.get(), req_start.data(), rc.data(), dgot.get(), sstart.data(),
                             scount.data(), sizeof(int64_t), comm->setup_stream);
      if (s != SPMAT_OK) {
        sf_free(sf);
        return s;
      }
      if (sf->nsend)
        e = cudaMemcpyAsync(sf->h_root_idx.data(), dgot.get(), sf->nsend * 8,
                            cudaMemcpyDeviceToHost, comm->setup_stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(comm->setup_stream);
    }
    if (e != cudaSuccess) {
      sf_free(sf);
      return fail(SPMAT_ERR_CUDA, "sf_create exchange: %s", cudaGetErrorString(e));
    }
  }
  for (int64_t t = 0; t < sf->nsend; ++t)
    if (sf->h_root_idx[t] >= nroots) bad = sf->h_root_idx[t];
  int64_t st2[1] = {bad >= 0 ? (int64_t)SPMAT_ERR_RANGE : (int64_t)SPMAT_OK};
  s = comm->allreduce_max_i64(st2, 1);
  if (s != SPMAT_OK || st2[0] != SPMAT_OK) {
    sf_free(sf);
    if (s != SPMAT_OK) return s;
    if (bad >= 0)
      return fail(SPMAT_ERR_RANGE, "sf_create: root offset %lld >= nroots %lld on rank %d",
                  (long long)bad, (long long)nroots, me);
    return fail(SPMAT_ERR_RANGE, "sf_create: root offset out of range on another rank");
  }
  for (int p = 0; p < P; ++p) {
    if (p == me || scount[p] == 0) continue;
    sf->snbr.push_back(p);
    sf->scount.push_back(scount[p]);
    sf->soff.push_back(sstart[p]);
    bool contig = true;
    for (int64_t t = 1; t < scount[p] && contig; ++t)
      contig = sf->h_root_idx[sstart[p] + t] == sf->h_root_idx[sstart[p]] + t;
    sf->root_start.push_back(contig ? sf->h_root_idx[sstart[p]] : -1);
    if (!contig) sf->need_pack = true;
  }
  // ---- device arrays
  DeviceGuard g(comm->device);
  auto up = [&](DevBuf<int64_t> &d, const std::vector<int64_t> &h) -> int {
    int r = d.alloc(h.size());
    if (r) return r;
    if (!h.empty()) {
      cudaError_t e = cudaMemcpy(d.get(), h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(SPMAT_ERR_CUDA, "sf upload: %s", cudaGetErrorString(e));
    }
    return SPMAT_OK;
  };
  if ((s = up(sf->d_leaf_idx, sf->h_leaf_idx)) || (s = up(sf->d_root_idx, sf->h_root_idx)) ||
      (s = up(sf->d_self_leaf, self_leaf)) || (s = up(sf->d_self_root, self_root)) ||
      (s = sf->d_sendbuf.alloc(sf->need_pack ? sf->nsend : 0)) ||
      (s = sf->d_recvbuf.alloc(sf->nrecv))) {
    sf_free(sf);
    return s;
  }
  // ---- reduce plan: every contribution (root, source rank, sequence) sorted; the sequence
  // within one source follows that source's leaf order (its leaves are sorted by
  // (owner, root offset, leaf index)), so a root sees ascending (source rank, leaf index)
  {
    struct Con { int64_t root, src, seq, code; };
    std::vector<Con> cons;
    cons.reserve(sf->nsend + self_root.size());
    for (size_t a = 0; a < sf->snbr.size(); ++a)
      for (int64_t t = 0; t < sf->scount[a]; ++t)
        cons.push_back({sf->h_root_idx[sf->soff[a] + t], sf->snbr[a], t, sf->soff[a] + t});
    for (size_t t = 0; t < self_root.size(); ++t)
      cons.push_back({self_root[t], me, (int64_t)t, -(int64_t)t - 1});
    std::sort(cons.begin(), cons.end(), [](const Con &x, const Con &y) {
      if (x.root != y.root) return x.root < y.root;
      if (x.src != y.src) return x.src < y.src;
      return x.seq < y.seq;
    });
    std::vector<int64_t> roots, ptr(1, 0), code;
    for (size_t t = 0; t < cons.size(); ++t) {
      if (t == 0 || cons[t].root != cons[t - 1].root) {
        if (t) ptr.push_back((int64_t)t);
        roots.push_back(cons[t].root);
      }
      code.push_back(cons[t].code);
    }
    if (!cons.empty()) ptr.push_back((int64_t)cons.size());
    sf->n_touched = (int64_t)roots.size();
    if ((s = up(sf->d_red_roots, roots)) || (s = up(sf->d_red_ptr, ptr)) ||
        (s = up(sf->d_red_code, code)) || (s = sf->d_redbuf.alloc(sf->nsend))) {
      sf_free(sf);
      return s;
    }
  }
  if (cudaEventCreateWithFlags(&sf->ev_begin, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&sf->ev_done, cudaEventDisableTiming) != cudaSuccess) {
    sf_free(sf);
    return fail(SPMAT_ERR_CUDA, "sf_create: event creation failed");
  }
  // a matrix's halo SF: its MatMult has its own NVLink buffers (halo.cu), so the SF's transport
  // is built on first use (MatMultTranspose, a borrowed SF, or the MatMult halo when that has
  // no NVLink path of its own)
  sf->peer_deferred = defer_peer && comm->nranks > 1;
  if (!sf->peer_deferred && (s = sf_peer_setup(sf)) != SPMAT_OK) {
    sf_free(sf);
    return s;
  }
  *out = sf;
  return SPMAT_OK;
}

// ------------------------------------------------------------------ NVLink transport
// The paper's NVSHMEM PetscSF with CUDA IPC instead of NVSHMEM: at creation every
// rank maps the staging buffers of the ranks it sends to; a Bcast/Reduce is then a put kernel
// (flagged lines straight into the consumer's buffer over NVLink, after the consumer released
// that buffer two epochs ago) and a consuming kernel that reads each line once it carries the
// epoch, applies the op, and releases the buffer.  No NCCL kernel, no host synchronisation.
int sf_ensure_peer(sf_s *sf) {
  if (!sf || !sf->peer_deferred) return SPMAT_OK;
  sf->peer_deferred = false;
  return sf_peer_setup(sf);
}

int sf_peer_setup(sf_s *sf) {
  spmat_comm_s *c = sf->comm;
  const int P = c->nranks, me = c->rank;
  sf->peer = false;
  if (P == 1) return SPMAT_OK;
  // SPMAT_SF=nccl (or SPMAT_HALO=nccl, which also covers the matrix halo's SF) keeps NCCL
  const char *env = getenv("SPMAT_SF"), *henv = getenv("SPMAT_HALO");
  int64_t vote0[1] = {((env && !strcmp(env, "nccl")) || (henv && !strcmp(henv, "nccl"))) ? 1 : 0};
  SP_TRY(c->allreduce_max_i64(vote0, 1));
  if (vote0[0]) return SPMAT_OK;
  DeviceGuard g(c->device);
  sf->bstride = std::max<int64_t>(sf->nrecv, 1);
  sf->rstride = std::max<int64_t>(sf->nsend, 1);
  SP_TRY(sf->bline.alloc(2 * (size_t)sf->bstride));
  SP_TRY(sf->rline.alloc(2 * (size_t)sf->rstride));
  // bulk segments (>= bulk_min values): plain doubles + one release flag per put chunk, the
  // chunk flags after the 2P done flags (bcast segments, then reduce segments).  Flagged lines
  // move twice the bytes but need no fence: measured (SF-pingpong, 2 B200) lines are faster up
  // to ~8 MB, bulk from ~32 MB (110 vs 121 us) -- hence the 2^21-value default.
  int64_t bulk_min = (int64_t)1 << 21;
  if (const char *e = getenv("SPMAT_SF_BULK_MIN")) bulk_min = std::max<int64_t>(1, atoll(e));
  std::vector<int64_t> bflag_off(P, -1), rflag_off(P, -1);
  int64_t nflags = 2 * (int64_t)P;
  for (size_t a = 0; a < sf->rnbr.size(); ++a)
    if (sf->rcount[a] >= bulk_min) {
      bflag_off[sf->rnbr[a]] = nflags;
      nflags += bulk_chunks_of(sf->rcount[a]);
    }
  for (size_t a = 0; a < sf->snbr.size(); ++a)
    if (sf->scount[a] >= bulk_min) {
      rflag_off[sf->snbr[a]] = nflags;
      nflags += bulk_chunks_of(sf->scount[a]);
    }
  SP_TRY(sf->pflags.alloc(nflags));
  SP_TRY(sf->d_ep.alloc(2));
  SP_TRY(sf->pcounter.alloc(1));
  SP_TRY(sf->perr.alloc(1));
  SP_CUDA(cudaEventCreateWithFlags(&sf->ev_take, cudaEventDisableTiming));
  SP_CUDA(cudaMemset(sf->bline.get(), 0, sf->bline.n * sizeof(uint4)));  // flag 0: no epoch
  SP_CUDA(cudaMemset(sf->rline.get(), 0, sf->rline.n * sizeof(uint4)));
  SP_CUDA(cudaMemset(sf->pflags.get(), 0, nflags * sizeof(unsigned long long)));
  SP_CUDA(cudaMemset(sf->d_ep.get(), 0, 2 * sizeof(unsigned long long)));
  SP_CUDA(cudaMemset(sf->pcounter.get(), 0, sizeof(unsigned)));
  SP_CUDA(cudaMemset(sf->perr.get(), 0, sizeof(int)));
  cudaIpcMemHandle_t h[3];
  memset(h, 0, sizeof h);
  int64_t fail_ = 0;
  if (cudaIpcGetMemHandle(&h[0], sf->bline.get()) != cudaSuccess ||
      cudaIpcGetMemHandle(&h[1], sf->rline.get()) != cudaSuccess ||
      cudaIpcGetMemHandle(&h[2], sf->pflags.get()) != cudaSuccess) {
    cudaGetLastError();
    fail_ = 1;
  }
  int64_t v1[1] = {fail_};
  SP_TRY(c->allreduce_max_i64(v1, 1));
  if (v1[0]) {
    note_fallback(c, "a star forest", "cudaIpcGetMemHandle failed on some rank");
    return SPMAT_OK;  // NCCL transport on every rank
  }
  // per rank: 3 handles, strides, and for every peer p the offset of p's data in my bline
  // (p sends me roots) and in my rline (p sends me leaves)
  const int W = 24 + 2 + 4 * P;
  std::vector<int64_t> mine(W, -1), all((size_t)W * P);
  memcpy(mine.data(), h, sizeof h);
  mine[24] = sf->bstride;
  mine[25] = sf->rstride;
  for (size_t a = 0; a < sf->rnbr.size(); ++a) mine[26 + sf->rnbr[a]] = sf->roff[a];
  for (size_t a = 0; a < sf->snbr.size(); ++a) mine[26 + P + sf->snbr[a]] = sf->soff[a];
  for (int q = 0; q < P; ++q) {
    mine[26 + 2 * P + q] = bflag_off[q];
    mine[26 + 3 * P + q] = rflag_off[q];
  }
  SP_TRY(c->allgather_i64(mine.data(), W, all.data()));
  std::vector<uint4 *> pb(P, nullptr), pr(P, nullptr);
  std::vector<unsigned long long *> pf(P, nullptr);
  int64_t open_fail = 0;
  auto open = [&](int q) {
    if (pf[q] || open_fail) return;
    cudaIpcMemHandle_t hq[3];
    memcpy(hq, all.data() + (size_t)W * q, sizeof hq);
    void *m[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < 3 && !open_fail; ++k) {
      if (cudaIpcOpenMemHandle(&m[k], hq[k], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        open_fail = 1;
      } else {
        sf->peer_mem.push_back(m[k]);
      }
    }
    pb[q] = (uint4 *)m[0];
    pr[q] = (uint4 *)m[1];
    pf[q] = (unsigned long long *)m[2];
  };
  for (int q : sf->snbr) open(q);
  for (int q : sf->rnbr) open(q);
  int64_t v2[1] = {open_fail};
  SP_TRY(c->allreduce_max_i64(v2, 1));
  if (v2[0]) {
    note_fallback(c, "a star forest", "cudaIpcOpenMemHandle failed on some rank (peers not on one node?)");
    for (void *m : sf->peer_mem) cudaIpcCloseMemHandle(m);
    sf->peer_mem.clear();
    return SPMAT_OK;
  }
  auto at = [&](int q, int k) { return all[(size_t)W * q + k]; };
  std::vector<HaloPut> bp, rp;
  std::vector<HaloWait> bw, rw;
  sf->bchunks = sf->rchunks = 0;
  for (size_t a = 0; a < sf->snbr.size(); ++a) {  // bcast: my roots -> q's leaves; reduce: q's leaves -> me
    const int q = sf->snbr[a];
    HaloPut p{};
    p.dst = pb[q] + at(q, 26 + me);
    p.dst_stride = at(q, 24);
    p.count = sf->scount[a];
    p.root_start = sf->root_start[a] >= 0 ? sf->root_start[a] : 0;
    p.root_idx = sf->root_start[a] >= 0 ? nullptr : sf->d_root_idx.get() + sf->soff[a];
    p.my_done = sf->pflags.get() + q;
    p.cflag = at(q, 26 + 2 * P + me) >= 0 ? pf[q] + at(q, 26 + 2 * P + me) : nullptr;
    p.nchunk = p.cflag ? bulk_chunks_of(p.count) : put_chunks_of(p.count);
    sf->bchunks += p.nchunk;
    bp.push_back(p);
    HaloWait w{};
    w.peer_done = pf[q] + P + me;  // I consumed q's leaves (reduce): release q's copy of them
    rw.push_back(w);
  }
  for (size_t a = 0; a < sf->rnbr.size(); ++a) {  // bcast: q's roots -> my leaves; reduce: my leaves -> q
    const int q = sf->rnbr[a];
    HaloPut p{};
    p.dst = pr[q] + at(q, 26 + P + me);
    p.dst_stride = at(q, 25);
    p.count = sf->rcount[a];
    p.root_start = sf->leaf_start[a] >= 0 ? sf->leaf_start[a] : 0;
    p.root_idx = sf->leaf_start[a] >= 0 ? nullptr : sf->d_leaf_idx.get() + sf->roff[a];
    p.my_done = sf->pflags.get() + P + q;
    p.cflag = at(q, 26 + 3 * P + me) >= 0 ? pf[q] + at(q, 26 + 3 * P + me) : nullptr;
    p.nchunk = p.cflag ? bulk_chunks_of(p.count) : put_chunks_of(p.count);
    sf->rchunks += p.nchunk;
    rp.push_back(p);
    HaloWait w{};
    w.peer_done = pf[q] + me;  // I consumed q's roots (bcast): release q's copy of them
    bw.push_back(w);
  }
  auto upload = [&](auto &dst, const auto &src) -> int {
    SP_TRY(dst.alloc(src.size()));
    if (!src.empty()) SP_CUDA(cudaMemcpy(dst.get(), src.data(), src.size() * sizeof(src[0]), cudaMemcpyHostToDevice));
    return SPMAT_OK;
  };
  // consumer segment tables (staging order): bcast = recv order, reduce = requester-major
  std::vector<SfSeg> bs, rs;
  for (size_t a = 0; a < sf->rnbr.size(); ++a) {
    const int64_t o = bflag_off[sf->rnbr[a]];
    const int nch = o >= 0 ? bulk_chunks_of(sf->rcount[a]) : put_chunks_of(sf->rcount[a]);
    bs.push_back({sf->roff[a], sf->rcount[a], o >= 0 ? sf->pflags.get() + o : nullptr,
                  (sf->rcount[a] + nch - 1) / nch});
  }
  for (size_t a = 0; a < sf->snbr.size(); ++a) {
    const int64_t o = rflag_off[sf->snbr[a]];
    const int nch = o >= 0 ? bulk_chunks_of(sf->scount[a]) : put_chunks_of(sf->scount[a]);
    rs.push_back({sf->soff[a], sf->scount[a], o >= 0 ? sf->pflags.get() + o : nullptr,
                  (sf->scount[a] + nch - 1) / nch});
  }
  SP_TRY(upload(sf->bsegs, bs));
  SP_TRY(upload(sf->rsegs, rs));
  SP_TRY(upload(sf->bputs, bp));
  SP_TRY(upload(sf->rputs, rp));
  SP_TRY(upload(sf->bwaits, bw));
  SP_TRY(upload(sf->rwaits, rw));
  sf->nbputs = (int)bp.size();
  sf->nrputs = (int)rp.size();
  sf->nbwaits = (int)bw.size();
  sf->nrwaits = (int)rw.size();
  sf->peer = true;
  int64_t sync[1] = {0};  // every buffer zeroed and mapped before the first put
  SP_TRY(c->allreduce_max_i64(sync, 1));
  return SPMAT_OK;
}

// The puts read the epoch the previous operation's consuming kernel advanced: order the
// caller's stream after it (a no-op when that kernel ran on the same stream).  Inside a stream capture only an event recorded in the same capture can be
// waited on; an operation ended before the capture began is the caller's to order (as any
// work preceding a capture).
static int sf_after_take(sf_s *sf, cudaStream_t stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  SP_CUDA(cudaStreamIsCapturing(stream, &st));
  const bool capturing = st == cudaStreamCaptureStatusActive;
  if (capturing != sf->take_captured) return SPMAT_OK;
  SP_CUDA(cudaStreamWaitEvent(stream, sf->ev_take, 0));
  return SPMAT_OK;
}

// Bcast consumer: leaf[leaf_idx[t]] (=|+=) the value of line t of this epoch; the last CTA
// releases the staging buffer to the senders and advances the epoch.
__global__ void k_sf_bcast_take(const uint4 *__restrict__ lines, int64_t stride, const int64_t *__restrict__ lidx,
                                int64_t n, const SfSeg *__restrict__ segs, int nseg, double *__restrict__ leaf,
                                int op, const HaloWait *__restrict__ waits, int nwaits, unsigned long long *ep,
                                unsigned int *counter, int *err) {
  pdl_wait();
  const unsigned long long epoch = *ep + 1ull;
  const uint4 *gl = lines + (int64_t)(epoch & 1) * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = sf_value(gl, t, segs, nseg, epoch, err);
    const int64_t l = lidx[t];
    leaf[l] = op == SF_REPLACE ? v : __dadd_rn(leaf[l], v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      atomicExch(counter, 0u);
      for (int w = 0; w < nwaits; ++w) st_release_sys(waits[w].peer_done, epoch);
      *ep = epoch;
    }
  }
}

// Reduce consumer: k_reduce_combine's ordered combine with the received values read from this
// epoch's lines; the last CTA releases the staging buffer and advances the epoch.
__global__ void k_sf_reduce_take(const int64_t *__restrict__ roots, const int64_t *__restrict__ ptr,
                                 const int64_t *__restrict__ code, int64_t n, const uint4 *__restrict__ lines,
                                 int64_t stride, const SfSeg *__restrict__ segs, int nseg,
                                 const double *__restrict__ leaf,
                                 const int64_t *__restrict__ self_leaf, double *__restrict__ root, int op,
                                 const HaloWait *__restrict__ waits, int nwaits, unsigned long long *ep,
                                 unsigned int *counter, int *err) {
  pdl_wait();
  const unsigned long long epoch = *ep + 1ull;
  const uint4 *gl = lines + (int64_t)(epoch & 1) * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = roots[t];
    double s = root[r];
    for (int64_t k = ptr[t]; k < ptr[t + 1]; ++k) {
      const int64_t cc = code[k];
      const double v = cc >= 0 ? sf_value(gl, cc, segs, nseg, epoch, err) : leaf[self_leaf[-cc - 1]];
      s = op == SF_REPLACE ? v : __dadd_rn(s, v);
    }
    root[r] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      atomicExch(counter, 0u);
      for (int w = 0; w < nwaits; ++w) st_release_sys(waits[w].peer_done, epoch);
      *ep = epoch;
    }
  }
}

// PetscSFReduce root side: one thread per touched root applies its contributions in
// ascending (source rank, leaf index) order -- REPLACE keeps the last, SUM adds one at a time.
__global__ void k_reduce_combine(const int64_t *__restrict__ roots, const int64_t *__restrict__ ptr,
                                 const int64_t *__restrict__ code, int64_t n,
                                 const double *__restrict__ redbuf, const double *__restrict__ leaf,
                                 const int64_t *__restrict__ self_leaf, double *__restrict__ root,
                                 int op) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = roots[t];
    double s = root[r];
    for (int64_t k = ptr[t]; k < ptr[t + 1]; ++k) {
      const int64_t c = code[k];
      const double v = c >= 0 ? redbuf[c] : leaf[self_leaf[-c - 1]];
      s = op == SF_REPLACE ? v : __dadd_rn(s, v);
    }
    root[r] = s;
  }
}

// leaf -> root: pack leaves per owner (unless contiguous), NCCL send to owners / receive from
// requesters, combine on the owners -- all on the comm stream after the work on `stream`
int sf_reduce_begin_impl(sf_s *sf, const double *leaf, double *root, int op, cudaStream_t stream) {
  if (sf->pending) return fail(SPMAT_ERR_STATE, "sf_reduce_begin: an operation is already pending");
  if (op != SF_REPLACE && op != SF_SUM) return fail(SPMAT_ERR_ARG, "sf_reduce: bad op %d", op);
  spmat_comm_s *c = sf->comm;
  if (sf->peer) {  // flagged-line puts of my leaves on the caller's stream; sf_reduce_end combines
    SP_TRY(sf_after_take(sf, stream));
    SP_TRY(peer_put_launch(sf->rputs.get(), sf->nrputs, sf->rchunks, leaf, sf->d_ep.get() + 1, sf->perr.get(),
                           stream));
    sf->pending = true;
    sf->p_kind = 2;
    sf->p_root = root;
    sf->p_leaf = const_cast<double *>(leaf);
    sf->p_op = op;
    return SPMAT_OK;
  }
  cudaStream_t cs = c->comm_stream;
  SP_CUDA(cudaEventRecord(sf->ev_begin, stream));
  SP_CUDA(cudaStreamWaitEvent(cs, sf->ev_begin, 0));
  const int T = 256;
  if (sf->need_unpack_any && sf->nrecv > 0) {  // non-contiguous leaves: pack into d_recvbuf
    k_gather<<<grid_for(sf->nrecv, T, c->num_sms), T, 0, cs>>>(leaf, sf->d_leaf_idx.get(),
                                                              sf->d_recvbuf.get(), sf->nrecv);
    SP_LAUNCH();
  }
  if (c->nranks > 1 && (!sf->rnbr.empty() || !sf->snbr.empty())) {
    NcclApi *api = c->api;
    SP_NCCL(api, api->GroupStart());
    for (size_t a = 0; a < sf->snbr.size(); ++a)
      SP_NCCL(api, api->Recv(sf->d_redbuf.get() + sf->soff[a], sf->scount[a], ncclFloat64,
                             sf->snbr[a], c->nccl, cs));
    for (size_t a = 0; a < sf->rnbr.size(); ++a) {
      const double *src = sf->leaf_start[a] >= 0 ? leaf + sf->leaf_start[a]
                                                 : sf->d_recvbuf.get() + sf->roff[a];
      SP_NCCL(api, api->Send(src, sf->rcount[a], ncclFloat64, sf->rnbr[a], c->nccl, cs));
    }
    SP_NCCL(api, api->GroupEnd());
  }
  if (sf->n_touched > 0) {
    k_reduce_combine<<<grid_for(sf->n_touched, T, c->num_sms), T, 0, cs>>>(
        sf->d_red_roots.get(), sf->d_red_ptr.get(), sf->d_red_code.get(), sf->n_touched,
        sf->d_redbuf.get(), leaf, sf->d_self_leaf.get(), root, op);
    SP_LAUNCH();
  }
  SP_CUDA(cudaEventRecord(sf->ev_done, cs));
  sf->pending = true;
  sf->p_kind = 2;
  sf->p_root = root;
  sf->p_leaf = const_cast<double *>(leaf);
  sf->p_op = op;
  return SPMAT_OK;
}

int sf_reduce_end_impl(sf_s *sf, const double *leaf, double *root, int op, cudaStream_t stream) {
  if (!sf->pending || sf->p_kind != 2)
    return fail(SPMAT_ERR_STATE, "sf_reduce_end without sf_reduce_begin");
  if (root != sf->p_root || leaf != sf->p_leaf || op != sf->p_op)
    return fail(SPMAT_ERR_STATE, "sf_reduce_end: buffers or op differ from sf_reduce_begin");
  if (!sf->peer) SP_CUDA(cudaStreamWaitEvent(stream, sf->ev_done, 0));
  if (sf->peer) {  // always launched: it also ends the epoch
    const unsigned grid = grid_for(std::max<int64_t>(sf->n_touched, 1), 256, sf->comm->num_sms);
    SP_CUDA(launch_pdl(k_sf_reduce_take, grid, 256, 0, stream, (const int64_t *)sf->d_red_roots.get(),
                       (const int64_t *)sf->d_red_ptr.get(), (const int64_t *)sf->d_red_code.get(), sf->n_touched,
                       (const uint4 *)sf->rline.get(), sf->rstride, (const SfSeg *)sf->rsegs.get(),
                       (int)sf->rsegs.n, (const double *)leaf,
                       (const int64_t *)sf->d_self_leaf.get(), root, op, (const HaloWait *)sf->rwaits.get(),
                       sf->nrwaits, sf->d_ep.get() + 1, sf->pcounter.get(), sf->perr.get()));
    SP_CUDA(cudaEventRecord(sf->ev_take, stream));
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    SP_CUDA(cudaStreamIsCapturing(stream, &cst));
    sf->take_captured = cst == cudaStreamCaptureStatusActive;
  }
  sf->pending = false;
  sf->p_kind = 0;
  return SPMAT_OK;
}

int sf_begin(sf_s *sf, const double *root, double *leaf, int op, cudaStream_t stream,
             cudaEvent_t *prof) {
  if (sf->pending) return fail(SPMAT_ERR_STATE, "sf_bcast_begin: an operation is already pending");
  if (op != SF_REPLACE && op != SF_SUM) return fail(SPMAT_ERR_ARG, "sf_bcast: bad op %d", op);
  spmat_comm_s *c = sf->comm;
  const int T = 256;
  if (sf->peer) {  // flagged-line puts on the caller's stream; sf_end consumes them there too
    if (prof) SP_CUDA(cudaEventRecord(prof[0], stream));
    SP_TRY(sf_after_take(sf, stream));
    SP_TRY(peer_put_launch(sf->bputs.get(), sf->nbputs, sf->bchunks, root, sf->d_ep.get(), sf->perr.get(),
                           stream));
    if (sf->nself > 0) {
      k_scatter<<<grid_for(sf->nself, T, c->num_sms), T, 0, stream>>>(
          root, sf->d_self_root.get(), leaf, sf->d_self_leaf.get(), sf->nself, op);
      SP_LAUNCH();
    }
    if (prof) SP_CUDA(cudaEventRecord(prof[1], stream));
    sf->pending = true;
    sf->p_kind = 1;
    sf->p_root = root;
    sf->p_leaf = leaf;
    sf->p_op = op;
    return SPMAT_OK;
  }
  cudaStream_t cs = c->comm_stream;
  SP_CUDA(cudaEventRecord(sf->ev_begin, stream));
  SP_CUDA(cudaStreamWaitEvent(cs, sf->ev_begin, 0));
  if (prof) SP_CUDA(cudaEventRecord(prof[0], cs));
  if (sf->need_pack && sf->nsend > 0) {
    k_gather<<<grid_for(sf->nsend, T, c->num_sms), T, 0, cs>>>(root, sf->d_root_idx.get(),
                                                              sf->d_sendbuf.get(), sf->nsend);
    SP_LAUNCH();
  }
  if (c->nranks > 1 && (!sf->rnbr.empty() || !sf->snbr.empty())) {
    NcclApi *api = c->api;
    SP_NCCL(api, api->GroupStart());
    for (size_t a = 0; a < sf->rnbr.size(); ++a) {
      double *dst = (op == SF_REPLACE && sf->leaf_start[a] >= 0) ? leaf + sf->leaf_start[a]
                                                                  : sf->d_recvbuf.get() + sf->roff[a];
      SP_NCCL(api, api->Recv(dst, sf->rcount[a], ncclFloat64, sf->rnbr[a], c->nccl, cs));
    }
    for (size_t a = 0; a < sf->snbr.size(); ++a) {
      const double *src = sf->root_start[a] >= 0 ? root + sf->root_start[a]
                                                 : sf->d_sendbuf.get() + sf->soff[a];
      SP_NCCL(api, api->Send(src, sf->scount[a], ncclFloat64, sf->snbr[a], c->nccl, cs));
    }
    SP_NCCL(api, api->GroupEnd());
  }
  if (sf->nself > 0) {
    k_scatter<<<grid_for(sf->nself, T, c->num_sms), T, 0, cs>>>(
        root, sf->d_self_root.get(), leaf, sf->d_self_leaf.get(), sf->nself, op);
    SP_LAUNCH();
  }
  for (size_t a = 0; a < sf->rnbr.size(); ++a) {
    bool in_place = op == SF_REPLACE && sf->leaf_start[a] >= 0;
    if (in_place) continue;
    k_scatter<<<grid_for(sf->rcount[a], T, c->num_sms), T, 0, cs>>>(
        sf->d_recvbuf.get() + sf->roff[a], nullptr, leaf, sf->d_leaf_idx.get() + sf->roff[a],
        sf->rcount[a], op);
    SP_LAUNCH();
  }
  if (prof) SP_CUDA(cudaEventRecord(prof[1], cs));
  SP_CUDA(cudaEventRecord(sf->ev_done, cs));
  sf->pending = true;
  sf->p_kind = 1;
  sf->p_root = root;
  sf->p_leaf = leaf;
  sf->p_op = op;
  return SPMAT_OK;
}

int sf_end(sf_s *sf, const double *root, double *leaf, int op, cudaStream_t stream) {
  if (!sf->pending || sf->p_kind != 1) return fail(SPMAT_ERR_STATE, "sf_bcast_end without sf_bcast_begin");
  if (root != sf->p_root || leaf != sf->p_leaf || op != sf->p_op)
    return fail(SPMAT_ERR_STATE, "sf_bcast_end: buffers or op differ from sf_bcast_begin");
  if (!sf->peer) SP_CUDA(cudaStreamWaitEvent(stream, sf->ev_done, 0));
  if (sf->peer) {  // always launched: it also ends the epoch
    const unsigned grid = grid_for(std::max<int64_t>(sf->nrecv, 1), 256, sf->comm->num_sms);
    SP_CUDA(launch_pdl(k_sf_bcast_take, grid, 256, 0, stream, (const uint4 *)sf->bline.get(), sf->bstride,
                       (const int64_t *)sf->d_leaf_idx.get(), sf->nrecv, (const SfSeg *)sf->bsegs.get(),
                       (int)sf->bsegs.n, leaf, op,
                       (const HaloWait *)sf->bwaits.get(), sf->nbwaits, sf->d_ep.get(), sf->pcounter.get(),
                       sf->perr.get()));
    SP_CUDA(cudaEventRecord(sf->ev_take, stream));
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    SP_CUDA(cudaStreamIsCapturing(stream, &cst));
    sf->take_captured = cst == cudaStreamCaptureStatusActive;
  }
  sf->pending = false;
  sf->p_kind = 0;
  return SPMAT_OK;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int sf_create(spmat_comm_t comm, int64_t nroots, int64_t nleaves, const int64_t *ilocal,
              const int32_t *remote_rank, const int64_t *remote_offset, sf_t *out) {
  SP_NVTX("sf_create");
  if (!comm || !out) return fail(SPMAT_ERR_ARG, "sf_create: null argument");
  *out = nullptr;
  if (nleaves > 0 && (!remote_rank || !remote_offset))
    return fail(SPMAT_ERR_ARG, "sf_create: null leaf arrays");
  DeviceGuard g(comm->device);
  // accept host or device leaf arrays (memtype detection)
  std::vector<int64_t> il, ro;
  std::vector<int32_t> rr;
  const int64_t *pil = ilocal;
  const int32_t *prr = remote_rank;
  const int64_t *pro = remote_offset;
  if (nleaves > 0) {
    SP_CUDA(cudaDeviceSynchronize());  // device leaf arrays: the caller's kernels may still write them
    if (ilocal && is_device_ptr(ilocal)) {
      il.resize(nleaves);
      SP_CUDA(cudaMemcpy(il.data(), ilocal, nleaves * 8, cudaMemcpyDeviceToHost));
      pil = il.data();
    }
    if (is_device_ptr(remote_rank)) {
      rr.resize(nleaves);
      SP_CUDA(cudaMemcpy(rr.data(), remote_rank, nleaves * 4, cudaMemcpyDeviceToHost));
      prr = rr.data();
    }
    if (is_device_ptr(remote_offset)) {
      ro.resize(nleaves);
      SP_CUDA(cudaMemcpy(ro.data(), remote_offset, nleaves * 8, cudaMemcpyDeviceToHost));
      pro = ro.data();
    }
  }
  return sf_build(comm, nroots, nleaves, pil, prr, pro, out);
}

int sf_bcast_begin(sf_t sf, const double *rootdata, double *leafdata, int op, void *stream) {
  SP_NVTX("sf_bcast_begin");
  if (!sf) return fail(SPMAT_ERR_ARG, "sf_bcast_begin: null sf");
  if ((sf->nsend > 0 || sf->nself > 0) && !rootdata)
    return fail(SPMAT_ERR_ARG, "sf_bcast_begin: null rootdata");
  if ((sf->nrecv > 0 || sf->nself > 0) && !leafdata)
    return fail(SPMAT_ERR_ARG, "sf_bcast_begin: null leafdata");
  DeviceGuard g(sf->comm->device);
  SP_TRY(sf_ensure_peer(sf));
  return sf_begin(sf, rootdata, leafdata, op, (cudaStream_t)stream, nullptr);
}

int sf_bcast_end(sf_t sf, const double *rootdata, double *leafdata, int op, void *stream) {
  SP_NVTX("sf_bcast_end");
  if (!sf) return fail(SPMAT_ERR_ARG, "sf_bcast_end: null sf");
  DeviceGuard g(sf->comm->device);
  return sf_end(sf, rootdata, leafdata, op, (cudaStream_t)stream);
}

int sf_reduce_begin(sf_t sf, const double *leafdata, double *rootdata, int op, void *stream) {
  SP_NVTX("sf_reduce_begin");
  if (!sf) return fail(SPMAT_ERR_ARG, "sf_reduce_begin: null sf");
  if ((sf->nrecv > 0 || sf->nself > 0) && !leafdata)
    return fail(SPMAT_ERR_ARG, "sf_reduce_begin: null leafdata");
  if (sf->n_touched > 0 && !rootdata) return fail(SPMAT_ERR_ARG, "sf_reduce_begin: null rootdata");
  DeviceGuard g(sf->comm->device);
  SP_TRY(sf_ensure_peer(sf));
  return sf_reduce_begin_impl(sf, leafdata, rootdata, op, (cudaStream_t)stream);
}

int sf_reduce_end(sf_t sf, const double *leafdata, double *rootdata, int op, void *stream) {
  SP_NVTX("sf_reduce_end");
  if (!sf) return fail(SPMAT_ERR_ARG, "sf_reduce_end: null sf");
  DeviceGuard g(sf->comm->device);
  return sf_reduce_end_impl(sf, leafdata, rootdata, op, (cudaStream_t)stream);
}

int sf_get_info(sf_t sf, int64_t info[8]) {
  if (!sf || !info) return fail(SPMAT_ERR_ARG, "sf_get_info: null argument");
  info[0] = sf->nroots;
  info[1] = sf->nleaves;
  info[2] = (int64_t)sf->snbr.size();
  info[3] = (int64_t)sf->rnbr.size();
  info[4] = sf->nsend;
  info[5] = sf->nrecv;
  info[6] = sf->nself;
  info[7] = (sf->need_pack || sf->need_unpack_any) ? 1 : 0;
  return SPMAT_OK;
}

int sf_export(sf_t sf, int what, void *host_buf, int64_t cap, int64_t *len) {
  if (!sf || !len) return fail(SPMAT_ERR_ARG, "sf_export: null argument");
  std::vector<int64_t> v;
  switch (what) {
    case 0: v.assign(sf->rnbr.begin(), sf->rnbr.end()); break;
    case 1: v = sf->rcount; break;
    case 2: v = sf->h_leaf_idx; break;
    case 3: v.assign(sf->snbr.begin(), sf->snbr.end()); break;
    case 4: v = sf->scount; break;
    case 5: v = sf->h_root_idx; break;
    default: return fail(SPMAT_ERR_ARG, "sf_export: unknown what=%d", what);
  }
  *len = (int64_t)v.size();
  if (host_buf && cap > 0) memcpy(host_buf, v.data(), sizeof(int64_t) * std::min<int64_t>(cap, *len));
  return SPMAT_OK;
}

int sf_transport(sf_t sf) {
  if (!sf) return 0;
  if (sf->peer) return 2;
  return sf->comm->nranks > 1 ? 1 : 0;
}

int sf_check(sf_t sf) {
  if (!sf) return fail(SPMAT_ERR_ARG, "sf_check: null sf");
  DeviceGuard g(sf->comm->device);
  SP_CUDA(cudaDeviceSynchronize());
  if (sf->peer) {
    int e = 0;
    SP_CUDA(cudaMemcpy(&e, sf->perr.get(), sizeof(int), cudaMemcpyDeviceToHost));
    if (e) return fail(SPMAT_ERR_NCCL, "star forest over NVLink: a peer did not answer (timeout)");
  }
  return SPMAT_OK;
}

int sf_destroy(sf_t sf) {
  if (!sf) return SPMAT_OK;
  DeviceGuard g(sf->comm->device);
  // the consuming kernels run on callers' streams (and maybe inside captured graphs, where
  // ev_take was never really recorded): wait for the whole device
  cudaDeviceSynchronize();
  sf_free(sf);
  cudaGetLastError();  // teardown errors (e.g. IPC unmapping) must not surface at a later launch
  return SPMAT_OK;
}

}  // extern "C"
