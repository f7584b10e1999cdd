// comm.cu -- errors, NCCL loading, communicator and setup collectives.
//
// The communication layer replaces the paper's MPI transport ("persistent MPI sends and
// receives by default") with NCCL point-to-point on a dedicated high-priority
// CUDA stream.  NCCL calls are stream-ordered, so the host never synchronises the device
// before a send -- the MPI/GPU mismatch of P:484-509 does not arise.
#include <dlfcn.h>

#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace spmat {

static thread_local std::string g_last_error = "no error";

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int fail(int status, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

bool pdl_on() {
  static const bool on = [] {
    const char *e = getenv("SPMAT_PDL");
    return !(e && !strcmp(e, "0"));
  }();
  return on;
}

void note_fallback(const Comm *c, const char *what, const char *why) {
  if (c->rank == 0) fprintf(stderr, "libspmat: %s uses NCCL instead of NVLink peer memory: %s\n", what, why);
}

int coop_mode() {
  static const int mode = [] {
    const char *e = getenv("SPMAT_COOP");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// NCCL is loaded lazily so that single-GPU use and the symbol-export tests do not need it.
// RTLD_NOLOAD first picks up the copy torch already mapped (same soname), avoiding two
// NCCL versions in one process.
static NcclApi g_nccl;
static std::mutex g_nccl_mu;
static std::string g_nccl_err;

int nccl_api(NcclApi **out) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (!g_nccl.loaded) {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(SPMAT_ERR_NCCL, "cannot load libnccl.so.2: %s", dlerror());
#define LOADSYM(field, name)                                                   \
  *(void **)(&g_nccl.field) = dlsym(h, name);                                 \
  if (!g_nccl.field) return fail(SPMAT_ERR_NCCL, "NCCL symbol %s missing", name);
    LOADSYM(GetUniqueId, "ncclGetUniqueId");
    LOADSYM(CommInitRank, "ncclCommInitRank");
    LOADSYM(CommDestroy, "ncclCommDestroy");
    LOADSYM(CommGetAsyncError, "ncclCommGetAsyncError");
    LOADSYM(GetErrorString, "ncclGetErrorString");
    LOADSYM(GroupStart, "ncclGroupStart");
    LOADSYM(GroupEnd, "ncclGroupEnd");
    LOADSYM(Send, "ncclSend");
    LOADSYM(Recv, "ncclRecv");
    LOADSYM(AllReduce, "ncclAllReduce");
    LOADSYM(AllGather, "ncclAllGather");
#undef LOADSYM
    *(void **)(&g_nccl.CommInitRankConfig) = dlsym(h, "ncclCommInitRankConfig");  // optional
    g_nccl.loaded = true;
  }
  *out = &g_nccl;
  return SPMAT_OK;
}

int Comm::allgather_i64(const int64_t *send, int64_t count, int64_t *recv_host) {
  if (nranks == 1) {
    memcpy(recv_host, send, sizeof(int64_t) * count);
    return SPMAT_OK;
  }
  DevBuf<int64_t> d;
  SP_TRY(d.alloc((size_t)count * (nranks + 1)));
  int64_t *dsend = d.get() + (size_t)count * nranks;
  SP_CUDA(cudaMemcpyAsync(dsend, send, sizeof(int64_t) * count, cudaMemcpyHostToDevice,
                          setup_stream));
  SP_NCCL(api, api->AllGather(dsend, d.get(), count, ncclInt64, nccl, setup_stream));
  SP_CUDA(cudaMemcpyAsync(recv_host, d.get(), sizeof(int64_t) * count * nranks,
                          cudaMemcpyDeviceToHost, setup_stream));
  SP_CUDA(cudaStreamSynchronize(setup_stream));
  return SPMAT_OK;
}

int Comm::allreduce_max_i64(int64_t *v, int64_t count) {
  if (nranks == 1) return SPMAT_OK;
  DevBuf<int64_t> d;
  SP_TRY(d.alloc(count));
  SP_CUDA(cudaMemcpyAsync(d.get(), v, sizeof(int64_t) * count, cudaMemcpyHostToDevice,
                          setup_stream));
  SP_NCCL(api, api->AllReduce(d.get(), d.get(), count, ncclInt64, ncclMax, nccl, setup_stream));
  SP_CUDA(cudaMemcpyAsync(v, d.get(), sizeof(int64_t) * count, cudaMemcpyDeviceToHost,
                          setup_stream));
  SP_CUDA(cudaStreamSynchronize(setup_stream));
  return SPMAT_OK;
}

int Comm::agree(int local_status, const char *what) {
  int64_t v = local_status;
  SP_TRY(allreduce_max_i64(&v, 1));
  if (v == SPMAT_OK) return SPMAT_OK;
  if (local_status != SPMAT_OK) return local_status;
  return fail((int)v, "%s: failed on another rank (status %lld)", what, (long long)v);
}

int Comm::exchange_dev(const void *d_send, const int64_t *soff, const int64_t *scount,
                       void *d_recv, const int64_t *roff, const int64_t *rcount,
                       size_t elem_bytes, cudaStream_t stream) {
  if (nranks == 1) return SPMAT_OK;
  SP_NCCL(api, api->GroupStart());
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    if (rcount[q] > 0)
      SP_NCCL(api, api->Recv((char *)d_recv + roff[q] * elem_bytes, rcount[q] * elem_bytes,
                             ncclChar, q, nccl, stream));
    if (scount[q] > 0)
      SP_NCCL(api, api->Send((const char *)d_send + soff[q] * elem_bytes,
                             scount[q] * elem_bytes, ncclChar, q, nccl, stream));
  }
  SP_NCCL(api, api->GroupEnd());
  return SPMAT_OK;
}

}  // namespace spmat

using namespace spmat;

extern "C" {

int spmat_version(void) { return 100; }

const char *spmat_last_error(void) { return g_last_error.c_str(); }

int spmat_comm_unique_id(unsigned char id[128]) {
  if (!id) return fail(SPMAT_ERR_ARG, "spmat_comm_unique_id: null id");
  NcclApi *api;
  SP_TRY(nccl_api(&api));
  ncclUniqueId uid;
  SP_NCCL(api, api->GetUniqueId(&uid));
  static_assert(sizeof(uid) == 128, "NCCL unique id is 128 bytes");
  memcpy(id, &uid, 128);
  return SPMAT_OK;
}

int spmat_comm_create(const unsigned char *id, int nranks, int rank, int device,
                      spmat_comm_t *out) {
  if (!out) return fail(SPMAT_ERR_ARG, "spmat_comm_create: null out");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || device < 0)
    return fail(SPMAT_ERR_ARG, "spmat_comm_create: bad nranks=%d rank=%d device=%d", nranks,
                rank, device);
  if (nranks > 1 && !id) return fail(SPMAT_ERR_ARG, "spmat_comm_create: null id with nranks>1");
  int ndev = 0;
  SP_CUDA(cudaGetDeviceCount(&ndev));
  if (device >= ndev) return fail(SPMAT_ERR_ARG, "device %d >= device count %d", device, ndev);
  DeviceGuard g(device);
  spmat_comm_s *c = new spmat_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaError_t e = cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->setup_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    delete c;
    return fail(SPMAT_ERR_CUDA, "spmat_comm_create: %s", cudaGetErrorString(e));
  }
  if (nranks > 1) {
    int st = nccl_api(&c->api);
    if (st != SPMAT_OK) {
      delete c;
      return st;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, 128);
    // NCCL's kernels share the SMs with the persistent SpMV (NCCL-mode halo, COO value
    // exchange); SURVEY §2.6 proposed capping them (ncclConfig_t.maxCTAs).  Measured on B200
    // (C4, P=2, NCCL halo): cap 4 -> 0.290 ms per MatMult vs 0.276 ms uncapped, and the 32 MB
    // SF-pingpong 481 vs 107 us -- so no cap by default; SPMAT_NCCL_MAX_CTAS=n sets one
    int max_ctas = 0;
    if (const char *e = getenv("SPMAT_NCCL_MAX_CTAS")) max_ctas = atoi(e);
    ncclResult_t r;
    if (c->api->CommInitRankConfig && max_ctas > 0) {
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.maxCTAs = max_ctas;
      cfg.minCTAs = 1;
      r = c->api->CommInitRankConfig(&c->nccl, nranks, uid, rank, &cfg);
      c->nccl_max_ctas = max_ctas;
    } else {
      r = c->api->CommInitRank(&c->nccl, nranks, uid, rank);
    }
    if (r != ncclSuccess) {
      const char *msg = c->api->GetErrorString(r);
      delete c;
      return fail(SPMAT_ERR_NCCL, "ncclCommInitRank: %s", msg);
    }
    int bs = board_setup(c);
    if (bs != SPMAT_OK) {
      c->api->CommDestroy(c->nccl);
      delete c;
      return bs;
    }
  }
  *out = c;
  return SPMAT_OK;
}

int spmat_comm_check(spmat_comm_t c) {
  if (!c) return fail(SPMAT_ERR_ARG, "spmat_comm_check: null comm");
  DeviceGuard g(c->device);
  cudaError_t e = cudaStreamQuery(c->comm_stream);
  if (e != cudaSuccess && e != cudaErrorNotReady)
    return fail(SPMAT_ERR_CUDA, "comm stream: %s", cudaGetErrorString(e));
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SPMAT_ERR_CUDA, "sticky CUDA error: %s", cudaGetErrorString(e));
  if (c->nccl) {
    ncclResult_t ar;
    SP_NCCL(c->api, c->api->CommGetAsyncError(c->nccl, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
      return fail(SPMAT_ERR_NCCL, "NCCL async error: %s", c->api->GetErrorString(ar));
  }
  return SPMAT_OK;
}

int spmat_comm_destroy(spmat_comm_t c) {
  if (!c) return SPMAT_OK;
  {
    DeviceGuard g(c->device);
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    board_release(c);
    if (c->nccl) c->api->CommDestroy(c->nccl);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->setup_stream) cudaStreamDestroy(c->setup_stream);
  }
  delete c;
  return SPMAT_OK;
}

}  // extern "C"
