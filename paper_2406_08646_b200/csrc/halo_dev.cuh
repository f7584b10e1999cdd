// halo_dev.cuh -- device side of the NVLink halo (shared by halo.cu and spmv.cu).
#pragma once
#include "internal.h"

namespace spmat {

constexpr int64_t kPutChunk = 1024;  // values per put warp
constexpr long long kSpinLimit = 20LL * 2000 * 1000 * 1000;  // ~20 s of SM clocks

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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

// bounded spin; returns false on timeout (and records it in *err)
__device__ __forceinline__ bool spin_until_geq(const unsigned long long *flag,
                                               unsigned long long target, int *err) {
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

// One warp moves put chunk c (global numbering over all destinations) of epoch `epoch`:
// wait until the destination has released the ghost buffer of epoch-2 (double buffering),
// store the owned x entries into the destination's lvec buffer (epoch & 1) over NVLink,
// fence at system scope, then bump the destination's ready counter.
__device__ __forceinline__ void halo_put_warp(const HaloPut *__restrict__ puts, int nputs, int c,
                                              const double *__restrict__ x,
                                              unsigned long long epoch, int *err) {
  const int lane = threadIdx.x & 31;
  int d = 0;
  while (d < nputs && c >= puts[d].nchunk) c -= puts[d++].nchunk;
  if (d >= nputs) return;
  const HaloPut p = puts[d];
  int ok = 1;
  if (lane == 0 && epoch > 2) ok = spin_until_geq(p.my_done, epoch - 2, err) ? 1 : 0;
  ok = __shfl_sync(0xffffffffu, ok, 0);
  if (!ok) return;
  double *dst = p.dst + (int64_t)(epoch & 1) * p.dst_stride;
  const int64_t per = (p.count + p.nchunk - 1) / p.nchunk;
  const int64_t lo = c * per, hi = min(p.count, lo + per);
  constexpr int U = 8;
  for (int64_t t0 = lo + lane; t0 < hi; t0 += 32 * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + 32 * u;
      v[u] = t < hi ? __ldg(x + (p.root_idx ? p.root_idx[t] : p.root_start + t)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + 32 * u;
      if (t < hi) dst[t] = v[u];
    }
  }
  __threadfence_system();
  __syncwarp();
  if (lane == 0) red_release_sys_add(p.peer_ready, 1ull);
}

}  // namespace spmat
