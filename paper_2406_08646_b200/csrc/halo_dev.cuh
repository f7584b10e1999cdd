// halo_dev.cuh -- device side of the NVLink transports: halo puts and flagged lines (halo.cu,
// spmv.cu), the fused off-diagonal tail, star-forest segments (sf.cu), the scalar board (krylov.cu).
#pragma once
#include "internal.h"
#include "ptx.cuh"

namespace spmat {

constexpr int64_t kPutChunk = 256;  // values per put warp
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

// ---- flagged lines ("LL" lines, as in NCCL's low-latency protocol)
// A double travels with its epoch: one 16-byte line {lo32, flag, hi32, flag}, written by a
// single 16-byte store and read by a single 16-byte load.  Each 8-byte half arrives whole, so
// a reader that sees both flags equal to the epoch it expects has the complete value -- no
// fence, no separate ready counter, no second NVLink round trip on the critical path.
__device__ __forceinline__ void ll_store(uint4 *p, double v, uint32_t flag) {
  const long long b = __double_as_longlong(v);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((uint32_t)b),
               "r"(flag), "r"((uint32_t)(b >> 32)), "r"(flag)
               : "memory");
}
__device__ __forceinline__ uint4 ll_load_raw(const uint4 *p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
// the value of line p once it carries `flag` (bounded spin; 0.0 and *err = 1 on timeout)
__device__ __forceinline__ double ll_load(const uint4 *p, uint32_t flag, int *err) {
  uint4 v = ll_load_raw(p);
  if (v.y != flag || v.w != flag) {
    const long long t0 = clock64();
    do {
      if (clock64() - t0 > kSpinLimit) {
        atomicExch(err, 1);
        return 0.0;
      }
      v = ll_load_raw(p);
    } while (v.y != flag || v.w != flag);
  }
  return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x));
}
__device__ __forceinline__ uint32_t ll_flag(unsigned long long epoch) { return (uint32_t)epoch; }
// finish a line already loaded as v (reload p until it carries `flag`)
__device__ __forceinline__ double ll_value(const uint4 *p, uint4 v, uint32_t flag, int *err) {
  if (v.y != flag || v.w != flag) return ll_load(p, flag, err);
  return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x));
}

// One warp moves put chunk c (global numbering over all destinations) of epoch `epoch`:
// wait until the destination has released the ghost buffer of epoch-2 (double buffering),
// then store the owned x entries as flagged lines into the destination's ghost buffer
// (epoch & 1) over NVLink.  Nothing else: the flags are the readiness signal.
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
  uint4 *dst = p.dst + (int64_t)(epoch & 1) * p.dst_stride;
  const uint32_t flag = ll_flag(epoch);
  const int64_t per = (p.count + p.nchunk - 1) / p.nchunk;
  const int64_t lo = c * per, hi = min(p.count, lo + per);
  constexpr int U = 8;
  if (p.cflag) {  // bulk: half the NVLink bytes of flagged lines, one release per chunk
    double *dd = reinterpret_cast<double *>(dst);
    const double *src = x + p.root_start;
    int64_t t0 = lo + lane;
    if (!p.root_idx && !(lo & 1) && !(((uintptr_t)src) & 15)) {  // 16-byte loads and stores
      const double2 *s2 = reinterpret_cast<const double2 *>(src + lo);
      double2 *d2 = reinterpret_cast<double2 *>(dd + lo);
      const int64_t n2 = (hi - lo) / 2;
      for (int64_t k0 = lane; k0 < n2; k0 += 32 * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = k0 + 32 * u;
          v[u] = k < n2 ? __ldg(s2 + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = k0 + 32 * u;
          if (k < n2) d2[k] = v[u];
        }
      }
      t0 = lo + 2 * n2 + lane;  // odd tail
    }
    for (; t0 < hi; t0 += 32 * U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t t = t0 + 32 * u;
        v[u] = t < hi ? __ldg(x + (p.root_idx ? p.root_idx[t] : p.root_start + t)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t t = t0 + 32 * u;
        if (t < hi) dd[t] = v[u];
      }
    }
    __threadfence_system();
    __syncwarp();
    if (lane == 0) st_release_sys(p.cflag + c, epoch);
    return;
  }
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
      if (t < hi) ll_store(dst + t, v[u], flag);
    }
  }
}

// Value t of this epoch's staging buffer gl (star forest): flagged line, or -- in a bulk
// segment -- a plain double once its chunk's flag carries the epoch.
__device__ __forceinline__ double sf_value(const uint4 *gl, int64_t t, const SfSeg *__restrict__ segs, int nseg,
                                           unsigned long long epoch, int *err) {
  int s = 0;
  while (s + 1 < nseg && t >= segs[s + 1].start) ++s;
  const SfSeg g = nseg ? segs[s] : SfSeg{0, 0, nullptr, 1};
  if (!g.cflag) return ll_load(gl + t, ll_flag(epoch), err);
  const int64_t k = t - g.start;
  spin_until_geq(g.cflag + k / g.per, epoch, err);
  return __ldcg(reinterpret_cast<const double *>(gl + g.start) + k);
}

// Off-diagonal SpMV-add with W lanes per row (W a power of two <= 32): thread t of a group
// handles row q's entries rowptr[q]+t, +W, ... and the group sums by a shuffle tree.  Every
// lane of the warp must call it (the shuffles); lanes with valid == false contribute nothing.
// W = 1 is the plain left-to-right row sum.  A lane loads the column/value of KB entries, then
// their KB ghost values, before it uses any (the work is latency-bound: a dependent ghost read
// per entry).  gl != nullptr: flagged ghost lines of `flag`; else the plain ghost vector lv.
__device__ __forceinline__ void offdiag_row_w(int64_t q, bool valid, int W,
                                              const int32_t *__restrict__ rows,
                                              const int32_t *__restrict__ rowptr,
                                              const int32_t *__restrict__ col,
                                              const double *__restrict__ val, const uint4 *gl,
                                              const double *lv, uint32_t flag, int *err, double *y,
                                              double *obuf = nullptr) {
  constexpr int KB = 4;
  const int sub = threadIdx.x & (W - 1);
  double s = 0.0;
  if (valid) {
    const int z = rowptr[q + 1];
    for (int e0 = rowptr[q] + sub; e0 < z; e0 += KB * W) {
      int c[KB];
      double v[KB];
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int e = e0 + k * W;
        c[k] = e < z ? col[e] : -1;
        v[k] = e < z ? val[e] : 0.0;
      }
      if (gl) {
        uint4 g[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k)
          if (c[k] >= 0) g[k] = ll_load_raw(gl + c[k]);
#pragma unroll
        for (int k = 0; k < KB; ++k)
          if (c[k] >= 0) s = __dadd_rn(s, __dmul_rn(v[k], ll_value(gl + c[k], g[k], flag, err)));
      } else {
        double g[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) g[k] = c[k] >= 0 ? __ldcg(lv + c[k]) : 0.0;
#pragma unroll
        for (int k = 0; k < KB; ++k)
          if (c[k] >= 0) s = __dadd_rn(s, __dmul_rn(v[k], g[k]));
      }
    }
  }
  for (int o = W >> 1; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o, W));
  if (valid && sub == 0) {
    if (obuf) {  // split tail: the sum alone, added into y after the sweep
      obuf[q] = s;
    } else {
      const int r = rows[q];
      y[r] = __dadd_rn(__ldcg(y + r), s);
    }
  }
}

// Off-diagonal SpMV-add for U rows per thread, one lane per row (rows q0, q0 + stride, ...):
// each level of the load chain (row pointers -> column/value -> ghost value, and row id -> y)
// is issued for all U rows before any of them is used, so U rows cost one chain of
// latencies instead of U.  Each row is summed left to right (the serial CSR order).
// gl != nullptr: flagged ghost lines of `flag`; else the plain ghost vector lv.
template <int U>
__device__ __forceinline__ void offdiag_rows_u(int64_t q0, int64_t stride, int64_t nro,
                                               const int32_t *__restrict__ rows,
                                               const int32_t *__restrict__ rowptr,
                                               const int32_t *__restrict__ col,
                                               const double *__restrict__ val, const uint4 *gl,
                                               const double *lv, uint32_t flag, int *err, double *y,
                                               double *obuf = nullptr) {
  int a[U], b[U];
  double s[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t q = q0 + u * stride;
    a[u] = q < nro ? rowptr[q] : 0;
    b[u] = q < nro ? rowptr[q + 1] : 0;
    s[u] = 0.0;
  }
  for (int k = 0;; ++k) {
    int c[U];
    double v[U];
    bool any = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool h = a[u] + k < b[u];
      any |= h;
      c[u] = h ? col[a[u] + k] : -1;
      v[u] = h ? val[a[u] + k] : 0.0;
    }
    if (!any) break;
    if (gl) {
      uint4 g[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) g[u] = ll_load_raw(gl + c[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) s[u] = __dadd_rn(s[u], __dmul_rn(v[u], ll_value(gl + c[u], g[u], flag, err)));
    } else {
      double g[U];
#pragma unroll
      for (int u = 0; u < U; ++u) g[u] = c[u] >= 0 ? __ldcg(lv + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) s[u] = __dadd_rn(s[u], __dmul_rn(v[u], g[u]));
    }
  }
  if (obuf) {  // split tail: the sums alone, added into y after the sweep
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q0 + u * stride < nro) obuf[q0 + u * stride] = s[u];
    return;
  }
  int r[U];
  double yo[U];
#pragma unroll
  for (int u = 0; u < U; ++u) r[u] = q0 + u * stride < nro ? rows[q0 + u * stride] : -1;
#pragma unroll
  for (int u = 0; u < U; ++u) yo[u] = r[u] >= 0 ? __ldcg(y + r[u]) : 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (r[u] >= 0) y[r[u]] = __dadd_rn(yo[u], s[u]);
}
constexpr int kRowsU = 4;  // rows per thread of the one-lane-per-row off-diagonal path

// Fused off-diagonal SpMV-add (k_spmv_tma, k_spmv_bsr3), run by the comm warps right after
// their puts: once every boundary row block is written (each of the consumer_warps consumer
// warps of every CTA adds its count of boundary blocks to tail.ctr[0]), claim chunks of off-diagonal rows from a counter and add
// A_o lvec into y, reading this epoch's flagged ghost lines.  The latency-bound chunks run
// beside the consumer warps' bandwidth-bound streaming (they used to be work items in the
// claim sequence, which idled whole CTAs on ghost-read latency: C4 P=2 kernel span 255 ->
// 251.6 us).  The last comm warp to finish releases the ghost buffer to the senders and
// resets the counters for the next launch.  Not inlined, and not called from the consumer
// path: either raised the streaming loop's register demand (C4 P=1 262 -> 302 us measured).
// Split tail (boundary rows in most row blocks, e.g. box partitions; natural claim order):
// while the consumers sweep, the comm warps compute every off-diagonal row's sum from the ghost
// lines into obuf -- no dependence on y; once all row blocks are written (every consumer warp
// adds its block count to ctr[0] when it finishes), they add obuf into y, a short
// bandwidth-bound pass instead of the whole latency-bound tail after the sweep.
static __device__ __forceinline__ bool wait_ctr(const unsigned *c, unsigned target, int *err) {
  const long long t0 = clock64();
  unsigned ns = 64;
  while (ld_acquire_gpu(c) < target) {
    if (clock64() - t0 > kSpinLimit) {
      atomicExch(err, 2);
      return false;
    }
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : ns;
  }
  return true;
}

static __device__ __noinline__ void split_tail(const SpmvTail tail, unsigned long long epoch, int *err,
                                               double *y, unsigned long long *trc, int consumer_warps) {
  const int lane = threadIdx.x & 31;
  const uint4 *gl = tail.ghost + (int64_t)(epoch & 1) * tail.ghost_stride;
  const uint32_t flag = ll_flag(epoch);
  const int w = tail.w;
  const int64_t per = w == 1 ? 32 * kRowsU : 32 / w;
  const int64_t n_chunks = (tail.n_ro + per - 1) / per;
  for (;;) {  // 1. sums
    int64_t c = 0;
    if (lane == 0) c = atomicAdd(tail.ctr + 1, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= n_chunks) break;
    if (w == 1) {
      offdiag_rows_u<kRowsU>(c * per + lane, 32, tail.n_ro, tail.rows, tail.rowptr, tail.col, tail.val, gl,
                             nullptr, flag, err, y, tail.obuf);
    } else {
      const int64_t q = c * per + lane / w;
      offdiag_row_w(q, q < tail.n_ro, w, tail.rows, tail.rowptr, tail.col, tail.val, gl, nullptr, flag, err, y,
                    tail.obuf);
    }
  }
  // 2. every warp's sums out (early: the sums take ~30 us of a ~250 us sweep).  The fence
  //    orders this warp's sums before the adds of any warp that reads them after the counter.
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    atomicAdd(tail.ctr + 3, 1u);  // comm warps whose sums are out
    wait_ctr(tail.ctr + 3, gridDim.x, err);
  }
  __syncwarp();
  // 3. y[rows[q]] += obuf[q] over static chunks of kAddU rows per lane (chunk c = CTA, + grid):
  //    the first chunk's rows and sums are loaded BEFORE the wait for the sweep, so after it
  //    only the y loads and stores remain on the critical path
  constexpr int kAddU = 10;
  const int64_t per2 = 32 * kAddU;
  const int64_t n2 = (tail.n_ro + per2 - 1) / per2;
  int r[kAddU];
  double o[kAddU], yv[kAddU];
  auto load_chunk = [&](int64_t c) {
#pragma unroll
    for (int u = 0; u < kAddU; ++u) {
      const int64_t q = c * per2 + u * 32 + lane;
      r[u] = q < tail.n_ro ? tail.rows[q] : -1;
      o[u] = q < tail.n_ro ? __ldcg(tail.obuf + q) : 0.0;
    }
  };
  int64_t c = blockIdx.x;
  if (c < n2) load_chunk(c);
  if (lane == 0) {  // every row block written
    wait_ctr(tail.ctr, (unsigned)(consumer_warps * tail.n_bblocks), err);
    if (trc) trc[4] = gtimer();
  }
  __syncwarp();
  for (; c < n2; c += gridDim.x) {
    if (c != blockIdx.x) load_chunk(c);
#pragma unroll
    for (int u = 0; u < kAddU; ++u) yv[u] = r[u] >= 0 ? __ldcg(y + r[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kAddU; ++u)
      if (r[u] >= 0) y[r[u]] = __dadd_rn(yv[u], o[u]);
  }
  __syncwarp();
  if (lane == 0) {
    if (trc) trc[5] = gtimer();
    __threadfence();
    if (atomicAdd(tail.ctr + 2, 1u) == gridDim.x - 1) {
      for (int k = 0; k < 5; ++k)
        if (k != 2) atomicExch(tail.ctr + k, 0u);
      atomicExch(tail.ctr + 2, 0u);
      __threadfence();
      for (int q = 0; q < tail.nwaits; ++q) st_release_sys(tail.waits[q].peer_done, epoch);
    }
  }
}

static __device__ __noinline__ void tail_warp(const SpmvTail tail, unsigned long long epoch, int *err,
                                              double *y, unsigned long long *trc, int consumer_warps) {
  const int lane = threadIdx.x & 31;
  if (tail.obuf) {  // split tail: sums first (ghost lines only), the y adds after the sweep
    split_tail(tail, epoch, err, y, trc, consumer_warps);
    return;
  }
  if (lane == 0) {
    // short backoff: with box partitions 444 warps may wait the whole sweep here
    const unsigned target = (unsigned)(consumer_warps * tail.n_bblocks);
    const long long t0 = clock64();
    unsigned ns = 64;
    while (ld_acquire_gpu(tail.ctr) < target) {
      if (clock64() - t0 > kSpinLimit) {
        atomicExch(err, 2);
        break;
      }
      __nanosleep(ns);
      ns = ns < 256 ? 2 * ns : ns;
    }
    if (trc) trc[4] = gtimer();
  }
  __syncwarp();
  const uint4 *gl = tail.ghost + (int64_t)(epoch & 1) * tail.ghost_stride;
  const uint32_t flag = ll_flag(epoch);
  const int w = tail.w;
  const int64_t per = w == 1 ? 32 * kRowsU : 32 / w;  // rows per chunk
  const int64_t n_chunks = (tail.n_ro + per - 1) / per;
  for (;;) {
    int64_t c = 0;
    if (lane == 0) c = atomicAdd(tail.ctr + 1, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= n_chunks) break;
    if (w == 1) {
      offdiag_rows_u<kRowsU>(c * per + lane, 32, tail.n_ro, tail.rows, tail.rowptr, tail.col, tail.val, gl,
                             nullptr, flag, err, y);
    } else {
      const int64_t q = c * per + lane / w;
      offdiag_row_w(q, q < tail.n_ro, w, tail.rows, tail.rowptr, tail.col, tail.val, gl, nullptr, flag, err, y);
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (trc) trc[5] = gtimer();
    __threadfence();
    // every warp stops claiming before it arrives here, so the last arrival may reset
    if (atomicAdd(tail.ctr + 2, 1u) == gridDim.x - 1) {
      atomicExch(tail.ctr, 0u);
      atomicExch(tail.ctr + 1, 0u);
      atomicExch(tail.ctr + 2, 0u);
      __threadfence();
      for (int q = 0; q < tail.nwaits; ++q) st_release_sys(tail.waits[q].peer_done, epoch);
    }
  }
}


}  // namespace spmat
