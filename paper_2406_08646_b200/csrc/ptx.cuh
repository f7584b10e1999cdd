// ptx.cuh -- inline-PTX helpers for sm_100a kernels (mbarrier, bulk copies, loads).
#pragma once
#include <stdint.h>

namespace spmat {

// Programmatic dependent launch: pdl_wait() blocks until the preceding grid of the stream has
// completed and its writes are visible (a no-op for a kernel launched without the attribute).
// Every kernel launched with launch_pdl calls it in every thread before it touches memory
// another kernel wrote -- so completion stays transitive along the stream.  No kernel calls
// griddepcontrol.launch_dependents early: measured on B200, letting the next grid's CTAs
// occupy SMs while a bandwidth-bound grid drains cost more (CG on a 3 M-row matrix: 96 ->
// 115 us per iteration) than the launch overlap saved; the implicit trigger at exit still
// takes ~2.5 us off each iteration.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// The one exception (bsr.cu): the 3x3 block SpMV triggers at entry when the next kernel is the
// block off-diagonal SpMV-add, which is sized to fit beside it on every SM and does all its
// latency-bound reads before its pdl_wait.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
// global -> shared bulk copy on the TMA engine, completion counted on an mbarrier.
// L2 evict_first: val/col/rowptr are streamed once; x should stay resident in L2.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         unsigned long long *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_stream(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// ------------------------------------------------------------------ TMA-fed row kernel
// Persistent, warp-specialised CTAs: warp kConsumerWarps is the producer, warp
// kConsumerWarps + 1 the comm warp (multi-GPU: stores this rank's boundary x entries into the
// neighbours' ghost vectors over NVLink while the SpMV streams -- halo.cu), the rest consume.  The producer claims row blocks from a global counter (dynamic scheduling: CTAs
// that start late -- e.g. behind an NCCL kernel -- simply take fewer blocks; blocks are
// claimed in increasing order, so all CTAs sweep the matrix together and a 3D stencil's
// +-plane x window stays L2-resident), and for each claimed block issues three bulk copies
// (val, col, row pointers) into a free stage, completing on that stage's `full` mbarrier.
// Consumers wait on `full`, compute W-lane row dot products straight out of shared memory,
// and release the stage on its `empty` mbarrier (one arrive per consumer warp).  A stage
// header with r0 = -1 ends the loop.  The last CTA to run out of blocks resets the counter
// for the next launch (stream order makes that safe; CUDA-graph safe too).
}  // namespace spmat
