// Streaming-read ceiling probes (lab tool, not product): TMA bulk ring vs cp.async
// ring vs plain loads, minimal consumer work (xor), to size the select kernels.
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  } while (!ok);
}
// TMA ring: 1 producer warp + W consumer warps; stage = SB bytes, S stages.
__global__ void tma_ring(const uint8_t* __restrict__ in, int64_t bytes, int SB, int S, int W, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + (size_t)S * SB);
  unsigned long long* empty = full + S;
  if (threadIdx.x < S) { mbar_init(full + threadIdx.x, 1); mbar_init(empty + threadIdx.x, W); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int64_t nst = bytes / SB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == W) {  // producer
    uint32_t seq = 0;
    for (int64_t st = blockIdx.x; st < nst; st += gridDim.x, ++seq) {
      const uint32_t slot = seq % S;
      if (seq >= (uint32_t)S) mbar_wait(empty + slot, ((seq / S) - 1) & 1);
      if (lane == 0) { mbar_expect_tx(full + slot, SB); bulk_g2s(sm + (size_t)slot * SB, in + st * SB, SB, full + slot); }
      __syncwarp();
    }
    return;
  }
  unsigned acc = 0;
  uint32_t seq = 0;
  const int per_warp = SB / 16 / W;
  for (int64_t st = blockIdx.x; st < nst; st += gridDim.x, ++seq) {
    const uint32_t slot = seq % S;
    mbar_wait(full + slot, (seq / S) & 1);
    const uint4* stage = reinterpret_cast<const uint4*>(sm + (size_t)slot * SB) + warp * per_warp;
    for (int q = lane; q < per_warp; q += 32) { uint4 v = stage[q]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + slot);
  }
  if (acc == 0x12345678u) out[0] = acc;
}
// cp.async (LDGSTS) ring: every thread copies its 16 B of each stage, D stages deep.
__global__ void cpasync_ring(const uint8_t* __restrict__ in, int64_t bytes, int D, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int T = blockDim.x;
  const int64_t SB = (int64_t)T * 16;
  const int64_t nst = bytes / SB;
  unsigned acc = 0;
  int64_t st = blockIdx.x;
  int issued = 0;
  // prologue
  for (int d = 0; d < D; ++d) {
    const int64_t s2 = st + (int64_t)d * gridDim.x;
    if (s2 < nst) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + ((size_t)d * T + threadIdx.x) * 16)), "l"(in + s2 * SB + threadIdx.x * 16) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int slot = 0;
  for (; st < nst; st += gridDim.x) {
    asm volatile("cp.async.wait_group %0;" ::"n"(7) : "memory");  // D must be 8
    const uint4 v = *reinterpret_cast<const uint4*>(sm + ((size_t)slot * T + threadIdx.x) * 16);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
    const int64_t s2 = st + (int64_t)D * gridDim.x;
    if (s2 < nst) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + ((size_t)slot * T + threadIdx.x) * 16)), "l"(in + s2 * SB + threadIdx.x * 16) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    slot = (slot + 1) % D;
    ++issued;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (acc == 0x12345678u) out[0] = acc;
}
extern "C" float probe_tma(const void* in, int64_t bytes, int SB, int S, int W, int ctas_per_sm, int iters) {
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned* out; cudaMalloc(&out, 4);
  size_t smem = (size_t)S * SB + 2 * S * 8;
  if (cudaFuncSetAttribute(tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  tma_ring<<<sms * ctas_per_sm, (W + 1) * 32, smem>>>((const uint8_t*)in, bytes, SB, S, W, out);
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) tma_ring<<<sms * ctas_per_sm, (W + 1) * 32, smem>>>((const uint8_t*)in, bytes, SB, S, W, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  if (cudaGetLastError() != cudaSuccess) return -2;
  float ms; cudaEventElapsedTime(&ms, a, b); cudaFree(out); return ms / iters;
}
extern "C" float probe_cpasync(const void* in, int64_t bytes, int T, int ctas_per_sm, int iters) {
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned* out; cudaMalloc(&out, 4);
  const int D = 8;
  size_t smem = (size_t)D * T * 16;
  if (cudaFuncSetAttribute(cpasync_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cpasync_ring<<<sms * ctas_per_sm, T, smem>>>((const uint8_t*)in, bytes, D, out);
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) cpasync_ring<<<sms * ctas_per_sm, T, smem>>>((const uint8_t*)in, bytes, D, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  if (cudaGetLastError() != cudaSuccess) return -2;
  float ms; cudaEventElapsedTime(&ms, a, b); cudaFree(out); return ms / iters;
}
