// Read-bandwidth ceiling probe (lab tool, not product): how fast can a kernel
// stream-read HBM with the same load instruction the select kernels use?
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_plain(const uint4* p) { return __ldg(p); }
template <int U, bool NA>
__global__ void read_kernel(const uint4* __restrict__ in, int64_t nvec, unsigned* out) {
  unsigned acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < nvec; base += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t g = base + (int64_t)u * blockDim.x;
      v[u] = g < nvec ? (NA ? ld_stream(in + g) : ld_plain(in + g)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
extern "C" float probe(const void* in, int64_t bytes, int variant, int blocks_per_sm, int threads, int iters) {
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned* out; cudaMalloc(&out, 4);
  const int64_t nvec = bytes / 16;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto launch = [&]() {
    const int grid = sms * blocks_per_sm;
    switch (variant) {
      case 0: read_kernel<4, true><<<grid, threads>>>((const uint4*)in, nvec, out); break;
      case 1: read_kernel<8, true><<<grid, threads>>>((const uint4*)in, nvec, out); break;
      case 2: read_kernel<4, false><<<grid, threads>>>((const uint4*)in, nvec, out); break;
      case 3: read_kernel<16, true><<<grid, threads>>>((const uint4*)in, nvec, out); break;
      default: read_kernel<2, true><<<grid, threads>>>((const uint4*)in, nvec, out); break;
    }
  };
  launch();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return ms / iters;
}
