// Green-context probe (lab tool, not product): can the streaming kernels and the
// commitment run on disjoint SM partitions of one B200 (driver green contexts), with
// runtime-API launches on the green contexts' streams, and how fast does a chunked
// streaming read run on the larger partition?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o greenctx tools/lab/greenctx.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <set>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("%s -> %s\n", #x, s_); exit(1); } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r_)); exit(1); } } while (0)

__global__ void smid_kernel(int* out) {
  if (threadIdx.x == 0) {
    int s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    out[blockIdx.x] = s;
  }
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// one warp per chunk, register double buffer (the select kernels' access pattern)
__global__ void chunked_warp(const uint4* __restrict__ in, int64_t nchunks, int chunk_vec, unsigned* out) {
  unsigned acc = 0;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < nchunks; j += nw) {
    const uint4* c = in + j * chunk_vec;
    uint4 a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { const int g = lane + u * 32; a[u] = g < chunk_vec ? ld_stream(c + g) : make_uint4(0, 0, 0, 0); }
    for (int base = lane; base < chunk_vec; base += 256) {
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int g = base + 256 + u * 32; b[u] = g < chunk_vec ? ld_stream(c + g) : make_uint4(0, 0, 0, 0); }
#pragma unroll
      for (int u = 0; u < 8; ++u) { acc ^= a[u].x ^ a[u].y ^ a[u].z ^ a[u].w; a[u] = b[u]; }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
  const int small_sms = argc > 1 ? atoi(argv[1]) : 24;
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource part, rest;
  unsigned int ngroups = 1;
  CK(cuDevSmResourceSplitByCount(&part, &ngroups, &all, &rest, 0, small_sms));
  printf("SMs: all %u, small %u, rest %u\n", all.sm.smCount, part.sm.smCount, rest.sm.smCount);
  CUdevResourceDesc d_small, d_rest;
  CK(cuDevResourceGenerateDesc(&d_small, &part, 1));
  CK(cuDevResourceGenerateDesc(&d_rest, &rest, 1));
  CUgreenCtx g_small, g_rest;
  CK(cuGreenCtxCreate(&g_small, d_small, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&g_rest, d_rest, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s_small, s_rest;
  CK(cuGreenCtxStreamCreate(&s_small, g_small, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&s_rest, g_rest, CU_STREAM_NON_BLOCKING, 0));

  // runtime launches on the green streams; memory from the primary context
  int* ids;
  RK(cudaMalloc(&ids, 4096 * sizeof(int)));
  std::set<int> a_set, b_set;
  std::vector<int> h(4096);
  smid_kernel<<<2048, 32, 0, (cudaStream_t)s_small>>>(ids);
  RK(cudaGetLastError());
  RK(cudaStreamSynchronize((cudaStream_t)s_small));
  RK(cudaMemcpy(h.data(), ids, 2048 * sizeof(int), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 2048; ++i) a_set.insert(h[i]);
  smid_kernel<<<4096, 32, 0, (cudaStream_t)s_rest>>>(ids);
  RK(cudaGetLastError());
  RK(cudaStreamSynchronize((cudaStream_t)s_rest));
  RK(cudaMemcpy(h.data(), ids, 4096 * sizeof(int), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 4096; ++i) b_set.insert(h[i]);
  int overlap = 0;
  for (int s : a_set) overlap += b_set.count(s);
  printf("distinct SMs used: small stream %zu, rest stream %zu, overlap %d\n", a_set.size(), b_set.size(), overlap);

  // streaming read on the rest partition vs the whole GPU
  const int64_t chunk_bytes = 32 * 5120 * 2, nchunks = 65536;
  const int64_t bytes = chunk_bytes * nchunks;
  uint4* buf;
  unsigned* o;
  RK(cudaMalloc(&buf, bytes));
  RK(cudaMalloc(&o, 4));
  RK(cudaMemset(buf, 1, bytes));
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  for (int cfg = 0; cfg < 2; ++cfg) {
    cudaStream_t st = cfg == 0 ? (cudaStream_t)0 : (cudaStream_t)s_rest;
    const int sms = cfg == 0 ? (int)all.sm.smCount : (int)rest.sm.smCount;
    for (int per : {16, 18, 20}) {
      const int grid = sms * per;
      chunked_warp<<<grid, 32, 0, st>>>(buf, nchunks, (int)(chunk_bytes / 16), o);
      RK(cudaEventRecord(e0, st));
      for (int it = 0; it < 5; ++it) chunked_warp<<<grid, 32, 0, st>>>(buf, nchunks, (int)(chunk_bytes / 16), o);
      RK(cudaEventRecord(e1, st));
      RK(cudaEventSynchronize(e1));
      float ms;
      RK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= 5;
      printf("%s (%d SMs) x %d warps/SM: %.3f ms  %.0f GB/s\n", cfg == 0 ? "whole GPU" : "rest partition", sms, per, ms,
             bytes / ms / 1e6);
    }
  }
  return 0;
}
