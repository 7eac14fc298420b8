// Read-bandwidth probe (lab tool, not product): how fast can a B200 stream HBM with
// (A) per-thread 128-bit non-allocating loads (the select/verify kernels' pattern) versus
// (B) TMA bulk copies (cp.async.bulk global -> shared, mbarrier ring) consumed from shared
// memory?  Answers whether a TMA-staged select could beat the ~7.3 TB/s LDG read ceiling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw tools/lab/readbw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int U>
__global__ void ldg_read(const uint4* __restrict__ in, int64_t n_vec, unsigned* out) {
  unsigned acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x) * U + threadIdx.x; base < n_vec; base += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      v[u] = i < n_vec ? ld_stream(in + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(bar)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

// One CTA: thread 0 issues bulk copies of STAGE bytes into a ring of NST stages; all warps
// consume each stage (XOR) and arrive on an "empty" barrier before it is refilled.
template <int NST>
__global__ void tma_read(const uint8_t* __restrict__ in, int64_t n_tiles, int stage_bytes, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[NST], empty[NST];
  const int nthr = blockDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nthr); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // tiles of this CTA: blockIdx.x, +gridDim.x, ...
  const int64_t my = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int64_t t = 0; t < my && t < NST; ++t) {
      mbar_expect_tx(&full[t], stage_bytes);
      bulk_g2s(sm + t * stage_bytes, in + (blockIdx.x + t * gridDim.x) * (int64_t)stage_bytes, stage_bytes, &full[t]);
    }
  }
  unsigned acc = 0;
  for (int64_t t = 0; t < my; ++t) {
    const int s = (int)(t % NST);
    const unsigned ph = (unsigned)((t / NST) & 1);
    mbar_wait(&full[s], ph);
    const uint4* v = reinterpret_cast<const uint4*>(sm + s * stage_bytes);
    for (int i = threadIdx.x; i < stage_bytes / 16; i += nthr) {
      const uint4 x = v[i];
      acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&empty[s])));
    if (threadIdx.x == 0 && t + NST < my) {
      mbar_wait(&empty[s], ph);
      mbar_expect_tx(&full[s], stage_bytes);
      bulk_g2s(sm + s * stage_bytes, in + (blockIdx.x + (t + NST) * gridDim.x) * (int64_t)stage_bytes, stage_bytes,
               &full[s]);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// The select kernels' shape: one warp per 320 KiB chunk, one-warp CTAs.
// (C) register double buffer of U x 32 x 16 B loads (the product's pattern).
__global__ void chunk_ldg(const uint4* __restrict__ in, int64_t nchunks, int chunk_vec, unsigned* out) {
  unsigned acc = 0;
  const int lane = threadIdx.x & 31;
  for (int64_t j = blockIdx.x; j < nchunks; j += gridDim.x) {
    const uint4* c = in + j * chunk_vec;
    uint4 a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = ld_stream(c + lane + u * 32);
    for (int base = 0; base < chunk_vec; base += 256) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int g = base + 256 + lane + u * 32;
        b[u] = g < chunk_vec ? ld_stream(c + g) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { acc ^= a[u].x ^ a[u].y ^ a[u].z ^ a[u].w; a[u] = b[u]; }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// (D) a per-warp ring of NST bulk copies of SB bytes, issued by lane 0, read with LDS.128.
template <int NST>
__global__ void chunk_tma(const uint8_t* __restrict__ in, int64_t nchunks, int chunk_bytes, int SB, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[NST];
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const int per_chunk = chunk_bytes / SB;
  const int64_t my_chunks = (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t total = my_chunks * per_chunk;  // stages over all of this CTA's chunks
  auto src_of = [&](int64_t t) {
    const int64_t cj = blockIdx.x + (t / per_chunk) * gridDim.x;
    return in + cj * (int64_t)chunk_bytes + (t % per_chunk) * (int64_t)SB;
  };
  if (lane == 0)
    for (int64_t t = 0; t < total && t < NST; ++t) {
      mbar_expect_tx(&full[t], SB);
      bulk_g2s(sm + t * SB, src_of(t), SB, &full[t]);
    }
  unsigned acc = 0;
  for (int64_t t = 0; t < total; ++t) {
    const int s = (int)(t % NST);
    mbar_wait(&full[s], (unsigned)((t / NST) & 1));
    const uint4* v = reinterpret_cast<const uint4*>(sm + s * SB);
    for (int i = lane; i < SB / 16; i += 32) {
      const uint4 x = v[i];
      acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    __syncwarp();
    if (lane == 0 && t + NST < total) {
      mbar_expect_tx(&full[s], SB);
      bulk_g2s(sm + s * SB, src_of(t + NST), SB, &full[s]);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int sms = 0;
  RK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t bytes = 8ll << 30;  // 8 GiB: far above L2
  uint8_t* buf;
  unsigned* o;
  RK(cudaMalloc(&buf, bytes));
  RK(cudaMalloc(&o, 4));
  RK(cudaMemset(buf, 1, bytes));
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  auto time_it = [&](auto launch) -> float {
    launch();
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
  };
  const int64_t nvec = bytes / 16;
  for (int per : {8, 16, 32}) {
    for (int thr : {256, 512}) {
      const int grid = sms * per * 256 / thr;
      float ms = time_it([&] { ldg_read<8><<<grid, thr>>>(reinterpret_cast<const uint4*>(buf), nvec, o); });
      RK(cudaGetLastError());
      printf("LDG   U=8  %3d thr x %5d CTAs: %.3f ms  %.0f GB/s\n", thr, grid, ms, bytes / ms / 1e6);
    }
  }
  for (int stage : {16384, 32768}) {
    for (int nst : {4, 6}) {
      for (int ctas : {1, 2}) {
        const int smem = stage * nst;
        if (smem * ctas > 220 * 1024) continue;
        const int64_t tiles = bytes / stage;
        float ms = -1;
        if (nst == 4) {
          RK(cudaFuncSetAttribute(tma_read<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          ms = time_it([&] { tma_read<4><<<sms * ctas, 256, smem>>>(buf, tiles, stage, o); });
        } else {
          RK(cudaFuncSetAttribute(tma_read<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          ms = time_it([&] { tma_read<6><<<sms * ctas, 256, smem>>>(buf, tiles, stage, o); });
        }
        RK(cudaGetLastError());
        RK(cudaDeviceSynchronize());
        printf("TMA   stage %5d x %d, %d CTA/SM: %.3f ms  %.0f GB/s\n", stage, nst, ctas, ms, bytes / ms / 1e6);
      }
    }
  }
  const int chunk_bytes = 32 * 5120 * 2;
  const int64_t nchunks = bytes / chunk_bytes;
  const int64_t cbytes = nchunks * chunk_bytes;
  for (int per : {16, 18, 20}) {
    float ms = time_it([&] { chunk_ldg<<<sms * per, 32>>>(reinterpret_cast<const uint4*>(buf), nchunks, chunk_bytes / 16, o); });
    RK(cudaGetLastError());
    printf("chunk LDG  %2d warps/SM: %.3f ms  %.0f GB/s\n", per, ms, cbytes / ms / 1e6);
  }
  struct Cfg { int per, nst, sb; };
  for (Cfg c : {Cfg{8, 4, 4096}, Cfg{12, 3, 4096}, Cfg{16, 2, 4096}, Cfg{12, 4, 4096}, Cfg{6, 4, 8192},
                Cfg{8, 3, 8192}, Cfg{4, 4, 16384}, Cfg{16, 3, 4096}, Cfg{8, 2, 16384}}) {
    const int smem = c.nst * c.sb;
    if (smem * c.per > 220 * 1024) continue;
    float ms;
    if (c.nst == 2) {
      RK(cudaFuncSetAttribute(chunk_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      ms = time_it([&] { chunk_tma<2><<<sms * c.per, 32, smem>>>(buf, nchunks, chunk_bytes, c.sb, o); });
    } else if (c.nst == 3) {
      RK(cudaFuncSetAttribute(chunk_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      ms = time_it([&] { chunk_tma<3><<<sms * c.per, 32, smem>>>(buf, nchunks, chunk_bytes, c.sb, o); });
    } else {
      RK(cudaFuncSetAttribute(chunk_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      ms = time_it([&] { chunk_tma<4><<<sms * c.per, 32, smem>>>(buf, nchunks, chunk_bytes, c.sb, o); });
    }
    RK(cudaGetLastError());
    RK(cudaDeviceSynchronize());
    printf("chunk TMA  %2d warps/SM, %d x %5d B: %.3f ms  %.0f GB/s\n", c.per, c.nst, c.sb, ms, cbytes / ms / 1e6);
  }
  return 0;
}
