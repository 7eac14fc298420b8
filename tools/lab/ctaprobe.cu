// CTA-ring read probe (lab tool, not product): one CTA streams whole 320 KiB chunks
// (configuration 2's chunk) through a TMA bulk-copy ring in shared memory, the way a
// TMA-fed select kernel would; consumer warps read every stage with LDS.128 and spend an
// artificial per-chunk tail (spin) after the last stage of each chunk while the producer
// keeps prefetching the next chunk.  Compared with the product's per-warp LDG pattern.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ctaprobe tools/lab/ctaprobe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n .reg .pred p;\n W_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(sa(b)),
               "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(bar)), "l"(pol) : "memory");
}

// Warp specialisation: warp 0 = producer (lane 0 issues), warps 1..W consume.
// Chunks are claimed dynamically by the producer (atomicAdd) and announced through a
// per-stage chunk id in shared memory.
template <int NST>
__global__ void ring_chunks(const uint8_t* __restrict__ in, int64_t nchunks, int chunk_bytes, int SB, int tail_cycles,
                            unsigned long long* counter, unsigned* out, int evict_first) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[NST], empty[NST];
  __shared__ int64_t stage_chunk[NST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwc = (blockDim.x >> 5) - 1;  // consumer warps
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nwc); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int per = chunk_bytes / SB;
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int64_t j = blockIdx.x;
      int q = 0;
      for (int64_t t = 0;; ++t) {
        if (q == per) {
          q = 0;
          j = gridDim.x + (int64_t)atomicAdd(counter, 1ull);
        }
        const int s = (int)(t % NST);
        if (t >= NST) mbar_wait(&empty[s], (unsigned)(((t / NST) - 1) & 1));
        if (j >= nchunks) {
          stage_chunk[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        stage_chunk[s] = j;
        mbar_expect_tx(&full[s], SB);
        const uint8_t* src = in + j * (int64_t)chunk_bytes + (int64_t)q * SB;
        if (evict_first) bulk_g2s_hint(sm + (size_t)s * SB, src, SB, &full[s], pol);
        else bulk_g2s(sm + (size_t)s * SB, src, SB, &full[s]);
        ++q;
      }
    }
    return;
  }
  unsigned acc = 0;
  const int cw = warp - 1;
  int q = 0;
  for (int64_t t = 0;; ++t) {
    const int s = (int)(t % NST);
    mbar_wait(&full[s], (unsigned)((t / NST) & 1));
    if (stage_chunk[s] < 0) break;
    const uint4* v = reinterpret_cast<const uint4*>(sm + (size_t)s * SB);
    for (int i = cw * 32 + lane; i < SB / 16; i += nwc * 32) {
      const uint4 x = v[i];
      acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++q == per) {
      q = 0;
      if (tail_cycles) {  // the chunk tail: final sort + merge, no loads
        const long long t0 = clock64();
        while (clock64() - t0 < tail_cycles) acc += (unsigned)t0;
      }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// The product's pattern: one warp per chunk, one-warp CTAs, 8 x 16 B per lane double-buffered.
__global__ void chunk_ldg(const uint4* __restrict__ in, int64_t nchunks, int chunk_vec, int tail_cycles, unsigned* out) {
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
    if (tail_cycles) {
      const long long t0 = clock64();
      while (clock64() - t0 < tail_cycles) acc += (unsigned)t0;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t chunk_bytes = 327680;
  const int64_t nchunks = argc > 1 ? atoll(argv[1]) : 65536;  // configuration 2: 21.5 GB
  const size_t bytes = (size_t)nchunks * chunk_bytes;
  uint8_t* d;
  unsigned* out;
  unsigned long long* ctr;
  RK(cudaMalloc(&d, bytes));
  RK(cudaMalloc(&out, 4));
  RK(cudaMalloc(&ctr, 8));
  RK(cudaMemset(d, 1, bytes));
  int sms;
  RK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
      cudaMemset(ctr, 0, 8);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    return best;
  };
  const int tails[] = {0, 4000, 12000};  // cycles at ~1.9 GHz: 0, ~2, ~6 us
  for (int tail : tails) {
    {
      float ms = timeit([&] { chunk_ldg<<<sms * 18, 32>>>((const uint4*)d, nchunks, (int)(chunk_bytes / 16), tail, out); });
      printf("chunk LDG 18 warps/SM                     tail %5d: %.3f ms %6.0f GB/s\n", tail, ms, bytes / ms / 1e6);
    }
    struct Cfg { int nst, sb, warps, ctas, ef; } cfgs[] = {
        {4, 32768, 8, 1, 0}, {6, 32768, 8, 1, 0}, {5, 32768, 16, 1, 0}, {6, 16384, 8, 1, 0}, {8, 16384, 8, 1, 0},
        {10, 16384, 16, 1, 0}, {3, 32768, 8, 2, 0}, {4, 16384, 8, 2, 0}, {6, 16384, 4, 2, 0}, {4, 32768, 8, 1, 1},
        {6, 16384, 8, 1, 1}, {3, 32768, 8, 2, 1}};
    for (const Cfg& c : cfgs) {
      const size_t smem = (size_t)c.nst * c.sb;
      float ms = 0;
      auto run = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        ms = timeit([&] { kern<<<sms * c.ctas, 32 * (c.warps + 1), smem>>>(d, nchunks, (int)chunk_bytes, c.sb, tail, ctr, out, c.ef); });
      };
      switch (c.nst) {
        case 3: run(ring_chunks<3>); break;
        case 4: run(ring_chunks<4>); break;
        case 5: run(ring_chunks<5>); break;
        case 6: run(ring_chunks<6>); break;
        case 8: run(ring_chunks<8>); break;
        default: run(ring_chunks<10>); break;
      }
      cudaError_t er = cudaGetLastError();
      printf("ring %2d x %5d B, %2d cons warps, %d CTA/SM%s tail %5d: %.3f ms %6.0f GB/s %s\n", c.nst, c.sb, c.warps,
             c.ctas, c.ef ? " evict_first" : "            ", tail, ms, bytes / ms / 1e6,
             er == cudaSuccess ? "" : cudaGetErrorString(er));
    }
  }
  return 0;
}
