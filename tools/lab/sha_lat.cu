// SHA-256 compression latency probe (lab tool, not product): cycles per 64-byte block for
// one chain per thread with one warp per SM sub-partition -- the exact-mode chain kernel's
// situation (a chain is serial; rollouts are the only parallelism).
//   (a) the product's round loop (message schedule computed inline);
//   (b) message schedule expanded before the rounds (W[64] + K folded);
//   (c) two independent chains interleaved per thread (the ILP ceiling).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sha_lat tools/lab/sha_lat.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__constant__ uint32_t K[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void compress_inline(uint32_t (&st)[8], uint32_t (&w)[16]) {
  uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
  for (int t = 0; t < 64; ++t) {
    uint32_t wt;
    if (t < 16) {
      wt = w[t];
    } else {
      const uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
      const uint32_t s0 = rotr(w15, 7) ^ rotr(w15, 18) ^ (w15 >> 3);
      const uint32_t s1 = rotr(w2, 17) ^ rotr(w2, 19) ^ (w2 >> 10);
      wt = w[t & 15] = w[t & 15] + s0 + w[(t - 7) & 15] + s1;
    }
    const uint32_t t1 = h + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[t] + wt;
    const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
    h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

__device__ __forceinline__ void compress_pre(uint32_t (&st)[8], const uint32_t (&w16)[16]) {
  uint32_t W[64];
#pragma unroll
  for (int t = 0; t < 16; ++t) W[t] = w16[t];
#pragma unroll
  for (int t = 16; t < 64; ++t) {
    const uint32_t s0 = rotr(W[t - 15], 7) ^ rotr(W[t - 15], 18) ^ (W[t - 15] >> 3);
    const uint32_t s1 = rotr(W[t - 2], 17) ^ rotr(W[t - 2], 19) ^ (W[t - 2] >> 10);
    W[t] = W[t - 16] + s0 + W[t - 7] + s1;
  }
#pragma unroll
  for (int t = 0; t < 64; ++t) W[t] += K[t];
  uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
  for (int t = 0; t < 64; ++t) {
    const uint32_t t1 = h + W[t] + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g));
    const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
    h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

template <int MODE>
__global__ void sha_kernel(int nblocks, uint32_t* out, long long* cycles) {
  uint32_t st[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au, 0x510e527fu, 0x9b05688cu, 0x1f83d9abu,
                    0x5be0cd19u};
  uint32_t st2[8] = {1u, 2u, 3u, 4u, 5u, 6u, 7u, 8u};
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const long long c0 = clock64();
  for (int b = 0; b < nblocks; ++b) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = tid * 16u + (uint32_t)b * 977u + i;  // data from registers
    if (MODE == 0) {
      compress_inline(st, w);
    } else if (MODE == 1) {
      compress_pre(st, w);
    } else {
      uint32_t w2[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) w2[i] = w[i] ^ 0x5a5a5a5au;
      compress_inline(st, w);
      compress_inline(st2, w2);
    }
  }
  const long long c1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= st[i] ^ (MODE == 2 ? st2[i] : 0u);
  out[tid] = acc;
  if (tid == 0) cycles[MODE] = c1 - c0;
}

int main() {
  const int nblocks = 2000;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 64);
  const char* names[3] = {"inline schedule (product)", "schedule expanded first", "two chains interleaved"};
  for (int warps_per_sm_subpart : {1, 2}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int grid = 148 * 4 * warps_per_sm_subpart;  // 32-thread CTAs: one warp per CTA
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&] {
        if (mode == 0) sha_kernel<0><<<grid, 32>>>(nblocks, out, cyc);
        else if (mode == 1) sha_kernel<1><<<grid, 32>>>(nblocks, out, cyc);
        else sha_kernel<2><<<grid, 32>>>(nblocks, out, cyc);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long c[3];
      cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      const int chains = mode == 2 ? 2 : 1;
      printf("%d warp(s)/sub-partition, %-28s: %6.0f cycles per block per thread, %.3f us per block, "
             "%.1f MB/s per chain\n",
             warps_per_sm_subpart, names[mode], (double)c[mode] / nblocks / chains, ms * 1e3 / nblocks / chains,
             64.0 * nblocks * chains / (ms * 1e-3) / 1e6 / chains);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
