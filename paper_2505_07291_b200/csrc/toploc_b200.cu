// toploc_b200.cu -- B200 (sm_100a) kernels + C ABI for TOPLOC prove / verify.
//
// Path (reference boundary, see include/toploc_b200.h):
//   prove  = streaming per-chunk top-K select  -> GF(p) commitment  -> 258-B proofs
//            (replaces swarm/worker/rollout.py:51-68, called at rollout.py:112)
//   verify = streaming per-chunk top-K select fused with proof evaluation,
//            exponent/mantissa statistics and verdicts
//            (replaces swarm/validator/checks.py:209-213)
// The CPU restatement these kernels are checked against is oracle/toploc_oracle.py
// (semantics pinned there).
//
// HBM roofline: both select kernels read every bf16 of the hidden states exactly
// once with 128-bit non-allocating loads; the per-element work is a 16x2-SIMD
// magnitude test against a running per-chunk threshold, so the kernels are
// HBM-bound.  Only the ~0.1 % of elements that can still enter the top-K take the
// slow path into a shared-memory candidate buffer.

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/toploc_b200.h"
#include "primes.inc"

namespace {

// ----------------------------------------------------------------------------- constants
#ifndef TL_RING
#define TL_RING 0  // TMA ring select (1) or direct register-double-buffered loads (0)
#endif
#ifndef TL_SEL_THREADS
#define TL_SEL_THREADS 96
#endif
constexpr int kSelThreads = TL_SEL_THREADS;   // select CTA consumer threads
#ifndef TL_SEL_U
#define TL_SEL_U 4
#endif
constexpr int kSelU = TL_SEL_U;               // 16-B vectors per thread per tile
#ifndef TL_SEL_MIN_BLOCKS
#define TL_SEL_MIN_BLOCKS (TL_RING ? 2 : 8)
#endif
constexpr int kSelMinBlocks = TL_SEL_MIN_BLOCKS;  // resident select CTAs per SM
constexpr int kTileVec = kSelThreads * kSelU; // 1024 vectors = 8192 bf16 per tile
constexpr int kTileElems = kTileVec * 8;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kWarpCap = 256;                 // per-warp candidate buffer (2 KiB)
static_assert(kWarpCap >= TL_MAX_K + 32, "a compaction must leave room for one full ballot");
constexpr int kFlushAt = 4;                   // flagged vectors per exact-test round (32 lanes / 8)
constexpr int kStageVec = 32 * kSelU + 8;     // per-warp flagged-vector queue (< kFlushAt pending + a tile)
#ifndef TL_SPEC_LO
#define TL_SPEC_LO 32   // adapt the margin so a chunk yields kk + [LO, HI] candidates
#endif
#ifndef TL_SPEC_HI
#define TL_SPEC_HI 128
#endif
#ifndef TL_SPEC_HIST
#define TL_SPEC_HIST 2  // speculation = min over the last TL_SPEC_HIST kk-th magnitudes (power of 2)
#endif
#ifndef TL_RING_STAGES
#define TL_RING_STAGES 5
#endif
constexpr int kRingStages = TL_RING_STAGES;   // 16 KiB TMA stages per CTA
constexpr int kRingStageBytes = kTileVec * 16;
constexpr unsigned kIdxMask = 0xFFFFFFu;      // flat index field (24 bits)
constexpr int kInvTables = 8;                 // precomputed inverse tables (first 8 primes)
#ifndef TL_COMMIT_WARPS
#define TL_COMMIT_WARPS 32
#endif
constexpr int kCommitWarps = TL_COMMIT_WARPS;
constexpr uint32_t kPMax = 65497u;

// ----------------------------------------------------------------------------- helpers
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Composite sort key of one element: |bits| (15) | ~idx (24) | bits (16).
// Descending order == magnitude descending, then flat index ascending.
__device__ __forceinline__ unsigned long long make_key(unsigned bits, unsigned idx) {
  return ((unsigned long long)(bits & 0x7FFFu) << 40) |
         ((unsigned long long)(kIdxMask - idx) << 16) | (unsigned long long)(bits & 0xFFFFu);
}
__device__ __forceinline__ unsigned key_idx(unsigned long long s) {
  return kIdxMask - (unsigned)((s >> 16) & kIdxMask);
}

// Arithmetic mod p (2 <= p < 2^16) on u32.  Reductions use the unsigned-min trick:
// for r in [0, 2p), min(r, r - p) (mod 2^32) is r mod p -- one VIADDMNMX.
struct ModP {
  uint32_t p, np, mu;  // np = -p mod 2^32, mu = floor(2^32 / p)
  __device__ __forceinline__ explicit ModP(uint32_t p_)
      : p(p_), np(0u - p_), mu((uint32_t)(0x100000000ull / p_)) {}
  __device__ __forceinline__ uint32_t red(uint32_t t) const {  // t < 2^32 -> t mod p (Barrett)
    const uint32_t r = t + __umulhi(t, mu) * np;                 // t - q p, in [0, 2p)
    return min(r, r + np);
  }
  __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return red(a * b); }
  __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const {
    const uint32_t t = a - b;  // a, b < p
    return min(t, t + p);
  }
  __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
    const uint32_t s = a + b;
    return min(s, s + np);
  }
  __device__ uint32_t pow(uint32_t a, uint32_t e) const {
    uint32_t r = 1;
    while (e) {
      if (e & 1) r = mul(r, a);
      a = mul(a, a);
      e >>= 1;
    }
    return r;
  }
};

// Chunk j -> (rollout, first row, rows) by binary search over the chunk prefix.
struct ChunkRef {
  int64_t row_start;
  int rows;
  int rollout;
};
__device__ __forceinline__ ChunkRef locate_chunk(const int64_t* __restrict__ prefix,
                                                 const int64_t* __restrict__ row_off, int n_roll,
                                                 int64_t j, int C) {
  int lo = 0, hi = n_roll - 1;  // largest r with prefix[r] <= j
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= j) lo = mid; else hi = mid - 1;
  }
  ChunkRef c;
  c.rollout = lo;
  const int64_t local = j - prefix[lo];
  const int64_t T = row_off[lo + 1] - row_off[lo];
  c.row_start = row_off[lo] + local * C;
  c.rows = (int)min((int64_t)C, T - local * C);
  return c;
}

// ----------------------------------------------------------------------------- streaming select
//
// One CTA owns one chunk at a time (persistent over its chunks j = blockIdx.x,
// + gridDim.x, ...).  TL_RING=1 (default): a producer warp streams the CTA's chunks
// through a ring of kRingStages x 16 KiB shared-memory stages with TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), running ahead across chunk boundaries so
// ~190 KiB per SM stay in flight -- the depth a pure read needs to approach the
// ~7.3 TB/s read ceiling measured on this part (tools/lab/bwprobe.py).  Eight
// consumer warps filter each stage (1024 vectors, 128 per warp).  TL_RING=0: the
// consumers load straight from HBM with a register double buffer.
//
// Each consumer warp keeps its own candidate buffer and threshold theta_w with
// the invariant
//     every element this warp has seen with key >= theta_w is in its buffer,
// and, once theta_w was raised by a compaction, >= kk seen elements are >= theta_w.
// The union of the warp buffers therefore contains the chunk's top-kk (an element
// below its warp's theta_w is beaten by kk others).  No barrier while streaming;
// the chunk ends with one consumer barrier and a warp bitonic sort.
//
// A chunk starts from a speculative theta (the previous chunk's kk-th magnitude
// minus an adaptive margin).  If the union ends with < kk entries the speculation
// was too high and the chunk is re-scanned from HBM/L2 with theta = 0.
struct SelState {
  unsigned long long wbuf[kSelWarps][kWarpCap];  // per-warp candidate keys
  int sidx[kSelWarps][kStageVec];                // per-warp flagged vector ids
  int lst_n[kSelWarps];                          // per-warp queue lengths
#if !TL_RING
  uint4 stage[kSelWarps][kStageVec];             // flagged vectors copied out of registers
#endif
  unsigned long long out[TL_MAX_K];              // selected keys, rank order
  unsigned long long theta;                      // chunk-start threshold (speculation)
  unsigned khist[TL_SPEC_HIST];                  // last kk-th magnitudes (speculation history)
  int khead;
  int retry;                                     // re-scans of the current chunk
  int wcnt[kSelWarps];
  unsigned hist[256];
  int delta;                                     // speculation margin, magnitude units
  int digit;
  int kr;
  int n_out;
  // verify-side scratch
  unsigned p;
  unsigned mism, nmatch, msum;
  unsigned mhist[128];
  uint32_t hpart[TL_MAX_K];
  uint16_t coef[TL_MAX_K];
};
constexpr size_t kSelStateBytes = (sizeof(SelState) + 127) & ~(size_t)127;
#if TL_RING
constexpr int kSelBlockThreads = kSelThreads + 32;  // + producer warp
constexpr size_t kSelSmem = kSelStateBytes + (size_t)kRingStages * kRingStageBytes + 2 * kRingStages * 8;
#else
constexpr int kSelBlockThreads = kSelThreads;
constexpr size_t kSelSmem = kSelStateBytes;
#endif

// Barrier over the consumer threads only (the producer warp never joins).
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(kSelThreads) : "memory"); }

__device__ __forceinline__ unsigned hmaxabs2(unsigned a, unsigned b) {
  unsigned d;  // per bf16 half: max(|a|, |b|) (sign = xor, masked off by the caller); NaN wins
  asm("max.NaN.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ bool coarse_hit(unsigned m, unsigned c2) {
  return (((m & 0x7FFF7FFFu) + c2) & 0x80008000u) != 0u;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// ---- TMA bulk copy + mbarrier primitives
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

// ---- chunk geometry
struct ChunkGeo {
  const uint16_t* base;  // first element
  int n;                 // elements
  int a0;                // scalar head elements before the first 16-B boundary
  int nvec;              // 16-B vectors after the head
  int nst;               // 1024-vector stages
};
struct SelArgs {
  const uint16_t* hidden;
  const int64_t* row_off;
  const int64_t* prefix;
  int n_roll, H, C, K;
  int64_t n_chunks;  // min(caller's n_chunks, prefix[n_roll])
};
__device__ __forceinline__ ChunkGeo chunk_geo(const SelArgs& a, int64_t j) {
  const ChunkRef cr = locate_chunk(a.prefix, a.row_off, a.n_roll, j, a.C);
  ChunkGeo g;
  g.base = a.hidden + cr.row_start * (int64_t)a.H;
  g.n = cr.rows * a.H;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(g.base);
  g.a0 = min(g.n, (int)(((16u - (unsigned)(addr & 15u)) & 15u) >> 1));
  g.nvec = (g.n - g.a0) >> 3;
  g.nst = (g.nvec + kTileVec - 1) / kTileVec;
  return g;
}

// Warp bitonic sort, descending, of NPER*32 keys held as a[r] at position r*32+lane.
template <int NPER>
__device__ __forceinline__ void warp_bitonic_desc(unsigned long long (&a)[NPER], int lane) {
  constexpr int N = NPER * 32;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int rj = j >> 5;
#pragma unroll
        for (int r = 0; r < NPER; ++r) {
          if ((r & rj) == 0) {
            const bool desc = (((r * 32 + lane) & k) == 0);
            const unsigned long long x = a[r], y = a[r | rj];
            const unsigned long long hi = x > y ? x : y, lo = x > y ? y : x;
            a[r] = desc ? hi : lo;
            a[r | rj] = desc ? lo : hi;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < NPER; ++r) {
          const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, a[r], j);
          const bool desc = (((r * 32 + lane) & k) == 0);
          const bool lower = (lane & j) == 0;
          const unsigned long long hi = a[r] > o ? a[r] : o, lo = a[r] > o ? o : a[r];
          a[r] = (desc == lower) ? hi : lo;
        }
      }
    }
  }
}

// Buffer full: keep the warp's kk largest keys; returns theta_w = the kk-th (rare path).
__device__ __noinline__ unsigned long long warp_compact(unsigned long long* wb, int cnt, int kk, int lane) {
  unsigned long long a[kWarpCap / 32];
#pragma unroll
  for (int r = 0; r < kWarpCap / 32; ++r) {
    const int q = r * 32 + lane;
    a[r] = q < cnt ? wb[q] : 0ull;
  }
  warp_bitonic_desc<kWarpCap / 32>(a, lane);
#pragma unroll
  for (int r = 0; r < kWarpCap / 32; ++r) wb[r * 32 + lane] = a[r];
  __syncwarp();
  return wb[kk - 1];
}

// Warp-uniform append of at most one key per lane.
__device__ __forceinline__ void warp_append(bool p, unsigned long long key, unsigned long long* wb, int& cnt,
                                            unsigned long long& theta, int kk, int lane) {
  unsigned bal = __ballot_sync(0xFFFFFFFFu, p);
  if (!bal) return;
  if (cnt + __popc(bal) > kWarpCap) {
    theta = warp_compact(wb, cnt, kk, lane);
    cnt = kk;
    p = p && key >= theta;
    bal = __ballot_sync(0xFFFFFFFFu, p);
  }
  if (p) wb[cnt + __popc(bal & lanemask_lt())] = key;
  cnt += __popc(bal);
  __syncwarp();
}

// k-th largest of buf[0..n) by 8-bit radix select over the 56 significant bits.
// All consumer threads call; contains barriers.  Rare path.
__device__ __noinline__ unsigned long long block_kth_largest(const unsigned long long* buf, int n, int k,
                                                             SelState& s) {
  unsigned long long prefix = 0, mask = 0;
  int kr = k;
  for (int shift = 48; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += kSelThreads) s.hist[b] = 0;
    csync();
    for (int e = threadIdx.x; e < n; e += kSelThreads) {
      const unsigned long long v = buf[e];
      if ((v & mask) == prefix) atomicAdd(&s.hist[(unsigned)(v >> shift) & 255u], 1u);
    }
    csync();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      unsigned c[8], sum = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) { c[t] = s.hist[255 - (lane * 8 + t)]; sum += c[t]; }
      unsigned incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned excl = incl - sum;
      if ((int)excl < kr && kr <= (int)incl) {
        unsigned acc = excl;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if ((int)acc < kr && kr <= (int)(acc + c[t])) {
            s.digit = 255 - (lane * 8 + t);
            s.kr = kr - (int)acc;
          }
          acc += c[t];
        }
      }
    }
    csync();
    prefix |= (unsigned long long)s.digit << shift;
    mask |= 0xFFull << shift;
    kr = s.kr;
    csync();
  }
  return prefix;
}

// Final ranking when the warp buffers hold more than 256 candidates (ties,
// degenerate chunks, theta = 0 restarts): radix-select the kk-th key over all
// buffers, collect the kk keys >= it, sort them.  All consumer threads call.
__device__ __noinline__ void rank_many(int kk, SelState& s) {
  unsigned long long* all = &s.wbuf[0][0];
  for (int e = threadIdx.x; e < kSelWarps * kWarpCap; e += kSelThreads)
    if ((e % kWarpCap) >= s.wcnt[e / kWarpCap]) all[e] = 0ull;
  if (threadIdx.x == 0) s.n_out = 0;
  csync();
  const unsigned long long th = block_kth_largest(all, kSelWarps * kWarpCap, kk, s);
  for (int e = threadIdx.x; e < kSelWarps * kWarpCap; e += kSelThreads)
    if (all[e] >= th && all[e] != 0ull) s.out[atomicAdd(&s.n_out, 1)] = all[e];
  csync();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    unsigned long long a[TL_MAX_K / 32];
#pragma unroll
    for (int r = 0; r < TL_MAX_K / 32; ++r) a[r] = (r * 32 + lane < kk) ? s.out[r * 32 + lane] : 0ull;
    __syncwarp();
    warp_bitonic_desc<TL_MAX_K / 32>(a, lane);
#pragma unroll
    for (int r = 0; r < TL_MAX_K / 32; ++r) s.out[r * 32 + lane] = a[r];
  }
}

// Per-warp streaming state (all members warp-uniform except the pointers' targets).
struct WarpScan {
  unsigned long long theta;
  int cnt;
  unsigned long long* wb;
  int* sidx;    // queued flagged vector ids
  uint4* stg;   // TL_RING=0: queued flagged vectors copied out of registers
  int* lst_n;   // queue length
};

__device__ __forceinline__ unsigned coarse_c2(unsigned long long theta, unsigned lo) {
  const unsigned tkey = (unsigned)(theta >> 40);
  // elements tied with theta's magnitude lose on index once lo > theta's index
  const unsigned tk = tkey + (lo > key_idx(theta) ? 1u : 0u);
  return ((0x8000u - tk) & 0xFFFFu) * 0x10001u;
}

// Test the elements of `nflag` flagged vectors lane-parallel and append survivors.
// Element e of the batch is vector sidx[e >> 3], bf16 (e & 7); its bits are read
// through `elem(e)`.
template <typename Elem>
__device__ __forceinline__ void test_flagged(int nflag, int a0, WarpScan& w, int kk, int lane, Elem elem) {
  const unsigned tkey = (unsigned)(w.theta >> 40);
  for (int e0 = 0; e0 < 8 * nflag; e0 += 32) {
    const int e = e0 + lane;
    bool p = false;
    unsigned long long key = 0;
    if (e < 8 * nflag) {
      const unsigned b = elem(e);
      if ((b & 0x7FFFu) >= tkey) {
        key = make_key(b, (unsigned)(a0 + 8 * w.sidx[e >> 3] + (e & 7)));
        p = key >= w.theta;
      }
    }
    warp_append(p, key, w.wb, w.cnt, w.theta, kk, lane);
  }
}

// Test the queued flagged vectors' elements lane-parallel and empty the queue.
template <bool STAGE>
__device__ __forceinline__ void flush_flagged(const ChunkGeo& cg, WarpScan& w, int n, int kk, int lane) {
  if (STAGE) {
    const uint16_t* stg16 = reinterpret_cast<const uint16_t*>(w.stg);
    test_flagged(n, cg.a0, w, kk, lane, [&](int e) { return (unsigned)stg16[e]; });
  } else {
    const uint16_t* el = cg.base + cg.a0;
    test_flagged(n, cg.a0, w, kk, lane, [&](int e) { return (unsigned)el[8 * w.sidx[e >> 3] + (e & 7)]; });
  }
  __syncwarp();
  if (lane == 0) *w.lst_n = 0;
  __syncwarp();
}

// Chunk pass straight from HBM/L2 with a register double buffer.  Vector g of tile
// t: t*1024 + u*256 + warp*32 + lane.  Flagged vectors are copied to w.stg
// (STAGE) or their elements re-read from global memory (L2-hot; the TL_RING
// restart path, which has no staging buffer).
template <bool STAGE>
__device__ __forceinline__ void pass_ldg(const ChunkGeo& cg, WarpScan& w, int kk, int warp, int lane) {
  const uint4* __restrict__ vb = reinterpret_cast<const uint4*>(cg.base + cg.a0);
  const int nvec = cg.nvec, a0 = cg.a0;
  uint4 vn[kSelU];
#pragma unroll
  for (int u = 0; u < kSelU; ++u) {
    const int g = warp * 32 + lane + u * kSelThreads;
    vn[u] = g < nvec ? ld_stream(vb + g) : make_uint4(0u, 0u, 0u, 0u);
  }
  for (int it = 0; it < cg.nst; ++it) {
    const int gbase = it * kTileVec + warp * 32 + lane;
    uint4 v[kSelU];
#pragma unroll
    for (int u = 0; u < kSelU; ++u) {
      v[u] = vn[u];
      const int g = gbase + kTileVec + u * kSelThreads;
      vn[u] = g < nvec ? ld_stream(vb + g) : make_uint4(0u, 0u, 0u, 0u);
    }
    const unsigned c2 = coarse_c2(w.theta, (unsigned)(a0 + it * kTileElems));
    unsigned mu[kSelU];
#pragma unroll
    for (int u = 0; u < kSelU; ++u) mu[u] = hmaxabs2(hmaxabs2(v[u].x, v[u].y), hmaxabs2(v[u].z, v[u].w));
    unsigned m = mu[0];
#pragma unroll
    for (int u = 1; u < kSelU; ++u) m = hmaxabs2(m, mu[u]);
    const bool hit = coarse_hit(m, c2);
    if (!__any_sync(0xFFFFFFFFu, hit)) continue;
    // queue this warp's flagged vectors (vectors past the chunk end are zero and
    // never flagged) with one shared-memory atomic per flagged lane; test queued
    // elements in full 32-lane rounds once >= kFlushAt vectors are pending
    if (hit) {
      unsigned hm = 0;
#pragma unroll
      for (int u = 0; u < kSelU; ++u)
        hm |= ((gbase + u * kSelThreads < nvec && coarse_hit(mu[u], c2)) ? 1u : 0u) << u;
      if (hm) {
        int pos = atomicAdd(w.lst_n, __popc(hm));
#pragma unroll
        for (int u = 0; u < kSelU; ++u) {
          if ((hm >> u) & 1u) {
            if (STAGE) w.stg[pos] = v[u];
            w.sidx[pos] = gbase + u * kSelThreads;
            ++pos;
          }
        }
      }
    }
    __syncwarp();
    const int pending = *reinterpret_cast<volatile int*>(w.lst_n);
    if (pending >= kFlushAt) flush_flagged<STAGE>(cg, w, pending, kk, lane);
  }
  const int pending = *reinterpret_cast<volatile int*>(w.lst_n);
  if (pending > 0) flush_flagged<STAGE>(cg, w, pending, kk, lane);
}

#if TL_RING
// Ring consumer: this warp's share (vectors warp*128 + u*32 + lane) of every stage
// of the chunk, in the producer's order.  Flagged elements are read straight from
// the stage, which is released to the producer afterwards.
struct Ring {
  const uint4* stages;           // [kRingStages][kTileVec]
  unsigned long long* full;      // [kRingStages] producer -> consumers
  unsigned long long* empty;     // [kRingStages] consumers -> producer (count = consumer warps)
  uint32_t seq;                  // stages consumed by this warp
};
__device__ __forceinline__ void pass_ring(const ChunkGeo& cg, WarpScan& w, Ring& r, int kk, int warp, int lane) {
  const int nvec = cg.nvec, a0 = cg.a0;
  const int q0 = warp * (kTileVec / kSelWarps) + lane;
  for (int st = 0; st < cg.nst; ++st) {
    const uint32_t slot = r.seq % kRingStages;
    mbar_wait(r.full + slot, (r.seq / kRingStages) & 1u);
    const uint4* __restrict__ stage = r.stages + (size_t)slot * kTileVec;
    const int g0 = st * kTileVec;  // vector id of stage slot 0
    unsigned mu[kSelU];
#pragma unroll
    for (int u = 0; u < kSelU; ++u) {
      const uint4 v = g0 + q0 + u * 32 < nvec ? stage[q0 + u * 32] : make_uint4(0u, 0u, 0u, 0u);
      mu[u] = hmaxabs2(hmaxabs2(v.x, v.y), hmaxabs2(v.z, v.w));
    }
    unsigned m = mu[0];
#pragma unroll
    for (int u = 1; u < kSelU; ++u) m = hmaxabs2(m, mu[u]);
    const unsigned c2 = coarse_c2(w.theta, (unsigned)(a0 + st * kTileElems));
    const bool hit = coarse_hit(m, c2);
    if (__any_sync(0xFFFFFFFFu, hit)) {
      // u-major list of flagged stage slots (ballots only)
      const unsigned lt = lanemask_lt();
      int tot = 0;
#pragma unroll
      for (int u = 0; u < kSelU; ++u) {
        const bool f = hit && g0 + q0 + u * 32 < nvec && coarse_hit(mu[u], c2);
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, f);
        if (f) w.sidx[tot + __popc(bal & lt)] = q0 + u * 32;
        tot += __popc(bal);
      }
      __syncwarp();
      const uint16_t* st16 = reinterpret_cast<const uint16_t*>(stage);
      const int a0s = a0 + 8 * g0;  // element index of stage slot 0
      test_flagged(tot, a0s, w, kk, lane, [&](int e) { return (unsigned)st16[w.sidx[e >> 3] * 8 + (e & 7)]; });
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(r.empty + slot);
    ++r.seq;
  }
}

// Producer warp: stream every chunk of this CTA, stage by stage, into the ring.
__device__ void ring_producer(const SelArgs& a, uint4* stages, unsigned long long* full,
                              unsigned long long* empty, int lane) {
  uint32_t seq = 0;
  for (int64_t j = blockIdx.x; j < a.n_chunks; j += gridDim.x) {
    const ChunkGeo g = chunk_geo(a, j);
    const uint4* src = reinterpret_cast<const uint4*>(g.base + g.a0);
    for (int st = 0; st < g.nst; ++st, ++seq) {
      const uint32_t slot = seq % kRingStages;
      if (seq >= (uint32_t)kRingStages) mbar_wait(empty + slot, ((seq / kRingStages) - 1u) & 1u);
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)min(kTileVec, g.nvec - st * kTileVec) * 16u;
        mbar_expect_tx(full + slot, bytes);
        bulk_g2s(stages + (size_t)slot * kTileVec, src + (size_t)st * kTileVec, bytes, full + slot);
      }
      __syncwarp();
    }
  }
}
#endif

// Top-kk of chunk cg -> s.out[0..kk) in rank order.  s.theta holds this chunk's
// speculative threshold on entry.  Consumer threads only; ends with a barrier.
template <typename Src>
__device__ void select_chunk(const ChunkGeo& cg, int kk, SelState& s, Src& src) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpScan w;
  w.wb = s.wbuf[warp];
  w.sidx = s.sidx[warp];
  w.lst_n = &s.lst_n[warp];
#if TL_RING
  w.stg = nullptr;
#else
  w.stg = s.stage[warp];
#endif
  const int tail0 = cg.a0 + (cg.nvec << 3);
  int total;
  bool first_pass = true;
  for (;;) {
    w.theta = s.theta;
    w.cnt = 0;
    const bool spec = w.theta != 0ull;
    if (warp == 0) {  // scalar head / tail elements (chunks not 16-B aligned)
      bool p = false;
      unsigned long long key = 0;
      if (lane < cg.a0) {
        key = make_key(cg.base[lane], lane);
        p = key >= w.theta;
      } else if (lane >= 8 && lane - 8 < cg.n - tail0) {
        key = make_key(cg.base[tail0 + lane - 8], tail0 + lane - 8);
        p = key >= w.theta;
      }
      warp_append(p, key, w.wb, w.cnt, w.theta, kk, lane);
    }
#if TL_RING
    if (first_pass) pass_ring(cg, w, src, kk, warp, lane);
    else pass_ldg<false>(cg, w, kk, warp, lane);
#else
    pass_ldg<true>(cg, w, kk, warp, lane);
#endif
    first_pass = false;
    if (lane == 0) s.wcnt[warp] = w.cnt;
    csync();
    total = 0;
#pragma unroll
    for (int q = 0; q < kSelWarps; ++q) total += s.wcnt[q];
    if (total >= kk) break;
    // the speculative theta excluded part of the top-kk: re-scan (L2-hot) with a
    // lower threshold -- 64, then 256 magnitude steps lower, then 0 (exact)
    if (!spec) __trap();  // unreachable: theta = 0 admits every element
    csync();
    if (tid == 0) {
      const unsigned key = (unsigned)(s.theta >> 40);
      const unsigned drop = s.retry == 0 ? 64u : 256u;
      s.theta = (s.retry < 2 && key > drop) ? ((unsigned long long)(key - drop) << 40) : 0ull;
      ++s.retry;
      s.delta = min(s.delta + 4, 0x4000);
    }
    csync();
  }

  if (total <= 256) {
    if (warp == 0) {
      unsigned long long a[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int q = r * 32 + lane;
        int run = 0, ww = 0, basew = 0;
#pragma unroll
        for (int t = 0; t < kSelWarps; ++t) {  // segment of q in the concatenated warp buffers
          if (q >= run) { ww = t; basew = run; }
          run += s.wcnt[t];
        }
        a[r] = q < total ? s.wbuf[ww][q - basew] : 0ull;
      }
      warp_bitonic_desc<8>(a, lane);
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r * 32 + lane < kk) s.out[r * 32 + lane] = a[r];
    }
  } else {
    rank_many(kk, s);
  }
  csync();
  if (tid == 0) {  // speculation for this CTA's next chunk
    int d = s.delta;
    if (total > kk + TL_SPEC_HI && d > 1) --d;
    else if (total < kk + TL_SPEC_LO) ++d;
    s.delta = d;
    s.khist[s.khead++ & (TL_SPEC_HIST - 1)] = (unsigned)(s.out[kk - 1] >> 40);
    unsigned kmag = s.khist[0];
#pragma unroll
    for (int q = 1; q < TL_SPEC_HIST; ++q) kmag = min(kmag, s.khist[q]);  // min of the last kk-th magnitudes
    s.theta = kmag > (unsigned)d ? ((unsigned long long)(kmag - (unsigned)d) << 40) : 0ull;
    s.retry = 0;
  }
}

struct NoSrc {};
#if TL_RING
using SelSrc = Ring;
#else
using SelSrc = NoSrc;
#endif

// Carve shared memory; the producer warp (TL_RING) streams and returns false,
// consumer threads get their ring view and return true.
__device__ __forceinline__ bool sel_setup(uint8_t* smem, const SelArgs& a, SelState*& sp, SelSrc& src) {
  SelState& s = *reinterpret_cast<SelState*>(smem);
  sp = &s;
  if (threadIdx.x < kSelWarps) s.lst_n[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    s.theta = 0;
    s.delta = 8;
    s.khead = 0;
    s.retry = 0;
    for (int i = 0; i < TL_SPEC_HIST; ++i) s.khist[i] = 0x7FFFu;
  }
#if TL_RING
  uint4* stages = reinterpret_cast<uint4*>(smem + kSelStateBytes);
  unsigned long long* full =
      reinterpret_cast<unsigned long long*>(smem + kSelStateBytes + (size_t)kRingStages * kRingStageBytes);
  unsigned long long* empty = full + kRingStages;
  if (threadIdx.x < kRingStages) {
    mbar_init(full + threadIdx.x, 1);
    mbar_init(empty + threadIdx.x, kSelWarps);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (threadIdx.x >= kSelThreads) {
    ring_producer(a, stages, full, empty, threadIdx.x & 31);
    return false;
  }
  src.stages = stages;
  src.full = full;
  src.empty = empty;
  src.seq = 0;
#else
  (void)a;
  (void)src;
  __syncthreads();
#endif
  return true;
}

// ----------------------------------------------------------------------------- kernels
__global__ void chunk_prefix_kernel(const int64_t* __restrict__ row_off, int n_roll, int C,
                                    int64_t* __restrict__ prefix) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) { carry = 0; prefix[0] = 0; }
  __syncthreads();
  for (int base = 0; base < n_roll; base += blockDim.x) {
    const int r = base + tid;
    int64_t cnt = 0;
    if (r < n_roll) {
      const int64_t T = row_off[r + 1] - row_off[r];
      cnt = T > 0 ? (T + C - 1) / C : 0;
    }
    int64_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      int64_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int64_t off = carry + (w ? warp_tot[w - 1] : 0);
    if (r < n_roll) prefix[r + 1] = off + incl;
    __syncthreads();
    if (tid == 0) carry += warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSelBlockThreads, kSelMinBlocks)
prove_select_kernel(SelArgs a, int32_t* __restrict__ idx_out, uint16_t* __restrict__ bits_out) {
  extern __shared__ __align__(128) uint8_t sel_smem[];
  a.n_chunks = min(a.n_chunks, a.prefix[a.n_roll]);
  SelState* sp;
  SelSrc src;
  if (!sel_setup(sel_smem, a, sp, src)) return;  // producer warp done
  SelState& s = *sp;
  const int K = a.K;
  for (int64_t j = blockIdx.x; j < a.n_chunks; j += gridDim.x) {
    const ChunkGeo g = chunk_geo(a, j);
    const int kk = min(K, g.n);
    select_chunk(g, kk, s, src);
    for (int i = threadIdx.x; i < K; i += kSelThreads) {
      if (i < kk) {
        const unsigned long long v = s.out[i];
        idx_out[j * K + i] = (int32_t)key_idx(v);
        bits_out[j * K + i] = (uint16_t)(v & 0xFFFFu);
      } else {
        idx_out[j * K + i] = -1;
        bits_out[j * K + i] = 0;
      }
    }
    csync();
  }
}

// Warp-wide bitonic sort (ascending over i = lane + 32 r) of 4 registers per lane.
__device__ __forceinline__ void warp_sort128(uint32_t (&v)[4], int lane) {
#pragma unroll
  for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj >= 32) {
        const int rj = jj >> 5;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if ((r & rj) == 0) {
            const int i = lane + 32 * r;
            const bool asc = (i & k) == 0;
            const uint32_t a = v[r], b = v[r | rj];
            const uint32_t lo = min(a, b), hi = max(a, b);
            v[r] = asc ? lo : hi;
            v[r | rj] = asc ? hi : lo;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v[r], jj);
          const int i = lane + 32 * r;
          const bool asc = (i & k) == 0;
          const bool lower = (lane & jj) == 0;
          v[r] = (asc == lower) ? min(v[r], o) : max(v[r], o);
        }
      }
    }
  }
}

__global__ void inv_table_kernel(uint16_t* __restrict__ tables) {
  const int q = blockIdx.y;
  const uint32_t p = kPrimesDesc[q];
  const ModP m(p);
  for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < 65536u; a += gridDim.x * blockDim.x)
    tables[(size_t)q * 65536u + a] = (a == 0 || a >= p) ? 0 : (uint16_t)m.pow(a, p - 2);
}

// Inverse source for the divided differences: the CTA's shared-memory table (first
// prime, almost every chunk), a precomputed global table (primes 2..8), or Fermat.
enum InvMode { kInvSmem = 0, kInvGlobal = 1, kInvFermat = 2, kInvSmemHalf = 3 };
constexpr int kHalfTab = 32768;  // half table: inv(d) for d < 2^15, inv(d) = p - inv(p - d) above

template <int MODE>
__device__ __forceinline__ uint32_t inv_of(const uint16_t* tab, uint32_t d, const ModP& m) {
  if (MODE == kInvSmem) return tab[d];
  if (MODE == kInvSmemHalf) {
    const bool lo = d < (uint32_t)kHalfTab;
    const uint32_t t = tab[lo ? d : m.p - d];
    return lo ? t : m.p - t;
  }
  if (MODE == kInvGlobal) return __ldg(tab + d);
  return m.pow(d, m.p - 2);
}

// Newton divided differences, levels jl in [j0, j1) with j1 <= 32 (R0 + 1): the
// register blocks r < R0 are complete (i < jl) and skipped at compile time; in
// block R0 lanes with i < jl keep their value.  c[i] <- (c[i] - c[i-1]) / (x[i] - x[i-jl]).
template <int MODE, int R0>
__device__ __forceinline__ void ndd_levels(int j0, int j1, const uint32_t (&x)[4], uint32_t (&c)[4],
                                           const uint32_t* xs, const ModP& m, const uint16_t* tab, int lane) {
  const int src = (lane + 31) & 31;
  for (int jl = j0; jl < j1; ++jl) {
    uint32_t t[4];
#pragma unroll
    for (int r = (R0 > 0 ? R0 - 1 : 0); r < 4; ++r) t[r] = __shfl_sync(0xFFFFFFFFu, c[r], src);
#pragma unroll
    for (int r = R0; r < 4; ++r) {
      const int i = lane + 32 * r;
      const uint32_t prev = lane ? t[r] : (r ? t[r > 0 ? r - 1 : 0] : 0u);
      const uint32_t xj = xs[r == R0 ? max(i - jl, 0) : i - jl];
      const uint32_t nv = m.mul(m.sub(c[r], prev), inv_of<MODE>(tab, m.sub(x[r], xj), m));
      if (r > R0 || i >= jl) c[r] = nv;
    }
  }
}

// Newton -> monomial steps i in [i_lo, i_hi] (descending): poly <- poly * (X - x_i) + c_i.
// The polynomial has degree kk-1-i <= 32 (RM + 1) - 1, so blocks r > RM stay zero.
template <int RM>
__device__ __forceinline__ void conv_steps(int i_hi, int i_lo, uint32_t (&poly)[4], const uint32_t* xs,
                                           const uint32_t* cs, const ModP& m, int lane) {
  const int src = (lane + 31) & 31;
  for (int i = i_hi; i >= i_lo; --i) {
    const uint32_t nxi = m.p - xs[i], ci = cs[i];  // prevk - x_i a == prevk + (p - x_i) a < 2^32
    uint32_t t[4];
#pragma unroll
    for (int r = 0; r <= RM; ++r) t[r] = __shfl_sync(0xFFFFFFFFu, poly[r], src);
#pragma unroll
    for (int r = 0; r <= RM; ++r) {
      const uint32_t prevk = lane ? t[r] : (r ? t[r > 0 ? r - 1 : 0] : (0u));
      uint32_t nv = m.red(prevk + nxi * poly[r]);
      if (r == 0 && lane == 0) nv = m.add(nv, ci);
      poly[r] = nv;
    }
  }
}

// Interpolate the warp's kk points (x_i, y_i), i = lane + 32 r, over GF(p):
// Newton divided differences, then Newton -> monomial.
template <int MODE>
__device__ __forceinline__ void interpolate_warp(const uint32_t (&x)[4], uint32_t (&c)[4], uint32_t (&poly)[4],
                                                 const uint32_t* xs, uint32_t* cs, int kk, const ModP& m,
                                                 const uint16_t* tab, int lane) {
  ndd_levels<MODE, 0>(1, min(kk, 32), x, c, xs, m, tab, lane);
  ndd_levels<MODE, 1>(32, min(kk, 64), x, c, xs, m, tab, lane);
  ndd_levels<MODE, 2>(64, min(kk, 96), x, c, xs, m, tab, lane);
  ndd_levels<MODE, 3>(96, kk, x, c, xs, m, tab, lane);
#pragma unroll
  for (int r = 0; r < 4; ++r) cs[lane + 32 * r] = c[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 4; ++r) poly[r] = 0u;
  if (lane == 0) poly[0] = cs[kk - 1];
  // step i yields degree kk-1-i: blocks r <= (kk-1-i) >> 5 are live
  conv_steps<0>(kk - 2, max(kk - 32, 0), poly, xs, cs, m, lane);
  conv_steps<1>(kk - 33, max(kk - 64, 0), poly, xs, cs, m, lane);
  conv_steps<2>(kk - 65, max(kk - 96, 0), poly, xs, cs, m, lane);
  conv_steps<3>(kk - 97, 0, poly, xs, cs, m, lane);
}

// One warp per chunk: modulus search, GF(p) interpolation, 258-byte serialisation.
// WARPS x 32 threads, one CTA per SM.  HALF = 64 KiB half inverse table and <= 64
// registers, so the CTA fits on an SM beside three select/verify CTAs (overlap mode).
template <int WARPS, bool HALF>
__global__ void __launch_bounds__(WARPS * 32, HALF ? 4 : (WARPS > 16 ? 1 : 1))
commit_kernel(const int32_t* __restrict__ idx, const uint16_t* __restrict__ bits, int64_t n_chunks,
              int K, const uint16_t* __restrict__ inv_tables, uint8_t* __restrict__ proofs) {
  constexpr int kTabEntries = HALF ? kHalfTab : 65536;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint16_t* inv0 = reinterpret_cast<uint16_t*>(smem_raw);
  uint32_t* xs_all = reinterpret_cast<uint32_t*>(smem_raw + kTabEntries * 2);  // [warps][128]
  uint32_t* cs_all = xs_all + WARPS * 128;                                     // [warps][128]
  {
    const uint4* src = reinterpret_cast<const uint4*>(inv_tables);
    uint4* dst = reinterpret_cast<uint4*>(inv0);
    for (int i = threadIdx.x; i < kTabEntries * 2 / 16; i += WARPS * 32) dst[i] = src[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* xs = xs_all + warp * 128;
  uint32_t* cs = cs_all + warp * 128;
  const int PB = 2 + 2 * K;

  for (int64_t j = (int64_t)blockIdx.x * WARPS + warp; j < n_chunks; j += (int64_t)gridDim.x * WARPS) {
    uint32_t raw[4], yb[4];
    int kk = 0;
    uint32_t maxidx = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      int32_t iv = -1;
      uint32_t b = 0;
      if (i < K) { iv = idx[j * K + i]; b = bits[j * K + i]; }
      raw[r] = (uint32_t)iv;
      yb[r] = b;
      kk += __popc(__ballot_sync(0xFFFFFFFFu, iv >= 0));
      if (iv >= 0) maxidx = max(maxidx, (uint32_t)iv);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxidx = max(maxidx, __shfl_xor_sync(0xFFFFFFFFu, maxidx, o));

    // ---- modulus: largest prime with injective residues
    int pi = 0;
    uint32_t p = kPMax;
    if (maxidx >= kPMax) {
      for (pi = 0; pi < TL_N_PRIMES; ++pi) {
        p = kPrimesDesc[pi];
        const ModP mp(p);
        uint32_t res[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = lane + 32 * r;
          res[r] = (i < kk) ? mp.red(raw[r]) : 0x10000u + (uint32_t)i;
        }
        warp_sort128(res, lane);
        bool dup = false;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, res[r], 1);
          const uint32_t first_next = __shfl_sync(0xFFFFFFFFu, res[r < 3 ? r + 1 : 3], 0);
          if (lane == 31) nxt = (r < 3) ? first_next : 0xFFFFFFFFu;
          dup |= (nxt == res[r]);
        }
        if (!__any_sync(0xFFFFFFFFu, dup)) break;
      }
      if (pi == TL_N_PRIMES) p = 0;
    }
    uint8_t* pr = proofs + j * PB;
    if (p == 0) {  // unprovable chunk: p = 0, zero coefficients
      for (int b = lane; b < PB; b += 32) pr[b] = 0;
      continue;
    }
    const ModP m(p);
    uint32_t x[4], c[4], poly[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      x[r] = (i < kk) ? m.red(raw[r]) : 0u;
      c[r] = (i < kk) ? m.red(yb[r]) : 0u;
      xs[i] = x[r];
    }
    __syncwarp();
    if (pi == 0) interpolate_warp<HALF ? kInvSmemHalf : kInvSmem>(x, c, poly, xs, cs, kk, m, inv0, lane);
    else if (pi < kInvTables)
      interpolate_warp<kInvGlobal>(x, c, poly, xs, cs, kk, m, inv_tables + (size_t)pi * 65536u, lane);
    else interpolate_warp<kInvFermat>(x, c, poly, xs, cs, kk, m, nullptr, lane);

    // ---- serialise: p, c_0..c_{K-1}, u16 big-endian
    uint16_t* pw = reinterpret_cast<uint16_t*>(pr);
    if (lane == 0) pw[0] = (uint16_t)(((p & 0xFFu) << 8) | (p >> 8));
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = lane + 32 * r;
      if (k < K) {
        const uint32_t v = poly[r];
        pw[1 + k] = (uint16_t)(((v & 0xFFu) << 8) | (v >> 8));
      }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kSelBlockThreads, kSelMinBlocks)
verify_kernel(SelArgs a, const uint8_t* __restrict__ proofs, tl_thresholds th,
              tl_chunk_stats* __restrict__ stats_out, uint8_t* __restrict__ accept_out) {
  extern __shared__ __align__(128) uint8_t sel_smem[];
  a.n_chunks = min(a.n_chunks, a.prefix[a.n_roll]);
  SelState* sp;
  SelSrc src;
  if (!sel_setup(sel_smem, a, sp, src)) return;  // producer warp done
  SelState& s = *sp;
  const int tid = threadIdx.x;
  const int K = a.K;
  const int PB = 2 + 2 * K;
  constexpr int kPW = (TL_MAX_K + 1 + kSelThreads - 1) / kSelThreads;  // proof words per thread
  for (int64_t j = blockIdx.x; j < a.n_chunks; j += gridDim.x) {
    const ChunkGeo g = chunk_geo(a, j);
    const int kk = min(K, g.n);
    // issue this chunk's proof loads (u16 t = p or c_{t-1}) before streaming, so
    // their latency hides behind the chunk instead of the tail
    const uint16_t* pw = reinterpret_cast<const uint16_t*>(proofs + j * PB);
    uint32_t pword[kPW];
#pragma unroll
    for (int q = 0; q < kPW; ++q) {
      const int t = tid + q * kSelThreads;
      pword[q] = t <= K ? (uint32_t)__ldg(pw + t) : 0u;
    }
    select_chunk(g, kk, s, src);

#pragma unroll
    for (int q = 0; q < kPW; ++q) {
      const int t = tid + q * kSelThreads;
      const uint16_t v = (uint16_t)(((pword[q] & 0xFFu) << 8) | (pword[q] >> 8));
      if (t == 0) s.p = v;
      else if (t <= K) s.coef[t - 1] = v;
    }
    if (tid == 0) { s.mism = 0; s.nmatch = 0; s.msum = 0; }
    for (int b = tid; b < 128; b += kSelThreads) s.mhist[b] = 0;
    csync();
    const unsigned p = s.p;
    const bool bad = p < 2;
    auto tally = [&](uint32_t claimed, unsigned long long v, const ModP& m) {
      const uint32_t obs = m.red((uint32_t)(v & 0xFFFFu));
      if (((claimed >> 7) & 0xFFu) != ((obs >> 7) & 0xFFu)) {
        atomicAdd(&s.mism, 1u);
      } else {
        const int d = abs((int)(claimed & 0x7Fu) - (int)(obs & 0x7Fu));
        atomicAdd(&s.mhist[d], 1u);
        atomicAdd(&s.msum, (unsigned)d);
        atomicAdd(&s.nmatch, 1u);
      }
    };
    if constexpr (kSelThreads >= 2 * TL_MAX_K) {
      // Horner split over two thread halves: thread t < 128 evaluates c_0..c_{h-1}
      // at point t, thread t + 128 evaluates c_h..c_{K-1} and scales by x^h
      const int pt = tid & 127, half = (tid >> 7) & 1, h = (K + 1) >> 1;
      const bool horner = tid < 256 && pt < kk;
      uint32_t acc = 0, x = 0;
      if (!bad && horner) {
        const ModP m(p);
        x = m.red(key_idx(s.out[pt]));
        const int k_lo = half ? h : 0, k_hi = half ? K : h;
        for (int k = k_hi - 1; k >= k_lo; --k) acc = m.red(acc * x + (uint32_t)s.coef[k]);
        if (half) s.hpart[pt] = m.mul(acc, m.pow(x, (uint32_t)h));
      }
      csync();
      if (!bad && horner && half == 0) {
        const ModP m(p);
        tally(m.add(acc, s.hpart[pt]), s.out[pt], m);
      }
    } else {
      // one Horner chain per point, TL_MAX_K / kSelThreads points per thread
      if (!bad) {
        const ModP m(p);
        for (int pt = tid; pt < kk; pt += kSelThreads) {
          const uint32_t x = m.red(key_idx(s.out[pt]));
          uint32_t acc = 0;
          for (int k = K - 1; k >= 0; --k) acc = m.red(acc * x + (uint32_t)s.coef[k]);
          tally(acc, s.out[pt], m);
        }
      }
    }
    csync();
    if (tid < 32) {  // median over the 128-bin histogram of |mantissa diff|
      const unsigned nm = s.nmatch;
      unsigned c4[4], sum = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) { c4[t] = s.mhist[tid * 4 + t]; sum += c4[t]; }
      unsigned incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (tid >= o) incl += y;
      }
      unsigned acc = incl - sum;
      int v1 = -1, v2 = -1;
      const unsigned q1 = nm ? (nm - 1) / 2 : 0, q2 = nm / 2;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (acc <= q1 && q1 < acc + c4[t]) v1 = tid * 4 + t;
        if (acc <= q2 && q2 < acc + c4[t]) v2 = tid * 4 + t;
        acc += c4[t];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v1 = max(v1, __shfl_xor_sync(0xFFFFFFFFu, v1, o));
        v2 = max(v2, __shfl_xor_sync(0xFFFFFFFFu, v2, o));
      }
      if (tid == 0) {
        tl_chunk_stats st;
        if (bad) {
          st.exp_mismatch = (uint32_t)kk; st.n_match = 0; st.mant_sum = 0;
          st.mant_mean = __longlong_as_double(0x7FF0000000000000ll);
          st.mant_median = st.mant_mean;
          st.flags = TL_STAT_BADPROOF;
        } else {
          st.exp_mismatch = s.mism; st.n_match = nm; st.mant_sum = s.msum;
          if (nm) {
            st.mant_mean = (double)s.msum / (double)nm;
            st.mant_median = ((double)v1 + (double)v2) * 0.5;
          } else {
            st.mant_mean = __longlong_as_double(0x7FF0000000000000ll);
            st.mant_median = st.mant_mean;
          }
          const bool acc_ok = (int)st.exp_mismatch <= th.max_exp_mismatch &&
                              st.mant_mean <= th.max_mant_mean && st.mant_median <= th.max_mant_median;
          st.flags = acc_ok ? TL_STAT_ACCEPT : 0u;
        }
        if (stats_out) stats_out[j] = st;
        accept_out[j] = (uint8_t)(st.flags & TL_STAT_ACCEPT);
      }
    }
    csync();
  }
}

__global__ void rollout_verdict_kernel(const uint8_t* __restrict__ chunk_accept,
                                       const int64_t* __restrict__ prefix, int n_roll,
                                       uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n_roll) return;
  int ok = 1;
  for (int64_t q = prefix[r] + lane; q < prefix[r + 1]; q += 32) ok &= chunk_accept[q] ? 1 : 0;
  ok = __all_sync(0xFFFFFFFFu, ok);
  if (lane == 0) out[r] = (uint8_t)ok;
}

// ----------------------------------------------------------------------------- exact mode
__device__ __forceinline__ double load_as_f64(const void* in, int dtype, int64_t i) {
  switch (dtype) {
    case 0: return reinterpret_cast<const double*>(in)[i];
    case 1: {
      const uint32_t b = reinterpret_cast<const uint32_t*>(in)[i];
      if ((b & 0x7FFFFFFFu) > 0x7F800000u)  // NaN: widen payload like x86 cvtss2sd
        return __longlong_as_double((long long)(((uint64_t)(b >> 31) << 63) | 0x7FF8000000000000ull |
                                                ((uint64_t)(b & 0x7FFFFFu) << 29)));
      return (double)__uint_as_float(b);
    }
    case 2: {
      const uint32_t b = (uint32_t)reinterpret_cast<const uint16_t*>(in)[i] << 16;
      if ((b & 0x7FFFFFFFu) > 0x7F800000u)
        return __longlong_as_double((long long)(((uint64_t)(b >> 31) << 63) | 0x7FF8000000000000ull |
                                                ((uint64_t)(b & 0x7FFFFFu) << 29)));
      return (double)__uint_as_float(b);
    }
    default: {
      const uint16_t h = reinterpret_cast<const uint16_t*>(in)[i];
      if ((h & 0x7FFFu) > 0x7C00u)
        return __longlong_as_double((long long)(((uint64_t)(h >> 15) << 63) | 0x7FF8000000000000ull |
                                                ((uint64_t)(h & 0x3FFu) << 42)));
      return (double)__half2float(__ushort_as_half(h));
    }
  }
}

__global__ void round6_kernel(const void* __restrict__ in, int dtype, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = load_as_f64(in, dtype, i);
    double r;
    if (x != x) {  // np.round keeps (and quiets) the NaN payload
      r = __longlong_as_double(__double_as_longlong(x) | 0x0008000000000000ll);
    } else {
      r = __ddiv_rn(rint(__dmul_rn(x, 1e6)), 1e6);
    }
    out[i] = r;
  }
}

// ----------------------------------------------------------------------------- synthetic input
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Massive { int c[6]; };

__global__ void synth_kernel(uint16_t* __restrict__ out, int64_t row0, int64_t n_rows, int H,
                             uint64_t sm, int dist, const uint16_t* __restrict__ table, Massive mv,
                             int jthr, uint64_t jm) {
  const int64_t G = (H + 3) / 4;
  const int64_t total = n_rows * G;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = q / G;
    const int g = (int)(q - row * G);
    const uint64_t ctr = (uint64_t)(row0 + row) * (uint64_t)G + (uint64_t)g;
    const uint64_t z = mix64(ctr + sm);
    const uint64_t jz = jthr > 0 ? mix64(ctr + jm) : 0ull;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int c = 4 * g + l;
      if (c >= H) break;
      uint32_t b;
      if (dist == 2) b = 0;
      else if (dist == 3) b = 0x3F80u;
      else {
        b = table[(z >> (16 * l)) & 0xFFFFu];
        if (dist == 1 && (c == mv.c[0] || c == mv.c[1] || c == mv.c[2] || c == mv.c[3] || c == mv.c[4] || c == mv.c[5])) {
          const float f = __fmul_rn(__uint_as_float(b << 16), 200.0f);
          b = __bfloat16_as_ushort(__float2bfloat16_rn(f));
        }
      }
      if (jthr > 0) {
        const uint32_t h = (uint32_t)((jz >> (16 * l)) & 0xFFFFu);
        if ((int)h < jthr) {
          uint32_t mag = b & 0x7FFFu;
          const uint32_t sign = b & 0x8000u;
          if (h & 1u) { if (mag < 0x7F7Fu) mag += 1; } else { if (mag > 0) mag -= 1; }
          b = sign | mag;
        }
      }
      out[row * H + c] = (uint16_t)b;
    }
  }
}

// ----------------------------------------------------------------------------- host helpers
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct WsLayout {
  size_t prefix, tables, idx, bits, accept, total;
};
WsLayout ws_layout(int32_t n_roll, int64_t n_chunks, int32_t K) {
  WsLayout L;
  size_t o = 0;
  L.prefix = o; o = align_up(o + (size_t)(n_roll + 1) * 8, 256);
  L.tables = o; o = align_up(o + (size_t)kInvTables * 65536 * 2, 256);
  L.idx = o; o = align_up(o + (size_t)n_chunks * K * 4, 256);
  L.bits = o; o = align_up(o + (size_t)n_chunks * K * 2, 256);
  L.accept = o; o = align_up(o + (size_t)n_chunks, 256);
  L.total = o;
  return L;
}

int check_shape(int32_t n_roll, int64_t n_rows, int32_t H, int32_t C, int32_t K, int64_t n_chunks) {
  if (n_roll < 0 || n_rows < 0 || H < 1 || C < 1 || K < 1 || n_chunks < 0) return TL_EINVAL;
  if (K > TL_MAX_K) return TL_EUNSUPPORTED;
  if ((int64_t)C * H >= (int64_t)kIdxMask) return TL_EUNSUPPORTED;
  return TL_OK;
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n;
}

int sel_grid(int64_t n_chunks, const void* kernel, int ctas_per_sm = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSelBlockThreads, kSelSmem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  if (ctas_per_sm > 0 && ctas_per_sm < per_sm) per_sm = ctas_per_sm;
  const int64_t g = (int64_t)sm_count() * per_sm;
  return (int)(n_chunks < g ? (n_chunks > 0 ? n_chunks : 1) : g);
}

int launch_status() { return cudaGetLastError() == cudaSuccess ? TL_OK : TL_ECUDA; }

template <int WARPS, bool HALF>
int launch_commit_t(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int K, const uint16_t* tables,
                    uint8_t* proofs, cudaStream_t st) {
  const size_t smem = (size_t)(HALF ? kHalfTab : 65536) * 2 + 2 * WARPS * 128 * 4;
  if (cudaFuncSetAttribute(commit_kernel<WARPS, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return TL_ECUDA;
  int grid = sm_count();
  if ((int64_t)grid * WARPS > n_chunks) grid = (int)((n_chunks + WARPS - 1) / WARPS);
  commit_kernel<WARPS, HALF><<<grid, WARPS * 32, smem, st>>>(idx, bits, n_chunks, K, tables, proofs);
  return launch_status();
}

// co_resident = 0: 16 warps, full 128 KiB table (fastest alone); 1: 8 warps, 64 KiB
// half table, <= 64 registers -- fits beside three select/verify CTAs per SM.
int launch_commit(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int K, const uint16_t* tables,
                  uint8_t* proofs, int co_resident, cudaStream_t st) {
  return co_resident ? launch_commit_t<8, true>(idx, bits, n_chunks, K, tables, proofs, st)
                     : launch_commit_t<kCommitWarps, false>(idx, bits, n_chunks, K, tables, proofs, st);
}

}  // namespace

// ============================================================================= C ABI
extern "C" {

const char* tl_strerror(int code) {
  switch (code) {
    case TL_OK: return "ok";
    case TL_EINVAL: return "invalid argument";
    case TL_EUNSUPPORTED: return "unsupported shape (K in [1,128], C*H < 2^24-1)";
    case TL_EWORKSPACE: return "workspace too small or misaligned";
    case TL_ECUDA: return "CUDA launch or runtime failure";
    default: return "unknown error";
  }
}

int tl_version(void) { return 1; }

int64_t tl_count_chunks(const int64_t* row_off_host, int32_t n_roll, int32_t C) {
  if (!row_off_host || n_roll < 0 || C < 1) return TL_EINVAL;
  int64_t n = 0;
  for (int32_t r = 0; r < n_roll; ++r) {
    const int64_t T = row_off_host[r + 1] - row_off_host[r];
    if (T < 0) return TL_EINVAL;
    n += (T + C - 1) / C;
  }
  return n;
}

size_t tl_workspace_bytes(int32_t n_roll, int64_t n_chunks, int32_t K) {
  return ws_layout(n_roll, n_chunks, K).total;
}

int tl_select(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
              int32_t H, int32_t C, int32_t K, int64_t n_chunks, int32_t* idx_out,
              uint16_t* bits_out, void* workspace, size_t workspace_bytes, void* stream) {
  return tl_select_ex(hidden, row_off, n_roll, n_rows, H, C, K, n_chunks, idx_out, bits_out, workspace,
                      workspace_bytes, 0, stream);
}

int tl_select_ex(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
                 int32_t H, int32_t C, int32_t K, int64_t n_chunks, int32_t* idx_out,
                 uint16_t* bits_out, void* workspace, size_t workspace_bytes, int32_t ctas_per_sm,
                 void* stream) {
  int rc = check_shape(n_roll, n_rows, H, C, K, n_chunks);
  if (rc) return rc;
  if (n_chunks == 0 || n_roll == 0) return TL_OK;
  if (!hidden || !row_off || !idx_out || !bits_out || !workspace) return TL_EINVAL;
  const WsLayout L = ws_layout(n_roll, n_chunks, K);
  if (workspace_bytes < L.total || (reinterpret_cast<uintptr_t>(workspace) & 255)) return TL_EWORKSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int64_t* prefix = reinterpret_cast<int64_t*>(ws + L.prefix);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  chunk_prefix_kernel<<<1, 1024, 0, st>>>(row_off, n_roll, C, prefix);
  const SelArgs a{hidden, row_off, prefix, n_roll, H, C, K, n_chunks};
  if (cudaFuncSetAttribute(prove_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelSmem) !=
      cudaSuccess)
    return TL_ECUDA;
  prove_select_kernel<<<sel_grid(n_chunks, (const void*)prove_select_kernel, ctas_per_sm), kSelBlockThreads,
                        kSelSmem, st>>>(
      a, idx_out, bits_out);
  return launch_status();
}

int tl_commit(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int32_t K,
              uint8_t* proofs_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_chunks < 0 || K < 1) return TL_EINVAL;
  if (K > TL_MAX_K) return TL_EUNSUPPORTED;
  if (n_chunks == 0) return TL_OK;
  if (!idx || !bits || !proofs_out || !workspace) return TL_EINVAL;
  const WsLayout L = ws_layout(0, n_chunks, K);
  if (workspace_bytes < L.tables + (size_t)kInvTables * 65536 * 2 || (reinterpret_cast<uintptr_t>(workspace) & 255))
    return TL_EWORKSPACE;
  uint16_t* tables = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(workspace) + L.tables);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  inv_table_kernel<<<dim3(64, kInvTables), 256, 0, st>>>(tables);
  return launch_commit(idx, bits, n_chunks, K, tables, proofs_out, 0, st);
}

int tl_commit_ex(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int32_t K, uint8_t* proofs_out,
                 void* workspace, size_t workspace_bytes, int32_t co_resident, void* stream) {
  if (n_chunks < 0 || K < 1) return TL_EINVAL;
  if (K > TL_MAX_K) return TL_EUNSUPPORTED;
  if (n_chunks == 0) return TL_OK;
  if (!idx || !bits || !proofs_out || !workspace) return TL_EINVAL;
  const WsLayout L = ws_layout(0, n_chunks, K);
  if (workspace_bytes < L.tables + (size_t)kInvTables * 65536 * 2 || (reinterpret_cast<uintptr_t>(workspace) & 255))
    return TL_EWORKSPACE;
  uint16_t* tables = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(workspace) + L.tables);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  inv_table_kernel<<<dim3(64, kInvTables), 256, 0, st>>>(tables);
  return launch_commit(idx, bits, n_chunks, K, tables, proofs_out, co_resident, st);
}

int tl_prove(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
             int32_t H, int32_t C, int32_t K, int64_t n_chunks, uint8_t* proofs_out,
             int32_t* idx_out, uint16_t* bits_out, void* workspace, size_t workspace_bytes,
             void* stream) {
  int rc = check_shape(n_roll, n_rows, H, C, K, n_chunks);
  if (rc) return rc;
  if (n_chunks == 0 || n_roll == 0) return TL_OK;
  if (!hidden || !row_off || !proofs_out || !workspace) return TL_EINVAL;
  const WsLayout L = ws_layout(n_roll, n_chunks, K);
  if (workspace_bytes < L.total || (reinterpret_cast<uintptr_t>(workspace) & 255)) return TL_EWORKSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int32_t* idx = idx_out ? idx_out : reinterpret_cast<int32_t*>(ws + L.idx);
  uint16_t* bits = bits_out ? bits_out : reinterpret_cast<uint16_t*>(ws + L.bits);
  rc = tl_select(hidden, row_off, n_roll, n_rows, H, C, K, n_chunks, idx, bits, workspace, workspace_bytes, stream);
  if (rc) return rc;
  return tl_commit(idx, bits, n_chunks, K, proofs_out, workspace, workspace_bytes, stream);
}

int tl_verify(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
              int32_t H, int32_t C, int32_t K, int64_t n_chunks, const uint8_t* proofs,
              const tl_thresholds* thresholds_host, tl_chunk_stats* stats_out,
              uint8_t* chunk_accept_out, uint8_t* rollout_accept_out, void* workspace,
              size_t workspace_bytes, void* stream) {
  return tl_verify_ex(hidden, row_off, n_roll, n_rows, H, C, K, n_chunks, proofs, thresholds_host, stats_out,
                      chunk_accept_out, rollout_accept_out, workspace, workspace_bytes, 0, stream);
}

int tl_verify_ex(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
                 int32_t H, int32_t C, int32_t K, int64_t n_chunks, const uint8_t* proofs,
                 const tl_thresholds* thresholds_host, tl_chunk_stats* stats_out,
                 uint8_t* chunk_accept_out, uint8_t* rollout_accept_out, void* workspace,
                 size_t workspace_bytes, int32_t ctas_per_sm, void* stream) {
  int rc = check_shape(n_roll, n_rows, H, C, K, n_chunks);
  if (rc) return rc;
  if (n_roll == 0) return TL_OK;
  if (!hidden || !row_off || !proofs || !thresholds_host || !workspace) return TL_EINVAL;
  const WsLayout L = ws_layout(n_roll, n_chunks, K);
  if (workspace_bytes < L.total || (reinterpret_cast<uintptr_t>(workspace) & 255)) return TL_EWORKSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int64_t* prefix = reinterpret_cast<int64_t*>(ws + L.prefix);
  uint8_t* accept = chunk_accept_out ? chunk_accept_out : ws + L.accept;
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  chunk_prefix_kernel<<<1, 1024, 0, st>>>(row_off, n_roll, C, prefix);
  if (n_chunks > 0) {
    const SelArgs a{hidden, row_off, prefix, n_roll, H, C, K, n_chunks};
    if (cudaFuncSetAttribute(verify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelSmem) !=
        cudaSuccess)
      return TL_ECUDA;
    verify_kernel<<<sel_grid(n_chunks, (const void*)verify_kernel, ctas_per_sm), kSelBlockThreads, kSelSmem,
                    st>>>(
        a, proofs, *thresholds_host, stats_out, accept);
  }
  if (rollout_accept_out)
    rollout_verdict_kernel<<<(n_roll + 7) / 8, 256, 0, st>>>(accept, prefix, n_roll, rollout_accept_out);
  return launch_status();
}

int tl_round6(const void* in, int32_t dtype, int64_t n, double* out, void* stream) {
  if (n < 0 || dtype < 0 || dtype > 3) return TL_EINVAL;
  if (n == 0) return TL_OK;
  if (!in || !out) return TL_EINVAL;
  const int64_t blocks = min((int64_t)sm_count() * 8, (n + 255) / 256);
  round6_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(in, dtype, n, out);
  return launch_status();
}

int tl_synth_bf16(uint16_t* out, int64_t row0, int64_t n_rows, int32_t H, uint64_t seed_mix,
                  int32_t dist, const uint16_t* normal_table, const int32_t* massive_host,
                  int32_t jitter_thr, uint64_t jitter_mix, void* stream) {
  if (n_rows < 0 || row0 < 0 || H < 1 || dist < 0 || dist > 3 || jitter_thr < 0) return TL_EINVAL;
  if (n_rows == 0) return TL_OK;
  if (!out || ((dist == 0 || dist == 1) && !normal_table)) return TL_EINVAL;
  Massive mv;
  for (int i = 0; i < 6; ++i) mv.c[i] = massive_host ? massive_host[i] : -1;
  const int64_t total = n_rows * ((H + 3) / 4);
  const int64_t blocks = min((int64_t)sm_count() * 16, (total + 255) / 256);
  synth_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out, row0, n_rows, H, seed_mix, dist, normal_table, mv, jitter_thr, jitter_mix);
  return launch_status();
}

}  // extern "C"
