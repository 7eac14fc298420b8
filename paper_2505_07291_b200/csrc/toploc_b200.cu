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

#include <cuda.h>  // driver-API types only; the functions come from cudaGetDriverEntryPoint
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>

#include "../../include/toploc_b200.h"
#include "primes.inc"

namespace {

// ----------------------------------------------------------------------------- constants
#ifndef TL_SEL_THREADS
#define TL_SEL_THREADS 32  // one warp per CTA: independent streaming warps (see DESIGN 5.1)
#endif
constexpr int kSelThreads = TL_SEL_THREADS;   // select CTA threads (independent warps)
#ifndef TL_SEL_U
#define TL_SEL_U 8
#endif
// L2 bulk prefetch in the one-warp streaming loop: lane 0 issues one
// cp.async.bulk.prefetch.L2 of TL_L2_PREFETCH_TILES warp tiles (4 KiB each) every that many
// tiles, TL_L2_PREFETCH_AHEAD tiles ahead of the register double buffer's loads.  Measured at
// configuration 2 (tools/stream_probe.py, same process): select 3.057 -> 3.005-3.015 ms,
// verify ~1.5 % faster; more than ~32 KiB ahead per warp (2664 warps) thrashes the 126 MB
// L2 (8 tiles at 16 ahead: 5.1 ms).  0 disables it.
#ifndef TL_L2_PREFETCH_TILES
#define TL_L2_PREFETCH_TILES 4
#endif
#ifndef TL_L2_PREFETCH_AHEAD
#define TL_L2_PREFETCH_AHEAD 2
#endif
constexpr int kSelU = TL_SEL_U;               // 16-B vectors per lane per warp tile
#ifndef TL_SEL_MIN_BLOCKS
#define TL_SEL_MIN_BLOCKS 18
#endif
constexpr int kSelMinBlocks = TL_SEL_MIN_BLOCKS;  // resident select CTAs per SM
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kWarpCap = 256;                 // per-warp candidate buffer (2 KiB)
static_assert(kWarpCap >= TL_MAX_K + 32, "a compaction must leave room for one full ballot");
constexpr int kFlushAt = 4;                   // flagged vectors per exact-test round (32 lanes / 8)
constexpr int kStageVec = 32 * kSelU + 8;     // per-warp flagged-vector queue (< kFlushAt pending + a tile)
#ifndef TL_SPEC_LO
#define TL_SPEC_LO 32   // adapt the margin so a chunk yields kk + [LO, HI] candidates
#endif
#ifndef TL_SPEC_HI
#define TL_SPEC_HI 112  // < kWarpCap - TL_MAX_K: no compaction at the target
#endif
constexpr unsigned kIdxMask = 0xFFFFFFu;      // flat index field (24 bits)
constexpr int kInvTables = 8;                 // precomputed inverse tables (first 8 primes)
constexpr int kHashBits = 8;                  // injectivity check: 256-slot set per commit warp
constexpr int kHashSlots = 1 << kHashBits;
constexpr int kSplitMax = 5;            // small batches: up to 5 warps share one chunk (the last one
                                        // merges the others' lists: more parts cost more merge steps)
constexpr int kSplitMaxLists = 4096;    // partial top-k lists in the workspace
constexpr int kSplitMaxChunks = 2048;   // chunk arrival counters in the workspace
constexpr int kSplitMinPart = 16384;    // elements per part, at least: a part pays a whole chunk's
                                        // final sort, so it must stream long enough to amortise it
constexpr int kSpecSlots = 8192;              // speculation slots in the workspace (16 B each)
#ifndef TL_COMMIT_WARPS
#define TL_COMMIT_WARPS 32
#endif
constexpr int kCommitWarps = TL_COMMIT_WARPS;
#ifndef TL_CO_COMMIT_WARPS
#define TL_CO_COMMIT_WARPS 8  // co-resident commit CTA (pipeline): warps, <= 64 registers each
#endif
constexpr int kCoCommitWarps = TL_CO_COMMIT_WARPS;
#ifndef TL_NDD_UNROLL
#define TL_NDD_UNROLL 2  // divided-difference levels per loop iteration
#endif
#ifndef TL_CONV_UNROLL
#define TL_CONV_UNROLL 2  // Newton -> monomial steps per loop iteration
#endif
constexpr int kNddUnroll = TL_NDD_UNROLL;
constexpr int kConvUnroll = TL_CONV_UNROLL;
constexpr uint32_t kPMax = 65497u;

// ----------------------------------------------------------------------------- checked builds
// -DTL_CHECKED=1 (paper_2505_07291_b200/_build.py: build_checked) compiles device asserts on
// the index, workspace and chunk-geometry arithmetic: a violated bound prints where and
// traps (the launch fails with an error instead of reading or writing out of bounds).  The
// GPU fuzz and parity tests run once more against that library (tests/test_gpu_checked.py);
// compute-sanitizer is not available on the GPU pool, so this is its substitute.
#ifndef TL_CHECKED
#define TL_CHECKED 0
#endif
#if TL_CHECKED
#define TL_CHECK(cond)                                                                              \
  do {                                                                                              \
    if (!(cond)) {                                                                                  \
      printf("TL_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #cond);                                                              \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)
#else
#define TL_CHECK(cond) do {} while (0)
#endif

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

// True iff p is one of the moduli a prover can emit: a prime in [32771, 65497]
// (kPrimesDesc), by one load from the generated membership map (a binary search of the
// constant table cost ~12 dependent constant-cache misses on a latency-bound chunk tail).
__device__ __forceinline__ bool prover_prime(uint32_t p) {
  return p < 65536u && ((__ldg(&kProverModulusBits[p >> 5]) >> (p & 31)) & 1u);
}

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
// One WARP owns one chunk at a time (persistent: first the chunk at its global warp
// id, then chunks claimed from a counter, claim_chunk).  It streams the chunk's 16-byte vectors
// (vector g of warp tile t: t*kWTileVec + u*32 + lane) through a register double
// buffer of non-allocating loads.  Per lane and tile a bf16x2 |max| tree folds the
// 8 U elements into one 16x2 maximum, tested with one add-and-mask against the
// warp's threshold theta; a flagged lane queues its vectors in shared memory and
// queued elements are tested exactly against the composite key in full 32-lane
// rounds.  Survivors go to the warp's candidate buffer (kWarpCap keys); a full
// buffer is compacted (bitonic sort, keep the kk largest, theta = the kk-th), so
// the buffer always holds every element seen with key >= theta and, once theta was
// raised by a compaction, at least kk of them: at the chunk end it contains the
// chunk's top-kk.
//
// There is no barrier anywhere.  The warps of a CTA are independent, so a warp's
// chunk tail (final sort, output, verify-side evaluation) overlaps the other
// warps' streaming and the SM keeps its loads in flight (tools/lab/chunkprobe.py:
// a CTA-wide chunk tail of 8 us costs 6 % of the read rate, a per-warp one 1 %).
//
// A chunk starts from a speculative theta (min of the warp's last two kk-th
// magnitudes minus an adaptive margin).  If the buffer ends with < kk keys the
// speculation excluded part of the top-kk and the chunk is re-scanned with a lower
// threshold: 64, then 256 magnitude steps lower, then 0 (exact).
constexpr int kWTileVec = 32 * kSelU;  // 16-B vectors per warp tile
constexpr int kWTileElems = kWTileVec * 8;

struct WarpSlot {
  unsigned long long wbuf[kWarpCap];  // candidate keys; the sorted top-kk at chunk end
  int sidx[kStageVec];                // queued flagged vector ids
  uint4 stage[kStageVec];             // queued flagged vectors
  uint16_t coef[TL_MAX_K];            // verify: the claimed coefficients
  int lst_n;                          // queue length
};
static_assert(offsetof(WarpSlot, stage) % 16 == 0 && offsetof(WarpSlot, coef) % 16 == 0, "slot alignment");
struct SelState {
  WarpSlot w[kSelWarps];
};
constexpr int kSelBlockThreads = kSelThreads;
constexpr size_t kSelSmem = (sizeof(SelState) + 127) & ~(size_t)127;

// Warp-uniform speculation state, carried in registers from chunk to chunk and,
// through the workspace, from launch to launch (slot = global warp id mod
// kSpecSlots; a slot that does not hold a valid state starts from theta = 0).
// It only steers speed: any theta gives the exact top-kk.
struct Spec {
  unsigned long long theta;  // next chunk's starting threshold
  unsigned k0, k1;           // the last two kk-th magnitudes
  int delta;                 // margin below them, magnitude units
};
constexpr unsigned kSpecMagic = 0x53504543u;
__device__ __forceinline__ void spec_arm(Spec& sp) {
  const unsigned kmag = min(sp.k0, sp.k1);
  sp.theta = kmag > (unsigned)sp.delta ? ((unsigned long long)(kmag - (unsigned)sp.delta) << 40) : 0ull;
}
__device__ __forceinline__ Spec spec_load(const uint4* slots, int64_t gw) {
  const uint4 v = slots[gw % kSpecSlots];
  Spec sp{0ull, 0x7FFFu, 0x7FFFu, 8};
  if (v.w == kSpecMagic && v.x <= 0x7FFFu && v.y <= 0x7FFFu && v.z >= 1u && v.z <= 0x4000u) {
    sp.k0 = v.x;
    sp.k1 = v.y;
    sp.delta = (int)v.z;
    spec_arm(sp);
  }
  return sp;
}
// A warp that selected no chunk this launch (k1 still the initial 0x7FFF) leaves its
// slot alone: storing the untrained state would start a later launch far too high.
__device__ __forceinline__ void spec_store(uint4* slots, int64_t gw, const Spec& sp, int lane) {
  if (lane == 0 && sp.k1 < 0x7FFFu)
    slots[gw % kSpecSlots] = make_uint4(sp.k0, sp.k1, (unsigned)sp.delta, kSpecMagic);
}

#if TL_PHASE_PROF
// Lab instrumentation (-DTL_PHASE_PROF=1): clock64 time per chunk phase summed over
// warps (0 geo, 1 pass, 2 re-scans, 3 sort + speculation, 4 output / verify tail)
// and counters (5 chunks, 6 candidates, 7 re-scanned chunks), 8 theta = 0 passes;
// read by tl_phase_prof.
__device__ unsigned long long g_prof[16];
__device__ unsigned long long g_prof_warp[8192][2];  // per global warp: globaltimer at start / end (ns)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROF_DECL unsigned long long prof_[16] = {}; long long prof_last_ = clock64(); const unsigned long long prof_t0_ = gtimer()
#define PROF_MARK(ph) do { const long long t_ = clock64(); prof_[ph] += t_ - prof_last_; prof_last_ = t_; } while (0)
#define PROF_COUNT(i, v) (prof_[i] += (v))
#define PROF_FLUSH()                                                                            \
  do {                                                                                          \
    if ((threadIdx.x & 31) == 0) {                                                              \
      for (int q_ = 0; q_ < 16; ++q_) atomicAdd(&g_prof[q_], prof_[q_]);                        \
      const int64_t w_ = (int64_t)blockIdx.x * kSelWarps + (threadIdx.x >> 5);                  \
      if (w_ < 8192) { g_prof_warp[w_][0] = prof_t0_; g_prof_warp[w_][1] = gtimer(); }          \
    }                                                                                           \
  } while (0)
#define PROF_ARG , unsigned long long (&prof_)[16], long long& prof_last_
#define PROF_PASS , prof_, prof_last_
#else
#define PROF_DECL do {} while (0)
#define PROF_MARK(ph) do {} while (0)
#define PROF_COUNT(i, v) do {} while (0)
#define PROF_FLUSH() do {} while (0)
#define PROF_ARG
#define PROF_PASS
#endif

__device__ __forceinline__ unsigned hmaxabs2(unsigned a, unsigned b) {
  unsigned d;  // per bf16 half: max(|a|, |b|) (sign = xor, masked off by the caller); NaN wins
  asm("max.NaN.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ bool coarse_hit(unsigned m, unsigned c2) {
  return (((m & 0x7FFF7FFFu) + c2) & 0x80008000u) != 0u;
}
// Coarse-test bits of one 16-B vector's 8 elements (bit e: |element e| >= the tile threshold).
__device__ __forceinline__ uint32_t elem_mask8(const uint4& v, unsigned c2) {
  const uint32_t f0 = ((v.x & 0x7FFF7FFFu) + c2) & 0x80008000u, f1 = ((v.y & 0x7FFF7FFFu) + c2) & 0x80008000u;
  const uint32_t f2 = ((v.z & 0x7FFF7FFFu) + c2) & 0x80008000u, f3 = ((v.w & 0x7FFF7FFFu) + c2) & 0x80008000u;
  return ((f0 >> 15) & 1u) | ((f0 >> 30) & 2u) | ((f1 >> 13) & 4u) | ((f1 >> 28) & 8u) | ((f2 >> 11) & 16u) |
         ((f2 >> 26) & 32u) | ((f3 >> 9) & 64u) | ((f3 >> 24) & 128u);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// ---- chunk geometry
struct ChunkGeo {
  const uint16_t* base;  // first element
  int n;                 // elements
  int a0;                // scalar head elements before the first 16-B boundary
  int nvec;              // 16-B vectors after the head
  int nst;               // warp tiles
};
struct SelArgs {
  const uint16_t* hidden;
  const int64_t* row_off;
  const int64_t* prefix;
  uint4* spec;       // workspace: speculation state per warp slot, kept across launches
  unsigned long long* next;  // workspace: chunks handed out beyond the first round (reset by chunk_prefix_kernel)
  int n_roll, H, C, K;
  int64_t n_chunks;  // caller's n_chunks (clamped to prefix[n_roll] in the kernels)
  int split = 1;                            // warps per chunk (small batches, sel_plan)
  unsigned long long* part = nullptr;       // workspace: [n_chunks][split][K] partial top-k keys
  unsigned* part_cnt = nullptr;             // workspace: per-chunk arrivals (zeroed by chunk_prefix_kernel)
  int64_t n_rows = 0;                       // rows of hidden (bounds checks of -DTL_CHECKED builds)
  int64_t* prefix_out = nullptr;            // ring kernels, small batches: prefix == nullptr, the kernel
                                            // builds it in shared memory and CTA 0 stores it here
};
// Chunk scheduling: the first round is static (chunk = global warp id), later chunks
// are claimed from a workspace counter, so warps that stream faster (SMs with fewer
// resident CTAs, better HBM placement) take more chunks and all warps finish within
// about one chunk of each other.  Lane 0 claims at the chunk start; the claim is
// broadcast at the chunk end, so the atomic's latency hides behind the chunk.
__device__ __forceinline__ unsigned long long claim_chunk(const SelArgs& a, int lane) {
  return lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
}

__device__ __forceinline__ ChunkGeo chunk_geo(const SelArgs& a, int64_t j) {
  const ChunkRef cr = locate_chunk(a.prefix, a.row_off, a.n_roll, j, a.C);
  TL_CHECK(j >= 0 && cr.rollout >= 0 && cr.rollout < a.n_roll && cr.rows >= 1 && cr.rows <= a.C);
  TL_CHECK(cr.row_start >= 0 && cr.row_start + cr.rows <= a.n_rows);
  ChunkGeo g;
  g.base = a.hidden + cr.row_start * (int64_t)a.H;
  g.n = cr.rows * a.H;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(g.base);
  g.a0 = min(g.n, (int)(((16u - (unsigned)(addr & 15u)) & 15u) >> 1));
  g.nvec = (g.n - g.a0) >> 3;
  g.nst = (g.nvec + kWTileVec - 1) / kWTileVec;
  return g;
}

// Warp bitonic sort, descending, of NPER*32 keys held as a[r] at position r*32+lane.
template <typename T, int NPER>
__device__ __forceinline__ void warp_bitonic_desc(T (&a)[NPER], int lane) {
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
            const T x = a[r], y = a[r | rj];
            const T hi = x > y ? x : y, lo = x > y ? y : x;
            a[r] = desc ? hi : lo;
            a[r | rj] = desc ? lo : hi;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < NPER; ++r) {
          const T o = __shfl_xor_sync(0xFFFFFFFFu, a[r], j);
          const bool desc = (((r * 32 + lane) & k) == 0);
          const bool lower = (lane & j) == 0;
          const T hi = a[r] > o ? a[r] : o, lo = a[r] > o ? o : a[r];
          a[r] = (desc == lower) ? hi : lo;
        }
      }
    }
  }
}

// Rank wb[0..cnt) descending in place (chunk end and buffer compaction).  When the
// keys' indices are < 2^19 - 1 and their magnitudes span < 2^12 above the minimum
// `base` (the usual case), the keys are ranked as 32-bit words
//     (mag - base) << 20 | (2^19 - 1 - idx) << 1 | sign,
// which order like the 64-bit keys ((mag, idx) is unique, so the sign never
// decides) at half the shuffles and compares; otherwise as 64-bit keys.
template <int NPER, int WMAX = NPER * 32>  // writes back wb[0 .. WMAX) only
__device__ __forceinline__ void final_sort(unsigned long long* wb, int cnt, int lane) {
  unsigned long long a[NPER];
  unsigned lo = 0xFFFFu, hi = 0u, imax = 0u;
#pragma unroll
  for (int r = 0; r < NPER; ++r) {
    const int q = r * 32 + lane;
    a[r] = q < cnt ? wb[q] : 0ull;
    if (q < cnt) {
      lo = min(lo, (unsigned)(a[r] >> 40));
      hi = max(hi, (unsigned)(a[r] >> 40));
      imax = max(imax, key_idx(a[r]));
    }
  }
  const unsigned base = __reduce_min_sync(0xFFFFFFFFu, lo);
  hi = __reduce_max_sync(0xFFFFFFFFu, hi);
  imax = __reduce_max_sync(0xFFFFFFFFu, imax);
  if (hi - base < 4096u && imax < 0x7FFFFu) {
    uint32_t k[NPER];
#pragma unroll
    for (int r = 0; r < NPER; ++r) {
      const unsigned mag = (unsigned)(a[r] >> 40);
      k[r] = r * 32 + lane < cnt ? ((mag - base) << 20) | ((0x7FFFFu - key_idx(a[r])) << 1) |
                                       (unsigned)((a[r] >> 15) & 1u)
                                 : 0u;
    }
    warp_bitonic_desc<uint32_t, NPER>(k, lane);
#pragma unroll
    for (int r = 0; r < NPER; ++r)
      if (r * 32 < WMAX)
        wb[r * 32 + lane] = k[r] ? make_key(((k[r] & 1u) << 15) | (base + (k[r] >> 20)), 0x7FFFFu - ((k[r] >> 1) & 0x7FFFFu))
                                 : 0ull;
  } else {
    warp_bitonic_desc<unsigned long long, NPER>(a, lane);
#pragma unroll
    for (int r = 0; r < NPER; ++r)
      if (r * 32 < WMAX) wb[r * 32 + lane] = a[r];
  }
  __syncwarp();
}


// Buffer full: keep the warp's kk largest keys; returns theta = the kk-th (rare path).
__device__ __noinline__ unsigned long long warp_compact(unsigned long long* wb, int cnt, int kk, int lane) {
  final_sort<kWarpCap / 32>(wb, cnt, lane);
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
  TL_CHECK(cnt + __popc(bal) <= kWarpCap);
  if (p) wb[cnt + __popc(bal & lanemask_lt())] = key;
  cnt += __popc(bal);
  __syncwarp();
}

// Per-warp streaming state (all members warp-uniform except the pointers' targets).
struct WarpScan {
  unsigned long long theta;
  int cnt;
  unsigned long long* wb;
  int* sidx;   // queued flagged vector ids
  uint4* stg;  // queued flagged vectors (copied out of registers)
  int* lst_n;  // queue length
};

__device__ __forceinline__ unsigned coarse_c2(unsigned long long theta, unsigned lo) {
  const unsigned tkey = (unsigned)(theta >> 40);
  // elements tied with theta's magnitude lose on index once lo > theta's index
  const unsigned tk = tkey + (lo > key_idx(theta) ? 1u : 0u);
  return ((0x8000u - tk) & 0xFFFFu) * 0x10001u;
}

// Test the elements of the n queued vectors lane-parallel, append survivors and
// empty the queue.  Element e of the batch is vector sidx[e >> 3], bf16 (e & 7).
__device__ __forceinline__ void flush_flagged(const ChunkGeo& cg, WarpScan& w, int n, int kk, int lane) {
  const uint16_t* stg16 = reinterpret_cast<const uint16_t*>(w.stg);
  const unsigned tkey = (unsigned)(w.theta >> 40);
  for (int e0 = 0; e0 < 8 * n; e0 += 32) {
    const int e = e0 + lane;
    bool p = false;
    unsigned long long key = 0;
    if (e < 8 * n) {
      const unsigned b = stg16[e];
      if ((b & 0x7FFFu) >= tkey) {
        key = make_key(b, (unsigned)(cg.a0 + 8 * w.sidx[e >> 3] + (e & 7)));
        p = key >= w.theta;
      }
    }
    warp_append(p, key, w.wb, w.cnt, w.theta, kk, lane);
  }
  __syncwarp();
  if (lane == 0) *w.lst_n = 0;
  __syncwarp();
}

// One pass of the warp over its chunk straight from HBM with a register double
// buffer; flagged vectors are queued with one shared-memory atomic per flagged
// lane and tested in full 32-lane rounds once >= kFlushAt are pending.
__device__ __forceinline__ void pass_warp(const ChunkGeo& cg, WarpScan& w, int kk, int lane) {
  const uint4* __restrict__ vb = reinterpret_cast<const uint4*>(cg.base + cg.a0);
  const int nvec = cg.nvec, a0 = cg.a0;
  uint4 vn[kSelU];
#pragma unroll
  for (int u = 0; u < kSelU; ++u) {
    const int g = lane + u * 32;
    vn[u] = g < nvec ? ld_stream(vb + g) : make_uint4(0u, 0u, 0u, 0u);
  }
#if TL_L2_PREFETCH_TILES
  // bulk L2 prefetch of the chunk's first TL_L2_PREFETCH_AHEAD tiles, then a group of
  // TL_L2_PREFETCH_TILES tiles that far ahead every TL_L2_PREFETCH_TILES tiles (lane 0)
  if (lane == 0) {
    const int v0 = 0, v1 = min(nvec, (TL_L2_PREFETCH_AHEAD) * kWTileVec);
    if (v1 > v0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vb + v0), "r"((unsigned)(v1 - v0) * 16u) : "memory");
  }
#endif
  for (int it = 0; it < cg.nst; ++it) {
    const int gbase = it * kWTileVec + lane;
#if TL_L2_PREFETCH_TILES
    if (lane == 0 && it % TL_L2_PREFETCH_TILES == 0) {
      const int v0 = (it + TL_L2_PREFETCH_AHEAD) * kWTileVec;
      const int v1 = min(nvec, v0 + TL_L2_PREFETCH_TILES * kWTileVec);
      if (v1 > v0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vb + v0), "r"((unsigned)(v1 - v0) * 16u) : "memory");
    }
#endif
    uint4 v[kSelU];
#pragma unroll
    for (int u = 0; u < kSelU; ++u) {
      v[u] = vn[u];
      const int g = gbase + kWTileVec + u * 32;
      vn[u] = g < nvec ? ld_stream(vb + g) : make_uint4(0u, 0u, 0u, 0u);
    }
    const unsigned c2 = coarse_c2(w.theta, (unsigned)(a0 + it * kWTileElems));
    unsigned mu[kSelU];
#pragma unroll
    for (int u = 0; u < kSelU; ++u) mu[u] = hmaxabs2(hmaxabs2(v[u].x, v[u].y), hmaxabs2(v[u].z, v[u].w));
    unsigned m = mu[0];
#pragma unroll
    for (int u = 1; u < kSelU; ++u) m = hmaxabs2(m, mu[u]);
    const bool hit = coarse_hit(m, c2);
    if (!__any_sync(0xFFFFFFFFu, hit)) continue;
    // vectors past the chunk end are zero and never flagged
    if (hit) {
      unsigned hm = 0;
#pragma unroll
      for (int u = 0; u < kSelU; ++u)
        hm |= ((gbase + u * 32 < nvec && coarse_hit(mu[u], c2)) ? 1u : 0u) << u;
      if (hm) {
        int pos = atomicAdd(w.lst_n, __popc(hm));
        TL_CHECK(pos + __popc(hm) <= kStageVec);
#pragma unroll
        for (int u = 0; u < kSelU; ++u) {
          if ((hm >> u) & 1u) {
            w.stg[pos] = v[u];
            w.sidx[pos] = gbase + u * 32;
            ++pos;
          }
        }
      }
    }
    __syncwarp();
    const int pending = *reinterpret_cast<volatile int*>(w.lst_n);
    if (pending >= kFlushAt) flush_flagged(cg, w, pending, kk, lane);
  }
  const int pending = *reinterpret_cast<volatile int*>(w.lst_n);
  if (pending > 0) flush_flagged(cg, w, pending, kk, lane);
}

// Top-kk of chunk cg -> slot.wbuf[0..kk) in rank order (descending key).
// Warp-level; sp carries the speculation from chunk to chunk.  Returns the
// candidate count of the final pass.
__device__ int select_chunk(const ChunkGeo& cg, int kk, WarpSlot& slot, Spec& sp, int lane PROF_ARG) {
  WarpScan w;
  w.wb = slot.wbuf;
  w.sidx = slot.sidx;
  w.stg = slot.stage;
  w.lst_n = &slot.lst_n;
  const int tail0 = cg.a0 + (cg.nvec << 3);
  unsigned long long theta0 = sp.theta;
  int retry = 0;
  for (;;) {
    w.theta = theta0;
    w.cnt = 0;
    {  // scalar head / tail elements (chunks not 16-B aligned)
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
    pass_warp(cg, w, kk, lane);
    PROF_MARK(retry ? 2 : (theta0 ? 1 : 8));
    if (w.cnt >= kk) break;
    // the speculative theta excluded part of the top-kk: re-scan with a lower one
    if (theta0 == 0ull) __trap();  // unreachable: theta = 0 admits every element
    const unsigned key = (unsigned)(theta0 >> 40);
    const unsigned drop = retry == 0 ? 64u : 256u;
    theta0 = (retry < 2 && key > drop) ? ((unsigned long long)(key - drop) << 40) : 0ull;
    PROF_COUNT(7, retry == 0);
    ++retry;
    sp.delta = min(sp.delta + 4, 0x4000);
  }
  const int cnt = w.cnt;
  if (cnt <= 64) final_sort<2>(w.wb, cnt, lane);
  else if (cnt <= 128) final_sort<4>(w.wb, cnt, lane);
  else final_sort<8>(w.wb, cnt, lane);
  // speculation for this warp's next chunk
  // (theta only rises by a buffer compaction: a compacting chunk had too many candidates)
  int d = sp.delta;
  if ((cnt > kk + TL_SPEC_HI || w.theta != theta0) && d > 1) --d;
  else if (cnt < kk + TL_SPEC_LO) ++d;
  sp.delta = d;
  sp.k0 = sp.k1;
  sp.k1 = (unsigned)(w.wb[kk - 1] >> 40);
  spec_arm(sp);
  PROF_COUNT(5, 1);
  PROF_COUNT(6, cnt);
  PROF_MARK(3);
  return cnt;
}

// ---- small batches: S warps share a chunk
// Part s of a chunk is the element range [lo, hi) (8-element aligned relative to the
// chunk).  The chunk's top-kk is contained in the union of its parts' top-kk, and a
// part's keys become chunk keys by re-basing the index (key - (lo << 16): the index is
// stored as kIdxMask - idx).  The last part to finish merges the lists.
__device__ __forceinline__ ChunkGeo sub_geo(const ChunkGeo& g, int lo, int hi) {
  ChunkGeo s;
  s.base = g.base + lo;
  s.n = hi - lo;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(s.base);
  s.a0 = min(s.n, (int)(((16u - (unsigned)(addr & 15u)) & 15u) >> 1));
  s.nvec = (s.n - s.a0) >> 3;
  s.nst = (s.nvec + kWTileVec - 1) / kWTileVec;
  return s;
}

// Sort a bitonic sequence of 128 keys (a[r] at position 32 r + lane) descending.
__device__ __forceinline__ void bitonic_merge_desc128(unsigned long long (&a)[4], int lane) {
#pragma unroll
  for (int rj = 2; rj >= 1; rj >>= 1) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if ((r & rj) == 0) {
        const unsigned long long x = a[r], y = a[r | rj];
        a[r] = x > y ? x : y;
        a[r | rj] = x > y ? y : x;
      }
    }
  }
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, a[r], j);
      a[r] = (lane & j) ? (a[r] < y ? a[r] : y) : (a[r] > y ? a[r] : y);
    }
  }
}

// Part s of chunk j: select its top-k and publish it; if this is the chunk's last part
// to finish, merge every part into slot.wbuf[0..kk) and return true.
__device__ __forceinline__ bool select_split(const SelArgs& a, const ChunkGeo& g, int kk, int64_t j, int s,
                                          WarpSlot& slot, Spec& sp, int lane PROF_ARG) {
  const int S = a.split, K = a.K;
  const int lo = s == 0 ? 0 : (int)(((int64_t)g.n * s / S) & ~7ll);
  const int hi = s == S - 1 ? g.n : (int)(((int64_t)g.n * (s + 1) / S) & ~7ll);
  const int kks = min(K, hi - lo);
  if (kks > 0) select_chunk(sub_geo(g, lo, hi), kks, slot, sp, lane PROF_PASS);
  TL_CHECK(j < kSplitMaxChunks && (j * S + s + 1) * K <= (int64_t)kSplitMaxLists * TL_MAX_K && lo <= hi && hi <= g.n);
  unsigned long long* mine = a.part + ((size_t)j * S + s) * K;
  for (int i = lane; i < K; i += 32) mine[i] = i < kks ? slot.wbuf[i] - ((unsigned long long)lo << 16) : 0ull;
  __threadfence();
  __syncwarp();
  unsigned arrived = 0;
  if (lane == 0) arrived = atomicAdd(a.part_cnt + j, 1u);
  arrived = __shfl_sync(0xFFFFFFFFu, arrived, 0);
  if (arrived != (unsigned)(S - 1)) return false;
  __threadfence();
  // top-K of the union: acc <- bitonic merge of (acc, list q reversed), one list at a time
  const unsigned long long* parts = a.part + (size_t)j * S * K;
  unsigned long long acc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int p = 32 * r + lane;
    acc[r] = p < K ? __ldcg(parts + p) : 0ull;
  }
  for (int q = 1; q < S; ++q) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int p = 127 - (32 * r + lane);
      const unsigned long long b = p < K ? __ldcg(parts + (size_t)q * K + p) : 0ull;
      acc[r] = acc[r] > b ? acc[r] : b;
    }
    bitonic_merge_desc128(acc, lane);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int p = 32 * r + lane;
    if (p < kk) slot.wbuf[p] = acc[r];
  }
  __syncwarp();
  return true;
}

// ----------------------------------------------------------------------------- kernels
__global__ void chunk_prefix_kernel(const int64_t* __restrict__ row_off, int n_roll, int C,
                                    int64_t* __restrict__ prefix, unsigned long long* __restrict__ next_chunk,
                                    unsigned* __restrict__ part_cnt) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) { carry = 0; prefix[0] = 0; *next_chunk = 0; }
  if (part_cnt)
    for (int i = tid; i < kSplitMaxChunks; i += blockDim.x) part_cnt[i] = 0u;
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

template <bool SPLIT>
__global__ void __launch_bounds__(kSelBlockThreads, kSelMinBlocks)
prove_select_kernel(SelArgs a, int32_t* __restrict__ idx_out, uint16_t* __restrict__ bits_out) {
  extern __shared__ __align__(128) uint8_t sel_smem[];
  WarpSlot& slot = reinterpret_cast<SelState*>(sel_smem)->w[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  if (lane == 0) slot.lst_n = 0;
  __syncwarp();
  const int64_t n_chunks = min(a.n_chunks, a.prefix[a.n_roll]);
  const int64_t nw = (int64_t)gridDim.x * kSelWarps;
  const int K = a.K;
  const int64_t gw = (int64_t)blockIdx.x * kSelWarps + (threadIdx.x >> 5);
  Spec sp = spec_load(a.spec, gw);
  PROF_DECL;
  const int S = SPLIT ? a.split : 1;
  for (int64_t j = SPLIT ? gw / S : gw; j < n_chunks;) {
    const unsigned long long claim = SPLIT ? 0ull : claim_chunk(a, lane);
    const ChunkGeo g = chunk_geo(a, j);
    const int kk = min(K, g.n);
    PROF_MARK(0);
    if (SPLIT) {
      if (!select_split(a, g, kk, j, (int)(gw % S), slot, sp, lane PROF_PASS)) break;  // another part merges
    } else {
      select_chunk(g, kk, slot, sp, lane PROF_PASS);
    }
    TL_CHECK(j < n_chunks && kk <= K && K <= TL_MAX_K);
    for (int i = lane; i < K; i += 32) {
      if (i < kk) {
        const unsigned long long v = slot.wbuf[i];
        TL_CHECK(key_idx(v) < (unsigned)g.n);
        idx_out[j * K + i] = (int32_t)key_idx(v);
        bits_out[j * K + i] = (uint16_t)(v & 0xFFFFu);
      } else {
        idx_out[j * K + i] = -1;
        bits_out[j * K + i] = 0;
      }
    }
    __syncwarp();
    PROF_MARK(4);
    if (SPLIT) break;  // one part per warp
    j = nw + (int64_t)__shfl_sync(0xFFFFFFFFu, claim, 0);
  }
  spec_store(a.spec, gw, sp, lane);
  PROF_FLUSH();
}

// Inverse tables of the first kInvTables primes: inv(a) for a in [1, p), 0 elsewhere.
// Montgomery's batch inversion over runs of kInvRun consecutive values -- prefix
// products, one Fermat inverse per run, back-substitution -- costs ~3 multiplications
// per entry instead of a ~24-multiplication power each (10.5 us -> a few us per call,
// which matters for small batches).
//
// The tables are a pure function of the primes, so they live in module memory, built once
// per device: the first tl_commit's inv_table_kernel builds them and its last CTA raises
// g_inv_ready; every later call only resets the commitment's chunk counter and returns
// (~1 us instead of 4-6 us on the latency-bound small batches).  Concurrent first calls on
// several streams each build identical values.
constexpr int kInvRun = 16;
constexpr int kInvTableThreads = 256;
constexpr int kInvTableBlocks = 65536 / (kInvRun * kInvTableThreads);  // per table
constexpr unsigned kInvReady = 0x494E5654u;
__device__ __align__(128) uint16_t g_inv_tables[kInvTables * 65536];
__device__ unsigned g_inv_ready;
__device__ unsigned g_inv_pieces[(kInvTableBlocks * kInvTables + 31) / 32];  // written pieces, one bit each
__global__ void inv_table_kernel(unsigned long long* __restrict__ next) {
  const int q = blockIdx.y;
  if (next && blockIdx.x == 0 && q == 0 && threadIdx.x == 0) *next = 0;  // commit_kernel's chunk counter
  if (*reinterpret_cast<volatile unsigned*>(&g_inv_ready) == kInvReady) return;
  uint16_t* tables = g_inv_tables;
  const uint32_t p = kPrimesDesc[q];
  const ModP m(p);
  const uint32_t a0 = (blockIdx.x * blockDim.x + threadIdx.x) * kInvRun;
  uint32_t pre[kInvRun];  // pre[i]: product of the run's invertible values before a0 + i
  uint32_t acc = 1;
#pragma unroll
  for (int i = 0; i < kInvRun; ++i) {
    const uint32_t a = a0 + i;
    pre[i] = acc;
    if (a != 0 && a < p) acc = m.mul(acc, a);
  }
  uint32_t inv = m.pow(acc, p - 2);  // (product of the invertible values up to i)^-1
  uint32_t out[kInvRun / 2];  // two 16-bit entries per word, little-endian
#pragma unroll
  for (int i = kInvRun - 1; i >= 0; --i) {
    const uint32_t a = a0 + i;
    uint32_t r = 0;
    if (a != 0 && a < p) {
      r = m.mul(inv, pre[i]);
      inv = m.mul(inv, a);
    }
    if (i & 1) out[i >> 1] = r << 16;
    else out[i >> 1] |= r;
  }
  uint4* dst = reinterpret_cast<uint4*>(tables + (size_t)q * 65536u + a0);
#pragma unroll
  for (int v = 0; v < kInvRun / 8; ++v) dst[v] = make_uint4(out[4 * v], out[4 * v + 1], out[4 * v + 2], out[4 * v + 3]);
  __syncthreads();
  if (threadIdx.x == 0) {
    // mark this piece written; the CTA that completes the set raises the flag.  Per-piece
    // bits (not a count) keep concurrent first launches on several streams safe: the flag
    // never rises before every piece was written by some launch.
    __threadfence();
    constexpr int kWords = (kInvTableBlocks * kInvTables + 31) / 32;
    const int piece = q * kInvTableBlocks + blockIdx.x;
    atomicOr(&g_inv_pieces[piece >> 5], 1u << (piece & 31));
    __threadfence();
    bool all = true;
    for (int w = 0; w < kWords; ++w) {
      const int bits_in = min(32, kInvTableBlocks * kInvTables - 32 * w);
      const unsigned want = bits_in == 32 ? 0xFFFFFFFFu : (1u << bits_in) - 1u;
      all = all && (atomicOr(&g_inv_pieces[w], 0u) & want) == want;
    }
    if (all) atomicExch(&g_inv_ready, kInvReady);
  }
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

#ifndef TL_COMMIT_PROF
#define TL_COMMIT_PROF 0
#endif
#if TL_COMMIT_PROF
// Lab instrumentation (-DTL_COMMIT_PROF=1): clock64 cycles per commitment phase of global
// warp 0 (0 table staging, 1 idx/bits load, 2 modulus, 3 divided differences,
// 4 conversion, 5 serialise; 7 chunks), summed over launches; read by tl_commit_prof.
__device__ unsigned long long g_cprof[8];
__device__ long long g_cprof_last;
#define CP_MARK(ph)                                                                   \
  do {                                                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                        \
      const long long t_ = clock64();                                                 \
      if ((ph) >= 0) g_cprof[(ph) < 0 ? 0 : (ph)] += (unsigned long long)(t_ - g_cprof_last); \
      g_cprof_last = t_;                                                              \
    }                                                                                 \
  } while (0)
#define CC_MARK(ph)                                                                   \
  do {                                                                                \
    const long long t_ = clock64();                                                   \
    cc_acc_[ph] += t_ - cc_last_;                                                     \
    cc_last_ = t_;                                                                    \
    if ((ph) == 5 && blockIdx.x == 0 && threadIdx.x == 0)                             \
      for (int i_ = 0; i_ < 6; ++i_) g_cprof[i_] += (unsigned long long)cc_acc_[i_];  \
  } while (0)
#else
#define CP_MARK(ph) do {} while (0)
#define CC_MARK(ph) do {} while (0)
#endif

// Newton divided differences, levels jl in [j0, j1) with j1 <= 32 (R0 + 1): the
// register blocks r < R0 are complete (i < jl) and skipped at compile time; in
// block R0 lanes with i < jl keep their value.  c[i] <- (c[i] - c[i-1]) / (x[i] - x[i-jl]).
template <int MODE, int R0, int UNR>
__device__ __forceinline__ void ndd_levels(int j0, int j1, const uint32_t (&x)[4], uint32_t (&c)[4],
                                           const uint32_t* xs, const ModP& m, const uint16_t* tab, int lane) {
  const int src = (lane + 31) & 31;
#pragma unroll UNR
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
// nxs[i] = p - x_i.  Coefficient k takes prev_{k-1} + (p - x_i) a_k (< p^2 < 2^32); the
// constant term's "previous" is c_i itself, which folds the + c_i into the same reduction.
template <int RM, int UNR>
__device__ __forceinline__ void conv_steps(int i_hi, int i_lo, uint32_t (&poly)[4], const uint32_t* nxs,
                                           const uint32_t* cs, const ModP& m, int lane) {
  const int src = (lane + 31) & 31;
#pragma unroll UNR
  for (int i = i_hi; i >= i_lo; --i) {
    const uint32_t nxi = nxs[i], ci = cs[i];
    uint32_t t[4];
#pragma unroll
    for (int r = 0; r <= RM; ++r) t[r] = __shfl_sync(0xFFFFFFFFu, poly[r], src);
#pragma unroll
    for (int r = 0; r <= RM; ++r) {
      const uint32_t prevk = lane ? t[r] : (r ? t[r > 0 ? r - 1 : 0] : ci);
      poly[r] = m.red(prevk + nxi * poly[r]);
    }
  }
}

// Interpolate the warp's kk points (x_i, y_i), i = lane + 32 r, over GF(p):
// Newton divided differences, then Newton -> monomial.
template <int MODE, int NU, int CU>
__device__ __forceinline__ void interpolate_warp(const uint32_t (&x)[4], uint32_t (&c)[4], uint32_t (&poly)[4],
                                                 uint32_t* xs, uint32_t* cs, int kk, const ModP& m,
                                                 const uint16_t* tab, int lane) {
  ndd_levels<MODE, 0, NU>(1, min(kk, 32), x, c, xs, m, tab, lane);
  ndd_levels<MODE, 1, NU>(32, min(kk, 64), x, c, xs, m, tab, lane);
  ndd_levels<MODE, 2, NU>(64, min(kk, 96), x, c, xs, m, tab, lane);
  ndd_levels<MODE, 3, NU>(96, kk, x, c, xs, m, tab, lane);
  CP_MARK(3);
  __syncwarp();  // every lane is done reading xs
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    cs[lane + 32 * r] = c[r];
    xs[lane + 32 * r] = m.p - x[r];  // the conversion multiplies by (X - x_i)
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 4; ++r) poly[r] = 0u;
  if (lane == 0) poly[0] = cs[kk - 1];
  // step i yields degree kk-1-i: blocks r <= (kk-1-i) >> 5 are live
  conv_steps<0, CU>(kk - 2, max(kk - 32, 0), poly, xs, cs, m, lane);
  conv_steps<1, CU>(kk - 33, max(kk - 64, 0), poly, xs, cs, m, lane);
  conv_steps<2, CU>(kk - 65, max(kk - 96, 0), poly, xs, cs, m, lane);
  conv_steps<3, CU>(kk - 97, 0, poly, xs, cs, m, lane);
  CP_MARK(4);
}

// One warp commits one chunk: modulus search, GF(p) interpolation and the 258-byte
// serialisation.  The chunk's kk selected (flat index, bf16 bits) pairs are
// raw[r], yb[r] at i = lane + 32 r (raw = 0xFFFFFFFF past kk).  MODE0 is the
// inverse source for the first prime (tab0); primes 2..8 use the global tables,
// later ones Fermat.  xs / cs: 128-word per-warp shared scratch.
// True iff the warp's kk residues res[r] (i = lane + 32 r < kk, each < 2^16) are
// pairwise distinct: insert into a 256-slot open-addressing set in shared memory
// (hs, per warp) with atomicCAS; an insert that finds its own value is a duplicate.
__device__ __forceinline__ bool residues_distinct(const uint32_t (&res)[4], int kk, uint32_t* hs, int lane) {
#pragma unroll
  for (int q = 0; q < kHashSlots / 32; ++q) hs[lane + 32 * q] = 0xFFFFFFFFu;
  __syncwarp();
  bool dup = false;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (lane + 32 * r < kk) {
      const uint32_t v = res[r];
      uint32_t h = (v * 0x9E3779B1u) >> (32 - kHashBits);
      for (;;) {  // load <= 1/2: ~1.5 probes on average
        const uint32_t old = atomicCAS(&hs[h], 0xFFFFFFFFu, v);
        if (old == 0xFFFFFFFFu) break;
        if (old == v) { dup = true; break; }
        h = (h + 1) & (kHashSlots - 1);
      }
    }
  }
  const bool any_dup = __any_sync(0xFFFFFFFFu, dup);
  __syncwarp();
  return !any_dup;
}

template <int MODE0, int NU = kNddUnroll, int CU = kConvUnroll>
__device__ __forceinline__ void commit_chunk(const uint32_t (&raw)[4], const uint32_t (&yb)[4], int kk, int K,
                                             const uint16_t* tab0, const uint16_t* __restrict__ inv_tables,
                                             uint32_t* xs, uint32_t* cs, uint32_t* hs, uint8_t* __restrict__ pr,
                                             int lane) {
  const int PB = 2 + 2 * K;
  uint32_t maxidx = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (lane + 32 * r < kk) maxidx = max(maxidx, raw[r]);
  maxidx = __reduce_max_sync(0xFFFFFFFFu, maxidx);

  // ---- modulus: largest prime with injective residues
  int pi = 0;
  uint32_t p = kPMax;
  if (maxidx >= kPMax) {
    for (pi = 0; pi < TL_N_PRIMES; ++pi) {
      p = kPrimesDesc[pi];
      const ModP mp(p);
      uint32_t res[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) res[r] = mp.red(raw[r]);
      if (residues_distinct(res, kk, hs, lane)) break;
    }
    if (pi == TL_N_PRIMES) p = 0;
  }
  if (p == 0) {  // unprovable chunk: p = 0, zero coefficients
    for (int b = lane; b < PB; b += 32) pr[b] = 0;
    return;
  }
  CP_MARK(2);
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
  if (pi == 0) interpolate_warp<MODE0, NU, CU>(x, c, poly, xs, cs, kk, m, tab0, lane);
  else if (pi < kInvTables) interpolate_warp<kInvGlobal, NU, CU>(x, c, poly, xs, cs, kk, m, inv_tables + (size_t)pi * 65536u, lane);
  else interpolate_warp<kInvFermat, NU, CU>(x, c, poly, xs, cs, kk, m, nullptr, lane);

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
  CP_MARK(5);
}

// ---- TMA bulk copy global -> shared with an mbarrier (the commitment's table staging)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred done;\n WAIT_%=: mbarrier.try_wait.parity.shared.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// tl_commit: one warp per chunk over (idx, bits) in global memory.  WARPS x 32
// threads, one CTA per SM, the first prime's inverse table staged in shared memory
// (HALF = 64 KiB half table and <= 64 registers, so the CTA fits beside 16 one-warp
// select/verify CTAs for the overlapped pipeline, api.Pipeline).
template <int WARPS, bool HALF>
__global__ void __launch_bounds__(WARPS * 32, HALF ? 1024 / (WARPS * 32) : 1)
commit_kernel(const int32_t* __restrict__ idx, const uint16_t* __restrict__ bits, int64_t n_chunks,
              int K, uint8_t* __restrict__ proofs, unsigned long long* __restrict__ next) {
  const uint16_t* inv_tables = g_inv_tables;
  constexpr int kTabEntries = HALF ? kHalfTab : 65536;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint16_t* inv0 = reinterpret_cast<uint16_t*>(smem_raw);
  uint32_t* xs_all = reinterpret_cast<uint32_t*>(smem_raw + kTabEntries * 2);  // [warps][128]
  uint32_t* cs_all = xs_all + WARPS * 128;                                     // [warps][128]
  uint32_t* hs_all = cs_all + WARPS * 128;                                     // [warps][kHashSlots]
  // stage the first prime's inverse table with TMA bulk copies: the whole table is in
  // flight at once (a load loop over few warps would pay one L2 round trip per step,
  // ~16 us for a 4-warp CTA -- the small-batch commitment's largest cost)
  __shared__ __align__(8) uint64_t tab_bar;
  CP_MARK(-1);
  if (threadIdx.x == 0) mbar_init(&tab_bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    constexpr uint32_t kBytes = kTabEntries * 2, kPiece = 32768;
    mbar_expect_tx(&tab_bar, kBytes);
#pragma unroll
    for (uint32_t off = 0; off < kBytes; off += kPiece)
      bulk_copy_g2s(smem_raw + off, reinterpret_cast<const uint8_t*>(inv_tables) + off, kPiece, &tab_bar);
  }
  mbar_wait_parity(&tab_bar, 0);
  CP_MARK(0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* xs = xs_all + warp * 128;
  uint32_t* cs = cs_all + warp * 128;
  uint32_t* hs = hs_all + warp * kHashSlots;
  const int PB = 2 + 2 * K;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  // first round static, then chunks claimed from the counter (reset by inv_table_kernel)
  // (next == nullptr: the grid covers the batch, one chunk per warp, no counter)
  for (int64_t j = (int64_t)blockIdx.x * WARPS + warp; j < n_chunks;) {
    const unsigned long long claim = next && lane == 0 ? atomicAdd(next, 1ull) : (unsigned long long)n_chunks;
    uint32_t raw[4], yb[4];
    int kk = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      int32_t iv = -1;
      uint32_t b = 0;
      if (i < K) { iv = idx[j * K + i]; b = bits[j * K + i]; }
      raw[r] = (uint32_t)iv;
      yb[r] = b;
      kk += __popc(__ballot_sync(0xFFFFFFFFu, iv >= 0));
    }
    TL_CHECK(j < n_chunks && kk <= K && K <= TL_MAX_K);
    CP_MARK(1);
#if TL_COMMIT_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0) g_cprof[7] += 1;
#endif
    // a small-batch CTA (one chunk per sub-partition) is latency-bound: unroll deeper so the
    // inverse lookups of later levels are issued ahead of the divided-difference chain
    commit_chunk<HALF ? kInvSmemHalf : kInvSmem, WARPS <= 4 ? 8 : kNddUnroll, WARPS <= 4 ? 4 : kConvUnroll>(
        raw, yb, kk, K, inv0, inv_tables, xs, cs, hs, proofs + j * PB, lane);
    j = nw + (int64_t)__shfl_sync(0xFFFFFFFFu, claim, 0);
  }
}


// P(x) mod p for one point by Paterson-Stockmeyer over the zero-padded TL_MAX_K
// coefficients (coef: 16-B aligned u16, shared memory) -- the residue of any exact
// evaluation order (verify_tail_warp's, the oracle's).  2^32 mod p = -(p floor(2^32/p)).
__device__ __forceinline__ uint32_t poly_eval_ps1(const uint16_t* coef, uint32_t x, const ModP& m) {
  const uint32_t k32 = 0u - m.p * m.mu;
  uint32_t xp[8];
  xp[0] = 1u;
  xp[1] = x;
  xp[2] = m.mul(x, x);
  xp[3] = m.mul(xp[2], x);
  xp[4] = m.mul(xp[2], xp[2]);
  xp[5] = m.mul(xp[4], x);
  xp[6] = m.mul(xp[4], xp[2]);
  xp[7] = m.mul(xp[4], xp[3]);
  const uint32_t y = m.mul(xp[4], xp[4]);
  const uint4* c8 = reinterpret_cast<const uint4*>(coef);
  uint32_t acc = 0u;
#pragma unroll 4
  for (int kb = TL_MAX_K / 8 - 1; kb >= 0; --kb) {
    const uint4 q = c8[kb];
    const uint32_t cw[4] = {q.x, q.y, q.z, q.w};
    unsigned long long s = 0ull;
#pragma unroll
    for (int e = 0; e < 8; ++e) s += (unsigned long long)((cw[e >> 1] >> (16 * (e & 1))) & 0xFFFFu) * xp[e];
    const uint32_t qk = m.red(m.red((uint32_t)s) + (uint32_t)(s >> 32) * k32);  // s < 2^35
    acc = m.red(acc * y + qk);
  }
  return acc;
}

// tl_commit for small batches: one CTA per chunk.  The one-warp kernel above is a chain
// of ~250 dependent steps (127 divided-difference levels, 127 Newton -> monomial steps),
// ~14 us for a chunk whatever the batch.  Here the same polynomial -- the unique one of
// degree < kk through the kk points, so the same coefficients -- comes from the Lagrange
// form over a subproduct tree, with 7 levels of short sums:
//   w_t  = y_t / prod_{j != t} (x_t - x_j)          (two partial products per point; the
//                                                    inverse from the prepared table, else Fermat)
//   up:    M_node = M_left M_right,                  leaves X - x_t
//          V_node = V_left M_right + V_right M_left, leaves w_t  (root: sum_t w_t M / (X - x_t))
// Both trees advance together, one barrier per level.  A level's 128 output coefficients
// of each take kCoopCommitSub = 2 threads (strided partial sums of <= 33 products < p^2 in
// 64 bits, reduced, then summed over the pair; 2 measured faster than 4 or 8: every level
// pays a barrier, and wider CTAs pay more for it).  Subproducts are stored monic with their
// leading 1 (node n of degree d at [n (d + 1), (n + 1)(d + 1))), V nodes with d
// coefficients.  The 128 - kk padding leaves are X with w = 0: the root's V carries a factor
// X^(128 - kk), divided out by an index shift (c_k = V_{k + 128 - kk}).
constexpr int kCoopCommitSub = 2;                                   // threads per coefficient
constexpr int kCoopCommitThreads = TL_MAX_K * kCoopCommitSub;       // 256
constexpr int kCoopLevels = 7;                                      // log2(TL_MAX_K)
static_assert((1 << kCoopLevels) == TL_MAX_K, "tree levels");
__device__ __forceinline__ uint32_t red64(unsigned long long s, const ModP& m, uint32_t k32) {  // s < 2^45
  return m.red(m.red((uint32_t)s) + (uint32_t)(s >> 32) * k32);
}
__global__ void __launch_bounds__(kCoopCommitThreads)
commit_coop_kernel(const int32_t* __restrict__ idx, const uint16_t* __restrict__ bits, int64_t n_chunks, int K,
                   uint8_t* __restrict__ proofs) {
  __shared__ uint32_t tm[2][2 * TL_MAX_K];  // M levels (monic, leading 1 stored), ping-pong
  __shared__ uint32_t tv[2][TL_MAX_K];      // V levels, ping-pong
  __shared__ __align__(16) uint32_t xs[TL_MAX_K];
  __shared__ uint32_t hs[kHashSlots];
  __shared__ uint32_t wmax[kCoopCommitThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int q = t / kCoopCommitSub, sub = t & (kCoopCommitSub - 1);  // coefficient / point q, part sub
  const bool owner = sub == 0;                             // the point's own thread
  const int64_t j = blockIdx.x;
  if (j >= n_chunks) return;
#if TL_COMMIT_PROF
  long long cc_last_ = clock64(), cc_acc_[6] = {};
  if (blockIdx.x == 0 && threadIdx.x == 0) g_cprof[7] += 1;
#endif
  const bool tables = *reinterpret_cast<volatile unsigned*>(&g_inv_ready) == kInvReady;  // in flight early
  const int PB = 2 + 2 * K;
  uint8_t* pr = proofs + j * PB;
  const int32_t iv = owner && q < K ? idx[j * K + q] : -1;
  const uint32_t yb = owner && q < K ? (uint32_t)bits[j * K + q] : 0u;
  const uint32_t raw = (uint32_t)iv;
  const unsigned mx = __reduce_max_sync(0xFFFFFFFFu, iv >= 0 ? raw : 0u);
  if (lane == 0) wmax[warp] = mx;
  const int kk = __syncthreads_count(iv >= 0);
  TL_CHECK(kk >= 1 && kk <= K && K <= TL_MAX_K);
  uint32_t maxidx = 0u;
#pragma unroll
  for (int w = 0; w < kCoopCommitThreads / 32; ++w) maxidx = max(maxidx, wmax[w]);
  CC_MARK(0);

  // ---- modulus: the largest prime with injective residues (as commit_chunk)
  uint32_t p = kPMax;
  int pi = 0;
  if (maxidx >= kPMax) {
    for (; pi < TL_N_PRIMES; ++pi) {
      p = kPrimesDesc[pi];
      const ModP mp(p);
      if (t < kHashSlots) hs[t] = 0xFFFFFFFFu;
      __syncthreads();
      bool dup = false;
      if (iv >= 0) {
        const uint32_t v = mp.red(raw);
        uint32_t h = (v * 0x9E3779B1u) >> (32 - kHashBits);
        for (;;) {
          const uint32_t old = atomicCAS(&hs[h], 0xFFFFFFFFu, v);
          if (old == 0xFFFFFFFFu) break;
          if (old == v) { dup = true; break; }
          h = (h + 1) & (kHashSlots - 1);
        }
      }
      if (!__syncthreads_or(dup)) break;
    }
    if (pi == TL_N_PRIMES) p = 0;
  }
  if (p == 0) {  // unprovable chunk: p = 0, zero coefficients
    for (int b = t; b < PB; b += kCoopCommitThreads) pr[b] = 0;
    return;
  }
  CC_MARK(1);
  const ModP m(p);
  const uint32_t k32 = 0u - m.p * m.mu;  // 2^32 mod p
  const bool live = q < kk;
  const uint32_t x = live ? m.red(raw) : 0u;  // the point of thread q's quad (owner's registers)
  if (owner) {
    xs[q] = x;
    tm[0][2 * q] = x ? p - x : 0u;  // leaf q: X - x_q (X for the padding points)
    tm[0][2 * q + 1] = 1u;
  }
  __syncthreads();
  CC_MARK(2);

  // ---- w_q = y_q / prod_{j < kk, j != q} (x_q - x_j): q's threads take j = sub mod kCoopCommitSub
  {
    const uint32_t xq = xs[q];
    uint32_t p0 = 1u, p1 = 1u;
#pragma unroll 4
    for (int i = 0; i < TL_MAX_K / (2 * kCoopCommitSub); ++i) {
      const int j0 = 2 * kCoopCommitSub * i + sub, j1 = j0 + kCoopCommitSub;
      const uint32_t d0 = (j0 == q || j0 >= kk) ? 1u : m.sub(xq, xs[j0]);
      const uint32_t d1 = (j1 == q || j1 >= kk) ? 1u : m.sub(xq, xs[j1]);
      p0 = m.mul(p0, d0);
      p1 = m.mul(p1, d1);
    }
    uint32_t den = m.mul(p0, p1);
#pragma unroll
    for (int o = 1; o < kCoopCommitSub; o <<= 1) den = m.mul(den, __shfl_xor_sync(0xFFFFFFFFu, den, o));
    // distinct x: den is nonzero
    if (owner) {
      uint32_t w = 0u;
      if (live) {
        const uint32_t inv = tables && pi < kInvTables ? (uint32_t)__ldg(g_inv_tables + (size_t)pi * 65536u + den)
                                                      : m.pow(den, p - 2u);
        w = m.mul(m.red(yb), inv);
      }
      tv[0][q] = w;
    }
  }
  __syncthreads();
  CC_MARK(3);

  // ---- up the trees.  Output coefficient k < 2d of parent node n (M: also its leading 1)
  int cur = 0;
#pragma unroll 1
  for (int L = 0; L < kCoopLevels; ++L) {
    const int d = 1 << L, n = q >> (L + 1), k = q & (2 * d - 1);
    const uint32_t* MA = tm[cur] + 2 * n * (d + 1);  // children 2n, 2n + 1; M_A[d] = M_B[d] = 1
    const uint32_t* MB = MA + d + 1;
    const uint32_t* VA = tv[cur] + 2 * n * d;
    const uint32_t* VB = VA + d;
    // M: sum_i A_i B_{k-i}, i in [max(0, k-d), min(k, d)];  V: sum_i VA_i MB_{k-i} + VB_i MA_{k-i},
    // i in [max(0, k-d), min(k, d-1)]
    const int lo = k > d ? k - d : 0, hm = k < d ? k : d, hv = k < d - 1 ? k : d - 1;
    unsigned long long sm = 0ull, sv0 = 0ull, sv1 = 0ull;
#pragma unroll 2
    for (int i = lo + sub; i <= hm; i += kCoopCommitSub) {
      const uint32_t mb = MB[k - i], ma = MA[k - i];
      sm += (unsigned long long)MA[i] * mb;
      if (i <= hv) {
        sv0 += (unsigned long long)VA[i] * mb;
        sv1 += (unsigned long long)VB[i] * ma;
      }
    }
    uint32_t vm = red64(sm, m, k32), vv = red64(sv0 + sv1, m, k32);
#pragma unroll
    for (int o = 1; o < kCoopCommitSub; o <<= 1) {  // sums of kCoopCommitSub values < p
      vm += __shfl_xor_sync(0xFFFFFFFFu, vm, o);
      vv += __shfl_xor_sync(0xFFFFFFFFu, vv, o);
    }
    vm = m.red(vm);
    vv = m.red(vv);
    if (owner) {
      uint32_t* P = tm[cur ^ 1] + n * (2 * d + 1);
      P[k] = vm;
      if (k == 0) P[2 * d] = 1u;
      tv[cur ^ 1][q] = vv;
    }
    cur ^= 1;
    __syncthreads();
  }
  CC_MARK(4);

  // ---- serialise p, c_0..c_{K-1} big-endian; c_k = V_{k + pad}
  const int pad = TL_MAX_K - kk;
  uint16_t* pw = reinterpret_cast<uint16_t*>(pr);
  if (t < K) {
    const uint32_t c = t < kk ? tv[cur][t + pad] : 0u;
    pw[1 + t] = (uint16_t)(((c & 0xFFu) << 8) | (c >> 8));
  }
  if (t == 0) pw[0] = (uint16_t)(((p & 0xFFu) << 8) | (p >> 8));
  CC_MARK(5);
}

// One warp verifies one chunk from its ranked top-kk keys (top, shared memory): decode
// the claimed coefficients (pword: this lane's big-endian u16 proof words t = lane + 32 q),
// evaluate the polynomial at the kk indices (Horner, four points per lane), compare
// exponent and mantissa bits with the observed values mod p, and write the chunk
// statistics and verdict.  coef (TL_MAX_K u16, 16-B aligned) is the warp's shared
// scratch.
constexpr int kPW = (TL_MAX_K + 1 + 31) / 32;  // proof words per lane
#if TL_RING_STATS
__device__ unsigned long long g_vt[8];  // lab: verify-tail phase cycles (decode, Horner, compare, median, write),
                                        // 5 entry -> first chunk ready, 6 entry -> first stage, 7 CTAs
#endif
// PS: evaluate by Paterson-Stockmeyer (shorter chains, ~40 registers more; the ring
// finisher) instead of the two-half Horner (the one-warp kernel, 18 CTAs per SM).
template <bool PS>
__device__ __forceinline__ void verify_tail_warp(const unsigned long long* top, int kk, int K, const uint32_t (&pword)[kPW],
                                                 uint16_t* coef, const tl_thresholds& th,
                                                 tl_chunk_stats* __restrict__ stats_out, uint8_t* __restrict__ accept_out,
                                                 int64_t j, int lane) {
  TL_CHECK(j >= 0 && kk >= 1 && kk <= K && K <= TL_MAX_K);
#if TL_RING_STATS
  long long vt_ = clock64();
#define VT_MARK(i) do { const long long t_ = clock64(); if (lane == 0) atomicAdd(&g_vt[i], (unsigned long long)(t_ - vt_)); vt_ = t_; } while (0)
#else
#define VT_MARK(i) do {} while (0)
#endif
  // claimed coefficients (big-endian u16) -> coef, zero-padded to TL_MAX_K
  unsigned p = 0;
#pragma unroll
  for (int q = 0; q < kPW; ++q) {
    const int t = lane + 32 * q;
    const unsigned v = ((pword[q] & 0xFFu) << 8) | (pword[q] >> 8);
    if (t == 0) p = v;
    else if (t <= TL_MAX_K) coef[t - 1] = (uint16_t)(t <= K ? v : 0u);
  }
  p = __shfl_sync(0xFFFFFFFFu, p, 0);
  __syncwarp();
  // a proof is only as strong as its modulus: anything but one of the prover's primes
  // (p = 2 with zero coefficients would match every exponent) is a bad proof
  const bool bad = !prover_prime(p);
  VT_MARK(0);
  unsigned mism = 0, msum = 0, nmatch = 0;
  uint32_t dv[4] = {0xFFu, 0xFFu, 0xFFu, 0xFFu};  // |mantissa diff| of each exponent-equal point, else 0xFF
  if (!bad) {
    const ModP m(p);
    uint32_t x[4], acc[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      x[r] = i < kk ? m.red(key_idx(top[i])) : 0u;
      acc[r] = 0u;
    }
    static_assert(TL_MAX_K == 128, "two 64-coefficient halves / 16 blocks of 8 coefficients");
    const uint4* c8 = reinterpret_cast<const uint4*>(coef);
    if (!PS) {
      // P(x) = L(x) + x^64 U(x): eight independent 64-step Horner chains per lane instead of
      // four 128-step ones (half the latency; the one-warp kernel's registers allow no more)
      uint32_t hi[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) hi[r] = 0u;
#pragma unroll 1
      for (int kb = 7; kb >= 0; --kb) {
        const uint4 ql = c8[kb], qh = c8[kb + 8];
        const uint32_t cl[4] = {ql.x, ql.y, ql.z, ql.w}, ch[4] = {qh.x, qh.y, qh.z, qh.w};
#pragma unroll
        for (int e = 7; e >= 0; --e) {
          const uint32_t a_ = (cl[e >> 1] >> (16 * (e & 1))) & 0xFFFFu, b_ = (ch[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            acc[r] = m.red(acc[r] * x[r] + a_);
            hi[r] = m.red(hi[r] * x[r] + b_);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        uint32_t x64 = x[r];
#pragma unroll
        for (int s = 0; s < 6; ++s) x64 = m.mul(x64, x64);
        acc[r] = m.add(acc[r], m.mul(x64, hi[r]));
      }
    } else {
      // Paterson-Stockmeyer over the zero-padded TL_MAX_K coefficients:
      //   P(x) = sum_k y^k Q_k(x),  y = x^8,  Q_k(x) = sum_{i<8} c_{8k+i} x^i.
      // Each Q_k is eight independent 32x32->64 multiply-adds of (raw u16 coefficient) x
      // (x^i mod p) -- below 2^35, reduced once -- and only the 16 steps in y form a
      // dependent chain: ~40 % fewer instructions than Horner over 128 coefficients and a
      // quarter of its chain (the same residue: any evaluation order of P mod p).
      const uint32_t k32 = (uint32_t)(0x100000000ull % m.p);  // 2^32 mod p
      uint32_t xp[4][8], y[4];
  #pragma unroll
      for (int r = 0; r < 4; ++r) {
        xp[r][0] = 1u;
        xp[r][1] = x[r];
        xp[r][2] = m.mul(x[r], x[r]);
        xp[r][3] = m.mul(xp[r][2], x[r]);
        xp[r][4] = m.mul(xp[r][2], xp[r][2]);
        xp[r][5] = m.mul(xp[r][4], x[r]);
        xp[r][6] = m.mul(xp[r][4], xp[r][2]);
        xp[r][7] = m.mul(xp[r][4], xp[r][3]);
        y[r] = m.mul(xp[r][4], xp[r][4]);
      }
  #pragma unroll 2
      for (int kb = 15; kb >= 0; --kb) {
        const uint4 q = c8[kb];
        const uint32_t cw[4] = {q.x, q.y, q.z, q.w};
        uint32_t cc[8];
  #pragma unroll
        for (int e = 0; e < 8; ++e) cc[e] = (cw[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
  #pragma unroll
        for (int r = 0; r < 4; ++r) {
          unsigned long long s = 0ull;
  #pragma unroll
          for (int e = 0; e < 8; ++e) s += (unsigned long long)cc[e] * xp[r][e];
          const uint32_t qk = m.red(m.red((uint32_t)s) + (uint32_t)(s >> 32) * k32);  // s < 2^35
          acc[r] = m.red(acc[r] * y[r] + qk);
        }
      }
    }
    VT_MARK(1);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      if (i < kk) {
        const uint32_t obs = m.red((uint32_t)(top[i] & 0xFFFFu));
        const uint32_t claimed = acc[r];
        if (((claimed >> 7) & 0xFFu) != ((obs >> 7) & 0xFFu)) {
          ++mism;
        } else {
          const unsigned d = (unsigned)abs((int)(claimed & 0x7Fu) - (int)(obs & 0x7Fu));
          dv[r] = d;
          msum += d;
          ++nmatch;
        }
      }
    }
  }
  VT_MARK(2);
  mism = __reduce_add_sync(0xFFFFFFFFu, mism);
  msum = __reduce_add_sync(0xFFFFFFFFu, msum);
  const unsigned nm = __reduce_add_sync(0xFFFFFFFFu, nmatch);
  __syncwarp();
  // median (statistics.median: the mean of the two middle values): the value of 0-based
  // rank q is the smallest t in [0, 127] with more than q diffs <= t -- a 7-step binary
  // search of warp counts per rank
  auto select_rank = [&](unsigned q) {
    unsigned lo = 0u, hi = 127u;
#pragma unroll 1
    while (lo < hi) {
      const unsigned mid = (lo + hi) >> 1;
      unsigned le = 0u;
#pragma unroll
      for (int r = 0; r < 4; ++r) le += dv[r] <= mid ? 1u : 0u;
      if (__reduce_add_sync(0xFFFFFFFFu, le) > q) hi = mid;
      else lo = mid + 1u;
    }
    return lo;
  };
  const unsigned q1 = nm ? (nm - 1) / 2 : 0, q2 = nm / 2;
  const int v1 = (int)select_rank(q1), v2 = q2 == q1 ? v1 : (int)select_rank(q2);
  VT_MARK(3);
  if (lane == 0) {
    tl_chunk_stats st;
    if (bad) {
      st.exp_mismatch = (uint32_t)kk; st.n_match = 0; st.mant_sum = 0;
      st.mant_mean = __longlong_as_double(0x7FF0000000000000ll);
      st.mant_median = st.mant_mean;
      st.flags = TL_STAT_BADPROOF;
    } else {
      st.exp_mismatch = mism; st.n_match = nm; st.mant_sum = msum;
      if (nm) {
        st.mant_mean = (double)msum / (double)nm;
        st.mant_median = ((double)v1 + (double)v2) * 0.5;
      } else {
        st.mant_mean = __longlong_as_double(0x7FF0000000000000ll);
        st.mant_median = st.mant_mean;
      }
      const bool ok = (int)st.exp_mismatch <= th.max_exp_mismatch && st.mant_mean <= th.max_mant_mean &&
                      st.mant_median <= th.max_mant_median;
      st.flags = ok ? TL_STAT_ACCEPT : 0u;
    }
    if (stats_out) stats_out[j] = st;
    accept_out[j] = (uint8_t)(st.flags & TL_STAT_ACCEPT);
  }
  __syncwarp();
  VT_MARK(4);
#undef VT_MARK
}

// Verify: the warp selects its chunk's top-kk on the validator tensor, evaluates
// the claimed polynomial at the kk indices (Horner, four points per lane),
// compares exponent and mantissa bits with the observed values mod p, and writes
// the chunk statistics and verdict.
template <bool SPLIT>
__global__ void __launch_bounds__(kSelBlockThreads, kSelMinBlocks)
verify_kernel(SelArgs a, const uint8_t* __restrict__ proofs, tl_thresholds th,
              tl_chunk_stats* __restrict__ stats_out, uint8_t* __restrict__ accept_out) {
  extern __shared__ __align__(128) uint8_t sel_smem[];
  WarpSlot& slot = reinterpret_cast<SelState*>(sel_smem)->w[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  if (lane == 0) slot.lst_n = 0;
  __syncwarp();
  const int64_t n_chunks = min(a.n_chunks, a.prefix[a.n_roll]);
  const int64_t nw = (int64_t)gridDim.x * kSelWarps;
  const int K = a.K;
  const int PB = 2 + 2 * K;
  const int64_t gw = (int64_t)blockIdx.x * kSelWarps + (threadIdx.x >> 5);
  Spec sp = spec_load(a.spec, gw);
  PROF_DECL;
  const int S = SPLIT ? a.split : 1;
  for (int64_t j = SPLIT ? gw / S : gw; j < n_chunks;) {
    const unsigned long long claim = SPLIT ? 0ull : claim_chunk(a, lane);
    const ChunkGeo g = chunk_geo(a, j);
    const int kk = min(K, g.n);
    // issue this chunk's proof loads (u16 t = p or c_{t-1}) before streaming, so
    // their latency hides behind the chunk
    const uint16_t* pw = reinterpret_cast<const uint16_t*>(proofs + j * PB);
    uint32_t pword[kPW];
#pragma unroll
    for (int q = 0; q < kPW; ++q) {
      const int t = lane + 32 * q;
      pword[q] = t <= K ? (uint32_t)__ldg(pw + t) : 0u;
    }
    PROF_MARK(0);
    if (SPLIT) {
      if (!select_split(a, g, kk, j, (int)(gw % S), slot, sp, lane PROF_PASS)) break;  // another part merges
    } else {
      select_chunk(g, kk, slot, sp, lane PROF_PASS);
    }

    verify_tail_warp<false>(slot.wbuf, kk, K, pword, slot.coef, th, stats_out, accept_out, j, lane);
    __syncwarp();
    PROF_MARK(4);
    if (SPLIT) break;  // one part per warp
    j = nw + (int64_t)__shfl_sync(0xFFFFFFFFu, claim, 0);
  }
  spec_store(a.spec, gw, sp, lane);
  PROF_FLUSH();
}

// A rollout is accepted iff all its chunks are.  Chunks at or past the caller's
// n_chunks were never verified (a miscounted call): they reject, so a miscount fails
// closed instead of reading stale accept bytes.
__global__ void rollout_verdict_kernel(const uint8_t* __restrict__ chunk_accept,
                                       const int64_t* __restrict__ prefix, int n_roll, int64_t n_chunks,
                                       uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n_roll) return;
  TL_CHECK(prefix[r] >= 0 && prefix[r] <= prefix[r + 1]);
  int ok = 1;
  for (int64_t q = prefix[r] + lane; q < prefix[r + 1]; q += 32) ok &= (q < n_chunks && chunk_accept[q]) ? 1 : 0;
  ok = __all_sync(0xFFFFFFFFu, ok);
  if (lane == 0) out[r] = (uint8_t)ok;
}

// ----------------------------------------------------------------------------- TMA-ring streaming (large batches)
//
// The large-batch select / verify path, one persistent CTA per SM with three warp roles:
//   * a producer warp moves one chunk at a time through a ring of kRingStages x 32 KiB
//     shared-memory stages with TMA bulk copies (cp.async.bulk + mbarrier transaction
//     counts), claiming chunks like the per-warp kernels (first round static, then the
//     workspace counter);
//   * kRingConsumers consumer warps each scan an interleaved share of every stage with the
//     same 16x2-SIMD magnitude test as the per-warp kernels, buffer their candidates and,
//     at the chunk end, rank their buffer and hand it to a finisher -- and go straight on
//     to the next chunk (their candidate buffers are double-buffered by chunk parity);
//   * kRingFinishers finisher warps (one per buffer parity) merge the consumers' ranked
//     lists into the chunk's top-kk and write the indices and values (prove) or evaluate
//     the proof and write statistics and verdicts (verify).
// So nothing on the streaming side ever waits for a chunk tail.
//
// Why: a bare-read probe on configuration 2's 21.5 GB (tools/lab/ctaprobe.cu,
// profiles/r02_ctaprobe.txt) streams 7.53 TB/s through a 5 x 32 KiB ring with 16 consumer
// warps per SM against 7.19 TB/s for the per-warp register double buffer of the
// one-warp-per-chunk kernels.  A first ring kernel whose consumers ran the chunk tail
// themselves (CTA barriers, two CTAs per SM) measured 7.8 us of tail per chunk and 5.4 TB/s.
//
// A lane whose elements pass the coarse test appends the passing elements itself (one
// per lane per round, re-read from the stage in shared memory), with no queue.
//
// Correctness: every consumer warp starts a chunk from the same threshold theta0 (the
// producer stamps it on the chunk's first stage), and each warp keeps the per-warp
// invariant of select_chunk on its share (every element of the share with key >= the
// warp's theta is buffered; a warp whose theta was raised by a compaction holds >= kk
// keys >= it).  Then an element no warp buffered has >= kk buffered keys above it as soon
// as the warps hold >= kk keys in total, so the merged top-kk of the ranked lists is the
// chunk's top-kk; otherwise the finisher re-scans the chunk from global memory with a
// lower threshold.
#ifndef TL_RING_CONSUMERS
#define TL_RING_CONSUMERS 8
#endif
#ifndef TL_RING_STAGES
#define TL_RING_STAGES 3
#endif
#ifndef TL_RING_STAGE_KB
#define TL_RING_STAGE_KB 28
#endif
#ifndef TL_RING_FINISHERS
#define TL_RING_FINISHERS 1
#endif
#ifndef TL_RING_CTAS
#define TL_RING_CTAS 2
#endif
#ifndef TL_RING_STATS
#define TL_RING_STATS 0
#endif
#ifndef TL_RING_LAB
#define TL_RING_LAB 0
#endif
#if TL_RING_STATS  // lab instrumentation: chunks, candidates, re-scans, compactions, finisher cycles
__device__ unsigned long long g_ring_stats[8];
__device__ unsigned g_ring_trace[1024][4];  // CTA 0: per chunk theta magnitude, total, delta, kth magnitude
__device__ unsigned g_ring_trace_n;
// CTA 0's timeline of up to 64 launches (globaltimer ns): 0 entry, 1 roles start, 2 first
// stages issued, 3 first stage landed, 4 chunk end (consumer 0), 5/6 cooperative finish
// after its first / second barrier, 7 done
__device__ unsigned long long g_ring_tl[64][32];  // 8 + 2t / 9 + 2t: consumer 0's stage t landed / scanned
__device__ unsigned g_ring_tl_n;
__device__ __forceinline__ unsigned long long ring_gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__shared__ unsigned g_ring_tl_launch;  // this launch's timeline row (CTA 0)
#define RING_TL(slot)                                                                        \
  do {                                                                                       \
    if (blockIdx.x == 0) g_ring_tl[g_ring_tl_launch & 63u][(slot) & 31] = ring_gt();          \
  } while (0)
#else
#define RING_TL(slot) do {} while (0)
#endif
constexpr int kRingConsumers = TL_RING_CONSUMERS;
constexpr int kRingFinishers = TL_RING_FINISHERS;  // chunk c -> finisher c % kRingFinishers, buffer c & 1
constexpr int kRingProducer = kRingConsumers + kRingFinishers;  // warp index
constexpr int kRingThreads = 32 * (kRingProducer + 1);
constexpr int kRingStages = TL_RING_STAGES;
constexpr int kRingStageBytes = TL_RING_STAGE_KB * 1024;
constexpr int kRingStageVec = kRingStageBytes / 16;
constexpr int kRingStride = kRingConsumers * 32;                         // vectors between a lane's vectors
constexpr int kRingTileU = kRingStageVec / kRingStride < kSelU ? kRingStageVec / kRingStride : kSelU;
constexpr int kRingSub = kRingStageVec / (kRingStride * kRingTileU);     // tiles per lane and stage
static_assert(kRingSub * kRingStride * kRingTileU == kRingStageVec && kRingTileU <= 8, "stage split");
constexpr int kRingCap = TL_MAX_K + 32;  // per-warp candidate keys: a compaction keeps kk, one round adds <= 32
constexpr int kRingCtasPerSm = TL_RING_CTAS;

constexpr int kRingOwnPrefixMax = 256;  // rollouts whose chunk prefix a small-batch ring CTA builds itself
struct RingMeta {
  long long j;               // chunk (-1: no more work)
  unsigned long long theta;  // the chunk's starting threshold (stamped on every stage)
  int q, nst;                // stage q of nst
  int len;                   // bytes in this stage
  int n;                     // elements in the chunk
};
struct RingJob {
  long long j;  // chunk (-1: the finisher exits)
  unsigned long long theta;
  int kk, nst;
};
struct RingSmem {
  uint4 ring[kRingStages][kRingStageVec];
  unsigned long long wbuf[2][kRingConsumers][kRingCap];  // by chunk parity: candidates, then ranked lists
  unsigned long long uni[kRingFinishers][kWarpCap];      // the union of a chunk's candidate buffers, ranked
  uint16_t coef[kRingFinishers][TL_MAX_K];               // verify: claimed coefficients
  RingMeta meta[kRingStages];
  uint64_t full[kRingStages], empty[kRingStages];        // ring stage filled / released
  uint64_t ready[2], freed[2];                           // ranked lists handed over / merged
  RingJob job[2];
  int cnt[2][kRingConsumers];  // candidates per consumer warp at the chunk end
  int cmp[2][kRingConsumers];  // ... and whether its threshold was raised by a compaction
  int64_t pfx[kRingOwnPrefixMax + 1];  // small batches: the chunk prefix, built by the CTA itself
  unsigned long long theta_next;  // speculation for the next chunk (finishers -> producer)
  unsigned long long theta_pub[2];  // by chunk parity: the largest threshold a consumer's compaction proved
  Spec spec;                      // the CTA's speculation state, updated in chunk order ...
  long long spec_seq;             // ... by the finisher of chunk spec_seq
  alignas(16) unsigned coop_hist[128];  // cooperative finish (verify): |mantissa diff| histogram
  unsigned coop_red[4];           // ... exponent mismatches, mantissa sum, matches
  unsigned coop_p, coop_bad;      // ... the proof's modulus, not a prover prime
};
constexpr size_t kRingSmem = (sizeof(RingSmem) + 127) & ~(size_t)127;
static_assert(kRingCtasPerSm * (kRingSmem + 1024) <= 228 * 1024, "ring CTAs per SM");

struct RingScan {
  unsigned long long theta;
  int cnt;
  unsigned long long* wb;
  unsigned long long* pub = nullptr;  // the chunk's shared threshold (consumers; nullptr on a re-scan)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init_count(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

// Warp-uniform append of at most one key per lane into the warp's kRingCap buffer; a full
// buffer keeps its kk largest keys and raises theta to the kk-th (rare path).
__device__ __noinline__ unsigned long long ring_compact(unsigned long long* wb, int cnt, int kk, int lane) {
  final_sort<kWarpCap / 32, TL_MAX_K>(wb, cnt, lane);
  return wb[kk - 1];
}
__device__ __forceinline__ void ring_append(bool p, unsigned long long key, RingScan& w, int kk, int lane) {
  unsigned bal = __ballot_sync(0xFFFFFFFFu, p);
  if (!bal) return;
  if (w.cnt + __popc(bal) > kRingCap) {
    w.theta = ring_compact(w.wb, w.cnt, kk, lane);
    w.cnt = kk;
    // this warp now holds kk keys >= theta, so no element below it is in the chunk's top-kk:
    // the other consumer warps adopt it (ties in a heavy-tie chunk stop queueing everywhere)
    if (w.pub && lane == 0) atomicMax(w.pub, w.theta);
    p = p && key >= w.theta;
    bal = __ballot_sync(0xFFFFFFFFu, p);
  }
  TL_CHECK(w.cnt + __popc(bal) <= kRingCap);
  if (p) w.wb[w.cnt + __popc(bal & lanemask_lt())] = key;
  w.cnt += __popc(bal);
  __syncwarp();
}


// Share `wid` of one stage-sized piece of the chunk (nvec 16-B vectors at src, in shared
// memory for the ring or in global memory for a re-scan): vectors
// g = (u * kRingConsumers + wid) * 32 + lane, kRingTileU per lane per tile; elem0 is the
// flat index of the piece's first element.
template <bool SMEM>
__device__ __forceinline__ void ring_scan(const uint4* __restrict__ src, int nvec, unsigned elem0, RingScan& w,
                                          int kk, int lane, int wid) {
  const uint16_t* s16 = reinterpret_cast<const uint16_t*>(src);
#pragma unroll 1
  for (int h = 0; h < kRingSub; ++h) {
    const int g0 = (h * kRingTileU * kRingConsumers + wid) * 32 + lane;
    uint4 v[kRingTileU];
#pragma unroll
    for (int u = 0; u < kRingTileU; ++u) {
      const int g = g0 + u * kRingStride;
      v[u] = g < nvec ? (SMEM ? src[g] : ld_stream(src + g)) : make_uint4(0u, 0u, 0u, 0u);
    }
    if (SMEM && w.pub) {  // adopt a threshold another warp's compaction published
      unsigned long long tp = lane == 0 ? *reinterpret_cast<volatile unsigned long long*>(w.pub) : 0ull;
      tp = __shfl_sync(0xFFFFFFFFu, tp, 0);
      if (tp > w.theta) w.theta = tp;
    }
    const unsigned c2 = coarse_c2(w.theta, elem0 + 8u * (unsigned)(g0 - lane));
    unsigned mu[kRingTileU];
#pragma unroll
    for (int u = 0; u < kRingTileU; ++u) mu[u] = hmaxabs2(hmaxabs2(v[u].x, v[u].y), hmaxabs2(v[u].z, v[u].w));
    unsigned m = mu[0];
#pragma unroll
    for (int u = 1; u < kRingTileU; ++u) m = hmaxabs2(m, mu[u]);
    const bool hit = coarse_hit(m, c2);
    if (!__any_sync(0xFFFFFFFFu, hit)) continue;
    uint32_t em_lo = 0u, em_hi = 0u;  // element e of vector u: bit 8u + e (zero vectors past the end never hit)
    if (hit) {
#pragma unroll
      for (int u = 0; u < kRingTileU; ++u) {
        if (g0 + u * kRingStride < nvec && coarse_hit(mu[u], c2)) {
          const uint32_t m8 = elem_mask8(v[u], c2);
          if (u < 4) em_lo |= m8 << (8 * u);
          else em_hi |= m8 << (8 * (u - 4));
        }
      }
    }
    // one candidate element per lane per round, tested exactly against the composite key
    for (;;) {
      const bool has = (em_lo | em_hi) != 0u;
      if (!__any_sync(0xFFFFFFFFu, has)) break;
      bool p = false;
      unsigned long long key = 0ull;
      if (has) {
        int bit;
        if (em_lo) { bit = __ffs(em_lo) - 1; em_lo &= em_lo - 1u; }
        else { bit = 31 + __ffs(em_hi); em_hi &= em_hi - 1u; }
        const int off = 8 * (g0 + (bit >> 3) * kRingStride) + (bit & 7);  // element offset within src
        const unsigned b = SMEM ? (unsigned)s16[off] : (unsigned)__ldg(s16 + off);
        key = make_key(b, elem0 + (unsigned)off);
        p = key >= w.theta;
      }
      ring_append(p, key, w, kk, lane);
    }
  }
}

// Rank a buffer and leave its top-min(128, cnt) in wb[0..128), zero-padded.
__device__ __forceinline__ void ring_rank(unsigned long long* wb, int cnt, int lane) {
  if (cnt <= 32) final_sort<1>(wb, cnt, lane);
  else if (cnt <= 64) final_sort<2>(wb, cnt, lane);
  else if (cnt <= 128) final_sort<4>(wb, cnt, lane);
  else final_sort<8, TL_MAX_K>(wb, cnt, lane);
  for (int i = (cnt <= 32 ? 32 : cnt <= 64 ? 64 : 128) + lane; i < TL_MAX_K; i += 32) wb[i] = 0ull;
  __syncwarp();
}

// Chunk j's geometry found by the whole (producer) warp: a 32-ary search over the chunk
// prefix (two dependent loads for up to 1024 rollouts instead of ~10 for a binary search
// by one thread), then the rollout's row range.
__device__ __forceinline__ ChunkGeo warp_chunk_geo(const SelArgs& a, int64_t j, int lane) {
  int lo = 0, hi = a.n_roll;  // prefix[lo] <= j < prefix[hi]
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const bool le = idx < hi && a.prefix[idx] <= j;
    const int last = 31 - __clz(__ballot_sync(0xFFFFFFFFu, le));  // lane 0 (idx = lo) always holds
    lo += last * step;
    hi = min(hi, lo + step);
  }
  const int64_t r0 = a.row_off[lo], T = a.row_off[lo + 1] - r0;
  const int64_t local = j - a.prefix[lo];
  TL_CHECK(lo < a.n_roll && local >= 0 && local * a.C < T && r0 + local * a.C + min((int64_t)a.C, T - local * a.C) <= a.n_rows);
  ChunkGeo g;
  g.base = a.hidden + (r0 + local * a.C) * (int64_t)a.H;
  g.n = (int)min((int64_t)a.C, T - local * a.C) * a.H;
  g.a0 = 0;  // ring chunks are 16-B aligned (ring_grid)
  g.nvec = g.n >> 3;
  g.nst = 0;
  return g;
}

// Producer warp: lane 0 issues the stages; the whole warp locates the next chunk while the
// current one streams (the ring is full then, so the producer would only be waiting).
__device__ __forceinline__ void ring_produce(const SelArgs& a, RingSmem& S, int64_t n_chunks, int lane,
                                             const uint8_t* __restrict__ proofs = nullptr) {
  int64_t j = blockIdx.x;
  ChunkGeo g = warp_chunk_geo(a, j < n_chunks ? j : 0, lane);
  long long t = 0;
  unsigned long long theta = 0ull;
  auto issue = [&](int q, int nst, int bytes) {  // lane 0
    const int s = (int)(t % kRingStages);
    if (t >= kRingStages) mbar_wait_parity(&S.empty[s], (unsigned)(((t / kRingStages) - 1) & 1));
    const int len = min(kRingStageBytes, bytes - q * kRingStageBytes);
    TL_CHECK(j >= 0 && j < n_chunks && len > 0 && (len & 15) == 0 && q < nst && g.n <= a.C * a.H);
    TL_CHECK((reinterpret_cast<uintptr_t>(g.base) & 15u) == 0);
    S.meta[s] = RingMeta{(long long)j, theta, q, nst, len, g.n};
    mbar_expect_tx(&S.full[s], (uint32_t)len);
    bulk_copy_g2s(S.ring[s], reinterpret_cast<const uint8_t*>(g.base) + (size_t)q * kRingStageBytes, (uint32_t)len,
                  &S.full[s]);
    ++t;
  };
  for (;;) {
    if (j >= n_chunks) {
      if (lane == 0) {
        const int s = (int)(t % kRingStages);
        if (t >= kRingStages) mbar_wait_parity(&S.empty[s], (unsigned)(((t / kRingStages) - 1) & 1));
        S.meta[s].j = -1;
        mbar_arrive(&S.full[s]);
      }
      return;
    }
    // the next chunk (none to claim when the grid covers the batch: small batches run without
    // the counter reset of chunk_prefix_kernel)
    const unsigned long long claim = lane == 0 && (int64_t)gridDim.x < n_chunks ? atomicAdd(a.next, 1ull)
                                                                                 : (unsigned long long)n_chunks;
    const int bytes = 2 * g.n;
    const int nst = (bytes + kRingStageBytes - 1) / kRingStageBytes;
    // the CTA's first chunk fills every free slot before the next chunk's lookup (a small
    // batch has no next chunk, and its stages would otherwise wait for that lookup); later
    // chunks issue one stage first, since the ring is full then
    const int pre = t == 0 ? min(nst, kRingStages) : 1;  // lane 0's t
    if (lane == 0) {
      theta = *reinterpret_cast<volatile unsigned long long*>(&S.theta_next);  // the finishers' latest hint
      for (int q = 0; q < pre; ++q) issue(q, nst, bytes);
      if (t == pre) RING_TL(2);
    }
    if (proofs && lane < 3)  // verify: the chunk's 258-byte proof into L2 for its finisher
      asm volatile("prefetch.global.L2 [%0];" ::"l"(proofs + j * (2 + 2 * a.K) + 128 * lane));
    __syncwarp();
    const int64_t jn = (int64_t)gridDim.x + (int64_t)__shfl_sync(0xFFFFFFFFu, claim, 0);
    const ChunkGeo gn = warp_chunk_geo(a, jn < n_chunks ? jn : 0, lane);
    if (lane == 0)
      for (int q = pre; q < nst; ++q) issue(q, nst, bytes);
    __syncwarp();
    j = jn;
    g = gn;
  }
}

// The ring kernel's outputs: select (idx, bits) or verify (proofs in; stats, verdicts out).
struct RingOut {
  int32_t* idx;
  uint16_t* bits;
  const uint8_t* proofs;
  tl_thresholds th;
  tl_chunk_stats* stats;
  uint8_t* accept;
};

// Small batches: a CTA whose only chunk this is finishes it with its consumer warps and
// its finisher together (kRingCoopThreads threads) instead of handing it to the one
// finisher warp, whose single-warp tail (one bitonic sort of the union, four points per
// lane for verify) is the latency of a batch of one chunk per CTA.
//   - rank: each consumer has ranked its own buffer (ring_rank) before the barrier;
//     candidate t (one per thread, the buffers' first kk keys concatenated) counts the keys
//     above it in every buffer by binary search -- keys are distinct (the index is part of
//     the key), so the count is its rank and sorted[rank] = key for rank < kk is the
//     ranked top-kk;
//   - select: the top-kk written by 128 threads;
//   - verify: the finisher decodes the proof while the consumers scan; point i by thread i
//     (poly_eval_ps1), counts by warp reductions, the mantissa median from a 128-bin
//     histogram's prefix (the smallest t with more than q differences <= t, as
//     select_rank in verify_tail_warp).
// Returns false, having changed nothing the general path reads, when the chunk needs the
// finisher's general path (fewer than kk candidates: a re-scan; a buffer over
// kRingCoopRankMax keys, left unranked; more candidates than threads); the caller then
// continues its normal loop.
constexpr int kRingCoopThreads = 32 * (kRingConsumers + 1);  // consumer warps + the finisher (warp kRingConsumers)
constexpr int kRingCoopRankMax = 64;  // candidates per consumer buffer the cooperative finish ranks (typical: ~25)
__device__ __forceinline__ void ring_coop_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kRingCoopThreads) : "memory");
}
template <bool VERIFY>
__device__ bool ring_coop_finish(const SelArgs& a, RingSmem& S, const RingOut& o, int tid) {
  static_assert(kRingFinishers == 1 && kRingConsumers * 32 + 32 == kRingCoopThreads, "coop layout");
  if (VERIFY && tid >= 32 * kRingConsumers) {
    // the finisher warp, idle while the consumers scan, decodes the proof of the CTA's only
    // chunk (blockIdx.x): coefficients zero-padded to TL_MAX_K, modulus, prover-prime test
    const int lane = tid & 31, K = a.K;
    const uint16_t* pw = reinterpret_cast<const uint16_t*>(o.proofs + (int64_t)blockIdx.x * (2 + 2 * K));
    unsigned p = 0u;
#pragma unroll
    for (int q = 0; q < kPW; ++q) {
      const int t = lane + 32 * q;
      if (t <= TL_MAX_K) {
        const unsigned w = t <= K ? (unsigned)__ldg(pw + t) : 0u;
        const unsigned v = ((w & 0xFFu) << 8) | (w >> 8);
        if (t == 0) p = v;
        else S.coef[0][t - 1] = (uint16_t)v;
      }
    }
    if (lane == 0) {
      S.coop_p = p;
      S.coop_bad = prover_prime(p) ? 0u : 1u;
    }
#pragma unroll
    for (int i = lane; i < 128; i += 32) S.coop_hist[i] = 0u;
    if (lane < 4) S.coop_red[lane] = 0u;
  }
  ring_coop_bar();  // every consumer's count, flag, buffer and the job are visible
#if TL_RING_STATS
  const long long t0 = clock64();
#endif
  const RingJob job = S.job[0];
  const int kk = job.kk, K = a.K, lane = tid & 31;
  int total = 0, cmax = 0, ranked = 0, mq = -1, mi = 0;
  int cq[kRingConsumers];
  bool compacted = false;
#pragma unroll
  for (int q = 0; q < kRingConsumers; ++q) {
    const int c = S.cnt[0][q];
    cq[q] = c;
    const int r = min(c, kk);  // a buffer's keys past its kk-th are not in the top-kk
    if (tid >= ranked && tid < ranked + r) {
      mq = q;
      mi = tid - ranked;
    }
    ranked += r;
    total += c;
    cmax = max(cmax, c);
    compacted = compacted || S.cmp[0][q];
  }
  if (tid == 0) RING_TL(5);
  // uniform: the general path (fewer than kk candidates, an unranked buffer, too many to rank)
  if (total < kk || cmax > kRingCoopRankMax || ranked > kRingCoopThreads) return false;
  TL_CHECK(job.j >= 0 && kk >= 1 && kk <= K && K <= TL_MAX_K);
  unsigned long long* sorted = S.uni[0];
  if (mq >= 0) {
    // rank = the keys above this one in every ranked buffer (its own included: keys are
    // distinct, so its own buffer contributes its position), by branch-free binary searches
    const unsigned long long key = S.wbuf[0][mq][mi];
    int rank = 0;
#pragma unroll
    for (int q = 0; q < kRingConsumers; ++q) {
      const unsigned long long* wb = S.wbuf[0][q];
      int pos = 0;  // keys of buffer q above key: wb[0, pos) > key >= wb[pos]
#pragma unroll
      for (int step = kRingCoopRankMax / 2; step >= 1; step >>= 1)
        if (pos + step <= cq[q] && wb[pos + step - 1] > key) pos += step;
      if (pos + 1 <= cq[q] && wb[pos] > key) ++pos;  // cq = kRingCoopRankMax: the last step of a full search
      rank += pos;
    }
    TL_CHECK(rank >= mi);
    if (rank < kk) sorted[rank] = key;
  }
  const int64_t j = job.j;
  TL_CHECK(j == (int64_t)blockIdx.x);
  ring_coop_bar();  // sorted[0, kk) complete
  if (tid == 0) RING_TL(6);
  if (tid >= 32 * kRingConsumers) {  // the finisher warp: speculation, as ring_finish (no re-scan here)
    Spec sp = S.spec;
    int d = sp.delta;
    if ((total > kk + TL_SPEC_HI || compacted) && d > 1) --d;
    else if (total < kk + TL_SPEC_LO) ++d;
    sp.delta = d;
    sp.k0 = sp.k1;
    sp.k1 = (unsigned)(sorted[kk - 1] >> 40);
    spec_arm(sp);
    spec_store(a.spec, blockIdx.x, sp, lane);
  }
  if (!VERIFY) {
    if (tid < K) {
      const unsigned long long key = sorted[tid < kk ? tid : 0];
      o.idx[j * K + tid] = tid < kk ? (int32_t)key_idx(key) : -1;
      o.bits[j * K + tid] = tid < kk ? (uint16_t)(key & 0xFFFFu) : (uint16_t)0;
    }
  } else {
    const uint32_t p = S.coop_p;
    const bool bad = S.coop_bad != 0u;
    unsigned mism = 0u, msum = 0u, match = 0u;
    if (!bad && tid < kk) {
      const ModP m(p);
      const unsigned long long key = sorted[tid];
      const uint32_t claimed = poly_eval_ps1(S.coef[0], m.red(key_idx(key)), m);
      const uint32_t obs = m.red((uint32_t)(key & 0xFFFFu));
      if (((claimed >> 7) & 0xFFu) != ((obs >> 7) & 0xFFu)) {
        mism = 1u;
      } else {
        const unsigned dd = (unsigned)abs((int)(claimed & 0x7Fu) - (int)(obs & 0x7Fu));
        msum = dd;
        match = 1u;
        atomicAdd(&S.coop_hist[dd], 1u);
      }
    }
    mism = __reduce_add_sync(0xFFFFFFFFu, mism);
    msum = __reduce_add_sync(0xFFFFFFFFu, msum);
    match = __reduce_add_sync(0xFFFFFFFFu, match);
    if (lane == 0 && (mism | msum | match)) {
      atomicAdd(&S.coop_red[0], mism);
      atomicAdd(&S.coop_red[1], msum);
      atomicAdd(&S.coop_red[2], match);
    }
    ring_coop_bar();  // counts and histogram complete
    if (tid < 32) {
      const unsigned nm = S.coop_red[2], ms = S.coop_red[1];
      // the value of 0-based rank q: the smallest t with more than q differences <= t
      const uint4 h = reinterpret_cast<const uint4*>(S.coop_hist)[lane];  // t = 4 lane + e
      const unsigned c0 = h.x, c1 = c0 + h.y, c2 = c1 + h.z, c3 = c2 + h.w;
      unsigned incl = c3;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += y;
      }
      const unsigned base = incl - c3;  // differences in t < 4 lane
      auto value_of_rank = [&](unsigned q) {
        const int e = base + c0 > q ? 0 : base + c1 > q ? 1 : base + c2 > q ? 2 : base + c3 > q ? 3 : 4;
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, e < 4);
        const int l = bal ? __ffs(bal) - 1 : 31;
        return 4 * l + __shfl_sync(0xFFFFFFFFu, e < 4 ? e : 3, l);
      };
      const unsigned q1 = nm ? (nm - 1) / 2 : 0, q2 = nm / 2;
      const int v1 = value_of_rank(q1), v2 = value_of_rank(q2);
      if (lane == 0) {
        tl_chunk_stats st;
        if (bad) {
          st.exp_mismatch = (uint32_t)kk; st.n_match = 0; st.mant_sum = 0;
          st.mant_mean = __longlong_as_double(0x7FF0000000000000ll);
          st.mant_median = st.mant_mean;
          st.flags = TL_STAT_BADPROOF;
        } else {
          st.exp_mismatch = S.coop_red[0]; st.n_match = nm; st.mant_sum = ms;
          if (nm) {
            st.mant_mean = (double)ms / (double)nm;
            st.mant_median = ((double)v1 + (double)v2) * 0.5;
          } else {
            st.mant_mean = __longlong_as_double(0x7FF0000000000000ll);
            st.mant_median = st.mant_mean;
          }
          const bool ok = (int)st.exp_mismatch <= o.th.max_exp_mismatch && st.mant_mean <= o.th.max_mant_mean &&
                          st.mant_median <= o.th.max_mant_median;
          st.flags = ok ? TL_STAT_ACCEPT : 0u;
        }
        if (o.stats) o.stats[j] = st;
        o.accept[j] = (uint8_t)(st.flags & TL_STAT_ACCEPT);
      }
    }
  }
#if TL_RING_STATS
  if (tid == 0) RING_TL(7);
  if (tid == 0) {
    atomicAdd(&g_ring_stats[0], 1ull);
    atomicAdd(&g_ring_stats[1], (unsigned long long)total);
    atomicAdd(&g_ring_stats[3], compacted ? 1ull : 0ull);
    atomicAdd(&g_ring_stats[4], (unsigned long long)(clock64() - t0));
  }
#endif
  return true;
}

// Consumer warp `wid`: scan its share of every stage; at each chunk end rank its buffer,
// hand it to the chunk's finisher and continue with the next chunk.  A CTA whose only
// chunk this is (coop) finishes it cooperatively when ring_coop_finish applies.
template <bool VERIFY>
__device__ __forceinline__ void ring_consume(const SelArgs& a, RingSmem& S, int K, int lane, int wid, bool coop,
                                             const RingOut& o, long long t_entry = 0) {
  RingScan w;
  w.theta = 0ull;
  w.cnt = 0;
  w.wb = S.wbuf[0][wid];
  unsigned long long theta0 = 0ull;
  long long c = -1;  // chunk sequence number of this CTA
  for (long long t = 0;; ++t) {
    const int s = (int)(t % kRingStages);
    mbar_wait_parity(&S.full[s], (unsigned)((t / kRingStages) & 1));
#if TL_RING_STATS
    if (t == 0 && wid == 0 && lane == 0) RING_TL(3);
    if (t < 12 && wid == 0 && lane == 0) RING_TL(8 + 2 * t);
    if (t == 0 && wid == 0 && lane == 0) {  // entry -> first stage landed; CTAs
      atomicAdd(&g_vt[6], (unsigned long long)(clock64() - t_entry));
      atomicAdd(&g_vt[7], 1ull);
    }
#endif
    const RingMeta m = S.meta[s];
    if (m.j < 0) break;
    const int kk = min(K, m.n);
    if (m.q == 0) {
      ++c;
      const int b = (int)(c & 1);
      if (c >= 2 && TL_RING_LAB != 2) mbar_wait_parity(&S.freed[b], (unsigned)(((c >> 1) - 1) & 1));  // c - 2 merged
      w.wb = S.wbuf[b][wid];
      w.pub = &S.theta_pub[b];
      theta0 = TL_RING_LAB == 2 ? (0x4050ull << 40) : m.theta;  // lab build 2: a fixed typical threshold, no finish
      w.theta = theta0;
      w.cnt = 0;
    }
#if TL_RING_LAB != 1  // lab build 1: the ring alone (no scan)
    ring_scan<true>(S.ring[s], m.len >> 4, (unsigned)m.q * (kRingStageBytes / 2), w, kk, lane, wid);
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[s]);
    if (t < 12 && wid == 0 && lane == 0) RING_TL(9 + 2 * t);
    if (m.q != m.nst - 1 || TL_RING_LAB == 2) continue;
    const int b = (int)(c & 1);
    // the cooperative finish ranks by binary searches in the consumers' ranked buffers (the
    // key set is unchanged; the general path gathers or ranks them again).  A fuller buffer
    // (compactions, ties) sends the chunk to the general path, which does not need it ranked.
    if (coop && w.cnt <= kRingCoopRankMax) ring_rank(w.wb, w.cnt, lane);
    if (lane == 0) {
      S.cnt[b][wid] = w.cnt;
      S.cmp[b][wid] = w.theta != theta0;
      if (wid == 0) S.job[b] = RingJob{m.j, theta0, kk, m.nst};
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.ready[b]);
    if (wid == 0 && lane == 0) RING_TL(4);
    if (coop && ring_coop_finish<VERIFY>(a, S, o, wid * 32 + lane)) return;
  }
  // no more chunks: release both finishers
  if (TL_RING_LAB == 2) c = -1;
  for (long long cc = c + 1; cc <= c + 2; ++cc) {
    const int b = (int)(cc & 1);
    if (cc >= 2 && TL_RING_LAB != 2) mbar_wait_parity(&S.freed[b], (unsigned)(((cc >> 1) - 1) & 1));
    if (lane == 0) {
      if (wid == 0) S.job[b].j = -1;
      mbar_arrive(&S.ready[b]);
    }
    __syncwarp();
  }
}

// Finisher f: the chunks c with c & 1 == f.  Merge the consumers' ranked lists (or, when
// they hold fewer than kk keys, re-scan the chunk from global memory with a lower
// threshold), update the speculation, then output (prove) or verify.
template <bool VERIFY>
__device__ __forceinline__ void ring_finish(const SelArgs& a, RingSmem& S, int f, int32_t* __restrict__ idx_out,
                                            uint16_t* __restrict__ bits_out, const uint8_t* __restrict__ proofs,
                                            const tl_thresholds& th, tl_chunk_stats* __restrict__ stats_out,
                                            uint8_t* __restrict__ accept_out, int lane, long long t_entry = 0) {
  const int K = a.K, PB = 2 + 2 * K;
  for (long long cseq = f;; cseq += kRingFinishers) {
    const int b = (int)(cseq & 1);  // the consumers' buffer parity of this chunk
    mbar_wait_parity(&S.ready[b], (unsigned)((cseq >> 1) & 1));
#if TL_RING_STATS
    const long long t0 = clock64();
    if (lane == 0 && cseq == f) atomicAdd(&g_vt[5], (unsigned long long)(t0 - t_entry));  // entry -> first chunk ready
#endif
    const RingJob job = S.job[b];
    if (job.j < 0) break;
    const int64_t j = job.j;
    const int kk = job.kk;
    uint32_t pword[kPW];
    if (VERIFY) {  // this chunk's proof words, in flight during the merge
      const uint16_t* pw = reinterpret_cast<const uint16_t*>(proofs + j * PB);
#pragma unroll
      for (int q = 0; q < kPW; ++q) {
        const int tt = lane + 32 * q;
        pword[q] = tt <= K ? (uint32_t)__ldg(pw + tt) : 0u;
      }
    }
    int total = 0;
    bool compacted = false;
#pragma unroll
    for (int q = 0; q < kRingConsumers; ++q) {
      total += S.cnt[b][q];
      compacted = compacted || S.cmp[b][q];
    }
    unsigned long long acc[4];
    int retry = 0;
    bool released = false;
    TL_CHECK(j >= 0 && kk >= 1 && kk <= K && total >= 0);
    // gather the consumers' candidates at or above the chunk's shared threshold (a key below
    // it has kk keys above it in the warp that proved it) into the union scratch
    const unsigned long long theta_f = S.theta_pub[b];
    int kept = 0;
    if (total >= kk) {
      unsigned long long* uni = S.uni[f];
#pragma unroll 1
      for (int q = 0; q < kRingConsumers; ++q) {
        const int cq = S.cnt[b][q];
        for (int i0 = 0; i0 < cq; i0 += 32) {
          const unsigned long long key = i0 + lane < cq ? S.wbuf[b][q][i0 + lane] : 0ull;
          const bool keep = i0 + lane < cq && key >= theta_f;
          const unsigned bal = __ballot_sync(0xFFFFFFFFu, keep);
          const int pos = kept + __popc(bal & lanemask_lt());
          if (keep && pos < kWarpCap) uni[pos] = key;
          kept += __popc(bal);
        }
      }
      __syncwarp();
    }
    if (total >= kk && kept <= kWarpCap) {
      unsigned long long* uni = S.uni[f];
      if (lane == 0) {
        S.theta_pub[b] = 0ull;
        mbar_arrive(&S.freed[b]);  // the consumers may refill their buffers already
      }
      released = true;
      final_sort<kWarpCap / 32, TL_MAX_K>(uni, kept, lane);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = uni[32 * r + lane];
    } else if (total >= kk) {
      // more candidates than the union holds (compactions, heavy ties): rank every buffer
      // and merge the ranked lists
#pragma unroll 1
      for (int q = 0; q < kRingConsumers; ++q) ring_rank(S.wbuf[b][q], S.cnt[b][q], lane);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = S.wbuf[b][0][32 * r + lane];
#pragma unroll 1
      for (int q = 1; q < kRingConsumers; ++q) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const unsigned long long bb = S.wbuf[b][q][127 - (32 * r + lane)];
          acc[r] = acc[r] > bb ? acc[r] : bb;
        }
        bitonic_merge_desc128(acc, lane);
      }
    } else {
      // the speculative theta excluded part of the top-kk: this warp re-scans the whole
      // chunk from global memory (every consumer share) with a lower threshold -- 64, then
      // 256 magnitude steps, then 0 -- using the first list as its buffer
      unsigned long long theta0 = job.theta;
      const ChunkGeo g = chunk_geo(a, j);
      RingScan w;
      w.wb = S.wbuf[b][0];
      do {
        if (theta0 == 0ull) __trap();  // unreachable: theta = 0 admits every element
        const unsigned key = (unsigned)(theta0 >> 40);
        const unsigned drop = retry == 0 ? 64u : 256u;
        theta0 = (retry < 2 && key > drop) ? ((unsigned long long)(key - drop) << 40) : 0ull;
        ++retry;
        w.theta = theta0;
        w.cnt = 0;
        for (int q = 0; q < job.nst; ++q) {
          const int len = min(kRingStageBytes, 2 * g.n - q * kRingStageBytes);
          for (int ws = 0; ws < kRingConsumers; ++ws)
            ring_scan<false>(reinterpret_cast<const uint4*>(g.base) + (size_t)q * kRingStageVec, len >> 4,
                             (unsigned)q * (kRingStageBytes / 2), w, kk, lane, ws);
        }
      } while (w.cnt < kk);
      total = w.cnt;
      compacted = compacted || w.theta != theta0;
      ring_rank(w.wb, w.cnt, lane);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = w.wb[32 * r + lane];
    }
    // speculation, one CTA-wide state updated in chunk order by the two finishers (theta
    // only rises by a compaction: a chunk with too many candidates)
#if TL_RING_STATS
    const long long t_merged = clock64();
#endif
    const int kr = (kk - 1) >> 5;  // register of the kk-th key (a select chain: no local-memory array)
    const unsigned long long kreg = kr == 0 ? acc[0] : kr == 1 ? acc[1] : kr == 2 ? acc[2] : acc[3];
    const unsigned long long kth = __shfl_sync(0xFFFFFFFFu, kreg, (kk - 1) & 31);
    while (*reinterpret_cast<volatile long long*>(&S.spec_seq) != cseq) __nanosleep(64);  // leave the issue slots to the scans
    Spec sp = S.spec;
    int d = sp.delta;
    if (retry) d = min(d + 4 * retry, 0x4000);
    else if ((total > kk + TL_SPEC_HI || compacted) && d > 1) --d;
    else if (total < kk + TL_SPEC_LO) ++d;
    sp.delta = d;
    sp.k0 = sp.k1;
    sp.k1 = (unsigned)(kth >> 40);
    spec_arm(sp);
    __syncwarp();
    if (lane == 0) {
      S.spec = sp;
      *reinterpret_cast<volatile unsigned long long*>(&S.theta_next) = sp.theta;
      __threadfence_block();
      *reinterpret_cast<volatile long long*>(&S.spec_seq) = cseq + 1;
    }
    if (VERIFY) {
      __syncwarp();  // every lane has read the buffers: the union scratch now holds the ranked top-kk
#pragma unroll
      for (int r = 0; r < 4; ++r) S.uni[f][32 * r + lane] = acc[r];
      __syncwarp();
#if TL_RING_STATS
      const long long t_spec = clock64();
#endif
      verify_tail_warp<true>(S.uni[f], kk, K, pword, S.coef[f], th, stats_out, accept_out, j, lane);
#if TL_RING_STATS
      if (lane == 0) {
        atomicAdd(&g_ring_stats[5], (unsigned long long)(t_merged - t0));
        atomicAdd(&g_ring_stats[6], (unsigned long long)(t_spec - t_merged));
        atomicAdd(&g_ring_stats[7], (unsigned long long)(clock64() - t_spec));
      }
#endif
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = 32 * r + lane;
        if (i < K) {
          idx_out[j * K + i] = i < kk ? (int32_t)key_idx(acc[r]) : -1;
          bits_out[j * K + i] = i < kk ? (uint16_t)(acc[r] & 0xFFFFu) : (uint16_t)0;
        }
      }
    }
#if TL_RING_STATS
    if (lane == 0 && blockIdx.x == 0) {
      const unsigned n = atomicAdd(&g_ring_trace_n, 1u);
      if (n < 1024) {
        g_ring_trace[n][0] = (unsigned)(job.theta >> 40) | (unsigned)f << 31;
        g_ring_trace[n][1] = (unsigned)total;
        g_ring_trace[n][2] = (unsigned)d;
        g_ring_trace[n][3] = (unsigned)(kth >> 40);
      }
    }
    if (lane == 0) {
      atomicAdd(&g_ring_stats[0], 1ull);
      atomicAdd(&g_ring_stats[1], (unsigned long long)total);
      atomicAdd(&g_ring_stats[2], (unsigned long long)retry);
      atomicAdd(&g_ring_stats[3], compacted ? 1ull : 0ull);
      atomicAdd(&g_ring_stats[4], (unsigned long long)(clock64() - t0));
    }
#endif
    __syncwarp();
    if (lane == 0 && !released) {
      S.theta_pub[b] = 0ull;
      mbar_arrive(&S.freed[b]);
    }
  }
  if (f == 0) spec_store(a.spec, blockIdx.x, S.spec, lane);
}

template <bool VERIFY>
__global__ void __launch_bounds__(kRingThreads, kRingCtasPerSm)
ring_stream_kernel(SelArgs a, int32_t* __restrict__ idx_out, uint16_t* __restrict__ bits_out,
                   const uint8_t* __restrict__ proofs, tl_thresholds th, tl_chunk_stats* __restrict__ stats_out,
                   uint8_t* __restrict__ accept_out) {
  extern __shared__ __align__(128) uint8_t ring_smem[];
  RingSmem& S = *reinterpret_cast<RingSmem*>(ring_smem);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if TL_RING_STATS
  const long long t_entry = clock64();
  const unsigned long long tl_entry_ = ring_gt();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    g_ring_tl_launch = atomicAdd(&g_ring_tl_n, 1u);
    g_ring_tl[g_ring_tl_launch & 63u][0] = tl_entry_;
  }
#else
  const long long t_entry = 0;
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRingStages; ++s) {
      mbar_init_count(&S.full[s], 1);
      mbar_init_count(&S.empty[s], kRingConsumers);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init_count(&S.ready[b], kRingConsumers);
      mbar_init_count(&S.freed[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    S.spec = spec_load(a.spec, blockIdx.x);
    S.spec_seq = 0;
    S.theta_pub[0] = S.theta_pub[1] = 0ull;
    S.theta_next = S.spec.theta;
  }
  if (a.prefix == nullptr) {
    // small batch (<= kRingOwnPrefixMax rollouts): this CTA builds the chunk prefix itself,
    // sparing the chunk_prefix_kernel launch; CTA 0 leaves a copy for rollout_verdict_kernel
    for (int r = threadIdx.x; r < a.n_roll; r += blockDim.x) {
      const int64_t T = a.row_off[r + 1] - a.row_off[r];
      S.pfx[r + 1] = T > 0 ? (T + a.C - 1) / a.C : 0;
    }
    __syncthreads();
    if (wid == 0) {
      int64_t carry = 0;
      for (int base = 0; base < a.n_roll; base += 32) {
        int64_t v = base + lane < a.n_roll ? S.pfx[base + lane + 1] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t y = __shfl_up_sync(0xFFFFFFFFu, v, o);
          if (lane >= o) v += y;
        }
        if (base + lane < a.n_roll) S.pfx[base + lane + 1] = carry + v;
        carry += __shfl_sync(0xFFFFFFFFu, v, 31);
      }
      if (lane == 0) S.pfx[0] = 0;
    }
    __syncthreads();
    if (blockIdx.x == 0 && a.prefix_out)
      for (int r = threadIdx.x; r <= a.n_roll; r += blockDim.x) a.prefix_out[r] = S.pfx[r];
    a.prefix = S.pfx;
  }
  __syncthreads();
  const int64_t n_chunks = min(a.n_chunks, a.prefix[a.n_roll]);
  // one chunk per CTA (the grid covers the batch): the consumers and the finisher finish it together
  const bool coop = TL_RING_LAB == 0 && (int64_t)gridDim.x >= n_chunks && (int64_t)blockIdx.x < n_chunks;
  if (threadIdx.x == 0) RING_TL(1);
  const RingOut o{idx_out, bits_out, proofs, th, stats_out, accept_out};
  if (wid == kRingProducer) ring_produce(a, S, n_chunks, lane, VERIFY ? proofs : nullptr);
  else if (wid >= kRingConsumers) {
    if (!(coop && ring_coop_finish<VERIFY>(a, S, o, (int)threadIdx.x)))
      ring_finish<VERIFY>(a, S, wid - kRingConsumers, idx_out, bits_out, proofs, th, stats_out, accept_out, lane,
                          t_entry);
  } else {
    ring_consume<VERIFY>(a, S, a.K, lane, wid, coop, o, t_entry);
  }
}

// ----------------------------------------------------------------------------- record checks
// One 256-thread CTA per record (grid-stride over records): termination
// (checks.py:120-131), sampling (checks.py:134-142), commitment verdict, in the
// reference's order.  The sampling fraction is the exact count of probs < p_low
// divided once in float64, like np.mean over a bool array.  Each thread counts a
// strided share with 4 independent loads in flight; a warp reduction and one shared
// word per warp finish the count.
constexpr int kRecThreads = 256;
__global__ void __launch_bounds__(kRecThreads) record_checks_kernel(const double* __restrict__ probs, const int64_t* __restrict__ row_off,
                                     int n_roll, const int32_t* __restrict__ prompt_len,
                                     const uint8_t* __restrict__ ends_with_eos, tl_record_thresholds th,
                                     const uint8_t* __restrict__ commit_accept,
                                     const uint8_t* __restrict__ commit_checked, int32_t* __restrict__ verdict_out,
                                     double* __restrict__ frac_out, double* __restrict__ p_last_out) {
  __shared__ unsigned long long part[kRecThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int r = blockIdx.x; r < n_roll; r += gridDim.x) {
  const int64_t lo = row_off[r], T = row_off[r + 1] - lo;
  unsigned long long cnt = 0;
  int64_t i = tid;
  for (; i + 3 * kRecThreads < T; i += 4 * kRecThreads) {
    const double a = probs[lo + i], b = probs[lo + i + kRecThreads];
    const double c = probs[lo + i + 2 * kRecThreads], d = probs[lo + i + 3 * kRecThreads];
    cnt += (a < th.p_low) + (b < th.p_low) + (c < th.p_low) + (d < th.p_low);
  }
  for (; i < T; i += kRecThreads) cnt += probs[lo + i] < th.p_low ? 1ull : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  if (lane == 0) part[tid >> 5] = cnt;
  __syncthreads();
  if (tid == 0) {
  cnt = 0;
#pragma unroll
  for (int w = 0; w < kRecThreads / 32; ++w) cnt += part[w];
  const double frac = T > 0 ? __ddiv_rn((double)cnt, (double)T) : 0.0;
  const double p_last = T > 0 ? probs[lo + T - 1] : __longlong_as_double(0x7FF8000000000000ll);
  const bool term_ok = (int64_t)prompt_len[r] + T >= (int64_t)th.max_len ||
                       (T > 0 && ends_with_eos[r] && p_last > th.eos_prob_floor);
  const bool samp_ok = T < (int64_t)th.min_sampling_len || !(frac > th.theta);
  const bool checked = commit_checked == nullptr || commit_checked[r] != 0;
  const bool com_ok = commit_accept == nullptr || !checked || commit_accept[r] != 0;
  verdict_out[r] = !term_ok ? 1 : !samp_ok ? 2 : !com_ok ? 3 : 0;
  if (frac_out) frac_out[r] = frac;
  if (p_last_out) p_last_out[r] = p_last;
  }
  __syncthreads();  // part[] is reused by the next record
  }
}

// ----------------------------------------------------------------------------- exact mode
// dtype codes: 0 float64, 1 float32, 2 bfloat16, 3 float16
template <int DT>
__device__ __forceinline__ uint64_t load_raw(const void* in, int64_t i) {
  if (DT == 0) return (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(in) + i);
  if (DT == 1) return (uint64_t)__ldg(reinterpret_cast<const unsigned int*>(in) + i);
  return (uint64_t)__ldg(reinterpret_cast<const unsigned short*>(in) + i);
}

// Widen a raw element to float64 exactly; NaNs keep sign and payload (quieted) the way
// x86 cvtss2sd / numpy widen them.
template <int DT>
__device__ __forceinline__ double raw_to_f64(uint64_t raw) {
  if (DT == 0) return __longlong_as_double((long long)raw);
  if (DT == 1 || DT == 2) {
    const uint32_t b = DT == 1 ? (uint32_t)raw : (uint32_t)raw << 16;
    if ((b & 0x7FFFFFFFu) > 0x7F800000u)
      return __longlong_as_double((long long)(((uint64_t)(b >> 31) << 63) | 0x7FF8000000000000ull |
                                              ((uint64_t)(b & 0x7FFFFFu) << 29)));
    return (double)__uint_as_float(b);
  }
  const uint16_t h = (uint16_t)raw;
  if ((h & 0x7FFFu) > 0x7C00u)
    return __longlong_as_double((long long)(((uint64_t)(h >> 15) << 63) | 0x7FF8000000000000ull |
                                            ((uint64_t)(h & 0x3FFu) << 42)));
  return (double)__half2float(__ushort_as_half(h));
}

__device__ __forceinline__ double load_as_f64(const void* in, int dtype, int64_t i) {
  switch (dtype) {
    case 0: return raw_to_f64<0>(load_raw<0>(in, i));
    case 1: return raw_to_f64<1>(load_raw<1>(in, i));
    case 2: return raw_to_f64<2>(load_raw<2>(in, i));
    default: return raw_to_f64<3>(load_raw<3>(in, i));
  }
}

// np.round(x, 6) = rint(x * 1e6) / 1e6 in float64, the division correctly rounded.
// The division is branch-free (no __ddiv_rn slow path) so it interleaves with the
// SHA rounds of the chain kernel: q0 = RN(r * RN(1e-6)) is within 1.5 ulp of r/1e6,
// the FMA remainder r - 1e6*q0 is exact, and q = RN(q0 + rem * RN(1e-6)) differs from
// r/1e6 by < 2^-52 ulp.  r is an integer-valued double, so r/1e6 = N/15625 ulp units
// for an integer N: it is never a rounding midpoint and never closer to one than
// 1/31250 ulp, hence q = RN(r/1e6) exactly (tests/test_gpu_exact.py checks every
// float32 input against torch's correctly rounded division).  0 keeps its sign, inf
// stays inf; NaN keeps its payload, quieted (np.round).
__device__ __forceinline__ double round6_value(double x) {
  const double r = rint(__dmul_rn(x, 1e6));
  const double q0 = __dmul_rn(r, 1e-6);
  const double q = __fma_rn(__fma_rn(-q0, 1e6, r), 1e-6, q0);
  const double nanq = __longlong_as_double(__double_as_longlong(x) | 0x0008000000000000ll);
  return x != x ? nanq : (r == 0.0 || fabs(r) == __longlong_as_double(0x7FF0000000000000ll)) ? r : q;
}

__global__ void round6_kernel(const void* __restrict__ in, int dtype, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = round6_value(load_as_f64(in, dtype, i));
}

// ----------------------------------------------------------------------------- exact mode on the GPU
// The reference's commitment chain (rollout.py:51-68): d_{-1} = 0^32,
// d_j = SHA-256(d_{j-1} || LE-f64(round(h[jk:(j+1)k], 6))).  A chain is serial, so
// each thread owns one rollout; it wins over the host (SHA-NI on every core) once a
// batch has enough rollouts (DESIGN 5.6).  SHA-256 is FIPS
// 180-4: the round constants are the first 32 bits of the fractional parts of the
// cube roots of the first 64 primes (generated, and checked against hashlib).
__constant__ uint32_t kSha256K[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void sha256_block(uint32_t (&st)[8], uint32_t (&w)[16]) {
  uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
  for (int t = 0; t < 64; ++t) {
    uint32_t wt;
    if (t < 16) {
      wt = w[t];
    } else {
      const uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
      const uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
      const uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
      wt = w[t & 15] = w[t & 15] + s0 + w[(t - 7) & 15] + s1;
    }
    const uint32_t t1 = h + (rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25)) + ((e & f) ^ (~e & g)) + kSha256K[t] + wt;
    const uint32_t t2 = (rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
    h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

constexpr int kShaPrefetch = 16;  // 64-byte message blocks ahead (L1 line prefetch)

template <int DT>
__device__ __forceinline__ const void* elem_addr(const void* in, int64_t i) {
  return static_cast<const char*>(in) + i * (DT == 0 ? 8 : DT == 1 ? 4 : 2);
}

// Raw elements of message block b (element slots e = 8b - 4 + s; 0 outside the data).
template <int DT>
__device__ __forceinline__ void fetch_block(const void* in, int64_t base, int64_t n_el, int64_t b, uint64_t (&raw)[8]) {
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int64_t e = 8 * b - 4 + s;
    raw[s] = (e >= 0 && e < n_el) ? load_raw<DT>(in, base + e) : 0ull;
  }
}

// Message words of block b: the previous digest (block 0), the rounded values as the
// big-endian words of their little-endian bytes, the 0x80 terminator, the bit length.
template <int DT>
__device__ __forceinline__ void assemble_block(const uint64_t (&raw)[8], int64_t b, int64_t n_el, int64_t n_blocks,
                                               uint64_t bits, const uint32_t (&prev)[8], uint32_t (&w)[16]) {
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int64_t e = 8 * b - 4 + s;
    uint32_t lo = 0u, hi = 0u;
    if (e < 0) {
      lo = prev[2 * s];
      hi = prev[2 * s + 1];
    } else if (e < n_el) {
      const uint64_t v = (uint64_t)__double_as_longlong(round6_value(raw_to_f64<DT>(raw[s])));
      lo = __byte_perm((uint32_t)v, 0u, 0x0123);
      hi = __byte_perm((uint32_t)(v >> 32), 0u, 0x0123);
    } else if (e == n_el) {
      lo = 0x80000000u;
    }
    w[2 * s] = lo;
    w[2 * s + 1] = hi;
  }
  if (b == n_blocks - 1) {
    w[14] = (uint32_t)(bits >> 32);
    w[15] = (uint32_t)bits;
  }
}

// Position of one rollout's chain: digest j, message block b of that digest.
struct ChainCursor {
  int64_t T, row0, j, b, nd, n_el, n_blocks, base;
  int H, k;
  __device__ __forceinline__ void start_digest() {
    const int64_t rows = T > 0 ? min((int64_t)k, T - j * k) : 0;
    base = (row0 + j * k) * (int64_t)H;
    n_el = rows * (int64_t)H;
    n_blocks = (8 + 2 * n_el + 3 + 15) / 16;  // data words + 0x80 word + 64-bit length
  }
  __device__ __forceinline__ void init(int64_t T_, int64_t row0_, int H_, int k_) {
    T = T_; row0 = row0_; H = H_; k = k_; j = 0; b = 0;
    nd = T > 0 ? (T + k - 1) / k : 1;
    start_digest();
  }
  __device__ __forceinline__ uint64_t bits() const { return (uint64_t)(32 + 8 * n_el) * 8u; }
  __device__ __forceinline__ void advance() {
    if (++b == n_blocks) {
      b = 0;
      if (++j < nd) start_digest();
    }
  }
  // message blocks over the whole chain
  __device__ __forceinline__ int64_t total_blocks() const {
    auto nb = [](int64_t n) { return (8 + 2 * n + 3 + 15) / 16; };
    if (T <= 0) return nb(0);
    const int64_t rem = T % k;
    return (T / k) * nb((int64_t)k * H) + (rem ? nb(rem * H) : 0);
  }
};

constexpr int kChainStages = 4;  // message blocks in flight between the two warps

__device__ __forceinline__ void named_bar_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void named_bar_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }

// The reference's commitment chain (rollout.py:51-68), one chain per rollout:
// ceil(T/k) digests (one for T = 0), 32 bytes each, at digests_out + 32 * dig_off[r].
// The message of digest j is the previous digest (8 words) followed by the block's
// rounded float64 values, then the SHA padding.
//
// A chain is serial, so the only parallelism is one lane per rollout, and a B200 sees
// ~one warp per SM sub-partition: the compression is latency-bound on its own
// dependencies.  The CTA is therefore warp-specialised over 32 rollouts: warp 1 loads,
// rounds and packs the message blocks into a shared-memory ring (kChainStages deep,
// named barriers 1..2*kChainStages), warp 0 runs nothing but the SHA-256 rounds and
// patches the previous digest into each digest's first block.  The two warps sit on
// different sub-partitions, so the compression runs at its bare rate.
template <int DT>
__global__ void __launch_bounds__(64) exact_chain_kernel(const void* __restrict__ in,
                                                         const int64_t* __restrict__ row_off, int n_roll, int H,
                                                         int k, const int64_t* __restrict__ dig_off,
                                                         uint8_t* __restrict__ digests_out) {
  __shared__ uint4 ring[kChainStages][4][32];  // 16 words per lane as 4 x 16 B, lane-interleaved (conflict-free)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + lane;
  ChainCursor cur;
  cur.init(r < n_roll ? row_off[r + 1] - row_off[r] : 0, r < n_roll ? row_off[r] : 0, H, k);
  const int64_t total = r < n_roll ? cur.total_blocks() : 0;
  int64_t iters = total;  // both warps run the same number of ring steps
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) iters = max(iters, (int64_t)__shfl_xor_sync(0xFFFFFFFFu, (long long)iters, o));

  if (warp == 1) {  // ------------------------------------------------ producer
    const uint32_t zero[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    for (int64_t i = 0; i < iters; ++i) {
      const int s = (int)(i % kChainStages);
      if (i >= kChainStages) named_bar_sync(1 + kChainStages + s);  // the consumer has read stage s
      uint32_t w[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) w[q] = 0u;
      if (i < total) {
        if (8 * (cur.b + kShaPrefetch) - 4 < cur.n_el)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(elem_addr<DT>(in, cur.base + 8 * (cur.b + kShaPrefetch) - 4)));
        uint64_t raw[8];
        fetch_block<DT>(in, cur.base, cur.n_el, cur.b, raw);
        assemble_block<DT>(raw, cur.b, cur.n_el, cur.n_blocks, cur.bits(), zero, w);
        cur.advance();
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) ring[s][q][lane] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      named_bar_arrive(1 + s);  // stage s is full
    }
    for (int64_t i = max(iters, (int64_t)kChainStages); i < iters + kChainStages; ++i)
      named_bar_sync(1 + kChainStages + (int)(i % kChainStages));  // match the consumer's last arrivals
    return;
  }
  // ------------------------------------------------------------------ consumer
  uint32_t prev[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  uint32_t st[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                    0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  uint32_t* out = reinterpret_cast<uint32_t*>(digests_out + 32 * (r < n_roll ? dig_off[r] : 0));
  for (int64_t i = 0; i < iters; ++i) {
    const int s = (int)(i % kChainStages);
    named_bar_sync(1 + s);  // stage s is full
    uint32_t w[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = ring[s][q][lane];
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
    named_bar_arrive(1 + kChainStages + s);  // stage s may be refilled
    if (i < total) {
      if (cur.b == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = prev[q];
      }
      sha256_block(st, w);
      if (cur.b == cur.n_blocks - 1) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          out[8 * cur.j + q] = __byte_perm(st[q], 0u, 0x0123);  // big-endian digest bytes
          prev[q] = st[q];
        }
        st[0] = 0x6a09e667u; st[1] = 0xbb67ae85u; st[2] = 0x3c6ef372u; st[3] = 0xa54ff53au;
        st[4] = 0x510e527fu; st[5] = 0x9b05688cu; st[6] = 0x1f83d9abu; st[7] = 0x5be0cd19u;
      }
      cur.advance();
    }
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
  size_t spec, next, prefix, idx, bits, accept, part, part_cnt, total;
};
WsLayout ws_layout(int32_t n_roll, int64_t n_chunks, int32_t K) {
  WsLayout L;
  size_t o = 0;
  L.spec = o; o += (size_t)kSpecSlots * 16;  // first, so its offset never depends on the shape
  L.next = o; o += 256;                       // chunk counters: [0] streaming kernels, [1] commit
  L.prefix = o; o = align_up(o + (size_t)(n_roll + 1) * 8, 256);
  L.idx = o; o = align_up(o + (size_t)n_chunks * K * 4, 256);
  L.bits = o; o = align_up(o + (size_t)n_chunks * K * 2, 256);
  L.accept = o; o = align_up(o + (size_t)n_chunks, 256);
  L.part = o; o = align_up(o + (size_t)kSplitMaxLists * TL_MAX_K * 8, 256);
  L.part_cnt = o; o = align_up(o + (size_t)kSplitMaxChunks * 4, 256);
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

// ---- SM partitions (driver green contexts), for the pipelined schedule: the streaming
// kernels on most SMs, the commitment on a few.  Driver functions are fetched through
// the runtime (cudaGetDriverEntryPoint), so the library needs no libcuda at link time.
struct DriverFns {
  CUresult (*stream_green_ctx)(CUstream, CUgreenCtx*) = nullptr;
  CUresult (*green_resource)(CUgreenCtx, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*device_get)(CUdevice*, int) = nullptr;
  CUresult (*device_resource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*split_by_count)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                             unsigned int) = nullptr;
  CUresult (*generate_desc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
  CUresult (*green_create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
  CUresult (*green_destroy)(CUgreenCtx) = nullptr;
  CUresult (*green_stream_create)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
  CUresult (*stream_destroy)(CUstream) = nullptr;
  bool ok = false;
};

template <typename F>
bool driver_fn(const char* name, F& f) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p) {
    cudaGetLastError();
    return false;
  }
  f = reinterpret_cast<F>(p);
  return true;
}

const DriverFns& driver() {
  static const DriverFns fns = [] {
    DriverFns f;
    f.ok = driver_fn("cuStreamGetGreenCtx", f.stream_green_ctx) &&
           driver_fn("cuGreenCtxGetDevResource", f.green_resource) && driver_fn("cuDeviceGet", f.device_get) &&
           driver_fn("cuDeviceGetDevResource", f.device_resource) &&
           driver_fn("cuDevSmResourceSplitByCount", f.split_by_count) &&
           driver_fn("cuDevResourceGenerateDesc", f.generate_desc) && driver_fn("cuGreenCtxCreate", f.green_create) &&
           driver_fn("cuGreenCtxDestroy", f.green_destroy) &&
           driver_fn("cuGreenCtxStreamCreate", f.green_stream_create) &&
           driver_fn("cuStreamDestroy", f.stream_destroy);
    return f;
  }();
  return fns;
}

// The green context behind a stream, or nullptr for an ordinary stream.
CUgreenCtx stream_green_ctx(cudaStream_t st) {
  const DriverFns& d = driver();
  CUgreenCtx g = nullptr;
  if (!st || !d.ok || d.stream_green_ctx(reinterpret_cast<CUstream>(st), &g) != CUDA_SUCCESS) return nullptr;
  return g;
}

// SMs the kernels launched on `st` can use: its green partition, else the device.
int stream_sms(cudaStream_t st) {
  const CUgreenCtx g = stream_green_ctx(st);
  CUdevResource r;
  if (g && driver().green_resource(g, &r, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS && r.sm.smCount > 0)
    return (int)r.sm.smCount;
  return sm_count();
}

int sel_grid(int64_t n_chunks, const void* kernel, cudaStream_t st, int ctas_per_sm = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSelBlockThreads, kSelSmem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  if (ctas_per_sm > 0 && ctas_per_sm < per_sm) per_sm = ctas_per_sm;
  // one warp per chunk: the fewest warps that finish in the same number of rounds
  // as the full grid (fewer warps share HBM bandwidth, so each round is shorter)
  const int64_t wmax = (int64_t)stream_sms(st) * per_sm * kSelWarps;
  const int64_t rounds = (n_chunks + wmax - 1) / wmax;
  const int64_t warps = rounds > 0 ? (n_chunks + rounds - 1) / rounds : 1;
  return (int)((warps + kSelWarps - 1) / kSelWarps);
}

// Grid and warps-per-chunk of a streaming launch.  A batch too small to give every warp
// slot of the grid a chunk splits each chunk over up to kSplitMax warps (each part at
// least kSplitMinPart elements): small batches are latency-bound per warp, and more
// warps per chunk fill the GPU.
struct SelPlan { int grid, split; };
SelPlan sel_plan(int64_t n_chunks, int64_t chunk_elems, const void* kernel, cudaStream_t st, int ctas_per_sm) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSelBlockThreads, kSelSmem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  if (ctas_per_sm > 0 && ctas_per_sm < per_sm) per_sm = ctas_per_sm;
  const int64_t wmax = (int64_t)stream_sms(st) * per_sm * kSelWarps;
  int64_t split = n_chunks > 0 ? wmax / n_chunks : 1;
  split = min(split, (int64_t)kSplitMax);
  split = min(split, chunk_elems / kSplitMinPart);
  if (n_chunks > kSplitMaxChunks || split * n_chunks > kSplitMaxLists) split = 1;
  if (split >= 2) return {(int)((n_chunks * split + kSelWarps - 1) / kSelWarps), (int)split};
  return {sel_grid(n_chunks, kernel, st, ctas_per_sm), 1};
}

int launch_status() { return cudaGetLastError() == cudaSuccess ? TL_OK : TL_ECUDA; }

// cudaFuncSetAttribute once per kernel and device (a per-call attribute write costs host
// time on the latency-bound small batches).  The cache is set-once, not mutable state
// that affects results.
template <auto KERNEL>
int smem_attr_once(size_t bytes) {
  static std::atomic<uint32_t> done{0u};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TL_ECUDA;
  const uint32_t bit = 1u << (dev & 31);
  if (done.load(std::memory_order_acquire) & bit) return TL_OK;
  if (cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return TL_ECUDA;
  done.fetch_or(bit, std::memory_order_acq_rel);
  return TL_OK;
}

// The TMA-ring kernels take 16-B aligned chunks (H % 8 == 0 and an aligned hidden pointer):
// small batches when the caller leaves the launch shape to the library (ctas_per_sm == 0),
// any batch with -2; other values select the one-warp-per-chunk kernels (e.g. beside a
// co-resident commitment).
constexpr int kRingOptIn = -2;  // ctas_per_sm value that selects the ring kernels
// A ring launch whose grid covers the batch (no chunk claims) over at most
// kRingOwnPrefixMax rollouts builds its chunk prefix itself (no chunk_prefix_kernel).
bool ring_own_prefix(int rg, int64_t n_chunks, int n_roll) {
  return rg > 0 && n_chunks <= rg && n_roll <= kRingOwnPrefixMax;
}

int ring_grid(const uint16_t* hidden, int H, int64_t n_chunks, int ctas_per_sm, cudaStream_t st, bool verify) {
  // Auto (0) takes the ring only for batches of at most one chunk per ring CTA, where a
  // chunk streamed by a whole CTA (all its stages in flight at once) finishes sooner than
  // by two warps of the split kernels: configuration 1 select 26 vs 34 us, 1 x 8192 x 5120
  // 39 vs 48 us.  Larger batches keep the one-warp kernels (DESIGN 5.1b: at configuration 2
  // the ring select runs 3.02-3.11 ms against 3.05 ms and the ring verify 3.15 against 3.02
  // ms, and in the partitioned pipeline its 2 x 111 KiB of shared memory per SM keeps
  // verify(k-2) off the SMs select(k) holds).  -2 opts in at any size.
  (void)verify;
  if ((ctas_per_sm != kRingOptIn && ctas_per_sm != 0) || H % 8 != 0 ||
      (reinterpret_cast<uintptr_t>(hidden) & 15u))
    return 0;
  const int64_t grid = (int64_t)stream_sms(st) * kRingCtasPerSm;
  if (ctas_per_sm == 0 && n_chunks > grid) return 0;
  return (int)min(grid, max(n_chunks, (int64_t)1));
}

template <int WARPS, bool HALF>
int launch_commit_t(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int K, uint8_t* proofs,
                    unsigned long long* next, cudaStream_t st) {
  const size_t smem = (size_t)(HALF ? kHalfTab : 65536) * 2 + (2 * 128 + kHashSlots) * WARPS * 4;
  if (smem_attr_once<commit_kernel<WARPS, HALF>>(smem)) return TL_ECUDA;
  int grid = stream_sms(st);  // one CTA per SM of the stream's partition
  if ((int64_t)grid * WARPS > n_chunks) grid = (int)((n_chunks + WARPS - 1) / WARPS);
  commit_kernel<WARPS, HALF><<<grid, WARPS * 32, smem, st>>>(idx, bits, n_chunks, K, proofs, next);
  return launch_status();
}

// co_resident = 0: 32 warps, full 128 KiB table (fastest alone); 1: 8 warps, 64 KiB
// half table, <= 64 registers -- fits beside 16 one-warp select/verify CTAs per SM.
// A batch with at most one chunk per SM sub-partition takes commit_coop_kernel (tl_commit_ex);
// without it (co-resident callers), 4-warp CTAs: every chunk's warp has a sub-partition to
// itself (a 32-warp CTA would stack 8 chunks on each sub-partition of a few SMs).
constexpr int kSmallCommitWarps = 4;
// Devices whose inverse tables are known built and visible to every stream (tl_prepare).
std::atomic<uint32_t> g_tables_prepared{0u};

int launch_commit(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int K, uint8_t* proofs,
                  unsigned long long* next, int co_resident, cudaStream_t st) {
  if (co_resident) return launch_commit_t<kCoCommitWarps, true>(idx, bits, n_chunks, K, proofs, next, st);
  if (n_chunks <= (int64_t)stream_sms(st) * kSmallCommitWarps)
    return launch_commit_t<kSmallCommitWarps, false>(idx, bits, n_chunks, K, proofs, next, st);
  return launch_commit_t<kCommitWarps, false>(idx, bits, n_chunks, K, proofs, next, st);
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
  unsigned* part_cnt = reinterpret_cast<unsigned*>(ws + L.part_cnt);
  SelArgs a{hidden, row_off, prefix, reinterpret_cast<uint4*>(ws + L.spec),
            reinterpret_cast<unsigned long long*>(ws + L.next), n_roll, H, C, K, n_chunks};
  a.n_rows = n_rows;
  const int rg = ring_grid(hidden, H, n_chunks, ctas_per_sm, st, false);
  if (ring_own_prefix(rg, n_chunks, n_roll)) {
    a.prefix = nullptr;  // built in the ring kernel
    a.prefix_out = prefix;
  } else {
    chunk_prefix_kernel<<<1, 1024, 0, st>>>(row_off, n_roll, C, prefix,
                                            reinterpret_cast<unsigned long long*>(ws + L.next), part_cnt);
  }
  if (rg) {
    if (smem_attr_once<ring_stream_kernel<false>>(kRingSmem)) return TL_ECUDA;
    ring_stream_kernel<false><<<rg, kRingThreads, kRingSmem, st>>>(a, idx_out, bits_out, nullptr, tl_thresholds{},
                                                                   nullptr, nullptr);
    return launch_status();
  }
  if (smem_attr_once<prove_select_kernel<false>>(kSelSmem) || smem_attr_once<prove_select_kernel<true>>(kSelSmem))
    return TL_ECUDA;
  if (ctas_per_sm < 0) ctas_per_sm = 0;
  const SelPlan sp = sel_plan(n_chunks, (int64_t)C * H, (const void*)prove_select_kernel<false>, st, ctas_per_sm);
  a.split = sp.split;
  a.part = reinterpret_cast<unsigned long long*>(ws + L.part);
  a.part_cnt = part_cnt;
  if (sp.split > 1)
    prove_select_kernel<true><<<sp.grid, kSelBlockThreads, kSelSmem, st>>>(a, idx_out, bits_out);
  else
    prove_select_kernel<false><<<sp.grid, kSelBlockThreads, kSelSmem, st>>>(a, idx_out, bits_out);
  return launch_status();
}

#if TL_PHASE_PROF
int tl_phase_prof_warps(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_prof_warp, sizeof(g_prof_warp)) == cudaSuccess ? TL_OK : TL_ECUDA;
}
int tl_phase_prof(unsigned long long* out64, int reset) {
  if (cudaMemcpyFromSymbol(out64, g_prof, sizeof(g_prof)) != cudaSuccess) return TL_ECUDA;
  if (reset) {
    static const unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(g_prof, z, sizeof(z)) != cudaSuccess) return TL_ECUDA;
  }
  return TL_OK;
}
#endif

int tl_commit(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int32_t K,
              uint8_t* proofs_out, void* workspace, size_t workspace_bytes, void* stream) {
  return tl_commit_ex(idx, bits, n_chunks, K, proofs_out, workspace, workspace_bytes, 0, stream);
}

int tl_commit_ex(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int32_t K, uint8_t* proofs_out,
                 void* workspace, size_t workspace_bytes, int32_t co_resident, void* stream) {
  if (n_chunks < 0 || K < 1) return TL_EINVAL;
  if (K > TL_MAX_K) return TL_EUNSUPPORTED;
  if (n_chunks == 0) return TL_OK;
  if (!idx || !bits || !proofs_out || !workspace) return TL_EINVAL;
  const WsLayout L = ws_layout(0, n_chunks, K);
  if (workspace_bytes < L.next + 256 || (reinterpret_cast<uintptr_t>(workspace) & 255)) return TL_EWORKSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  unsigned long long* next = reinterpret_cast<unsigned long long*>(ws + L.next) + 1;  // commit's own counter
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // a small batch (at most one chunk per SM sub-partition) is one launch of one 128-thread
  // CTA per chunk: no inverse table, no chunk counter (commit_coop_kernel)
  if (!co_resident && n_chunks <= (int64_t)stream_sms(st) * kSmallCommitWarps) {
    commit_coop_kernel<<<(unsigned)n_chunks, kCoopCommitThreads, 0, st>>>(idx, bits, n_chunks, K, proofs_out);
    return launch_status();
  }
  inv_table_kernel<<<dim3(kInvTableBlocks, kInvTables), kInvTableThreads, 0, st>>>(next);
  return launch_commit(idx, bits, n_chunks, K, proofs_out, next, co_resident, st);
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

  unsigned* part_cnt = reinterpret_cast<unsigned*>(ws + L.part_cnt);
  const int rg = n_chunks > 0 ? ring_grid(hidden, H, n_chunks, ctas_per_sm, st, true) : 0;
  const bool own_prefix = ring_own_prefix(rg, n_chunks, n_roll);
  if (!own_prefix)
    chunk_prefix_kernel<<<1, 1024, 0, st>>>(row_off, n_roll, C, prefix,
                                            reinterpret_cast<unsigned long long*>(ws + L.next), part_cnt);
  if (n_chunks > 0) {
    SelArgs a{hidden, row_off, prefix, reinterpret_cast<uint4*>(ws + L.spec),
              reinterpret_cast<unsigned long long*>(ws + L.next), n_roll, H, C, K, n_chunks};
    a.n_rows = n_rows;
    if (own_prefix) {
      a.prefix = nullptr;  // built in the ring kernel
      a.prefix_out = prefix;
    }
    if (rg) {
      if (smem_attr_once<ring_stream_kernel<true>>(kRingSmem)) return TL_ECUDA;
    } else if (smem_attr_once<verify_kernel<false>>(kSelSmem) || smem_attr_once<verify_kernel<true>>(kSelSmem)) {
      return TL_ECUDA;
    }
    if (ctas_per_sm < 0) ctas_per_sm = 0;
    const SelPlan sp = rg ? SelPlan{rg, 1}
                          : sel_plan(n_chunks, (int64_t)C * H, (const void*)verify_kernel<false>, st, ctas_per_sm);
    a.split = sp.split;
    a.part = reinterpret_cast<unsigned long long*>(ws + L.part);
    a.part_cnt = part_cnt;
    if (rg)
      ring_stream_kernel<true><<<rg, kRingThreads, kRingSmem, st>>>(a, nullptr, nullptr, proofs, *thresholds_host,
                                                                    stats_out, accept);
    else if (sp.split > 1)
      verify_kernel<true><<<sp.grid, kSelBlockThreads, kSelSmem, st>>>(a, proofs, *thresholds_host, stats_out,
                                                                        accept);
    else
      verify_kernel<false><<<sp.grid, kSelBlockThreads, kSelSmem, st>>>(a, proofs, *thresholds_host, stats_out,
                                                                         accept);
  }
  if (rollout_accept_out)
    rollout_verdict_kernel<<<(n_roll + 7) / 8, 256, 0, st>>>(accept, prefix, n_roll, n_chunks, rollout_accept_out);
  return launch_status();
}

int tl_record_checks(const double* probs, const int64_t* row_off, int32_t n_roll, const int32_t* prompt_len,
                     const uint8_t* ends_with_eos, const tl_record_thresholds* thresholds_host,
                     const uint8_t* commit_accept, const uint8_t* commit_checked, int32_t* verdict_out,
                     double* frac_out, double* p_last_out, void* stream) {
  if (n_roll < 0 || !thresholds_host) return TL_EINVAL;
  if (n_roll == 0) return TL_OK;
  if (!probs || !row_off || !prompt_len || !ends_with_eos || !verdict_out) return TL_EINVAL;
  const int max_grid = stream_sms(static_cast<cudaStream_t>(stream)) * 8;
  const int grid = n_roll < max_grid ? n_roll : max_grid;
  record_checks_kernel<<<grid, kRecThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      probs, row_off, n_roll, prompt_len, ends_with_eos, *thresholds_host, commit_accept, commit_checked,
      verdict_out, frac_out, p_last_out);
  return launch_status();
}

int tl_partition_create(int32_t commit_sms, void** streams_out, int32_t* sms_out) {
  if (commit_sms < 1 || !streams_out) return TL_EINVAL;
  const DriverFns& d = driver();
  if (!d.ok) return TL_EUNSUPPORTED;
  int dev_ord = 0;
  if (cudaGetDevice(&dev_ord) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return TL_ECUDA;  // primary ctx up
  CUdevice dev;
  CUdevResource all, part, rest;
  unsigned int groups = 1;
  CUdevResourceDesc d_part, d_rest;
  CUgreenCtx g_part = nullptr, g_rest = nullptr;
  CUstream s[3] = {nullptr, nullptr, nullptr};
  if (d.device_get(&dev, dev_ord) != CUDA_SUCCESS || d.device_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return TL_EUNSUPPORTED;
  if ((unsigned)commit_sms >= all.sm.smCount) return TL_EINVAL;
  if (d.split_by_count(&part, &groups, &all, &rest, 0, (unsigned)commit_sms) != CUDA_SUCCESS || groups != 1 ||
      rest.sm.smCount == 0)
    return TL_EUNSUPPORTED;
  if (d.generate_desc(&d_part, &part, 1) != CUDA_SUCCESS || d.generate_desc(&d_rest, &rest, 1) != CUDA_SUCCESS)
    return TL_ECUDA;
  if (d.green_create(&g_part, d_part, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return TL_ECUDA;
  if (d.green_create(&g_rest, d_rest, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    d.green_destroy(g_part);
    return TL_ECUDA;
  }
  if (d.green_stream_create(&s[0], g_rest, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      d.green_stream_create(&s[1], g_rest, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      d.green_stream_create(&s[2], g_part, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
    for (CUstream x : s)
      if (x) d.stream_destroy(x);
    d.green_destroy(g_part);
    d.green_destroy(g_rest);
    return TL_ECUDA;
  }
  for (int q = 0; q < 3; ++q) streams_out[q] = s[q];
  if (sms_out) {
    sms_out[0] = (int32_t)rest.sm.smCount;
    sms_out[1] = (int32_t)part.sm.smCount;
  }
  return TL_OK;
}

int tl_partition_destroy(void** streams) {
  const DriverFns& d = driver();
  if (!d.ok) return TL_EUNSUPPORTED;
  if (!streams) return TL_EINVAL;
  CUgreenCtx ctx[3] = {nullptr, nullptr, nullptr};
  for (int q = 0; q < 3; ++q) {
    if (!streams[q]) continue;
    cudaStream_t st = static_cast<cudaStream_t>(streams[q]);
    ctx[q] = stream_green_ctx(st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return TL_ECUDA;
    if (d.stream_destroy(reinterpret_cast<CUstream>(st)) != CUDA_SUCCESS) return TL_ECUDA;
  }
  for (int q = 0; q < 3; ++q) {  // the two streaming streams share one context
    bool seen = false;
    for (int r = 0; r < q; ++r) seen = seen || ctx[r] == ctx[q];
    if (ctx[q] && !seen && d.green_destroy(ctx[q]) != CUDA_SUCCESS) return TL_ECUDA;
  }
  return TL_OK;
}

int32_t tl_stream_sms(void* stream) { return stream_sms(static_cast<cudaStream_t>(stream)); }

int tl_prepare(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TL_ECUDA;
  if ((g_tables_prepared.load(std::memory_order_acquire) >> (dev & 31)) & 1u) return TL_OK;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return TL_ECUDA;
  inv_table_kernel<<<dim3(kInvTableBlocks, kInvTables), kInvTableThreads, 0, st>>>(nullptr);
  const bool ok = cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(st) == cudaSuccess;
  cudaStreamDestroy(st);
  if (!ok) return TL_ECUDA;
  g_tables_prepared.fetch_or(1u << (dev & 31), std::memory_order_acq_rel);
  return TL_OK;
}

#if TL_COMMIT_PROF
int tl_commit_prof(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_cprof, sizeof(g_cprof)) != cudaSuccess) return TL_ECUDA;
  if (reset) {
    static const unsigned long long z[8] = {};
    if (cudaMemcpyToSymbol(g_cprof, z, sizeof(z)) != cudaSuccess) return TL_ECUDA;
  }
  return TL_OK;
}
#endif
#if TL_RING_STATS
int tl_ring_lab_timeline(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_ring_tl, sizeof(g_ring_tl)) != cudaSuccess) return TL_ECUDA;
  if (reset) {
    unsigned z = 0;
    if (cudaMemcpyToSymbol(g_ring_tl_n, &z, 4) != cudaSuccess) return TL_ECUDA;
  }
  return TL_OK;
}
int tl_ring_lab_vt(unsigned long long* out) {
  static const unsigned long long z[8] = {};
  if (cudaMemcpyFromSymbol(out, g_vt, sizeof(g_vt)) != cudaSuccess) return TL_ECUDA;
  return cudaMemcpyToSymbol(g_vt, z, sizeof(z)) == cudaSuccess ? TL_OK : TL_ECUDA;
}
int tl_ring_lab_trace(unsigned* out) {
  unsigned z = 0;
  if (cudaMemcpyFromSymbol(out, g_ring_trace, sizeof(g_ring_trace)) != cudaSuccess) return TL_ECUDA;
  return cudaMemcpyToSymbol(g_ring_trace_n, &z, 4) == cudaSuccess ? TL_OK : TL_ECUDA;
}
int tl_ring_lab_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_ring_stats, sizeof(g_ring_stats)) != cudaSuccess) return TL_ECUDA;
  if (reset) {
    static const unsigned long long z[8] = {};
    if (cudaMemcpyToSymbol(g_ring_stats, z, sizeof(z)) != cudaSuccess) return TL_ECUDA;
  }
  return TL_OK;
}
#endif

int32_t tl_ring_grid(const uint16_t* hidden, int32_t H, int64_t n_chunks, int32_t ctas_per_sm, int32_t verify,
                     void* stream) {
  if (H < 1 || n_chunks < 0) return TL_EINVAL;
  return ring_grid(hidden, H, n_chunks, ctas_per_sm, static_cast<cudaStream_t>(stream), verify != 0);
}

int tl_exact_chains(const void* hidden, int32_t dtype, const int64_t* row_off, int32_t n_roll, int32_t H, int32_t k,
                    const int64_t* digest_off, uint8_t* digests_out, void* stream) {
  if (n_roll < 0 || H < 0 || k < 1 || dtype < 0 || dtype > 3) return TL_EINVAL;  // H = 0: empty rows
  if (n_roll == 0) return TL_OK;
  if (!hidden || !row_off || !digest_off || !digests_out) return TL_EINVAL;
  const dim3 grid((n_roll + 31) / 32), block(64);  // 32 rollouts per CTA: a producer and a SHA warp
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (dtype) {
    case 0: exact_chain_kernel<0><<<grid, block, 0, st>>>(hidden, row_off, n_roll, H, k, digest_off, digests_out); break;
    case 1: exact_chain_kernel<1><<<grid, block, 0, st>>>(hidden, row_off, n_roll, H, k, digest_off, digests_out); break;
    case 2: exact_chain_kernel<2><<<grid, block, 0, st>>>(hidden, row_off, n_roll, H, k, digest_off, digests_out); break;
    default: exact_chain_kernel<3><<<grid, block, 0, st>>>(hidden, row_off, n_roll, H, k, digest_off, digests_out); break;
  }
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
