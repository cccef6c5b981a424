// kernels_topk.cu — top-k sparsification with error feedback (§2.2 P:216-224,
// Algorithm 1).
//
// Global top-k: ONE persistent cooperative kernel, one CTA of 16 warps per SM.
// Every warp owns a contiguous run of 256-element chunks and streams it
// through its own 4-stage TMA ring (cp.async.bulk global -> shared, mbarrier
// completion), so HBM reads are in flight continuously and no block barrier
// sits in the streaming loop.
//
//   S  sample : every CTA reads the SAME 4096 values (1024 float4 granules,
//               one in the last chunk of every W/1024-th warp) and derives the
//               same candidate threshold tau and histogram range [tau, split)
//               -- no grid barrier.  (EF: a warp overwrites its last chunk only
//               after every CTA has sampled: a counter, checked once per warp.)
//   F  filter : (EF) acc = fmaf(alpha, g, eps), eps <- acc (st.global.v4);
//               |acc| >= tau -> appended to the warp's candidate list in index
//               order (shared memory, spilling to its global region) and
//               binned into a 4096-bin shared histogram -> flushed to global.
//   -- grid barrier A --
//   R  every CTA reads the global histogram and finds the bin holding the
//               k-th magnitude.  Width 1: exact.  At most 4096 candidates in
//               it: LIST.  Otherwise refine (histogram those candidates, grid
//               barrier, again).  Fewer than k candidates in all (the sample
//               over-estimated tau): exact re-filter with tau = 0.
//   L  each CTA publishes (#candidates above the bin, #in it) and appends the
//               bin's candidates to a global list.
//   -- grid barrier B --
//   P  every CTA resolves the exact k-th magnitude and the number of its ties
//               to take (lower index first, R-18) from the list, its own
//               output offset from the per-CTA counts, then writes its
//               selected pairs in index order and zeroes them in the residual.
// Two grid barriers in the common case; all histogram slots are cleared after
// barrier B (so a workspace can be reused at any N <= its size).
#include <algorithm>
#include <cmath>

#include "kernels.h"

namespace sparcml {

constexpr int kTkWarps = 16;
constexpr int kTkThreads = kTkWarps * 32;
constexpr int kChunk = 256;                   // elements per pipeline chunk (1 KB per array)
#ifndef SPARCML_TOPK_RING_KB
#define SPARCML_TOPK_RING_KB 8               // TMA ring bytes per warp (x, or eps and grad)
#endif
#ifndef SPARCML_TOPK_LATE_PRO
#define SPARCML_TOPK_LATE_PRO 0              // 1: issue the TMA prologue after the sample (A/B diagnostics)
#endif
#ifndef SPARCML_TOPK_EPS_EF
#define SPARCML_TOPK_EPS_EF 0                // 1: eps / residual stores with an L2 evict-first hint (A/B)
#endif
#ifndef SPARCML_TOPK_FENCE
#define SPARCML_TOPK_FENCE 0                 // 1: proxy fence before every ring refill (A/B diagnostics)
#endif
#ifndef SPARCML_TOPK_ROLES
#define SPARCML_TOPK_ROLES 1                 // 1: warps 0-7 issue the sample loads first, warps 8-15 set up the rings
#endif
#ifndef SPARCML_TOPK_BITSEL
#define SPARCML_TOPK_BITSEL 0                // 1: sample quantiles by a bitwise block search (no sample histogram)
#endif
#ifndef SPARCML_TOPK_WARM
#define SPARCML_TOPK_WARM 1                  // 1: tau / split from the previous call's k-th magnitude (no sample)
#endif
#ifndef SPARCML_TOPK_WARM_LO
#define SPARCML_TOPK_WARM_LO 64                // warm tau = m (1 - 1/LO)  (128: -1-2 us in a seed-cycling loop, but low-side misses when one gradient repeats: bench top-k 55 us)
#endif
#ifndef SPARCML_TOPK_WARM_HI
#define SPARCML_TOPK_WARM_HI 8                 // warm split = m (1 + 1/HI)
#endif
#ifndef SPARCML_TOPK_COOP
#define SPARCML_TOPK_COOP 1                  // 0: plain launch (one CTA per SM fits; A/B diagnostics)
#endif
constexpr int kBins = 4096;                   // bins per histogram level (last one: overflow [split, hi))
constexpr int kLevels = 6;                    // histogram slots per call (filter, re-filter, refinements)
constexpr int kListCap = 4096;                // crossing-bin candidates resolved in shared memory
constexpr int kSampleGran = 1024;             // sampled float4 granules (4096 values)
constexpr uint64_t kSampleMinN = 1u << 16;    // below this: tau = 0 (every value is a candidate)
constexpr int kMaxGrid = 1024;
constexpr uint64_t kKeyEnd = 0x80000000ull;   // one past the largest |x| key (NaN included)

template <bool EF>
struct TkCfg {
  static constexpr int kArr = EF ? 2 : 1;               // eps and grad, or x
  static constexpr int kStages = SPARCML_TOPK_RING_KB * 1024 / (kArr * kChunk * 4);   // chunks in flight per warp
  static constexpr int kCap = 512;                      // candidates per warp kept in shared memory
  static constexpr size_t kRing = (size_t)kTkWarps * kStages * kArr * kChunk * 4;
  static constexpr size_t kBar = (size_t)kTkWarps * kStages * 8;
  static constexpr size_t kSmem = kRing + kBar + (size_t)kBins * 4 + (size_t)kTkWarps * kCap * 8;
  static_assert(kRing >= (size_t)kListCap * 8 + 2 * kMaxGrid * 4, "list staging reuses the ring");
};

struct TopkCtl {
  uint32_t arrive;          // arrivals at the current grid barrier (reset by the last arriver)
  uint32_t flag;            // grid barriers released so far (wrapping)
  uint32_t calls;           // completed calls; parity p = calls & 1 selects the per-call slots below
  uint32_t status, passes;  // last call: non-finite input seen, filter passes (1; +1 per re-filter)
  uint32_t bad[2];          // per call parity: a non-finite value was seen
  uint32_t sampled[2];      // per call parity: CTAs done sampling (EF write guard)
  uint32_t list_n[2];       // per call parity: length of the crossing-bin list
  uint32_t nofast[2];       // per call parity: some CTA could not sort its candidates (slow path)
  uint32_t pad[1];
  uint64_t t_phase[16];     // %globaltimer phase ends (SPARCML_DEBUG_MARKS); [15] = bucketed status
  uint64_t dbg[32];         // CTA 0's fine-grained %globaltimer marks (SPARCML_DEBUG_MARKS)
  alignas(16) uint32_t hist[2][kLevels][kBins];   // [call parity][slot]; 16-byte aligned (uint4 reads)
  uint32_t cta_a[kMaxGrid];  // per CTA: candidates with key >= hi of the final range
  uint32_t cta_e[kMaxGrid];  // per CTA: candidates in [lo, hi) of the final range
  uint64_t t_cta[2][kMaxGrid];   // per CTA: %globaltimer at start and filter end (SPARCML_DEBUG_MARKS)
  uint32_t warm_kth;        // last call's k-th magnitude key (0: none, or that call missed; sample instead)
  uint32_t warm_ef;         // ... of an EF call (1) or a plain sparsify (0)
  uint64_t warm_N, warm_k;  // ... for this (N, k)
};

struct TopkLayout {
  TopkCtl* ctl;
  uint4* list;              // (index, key, cta, 0) of the crossing bin's candidates
  uint32_t* sp_idx;         // per-warp candidate spill regions (the warp's element range)
  float* sp_val;
};

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static TopkLayout topk_layout(void* ws, uint64_t N) {
  TopkLayout L;
  char* p = static_cast<char*>(ws);
  L.ctl = reinterpret_cast<TopkCtl*>(p);
  p += align256(sizeof(TopkCtl));
  L.list = reinterpret_cast<uint4*>(p);
  p += align256((size_t)kListCap * sizeof(uint4));
  L.sp_idx = reinterpret_cast<uint32_t*>(p);
  p += align256(N * sizeof(uint32_t));
  L.sp_val = reinterpret_cast<float*>(p);
  return L;
}

size_t topk_workspace_bytes(uint64_t N, uint64_t /*k*/) {
  return align256(sizeof(TopkCtl)) + align256((size_t)kListCap * sizeof(uint4)) + 2 * align256(N * sizeof(uint32_t));
}

__device__ __forceinline__ uint32_t abs_key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

__host__ __device__ __forceinline__ uint32_t shift_for(uint64_t span, uint64_t nbins) {
  uint32_t s = 0;
  while ((nbins << s) < span) ++s;
  return s;
}

// bins 0..kBins-2 cover [lo, split) in steps of 2^shift; kBins-1 holds keys >= split
__device__ __forceinline__ uint32_t bin_of(uint32_t key, uint32_t lo, uint64_t split, uint32_t shift) {
  if ((uint64_t)key >= split) return kBins - 1;
  const uint32_t b = (key - lo) >> shift;
  return b < (uint32_t)(kBins - 1) ? b : (uint32_t)(kBins - 2);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- TMA bulk copies and mbarriers (PTX) ---------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TK_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TK_DONE;\n\t"
      "bra TK_WAIT;\n"
      "TK_DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ float4 lds_f4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// ---- diagnostics (compiled in only with -DSPARCML_DEBUG_MARKS) -------------------
__device__ __forceinline__ void tk_mark(TopkCtl* c, int i) {
  // [0] CTA 0's start, [1..7] the latest CTA's end of phase i, [8] the latest
  // CTA's start, [9..14] CTA 0's end of phases 1..6
#ifdef SPARCML_DEBUG_MARKS
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (i == 0) {
      if (blockIdx.x == 0) c->t_phase[0] = t;
      atomicMax(reinterpret_cast<unsigned long long*>(&c->t_phase[8]), (unsigned long long)t);
    } else {
      atomicMax(reinterpret_cast<unsigned long long*>(&c->t_phase[i]), (unsigned long long)t);
      if (blockIdx.x == 0 && i <= 6) c->t_phase[8 + i] = t;
    }
  }
#else
  (void)c;
  (void)i;
#endif
}

#ifdef SPARCML_DEBUG_MARKS
#define TK_D(i)                                                        \
  do {                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                         \
      uint64_t t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));           \
      c->dbg[i] = t_;                                                  \
    }                                                                  \
  } while (0)
#define TK_C(j)                                                        \
  do {                                                                 \
    if (threadIdx.x == 0) {                                            \
      uint64_t t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));           \
      c->t_cta[j][blockIdx.x] = t_;                                    \
    }                                                                  \
  } while (0)
#define TK_V(i, v)                                                     \
  do {                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) c->dbg[i] = (uint64_t)(v); \
  } while (0)
#else
#define TK_D(i) \
  do {          \
  } while (0)
#define TK_V(i, v) \
  do {             \
  } while (0)
#define TK_C(j) \
  do {          \
  } while (0)
#endif

// ---- block primitives (kTkThreads) ------------------------------------------------
template <typename T>
__device__ __forceinline__ T blk_excl_sum(T x, T* sc, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_inclusive_sum(x);
  if (lane == 31) sc[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const T w = lane < kTkWarps ? sc[lane] : T(0);
    const T wi = warp_inclusive_sum(w);
    if (lane < kTkWarps) sc[lane] = wi - w;
    if (lane == kTkWarps - 1) sc[kTkWarps] = wi;
  }
  __syncthreads();
  const T r = sc[warp] + inc - x;
  *total = sc[kTkWarps];
  __syncthreads();
  return r;
}

// two exclusive block sums with one set of barriers
__device__ __forceinline__ void blk_excl_sum2(uint64_t x, uint64_t y, uint64_t* sc /*2*(kTkWarps+1)*/, uint64_t* ex,
                                              uint64_t* ey) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ix = warp_inclusive_sum(x), iy = warp_inclusive_sum(y);
  if (lane == 31) {
    sc[warp] = ix;
    sc[kTkWarps + 1 + warp] = iy;
  }
  __syncthreads();
  if (warp == 0) {
    const uint64_t wx = lane < kTkWarps ? sc[lane] : 0, wy = lane < kTkWarps ? sc[kTkWarps + 1 + lane] : 0;
    const uint64_t jx = warp_inclusive_sum(wx), jy = warp_inclusive_sum(wy);
    if (lane < kTkWarps) {
      sc[lane] = jx - wx;
      sc[kTkWarps + 1 + lane] = jy - wy;
    }
  }
  __syncthreads();
  *ex = sc[warp] + ix - x;
  *ey = sc[kTkWarps + 1 + warp] + iy - y;
  __syncthreads();
}

struct Cross {
  uint32_t bin;    // crossing bin
  uint32_t cnt;    // its count
  uint64_t above;  // count in the bins above it (or the histogram total if !ok)
  int ok;          // the histogram reaches the target
};

// Whole block, shared histogram h[NB] (NB = 512 * per): for each target t, the
// highest bin b with sum_{bins > b} < t <= sum_{bins >= b}.  Thread i scans bins
// NB-1-per*i down to NB-per*(i+1).  Results in s_out[0..1].
template <int NB>
__device__ __forceinline__ void find2(const uint32_t* h, uint64_t t0, uint64_t t1, uint64_t* sc, Cross* s_out) {
  constexpr int per = NB / kTkThreads;
  static_assert(per % 4 == 0, "uint4 reads");
  const int tid = threadIdx.x;
  const int base = NB - per * (tid + 1);
  uint32_t v[per];   // v[i] = bin base+i
#pragma unroll
  for (int q = 0; q < per; q += 4) {
    const uint4 u = *reinterpret_cast<const uint4*>(h + base + q);
    v[q] = u.x;
    v[q + 1] = u.y;
    v[q + 2] = u.z;
    v[q + 3] = u.w;
  }
  uint64_t loc = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) loc += v[i];
  uint64_t tot;
  const uint64_t ex = blk_excl_sum<uint64_t>(loc, sc, &tot);
  const uint64_t tg[2] = {t0, t1};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (tid == 0 && tot < tg[q]) s_out[q] = Cross{0u, 0u, tot, 0};
    if (ex < tg[q] && ex + loc >= tg[q]) {
      uint64_t cum = ex;
#pragma unroll
      for (int i = per - 1; i >= 0; --i) {
        if (cum < tg[q] && cum + v[i] >= tg[q]) s_out[q] = Cross{(uint32_t)(base + i), v[i], cum, 1};
        cum += v[i];
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ Cross find_desc(const uint32_t* h, uint64_t t, uint64_t* sc, Cross* s_out) {
  find2<kBins>(h, t, t, sc, s_out);
  const Cross r = s_out[0];
  __syncthreads();
  return r;
}

// Grid barrier of a cooperative launch: arrivals on a counter (the last
// arriver resets it) and a wrapping release flag; `target` = the flag value
// that releases this barrier.
#ifndef SPARCML_TOPK_BAR_ACQREL
#define SPARCML_TOPK_BAR_ACQREL 1   // 1: acq_rel fences (0: membar.gl, i.e. fence.sc, A/B diagnostics)
#endif
__device__ __forceinline__ void tk_grid_barrier(TopkCtl* c, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (SPARCML_TOPK_BAR_ACQREL) fence_acq_rel_gpu();   // release: this CTA's writes (cumulative over the bar.sync)
    else __threadfence();
    const uint32_t old = atomicAdd(&c->arrive, 1u);
    if (old == gridDim.x - 1) {
      atomicExch(&c->arrive, 0u);
      if (SPARCML_TOPK_BAR_ACQREL) fence_acq_rel_gpu();   // acquire the other CTAs' arrivals, release to the waiters
      else __threadfence();
      st_release_gpu(&c->flag, target);
    } else {
      while ((int)(ld_relaxed_gpu_u32(&c->flag) - target) < 0) {
      }
      (void)ld_acquire_gpu(&c->flag);
    }
    if (!SPARCML_TOPK_BAR_ACQREL) __threadfence();
  }
  __syncthreads();
}

// Chunk split: C chunks over W warps, warp w owns [wstart(w), wstart(w) + wcount(w))
// (32-bit: C < 2^24 for N < 2^32, W <= 16384).
struct WSplit {
  uint32_t base, rem;
};
__host__ __device__ __forceinline__ uint32_t wstart(const WSplit& s, uint32_t w) {
  return w * s.base + (w < s.rem ? w : s.rem);
}
__host__ __device__ __forceinline__ uint32_t wcount(const WSplit& s, uint32_t w) { return s.base + (w < s.rem ? 1u : 0u); }

// The float4 granule of sample q: in the last chunk of warp q*W/1024 (so EF can
// guard its overwrite with one check per warp).  False if the granule does not
// exist (the ragged final chunk of the vector holding < 4 values).
__host__ __device__ __forceinline__ bool sample_pos(uint32_t q, uint64_t N, uint32_t C, uint32_t W, const WSplit& sp,
                                                    uint64_t* pos) {
  const uint32_t wq = (q * W) / kSampleGran;
  const uint32_t cl = wstart(sp, wq) + wcount(sp, wq) - 1;
  uint32_t gr = (q * 17u) & 63u;
  if (cl + 1 == C) {
    const uint32_t nval = (uint32_t)((N - (uint64_t)cl * kChunk < (uint64_t)kChunk ? N - (uint64_t)cl * kChunk
                                                                                    : (uint64_t)kChunk) / 4);
    if (nval == 0) return false;
    gr %= nval;
  }
  *pos = (uint64_t)cl * kChunk + gr * 4;
  return true;
}

struct TkArgs {
  const float* x;   // EF: eps (read, then overwritten by acc through dst); else the input
  const float* g;   // EF: the gradient
  float alpha;
  float* dst;       // STORE: EF -> eps (== x), sparsify -> residual (!= x)
  float* zero_at;   // selected coordinates zeroed here (EF: eps; residual; x in place; or null)
  uint64_t N, k;
  uint32_t* idx_out;
  float* val_out;
  TopkLayout L;
};

// Per-warp candidate storage: the first kCap in shared memory, the rest in the
// warp's global spill region (its element range, so it never overflows).
template <bool EF>
struct CandStore {
  uint32_t* si;
  float* sv;
  uint32_t* gi;
  float* gv;
  uint32_t range;   // the warp's element count: the spill region's capacity
  __device__ __forceinline__ void put(uint32_t pos, uint32_t idx, float v) const {
    SPARCML_CHECK(pos < (uint32_t)TkCfg<EF>::kCap + range);
    if (pos < (uint32_t)TkCfg<EF>::kCap) {
      si[pos] = idx;
      sv[pos] = v;
    } else {
      gi[pos - TkCfg<EF>::kCap] = idx;
      gv[pos - TkCfg<EF>::kCap] = v;
    }
  }
  __device__ __forceinline__ void get(uint32_t pos, uint32_t* idx, float* v) const {
    if (pos < (uint32_t)TkCfg<EF>::kCap) {
      *idx = si[pos];
      *v = sv[pos];
    } else {
      *idx = gi[pos - TkCfg<EF>::kCap];
      *v = gv[pos - TkCfg<EF>::kCap];
    }
  }
};

// One 128-element row of a chunk (4 consecutive values per lane): optional
// store, non-finite check, in-order compaction of |v| >= tau, histogram.
template <bool EF, bool STORE>
__device__ __forceinline__ void consume_row(const float v[4], uint64_t gp, bool full, uint64_t N, float* dst,
                                            uint32_t tau, uint64_t split, uint32_t shift, uint32_t* sh,
                                            const CandStore<EF>& cs, uint32_t& nw, uint32_t& bad) {
  if (STORE) {
    if (full) {
      *reinterpret_cast<float4*>(dst + gp) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (gp + j < N) dst[gp + j] = v[j];
    }
  }
  uint32_t fl = 0;
  uint32_t key[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    key[j] = abs_key(v[j]);
    const bool valid = full || gp + j < N;
    if (valid) {
      bad |= key[j] >= 0x7F800000u ? 1u : 0u;
      if (key[j] >= tau) fl |= 1u << j;
    }
  }
  const uint32_t lt = lanemask_lt();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t bj = __ballot_sync(0xffffffffu, (fl >> j) & 1u);
    before += __popc(bj & lt);
    tot += __popc(bj);
  }
  if (fl) {
    uint32_t pos = nw + before;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((fl >> j) & 1u) {
        cs.put(pos, (uint32_t)(gp + j), v[j]);
        atomicAdd(&sh[bin_of(key[j], tau, split, shift)], 1u);
        ++pos;
      }
  }
  nw += tot;
}

// bins for the hot loop (32-bit: split <= 2^31)
__device__ __forceinline__ uint32_t bin_of32(uint32_t key, uint32_t lo, uint32_t split, uint32_t shift) {
  if (key >= split) return kBins - 1;
  return min((key - lo) >> shift, (uint32_t)(kBins - 2));
}

// One full chunk from the TMA ring (the hot loop, kept short: it is issue-bound
// otherwise).  Lane l holds elements 4l..4l+3 (row 0) and 128+4l..128+4l+3
// (row 1).  Candidates (|v| >= tau, or unordered: NaN) are rare; their
// in-order positions come from one packed warp scan of the per-row counts,
// and each lane walks only its own set bits, re-reading the value from the
// stage (EF: recomputing the same fma) instead of indexing registers.
template <bool EF, bool STORE>
__device__ __forceinline__ void hot_chunk(const float* sx, uint32_t e0, float alpha, float* dst, float tauf,
                                          uint32_t lo, uint32_t split, uint32_t shift, uint32_t* sh,
                                          const CandStore<EF>& cs, uint32_t& nw, uint32_t& bad) {
  const int lane = threadIdx.x & 31;
  float4 r0 = lds_f4(sx + lane * 4), r1 = lds_f4(sx + 128 + lane * 4);
  if (EF) {
    const float4 g0 = lds_f4(sx + kChunk + lane * 4), g1 = lds_f4(sx + kChunk + 128 + lane * 4);
    r0 = make_float4(__fmaf_rn(alpha, g0.x, r0.x), __fmaf_rn(alpha, g0.y, r0.y), __fmaf_rn(alpha, g0.z, r0.z),
                     __fmaf_rn(alpha, g0.w, r0.w));
    r1 = make_float4(__fmaf_rn(alpha, g1.x, r1.x), __fmaf_rn(alpha, g1.y, r1.y), __fmaf_rn(alpha, g1.z, r1.z),
                     __fmaf_rn(alpha, g1.w, r1.w));
  }
  if (STORE) {
    if (SPARCML_TOPK_EPS_EF) {
      const uint64_t pol = l2_evict_first_policy();
      st_stream_f4_ef(reinterpret_cast<float4*>(dst + e0 + lane * 4), r0, pol);
      st_stream_f4_ef(reinterpret_cast<float4*>(dst + e0 + 128 + lane * 4), r1, pol);
    } else {
      *reinterpret_cast<float4*>(dst + e0 + lane * 4) = r0;
      *reinterpret_cast<float4*>(dst + e0 + 128 + lane * 4) = r1;
    }
  }
  uint32_t m = 0;
  m |= !(fabsf(r0.x) < tauf) ? 0x01u : 0u;
  m |= !(fabsf(r0.y) < tauf) ? 0x02u : 0u;
  m |= !(fabsf(r0.z) < tauf) ? 0x04u : 0u;
  m |= !(fabsf(r0.w) < tauf) ? 0x08u : 0u;
  m |= !(fabsf(r1.x) < tauf) ? 0x10u : 0u;
  m |= !(fabsf(r1.y) < tauf) ? 0x20u : 0u;
  m |= !(fabsf(r1.z) < tauf) ? 0x40u : 0u;
  m |= !(fabsf(r1.w) < tauf) ? 0x80u : 0u;
  if (!__any_sync(0xffffffffu, m)) return;
  const uint32_t pk = (uint32_t)__popc(m & 0xFu) | ((uint32_t)__popc(m >> 4) << 16);
  const uint32_t inc = warp_inclusive_sum<uint32_t>(pk);
  const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
  const uint32_t ex = inc - pk;
  uint32_t pos0 = nw + (ex & 0xFFFFu), pos1 = nw + (tot & 0xFFFFu) + (ex >> 16);
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    const uint32_t el = (j < 4 ? 0u : 124u) + lane * 4 + j;   // j >= 4: 128 + 4l + (j - 4)
    const float v = EF ? __fmaf_rn(alpha, sx[kChunk + el], sx[el]) : sx[el];
    const uint32_t pos = j < 4 ? pos0++ : pos1++;
    cs.put(pos, e0 + el, v);
    const uint32_t key = abs_key(v);
    bad |= key >= 0x7F800000u ? 1u : 0u;
    atomicAdd(&sh[bin_of32(key, lo, split, shift)], 1u);
  }
  nw += (tot & 0xFFFFu) + (tot >> 16);
}

template <bool EF, bool STORE>
__global__ void __launch_bounds__(kTkThreads, 1) topk_stream_kernel(TkArgs a) {
  using Cfg = TkCfg<EF>;
  constexpr int kCap = Cfg::kCap;
  constexpr int kStages = Cfg::kStages;
  extern __shared__ __align__(128) unsigned char tk_smem[];
  float* ring = reinterpret_cast<float*>(tk_smem);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tk_smem + Cfg::kRing);
  uint32_t* sh = reinterpret_cast<uint32_t*>(tk_smem + Cfg::kRing + Cfg::kBar);
  uint32_t* cidx = sh + kBins;
  float* cval = reinterpret_cast<float*>(cidx + kTkWarps * kCap);
  __shared__ uint64_t s_sc[2 * (kTkWarps + 1)];
  __shared__ Cross s_cross[2];
  __shared__ uint32_t s_w[kTkWarps][2];
  __shared__ uint32_t s_wn[kTkWarps];
  __shared__ uint32_t s_bad, s_spill, s_nofast, s_lbase, s_quota;
  __shared__ uint64_t s_off;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  TopkCtl* c = a.L.ctl;
  const uint64_t N = a.N, k = a.k;
  const uint32_t C = (uint32_t)((N + kChunk - 1) / kChunk);
  const uint32_t W = G * kTkWarps, gw = b * kTkWarps + warp;
  const WSplit sp{C / W, C % W};
  const uint32_t c0 = wstart(sp, gw), nch = wcount(sp, gw);
  const uint64_t wbase = (uint64_t)c0 * kChunk;
  const uint32_t p = ld_relaxed_gpu_u32(&c->calls) & 1u;
  uint32_t bar_t = ld_relaxed_gpu_u32(&c->flag);
  const CandStore<EF> cs{cidx + warp * kCap, cval + warp * kCap, a.L.sp_idx + wbase, a.L.sp_val + wbase,
                         (uint32_t)(std::min<uint64_t>(N, (uint64_t)(c0 + nch) * kChunk) - wbase)};
  tk_mark(c, 0);
  TK_C(0);

  // ---- ring set-up, prologue and the shared sample ---------------------------------
  // ROLES: warps [0, 8) issue the sample's loads at once (ahead of the ring's bulk
  // copies in the memory queues: the threshold is what every warp waits for),
  // while lanes 0-1 of warps [8, 16) each set up one warp's ring (mbarrier init,
  // fences, the first kStages chunks).  A fence only orders its own thread's
  // accesses, so the ring warps' fences do not wait for the sample's loads.
  // Otherwise every warp's lane 0 sets up its own ring before the sample.
  uint64_t* wbar = mbar + warp * kStages;
  float* wring = ring + (size_t)warp * kStages * Cfg::kArr * kChunk;
  const uint64_t pol = l2_evict_first_policy();
  auto issue_w = [&](uint32_t w, uint32_t cc, int s) {
    if ((uint64_t)(cc + 1) * kChunk > N) return;   // the ragged final chunk is read directly
    float* d = ring + ((size_t)w * kStages + s) * Cfg::kArr * kChunk;
    uint64_t* bar = mbar + w * kStages + s;
    mbar_expect_tx(bar, Cfg::kArr * kChunk * 4);
    bulk_g2s(d, a.x + (uint64_t)cc * kChunk, kChunk * 4, bar, pol);
    if (EF) bulk_g2s(d + kChunk, a.g + (uint64_t)cc * kChunk, kChunk * 4, bar, pol);
  };
  auto setup_ring = [&](uint32_t w) {   // one thread: warp w's mbarriers and prologue
    for (int s = 0; s < kStages; ++s) mbar_init(mbar + w * kStages + s, 1);
    fence_mbar_init();
    fence_proxy_async_smem();
    if (!SPARCML_TOPK_LATE_PRO) {
      const uint32_t gw_ = b * kTkWarps + w;
      const uint32_t c0_ = wstart(sp, gw_), n_ = wcount(sp, gw_);
      for (int s = 0; s < kStages && (uint32_t)s < n_; ++s) issue_w(w, c0_ + s, s);
    }
  };
  auto issue = [&](uint32_t cc, int s) { issue_w((uint32_t)warp, cc, s); };
  // Warm start: a previous call on this workspace with the same (N, k) found the
  // k-th magnitude m without a miss; take tau = m (1 - 1/64), split = m (1 + 1/8)
  // and skip the sample.  Under error feedback m drifts by < 1% per step once the
  // accumulator's distribution settles; a miss is still exact
  // (m < tau: the tau = 0 re-filter; m >= split: the overflow bin's refinement)
  // and makes the next call sample again.
  const uint32_t wk = SPARCML_TOPK_WARM ? c->warm_kth : 0u;
  const bool warm = SPARCML_TOPK_WARM && N >= kSampleMinN && wk > 0u && wk < 0x7F800000u && c->warm_N == N &&
                    c->warm_k == k && c->warm_ef == (EF ? 1u : 0u);
  const bool sampling = N >= kSampleMinN && !warm;
  constexpr int kSThreads = SPARCML_TOPK_ROLES ? kTkThreads / 2 : kTkThreads;   // sampling threads
  constexpr int kSPer = kSampleGran / kSThreads;                                  // granules per sampling thread
  float4 smp[kSPer], smg[kSPer];
  bool sok[kSPer];
#pragma unroll
  for (int j = 0; j < kSPer; ++j) {   // threads without samples (the ring warps) hold none
    sok[j] = false;
    smp[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    smg[j] = smp[j];
  }
  auto sample_loads = [&]() {
#pragma unroll
    for (int j = 0; j < kSPer; ++j) {
      uint64_t pos = 0;
      sok[j] = sampling && tid < kSThreads && sample_pos((uint32_t)(tid + j * kSThreads), N, C, W, sp, &pos);
      smp[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      smg[j] = smp[j];
      if (sok[j]) {
        smp[j] = __ldcg(reinterpret_cast<const float4*>(a.x + pos));
        if (EF) smg[j] = __ldcg(reinterpret_cast<const float4*>(a.g + pos));
      }
    }
  };
  if (SPARCML_TOPK_ROLES && sampling) {
    static_assert(kTkWarps == 16, "two ring warps per set-up warp");
    if (warp < kTkWarps / 2) {
      sample_loads();
    } else if (lane < 2) {
      setup_ring((uint32_t)(2 * (warp - kTkWarps / 2) + lane));
    }
    __syncwarp();
    TK_D(18);
  } else {
    if (lane == 0) setup_ring((uint32_t)warp);
    __syncwarp();
    TK_D(18);
  }

  constexpr int kSBins = 8192;    // sample histogram: key >> 18 (1/32 octave), in the candidate area
  static_assert(kSBins * 4 <= kTkWarps * kCap * 8, "sample histogram fits the candidate area");
  uint32_t* shs = cidx;
  for (int i = tid; i < kBins; i += kTkThreads) sh[i] = 0;
  if (sampling && !SPARCML_TOPK_BITSEL)
    for (int i = tid; i < kSBins / 4; i += kTkThreads) reinterpret_cast<uint4*>(shs)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) {
    s_bad = 0;
    s_spill = 0;
  }
  __syncthreads();   // (also: every ring's mbarriers are initialised before any warp waits on them)
  TK_D(0);
  if (!SPARCML_TOPK_ROLES) sample_loads();   // behind the rings' prologue in the memory queues

  uint32_t tau = 0;
  uint64_t split = kKeyEnd;
  if (sampling) {
    uint32_t ns = 0;
#pragma unroll
    for (int j = 0; j < kSPer; ++j) {
      if (EF)   // acc = fmaf(alpha, g, eps) at the sampled positions
        smp[j] = make_float4(__fmaf_rn(a.alpha, smg[j].x, smp[j].x), __fmaf_rn(a.alpha, smg[j].y, smp[j].y),
                             __fmaf_rn(a.alpha, smg[j].z, smp[j].z), __fmaf_rn(a.alpha, smg[j].w, smp[j].w));
      ns += sok[j] ? 4u : 0u;
    }
    TK_D(1);
    // tau where the sample count from the top reaches t_lo = mean + 5 sigma + 4
    // (to 1/32 octave): the k-th magnitude is >= tau unless the sample holds >=
    // t_lo values above it (a 5.6-sigma event; then the exact re-filter runs).
    // split where the count reaches mean - 4 sigma - 16: the level-0 bins cover
    // [tau, split) finely.  Same result in every CTA.
    uint64_t S;
    (void)blk_excl_sum<uint64_t>(ns, s_sc, &S);
    TK_D(2);
    const float mean = (float)((double)k * (double)S / (double)N);
    const float sd = sqrtf(mean);
    const uint64_t t_lo = (uint64_t)ceilf(mean + 5.0f * sd + 4.0f);
    const float th = mean - 4.0f * sd - 16.0f;
    const uint64_t t_hi = th > 1.0f ? (uint64_t)th : 1;
    if (SPARCML_TOPK_BITSEL) {
      // the 1/32-octave bin holding the t-th largest sample key, bit by bit from
      // the top (bits 30..18): the largest T = m * 2^18 with #(keys >= T) >= t.
      // Both targets per round, counts packed in 16-bit halves (S <= 4096).
      uint32_t key[4 * kSPer];
#pragma unroll
      for (int j = 0; j < kSPer; ++j) {
        key[4 * j] = sok[j] ? abs_key(smp[j].x) : 0u;
        key[4 * j + 1] = sok[j] ? abs_key(smp[j].y) : 0u;
        key[4 * j + 2] = sok[j] ? abs_key(smp[j].z) : 0u;
        key[4 * j + 3] = sok[j] ? abs_key(smp[j].w) : 0u;
      }
      uint32_t* s_red = reinterpret_cast<uint32_t*>(shs);   // 2 x kTkWarps round counts (candidate area, unused yet)
      uint32_t Tlo = 0, Thi = 0;
#pragma unroll 1
      for (int bit = 30; bit >= 18; --bit) {
        const uint32_t cl = Tlo | (1u << bit), ch = Thi | (1u << bit);
        uint32_t cnt = 0;
        if (tid < kSThreads) {
#pragma unroll
          for (int j = 0; j < 4 * kSPer; ++j) cnt += (key[j] >= cl ? 1u : 0u) + (key[j] >= ch ? 0x10000u : 0u);
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) s_red[(bit & 1) * kTkWarps + warp] = cnt;
        __syncthreads();
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kTkWarps; ++w) tot += s_red[(bit & 1) * kTkWarps + w];
        if ((tot & 0xFFFFu) >= t_lo) Tlo = cl;
        if ((tot >> 16) >= t_hi) Thi = ch;
      }
      tau = S >= t_lo ? Tlo : 0u;
      split = S >= t_hi ? (uint64_t)Thi + (1u << 18) : kKeyEnd;
      __syncthreads();   // s_red (the candidate area) is free again
    } else {
#pragma unroll
      for (int j = 0; j < kSPer; ++j)
        if (sok[j]) {
          atomicAdd(&shs[abs_key(smp[j].x) >> 18], 1u);
          atomicAdd(&shs[abs_key(smp[j].y) >> 18], 1u);
          atomicAdd(&shs[abs_key(smp[j].z) >> 18], 1u);
          atomicAdd(&shs[abs_key(smp[j].w) >> 18], 1u);
        }
      __syncthreads();
      find2<kSBins>(shs, t_lo, t_hi, s_sc, s_cross);
      const Cross f0 = s_cross[0], f1 = s_cross[1];
      tau = f0.ok ? (f0.bin << 18) : 0u;
      split = f1.ok ? (uint64_t)(f1.bin + 1) << 18 : kKeyEnd;
    }
    if (EF && tid == 0) atomicAdd(&c->sampled[p], 1u);   // this CTA's sample reads are complete
    if (split <= tau) split = (uint64_t)tau + 1;
    TK_D(3);
  } else if (warm) {
    const float m = __uint_as_float(wk);
    tau = abs_key(m * (1.0f - 1.0f / (float)SPARCML_TOPK_WARM_LO));
    split = (uint64_t)abs_key(m * (1.0f + 1.0f / (float)SPARCML_TOPK_WARM_HI)) + 1u;   // <= Inf's key + 1 < kKeyEnd
  }
  uint32_t shift = shift_for(split - tau, kBins - 1);
  if (SPARCML_TOPK_LATE_PRO && lane == 0)
    for (int s = 0; s < kStages && (uint32_t)s < nch; ++s) issue(c0 + s, s);
  tk_mark(c, 1);

  // ---- F: the streaming pass ---------------------------------------------------------
  if (tau > 0x7F800000u) tau = 0x7F800000u;   // a sample holding NaN: Inf must stay a candidate
  const float tauf = __uint_as_float(tau);
  const uint32_t split32 = (uint32_t)split;
  uint32_t nw = 0, bad = 0;
  const bool ragged = nch > 0 && (uint64_t)(c0 + nch) * kChunk > N;   // this warp owns the vector's partial last chunk
  const uint32_t nfull = ragged ? nch - 1 : nch;
  auto guard = [&](uint32_t i) {   // EF: the warp's last chunk may hold sampled values
    if (EF && STORE && sampling && i + 1 == nch) {
      if (lane == 0) {
        while ((int)(ld_relaxed_gpu_u32(&c->sampled[p]) - G) < 0) {
        }
        (void)ld_acquire_gpu(&c->sampled[p]);
      }
      __syncwarp();
    }
  };
  for (uint32_t i = 0; i < nfull; ++i) {
    const int s = (int)(i % kStages);
    const float* sx = wring + (size_t)s * Cfg::kArr * kChunk;
    mbar_wait(&wbar[s], (i / kStages) & 1u);
    guard(i);
    hot_chunk<EF, STORE>(sx, (c0 + i) * kChunk, a.alpha, a.dst, tauf, tau, split32, shift, sh, cs, nw, bad);
    __syncwarp();
    if (lane == 0 && i + kStages < nch) {
      // every lane has consumed stage s (its values fed the vote above the
      // __syncwarp), so the async refill cannot overwrite unread data
      if (SPARCML_TOPK_FENCE) fence_proxy_async_smem();
      issue(c0 + i + kStages, s);
    }
  }
  if (ragged) {   // the partial final chunk of the vector, read directly
    const uint64_t cc = c0 + nch - 1;
    guard(nch - 1);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint64_t gp = cc * kChunk + r * 128 + lane * 4;
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[j] = 0.0f;
        if (gp + j < N) v[j] = EF ? __fmaf_rn(a.alpha, a.g[gp + j], a.x[gp + j]) : a.x[gp + j];
      }
      consume_row<EF, STORE>(v, gp, false, N, a.dst, tau, split, shift, sh, cs, nw, bad);
    }
  }
  TK_D(5);
  bad = __any_sync(0xffffffffu, bad) ? 1u : 0u;
  if (lane == 0) {
    s_wn[warp] = nw;
    if (nw > (uint32_t)kCap) s_spill = 1u;
    if (bad) s_bad = 1u;
  }
  __syncthreads();
  TK_D(4);
  TK_C(1);

  // ---- counting sort of this CTA's candidates by bin (fast path) -------------------
  // The CTA's element range [r0, r1) doubles as its sorted region: sp_idx[r0 ..
  // r0+kBins) = per-bin counts ABOVE the bin (descending exclusive scan),
  // sp_idx/sp_val[r0+kBins + i] = the candidates in descending bin order.  After
  // barrier A any CTA reads the crossing bin's segment of every CTA directly.
  uint32_t cta_n = 0;
#pragma unroll
  for (int w = 0; w < kTkWarps; ++w) cta_n += s_wn[w];
  const uint64_t r0 = (uint64_t)wstart(sp, b * kTkWarps) * kChunk;
  const uint64_t r1 = std::min<uint64_t>(N, (uint64_t)(wstart(sp, b * kTkWarps + kTkWarps - 1) +
                                                         wcount(sp, b * kTkWarps + kTkWarps - 1)) * kChunk);
  const bool fast_ok = !s_spill && (uint64_t)cta_n + kBins <= r1 - r0;
  TK_V(20, tau);
  TK_V(21, split);
  TK_V(22, cta_n);
  TK_V(23, fast_ok);
  if (fast_ok) {
    uint32_t* ab = reinterpret_cast<uint32_t*>(ring);   // per-bin cursors (the ring is drained)
    {
      constexpr int per = kBins / kTkThreads;
      const int base = kBins - per * (tid + 1);
      const uint4 lo4 = *reinterpret_cast<const uint4*>(sh + base);
      const uint4 hi4 = *reinterpret_cast<const uint4*>(sh + base + 4);
      const uint32_t v[per] = {hi4.w, hi4.z, hi4.y, hi4.x, lo4.w, lo4.z, lo4.y, lo4.x};
      uint32_t loc = 0;
#pragma unroll
      for (int i = 0; i < per; ++i) loc += v[i];
      uint64_t tot;
      uint32_t cum = (uint32_t)blk_excl_sum<uint64_t>(loc, s_sc, &tot);
      uint32_t o[per];
#pragma unroll
      for (int i = 0; i < per; ++i) {
        o[i] = cum;
        cum += v[i];
      }
      const uint4 olo = make_uint4(o[7], o[6], o[5], o[4]), ohi = make_uint4(o[3], o[2], o[1], o[0]);
      *reinterpret_cast<uint4*>(ab + base) = olo;
      *reinterpret_cast<uint4*>(ab + base + 4) = ohi;
      *reinterpret_cast<uint4*>(a.L.sp_idx + r0 + base) = olo;
      *reinterpret_cast<uint4*>(a.L.sp_idx + r0 + base + 4) = ohi;
    }
    __syncthreads();
    TK_D(12);
    uint32_t* si = a.L.sp_idx + r0 + kBins;
    float* sv = a.L.sp_val + r0 + kBins;
    // sorted into shared memory behind the cursors (the drained ring), then
    // copied out coalesced: scattered 4-byte global stores cost a sector each
    constexpr uint32_t kStageCap = (uint32_t)((Cfg::kRing - (size_t)kBins * 4) / 8);
    const bool staged = cta_n <= kStageCap;
    uint32_t* qi = ab + kBins;
    float* qv = reinterpret_cast<float*>(qi + kStageCap);
    for (uint32_t i = lane; i < nw; i += 32) {
      uint32_t idx;
      float v;
      cs.get(i, &idx, &v);
      const uint32_t key = abs_key(v);
      const uint32_t at = atomicAdd(&ab[bin_of(key, tau, split, shift)], 1u);
      SPARCML_CHECK(at < cta_n && r0 + kBins + at < r1);
      if (staged) {
        qi[at] = idx;
        qv[at] = v;
      } else {
        si[at] = idx;
        sv[at] = v;
      }
    }
    if (staged) {
      __syncthreads();
      for (uint32_t i = tid; i < cta_n; i += kTkThreads) {
        si[i] = qi[i];
        sv[i] = qv[i];
      }
    }
    TK_D(13);
  }
  // the level-0 histogram to global; per-call flags
  for (int i = tid; i < kBins; i += kTkThreads) {
    const uint32_t v = sh[i];
    if (v) atomicAdd(&c->hist[p][0][i], v);
    sh[i] = 0;
  }
  if (tid == 0) {
    if (s_bad) atomicOr(&c->bad[p], 1u);
    if (!fast_ok) atomicOr(&c->nofast[p], 1u);
    c->cta_a[b] = cta_n;
  }
  TK_D(6);
  tk_mark(c, 2);
  tk_grid_barrier(c, ++bar_t);   // ---- A
  TK_D(7);
  tk_mark(c, 3);
  if (b == 0 && tid == 0) {
    c->status = __ldcg(&c->bad[p]) ? 1u : 0u;
    c->bad[p ^ 1u] = 0;       // the next call's slots (the previous call has ended)
    c->sampled[p ^ 1u] = 0;
    c->list_n[p ^ 1u] = 0;
    c->nofast[p ^ 1u] = 0;
  }
  {   // the previous call's histogram slots, for the next call (every CTA has read them)
    uint4* hz = reinterpret_cast<uint4*>(&c->hist[p ^ 1u][0][0]);
    for (uint32_t i = b * kTkThreads + tid; i < (uint32_t)(kLevels * kBins / 4); i += G * kTkThreads)
      hz[i] = make_uint4(0u, 0u, 0u, 0u);
  }

  // ---- R: locate the k-th magnitude -------------------------------------------------
  uint32_t slot = 0;
  uint32_t lo = tau;
  uint64_t spl = split, hi = kKeyEnd, above = 0;
  uint32_t passes = 1;
  bool exact = false, fast = false, resampled = false;
  uint32_t kth = 0;
  uint64_t need = 0;
  {
    const uint4* gh = reinterpret_cast<const uint4*>(c->hist[p][0]);
    if (tid == 0) s_nofast = __ldcg(&c->nofast[p]);
    for (int i = tid; i < kBins / 4; i += kTkThreads) reinterpret_cast<uint4*>(sh)[i] = __ldcg(gh + i);
    __syncthreads();
    const Cross f = find_desc(sh, k, s_sc, &s_cross[0]);
    for (int i = tid; i < kBins; i += kTkThreads) sh[i] = 0;
    __syncthreads();
    TK_D(8);
    if (f.ok && !s_nofast) {
      const uint32_t B = f.bin;
      TK_V(24, f.cnt);
      TK_V(25, B);
      uint64_t blo, bhi;
      if (B == kBins - 1) {
        blo = split;
        bhi = kKeyEnd;
      } else {
        blo = (uint64_t)tau + ((uint64_t)B << shift);
        bhi = std::min<uint64_t>(split, (uint64_t)tau + ((uint64_t)(B + 1) << shift));
      }
      if (bhi - blo == 1 || f.cnt <= (uint32_t)kListCap) {
        // ---- fast path: the crossing bin's entries of every CTA, straight from
        // their sorted regions (no second barrier) ----
        fast = true;
        uint32_t* lk = reinterpret_cast<uint32_t*>(ring);   // crossing-bin keys
        uint32_t* lc = lk + kListCap;                        // their CTAs
        uint32_t* abh = lc + kListCap;                       // per CTA: candidates above the bin
        uint32_t* cnb = abh + kMaxGrid;                      // per CTA: candidates in the bin
        uint32_t* sof = cnb + kMaxGrid;                      // per CTA: offset of its entries in lk
        uint32_t* gtl = sof + kMaxGrid;                      // per CTA: bin entries > kth
        uint32_t* eql = gtl + kMaxGrid;                      // per CTA: bin entries == kth
        const uint32_t bb0 = 2 * tid, bb1 = 2 * tid + 1;
        auto cta_r0 = [&](uint32_t bq) { return (uint64_t)wstart(sp, bq * kTkWarps) * kChunk; };
        uint32_t ah0 = 0, al0 = 0, ah1 = 0, al1 = 0;
        if (bb0 < G) {
          const uint32_t* g0 = a.L.sp_idx + cta_r0(bb0);
          ah0 = __ldcg(g0 + B);
          al0 = B == 0 ? __ldcg(&c->cta_a[bb0]) : __ldcg(g0 + B - 1);
        }
        if (bb1 < G) {
          const uint32_t* g1 = a.L.sp_idx + cta_r0(bb1);
          ah1 = __ldcg(g1 + B);
          al1 = B == 0 ? __ldcg(&c->cta_a[bb1]) : __ldcg(g1 + B - 1);
        }
        const uint32_t n0 = al0 - ah0, n1 = al1 - ah1;
        uint64_t ntot;
        const uint32_t so0 = (uint32_t)blk_excl_sum<uint64_t>((uint64_t)n0 + n1, s_sc, &ntot);
        if (bb0 < G) {
          abh[bb0] = ah0;
          cnb[bb0] = n0;
          sof[bb0] = so0;
          gtl[bb0] = 0;
          eql[bb0] = 0;
        }
        if (bb1 < G) {
          abh[bb1] = ah1;
          cnb[bb1] = n1;
          sof[bb1] = so0 + n0;
          gtl[bb1] = 0;
          eql[bb1] = 0;
        }
        above = f.above;
        if (bhi - blo == 1) {   // the bin is one magnitude: every entry is a tie
          kth = (uint32_t)blo;
          need = k - above;
          __syncthreads();
          if (bb0 < G) eql[bb0] = n0;
          if (bb1 < G) eql[bb1] = n1;
          exact = true;
        } else {
          // gather every CTA's segment in one round of loads: entry e belongs to
          // the CTA bq with sof[bq] <= e < sof[bq + 1] (binary search)
          __syncthreads();
          for (uint32_t e = tid; e < (uint32_t)ntot; e += kTkThreads) {
            uint32_t lo_b = 0, hi_b = G;   // largest bq with sof[bq] <= e and cnb[bq] > 0
            while (hi_b - lo_b > 1) {
              const uint32_t mid = (lo_b + hi_b) >> 1;
              if (sof[mid] <= e) lo_b = mid;
              else hi_b = mid;
            }
            while (cnb[lo_b] == 0 || sof[lo_b] + cnb[lo_b] <= e) ++lo_b;   // skip empty segments
            SPARCML_CHECK(lo_b < G && e >= sof[lo_b] && e - sof[lo_b] < cnb[lo_b]);
            lk[e] = abs_key(__ldcg(a.L.sp_val + cta_r0(lo_b) + kBins + abh[lo_b] + (e - sof[lo_b])));
            lc[e] = lo_b;
          }
          __syncthreads();
          TK_D(9);
          const uint32_t n = (uint32_t)ntot;
          uint64_t t = k - above;
          {
            uint64_t rlo = blo, rhi = bhi;
            while (rhi - rlo > 1) {
              const uint32_t s = shift_for(rhi - rlo, kBins);
              for (uint32_t i = tid; i < n; i += kTkThreads) {
                const uint32_t key = lk[i];
                if (key >= rlo && key < rhi) atomicAdd(&sh[(uint32_t)(key - rlo) >> s], 1u);
              }
              __syncthreads();
              const Cross fr = find_desc(sh, t, s_sc, &s_cross[0]);
              for (int i = tid; i < kBins; i += kTkThreads) sh[i] = 0;
              __syncthreads();
              t -= fr.above;
              const uint64_t nlo = rlo + ((uint64_t)fr.bin << s);
              rhi = std::min<uint64_t>(rhi, rlo + ((uint64_t)(fr.bin + 1) << s));
              rlo = nlo;
            }
            kth = (uint32_t)rlo;
            need = t;
          }
          for (uint32_t i = tid; i < n; i += kTkThreads) {
            if (lk[i] > kth) atomicAdd(&gtl[lc[i]], 1u);
            else if (lk[i] == kth) atomicAdd(&eql[lc[i]], 1u);
          }
        }
        __syncthreads();
        TK_D(10);
        // per CTA (index order): ties are taken in CTA order, so the ties taken
        // before CTA b' are min(E_b', need) with E the prefix of the tie counts:
        // offset(b') = prefix(above-bin + above-kth) + min(E_b', need)
        const uint32_t e0 = bb0 < G ? eql[bb0] : 0u, e1 = bb1 < G ? eql[bb1] : 0u;
        const uint64_t g0 = bb0 < G ? (uint64_t)ah0 + gtl[bb0] : 0, g1 = bb1 < G ? (uint64_t)ah1 + gtl[bb1] : 0;
        uint64_t AG0, E0;
        blk_excl_sum2(g0 + g1, (uint64_t)e0 + e1, s_sc, &AG0, &E0);
        const uint64_t E1 = E0 + e0;
        if (bb0 == b) {
          s_off = AG0 + std::min<uint64_t>(E0, need);
          s_quota = (uint32_t)std::min<uint64_t>(e0, need > E0 ? need - E0 : 0);
        }
        if (bb1 == b) {
          s_off = AG0 + g0 + std::min<uint64_t>(E1, need);
          s_quota = (uint32_t)std::min<uint64_t>(e1, need > E1 ? need - E1 : 0);
        }
        __syncthreads();
      }
    }
  }

  if (!fast) {
    // ---- slow path: refinement levels / exact re-filter, then the list + barrier B --
    while (true) {
      {
        const uint4* gh = reinterpret_cast<const uint4*>(c->hist[p][slot]);
        for (int i = tid; i < kBins / 4; i += kTkThreads) reinterpret_cast<uint4*>(sh)[i] = __ldcg(gh + i);
      }
      __syncthreads();
      const Cross f = find_desc(sh, k - above, s_sc, &s_cross[0]);
      for (int i = tid; i < kBins; i += kTkThreads) sh[i] = 0;
      __syncthreads();
      if (!f.ok) {
        // fewer than k candidates: tau over-estimated the k-th magnitude.  Re-filter
        // the current vector (EF: acc, now in eps).  After a warm-start miss the
        // threshold comes from the sample of that vector (one more streaming pass);
        // otherwise -- or if that misses too -- exactly, with tau = 0 (every value
        // a candidate: far slower, a 5.6-sigma event for the sample).
        ++passes;
        ++slot;
        lo = 0;
        spl = kKeyEnd;
        hi = kKeyEnd;
        above = 0;
        nw = 0;
        const float* src = EF ? a.dst : a.x;
        if (warm && !resampled) {
          resampled = true;
          uint32_t* shs = cidx;   // the sample histogram, in the (discarded) candidate area
          constexpr int kSBins2 = 8192;
          for (int i = tid; i < kSBins2 / 4; i += kTkThreads)
            reinterpret_cast<uint4*>(shs)[i] = make_uint4(0u, 0u, 0u, 0u);
          __syncthreads();
          uint32_t ns = 0;
          for (uint32_t q = tid; q < (uint32_t)kSampleGran; q += kTkThreads) {
            uint64_t pos = 0;
            if (!sample_pos(q, N, C, W, sp, &pos)) continue;
            const float4 v = __ldcg(reinterpret_cast<const float4*>(src + pos));
            atomicAdd(&shs[abs_key(v.x) >> 18], 1u);
            atomicAdd(&shs[abs_key(v.y) >> 18], 1u);
            atomicAdd(&shs[abs_key(v.z) >> 18], 1u);
            atomicAdd(&shs[abs_key(v.w) >> 18], 1u);
            ns += 4;
          }
          uint64_t S;
          (void)blk_excl_sum<uint64_t>(ns, s_sc, &S);   // (ends with a block barrier)
          const float mean = (float)((double)k * (double)S / (double)N);
          const float sd = sqrtf(mean);
          const uint64_t t_lo = (uint64_t)ceilf(mean + 5.0f * sd + 4.0f);
          const float th = mean - 4.0f * sd - 16.0f;
          const uint64_t t_hi = th > 1.0f ? (uint64_t)th : 1;
          find2<kSBins2>(shs, t_lo, t_hi, s_sc, s_cross);
          const Cross f0 = s_cross[0], f1 = s_cross[1];
          __syncthreads();   // every thread has its crossings; the candidate area is free again
          lo = f0.ok ? (f0.bin << 18) : 0u;
          if (lo > 0x7F800000u) lo = 0x7F800000u;
          spl = f1.ok ? (uint64_t)(f1.bin + 1) << 18 : kKeyEnd;
          if (spl <= lo) spl = (uint64_t)lo + 1;
        }
        shift = shift_for(spl - lo, kBins - 1);
        for (uint32_t i = 0; i < nch; ++i) {
          const uint64_t cc = c0 + i;
          const bool full = (cc + 1) * kChunk <= N;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const uint64_t gp = cc * kChunk + r * 128 + lane * 4;
            float v[4];
            if (full) {
              const float4 xv = __ldcg(reinterpret_cast<const float4*>(src + gp));
              v[0] = xv.x; v[1] = xv.y; v[2] = xv.z; v[3] = xv.w;
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) v[j] = gp + j < N ? __ldcg(src + gp + j) : 0.0f;
            }
            uint32_t dummy = 0;
            consume_row<EF, false>(v, gp, full, N, nullptr, lo, spl, shift, sh, cs, nw, dummy);
          }
        }
        __syncthreads();
        for (int i = tid; i < kBins; i += kTkThreads) {
          const uint32_t v = sh[i];
          if (v) atomicAdd(&c->hist[p][slot][i], v);
          sh[i] = 0;
        }
        tk_grid_barrier(c, ++bar_t);
        continue;
      }
      uint64_t blo, bhi;
      if (f.bin == kBins - 1) {
        blo = spl;
        bhi = hi;
      } else {
        blo = (uint64_t)lo + ((uint64_t)f.bin << shift);
        bhi = std::min<uint64_t>(spl, (uint64_t)lo + ((uint64_t)(f.bin + 1) << shift));
      }
      above += f.above;
      lo = (uint32_t)blo;
      hi = bhi;
      if (bhi - blo == 1) {
        exact = true;
        break;
      }
      if (f.cnt <= (uint32_t)kListCap) break;
      // refine: histogram the candidates in [lo, hi) at a finer step
      ++slot;
      spl = hi;
      shift = shift_for(hi - lo, kBins - 1);
      for (uint32_t i0 = 0; i0 < nw; i0 += 32) {
        const uint32_t i = i0 + lane;
        if (i < nw) {
          uint32_t idx;
          float v;
          cs.get(i, &idx, &v);
          const uint32_t key = abs_key(v);
          if (key >= lo && (uint64_t)key < hi) atomicAdd(&sh[bin_of(key, lo, spl, shift)], 1u);
        }
      }
      __syncthreads();
      for (int i = tid; i < kBins; i += kTkThreads) {
        const uint32_t v = sh[i];
        if (v) atomicAdd(&c->hist[p][slot][i], v);
        sh[i] = 0;
      }
      tk_grid_barrier(c, ++bar_t);
    }
    tk_mark(c, 4);

    // ---- L: per-CTA counts above / in [lo, hi); the bin's candidates to the list --
    {
      uint32_t aw = 0, ew = 0;
      for (uint32_t i0 = 0; i0 < nw; i0 += 32) {
        const uint32_t i = i0 + lane;
        uint32_t key = 0;
        const bool in = i < nw;
        if (in) {
          uint32_t idx;
          float v;
          cs.get(i, &idx, &v);
          key = abs_key(v);
        }
        aw += __popc(__ballot_sync(0xffffffffu, in && (uint64_t)key >= hi));
        ew += __popc(__ballot_sync(0xffffffffu, in && key >= lo && (uint64_t)key < hi));
      }
      if (lane == 0) {
        s_w[warp][0] = aw;
        s_w[warp][1] = ew;
      }
      __syncthreads();
      if (tid == 0) {   // one list reservation per CTA; warp w's entries follow warps < w
        uint32_t sa = 0, se = 0;
        for (int w = 0; w < kTkWarps; ++w) {
          sa += s_w[w][0];
          const uint32_t e = s_w[w][1];
          s_w[w][1] = se;
          se += e;
        }
        c->cta_a[b] = sa;
        c->cta_e[b] = se;
        s_lbase = (!exact && se) ? atomicAdd(&c->list_n[p], se) : 0u;
      }
      __syncthreads();
      if (!exact && ew) {
        const uint32_t lt = lanemask_lt();
        uint32_t at = s_lbase + s_w[warp][1];
        for (uint32_t i0 = 0; i0 < nw; i0 += 32) {
          const uint32_t i = i0 + lane;
          uint32_t idx = 0, key = 0;
          float v = 0.0f;
          const bool in = i < nw;
          if (in) {
            cs.get(i, &idx, &v);
            key = abs_key(v);
          }
          const bool e = in && key >= lo && (uint64_t)key < hi;
          const uint32_t eb = __ballot_sync(0xffffffffu, e);
          if (e && at + __popc(eb & lt) < (uint32_t)kListCap)
            a.L.list[at + __popc(eb & lt)] = make_uint4(idx, key, b, 0u);
          at += __popc(eb);
        }
      }
    }
    tk_grid_barrier(c, ++bar_t);   // ---- B
    tk_mark(c, 5);

    // ---- exact k-th magnitude, ties, this CTA's offset ---------------------------
    {
      uint32_t* lk = reinterpret_cast<uint32_t*>(ring);       // list keys
      uint32_t* lc = lk + kListCap;                            // list CTAs
      uint32_t* gtl = lc + kListCap;                           // per CTA: list entries > kth
      uint32_t* eql = gtl + kMaxGrid;                          // per CTA: entries == kth (ties)
      const uint32_t b0 = 2 * tid, b1 = 2 * tid + 1;
      const uint32_t a0 = b0 < G ? __ldcg(&c->cta_a[b0]) : 0u, a1 = b1 < G ? __ldcg(&c->cta_a[b1]) : 0u;
      uint32_t ce0 = 0, ce1 = 0;
      if (exact) {
        ce0 = b0 < G ? __ldcg(&c->cta_e[b0]) : 0u;
        ce1 = b1 < G ? __ldcg(&c->cta_e[b1]) : 0u;
      }
      const uint32_t n = exact ? 0u : std::min<uint32_t>(__ldcg(&c->list_n[p]), (uint32_t)kListCap);
      for (uint32_t i = tid; i < G; i += kTkThreads) {
        gtl[i] = 0;
        eql[i] = 0;
      }
      for (uint32_t i = tid; i < n; i += kTkThreads) {
        const uint4 e = __ldcg(&a.L.list[i]);
        lk[i] = e.y;
        lc[i] = e.z;
      }
      __syncthreads();
      if (!exact) {
        uint64_t t = k - above;
        uint64_t rlo = lo, rhi = hi;
        while (rhi - rlo > 1) {
          const uint32_t s = shift_for(rhi - rlo, kBins);
          for (uint32_t i = tid; i < n; i += kTkThreads) {
            const uint32_t key = lk[i];
            if (key >= rlo && key < rhi) atomicAdd(&sh[(uint32_t)(key - rlo) >> s], 1u);
          }
          __syncthreads();
          const Cross fr = find_desc(sh, t, s_sc, &s_cross[0]);
          for (int i = tid; i < kBins; i += kTkThreads) sh[i] = 0;
          __syncthreads();
          t -= fr.above;
          const uint64_t nlo = rlo + ((uint64_t)fr.bin << s);
          rhi = std::min<uint64_t>(rhi, rlo + ((uint64_t)(fr.bin + 1) << s));
          rlo = nlo;
        }
        kth = (uint32_t)rlo;
        need = t;
        for (uint32_t i = tid; i < n; i += kTkThreads) {
          if (lk[i] > kth) atomicAdd(&gtl[lc[i]], 1u);
          else if (lk[i] == kth) atomicAdd(&eql[lc[i]], 1u);
        }
        __syncthreads();
      } else {
        kth = lo;
        need = k - above;
      }
      const uint32_t e0 = exact ? ce0 : (b0 < G ? eql[b0] : 0u), e1 = exact ? ce1 : (b1 < G ? eql[b1] : 0u);
      const uint32_t g0 = exact ? 0u : (b0 < G ? gtl[b0] : 0u), g1 = exact ? 0u : (b1 < G ? gtl[b1] : 0u);
      uint64_t etot;
      const uint64_t E0 = blk_excl_sum<uint64_t>((uint64_t)e0 + e1, s_sc, &etot);
      const uint64_t E1 = E0 + e0;
      const uint32_t q0 = (uint32_t)std::min<uint64_t>(e0, need > E0 ? need - E0 : 0);
      const uint32_t q1 = (uint32_t)std::min<uint64_t>(e1, need > E1 ? need - E1 : 0);
      const uint64_t s0 = (uint64_t)a0 + g0 + q0;
      const uint64_t s1 = (uint64_t)a1 + g1 + q1;
      uint64_t stot;
      const uint64_t O0 = blk_excl_sum<uint64_t>(s0 + s1, s_sc, &stot);
      if (b0 == b) {
        s_off = O0;
        s_quota = q0;
      }
      if (b1 == b) {
        s_off = O0 + s0;
        s_quota = q1;
      }
      __syncthreads();
    }
  }
  TK_D(11);
  TK_V(26, fast);
  TK_V(27, kth);
  if (b == 0 && tid == 0) {
    c->passes = passes;
    c->calls = c->calls + 1u;
    // warm start for the next call: only when the k-th magnitude fell inside this
    // call's level-0 range [tau, split) (a miss samples next time)
    c->warm_kth = (passes == 1u && kth >= tau && (uint64_t)kth < split) ? kth : 0u;
    c->warm_ef = EF ? 1u : 0u;
    c->warm_N = N;
    c->warm_k = k;
  }
  // ---- placement: per warp, pass 1 counts (> kth, == kth), every warp scans the
  // 16 pairs (offsets, tie quotas), pass 2 writes in index order.  Compact loops:
  // this code runs once per call, so its instruction footprint is its cost.
  tk_mark(c, 6);
  TK_D(16);
  {
    uint32_t gtw = 0, eqw = 0;
#pragma unroll 1
    for (uint32_t i0 = 0; i0 < nw; i0 += 32) {
      const uint32_t i = i0 + lane;
      uint32_t idx = 0, key = 0;
      float v = 0.0f;
      if (i < nw) {
        cs.get(i, &idx, &v);
        key = abs_key(v);
      }
      gtw += __popc(__ballot_sync(0xffffffffu, i < nw && key > kth));
      eqw += __popc(__ballot_sync(0xffffffffu, i < nw && key == kth));
    }
    if (lane == 0) {
      s_w[warp][0] = gtw;
      s_w[warp][1] = eqw;
    }
    __syncthreads();
    uint64_t o;
    uint32_t tq;
    {   // every warp scans the 16 (gt, eq) pairs itself: no second barrier
      const uint32_t gv = lane < kTkWarps ? s_w[lane][0] : 0u, ev = lane < kTkWarps ? s_w[lane][1] : 0u;
      const uint32_t E = warp_inclusive_sum<uint32_t>(ev) - ev;
      const uint32_t q = s_quota;
      const uint32_t t = q > E ? std::min(q - E, ev) : 0u;
      const uint32_t sel = gv + t;
      const uint32_t Sx = warp_inclusive_sum<uint32_t>(sel) - sel;
      o = s_off + __shfl_sync(0xffffffffu, Sx, warp);
      tq = __shfl_sync(0xffffffffu, t, warp);
    }
    const uint32_t lt = lanemask_lt();
    uint32_t run = 0, eq_run = 0;
#pragma unroll 1
    for (uint32_t i0 = 0; i0 < nw; i0 += 32) {
      const uint32_t i = i0 + lane;
      uint32_t idx = 0, key = 0;
      float v = 0.0f;
      if (i < nw) {
        cs.get(i, &idx, &v);
        key = abs_key(v);
      }
      const bool gsel = i < nw && key > kth, esel = i < nw && key == kth;
      const uint32_t eb = __ballot_sync(0xffffffffu, esel);
      const uint32_t eq_before = eq_run + __popc(eb & lt);
      const bool take = gsel || (esel && eq_before < tq);
      const uint32_t tb = __ballot_sync(0xffffffffu, take);
      if (take) {
        const uint64_t pos = o + run + __popc(tb & lt);
        SPARCML_CHECK(pos < k && idx < N);
        a.idx_out[pos] = idx;
        a.val_out[pos] = v;
        if (a.zero_at) a.zero_at[idx] = 0.0f;   // acc - TopK(acc)
      }
      run += __popc(tb);
      eq_run += __popc(eb);
    }
  }
  TK_D(17);
  tk_mark(c, 7);
}

// ------------------------------------------------------- bucketed ---------
// Bucketed top-k (§7; reading R-26): one warp per bucket
// of B = 128*R consecutive values, held in registers (R float4 per lane).
// The k-th largest |v| of the bucket is found by a 4-pass 8-bit radix select
// over the magnitude bit patterns (per-warp 256-bin shared histogram); the
// selected pairs are written in index order at bucket * min(k, B), and the
// residual / new eps (the unselected values, "saving the rest
// locally") is stored in the same pass.  HBM-bound: one read of x (+ g), one
// write of the residual.
struct BucketCtl {   // in the top-k workspace's control block (status only)
  uint32_t bad, done;
};

template <int R, bool EF, bool STORE>
__global__ void __launch_bounds__(kThreads, (R <= 4 ? 4 : 2)) topk_bucketed_kernel(const float* __restrict__ x,
                                                                 const float* __restrict__ g, float alpha,
                                                                 float* __restrict__ dst, uint64_t N, uint32_t k,
                                                                 uint32_t* __restrict__ idx_out,
                                                                 float* __restrict__ val_out, TopkCtl* ctl) {
  constexpr int B = 128 * R;
  __shared__ uint32_t hist[kWarps][256];
  __shared__ uint32_t s_bad;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  uint32_t* h = hist[warp];
  const uint64_t nb = (N + B - 1) / B;
  const uint32_t kb = k < (uint32_t)B ? k : (uint32_t)B;   // outputs of a full bucket
  const uint64_t pol = l2_evict_first_policy();
  uint32_t bad = 0;
  for (uint64_t bk = (uint64_t)blockIdx.x * kWarps + warp; bk < nb; bk += (uint64_t)gridDim.x * kWarps) {
    const uint64_t b0 = bk * B;
    const uint32_t n = (uint32_t)std::min<uint64_t>(B, N - b0);
    float v[R][4];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const uint32_t e = c * 128 + lane * 4;
      if (e + 4 <= n) {
        const float4 a = ld_stream_f4_ef(reinterpret_cast<const float4*>(x + b0 + e), pol);
        v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
        if (EF) {
          const float4 q = ld_stream_f4_ef(reinterpret_cast<const float4*>(g + b0 + e), pol);
          v[c][0] = __fmaf_rn(alpha, q.x, v[c][0]);
          v[c][1] = __fmaf_rn(alpha, q.y, v[c][1]);
          v[c][2] = __fmaf_rn(alpha, q.z, v[c][2]);
          v[c][3] = __fmaf_rn(alpha, q.w, v[c][3]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[c][q] = e + q < n ? x[b0 + e + q] : 0.0f;
          if (EF && e + q < n) v[c][q] = __fmaf_rn(alpha, g[b0 + e + q], v[c][q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) bad |= (e + q < n) && abs_key(v[c][q]) >= 0x7F800000u;
    }
    const uint32_t m = k < n ? k : n;   // selected in this bucket
    // selected: (key & selmask) > kth, plus the first `ties` (index order) of
    // the group (key & selmask) == kth with key >= T
    uint32_t kth = 0, ties = n, selmask = 0xFFFFFFFFu, T = 0;
    if (m < n) {
      // prefilter: T = the m-th largest lane maximum (m <= 32).  At least m
      // elements are >= T, so the k-th largest is >= T: only elements >= T
      // (usually about m of them) enter the radix select.
      if (m <= 32) {
        uint32_t lm = 0;
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c * 128 + lane * 4 + q < n) lm = max(lm, abs_key(v[c][q]));
        // bitonic sort of the 32 lane maxima, descending along the lanes
        uint32_t sv = lm;
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
          for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, sv, jj);
            const bool up = ((lane & kk) == 0) == ((lane & jj) == 0);   // keep the larger
            sv = up ? max(sv, o) : min(sv, o);
          }
        T = __shfl_sync(0xffffffffu, sv, (int)m - 1);
      }
      uint32_t C = 0;
#pragma unroll
      for (int c = 0; c < R; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) C += (c * 128 + lane * 4 + q < n && abs_key(v[c][q]) >= T) ? 1u : 0u;
      C = warp_sum<uint32_t>(C);
      if (C == m) {   // exactly the candidates: select key >= T
        kth = T;
        ties = n;
      } else {
        uint32_t prefix = 0, pmask = 0, need = m;
#pragma unroll
        for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
          for (int i = 0; i < 8; ++i) h[lane * 8 + i] = 0;
          __syncwarp();
#pragma unroll
          for (int c = 0; c < R; ++c)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (c * 128 + lane * 4 + q < n && abs_key(v[c][q]) >= T && (abs_key(v[c][q]) & pmask) == prefix)
                atomicAdd(&h[(abs_key(v[c][q]) >> shift) & 255u], 1u);
          __syncwarp();
          // lane l scans digits 255-8l .. 248-8l (descending)
          uint32_t cnt[8], loc = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            cnt[i] = h[255 - lane * 8 - i];
            loc += cnt[i];
          }
          const uint32_t incl = warp_inclusive_sum<uint32_t>(loc);
          const uint32_t before = incl - loc;
          const bool mine = before < need && incl >= need;
          uint32_t d = 0, above = 0, grp = 0;
          if (mine) {
            uint32_t cum = before;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (cum + cnt[i] >= need && cum < need) {
                d = 255 - lane * 8 - i;
                above = cum;
                grp = cnt[i];
              }
              cum += cnt[i];
            }
          }
          const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
          d = __shfl_sync(0xffffffffu, d, src);
          above = __shfl_sync(0xffffffffu, above, src);
          grp = __shfl_sync(0xffffffffu, grp, src);
          need -= above;
          prefix |= d << shift;
          pmask |= 0xFFu << shift;
          __syncwarp();
          if (grp == need) break;   // the whole group is selected: stop at this digit
        }
        kth = prefix;
        selmask = pmask;
        ties = need;
      }
    }
    // index order: chunk c, then lane, then q
    const uint64_t obase = bk * kb;
    uint32_t run_sel = 0, run_eq = 0;
#pragma unroll
    for (int c = 0; c < R; ++c) {
      uint32_t gtf = 0, eqf = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool in = c * 128 + lane * 4 + q < n;
        const uint32_t mk = abs_key(v[c][q]) & selmask;
        if (in && (m == n || mk > kth)) gtf |= 1u << q;
        else if (in && mk == kth && abs_key(v[c][q]) >= T) eqf |= 1u << q;
      }
      uint32_t self = gtf | eqf;
      if (ties < n) {   // only a prefix of the group (index order) is selected
        const uint32_t ne = __popc(eqf);
        const uint32_t eq_incl = warp_inclusive_sum<uint32_t>(ne);
        uint32_t eq_before = run_eq + eq_incl - ne;
        self = gtf;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (eqf & (1u << q)) {
            if (eq_before < ties) self |= 1u << q;
            ++eq_before;
          }
        run_eq += __shfl_sync(0xffffffffu, eq_incl, 31);
      }
      const uint32_t ns = __popc(self);
      const uint32_t s_incl = warp_inclusive_sum<uint32_t>(ns);
      uint32_t pos = run_sel + s_incl - ns;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (self & (1u << q)) {
          idx_out[obase + pos] = (uint32_t)(b0 + c * 128 + lane * 4 + q);
          val_out[obase + pos] = v[c][q];
          ++pos;
        }
      run_sel += __shfl_sync(0xffffffffu, s_incl, 31);
      if (STORE) {   // residual / new eps: the unselected values
        const uint32_t e = c * 128 + lane * 4;
        float o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = (self & (1u << q)) ? 0.0f : v[c][q];
        if (e + 4 <= n) st_stream_f4_ef(reinterpret_cast<float4*>(dst + b0 + e), make_float4(o[0], o[1], o[2], o[3]), pol);
        else
          for (int q = 0; q < 4; ++q)
            if (e + q < n) dst[b0 + e + q] = o[q];
      }
    }
  }
  // status: non-finite input seen by any block (the last block publishes it)
  if (ctl) {
    if (bad) s_bad = 1;
    __syncthreads();
    if (tid == 0) {
      BucketCtl* bc = reinterpret_cast<BucketCtl*>(&ctl->t_phase[15]);
      if (s_bad) atomicOr(&bc->bad, 1u);
      __threadfence();
      if (atomicAdd(&bc->done, 1u) == gridDim.x - 1) {
        __threadfence();
        ctl->status = atomicExch(&bc->bad, 0u) ? 1u : 0u;
        ctl->passes = 1;
        bc->done = 0;
      }
    }
  }
}

template <int R>
static cudaError_t launch_bucketed_r(const float* x, const float* grad, float alpha, int ef, float* dst, uint64_t N,
                                     uint32_t k, uint32_t* io, float* vo, TopkCtl* ctl, cudaStream_t s) {
  const uint64_t nb = (N + 128 * R - 1) / (128 * R);
  const unsigned blocks = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((nb + kWarps - 1) / kWarps, (uint64_t)device_sm_count() * 8));
  if (ef) topk_bucketed_kernel<R, true, true><<<blocks, kThreads, 0, s>>>(x, grad, alpha, dst, N, k, io, vo, ctl);
  else if (dst) topk_bucketed_kernel<R, false, true><<<blocks, kThreads, 0, s>>>(x, nullptr, 0.0f, dst, N, k, io, vo, ctl);
  else topk_bucketed_kernel<R, false, false><<<blocks, kThreads, 0, s>>>(x, nullptr, 0.0f, nullptr, N, k, io, vo, ctl);
  return cudaGetLastError();
}

cudaError_t launch_topk_bucketed(const float* x, const float* grad, float alpha, int ef, float* dst, uint64_t N,
                                 uint64_t k, uint64_t bucket, uint32_t* io, float* vo, void* ws, cudaStream_t s) {
  TopkCtl* ctl = ws ? reinterpret_cast<TopkCtl*>(ws) : nullptr;
  const uint32_t kk = (uint32_t)std::min<uint64_t>(k, bucket);
  SPARCML_PROF("topk_bucketed", s);
  cudaError_t e;
  switch (bucket / 128) {
    case 1: e = launch_bucketed_r<1>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    case 2: e = launch_bucketed_r<2>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    case 3: e = launch_bucketed_r<3>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    case 4: e = launch_bucketed_r<4>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    case 5: e = launch_bucketed_r<5>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    case 6: e = launch_bucketed_r<6>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    case 7: e = launch_bucketed_r<7>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    case 8: e = launch_bucketed_r<8>(x, grad, alpha, ef, dst, N, kk, io, vo, ctl, s); break;
    default: return cudaErrorInvalidValue;
  }
  ++g_launches;
  return e;
}

// --------------------------------------------------------- k >= N ---------
template <bool EF>
__global__ void topk_all_kernel(const float* x, const float* __restrict__ g, float alpha,
                                float* xout, float* __restrict__ resid, uint64_t N,   // EF: x == xout
                                uint32_t* __restrict__ idx_out, float* __restrict__ val_out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
    float v = x[i];
    if (EF) {
      v = __fmaf_rn(alpha, g[i], v);
      xout[i] = 0.0f;
    }
    idx_out[i] = (uint32_t)i;
    val_out[i] = v;
    if (!EF && resid) resid[i] = 0.0f;
  }
}


// ------------------------------------------------------------ launcher -----
static uint64_t topk_grid(uint64_t N) {
  const uint64_t C = (N + kChunk - 1) / kChunk;
  return std::max<uint64_t>(1, std::min<uint64_t>({(uint64_t)device_sm_count(), C / kTkWarps, (uint64_t)kMaxGrid}));
}

template <bool EF, bool STORE>
static cudaError_t launch_stream(const TkArgs& a, cudaStream_t s) {
  static unsigned attr_set = 0;   // per device: dynamic shared memory opt-in done
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 32 && !(attr_set & (1u << dev))) {
    const cudaError_t e = cudaFuncSetAttribute(topk_stream_kernel<EF, STORE>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TkCfg<EF>::kSmem);
    if (e != cudaSuccess) return e;
    attr_set |= 1u << dev;
  }
  TkArgs ac = a;
  void* args[] = {(void*)&ac};
  if (!SPARCML_TOPK_COOP) {   // one CTA per SM and a grid <= the SM count: co-resident once the SMs drain
    topk_stream_kernel<EF, STORE><<<dim3((unsigned)topk_grid(a.N)), dim3(kTkThreads), TkCfg<EF>::kSmem, s>>>(ac);
    return cudaGetLastError();
  }
  return cudaLaunchCooperativeKernel((const void*)topk_stream_kernel<EF, STORE>, dim3((unsigned)topk_grid(a.N)),
                                     dim3(kTkThreads), args, TkCfg<EF>::kSmem, s);
}

cudaError_t launch_topk(const float* x, const float* grad, float alpha, int ef, float* x_out, uint64_t N,
                        uint64_t k, uint32_t* idx_out, float* val_out, float* residual, void* ws,
                        cudaStream_t s) {
  const int sms = device_sm_count();
  if (k >= N) {
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((N + 255) / 256, (uint64_t)sms * 8));
    SPARCML_PROF("topk_all", s);
    if (ef) topk_all_kernel<true><<<blocks, 256, 0, s>>>(x, grad, alpha, x_out, nullptr, N, idx_out, val_out);
    else topk_all_kernel<false><<<blocks, 256, 0, s>>>(x, nullptr, 0.0f, nullptr, residual, N, idx_out, val_out);
    ++g_launches;
    return cudaGetLastError();
  }
  TkArgs a;
  a.x = x;
  a.g = grad;
  a.alpha = alpha;
  a.N = N;
  a.k = k;
  a.idx_out = idx_out;
  a.val_out = val_out;
  a.L = topk_layout(ws, N);
  cudaError_t e;
  {
    SPARCML_PROF("topk", s);
    if (ef) {   // eps is read through x and overwritten with acc, then zeroed at the selection
      a.dst = x_out;
      a.zero_at = x_out;
      e = launch_stream<true, true>(a, s);
    } else if (residual && residual != x) {
      a.dst = residual;
      a.zero_at = residual;
      e = launch_stream<false, true>(a, s);
    } else {    // no residual, or the residual is x itself (zeroed in place at the selection)
      a.dst = nullptr;
      a.zero_at = residual;
      e = launch_stream<false, false>(a, s);
    }
  }
  ++g_launches;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// host replica of sample_pos (diagnostics: lets a test build an input that
// defeats the sample and so exercises the exact re-filter)
size_t topk_sample_positions(uint64_t N, uint64_t* pos, size_t cap) {
  if (N < kSampleMinN) return 0;
  const uint32_t C = (uint32_t)((N + kChunk - 1) / kChunk), W = (uint32_t)topk_grid(N) * kTkWarps;
  const WSplit sp{C / W, C % W};
  size_t n = 0;
  for (uint32_t q = 0; q < (uint32_t)kSampleGran; ++q) {
    uint64_t p;
    if (!sample_pos(q, N, C, W, sp, &p)) continue;
    if (n < cap) pos[n] = p;
    ++n;
  }
  return n;
}

// status readback helper for the API
cudaError_t topk_read_status(const void* ws, uint32_t* status, uint32_t* passes, cudaStream_t s) {
  const TopkCtl* c = reinterpret_cast<const TopkCtl*>(ws);
  uint32_t tmp[2];
  cudaError_t e = cudaMemcpyAsync(tmp, &c->status, sizeof(tmp), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *status = tmp[0] ? SPARCML_ERR_NONFINITE : 0;
  *passes = tmp[1];
  return cudaSuccess;
}

}  // namespace sparcml
