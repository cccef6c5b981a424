// kernels_topk.cu — top-k sparsification with error feedback (§2.2 P:216-224,
// Algorithm 1) in one HBM pass over the N-vector, as ONE persistent
// cooperative kernel (grid = SMs x resident blocks).  Between phases the grid
// meets at a barrier whose LAST arriving block computes the next decision
// (threshold, bin, prefix) and publishes it before releasing the others.
//
//   S  sample : 8192 chunks of 8 values (one 32-byte sector every N/8192) ->
//               magnitude histogram -> conservative candidate threshold tau
//               (expected candidates ~ k + 4 sigma + 16 of the sample)
//   F  filter : the streaming pass over the block's contiguous 4096-tiles:
//               (EF) acc = fmaf(alpha, g, eps), eps <- acc; values with
//               |x| >= tau compacted per tile in index order; histogram of
//               candidate magnitudes in 4096 bins of width 2^s above tau
//   R  refine : histogram the candidates of the crossing bin until the bin is a
//               single magnitude: the exact k-th magnitude `kth` and how many
//               of its ties to keep (usually one refine level)
//   C  place  : per-block (gt, eq) counts -> grid prefix -> ordered placement of
//               |x| > kth and the first `need` ties (lower index wins, R-18);
//               the residual at the selected indices is zeroed.
// If the sample under-estimates (fewer than k candidates) every block
// re-filters with tau = 0 (exact; rare slow path, counted in `passes`).
#include <algorithm>
#include <cmath>

#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace sparcml {

constexpr int kTopkTile = 4096;           // elements per filter tile (16 per thread)
constexpr int kBins = 4096;
constexpr int kCoarse = 64;                   // coarse bins of 64 fine bins each, stored after the fine ones
constexpr int kHist = kBins + kCoarse;
constexpr uint64_t kSampleMinN = 1u << 16;   // below this: tau = 0 (all candidates)
constexpr uint32_t kSampleChunks = 8192;     // 8-value chunks sampled
constexpr int kMaxGrid = 4096;
#define kKeyEnd 0x80000000ull  // one past the largest |x| key (NaN included)
constexpr int kLevels = 4;                   // histogram levels (12 + 12 + 7 key bits worst case)

struct TopkCtl {
  uint64_t t_phase[16];     // %globaltimer at phase ends (block 0), diagnostics only
  uint32_t hist_s[kHist];   // sample histogram (key >> 19), then its 64 coarse sums
  uint32_t hist[kLevels][kHist];   // candidate histogram per refinement level (+ coarse sums)
  uint64_t blk[kMaxGrid];   // per-block (gt | eq << 32) selected counts
  uint32_t status, passes;
  uint32_t smax;            // largest sampled key
  uint32_t tile_ticket;     // filter tiles handed out dynamically
  uint32_t spill;           // some block could not keep its candidates in shared memory
  uint64_t t_blk[kMaxGrid][8];   // %globaltimer per block at phase ends (diagnostics)
};

struct TopkLayout {
  TopkCtl* ctl;
  uint64_t* tile_sel;       // per-tile (gt | eq << 32) selected counts
  uint32_t* tile_count;
  uint32_t* cand_idx;
  float* cand_val;
  uint64_t* gsum;           // per 64-tile group: sum of tile_sel (fast placement path)
  uint64_t ntiles, ngroups;
};

constexpr int kGroupTiles = 64;

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static TopkLayout topk_layout(void* ws, uint64_t N) {
  TopkLayout L;
  char* p = static_cast<char*>(ws);
  L.ntiles = (N + kTopkTile - 1) / kTopkTile;
  L.ctl = reinterpret_cast<TopkCtl*>(p);
  p += align256(sizeof(TopkCtl));
  L.tile_sel = reinterpret_cast<uint64_t*>(p);
  p += align256(L.ntiles * sizeof(uint64_t));
  L.tile_count = reinterpret_cast<uint32_t*>(p);
  p += align256(L.ntiles * sizeof(uint32_t));
  L.cand_idx = reinterpret_cast<uint32_t*>(p);
  p += align256(L.ntiles * kTopkTile * sizeof(uint32_t));
  L.cand_val = reinterpret_cast<float*>(p);
  p += align256(L.ntiles * kTopkTile * sizeof(float));
  L.ngroups = (L.ntiles + kGroupTiles - 1) / kGroupTiles;
  L.gsum = reinterpret_cast<uint64_t*>(p);
  return L;
}

size_t topk_workspace_bytes(uint64_t N, uint64_t /*k*/) {
  const uint64_t nt = (N + kTopkTile - 1) / kTopkTile;
  return align256(sizeof(TopkCtl)) + align256(nt * sizeof(uint64_t)) + align256(nt * sizeof(uint32_t)) +
         2 * align256(nt * kTopkTile * sizeof(uint32_t)) + align256(((nt + 63) / 64) * sizeof(uint64_t));
}

__device__ __forceinline__ uint32_t abs_key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

__device__ __forceinline__ void mark(TopkCtl* c, int i) {
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == 0) c->t_phase[i] = t;
    if (i < 8) c->t_blk[blockIdx.x][i] = t;
  }
}

// level binning: bins 0..kBins-2 cover [lo, split) in steps of 2^shift (the
// shift is chosen so that they do), bin kBins-1 collects every key >= split
__device__ __forceinline__ uint32_t bin_of(uint32_t key, uint64_t lo, uint64_t split, uint32_t shift) {
  if ((uint64_t)key >= split) return kBins - 1;
  const uint64_t b = ((uint64_t)key - lo) >> shift;
  return b < (uint64_t)(kBins - 1) ? (uint32_t)b : (uint32_t)(kBins - 2);
}

__host__ __device__ __forceinline__ uint32_t shift_for(uint64_t span, uint64_t nbins) {
  uint32_t s = 0;
  while ((nbins << s) < span) ++s;
  return s;
}

// Grid-wide barrier of a cooperative launch.  The last block to arrive runs
// f() (whole block) before releasing the others; f's global writes are
// visible to every block after the barrier.
// Whole block: the highest bin b with above0 + (count in bins > b) < target
// <= above0 + (count in bins >= b).  h is staged through shared memory
// (coalesced).  Returns b and the count strictly above it (including above0).
// If the histogram cannot reach the target: b = 0 and *reached = false.
struct BinFind {
  uint32_t bin;
  uint64_t above;
  bool reached;
};

// Up to two targets.  Two small reads instead of one 16 KB one (every block
// runs this on the same histogram right after a grid barrier, so the read is
// the contended part): warp 0 scans the 64 coarse sums from the top, then warp
// q scans the 64 fine bins of target q's coarse bin.  Same result as a scan of
// the fine bins (the coarse sums are their exact sums).
__device__ __forceinline__ bool pair_find(uint32_t hi, uint32_t lo, uint64_t base, uint64_t tg, uint32_t* which,
                                          uint64_t* above) {
  // lane holds bins (hi, lo) of a descending scan; base = count above them
  if (!(base < tg && base + hi + lo >= tg)) return false;
  if (base + hi >= tg) {
    *which = 0;
    *above = base;
  } else {
    *which = 1;
    *above = base + hi;
  }
  return true;
}

__device__ void find_bins(const uint32_t* h, uint64_t above0, const uint64_t* target, int ntarget, uint32_t* /*sm*/,
                          BinFind* out) {
  __shared__ uint32_t s_cb[2];
  __shared__ uint64_t s_ca[2];
  __shared__ int s_ok[2];
  __shared__ BinFind s_res[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    const uint32_t* hc = h + kBins;
    const uint32_t chi = __ldcg(&hc[63 - 2 * lane]), clo = __ldcg(&hc[62 - 2 * lane]);
    const uint32_t s = chi + clo;
    const uint64_t excl = warp_inclusive_sum<uint64_t>(s) - s;
    for (int q = 0; q < ntarget; ++q) {
      uint32_t which = 0;
      uint64_t ab = 0;
      const bool hit = pair_find(chi, clo, above0 + excl, target[q], &which, &ab);
      const uint32_t m = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) s_ok[q] = m != 0;
      if (hit) {
        s_cb[q] = 63 - 2 * lane - which;
        s_ca[q] = ab;
      }
    }
  }
  __syncthreads();
  if (warp < ntarget) {
    const int q = warp;
    if (!s_ok[q]) {
      if (lane == 0) s_res[q] = BinFind{0u, above0, false};
    } else {
      const uint32_t* hf = h + (size_t)s_cb[q] * 64;
      const uint32_t fhi = __ldcg(&hf[63 - 2 * lane]), flo = __ldcg(&hf[62 - 2 * lane]);
      const uint32_t s = fhi + flo;
      const uint64_t excl = warp_inclusive_sum<uint64_t>(s) - s;
      uint32_t which = 0;
      uint64_t ab = 0;
      if (pair_find(fhi, flo, s_ca[q] + excl, target[q], &which, &ab))
        s_res[q] = BinFind{s_cb[q] * 64 + 63 - 2 * lane - which, ab, true};
    }
  }
  __syncthreads();
  for (int q = 0; q < ntarget; ++q) out[q] = s_res[q];
  __syncthreads();
}

// One tile: 16 values per thread (4 coalesced float4 rows).  Candidates are
// written in index order to the tile's region and binned into `sh`.
#ifndef SPARCML_TOPK_KEEP
#define SPARCML_TOPK_KEEP 1      // 0: always take the global-memory path (A/B diagnostics)
#endif
#ifndef SPARCML_TOPK_CANDCAP
#define SPARCML_TOPK_CANDCAP 2048
#endif
#ifndef SPARCML_TOPK_MINB
#define SPARCML_TOPK_MINB 3      // blocks per SM (A/B at N = 2^24: 3 beats 4 by 1.5 us, 2 loses 2.5 us)
#endif
constexpr int kCandCap = SPARCML_TOPK_CANDCAP;   // candidates a block keeps in shared memory
constexpr int kTileCap = 32;     // tiles a block tracks

// The block's filtered tiles and their candidates, kept in shared memory for
// the refine / count / place phases (no global re-reads).  spill = some tile
// did not fit: the whole grid then takes the global-memory path.
struct KeepSmem {
  uint32_t ci[kCandCap];
  float cv[kCandCap];
  uint32_t tl[kTileCap], tn[kTileCap], to[kTileCap];
  uint64_t tp[kTileCap];
  uint32_t ntl, nc, spill;
};

template <bool EF, bool RESID, bool STORE>
__device__ __forceinline__ void filter_tile(const float* __restrict__ x, const float* __restrict__ g, float alpha,
                                            float* __restrict__ xout, float* __restrict__ resid, uint64_t N, uint64_t t,
                                            uint32_t tau, uint64_t split, uint32_t shift, const TopkLayout& L,
                                            uint32_t* sh, uint32_t* s_wt, uint32_t* s_status, KeepSmem* ks) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t base = t * kTopkTile;
  const uint64_t pol = l2_evict_first_policy();
  float v[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t p = base + (uint64_t)(j * kThreads + tid) * 4;
    if (p + 4 <= N) {
      const float4 a = ld_stream_f4_ef(reinterpret_cast<const float4*>(x + p), pol);
      v[j][0] = a.x; v[j][1] = a.y; v[j][2] = a.z; v[j][3] = a.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[j][q] = (p + q < N) ? x[p + q] : 0.0f;
    }
  }
  if (EF) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t p = base + (uint64_t)(j * kThreads + tid) * 4;
      if (p + 4 <= N) {
        const float4 a = ld_stream_f4_ef(reinterpret_cast<const float4*>(g + p), pol);
        v[j][0] = __fmaf_rn(alpha, a.x, v[j][0]);
        v[j][1] = __fmaf_rn(alpha, a.y, v[j][1]);
        v[j][2] = __fmaf_rn(alpha, a.z, v[j][2]);
        v[j][3] = __fmaf_rn(alpha, a.w, v[j][3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (p + q < N) v[j][q] = __fmaf_rn(alpha, g[p + q], v[j][q]);
      }
    }
  }
  if (STORE) {   // EF: eps <- acc ; sparsify: residual <- x
    float* dst = EF ? xout : resid;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t p = base + (uint64_t)(j * kThreads + tid) * 4;
      if (p + 4 <= N) {
        st_stream_f4_ef(reinterpret_cast<float4*>(dst + p), make_float4(v[j][0], v[j][1], v[j][2], v[j][3]), pol);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (p + q < N) dst[p + q] = v[j][q];
      }
    }
  }
  // candidate flags and in-order compaction over (row j, warp, lane, q)
  uint32_t flags[4];
  uint32_t bad = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    flags[j] = 0;
    const uint64_t p = base + (uint64_t)(j * kThreads + tid) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t key = abs_key(v[j][q]);
      if (p + q < N) {
        bad |= key >= 0x7F800000u;
        if (key >= tau) flags[j] |= 1u << q;
      }
    }
  }
  if (bad) *s_status = 1;
  uint32_t incl[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    incl[j] = warp_inclusive_sum<uint32_t>(__popc(flags[j]));
    if (lane == 31) s_wt[j * kWarps + warp] = incl[j];
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = s_wt[lane];   // 4 * 8 = 32 entries, (j, warp) order
    const uint32_t wi = warp_inclusive_sum<uint32_t>(w);
    s_wt[32 + lane] = wi - w;
    if (lane == 31) s_wt[64] = wi;
  }
  __syncthreads();
  const uint32_t tcount = s_wt[64];
  const uint32_t kb = ks ? ks->nc : 0u;
  const bool keep = ks && kb + tcount <= (uint32_t)kCandCap && ks->ntl < (uint32_t)kTileCap;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t pos = s_wt[32 + j * kWarps + warp] + incl[j] - __popc(flags[j]);
    const uint64_t p = base + (uint64_t)(j * kThreads + tid) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (flags[j] & (1u << q)) {
        L.cand_idx[base + pos] = (uint32_t)(p + q);
        L.cand_val[base + pos] = v[j][q];
        if (keep) {
          ks->ci[kb + pos] = (uint32_t)(p + q);
          ks->cv[kb + pos] = v[j][q];
        }
        const uint32_t bn = bin_of(abs_key(v[j][q]), tau, split, shift);
        atomicAdd(&sh[bn], 1u);
        atomicAdd(&sh[kBins + (bn >> 6)], 1u);
        ++pos;
      }
    }
  }
  if (tid == 0) L.tile_count[t] = tcount;
  __syncthreads();
  if (ks && tid == 0) {   // read by every thread only after the next tile's first barrier
    if (keep) {
      ks->tl[ks->ntl] = (uint32_t)t;
      ks->tn[ks->ntl] = tcount;
      ks->to[ks->ntl] = kb;
      ks->ntl = ks->ntl + 1;
      ks->nc = kb + tcount;
    } else {
      ks->spill = 1;
    }
  }
}

// A refinement level: bins 0..kBins-2 cover [lo, split) in steps of 2^shift,
// bin kBins-1 is [split, hi); `above` counts candidates with key >= hi.
struct Level {
  uint64_t lo, split, hi, above;
  uint32_t shift;
  int exact;
  uint32_t kth;
  uint64_t need;
};

// Narrow the level to the crossing bin f (found in this level's histogram).
__device__ __forceinline__ void apply_narrow(Level& lv, const BinFind& f, uint64_t k) {
  uint64_t nlo, nhi;
  if (f.bin == kBins - 1) {
    nlo = lv.split;
    nhi = lv.hi;
  } else {
    nlo = lv.lo + ((uint64_t)f.bin << lv.shift);
    nhi = min(lv.split, lv.lo + ((uint64_t)(f.bin + 1) << lv.shift));
  }
  lv.above = f.above;
  lv.lo = nlo;
  lv.split = nhi;
  lv.hi = nhi;
  if (nhi - nlo <= 1) {
    lv.exact = 1;
    lv.kth = (uint32_t)nlo;
    lv.need = k - f.above;
  } else {
    lv.shift = shift_for(nhi - nlo, kBins - 1);
  }
}

// Whole block (every block computes the same result from the same global
// histogram): locate the crossing bin of `h` and narrow the level.
__device__ __forceinline__ void narrow(Level& lv, const uint32_t* h, uint64_t k, uint32_t* sm) {
  BinFind f;
  find_bins(h, lv.above, &k, 1, sm, &f);
  apply_narrow(lv, f, k);
}

// Warp: load the (up to 128) candidates [i0, i0+128) of a tile, 4 per lane in flight.
__device__ __forceinline__ void load4(const float* cv, uint32_t n, uint32_t i0, float v[4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t i = i0 + r * 32 + lane;
    v[r] = i < n ? __ldcg(&cv[i]) : 0.0f;
  }
}

__device__ __forceinline__ void flush_hist(const uint32_t* sh, uint32_t* gh) {
  __syncthreads();
  for (int i = threadIdx.x; i < kHist; i += kThreads) {
    const uint32_t v = sh[i];
    if (v) atomicAdd(&gh[i], v);
  }
}

constexpr int kGroup = 32;   // tiles per placement group (one warp scans their prefix)

template <bool EF, bool RESID>
__global__ void __launch_bounds__(kThreads, SPARCML_TOPK_MINB) topk_fused_kernel(const float* __restrict__ x,
                                                                 const float* __restrict__ g, float alpha,
                                                                 float* __restrict__ xout, float* __restrict__ resid,
                                                                 uint64_t N, uint64_t k, uint32_t* __restrict__ idx_out,
                                                                 float* __restrict__ val_out, float* zero_at,
                                                                 TopkLayout L) {
  __shared__ uint32_t sh[kBins + kBins / 16];   // histogram; find_bin staging (padded)
  __shared__ uint32_t s_wt[65];
  __shared__ uint32_t s_status, s_ticket;
  __shared__ uint64_t s_sum[kWarps + 1];
  __shared__ uint64_t s_pref[kGroup];
  __shared__ uint64_t s_base;
  __shared__ KeepSmem ks;
  __shared__ uint32_t s_fast;
  cg::grid_group grid = cg::this_grid();
  TopkCtl* c = L.ctl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t gwarp = b * kWarps + warp, nwarps = G * kWarps;
  const uint64_t t0 = L.ntiles * b / G, t1 = L.ntiles * (b + 1) / G;   // this block's tiles in C
  for (int i = tid; i < kHist; i += kThreads) sh[i] = 0;
  if (tid == 0) {
    s_status = 0;
    ks.ntl = 0;
    ks.nc = 0;
    ks.spill = SPARCML_TOPK_KEEP ? 0u : 1u;
  }
  if (b == 0 && tid == 0) {
    c->tile_ticket = 0;
    c->status = 0;
    c->spill = 0;
  }
  for (uint64_t i = (uint64_t)b * kThreads + tid; i < L.ngroups; i += (uint64_t)G * kThreads) L.gsum[i] = 0;
  mark(c, 0);

  // ---- S: sample ----------------------------------------------------------------
  const uint64_t nchunk = N >= kSampleMinN ? std::min<uint64_t>(kSampleChunks, N / 8) : 0;
  const uint32_t sblocks = (uint32_t)std::min<uint64_t>(G, (nchunk + kThreads - 1) / kThreads);
  __syncthreads();
  if (b < sblocks) {
    const uint64_t ch = (uint64_t)b * kThreads + tid;
    uint32_t mx = 0;
    if (ch < nchunk) {
      const uint64_t pos = (ch * (N / 8) / nchunk) * 8;
      float v[8];
      const float4 a0 = *reinterpret_cast<const float4*>(x + pos);
      const float4 a1 = *reinterpret_cast<const float4*>(x + pos + 4);
      v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w;
      v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
      if (EF) {
        const float4 g0 = *reinterpret_cast<const float4*>(g + pos);
        const float4 g1 = *reinterpret_cast<const float4*>(g + pos + 4);
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fmaf_rn(alpha, gg[i], v[i]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t key = abs_key(v[i]);
        mx = max(mx, key);
        atomicAdd(&sh[key >> 19], 1u);
        atomicAdd(&sh[kBins + (key >> 25)], 1u);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx) atomicMax(&c->smax, mx);
    flush_hist(sh, c->hist_s);
    __syncthreads();
    for (int i = tid; i < kHist; i += kThreads) sh[i] = 0;
  }
  mark(c, 1);
  grid.sync();
  // tau: where the sample's count from the top reaches mean + 4 sigma + 16;
  // split: where it reaches mean - 4 sigma - 16.  The k-th magnitude lies in
  // [tau, split) with overwhelming probability: level-1 bins cover that range
  // finely, everything above it is one bin.  (Same result in every block.)
  Level lv;
  lv.lo = 0;
  lv.split = kKeyEnd;
  lv.hi = kKeyEnd;
  lv.above = 0;
  lv.shift = shift_for(kKeyEnd, kBins - 1);
  lv.exact = 0;
  lv.kth = 0;
  lv.need = 0;
  if (nchunk) {
    const double S = (double)nchunk * 8.0;
    const double mean = (double)k * S / (double)N;
    const uint64_t t_lo = (uint64_t)ceil(mean + 4.0 * sqrt(mean) + 16.0);
    const double th = mean - 4.0 * sqrt(mean) - 16.0;
    const uint64_t t_hi = th > 1.0 ? (uint64_t)th : 1;
    const uint64_t tg[2] = {t_lo, t_hi};
    BinFind fb[2];
    find_bins(c->hist_s, 0, tg, 2, sh, fb);
    const bool ok = fb[0].reached, okh = fb[1].reached;
    const uint32_t bn = fb[0].bin, bh = fb[1].bin;
    const uint64_t tau = ok ? ((uint64_t)bn << 19) : 0ull;
    const uint64_t top = (uint64_t)__ldcg(&c->smax) + (1ull << 23);   // 2 x the largest sample
    uint64_t split = okh ? min((uint64_t)(bh + 1) << 19, (uint64_t)kKeyEnd) : min(top, (uint64_t)kKeyEnd);
    if (split <= tau) split = tau + 1;
    lv.lo = tau;
    lv.split = split;
    lv.shift = shift_for(split - tau, kBins - 1);
  }
  for (int i = tid; i < kHist; i += kThreads) sh[i] = 0;
  __syncthreads();
  mark(c, 2);
  const uint32_t tau = (uint32_t)lv.lo;

  // ---- F: the streaming pass (tiles handed out dynamically for balance) ------
  while (true) {
    if (tid == 0) s_ticket = atomicAdd(&c->tile_ticket, 1u);
    __syncthreads();
    const uint64_t t = s_ticket;
    if (t >= L.ntiles) break;
    filter_tile<EF, RESID, EF || RESID>(x, g, alpha, xout, resid, N, t, tau, lv.split, lv.shift, L, sh, s_wt,
                                        &s_status, SPARCML_TOPK_KEEP ? &ks : nullptr);
  }
  mark(c, 3);
  flush_hist(sh, c->hist[0]);
  if (tid == 0 && s_status) atomicOr(&c->status, 1u);
  if (tid == 0 && ks.spill) atomicOr(&c->spill, 1u);
  grid.sync();
  if (tid == 0) s_fast = __ldcg(&c->spill) == 0u;
  mark(c, 4);
  {
    BinFind f0;
    find_bins(c->hist[0], lv.above, &k, 1, sh, &f0);
    if (!f0.reached) {   // fewer than k candidates: the sample under-estimated; exact re-filter with tau = 0 (rare)
      grid.sync();   // every block has read hist[0]
      if (b == 0) {
        for (int i = tid; i < kHist; i += kThreads) c->hist[0][i] = 0;
        if (tid == 0) {
          c->tile_ticket = 0;
          c->passes = 2;
        }
      }
      for (int i = tid; i < kHist; i += kThreads) sh[i] = 0;
      if (tid == 0) s_fast = 0;   // the re-filtered candidates live in global memory only
      grid.sync();
      lv.lo = 0;
      lv.split = kKeyEnd;
      lv.shift = shift_for(kKeyEnd, kBins - 1);
      const float* src = EF ? xout : x;
      while (true) {
        if (tid == 0) s_ticket = atomicAdd(&c->tile_ticket, 1u);
        __syncthreads();
        const uint64_t t = s_ticket;
        if (t >= L.ntiles) break;
        filter_tile<false, false, false>(src, nullptr, 0.0f, nullptr, nullptr, N, t, 0u, lv.split, lv.shift, L, sh,
                                         s_wt, &s_status, nullptr);
      }
      flush_hist(sh, c->hist[0]);
      grid.sync();
      narrow(lv, c->hist[0], k, sh);
    } else {
      if (b == 0 && tid == 0) c->passes = 1;
      apply_narrow(lv, f0, k);
    }
  }
  mark(c, 5);

  // ---- R: refine the crossing bin until it is one magnitude ------------------
  int level = 1;
  while (!lv.exact) {
    uint32_t* gh = c->hist[level < kLevels ? level : kLevels - 1];
    if (s_fast) {
      for (uint32_t i = tid; i < ks.nc; i += kThreads) {
        const uint32_t key = abs_key(ks.cv[i]);
        if (key >= lv.lo && key < lv.hi) {
          const uint32_t bn = bin_of(key, lv.lo, lv.split, lv.shift);
          atomicAdd(&gh[bn], 1u);
          atomicAdd(&gh[kBins + (bn >> 6)], 1u);
        }
      }
    } else
    for (uint64_t t = gwarp; t < L.ntiles; t += nwarps) {
      const uint32_t n = __ldcg(&L.tile_count[t]);
      const float* cv = L.cand_val + t * kTopkTile;
      for (uint32_t i0 = 0; i0 < n; i0 += 128) {
        float v[4];
        load4(cv, n, i0, v);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t key = abs_key(v[r]);
          if (i0 + r * 32 + lane < n && key >= lv.lo && key < lv.hi) {
            const uint32_t bn = bin_of(key, lv.lo, lv.split, lv.shift);
            atomicAdd(&gh[bn], 1u);
            atomicAdd(&gh[kBins + (bn >> 6)], 1u);
          }
        }
      }
    }
    grid.sync();
    narrow(lv, gh, k, sh);
    ++level;
  }
  mark(c, 6);
  const uint32_t kth = lv.kth;
  const uint64_t need = lv.need;

  // ---- C: ordered placement (index order = tile order, then in-tile order) --
  if (s_fast) {
    // per kept tile: (#|v| > kth) | (#|v| == kth) << 32, from shared memory
    for (uint32_t j = warp; j < ks.ntl; j += kWarps) {
      const uint32_t n = ks.tn[j], o = ks.to[j];
      uint32_t ng = 0, ne = 0;
      for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t key = abs_key(ks.cv[o + i]);
        ng += key > kth;
        ne += key == kth;
      }
      ng = warp_sum<uint32_t>(ng);
      ne = warp_sum<uint32_t>(ne);
      if (lane == 0) {
        const uint64_t sel = (uint64_t)ng | ((uint64_t)ne << 32);
        L.tile_sel[ks.tl[j]] = sel;
        if (sel) atomicAdd(reinterpret_cast<unsigned long long*>(&L.gsum[ks.tl[j] / kGroupTiles]), sel);
      }
    }
    mark(c, 10);
  } else {
    uint64_t bsum = 0;
    for (uint64_t t = t0 + warp; t < t1; t += kWarps) {
      const uint32_t n = __ldcg(&L.tile_count[t]);
      const float* cv = L.cand_val + t * kTopkTile;
      uint32_t ng = 0, ne = 0;
      for (uint32_t i0 = 0; i0 < n; i0 += 128) {
        float v[4];
        load4(cv, n, i0, v);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const bool in = i0 + r * 32 + lane < n;
          const uint32_t key = abs_key(v[r]);
          ng += __popc(__ballot_sync(0xffffffffu, in && key > kth));
          ne += __popc(__ballot_sync(0xffffffffu, in && key == kth));
        }
      }
      const uint64_t sel = (uint64_t)ng | ((uint64_t)ne << 32);
      if (lane == 0) {
        L.tile_sel[t] = sel;
        bsum += sel;
      }
    }
    {
      uint64_t tot;
      block_exclusive_sum<uint64_t>(bsum, s_sum, &tot);
      if (tid == 0) c->blk[b] = tot;
    }
  }
  grid.sync();
  mark(c, 8);
  // every histogram has been read by every block: clear them for the next call
  if (b < (uint32_t)(kLevels + 1)) {
    uint32_t* h = b == 0 ? c->hist_s : c->hist[b - 1];
    for (int i = tid; i < kHist; i += kThreads) h[i] = 0;
    if (b == 0 && tid == 0) c->smax = 0;
  }
  if (s_fast) {
    // exclusive prefix of tile_sel at each kept tile: the group sums before
    // its 64-tile group plus the tiles before it in the group (one warp per tile)
    for (uint32_t j = warp; j < ks.ntl; j += kWarps) {
      const uint64_t t = ks.tl[j], g0 = t / kGroupTiles;
      uint64_t v = 0;
      for (uint64_t i = lane; i < g0; i += 32) v += __ldcg(reinterpret_cast<const unsigned long long*>(&L.gsum[i]));
#pragma unroll
      for (int q = 0; q < kGroupTiles / 32; ++q) {
        const uint64_t tt = g0 * kGroupTiles + q * 32 + lane;
        if (tt < t) v += __ldcg(reinterpret_cast<const unsigned long long*>(&L.tile_sel[tt]));
      }
      v = warp_sum<uint64_t>(v);
      if (lane == 0) ks.tp[j] = v;
    }
    __syncthreads();
    mark(c, 9);
    for (uint32_t j = warp; j < ks.ntl; j += kWarps) {
      const uint32_t n = ks.tn[j], o = ks.to[j];
      uint64_t gt_run = ks.tp[j] & 0xFFFFFFFFull, eq_run = ks.tp[j] >> 32;
      for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const float vv = i < n ? ks.cv[o + i] : 0.0f;
        const uint32_t key = abs_key(vv);
        const bool gsel = i < n && key > kth, esel = i < n && key == kth;
        const uint32_t gbal = __ballot_sync(0xffffffffu, gsel), ebal = __ballot_sync(0xffffffffu, esel);
        const uint32_t lower = (1u << lane) - 1u;
        const uint64_t gt_before = gt_run + __popc(gbal & lower);
        const uint64_t eq_before = eq_run + __popc(ebal & lower);
        if (gsel || (esel && eq_before < need)) {
          const uint64_t pos = gt_before + (eq_before < need ? eq_before : need);
          const uint32_t j2 = ks.ci[o + i];
          idx_out[pos] = j2;
          val_out[pos] = vv;
          if (zero_at) zero_at[j2] = 0.0f;   // acc - TopK(acc)
        }
        gt_run += __popc(gbal);
        eq_run += __popc(ebal);
      }
    }
  } else {
    {
      uint64_t v = 0;
      for (uint32_t j = tid; j < b; j += kThreads) v += __ldcg(reinterpret_cast<const unsigned long long*>(&c->blk[j]));
      uint64_t tot;
      block_exclusive_sum<uint64_t>(v, s_sum, &tot);
      if (tid == 0) s_base = tot;
    }
    __syncthreads();
    for (uint64_t gs = t0; gs < t1; gs += kGroup) {
      const int nt = (int)std::min<uint64_t>(kGroup, t1 - gs);
      if (warp == 0) {
        const uint64_t v = lane < nt ? __ldcg(reinterpret_cast<const unsigned long long*>(&L.tile_sel[gs + lane])) : 0ull;
        const uint64_t inc = warp_inclusive_sum<uint64_t>(v);
        s_pref[lane] = s_base + inc - v;
        __syncwarp();
        if (lane == 31) s_base += inc;
      }
      __syncthreads();
      for (int j = warp; j < nt; j += kWarps) {
        const uint64_t t = gs + j;
        const uint32_t n = __ldcg(&L.tile_count[t]);
        const uint32_t* ci = L.cand_idx + t * kTopkTile;
        const float* cv = L.cand_val + t * kTopkTile;
        uint64_t gt_run = s_pref[j] & 0xFFFFFFFFull, eq_run = s_pref[j] >> 32;
        for (uint32_t i0 = 0; i0 < n; i0 += 128) {
          float v[4];
          load4(cv, n, i0, v);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t i = i0 + r * 32 + lane;
            const uint32_t key = abs_key(v[r]);
            const bool gsel = i < n && key > kth, esel = i < n && key == kth;
            const uint32_t gbal = __ballot_sync(0xffffffffu, gsel), ebal = __ballot_sync(0xffffffffu, esel);
            const uint32_t lower = (1u << lane) - 1u;
            const uint64_t gt_before = gt_run + __popc(gbal & lower);
            const uint64_t eq_before = eq_run + __popc(ebal & lower);
            if (gsel || (esel && eq_before < need)) {
              const uint64_t pos = gt_before + (eq_before < need ? eq_before : need);
              const uint32_t j2 = ci[i];
              idx_out[pos] = j2;
              val_out[pos] = v[r];
              if (zero_at) zero_at[j2] = 0.0f;   // acc - TopK(acc)
            }
            gt_run += __popc(gbal);
            eq_run += __popc(ebal);
          }
        }
      }
      __syncthreads();
    }
  }
  mark(c, 7);
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
__global__ void topk_all_kernel(const float* __restrict__ x, const float* __restrict__ g, float alpha,
                                float* __restrict__ xout, float* __restrict__ resid, uint64_t N,
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
template <bool EF, bool RESID>
static cudaError_t launch_fused(const float* x, const float* grad, float alpha, float* x_out, float* residual,
                                uint64_t N, uint64_t k, uint32_t* idx_out, float* val_out, float* zero_at,
                                const TopkLayout& L, cudaStream_t s) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, topk_fused_kernel<EF, RESID>, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
  }
  const uint64_t G = std::max<uint64_t>(1, std::min<uint64_t>({(uint64_t)per_sm * device_sm_count(), L.ntiles,
                                                                (uint64_t)kMaxGrid}));
  TopkLayout Lc = L;
  void* args[] = {(void*)&x,      (void*)&grad,    (void*)&alpha,   (void*)&x_out,   (void*)&residual, (void*)&N,
                  (void*)&k,      (void*)&idx_out, (void*)&val_out, (void*)&zero_at, (void*)&Lc};
  return cudaLaunchCooperativeKernel((const void*)topk_fused_kernel<EF, RESID>, dim3((unsigned)G), dim3(kThreads), args,
                                     0, s);
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
  TopkLayout L = topk_layout(ws, N);
  cudaError_t e;
  {
    SPARCML_PROF("topk", s);
    if (ef) e = launch_fused<true, false>(x, grad, alpha, x_out, nullptr, N, k, idx_out, val_out, x_out, L, s);
    else if (residual && residual != x)
      e = launch_fused<false, true>(x, nullptr, 0.0f, nullptr, residual, N, k, idx_out, val_out, residual, L, s);
    else   // no residual, or residual aliasing x (in place)
      e = launch_fused<false, false>(x, nullptr, 0.0f, nullptr, nullptr, N, k, idx_out, val_out, residual, L, s);
  }
  ++g_launches;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
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
