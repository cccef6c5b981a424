// kernels_topk.cu — top-k sparsification with error feedback (§2.2 P:216-224,
// Algorithm 1) in one HBM pass over the N-vector.
//
//   1 sample   : ~N/256 values (every 256th 32-byte sector) -> 12-bit
//                magnitude histogram -> conservative candidate threshold tau
//                (expected candidates ~ k + 4 sigma + 16 of the sample)
//   2 filter   : the single streaming pass: (EF) acc = fmaf(alpha, g, eps),
//                eps <- acc; candidates |x| >= tau compacted per 4096-tile in
//                index order; 12-bit histogram of candidate magnitudes
//   3 hist2/3  : refine the k-th magnitude on the candidates only (12 + 7 bits)
//   4 compact  : ordered single pass (decoupled look-back) keeping |x| > kth
//                and the lowest-index ties (reading R-18); zero the residual.
// If the sample under-estimates (fewer than k candidates) the filter's last
// block re-filters with tau = 0 (exact; rare slow path, counted in `passes`).
#include <algorithm>
#include <cmath>

#include "kernels.h"

namespace sparcml {

constexpr int kTopkTile = 4096;           // elements per filter tile (16 per thread)
constexpr int kBins = 4096;
constexpr int kBins3 = 128;
constexpr uint64_t kSampleMinN = 1u << 16;   // below this: tau = 0 (all candidates)
constexpr uint32_t kSampleChunks = 16384;    // 8-value chunks sampled

struct TopkCtl {
  uint32_t hist_s[kBins];
  uint32_t hist1[kBins];
  uint32_t hist2[kBins];
  uint32_t hist3[kBins3];
  uint32_t tau_key;
  uint32_t b1, b2, kth;
  uint64_t above1, above2, above_k, need;
  uint32_t done_s, done_f, done_2, done_3;
  uint32_t status, passes;
  uint32_t pad[2];
  ScanCounters scan;
};

struct TopkLayout {
  TopkCtl* ctl;
  uint32_t* tile_count;
  TileStatus* status;
  uint32_t* cand_idx;
  float* cand_val;
  uint64_t ntiles;
};

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static TopkLayout topk_layout(void* ws, uint64_t N) {
  TopkLayout L;
  char* p = static_cast<char*>(ws);
  L.ntiles = (N + kTopkTile - 1) / kTopkTile;
  L.ctl = reinterpret_cast<TopkCtl*>(p);
  p += align256(sizeof(TopkCtl));
  L.tile_count = reinterpret_cast<uint32_t*>(p);
  p += align256(L.ntiles * sizeof(uint32_t));
  L.status = reinterpret_cast<TileStatus*>(p);
  p += align256(L.ntiles * sizeof(TileStatus));
  L.cand_idx = reinterpret_cast<uint32_t*>(p);
  p += align256(L.ntiles * kTopkTile * sizeof(uint32_t));
  L.cand_val = reinterpret_cast<float*>(p);
  return L;
}

size_t topk_workspace_bytes(uint64_t N, uint64_t /*k*/) {
  const uint64_t nt = (N + kTopkTile - 1) / kTopkTile;
  return align256(sizeof(TopkCtl)) + align256(nt * sizeof(uint32_t)) + align256(nt * sizeof(TileStatus)) +
         2 * align256(nt * kTopkTile * sizeof(uint32_t));
}

__device__ __forceinline__ uint32_t abs_key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

// Whole block: find the highest bin b such that (count in bins > b) < target <=
// (count in bins >= b).  Returns b and the count strictly above it in *above.
// If the histogram holds fewer than `target`, returns bin 0 with above =
// total - h[0].
__device__ void find_bin_from_top(const uint32_t* h, int nbins, uint64_t target, uint32_t* bin_out,
                                  uint64_t* above_out) {
  __shared__ uint64_t scan[kWarps + 1];
  __shared__ uint32_t s_bin;
  __shared__ uint64_t s_above;
  const int tid = threadIdx.x;
  const int per = (nbins + kThreads - 1) / kThreads;
  // thread t owns bins [top - (t+1)*per, top - t*per) counted from the top
  const int hiB = nbins - tid * per;
  const int loB = max(0, hiB - per);
  uint64_t local = 0;
  for (int b = loB; b < hiB; ++b) local += h[b];
  if (tid == 0) {
    s_bin = 0;
    s_above = 0;
  }
  uint64_t total;
  const uint64_t before = block_exclusive_sum<uint64_t>(local, scan, &total);
  if (total < target) {
    if (tid == 0) {
      s_bin = 0;
      s_above = total - h[0];
    }
  } else if (before < target && before + local >= target) {
    uint64_t cum = before;
    for (int b = hiB - 1; b >= loB; --b) {
      if (cum + h[b] >= target) {
        s_bin = (uint32_t)b;
        s_above = cum;
        break;
      }
      cum += h[b];
    }
  }
  __syncthreads();
  *bin_out = s_bin;
  *above_out = s_above;
  __syncthreads();
}

__device__ __forceinline__ bool last_block(uint32_t* done) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t d = atomicAdd(done, 1u);
    s_last = (d == gridDim.x - 1);
    if (s_last) *done = 0;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

__device__ __forceinline__ void flush_hist(uint32_t* sh, uint32_t* gh, int nbins) {
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += kThreads) {
    const uint32_t c = sh[b];
    if (c) atomicAdd(&gh[b], c);
  }
}

// ---------------------------------------------------------------- sample ---
template <bool EF>
__global__ void __launch_bounds__(kThreads) topk_sample_kernel(const float* __restrict__ x,
                                                               const float* __restrict__ g, float alpha,
                                                               uint64_t N, uint64_t k, TopkLayout L) {
  __shared__ uint32_t sh[kBins];
  TopkCtl* c = L.ctl;
  if (blockIdx.x == 0 && threadIdx.x == 0) c->status = 0;   // per-call device status
  if (N < kSampleMinN) {
    if (blockIdx.x == 0 && threadIdx.x == 0) c->tau_key = 0;
    return;
  }
  for (int b = threadIdx.x; b < kBins; b += kThreads) sh[b] = 0;
  __syncthreads();
  const uint64_t nchunk = std::min<uint64_t>(kSampleChunks, N / 8);
  for (uint64_t ch = (uint64_t)blockIdx.x * kThreads + threadIdx.x; ch < nchunk;
       ch += (uint64_t)gridDim.x * kThreads) {
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
    for (int i = 0; i < 8; ++i) atomicAdd(&sh[abs_key(v[i]) >> 19], 1u);
  }
  flush_hist(sh, c->hist_s, kBins);
  if (last_block(&c->done_s)) {
    const double S = (double)nchunk * 8.0;
    const double mean = (double)k * S / (double)N;
    const uint64_t target = (uint64_t)ceil(mean + 4.0 * sqrt(mean) + 16.0);
    uint32_t bin;
    uint64_t above;
    find_bin_from_top(c->hist_s, kBins, target, &bin, &above);
    if (threadIdx.x == 0) c->tau_key = bin << 19;
    for (int b = threadIdx.x; b < kBins; b += kThreads) c->hist_s[b] = 0;
  }
}

// ---------------------------------------------------------------- filter ---
// One tile: 16 values per thread (4 coalesced float4 rows).  Candidates are
// written in index order to the tile's region; returns nothing.
template <bool EF, bool RESID, bool STORE>
__device__ __forceinline__ void filter_tile(const float* __restrict__ x, const float* __restrict__ g,
                                            float alpha, float* __restrict__ xout, float* __restrict__ resid,
                                            uint64_t N, uint64_t t, uint32_t tau, const TopkLayout& L,
                                            uint32_t* sh, uint32_t* s_wt, uint32_t* s_status) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t base = t * kTopkTile;
  float v[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t p = base + (uint64_t)(j * kThreads + tid) * 4;
    if (p + 4 <= N) {
      const float4 a = ld_stream_f4(reinterpret_cast<const float4*>(x + p));
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
        const float4 a = ld_stream_f4(reinterpret_cast<const float4*>(g + p));
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
        *reinterpret_cast<float4*>(dst + p) = make_float4(v[j][0], v[j][1], v[j][2], v[j][3]);
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
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t pos = s_wt[32 + j * kWarps + warp] + incl[j] - __popc(flags[j]);
    const uint64_t p = base + (uint64_t)(j * kThreads + tid) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (flags[j] & (1u << q)) {
        L.cand_idx[base + pos] = (uint32_t)(p + q);
        L.cand_val[base + pos] = v[j][q];
        atomicAdd(&sh[abs_key(v[j][q]) >> 19], 1u);
        ++pos;
      }
    }
  }
  if (tid == 0) L.tile_count[t] = s_wt[64];
  __syncthreads();
}

template <bool EF, bool RESID>
__global__ void __launch_bounds__(kThreads) topk_filter_kernel(const float* __restrict__ x,
                                                               const float* __restrict__ g, float alpha,
                                                               float* __restrict__ xout,
                                                               float* __restrict__ resid, uint64_t N,
                                                               uint64_t k, TopkLayout L) {
  __shared__ uint32_t sh[kBins];
  __shared__ uint32_t s_wt[65];
  __shared__ uint32_t s_status;
  TopkCtl* c = L.ctl;
  for (int b = threadIdx.x; b < kBins; b += kThreads) sh[b] = 0;
  if (threadIdx.x == 0) s_status = 0;
  __syncthreads();
  const uint32_t tau = c->tau_key;
  for (uint64_t t = blockIdx.x; t < L.ntiles; t += gridDim.x)
    filter_tile<EF, RESID, EF || RESID>(x, g, alpha, xout, resid, N, t, tau, L, sh, s_wt, &s_status);
  flush_hist(sh, c->hist1, kBins);
  if (threadIdx.x == 0 && s_status) atomicOr(&c->status, 1u);
  if (last_block(&c->done_f)) {
    __shared__ uint64_t s_scan[kWarps + 1];
    uint64_t local = 0;
    for (uint64_t t = threadIdx.x; t < L.ntiles; t += kThreads) local += L.tile_count[t];
    uint64_t C;
    block_exclusive_sum<uint64_t>(local, s_scan, &C);
    uint32_t passes = 1;
    if (C < k) {
      // the sample under-estimated: exact re-filter with tau = 0 (every value
      // is a candidate), reading the stored accumulator in the EF case
      passes = 2;
      for (int b = threadIdx.x; b < kBins; b += kThreads) {
        c->hist1[b] = 0;
        sh[b] = 0;
      }
      __syncthreads();
      const float* src = EF ? xout : x;
      for (uint64_t t = 0; t < L.ntiles; ++t)
        filter_tile<false, false, false>(src, nullptr, 0.0f, nullptr, nullptr, N, t, 0u, L, sh, s_wt, &s_status);
      __syncthreads();
      for (int b = threadIdx.x; b < kBins; b += kThreads) c->hist1[b] = sh[b];
      __syncthreads();
    }
    uint32_t b1;
    uint64_t above1;
    find_bin_from_top(c->hist1, kBins, k, &b1, &above1);
    if (threadIdx.x == 0) {
      c->b1 = b1;
      c->above1 = above1;
      c->passes = passes;
      if (passes == 2) c->tau_key = 0;
    }
    for (int b = threadIdx.x; b < kBins; b += kThreads) c->hist1[b] = 0;
  }
}

// -------------------------------------------------------------- refine -----
template <int LEVEL>
__global__ void __launch_bounds__(kThreads) topk_refine_kernel(uint64_t k, TopkLayout L) {
  constexpr int NB = LEVEL == 2 ? kBins : kBins3;
  __shared__ uint32_t sh[NB];
  TopkCtl* c = L.ctl;
  for (int b = threadIdx.x; b < NB; b += kThreads) sh[b] = 0;
  __syncthreads();
  const uint32_t b1 = c->b1;
  const uint32_t pre = LEVEL == 2 ? b1 : ((b1 << 12) | c->b2);
  const int shift = LEVEL == 2 ? 19 : 7;
  // warp per tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint64_t t = (uint64_t)blockIdx.x * kWarps + warp; t < L.ntiles; t += (uint64_t)gridDim.x * kWarps) {
    const uint32_t n = L.tile_count[t];
    const float* cv = L.cand_val + t * kTopkTile;
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t key = abs_key(cv[i]);
      if ((key >> shift) == pre) atomicAdd(&sh[LEVEL == 2 ? ((key >> 7) & 4095u) : (key & 127u)], 1u);
    }
  }
  flush_hist(sh, LEVEL == 2 ? c->hist2 : c->hist3, NB);
  if (last_block(LEVEL == 2 ? &c->done_2 : &c->done_3)) {
    uint32_t* gh = LEVEL == 2 ? c->hist2 : c->hist3;
    const uint64_t above_prev = LEVEL == 2 ? c->above1 : c->above2;
    uint32_t b;
    uint64_t above;
    find_bin_from_top(gh, NB, k - above_prev, &b, &above);
    if (threadIdx.x == 0) {
      if (LEVEL == 2) {
        c->b2 = b;
        c->above2 = above_prev + above;
      } else {
        c->kth = (c->b1 << 19) | (c->b2 << 7) | b;
        c->above_k = above_prev + above;
        c->need = k - (above_prev + above);
      }
    }
    for (int i = threadIdx.x; i < NB; i += kThreads) gh[i] = 0;
  }
}

// ------------------------------------------------------------- compact -----
// One ticket = a chunk of kCompactTiles filter tiles, processed warp-per-tile.
// Selected = |x| > kth, or |x| == kth among the first `need` in index order
// (ties to the lower index, R-18).  Chunk prefixes (gt count in the low 32
// bits, eq count in the high 32) come from a warp-parallel decoupled look-back.
constexpr int kCompactTiles = 16;

__device__ __forceinline__ void count_tile(const float* cv, uint32_t n, uint32_t kth, uint32_t* gt, uint32_t* eq) {
  const int lane = threadIdx.x & 31;
  uint32_t g = 0, e = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t key = i < n ? abs_key(cv[i]) : 0u;
    g += __popc(__ballot_sync(0xffffffffu, i < n && key > kth));
    e += __popc(__ballot_sync(0xffffffffu, i < n && key == kth));
  }
  *gt = g;
  *eq = e;
}

template <bool ZERO>
__global__ void __launch_bounds__(kThreads) topk_compact_kernel(uint32_t* __restrict__ idx_out,
                                                                float* __restrict__ val_out,
                                                                float* __restrict__ zero_at, TopkLayout L) {
  __shared__ uint32_t s_gt[kCompactTiles], s_eq[kCompactTiles];
  __shared__ uint32_t s_ticket, s_gen;
  __shared__ uint64_t s_excl;
  TopkCtl* c = L.ctl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t kth = c->kth;
  const uint64_t need = c->need;
  if (tid == 0) s_gen = c->scan.gen;
  __syncthreads();
  const uint32_t gen = s_gen;
  const uint32_t nchunks = (uint32_t)((L.ntiles + kCompactTiles - 1) / kCompactTiles);
  while (true) {
    if (tid == 0) s_ticket = atomicAdd(&c->scan.ticket, 1u);
    __syncthreads();
    const uint32_t ch = s_ticket;
    if (ch >= nchunks) break;
    const uint64_t t0 = (uint64_t)ch * kCompactTiles;
    const int nt = (int)(L.ntiles - t0 < (uint64_t)kCompactTiles ? L.ntiles - t0 : (uint64_t)kCompactTiles);
    for (int j = warp; j < nt; j += kWarps) {
      uint32_t g, e;
      count_tile(L.cand_val + (t0 + j) * kTopkTile, L.tile_count[t0 + j], kth, &g, &e);
      if (lane == 0) {
        s_gt[j] = g;
        s_eq[j] = e;
      }
    }
    __syncthreads();
    if (warp == 0) {
      // exclusive scan over the chunk's tiles (lanes = tiles)
      const uint32_t g = lane < nt ? s_gt[lane] : 0u, e = lane < nt ? s_eq[lane] : 0u;
      const uint32_t gi = warp_inclusive_sum<uint32_t>(g), ei = warp_inclusive_sum<uint32_t>(e);
      const uint32_t gtot = __shfl_sync(0xffffffffu, gi, 31), etot = __shfl_sync(0xffffffffu, ei, 31);
      const uint64_t agg = (uint64_t)gtot | ((uint64_t)etot << 32);
      const uint64_t ex = warp_tile_lookback(L.status, ch, 0, agg, gen);
      __syncwarp();
      if (lane < nt) {
        s_gt[lane] = gi - g;
        s_eq[lane] = ei - e;
      }
      if (lane == 0) s_excl = ex;
    }
    __syncthreads();
    const uint64_t ex = s_excl;
    for (int j = warp; j < nt; j += kWarps) {
      const uint64_t t = t0 + j;
      const uint32_t n = L.tile_count[t];
      const uint32_t* ci = L.cand_idx + t * kTopkTile;
      const float* cv = L.cand_val + t * kTopkTile;
      uint64_t gt_run = (ex & 0xFFFFFFFFull) + s_gt[j];
      uint64_t eq_run = (ex >> 32) + s_eq[j];
      for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const float v = i < n ? cv[i] : 0.0f;
        const uint32_t key = abs_key(v);
        const bool g = i < n && key > kth, e = i < n && key == kth;
        const uint32_t gb = __ballot_sync(0xffffffffu, g), eb = __ballot_sync(0xffffffffu, e);
        const uint32_t lower = (1u << lane) - 1u;
        const uint64_t gt_before = gt_run + __popc(gb & lower);
        const uint64_t eq_before = eq_run + __popc(eb & lower);
        if (g || (e && eq_before < need)) {
          const uint64_t pos = gt_before + (eq_before < need ? eq_before : need);
          const uint32_t j2 = ci[i];
          idx_out[pos] = j2;
          val_out[pos] = v;
          if (ZERO) zero_at[j2] = 0.0f;
        }
        gt_run += __popc(gb);
        eq_run += __popc(eb);
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const uint32_t d = atomicAdd(&c->scan.done, 1u);
    if (d == gridDim.x - 1) {
      c->scan.ticket = 0;
      c->scan.done = 0;
      c->scan.gen = c->scan.gen + 1;
      __threadfence();
    }
  }
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
  const unsigned sgrid = N < kSampleMinN ? 1u : 64u;
  const unsigned fgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(L.ntiles, (uint64_t)sms * 4));
  const unsigned rgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((L.ntiles + kWarps - 1) / kWarps, 64));
  const unsigned cgrid = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((L.ntiles + kCompactTiles - 1) / kCompactTiles, (uint64_t)sms * 4));
  {
    SPARCML_PROF("topk_sample", s);
    if (ef) topk_sample_kernel<true><<<sgrid, kThreads, 0, s>>>(x, grad, alpha, N, k, L);
    else topk_sample_kernel<false><<<sgrid, kThreads, 0, s>>>(x, nullptr, 0.0f, N, k, L);
  }
  {
    SPARCML_PROF("topk_filter", s);
    if (ef) topk_filter_kernel<true, false><<<fgrid, kThreads, 0, s>>>(x, grad, alpha, x_out, nullptr, N, k, L);
    else if (residual && residual != x)
      topk_filter_kernel<false, true><<<fgrid, kThreads, 0, s>>>(x, nullptr, 0.0f, nullptr, residual, N, k, L);
    else topk_filter_kernel<false, false><<<fgrid, kThreads, 0, s>>>(x, nullptr, 0.0f, nullptr, nullptr, N, k, L);
  }
  {
    SPARCML_PROF("topk_refine", s);
    topk_refine_kernel<2><<<rgrid, kThreads, 0, s>>>(k, L);
  }
  {
    SPARCML_PROF("topk_refine", s);
    topk_refine_kernel<3><<<rgrid, kThreads, 0, s>>>(k, L);
  }
  float* zero_at = ef ? x_out : residual;
  {
    SPARCML_PROF("topk_compact", s);
    if (zero_at) topk_compact_kernel<true><<<cgrid, kThreads, 0, s>>>(idx_out, val_out, zero_at, L);
    else topk_compact_kernel<false><<<cgrid, kThreads, 0, s>>>(idx_out, val_out, nullptr, L);
  }
  g_launches += 5;
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
