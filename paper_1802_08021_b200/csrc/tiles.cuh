// tiles.cuh — the two reduction tiles every collective is built from.
//
//  merge tile  : union-merge-with-sum of two sorted sparse streams over one
//                merge-path tile (§5.1 "Efficient Summation", both sparse,
//                overlapping indices).
//  window tile : coordinate window [wlo, whi) of a P-way reduction whose
//                sources are sparse or dense (§5.1 sparse+dense / dense+dense,
//                P:528-530; the DSAR owner's sparse->dense switch),
//                combined in the canonical rank-order tree (R-8),
//                emitted dense, compacted sparse, or QSGD-encoded (§6).
#pragma once

#include "common.cuh"

namespace sparcml {

// ---------------------------------------------------------------------------
// merge chunk: the union-merge-with-sum of two sorted sparse streams (§5.1
// "Efficient Summation", both sparse, overlapping indices), one
// pass over the inputs.  The merged sequence is cut into chunks of kSpanItems
// * kThreads diagonal positions; a block takes chunks by ticket (so every
// predecessor of a chunk is held by a running or finished block).  Per chunk:
// two warps locate its ends on the merge path in global memory (33-ary
// searches), the A and B windows are staged into shared memory with 16-byte
// loads (one round trip), every thread merges kSpanItems consecutive outputs
// from its own diagonal, a block scan compacts the emitted pairs in place,
// warp 0 publishes the chunk's count and looks back for its offset (decoupled
// look-back), and the block writes the run coalesced.
// ---------------------------------------------------------------------------
#ifndef SPARCML_SPAN_ITEMS
#define SPARCML_SPAN_ITEMS 16   // outputs per thread for 4-byte values (8-byte: half)
#endif
template <typename V>
struct SpanCfg {
  static constexpr int kItems = sizeof(V) == 4 ? SPARCML_SPAN_ITEMS : SPARCML_SPAN_ITEMS / 2;   // outputs per thread
  static constexpr int kChunk = kItems * kThreads;          // diagonal positions per chunk
};

#ifndef SPARCML_MERGE_PAD
#define SPARCML_MERGE_PAD 0   // 1: one pad word per 8 in the staged windows (A/B: 44 vs 42 us unpadded, not kept)
#endif
// Logical index i of a staged window lives at mpad(i): every thread walks its
// own run of ~kItems/2 elements of each window, so lane t reads near 8t -- with
// a pad word per 8 the lanes fall into distinct banks instead of 4.
__device__ __forceinline__ int mpad(int i) { return SPARCML_MERGE_PAD ? i + (i >> 3) : i; }

template <typename V = float>
struct MergeSmem {
  static constexpr int kC = SpanCfg<V>::kChunk;
  static constexpr int kN = SPARCML_MERGE_PAD ? kC + 4 + (kC + 4) / 8 + 1 : kC + 4;   // padded length
  alignas(16) uint32_t ak[kN];   // ak[0] = A[a0-1] (look-behind), ak[1+i] = A[a0+i] (at mpad)
  alignas(16) uint32_t bk[kN];   // bk[i] = B[b0+i], bk[lb] = B[b1] (look-ahead)
  alignas(16) V av[kN];
  alignas(16) V bv[kN];
  uint64_t split[2];
  uint32_t scan[kWarps + 1];
  uint64_t red[kWarps];
  int near;
};

template <typename V = float>
struct MergeOutput {
  uint32_t* idx;
  V* val;
  uint64_t* n;          // receives the output count (written by the last chunk)
  uint32_t* idx2;       // optional mirror (a peer's receive buffer over NVLink)
  V* val2;
  uint64_t* n2;
  int op;               // reduction operator (R-30)
};

__device__ __forceinline__ uint64_t umin64(uint64_t x, uint64_t y) { return x < y ? x : y; }


// n consecutive elements src[s0 ..) -> dst[0 ..) with 4- or 8-byte cp.async
// (LDGSTS, consecutive lanes on consecutive words: coalesced, no alignment
// needed); the caller commits and waits once for all four windows, so the
// block has a single load round trip instead of one per window.
template <typename T>
__device__ __forceinline__ void stage_run_async(T* dst, int dst0, const T* __restrict__ src, uint64_t s0, int n) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte elements");
  for (int i = threadIdx.x; i < n; i += kThreads) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + mpad(dst0 + i));
    if (sizeof(T) == 4)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src + s0 + i) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src + s0 + i) : "memory");
  }
}
__device__ __forceinline__ void stage_async_wait() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// diagnostics (-DSPARCML_DEBUG_MARKS): mk[0][i] = block 0's first chunk reaching
// point i, mk[1][i] = the latest chunk (%globaltimer ns)
__device__ __forceinline__ void merge_mark(uint64_t* mk, int i, bool first) {
#ifdef SPARCML_DEBUG_MARKS
  if (mk && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (first && blockIdx.x == 0) mk[i] = t;
    atomicMax(reinterpret_cast<unsigned long long*>(&mk[12 + i]), (unsigned long long)t);
  }
#else
  (void)mk;
  (void)i;
  (void)first;
#endif
}

#ifndef SPARCML_MERGE_BSEARCH
#define SPARCML_MERGE_BSEARCH 0   // 1: both chunk ends searched by the whole block, 129-ary (A/B: 47 vs 42 us, not kept)
#endif
// Both ends of a chunk on the merge path at once, the whole block: warps 0-3
// search diagonal d0, warps 4-7 diagonal d1, 128 probes per round (129-ary:
// 4 dependent load rounds for 2 x 1.68M pairs instead of 6).  The probe
// predicate A[p] <= B[d-1-p] is monotone in p; c true probes put the split in
// (p_c, p_c+1].  out[g] = the split of diagonal g (A elements before it).
__device__ __forceinline__ void block_merge_path2(const uint32_t* __restrict__ A, uint64_t na,
                                                  const uint32_t* __restrict__ B, uint64_t nb, uint64_t d0,
                                                  uint64_t d1, uint32_t* s_cnt /* kWarps */, uint64_t* out) {
  static_assert(kWarps == 8, "two groups of four warps");
  const int tid = threadIdx.x, warp = tid >> 5, g = warp >> 2, l = tid & 127;
  const uint64_t d = g ? d1 : d0;
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  while (__syncthreads_or(hi - lo > 128)) {   // (also orders s_cnt's reads before the next writes)
    const uint64_t span = hi - lo;
    bool pred = false;
    if (span > 128) {
      const uint64_t p = lo + (span * (uint64_t)(l + 1)) / 129;
      pred = A[p] <= B[d - 1 - p];
    }
    const uint32_t b = __ballot_sync(0xffffffffu, pred);
    if ((tid & 31) == 0) s_cnt[warp] = __popc(b);
    __syncthreads();
    if (span > 128) {
      const int c = (int)(s_cnt[4 * g] + s_cnt[4 * g + 1] + s_cnt[4 * g + 2] + s_cnt[4 * g + 3]);
      const uint64_t plo = lo + (span * (uint64_t)c) / 129;
      const uint64_t phi = lo + (span * (uint64_t)(c + 1)) / 129;
      lo = c > 0 ? plo + 1 : lo;
      hi = c < 128 ? phi : hi;
    }
  }
  const uint64_t p = lo + (uint64_t)l;
  const bool pred = p < hi && A[p] <= B[d - 1 - p];
  const uint32_t b = __ballot_sync(0xffffffffu, pred);
  if ((tid & 31) == 0) s_cnt[warp] = __popc(b);
  __syncthreads();
  if (l == 0) out[g] = lo + s_cnt[4 * g] + s_cnt[4 * g + 1] + s_cnt[4 * g + 2] + s_cnt[4 * g + 3];
}

template <typename V>
__device__ __forceinline__ void merge_chunk(const uint32_t* __restrict__ A, const V* __restrict__ Av, uint64_t na,
                                            const uint32_t* __restrict__ B, const V* __restrict__ Bv, uint64_t nb,
                                            uint64_t d0, MergeSmem<V>& sm, TileStatus* st, uint32_t tile,
                                            uint32_t first, uint32_t gen, const MergeOutput<V>& out,
                                            uint64_t* mk = nullptr, bool mfirst = false) {
  constexpr int kItems = SpanCfg<V>::kItems;
  merge_mark(mk, 0, mfirst);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t total = na + nb;
  const uint64_t d1 = umin64(d0 + SpanCfg<V>::kChunk, total);
  if (SPARCML_MERGE_BSEARCH) {
    block_merge_path2(A, na, B, nb, d0, d1, sm.scan, sm.split);
  } else if (warp == 0) {
    const uint64_t s = warp_merge_path(A, na, B, nb, d0);
    if (lane == 0) sm.split[0] = s;
  } else if (warp == 1) {
    const uint64_t s = warp_merge_path(A, na, B, nb, d1);
    if (lane == 0) sm.split[1] = s;
  }
  __syncthreads();
  merge_mark(mk, 1, mfirst);
  const uint64_t a0 = sm.split[0], a1 = sm.split[1];
  const uint64_t b0 = d0 - a0, b1 = d1 - a1;
  const int la = (int)(a1 - a0), lb = (int)(b1 - b0);
  const bool has_prev_a = a0 > 0;
  const int wb = lb + (b1 < nb ? 1 : 0);   // + the look-ahead B[b1]
  stage_run_async(sm.ak, 1, A, a0, la);
  stage_run_async(sm.bk, 0, B, b0, wb);
  stage_run_async(sm.av, 1, Av, a0, la);
  stage_run_async(sm.bv, 0, Bv, b0, wb);
  if (tid == 0 && has_prev_a) sm.ak[0] = __ldcg(&A[a0 - 1]);
  stage_async_wait();
  __syncthreads();
  merge_mark(mk, 2, mfirst);
  // this thread's outputs: diagonal dt of the chunk
  const int L = la + lb;
  const int dt = min(tid * kItems, L);
  int lo = max(0, dt - lb), hi = min(dt, la);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sm.ak[mpad(mid + 1)] <= sm.bk[mpad(dt - 1 - mid)]) lo = mid + 1; else hi = mid;
  }
  int ia = lo, ib = dt - lo;
  uint32_t ok[kItems];
  V ov[kItems];
  uint32_t emit = 0;
#pragma unroll
  for (int s = 0; s < kItems; ++s) {
    ok[s] = 0;
    ov[s] = V(0);
    if (dt + s < L) {
      const uint32_t ka = ia < la ? sm.ak[mpad(ia + 1)] : 0xFFFFFFFFu;
      const uint32_t kb = ib < wb ? sm.bk[mpad(ib)] : 0xFFFFFFFFu;
      const bool takeA = ib >= lb || (ia < la && ka <= kb);
      if (takeA) {
        V v = sm.av[mpad(ia + 1)];
        // the element following A[ia] in merged order is B[ib] (in the window or the look-ahead)
        if (ib < wb && kb == ka) v = op_combine(out.op, v, sm.bv[mpad(ib)]);
        ok[s] = ka;
        ov[s] = v;
        emit |= 1u << s;
        ++ia;
      } else {
        // a B element equal to the preceding A element was already combined into it
        const bool dup = (ia > 0 || has_prev_a) && sm.ak[mpad(ia)] == kb;
        if (!dup) {
          ok[s] = kb;
          ov[s] = sm.bv[mpad(ib)];
          emit |= 1u << s;
        }
        ++ib;
      }
    }
  }
  uint32_t tile_total;
  const uint32_t my_off = block_exclusive_sum<uint32_t>(__popc(emit), sm.scan, &tile_total);
  // (the scan ended with __syncthreads: the staged windows are consumed)
  merge_mark(mk, 3, mfirst);
  const uint64_t o = block_tile_lookback(st, tile, first, tile_total, gen, sm.red, &sm.near);
  merge_mark(mk, 4, mfirst);
  uint32_t pos = my_off;
#pragma unroll
  for (int s = 0; s < kItems; ++s)
    if (emit & (1u << s)) {
      sm.ak[mpad(pos)] = ok[s];
      sm.av[mpad(pos)] = ov[s];
      ++pos;
    }
  __syncthreads();
  for (uint32_t i = tid; i < tile_total; i += kThreads) {   // coalesced
    SPARCML_CHECK(o + i < total);
    const uint32_t k = sm.ak[mpad(i)];
    const V v = sm.av[mpad(i)];
    out.idx[o + i] = k;
    out.val[o + i] = v;
    if (out.idx2) {
      out.idx2[o + i] = k;
      out.val2[o + i] = v;
    }
  }
  if (tid == 0 && d1 == total) {
    if (out.n) *out.n = o + tile_total;
    if (out.n2) *out.n2 = o + tile_total;
  }
  __syncthreads();   // sm is reused by the block's next chunk
  merge_mark(mk, 5, mfirst);
}

// The whole merge on the grid: chunks by ticket from `ctr` (tickets [t0, t0 +
// nchunks) belong to this merge; status entries are indexed by ticket).
template <typename V>
__device__ void merge_span(const uint32_t* __restrict__ A, const V* __restrict__ Av, uint64_t na,
                           const uint32_t* __restrict__ B, const V* __restrict__ Bv, uint64_t nb, MergeSmem<V>& sm,
                           TileStatus* st, uint32_t gen, const MergeOutput<V>& out, ScanCounters* ctr,
                           uint32_t* s_ticket) {
  const uint64_t total = na + nb;
  const uint32_t nchunks = (uint32_t)((total + SpanCfg<V>::kChunk - 1) / SpanCfg<V>::kChunk);
  while (true) {
    if (threadIdx.x == 0) *s_ticket = atomicAdd(&ctr->ticket, 1u);
    __syncthreads();
    const uint32_t t = *s_ticket;
    __syncthreads();
    if (t >= nchunks) break;
    merge_chunk(A, Av, na, B, Bv, nb, (uint64_t)t * SpanCfg<V>::kChunk, sm, st, t, 0u, gen, out);
  }
  if (total == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    if (out.n) *out.n = 0;
    if (out.n2) *out.n2 = 0;
  }
}

// ---------------------------------------------------------------------------
// window tile
// ---------------------------------------------------------------------------
template <typename V = float>
struct WinSource {
  const uint32_t* idx;   // sparse: global indices
  const V* val;          // sparse values, or dense values indexed by (g - dense_base)
  uint64_t n;            // sparse count
  uint64_t dense_base;   // dense: global index of val[0]
  int dense;
};

enum WinMode : int { WIN_DENSE = 0, WIN_SPARSE = 1, WIN_QUANT = 2 };

template <typename V = float>
struct WinOutput {
  int mode;
  // WIN_DENSE: out[g - dense_base] (and mirror)
  V* dense;
  V* dense2;
  uint64_t dense_base;
  // WIN_SPARSE: compacted (g, v); count to *n (and mirrors)
  uint32_t* idx;
  V* val;
  uint64_t* n;
  uint32_t* idx2;
  V* val2;
  uint64_t* n2;
  // WIN_QUANT (fp32 only): QSGD of the window, positions relative to qbase (= partition start)
  uint8_t* codes;
  float* scales;
  uint64_t qbase;
  int op;               // reduction operator (R-30): combine and neutral fill
  int bits;
  uint32_t bucket;
  uint32_t seed_lo, seed_hi;
};

// Dynamic shared memory: pres[kWin] | vals[nsrc][kWin] | misc
struct WinMisc {
  uint64_t rng[kMaxRanks][2];
  uint64_t epre[kMaxRanks + 1];
  uint32_t scan[kWarps + 1];
  uint64_t excl;
  uint32_t bmax[kWin / 8];
};

__host__ __device__ constexpr size_t win_smem_bytes(int nsrc, size_t vbytes = 4) {
  return sizeof(uint32_t) * kWin + vbytes * kWin * (size_t)nsrc + sizeof(WinMisc);
}

// Canonical tree schedule (reading R-8): post-order list of (dst, src) slot
// pairs for tree(lo, hi) with mid = lo + (hi - lo)/2, result in slot lo.
constexpr int kMaxTreeH = 5;   // ceil(log2(kMaxRanks)) + 1

struct TreeSched {
  uint8_t dst[kMaxRanks];
  uint8_t src[kMaxRanks];
  uint8_t h[kMaxRanks];   // node height (leaves 0): nodes of one height touch disjoint slots
  int n;
  int hmax;
  // per height h (index h-1), per slot: 0 untouched, 1 left child (dst), 2 right child (src)
  uint8_t role[kMaxTreeH][kMaxRanks];
  uint8_t part[kMaxTreeH][kMaxRanks];   // the other child of the same node
};

// QSGD-encode 4 consecutive values v[0..3] at partition-relative position e
// (e % 4 == 0), global counter c0 = qbase + e, valid = how many of the 4 exist.
__device__ __forceinline__ void qsgd_encode4(const float v[4], float scale, uint64_t e, uint64_t c0,
                                             int valid, int bits, uint32_t k0, uint32_t k1,
                                             uint8_t* __restrict__ codes) {
  const uint32_t s = (1u << (bits - 1)) - 1u;
  uint32_t packed = 0;
  // a zero value always codes to 0 (level = floor(0 + u) = 0 since u < 1, R-16):
  // no random word and no division for it, and no Philox block for 4 zeros
  bool any = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) any |= i < valid && v[i] != 0.0f;
  if (any && scale != 0.0f) {
    const uint4 blk = philox4x32_10(make_uint4((uint32_t)(c0 >> 2), (uint32_t)(c0 >> 34), 0u, 0u), k0, k1);
    if ((c0 & 3) == 0) {   // the 4 counters are one Philox block: word i is element i's
      const uint32_t wv[4] = {blk.x, blk.y, blk.z, blk.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t code = (i < valid && v[i] != 0.0f) ? qsgd_code(v[i], scale, s, bits, wv[i]) : 0u;
        packed |= code << (i * bits);
      }
    } else {
      const uint64_t nb = (c0 >> 2) + 1;
      const uint4 blk2 = philox4x32_10(make_uint4((uint32_t)nb, (uint32_t)(nb >> 32), 0u, 0u), k0, k1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t c = c0 + i;
        const uint32_t w = ((c >> 2) == (c0 >> 2)) ? u4_get(blk, (int)(c & 3)) : u4_get(blk2, (int)(c & 3));
        const uint32_t code = (i < valid && v[i] != 0.0f) ? qsgd_code(v[i], scale, s, bits, w) : 0u;
        packed |= code << (i * bits);
      }
    }
  }
  if (valid == 4) {
    if (bits == 2) codes[e / 4] = (uint8_t)packed;
    else if (bits == 4) *reinterpret_cast<uint16_t*>(codes + e / 2) = (uint16_t)packed;
    else *reinterpret_cast<uint32_t*>(codes + e) = packed;
  } else if (valid > 0) {
    const int nbytes = (valid * bits + 7) / 8;
    uint8_t* dst = codes + (e * (uint64_t)bits) / 8;
    for (int b = 0; b < nbytes; ++b) dst[b] = (uint8_t)(packed >> (8 * b));
  }
}

// Whole block (kThreads): QSGD-encode one window of kThreads*4 consecutive
// values, thread t holding positions [e, e+4) (e % 4 == 0, partition-relative)
// with global Philox counter c0 = ctr_base + e.  Buckets of B positions (a
// power of two, 8 <= B <= 1024) start at multiples of B: scale = max |v|
// (P:845-849), one thread per bucket stores it.  bmax: kWin/8 smem words.
__device__ __forceinline__ void qsgd_block_encode(const float r[4], int valid, uint64_t e, uint64_t c0, int bits,
                                                  uint32_t B, uint32_t k0, uint32_t k1, uint8_t* __restrict__ codes,
                                                  float* __restrict__ scales, uint32_t* bmax, int norm = 0) {
  const int tid = threadIdx.x;
  const uint32_t lgB = 31u - __clz(B);    // B is a power of two (8..1024)
  const uint32_t lgt = lgB - 2;           // threads per bucket = B/4 (>= 2)
  const uint32_t seg = lgt < 5 ? (1u << lgt) : 32u;
  float scale;
  if (norm == 0) {   // max |v| (R-16)
    float m = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) m = fmaxf(m, i < valid ? fabsf(r[i]) : 0.0f);
    for (uint32_t o = 1; o < seg; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const int nb_win = (kThreads * 4) >> lgB;
    for (int b = tid; b < nb_win; b += kThreads) bmax[b] = 0u;
    __syncthreads();
    if ((tid & (seg - 1)) == 0) atomicMax(&bmax[tid >> lgt], __float_as_uint(m));
    __syncthreads();
    scale = __uint_as_float(bmax[tid >> lgt]);
  } else {           // l2 (R-31): balanced pairwise tree of fl(v*v) in index order, then sqrt
    float q[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = i < valid ? __fmul_rn(r[i], r[i]) : 0.0f;
    float t = __fadd_rn(__fadd_rn(q[0], q[1]), __fadd_rn(q[2], q[3]));
    for (uint32_t o = 1; o < seg; o <<= 1) t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
    float* wsum = reinterpret_cast<float*>(bmax);   // one partial per warp
    __syncthreads();
    if ((tid & 31) == 0) wsum[tid >> 5] = t;
    __syncthreads();
    if (lgt > 5) {   // buckets spanning 2, 4 or 8 warps: the tree continues over them
      const int nw = 1 << (lgt - 5), w0 = (tid >> 5) & ~(nw - 1);
      float a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = i < nw ? wsum[w0 + i] : 0.0f;
      for (int len = nw; len > 1; len >>= 1)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < len / 2) a[i] = __fadd_rn(a[2 * i], a[2 * i + 1]);
      t = a[0];
    }
    scale = __fsqrt_rn(t);
  }
  if (valid > 0) {
    qsgd_encode4(r, scale, e, c0, valid, bits, k0, k1, codes);
    if ((e & (B - 1)) == 0) scales[e >> lgB] = scale;
  }
}

// Processes window w of [lo, hi): positions [lo + w*kWin, min(lo+(w+1)*kWin, hi)).
// ticket order == window order (required for WIN_SPARSE's look-back).
template <typename V>
__device__ __forceinline__ void window_tile(const WinSource<V>* src, int nsrc, const TreeSched& ts,
                                            uint64_t lo, uint64_t hi, uint32_t w,
                                            unsigned char* smem, TileStatus* st, uint32_t gen,
                                            uint32_t nwin, const WinOutput<V>& out) {
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t* pres = reinterpret_cast<uint32_t*>(smem);
  V* vals = reinterpret_cast<V*>(smem + sizeof(uint32_t) * kWin);
  WinMisc& mc = *reinterpret_cast<WinMisc*>(smem + sizeof(uint32_t) * kWin + sizeof(V) * kWin * nsrc);
  const uint64_t wlo = lo + (uint64_t)w * kWin;
  const uint64_t whi = (wlo + kWin < hi) ? wlo + kWin : hi;
  const int wn = (int)(whi - wlo);

  for (int s = warp; s < nsrc; s += kWarps) {
    if (!src[s].dense) {
      const uint64_t p0 = warp_lower_bound(src[s].idx, src[s].n, wlo);
      const uint64_t p1 = p0 + warp_lower_bound(src[s].idx + p0, src[s].n - p0, whi);
      if ((tid & 31) == 0) {
        mc.rng[s][0] = p0;
        mc.rng[s][1] = p1;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kWinPerThread; ++i) pres[tid + i * kThreads] = 0u;
  __syncthreads();
  // dense sources: their window values; sparse sources: all elements of all
  // sources at once (one load latency for the window, not one per source)
  for (int s = 0; s < nsrc; ++s) {
    if (src[s].dense) {
      const V* dv = src[s].val + (wlo - src[s].dense_base);
      for (int p = tid; p < wn; p += kThreads) vals[s * kWin + p] = dv[p];
      for (int p = tid; p < wn; p += kThreads) atomicOr(&pres[p], 1u << s);
    }
  }
  if (tid == 0) {
    uint64_t run = 0;
    for (int s = 0; s < nsrc; ++s) {
      mc.epre[s] = run;
      if (!src[s].dense) run += mc.rng[s][1] - mc.rng[s][0];
    }
    mc.epre[nsrc] = run;
  }
  __syncthreads();
  for (uint64_t u = tid; u < mc.epre[nsrc]; u += kThreads) {
    int s = 0;
    while (u >= mc.epre[s + 1]) ++s;
    const uint64_t e = mc.rng[s][0] + (u - mc.epre[s]);
    const uint32_t pos = src[s].idx[e] - (uint32_t)wlo;
    if (pos < (uint32_t)wn) {   // guards against unsorted (invalid) input only
      vals[s * kWin + pos] = src[s].val[e];
      atomicOr(&pres[pos], 1u << s);
    }
  }
  __syncthreads();

  // each thread: 4 consecutive positions
  const int p0 = tid * kWinPerThread;
  V r[kWinPerThread];
  uint32_t present = 0;
#pragma unroll
  for (int i = 0; i < kWinPerThread; ++i) {
    const int p = p0 + i;
    uint32_t m = (p < wn) ? pres[p] : 0u;
    for (int q = 0; q < ts.n; ++q) {
      const int d = ts.dst[q], s = ts.src[q];
      if (m & (1u << s)) {
        if (m & (1u << d)) {
          vals[d * kWin + p] = op_combine(out.op, vals[d * kWin + p], vals[s * kWin + p]);
        } else {
          vals[d * kWin + p] = vals[s * kWin + p];
          m |= 1u << d;
        }
      }
    }
    r[i] = (m & 1u) ? vals[p] : op_neutral_v<V>(out.op);
    if (m & 1u) present |= 1u << i;
  }

  if (out.mode == WIN_DENSE) {
    const uint64_t g0 = wlo + p0;
    if (p0 < wn) {
      store4(out.dense + (g0 - out.dense_base), r, wn - p0);
      if (out.dense2) store4(out.dense2 + (g0 - out.dense_base), r, wn - p0);
    }
  } else if (out.mode == WIN_SPARSE) {
    uint32_t total;
    const uint32_t off = block_exclusive_sum<uint32_t>(__popc(present), mc.scan, &total);
    if (warp == 0) {
      const uint64_t e = warp_tile_lookback(st, w, 0, total, gen);
      if ((tid & 31) == 0) mc.excl = e;
    }
    __syncthreads();
    const uint64_t base = mc.excl + off;
    int c = 0;
#pragma unroll
    for (int i = 0; i < kWinPerThread; ++i) {
      if (present & (1u << i)) {
        out.idx[base + c] = (uint32_t)(wlo + p0 + i);
        out.val[base + c] = r[i];
        if (out.idx2) {
          out.idx2[base + c] = (uint32_t)(wlo + p0 + i);
          out.val2[base + c] = r[i];
        }
        ++c;
      }
    }
    if (tid == 0 && w == nwin - 1) {
      if (out.n) *out.n = mc.excl + total;
      if (out.n2) *out.n2 = mc.excl + total;
    }
  } else if constexpr (sizeof(V) == sizeof(float)) {
    const uint64_t e = (wlo - out.qbase) + p0;   // partition-relative position
    const int valid = max(0, min(kWinPerThread, wn - p0));
    qsgd_block_encode(r, valid, e, wlo + p0, out.bits, out.bucket, out.seed_lo, out.seed_hi, out.codes,
                      out.scales, mc.bmax);
  }
  __syncthreads();
}

}  // namespace sparcml
