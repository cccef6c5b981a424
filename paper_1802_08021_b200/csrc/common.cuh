// common.cuh — device helpers and shared layouts of libsparcml (sm_100a).
//
// Nothing here is shared with oracle/ (which is plain C); this header is
// product code only.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sparcml.h"

// Bounds checks compiled in with -DSPARCML_CHECKS (a diagnostics build: a
// failed check traps with cudaErrorAssert; compute-sanitizer is not available
// on this pool, so the test suite runs against this build instead).
#ifdef SPARCML_CHECKS
#include <cassert>
#define SPARCML_CHECK(cond) assert(cond)
#else
#define SPARCML_CHECK(cond) \
  do {                      \
  } while (0)
#endif

namespace sparcml {

constexpr int kMaxRanks = SPARCML_MAX_RANKS;
constexpr int kThreads = 256;            // every tile kernel: 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kMergeItems = 8;           // merge-path items per thread
constexpr int kMergeTile = kThreads * kMergeItems;   // 2048 merged inputs per tile
constexpr int kWin = 1024;               // window kernel: index positions per window
constexpr int kWinPerThread = kWin / kThreads;       // 4
constexpr int kTab = 256;                // window-offset table granularity (index positions)
constexpr int kTabPerWin = kWin / kTab;  // 4
constexpr int kMaxJobs = kMaxRanks / 2;  // batched merges per launch

// ---------------------------------------------------------------------------
// memory-model helpers (PTX)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Spin loops poll with relaxed loads (an acquire load also invalidates the
// SM's L1, which starves the other warps' LSU traffic) and order the data
// reads with one acquire fence after the flag is seen.
__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// acquire-release fences: ordering without the sequentially-consistent drain
// (__threadfence_system() is fence.sc.sys, several microseconds under load)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// relaxed system-scope add (no return value): an arrival after a release fence
__device__ __forceinline__ void red_add_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// streaming (read-once) vector load, no L1 allocation
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// streaming access with an L2 evict-first policy: data touched once (the N-vector
// pass) should not push reusable lines (candidates, control) out of L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float4 ld_stream_f4_ef(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_stream_f4_ef(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

// ---------------------------------------------------------------------------
// warp / block scans (256 threads)
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Exclusive block sum of `x` over kThreads threads; returns the prefix and
// writes the block total to *total.  `scratch` holds kWarps+1 elements.
template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T x, T* scratch, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_inclusive_sum(x);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kWarps ? scratch[lane] : T(0);
    T wi = warp_inclusive_sum(w);
    if (lane < kWarps) scratch[lane] = wi - w;
    if (lane == kWarps - 1) scratch[kWarps] = wi;
  }
  __syncthreads();
  T r = scratch[warp] + inc - x;
  *total = scratch[kWarps];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// ordered tile scan: dynamic tickets + decoupled look-back (single pass)
// ---------------------------------------------------------------------------
struct ScanCounters {
  uint32_t ticket;   // next tile ticket
  uint32_t done;     // blocks finished
  uint32_t gen;      // launch generation (tags TileStatus entries)
  uint32_t pad;
};

struct alignas(32) TileStatus {   // one 32-byte sector each: neighbours' writes never share a sector
  uint64_t word;     // ((gen << 2 | state) << 32) | value; state 1 = aggregate, 2 = inclusive prefix
  uint64_t pad[3];
};

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Called by ONE full warp.  Publishes this tile's aggregate, then looks back
// 32 predecessors at a time (within [first, tile)) until it meets an
// inclusive prefix; publishes its own inclusive prefix and returns the
// exclusive one (to every lane).  `first` is the job's first global tile.
__device__ __forceinline__ uint64_t warp_tile_lookback(TileStatus* st, uint32_t tile, uint32_t first,
                                                       uint64_t agg, uint32_t gen) {
  // (status and value in one 64-bit word, as in block_tile_lookback below)
  const int lane = threadIdx.x & 31;
  const uint64_t tag = (uint64_t)(gen << 2) << 32;
  const uint64_t tmask = (uint64_t)0xFFFFFFFCu << 32;
  SPARCML_CHECK(agg <= 0xFFFFFFFFull);
  if (tile == first) {
    if (lane == 0) st_relaxed_gpu(&st[tile].word, tag | (2ull << 32) | agg);
    return 0;
  }
  if (lane == 0) st_relaxed_gpu(&st[tile].word, tag | (1ull << 32) | agg);
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t t = base - lane;
    uint32_t state = 2;
    uint64_t v = 0;
    if (t >= (int64_t)first) {
      uint64_t w;
      do {
        w = ld_relaxed_gpu(&st[t].word);
      } while ((w & tmask) != tag || (w & (3ull << 32)) == 0);
      state = (uint32_t)(w >> 32) & 3u;
      v = w & 0xFFFFFFFFull;
    }
    const uint32_t im = __ballot_sync(0xffffffffu, state == 2u);
    if (im) {
      const int j = __ffs(im) - 1;   // nearest predecessor holding an inclusive prefix
      excl += warp_sum<uint64_t>(lane <= j ? v : 0ull);
      break;
    }
    excl += warp_sum<uint64_t>(v);
    base -= 32;
  }
  SPARCML_CHECK(excl + agg <= 0xFFFFFFFFull);
  if (lane == 0) st_relaxed_gpu(&st[tile].word, tag | (2ull << 32) | (excl + agg));
  return excl;
}

// Called by the WHOLE block (kThreads).  Like warp_tile_lookback, but every
// thread inspects one predecessor, so a step covers kThreads tiles: tiles taken
// in one wave resolve in one round trip instead of (tile / 32) chained ones.
// Returns the exclusive prefix to every thread.
__device__ __forceinline__ uint64_t block_tile_lookback(TileStatus* st, uint32_t tile, uint32_t first, uint64_t agg,
                                                        uint32_t gen, uint64_t* s_red /* kWarps */,
                                                        int* s_near) {
  // Status and value share one 64-bit word, written and read with single
  // relaxed accesses: a reader that sees the state also sees its value, so no
  // acquire load (each one invalidates the SM's L1) and no fence is needed.
  // Values are per-job output counts: < 2^32 (indices are u32).
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t tag = (uint64_t)(gen << 2) << 32;
  const uint64_t tmask = (uint64_t)0xFFFFFFFCu << 32;
  SPARCML_CHECK(agg <= 0xFFFFFFFFull);
  if (tid == 0) st_relaxed_gpu(&st[tile].word, tag | (1ull << 32) | agg);
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t t = base - tid;
    uint32_t state = 2;   // before the job's first tile: an inclusive prefix of 0
    uint64_t v = 0;
    int j;
    // Polling rounds: each thread reads its predecessor's word once per round; the
    // round ends when every predecessor nearer than the nearest inclusive prefix
    // has published at least its aggregate (a farther one is never waited for).
    bool have = t < (int64_t)first;
    while (true) {
      if (!have) {
        const uint64_t w = ld_relaxed_gpu(&st[t].word);
        if ((w & tmask) == tag && (w & (3ull << 32)) != 0) {
          state = (uint32_t)(w >> 32) & 3u;
          v = w & 0xFFFFFFFFull;
          have = true;
        }
      }
      if (tid == 0) *s_near = kThreads;
      __syncthreads();
      if (have && state == 2u) atomicMin(s_near, tid);
      __syncthreads();
      j = *s_near;
      if (!__syncthreads_or(!have && tid <= j)) break;
    }
    const uint64_t w = warp_sum<uint64_t>(tid <= j ? v : 0ull);
    if (lane == 0) s_red[warp] = w;
    __syncthreads();
    uint64_t sum = 0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) sum += s_red[i];
    excl += sum;
    __syncthreads();   // s_red / s_near are reused by the next step
    if (j < kThreads) break;
    base -= kThreads;
  }
  SPARCML_CHECK(excl + agg <= 0xFFFFFFFFull);
  if (tid == 0) st_relaxed_gpu(&st[tile].word, tag | (2ull << 32) | (excl + agg));
  return excl;
}

// End-of-kernel protocol for ticketed kernels: the last block to finish
// resets the ticket/done counters and bumps the generation.
__device__ __forceinline__ void scan_block_exit(ScanCounters* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t d = atomicAdd(&c->done, 1u);
    if (d == gridDim.x - 1) {
      c->ticket = 0;
      c->done = 0;
      c->gen = c->gen + 1;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11).  Independent implementation from the
// oracle's; equality is checked by the parity tests.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint32_t u4_get(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// QSGD level for |v| with bucket scale `scale`, s levels, uniform word w
// (reading R-16): level = min(s, floor(fl(fl(fl(|v|/scale)*s) + u))).
__device__ __forceinline__ uint32_t qsgd_code(float v, float scale, uint32_t s, int bits, uint32_t w) {
  uint32_t level = 0;
  if (scale != 0.0f) {
    const float u = __fmul_rn(__uint2float_rn(w >> 8), 5.9604644775390625e-8f);  // 2^-24
    const float r = __fdiv_rn(fabsf(v), scale);
    const float t = __fmul_rn(r, __uint2float_rn(s));
    const float f = floorf(__fadd_rn(t, u));
    level = (uint32_t)f;
    if (level > s) level = s;
  }
  const uint32_t neg = (v < 0.0f && level > 0) ? 1u : 0u;
  return (neg << (bits - 1)) | level;
}

__device__ __forceinline__ float qsgd_decode(uint32_t code, float scale, uint32_t s, int bits) {
  const uint32_t level = code & s;
  const float mag = __fmul_rn(__fdiv_rn(__uint2float_rn(level), __uint2float_rn(s)), scale);
  return (code >> (bits - 1)) ? -mag : mag;
}

// ---------------------------------------------------------------------------
// reduction operator (§5; reading R-30): 0 SUM, 1 MAX, 2 MIN
// ---------------------------------------------------------------------------
__device__ __forceinline__ float op_combine(int op, float a, float b) {
  return op == 0 ? __fadd_rn(a, b) : (op == 1 ? fmaxf(a, b) : fminf(a, b));
}
__device__ __forceinline__ float op_neutral(int op) {
  return op == 0 ? 0.0f : (op == 1 ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000));
}
// fp64 values ("single or double precision"): one rounding per combine
__device__ __forceinline__ double op_combine(int op, double a, double b) {
  return op == 0 ? __dadd_rn(a, b) : (op == 1 ? fmax(a, b) : fmin(a, b));
}
template <typename V>
__device__ __forceinline__ V op_neutral_v(int op) { return (V)op_neutral(op); }   // 0, -inf, +inf exact

// four consecutive values to d (16-byte vector stores when aligned)
__device__ __forceinline__ void store4(float* d, const float r[4], int n) {
  if (n == 4 && (reinterpret_cast<uintptr_t>(d) & 15u) == 0) {
    *reinterpret_cast<float4*>(d) = make_float4(r[0], r[1], r[2], r[3]);
  } else {
    for (int i = 0; i < 4 && i < n; ++i) d[i] = r[i];
  }
}
__device__ __forceinline__ void store4(double* d, const double r[4], int n) {
  if (n == 4 && (reinterpret_cast<uintptr_t>(d) & 15u) == 0) {
    reinterpret_cast<double2*>(d)[0] = make_double2(r[0], r[1]);
    reinterpret_cast<double2*>(d)[1] = make_double2(r[2], r[3]);
  } else {
    for (int i = 0; i < 4 && i < n; ++i) d[i] = r[i];
  }
}

// ---------------------------------------------------------------------------
// warp-cooperative searches (32 probes per step)
// ---------------------------------------------------------------------------
// first position p in a[0..n) with a[p] >= key (all lanes return it)
__device__ __forceinline__ uint64_t warp_lower_bound(const uint32_t* __restrict__ a, uint64_t n,
                                                     uint64_t key) {
  const int lane = threadIdx.x & 31;
  uint64_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const uint64_t span = hi - lo;
    const uint64_t p = lo + (span * (uint64_t)(lane + 1)) / 33;
    const bool pred = (uint64_t)a[p] < key;
    const uint32_t b = __ballot_sync(0xffffffffu, pred);
    const int c = __popc(b);
    const uint64_t plo = lo + (span * (uint64_t)c) / 33;          // probe c-1 (+1)
    const uint64_t phi = lo + (span * (uint64_t)(c + 1)) / 33;    // probe c
    const uint64_t nlo = c > 0 ? plo + 1 : lo;
    const uint64_t nhi = c < 32 ? phi : hi;
    lo = nlo;
    hi = nhi;
  }
  const bool pred = (lo + lane < hi) && ((uint64_t)a[lo + lane] < key);
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}

// merge-path split of diagonal d for A-first ties: the number of A elements
// among the first d elements of merge(A, B) where A[i] precedes B[j] iff
// A[i] <= B[j].
__device__ __forceinline__ uint64_t warp_merge_path(const uint32_t* __restrict__ A, uint64_t na,
                                                    const uint32_t* __restrict__ B, uint64_t nb,
                                                    uint64_t d) {
  const int lane = threadIdx.x & 31;
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  while (hi - lo > 32) {
    const uint64_t span = hi - lo;
    const uint64_t p = lo + (span * (uint64_t)(lane + 1)) / 33;
    const bool pred = A[p] <= B[d - 1 - p];
    const uint32_t b = __ballot_sync(0xffffffffu, pred);
    const int c = __popc(b);
    const uint64_t plo = lo + (span * (uint64_t)c) / 33;
    const uint64_t phi = lo + (span * (uint64_t)(c + 1)) / 33;
    const uint64_t nlo = c > 0 ? plo + 1 : lo;
    const uint64_t nhi = c < 32 ? phi : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint64_t p = lo + lane;
  const bool pred = (p < hi) && (A[p] <= B[d - 1 - p]);
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}

constexpr int kMaxStages = 5;   // recursive doubling: log2(16) stages (+1)

// ---------------------------------------------------------------------------
// per-rank control block at offset 0 of the symmetric workspace
// ---------------------------------------------------------------------------
struct alignas(128) Ctrl {
  uint32_t flags[kMaxRanks];      // sparcml_barrier arrivals; slot p written by rank p
  uint32_t epoch;                 // this rank's barrier epoch
  uint32_t seq;                   // collectives this rank has completed
  uint32_t dsar;                  // split-allgather decision of the current call
  uint32_t status;                // device-detected sparcml_status bits
  uint32_t src_done[kMaxRanks];   // split: rank i's slice of call seq+1 is in my receive region i
  uint32_t owner_done[kMaxRanks]; // split: owner j's partition result of call seq+1 is ready
  uint32_t done_ctr[4];           // last-block detection counters (push, stage, concat, owner)
  uint32_t pad0[12];
  uint64_t k_in[kMaxRanks];       // nnz of rank i (written by rank i)
  uint64_t slice_cnt[kMaxRanks];  // pairs rank i pushed into my receive region i
  uint64_t slice_out[kMaxRanks];  // pairs I pushed to owner j
  uint64_t owner_K;               // my partition's reduced pair count
  uint64_t k_sum;                 // sum of k_i
  // recursive doubling, per call parity (seq & 1) and stage t = 1..L: the
  // partner's stream in my receive buffer [par][t] and its flag
  uint32_t rd_flag[2][kMaxStages];
  uint32_t rd_dense[2][kMaxStages];
  uint64_t rd_n[2][kMaxStages];
  uint64_t rd_ksum[2][kMaxStages];
  uint32_t own_dense[2];          // my own stream in cur[b]
  uint64_t own_n[2];
  uint64_t own_ksum[2];
  uint64_t rd_sent[8];            // bytes I pushed for stage t (index t-1)
  uint64_t rd_recv[8];            // bytes I received for stage t
  ScanCounters scan[4];           // ticket counters of the tile kernels
  uint64_t dbg[2][16];            // %globaltimer phase marks (diagnostics): block 0, last block
  uint64_t owner_k[16];           // K_j of owner j's sparse partition result, stored by owner j with its flag
  // sparse allgather: rank i's published stream (count, index range) and its flag
  // sparse allgather, per call parity (seq & 1): rank i's published stream
  // (count, index range, call signature) and its flag.  Two slots: a rank that
  // has finished call s may publish s+1 while a slower peer still pulls s.
  uint64_t ag_n[2][16];
  uint32_t ag_first[2][16], ag_last[2][16];
  uint32_t ag_done[2][16];
  uint64_t ag_sig[2][16];
  uint64_t fold_recv;             // RD folding (R-28): bytes received from my extra rank
  // collective discipline: every rank's call signature (N, op, algo,
  // options) travels with its data; a consumer that sees another signature sets
  // SPARCML_ERR_MISMATCH.  RD stage inputs carry the sender's signature, xor 1
  // once the sender has seen a mismatch (so it propagates to every rank).
  uint64_t sig_in[kMaxRanks];     // split: source i's signature (with its slice)
  uint64_t rd_sig[2][kMaxStages + 2];
  uint64_t slice_rx[2][kMaxRanks];   // split owner: pairs received from source i in call parity p
  uint64_t timeout_ns;            // flag waits give up after this long (SPARCML_ERR_TIMEOUT)
  // fused split-allgather (split_fused_kernel): arrival counters, one 128-byte
  // line per peer -- each of the peer's G CTAs adds 1 per call, so call c is
  // complete at (c + 1) * G (wrap-safe compares) -- this rank's count of fused
  // calls and its CTA ticket
  alignas(128) uint32_t fz_push_arr[kMaxRanks * 32];   // [src * 32]: source src's CTAs whose slices are in my receive region
  uint32_t fz_data_arr[kMaxRanks * 32];                // [j * 32]: owner j's CTAs whose pieces are in my staging area
  alignas(128) uint32_t fz_calls;      // fused calls completed on this rank
  uint32_t fz_ticket;                   // CTAs of this rank done with the current call
};

// ---------------------------------------------------------------------------
// cross-GPU signalling: a flag holds the sequence number of the call that set
// it; waiters compare wrap-safely against seq + 1 of their own call.  A wait
// gives up after ctl->timeout_ns (a dead, hung or mismatched peer), sets
// SPARCML_ERR_TIMEOUT in the rank's status and returns false; once that bit is
// set, later waits of the call return at once, so the call completes (its
// header reports the timeout) instead of hanging the GPU.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool wait_flag_geq(const uint32_t* f, uint32_t target, Ctrl* ctl) {
  // relaxed polling, then one acquire load of the (already satisfied) flag:
  // synchronizes-with the producer's release without a full system fence
  if ((int)(ld_acquire_sys(f) - target) >= 0) return true;
  if (ld_relaxed_gpu_u32(&ctl->status) & (1u << SPARCML_ERR_TIMEOUT)) return false;
  const uint64_t limit = *(volatile uint64_t*)&ctl->timeout_ns;
  const uint64_t t0 = global_ns();
  uint32_t spins = 0;
  while ((int)(ld_relaxed_sys_u32(f) - target) < 0) {
    if (++spins > 64) {   // tight polling first: a flag is usually microseconds away
      __nanosleep(32);
      if ((spins & 255u) == 0 && limit && global_ns() - t0 > limit) {
        atomicOr(&ctl->status, 1u << SPARCML_ERR_TIMEOUT);
        return false;
      }
    }
  }
  (void)ld_acquire_sys(f);
  return true;
}

// signature checks (see Ctrl::sig_in)
__device__ __forceinline__ void check_sig(Ctrl* ctl, uint64_t got, uint64_t mine) {
  if (got != mine) atomicOr(&ctl->status, 1u << SPARCML_ERR_MISMATCH);
}
__device__ __forceinline__ uint64_t sig_out(const Ctrl* ctl, uint64_t mine) {
  return mine ^ ((*(volatile const uint32_t*)&ctl->status >> SPARCML_ERR_MISMATCH) & 1u);
}

__device__ __forceinline__ void dbg_mark(Ctrl* c, int slot) {
  // dbg[0][slot] = %globaltimer (ns) of block 0, dbg[1][slot] = the latest
  // block's.  Compiled in only with -DSPARCML_DEBUG_MARKS (diagnostics).
#ifdef SPARCML_DEBUG_MARKS
  uint64_t t;
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == 0) c->dbg[0][slot] = t;
    atomicMax(reinterpret_cast<unsigned long long*>(&c->dbg[1][slot]), (unsigned long long)t);
  }
#else
  (void)c;
  (void)slot;
#endif
}

}  // namespace sparcml
