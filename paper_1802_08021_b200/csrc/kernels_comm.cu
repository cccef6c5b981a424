// kernels_comm.cu — collective kernels of the sparse allreduce (§5.3).
//
// Exchange model: every rank owns a symmetric workspace that
// its peers map over NVLink (CUDA IPC).  Data moves by *pushes* fused into
// the producing kernel (split phase, RD stage outputs) and *pulls* fused into
// the consuming kernel (allgather phase); ranks synchronise with a one-warp
// flag barrier.  No host round trip, no NCCL on the data path.
#include <algorithm>

#include "kernels.h"

namespace sparcml {

unsigned long long g_launches = 0;

int device_sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Returns true in the last block to finish (after the counters are reset).
__device__ __forceinline__ bool scan_block_exit_last(ScanCounters* c) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t d = atomicAdd(&c->done, 1u);
    s_last = (d == gridDim.x - 1);
    if (s_last) {
      c->ticket = 0;
      c->done = 0;
      c->gen = c->gen + 1;
      __threadfence();
    }
  }
  __syncthreads();
  return s_last != 0;
}

__device__ __forceinline__ uint32_t next_ticket(ScanCounters* c, uint32_t* s_ticket) {
  if (threadIdx.x == 0) *s_ticket = atomicAdd(&c->ticket, 1u);
  __syncthreads();
  const uint32_t t = *s_ticket;
  return t;
}

__device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// ===========================================================================
// batched union-merge-with-sum (split owner tree levels; stand-alone merge)
// ===========================================================================
__global__ void __launch_bounds__(kThreads) merge_jobs_kernel(MergeJobsArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  MergeSmem& sm = *reinterpret_cast<MergeSmem*>(smem);
  __shared__ uint64_t s_na[kMaxJobs], s_nb[kMaxJobs];
  __shared__ uint32_t s_base[kMaxJobs + 1];
  __shared__ uint32_t s_ticket, s_gen;
  if (a.gate.ptr && *a.gate.ptr != a.gate.value) return;   // grid-uniform
  const int tid = threadIdx.x;
  if (tid < a.njobs) {
    const MergeJob& j = a.job[tid];
    s_na[tid] = j.a_n_dev ? *j.a_n_dev : j.a_n;
    s_nb[tid] = j.b_n_dev ? *j.b_n_dev : j.b_n;
  }
  __syncthreads();
  if (tid == 0) {
    s_base[0] = 0;
    for (int j = 0; j < a.njobs; ++j)
      s_base[j + 1] = s_base[j] + (uint32_t)ceil_div(s_na[j] + s_nb[j], kMergeTile);
    s_gen = a.ctr->gen;
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid < a.njobs && s_na[tid] + s_nb[tid] == 0) {
    const MergeOutput& o = a.job[tid].out;
    if (o.n) *o.n = 0;
    if (o.n2) *o.n2 = 0;
  }
  const uint32_t total = s_base[a.njobs];
  while (true) {
    const uint32_t t = next_ticket(a.ctr, &s_ticket);
    if (t >= total) break;
    int j = 0;
    while (t >= s_base[j + 1]) ++j;
    const MergeJob& jb = a.job[j];
    merge_tile(jb.a_idx, jb.a_val, s_na[j], jb.b_idx, jb.b_val, s_nb[j],
               (uint64_t)(t - s_base[j]) * kMergeTile, sm, a.status, t, s_base[j], s_gen, jb.out);
  }
  scan_block_exit_last(a.ctr);
}

cudaError_t launch_merge_jobs(const MergeJobsArgs& a, int grid_cap, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = sizeof(MergeSmem);
  if (!attr) {
    cudaFuncSetAttribute(merge_jobs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int grid = std::max(1, std::min(grid_cap, device_sm_count() * 4));
  SPARCML_PROF("merge", s);
  merge_jobs_kernel<<<grid, kThreads, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// window kernel (DSAR owner: P sparse slices -> dense / QSGD partition)
// ===========================================================================
__device__ __forceinline__ void resolve_sources(const WinSourceDesc* d, int n, WinSource* s) {
  const int tid = threadIdx.x;
  if (tid < n) {
    s[tid].idx = d[tid].idx;
    s[tid].val = d[tid].val;
    s[tid].n = d[tid].n_dev ? *d[tid].n_dev : d[tid].n;
    s[tid].dense = d[tid].dense_dev ? (int)*d[tid].dense_dev : d[tid].dense;
    s[tid].dense_base = d[tid].dense_base;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) window_kernel(WindowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ WinSource s_src[kMaxRanks];
  __shared__ uint32_t s_ticket, s_gen;
  if (a.gate.ptr && *a.gate.ptr != a.gate.value) return;
  resolve_sources(a.src, a.nsrc, s_src);
  if (threadIdx.x == 0) s_gen = a.ctr->gen;
  __syncthreads();
  const uint32_t nwin = (uint32_t)ceil_div(a.hi - a.lo, kWin);
  if (nwin == 0 && blockIdx.x == 0 && threadIdx.x == 0 && a.out.mode == WIN_SPARSE) {
    if (a.out.n) *a.out.n = 0;
    if (a.out.n2) *a.out.n2 = 0;
  }
  while (true) {
    const uint32_t w = next_ticket(a.ctr, &s_ticket);
    if (w >= nwin) break;
    window_tile(s_src, a.nsrc, a.sched, a.lo, a.hi, w, smem, a.status, s_gen, nwin, a.out);
  }
  scan_block_exit_last(a.ctr);
}

cudaError_t launch_window(const WindowArgs& a, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = win_smem_bytes(a.nsrc);
  if (!attr) {
    cudaFuncSetAttribute(window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)win_smem_bytes(kMaxRanks));
    attr = true;
  }
  const uint64_t nwin = (a.hi - a.lo + kWin - 1) / kWin;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(nwin, (uint64_t)device_sm_count() * 4));
  SPARCML_PROF("window", s);
  window_kernel<<<grid, kThreads, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// recursive doubling (§5.3.1): push of the input, then one kernel per stage
// ===========================================================================
__global__ void __launch_bounds__(kThreads) rd_push_kernel(RdPushArgs a) {
  uint32_t* di = reinterpret_cast<uint32_t*>(a.dst.base);
  float* dv = reinterpret_cast<float*>(a.dst.base + a.dst.val_off);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < a.n; e += stride) {
    const uint32_t x = a.idx[e];
    const float v = a.val[e];
    di[e] = x;
    dv[e] = v;
    if (a.validate) {
      if (x >= a.N || (e + 1 < a.n && a.idx[e + 1] <= x)) atomicOr(&a.ctl->status, 1u << SPARCML_ERR_UNSORTED);
      if (!isfinite(v)) atomicOr(&a.ctl->status, 1u << SPARCML_ERR_NONFINITE);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.dst_n = a.n;
    *a.dst_dense = 0;
    *a.dst_ksum = a.n;
    a.ctl->rd_sent[0] = 8 * a.n;
  }
}

cudaError_t launch_rd_push(const RdPushArgs& a, cudaStream_t s) {
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((a.n + kThreads - 1) / kThreads,
                                                                    (uint64_t)device_sm_count() * 8));
  SPARCML_PROF("rd_push", s);
  rd_push_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

__device__ __forceinline__ void write_header(sparcml_header* h, uint32_t repr, uint64_t nnz, uint64_t N,
                                             uint64_t ksum, uint64_t sent, uint64_t recv, uint32_t algo,
                                             uint32_t status_bits, uint64_t val_offset) {
  uint32_t st = 0;
  for (uint32_t b = 1; b < 32; ++b)
    if (status_bits & (1u << b)) { st = b; break; }
  h->magic = SPARCML_HEADER_MAGIC;
  h->repr = repr;
  h->nnz = nnz;
  h->N = N;
  h->k_sum = ksum;
  h->bytes_sent = sent;
  h->bytes_recv = recv;
  h->algo_used = algo;
  h->status = st;
  h->val_offset = val_offset;
}

__global__ void __launch_bounds__(kThreads) rd_stage_kernel(RdStageArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t s_ticket, s_gen;
  __shared__ WinSource s_src[2];
  const int tid = threadIdx.x;
  const uint64_t an = a.a_n_dev ? *a.a_n_dev : a.a_n;
  const uint32_t ad = a.a_dense_dev ? *a.a_dense_dev : 0u;
  const uint64_t aks = a.a_ksum_dev ? *a.a_ksum_dev : a.a_n;
  const uint64_t bn = *a.b_n_dev;
  const uint32_t bd = *a.b_dense_dev;
  const uint64_t bks = *a.b_ksum_dev;
  // dense switch: upper bound |H1|+|H2| > delta; once dense, dense
  const bool sparse_out = !ad && !bd && (an + bn <= a.delta);
  if (tid == 0) s_gen = a.ctr->gen;
  const uint32_t* b_idx = reinterpret_cast<const uint32_t*>(a.b.base);
  const float* b_val = reinterpret_cast<const float*>(a.b.base + a.b.val_off);
  if (sparse_out) {
    MergeSmem& sm = *reinterpret_cast<MergeSmem*>(smem);
    MergeOutput o;
    o.idx = reinterpret_cast<uint32_t*>(a.o.base);
    o.val = reinterpret_cast<float*>(a.o.base + a.o.val_off);
    o.n = a.o_n_dev;
    o.idx2 = a.m.base ? reinterpret_cast<uint32_t*>(a.m.base) : nullptr;
    o.val2 = a.m.base ? reinterpret_cast<float*>(a.m.base + a.m.val_off) : nullptr;
    o.n2 = a.m.base ? a.m_n_dev : nullptr;
    __syncthreads();
    const uint32_t total = (uint32_t)ceil_div(an + bn, kMergeTile);
    if (total == 0 && blockIdx.x == 0 && tid == 0) {
      if (o.n) *o.n = 0;
      if (o.n2) *o.n2 = 0;
    }
    while (true) {
      const uint32_t t = next_ticket(a.ctr, &s_ticket);
      if (t >= total) break;
      merge_tile(a.a_idx, a.a_val, an, b_idx, b_val, bn, (uint64_t)t * kMergeTile, sm, a.status, t, 0,
                 s_gen, o);
    }
  } else {
    // densify: window over [0, N) with the two streams (sparse or dense)
    if (tid == 0) {
      s_src[0].idx = a.a_idx;
      s_src[0].val = ad ? reinterpret_cast<const float*>(a.a_idx) : a.a_val;
      s_src[0].n = an;
      s_src[0].dense = (int)ad;
      s_src[0].dense_base = 0;
      s_src[1].idx = b_idx;
      s_src[1].val = bd ? reinterpret_cast<const float*>(a.b.base) : b_val;
      s_src[1].n = bn;
      s_src[1].dense = (int)bd;
      s_src[1].dense_base = 0;
    }
    __syncthreads();
    TreeSched ts;
    ts.n = 1;
    ts.dst[0] = 0;
    ts.src[0] = 1;
    WinOutput o = {};
    o.mode = WIN_DENSE;
    o.dense = reinterpret_cast<float*>(a.o.base);
    o.dense2 = a.m.base ? reinterpret_cast<float*>(a.m.base) : nullptr;
    o.dense_base = 0;
    const uint32_t nwin = (uint32_t)ceil_div(a.N, kWin);
    while (true) {
      const uint32_t w = next_ticket(a.ctr, &s_ticket);
      if (w >= nwin) break;
      window_tile(s_src, 2, ts, 0, a.N, w, smem, a.status, s_gen, nwin, o);
    }
  }
  if (scan_block_exit_last(a.ctr) && tid == 0) {
    __threadfence();
    const uint64_t on = sparse_out ? *(volatile uint64_t*)a.o_n_dev : a.N;
    const uint64_t ksum = aks + bks;
    const uint64_t obytes = sparse_out ? 8 * on : 4 * a.N;
    const uint64_t bbytes = bd ? 4 * a.N : 8 * bn;
    *a.o_n_dev = on;
    *a.o_dense_dev = sparse_out ? 0u : 1u;
    *a.o_ksum_dev = ksum;
    Ctrl* ctl = a.ctl;
    ctl->rd_recv[a.stage - 1] = bbytes;
    if (a.m.base) {
      *a.m_n_dev = on;
      *a.m_dense_dev = sparse_out ? 0u : 1u;
      *a.m_ksum_dev = ksum;
      ctl->rd_sent[a.stage] = obytes;
    }
    if (a.last && a.hdr) {
      uint64_t sent = 0, recv = 0;
      for (int t = 0; t < a.stage; ++t) {
        sent += ctl->rd_sent[t];
        recv += ctl->rd_recv[t];
      }
      write_header(a.hdr, sparse_out ? SPARCML_REPR_SPARSE : SPARCML_REPR_DENSE, on, a.N, ksum, sent, recv,
                   SPARCML_SSAR_RECURSIVE_DOUBLE, ctl->status,
                   sparse_out ? (uint64_t)((char*)a.o.base + a.o.val_off - (char*)a.hdr)
                              : (uint64_t)SPARCML_HEADER_BYTES);
      ctl->status = 0;
    }
  }
}

cudaError_t launch_rd_stage(const RdStageArgs& a, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = std::max(sizeof(MergeSmem), win_smem_bytes(2));
  if (!attr) {
    cudaFuncSetAttribute(rd_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int grid = device_sm_count() * 4;
  SPARCML_PROF("rd_stage", s);
  rd_stage_kernel<<<grid, kThreads, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// split phase (§5.3.2): slice by partition, push each slice to its
// owner's receive region over NVLink
// ===========================================================================
constexpr int kPushItems = 4;

__global__ void __launch_bounds__(kThreads) split_push_kernel(PushArgs a) {
  __shared__ uint64_t s_off[kMaxRanks + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // slice boundaries: first position with idx >= b_j (P binary searches)
  for (int j = warp; j <= a.P; j += kWarps) {
    uint64_t o;
    if (j == 0) o = 0;
    else if (j == a.P) o = a.n;
    else o = warp_lower_bound(a.idx, a.n, a.bnd[j]);
    if (lane == 0) s_off[j] = o;
  }
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kThreads * kPushItems;
#pragma unroll
  for (int i = 0; i < kPushItems; ++i) {
    const uint64_t e = base + (uint64_t)i * kThreads + tid;
    if (e < a.n) {
      const uint32_t x = a.idx[e];
      const float v = a.val[e];
      int j = 0;
      while (j + 1 < a.P && e >= s_off[j + 1]) ++j;
      const uint64_t p = e - s_off[j];
      a.dst_idx[j][p] = x;
      a.dst_val[j][p] = v;
      if (a.validate) {
        if (x >= a.N || (e + 1 < a.n && a.idx[e + 1] <= x)) atomicOr(&a.ctl->status, 1u << SPARCML_ERR_UNSORTED);
        if (!isfinite(v)) atomicOr(&a.ctl->status, 1u << SPARCML_ERR_NONFINITE);
      }
    }
  }
  if (blockIdx.x == 0 && tid < a.P) {
    const uint64_t c = s_off[tid + 1] - s_off[tid];
    *a.dst_cnt[tid] = c;
    *a.dst_k[tid] = a.n;
    a.ctl->slice_out[tid] = c;
  }
}

cudaError_t launch_split_push(const PushArgs& a, cudaStream_t s) {
  const uint64_t per = (uint64_t)kThreads * kPushItems;
  const uint64_t blocks = std::max<uint64_t>(1, (a.n + per - 1) / per);
  SPARCML_PROF("split_push", s);
  split_push_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// flag barrier over NVLink (one warp); optional SSAR/DSAR decision after it
// ===========================================================================
struct BarrierDecide {
  int enabled;
  DecideArgs d;
};

__global__ void barrier_kernel(BarrierArgs a, BarrierDecide dec) {
  const int lane = threadIdx.x;
  uint32_t e = 0;
  if (lane == 0) {
    e = a.my->epoch + 1;
    a.my->epoch = e;
    if (a.first_in_call) a.my->call_count = a.my->call_count + 1;
  }
  e = __shfl_sync(0xffffffffu, e, 0);
  __threadfence_system();
  if (!a.loopback && lane < a.P && lane != a.rank) {
    st_release_sys(a.peer_flags[lane], e);
    while ((int)(ld_acquire_sys(&a.my->flags[lane]) - e) < 0) {
    }
  }
  __syncwarp();
  __threadfence_system();
  if (dec.enabled && lane == 0) {
    uint64_t ks = 0;
    for (int i = 0; i < dec.d.P; ++i) ks += *(volatile const uint64_t*)&dec.d.k_in[i];
    uint32_t dsar;
    if (dec.d.algo == SPARCML_DSAR_SPLIT_ALLGATHER) dsar = 1;
    else if (dec.d.algo == SPARCML_SSAR_SPLIT_ALLGATHER) dsar = 0;
    else dsar = ks > dec.d.delta ? 1u : 0u;   // AUTO: upper bound sum k_i > delta (R-5)
    *dec.d.dsar_out = dsar;
    *dec.d.k_sum_out = ks;
  }
}

cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s) {
  BarrierDecide d = {};
  SPARCML_PROF("barrier", s);
  barrier_kernel<<<1, 32, 0, s>>>(a, d);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_barrier_decide(const BarrierArgs& a, const DecideArgs& da, cudaStream_t s) {
  BarrierDecide d;
  d.enabled = 1;
  d.d = da;
  SPARCML_PROF("barrier", s);
  barrier_kernel<<<1, 32, 0, s>>>(a, d);
  ++g_launches;
  return cudaGetLastError();
}

// P == 1: the collective is the identity on the stream (or its densified /
// QSGD-coded form); validate and fill the control block the concat reads.
__global__ void __launch_bounds__(kThreads) p1_prep_kernel(P1PrepArgs a) {
  if (a.validate) {
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < a.n; e += stride) {
      const uint32_t x = a.idx[e];
      if (x >= a.N || (e + 1 < a.n && a.idx[e + 1] <= x)) atomicOr(&a.ctl->status, 1u << SPARCML_ERR_UNSORTED);
      if (!isfinite(a.val[e])) atomicOr(&a.ctl->status, 1u << SPARCML_ERR_NONFINITE);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctrl* c = a.ctl;
    c->k_in[0] = a.n;
    c->slice_cnt[0] = a.n;
    c->slice_out[0] = a.n;
    c->owner_K = a.n;
    c->k_sum = a.n;
    if (a.algo == SPARCML_DSAR_SPLIT_ALLGATHER) c->dsar = 1;
    else if (a.algo == SPARCML_SSAR_SPLIT_ALLGATHER || a.algo == SPARCML_SSAR_RECURSIVE_DOUBLE) c->dsar = 0;
    else c->dsar = a.n > a.delta ? 1u : 0u;
  }
}

cudaError_t launch_p1_prep(const P1PrepArgs& a, cudaStream_t s) {
  const uint64_t blocks = a.validate ? std::max<uint64_t>(1, std::min<uint64_t>((a.n + kThreads - 1) / kThreads, 1024)) : 1;
  SPARCML_PROF("p1_prep", s);
  p1_prep_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// allgather phase (§5.3.2 P:757-758 / §5.3.3): pull every owner's
// partition result over NVLink into the caller's out (concatenation,
// densification, or QSGD decode), then write the header
// ===========================================================================
__global__ void __launch_bounds__(kThreads) concat_kernel(ConcatArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t s_pref[kMaxRanks + 1];
  __shared__ uint32_t s_dsar;
  __shared__ uint32_t s_gen;
  __shared__ WinSource s_src[1];
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_dsar = a.ctl->dsar;
    s_pref[0] = 0;
    for (int j = 0; j < a.P; ++j) s_pref[j + 1] = s_pref[j] + (s_dsar ? 0 : *(volatile const uint64_t*)a.r_n[j]);
    s_gen = a.ctr->gen;
  }
  __syncthreads();
  const bool dsar = s_dsar != 0;
  const uint64_t K = s_pref[a.P];
  float* out_dense = reinterpret_cast<float*>(a.out + SPARCML_HEADER_BYTES);
  uint32_t* out_idx = reinterpret_cast<uint32_t*>(a.out + SPARCML_HEADER_BYTES);
  float* out_val = reinterpret_cast<float*>(a.out + a.val_offset);
  const uint64_t gstride = (uint64_t)gridDim.x * kThreads;
  const uint64_t gtid = (uint64_t)blockIdx.x * kThreads + tid;
  bool dense_result = dsar;
  if (dsar) {
    // decode partitions in groups of 8 (partition-relative)
    uint64_t groups[kMaxRanks + 1];
    groups[0] = 0;
    for (int j = 0; j < a.P; ++j) groups[j + 1] = groups[j] + ceil_div(a.bnd[j + 1] - a.bnd[j], 8);
    const uint32_t s = a.bits ? (1u << (a.bits - 1)) - 1u : 0u;
    for (uint64_t g = gtid; g < groups[a.P]; g += gstride) {
      int j = 0;
      while (g >= groups[j + 1]) ++j;
      const uint64_t e = (g - groups[j]) * 8;
      const uint64_t nj = a.bnd[j + 1] - a.bnd[j];
      const int cnt = (int)((nj - e) < 8 ? (nj - e) : 8);
      float v[8];
      if (a.bits) {
        const uint8_t* cp = a.r_codes[j] + (e * a.bits) / 8;
        uint64_t word = 0;
        const int nbytes = (cnt * a.bits + 7) / 8;
        if (cnt == 8 && a.bits == 4) word = *reinterpret_cast<const uint32_t*>(cp);
        else if (cnt == 8 && a.bits == 8) word = *reinterpret_cast<const unsigned long long*>(cp);
        else if (cnt == 8 && a.bits == 2) word = *reinterpret_cast<const uint16_t*>(cp);
        else
          for (int b = 0; b < nbytes; ++b) word |= (uint64_t)cp[b] << (8 * b);
        const float scale = a.r_scales[j][e / a.bucket];
        const uint32_t mask = (1u << a.bits) - 1u;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = qsgd_decode((uint32_t)(word >> (i * a.bits)) & mask, scale, s, a.bits);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = i < cnt ? a.r_dense[j][e + i] : 0.0f;
      }
      float* d = out_dense + a.bnd[j] + e;
      if (cnt == 8 && ((reinterpret_cast<uintptr_t>(d) & 15u) == 0)) {
        reinterpret_cast<float4*>(d)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(d)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
        for (int i = 0; i < cnt; ++i) d[i] = v[i];
      }
    }
  } else if (K <= a.delta) {
    // sparse concatenation: disjoint ranges, globally sorted by construction
    for (uint64_t o = gtid; o < K; o += gstride) {
      int j = 0;
      while (o >= s_pref[j + 1]) ++j;
      const uint64_t p = o - s_pref[j];
      out_idx[o] = a.r_idx[j][p];
      out_val[o] = a.r_val[j][p];
    }
  } else {
    // K > delta cannot be stored sparse: densify partition by partition
    dense_result = true;
    TreeSched ts;
    ts.n = 0;
    WinOutput wo = {};
    wo.mode = WIN_DENSE;
    wo.dense = out_dense;
    wo.dense_base = 0;
    for (int j = 0; j < a.P; ++j) {
      if (tid == 0) {
        s_src[0].idx = a.r_idx[j];
        s_src[0].val = a.r_val[j];
        s_src[0].n = s_pref[j + 1] - s_pref[j];
        s_src[0].dense = 0;
        s_src[0].dense_base = 0;
      }
      __syncthreads();
      const uint32_t nwin = (uint32_t)ceil_div(a.bnd[j + 1] - a.bnd[j], kWin);
      for (uint32_t w = blockIdx.x; w < nwin; w += gridDim.x)
        window_tile(s_src, 1, ts, a.bnd[j], a.bnd[j + 1], w, smem, a.status, s_gen, nwin, wo);
      __syncthreads();
    }
  }
  if (scan_block_exit_last(a.ctr) && tid == 0) {
    // bytes this rank put on / took off NVLink (pull model counted at the owner)
    uint64_t sent = 0, recv = 0;
    for (int j = 0; j < a.P; ++j) {
      if (j == a.rank) continue;
      sent += 8 * a.ctl->slice_out[j];
      recv += 8 * a.ctl->slice_cnt[j];
    }
    for (int j = 0; j < a.P; ++j) {
      uint64_t w;
      const uint64_t nj = a.bnd[j + 1] - a.bnd[j];
      if (dsar) w = a.bits ? (nj * a.bits + 7) / 8 + 4 * ceil_div(nj, a.bucket) : 4 * nj;
      else w = 8 * (s_pref[j + 1] - s_pref[j]);
      if (j == a.rank) sent += (uint64_t)(a.P - 1) * w;
      else recv += w;
    }
    Ctrl* ctl = a.ctl;
    const uint32_t st = ctl->status;
    write_header(reinterpret_cast<sparcml_header*>(a.out), dense_result ? SPARCML_REPR_DENSE : SPARCML_REPR_SPARSE,
                 dense_result ? a.N : K, a.N, ctl->k_sum, sent, recv,
                 dsar ? SPARCML_DSAR_SPLIT_ALLGATHER : a.algo, st,
                 dense_result ? (uint64_t)SPARCML_HEADER_BYTES : a.val_offset);
    ctl->status = 0;
  }
}

cudaError_t launch_concat(const ConcatArgs& a, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = win_smem_bytes(1);
  if (!attr) {
    cudaFuncSetAttribute(concat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int grid = device_sm_count() * 4;
  SPARCML_PROF("concat", s);
  concat_kernel<<<grid, kThreads, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace sparcml
