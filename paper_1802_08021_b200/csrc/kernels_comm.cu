// kernels_comm.cu — collective kernels of the sparse allreduce (§5.3).
//
// Exchange model: every rank owns a symmetric workspace that
// its peers map over NVLink (CUDA IPC).  Data moves inside the kernels:
// *pushes* fused into the producer (split phase, recursive-doubling stage
// outputs) and *pulls* fused into the consumer (allgather phase).  Phases are
// ordered by per-call flags (the call's sequence number) that the producer's
// last block stores into the consumer's control block with release semantics
// at system scope — no barrier kernels, no host round trip, no NCCL.
#include <algorithm>
#include <cstdlib>
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace sparcml {

unsigned long long g_launches = 0;

int device_sm_count() {
  static int cached_dev = -1, cached = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    cached_dev = dev;
  }
  return cached;
}

__device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Returns true in the last block to finish (after the ticket counters are reset).
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

// Last block to finish.  Every block releases its writes (at system scope when
// `sys`, i.e. when they went to peers over NVLink) before counting itself; the
// last block acquires them before it returns true.
template <bool SYS>
__device__ __forceinline__ bool last_block(uint32_t* ctr) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (SYS) fence_acq_rel_sys(); else fence_acq_rel_gpu();
    const uint32_t d = atomicAdd(ctr, 1u);
    s_last = (d == gridDim.x - 1);
    if (s_last) {
      *ctr = 0;
      if (SYS) fence_acq_rel_sys(); else fence_acq_rel_gpu();
    }
  }
  __syncthreads();
  return s_last != 0;
}

__device__ __forceinline__ uint32_t next_ticket(ScanCounters* c, uint32_t* s_ticket) {
  if (threadIdx.x == 0) *s_ticket = atomicAdd(&c->ticket, 1u);
  __syncthreads();
  return *s_ticket;
}

__device__ __forceinline__ void write_header(sparcml_header* h, uint32_t repr, uint64_t nnz, uint64_t N,
                                             uint64_t ksum, uint64_t sent, uint64_t recv, uint32_t algo,
                                             uint32_t status_bits, uint64_t val_offset,
                                             uint32_t magic = SPARCML_HEADER_MAGIC) {
  uint32_t st = 0;
  for (uint32_t b = 1; b < 32; ++b)
    if (status_bits & (1u << b)) {
      st = b;
      break;
    }
  h->magic = magic;
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

template <typename V>
__device__ __forceinline__ void check_input(const uint32_t* idx, uint64_t e, uint64_t n, uint64_t N, uint32_t x,
                                            V v, uint32_t* status) {
  if (x >= N || (e + 1 < n && idx[e + 1] <= x)) atomicOr(status, 1u << SPARCML_ERR_UNSORTED);
  if (!isfinite(v)) atomicOr(status, 1u << SPARCML_ERR_NONFINITE);
}

// Programmatic dependent launch: the next kernel of the call (owner after the
// push, concat after the owner) may be scheduled as soon as every block of
// this one has started; it orders itself on device flags, not on stream order.
__device__ __forceinline__ void allow_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch with the programmatic-stream-serialization attribute (and cooperative if asked).
static cudaError_t launch_pdl(const void* fn, dim3 grid, size_t smem, cudaStream_t s, void** args, bool coop) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (coop) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// value type traits: header magic, bytes of a (u32, value) pair and of a dense word
template <typename V>
__host__ __device__ constexpr uint32_t hdr_magic() {
  return sizeof(V) == 8 ? SPARCML_HEADER_MAGIC_F64 : SPARCML_HEADER_MAGIC;
}
template <typename V>
__host__ __device__ constexpr uint64_t pair_bytes() { return 4 + sizeof(V); }

// four consecutive values from src (cnt of them valid; 16-byte loads when aligned)
__device__ __forceinline__ void load4(const float* src, int cnt, float v[4]) {
  if (cnt == 4 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
    const float4 q = *reinterpret_cast<const float4*>(src);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = i < cnt ? src[i] : 0.0f;
  }
}
__device__ __forceinline__ void load4(const double* src, int cnt, double v[4]) {
  if (cnt == 4 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
    const double2 q0 = reinterpret_cast<const double2*>(src)[0];
    const double2 q1 = reinterpret_cast<const double2*>(src)[1];
    v[0] = q0.x; v[1] = q0.y; v[2] = q1.x; v[3] = q1.y;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = i < cnt ? src[i] : 0.0;
  }
}

// ===========================================================================
// stand-alone union-merge-with-sum (sparcml_merge_sum)
// ===========================================================================
__global__ void __launch_bounds__(kThreads) merge_jobs_kernel(MergeJobsArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  MergeSmem<float>& sm = *reinterpret_cast<MergeSmem<float>*>(smem);
  constexpr int kC = SpanCfg<float>::kChunk;
  __shared__ uint64_t s_na[kMaxJobs], s_nb[kMaxJobs];
  __shared__ uint32_t s_base[kMaxJobs + 1];
  __shared__ uint32_t s_ticket, s_gen;
  const int tid = threadIdx.x;
  if (tid < a.njobs) {
    const MergeJob& j = a.job[tid];
    s_na[tid] = j.a_n_dev ? *j.a_n_dev : j.a_n;
    s_nb[tid] = j.b_n_dev ? *j.b_n_dev : j.b_n;
  }
  __syncthreads();
  if (tid == 0) {
    s_base[0] = 0;
    for (int j = 0; j < a.njobs; ++j) s_base[j + 1] = s_base[j] + (uint32_t)ceil_div(s_na[j] + s_nb[j], kC);
    s_gen = a.ctr->gen;
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid < a.njobs && s_na[tid] + s_nb[tid] == 0) {
    const MergeOutput<float>& o = a.job[tid].out;
    if (o.n) *o.n = 0;
    if (o.n2) *o.n2 = 0;
  }
  // one ticket space over every job's chunks: ticket t is chunk t - base[j] of
  // job j, its status entry is t, and its look-back stops at base[j]
  uint64_t* mk = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(a.ctr) + 64);   // (diagnostics)
  bool mfirst = true;
  while (true) {
    const uint32_t t = next_ticket(a.ctr, &s_ticket);
    __syncthreads();
    if (t >= s_base[a.njobs]) break;
    int j = 0;
    while (t >= s_base[j + 1]) ++j;
    const MergeJob& jb = a.job[j];
    merge_chunk(jb.a_idx, jb.a_val, s_na[j], jb.b_idx, jb.b_val, s_nb[j], (uint64_t)(t - s_base[j]) * kC, sm,
                a.status, t, s_base[j], s_gen, jb.out, mk, mfirst);
    mfirst = false;
  }
  scan_block_exit_last(a.ctr);
}

cudaError_t launch_merge_jobs(const MergeJobsArgs& a, int grid_cap, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = sizeof(MergeSmem<float>);
  if (!attr) {
    cudaFuncSetAttribute(merge_jobs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int grid = std::max(1, std::min(grid_cap, device_sm_count() * 3));
  SPARCML_PROF("merge", s);
  merge_jobs_kernel<<<grid, kThreads, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}


// ===========================================================================
// recursive doubling (§5.3.1): push of the input, one kernel per stage
// ===========================================================================
template <typename V>
__global__ void __launch_bounds__(kThreads) rd_push_kernel(RdPushArgs a) {
  const uint32_t seq = a.ctl->seq;
  const int par = seq & 1;
  uint32_t* di = reinterpret_cast<uint32_t*>(a.dst[par].base);
  V* dv = reinterpret_cast<V*>(a.dst[par].base + a.dst[par].val_off);
  const V* sv = static_cast<const V*>(a.val);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < a.n; e += stride) {
    const uint32_t x = a.idx[e];
    const V v = sv[e];
    di[e] = x;
    dv[e] = v;
    if (a.validate) check_input(a.idx, e, a.n, a.N, x, v, &a.ctl->status);
  }
  if (last_block<false>(&a.ctl->done_ctr[0]) && threadIdx.x == 0) {   // see split_push_kernel
    a.peer->rd_n[par][a.tgt] = a.n;
    a.peer->rd_dense[par][a.tgt] = 0;
    a.peer->rd_ksum[par][a.tgt] = a.n;
    a.peer->rd_sig[par][a.tgt] = sig_out(a.ctl, a.sig);
    a.ctl->rd_sent[0] = pair_bytes<V>() * a.n;
    st_release_sys(&a.peer->rd_flag[par][a.tgt], seq + 1);
  }
}

cudaError_t launch_rd_push(const RdPushArgs& a, cudaStream_t s) {
  const uint64_t blocks =
      std::max<uint64_t>(1, std::min<uint64_t>((a.n + kThreads - 1) / kThreads, (uint64_t)device_sm_count() * 8));
  SPARCML_PROF("rd_push", s);
  if (a.f64) rd_push_kernel<double><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  else rd_push_kernel<float><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

template <typename V>
__global__ void __launch_bounds__(kThreads) rd_stage_kernel(RdStageArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t s_ticket, s_gen;
  __shared__ WinSource<V> s_src[2];
  const int tid = threadIdx.x;
  Ctrl* ctl = a.ctl;
  const uint32_t seq = ctl->seq;
  const int par = seq & 1, t = a.stage;
  __shared__ uint32_t s_ok;
  if (tid == 0) {   // the partner's stream is in place (or it timed out: then treat it as empty)
    s_ok = wait_flag_geq(&ctl->rd_flag[par][t], seq + 1, ctl) ? 1u : 0u;
    if (s_ok) check_sig(ctl, *(volatile uint64_t*)&ctl->rd_sig[par][t], a.sig);
  }
  __syncthreads();
  const bool got = s_ok != 0;
  const int cp = (t - 1) & 1;   // cur buffer holding my stage t-1 output
  const uint32_t* a_idx = a.a_from_cur ? reinterpret_cast<const uint32_t*>(a.cur[cp].base) : a.a_idx;
  const V* a_val = a.a_from_cur ? reinterpret_cast<const V*>(a.cur[cp].base + a.cur[cp].val_off)
                                : static_cast<const V*>(a.a_val);
  const uint64_t an = a.a_from_cur ? *(volatile uint64_t*)&ctl->own_n[cp] : a.a_n;
  const uint32_t ad = a.a_from_cur ? *(volatile uint32_t*)&ctl->own_dense[cp] : 0u;
  const uint64_t aks = a.a_from_cur ? *(volatile uint64_t*)&ctl->own_ksum[cp] : a.a_n;
  const uint64_t bn = got ? *(volatile uint64_t*)&ctl->rd_n[par][t] : 0;
  const uint32_t bd = got ? *(volatile uint32_t*)&ctl->rd_dense[par][t] : 0u;
  const uint64_t bks = got ? *(volatile uint64_t*)&ctl->rd_ksum[par][t] : 0;
  const StreamBuf b = a.b[par];
  const StreamBuf o = a.o_cur ? a.cur[t & 1] : a.o;
  const StreamBuf m = a.mpeer ? a.m[par] : StreamBuf{nullptr, 0};
  // dense switch: upper bound |H1|+|H2| > delta; once dense, dense
  const bool sparse_out = !ad && !bd && (an + bn <= a.delta);
  if (tid == 0) s_gen = a.ctr->gen;
  const uint32_t* b_idx = reinterpret_cast<const uint32_t*>(b.base);
  const V* b_val = reinterpret_cast<const V*>(b.base + b.val_off);
  if (sparse_out) {
    MergeSmem<V>& sm = *reinterpret_cast<MergeSmem<V>*>(smem);
    MergeOutput<V> mo;
    mo.op = a.op;
    mo.idx = reinterpret_cast<uint32_t*>(o.base);
    mo.val = reinterpret_cast<V*>(o.base + o.val_off);
    mo.n = &ctl->own_n[t & 1];
    mo.idx2 = m.base ? reinterpret_cast<uint32_t*>(m.base) : nullptr;
    mo.val2 = m.base ? reinterpret_cast<V*>(m.base + m.val_off) : nullptr;
    mo.n2 = nullptr;
    __syncthreads();
    merge_span(a_idx, a_val, an, b_idx, b_val, bn, sm, a.status, s_gen, mo, a.ctr, &s_ticket);
  } else {
    // densify: window over [0, N) with the two streams (sparse or dense)
    if (tid == 0) {
      s_src[0].idx = a_idx;
      s_src[0].val = ad ? reinterpret_cast<const V*>(a_idx) : a_val;
      s_src[0].n = an;
      s_src[0].dense = (int)ad;
      s_src[0].dense_base = 0;
      s_src[1].idx = b_idx;
      s_src[1].val = bd ? reinterpret_cast<const V*>(b.base) : b_val;
      s_src[1].n = bn;
      s_src[1].dense = (int)bd;
      s_src[1].dense_base = 0;
    }
    __syncthreads();
    TreeSched ts;
    ts.n = 1;
    ts.dst[0] = 0;
    ts.src[0] = 1;
    WinOutput<V> wo = {};
    wo.mode = WIN_DENSE;
    wo.op = a.op;
    wo.dense = reinterpret_cast<V*>(o.base);
    wo.dense2 = m.base ? reinterpret_cast<V*>(m.base) : nullptr;
    wo.dense_base = 0;
    const uint32_t nwin = (uint32_t)ceil_div(a.N, kWin);
    while (true) {
      const uint32_t w = next_ticket(a.ctr, &s_ticket);
      if (w >= nwin) break;
      window_tile(s_src, 2, ts, 0, a.N, w, smem, a.status, s_gen, nwin, wo);
    }
  }
  // every block completes its (remote) stores at gpu scope before the last
  // block publishes the stream metadata and the partner's flag (system-scope
  // release, cumulative over the blocks it synchronized with)
  __syncthreads();
  if (tid == 0) fence_acq_rel_gpu();
  if (scan_block_exit_last(a.ctr) && tid == 0) {
    fence_acq_rel_gpu();
    const uint64_t on = sparse_out ? *(volatile uint64_t*)&ctl->own_n[t & 1] : a.N;
    const uint64_t ksum = aks + bks;
    const uint64_t obytes = sparse_out ? pair_bytes<V>() * on : sizeof(V) * a.N;
    const uint64_t bbytes = bd ? sizeof(V) * a.N : pair_bytes<V>() * bn;
    ctl->own_n[t & 1] = on;
    ctl->own_dense[t & 1] = sparse_out ? 0u : 1u;
    ctl->own_ksum[t & 1] = ksum;
    if (t > 0) ctl->rd_recv[t - 1] = bbytes;
    else ctl->fold_recv = bbytes;   // the fold step (R-28)
    if (a.mpeer) {
      a.mpeer->rd_n[par][t + 1] = on;
      a.mpeer->rd_dense[par][t + 1] = sparse_out ? 0u : 1u;
      a.mpeer->rd_ksum[par][t + 1] = ksum;
      a.mpeer->rd_sig[par][t + 1] = sig_out(ctl, a.sig);
      ctl->rd_sent[t] = obytes;
      st_release_sys(&a.mpeer->rd_flag[par][t + 1], seq + 1);
    }
    if (a.last && a.hdr) {
      uint64_t sent = 0, recv = 0;
      for (int i = 0; i < t; ++i) {
        sent += ctl->rd_sent[i];
        recv += ctl->rd_recv[i];
      }
      if (a.fold) {   // R-28: the extra rank's stream came in, the result goes out to it
        sent += ctl->rd_sent[t];
        recv += ctl->fold_recv;
      }
      write_header(a.hdr, sparse_out ? SPARCML_REPR_SPARSE : SPARCML_REPR_DENSE, on, a.N, ksum, sent, recv,
                   SPARCML_SSAR_RECURSIVE_DOUBLE, ctl->status,
                   sparse_out ? (uint64_t)((char*)o.base + o.val_off - (char*)a.hdr) : (uint64_t)SPARCML_HEADER_BYTES,
                   hdr_magic<V>());
      ctl->status = 0;
      __threadfence();
      ctl->seq = seq + 1;   // the call is complete on this rank
    }
  }
}

template <typename V>
__global__ void __launch_bounds__(kThreads) rd_unfold_kernel(RdUnfoldArgs a) {
  __shared__ uint64_t s_n;
  __shared__ uint32_t s_d;
  Ctrl* ctl = a.ctl;
  const uint32_t seq = ctl->seq;
  const int par = seq & 1, t = a.stage;
  if (threadIdx.x == 0) {
    const bool ok = wait_flag_geq(&ctl->rd_flag[par][t], seq + 1, ctl);
    if (ok) check_sig(ctl, *(volatile uint64_t*)&ctl->rd_sig[par][t], a.sig);
    s_n = ok ? *(volatile uint64_t*)&ctl->rd_n[par][t] : 0;
    s_d = ok ? *(volatile uint32_t*)&ctl->rd_dense[par][t] : 0u;
  }
  __syncthreads();
  const uint64_t n = s_n;
  const bool dense = s_d != 0;
  const StreamBuf b = a.src[par];
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  if (dense) {
    const V* src = reinterpret_cast<const V*>(b.base);
    V* d = reinterpret_cast<V*>(a.out + SPARCML_HEADER_BYTES);
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < a.N; e += stride) d[e] = __ldcg(&src[e]);
  } else {
    const uint32_t* si = reinterpret_cast<const uint32_t*>(b.base);
    const V* sv = reinterpret_cast<const V*>(b.base + b.val_off);
    uint32_t* oi = reinterpret_cast<uint32_t*>(a.out + SPARCML_HEADER_BYTES);
    V* ov = reinterpret_cast<V*>(a.out + a.val_offset);
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < n; e += stride) {
      oi[e] = __ldcg(&si[e]);
      ov[e] = __ldcg(&sv[e]);
    }
  }
  if (last_block<false>(&ctl->done_ctr[1]) && threadIdx.x == 0) {
    const uint64_t ksum = *(volatile uint64_t*)&ctl->rd_ksum[par][t];
    write_header(reinterpret_cast<sparcml_header*>(a.out), dense ? SPARCML_REPR_DENSE : SPARCML_REPR_SPARSE,
                 dense ? a.N : n, a.N, ksum, ctl->rd_sent[0], dense ? sizeof(V) * a.N : pair_bytes<V>() * n,
                 SPARCML_SSAR_RECURSIVE_DOUBLE, ctl->status, dense ? (uint64_t)SPARCML_HEADER_BYTES : a.val_offset,
                 hdr_magic<V>());
    ctl->status = 0;
    __threadfence();
    ctl->seq = seq + 1;   // the call is complete on this rank
  }
}

cudaError_t launch_rd_unfold(const RdUnfoldArgs& a, cudaStream_t s) {
  SPARCML_PROF("rd_unfold", s);
  if (a.f64) rd_unfold_kernel<double><<<device_sm_count() * 2, kThreads, 0, s>>>(a);
  else rd_unfold_kernel<float><<<device_sm_count() * 2, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

template <typename V>
static size_t rd_stage_smem() {
  static bool attr = false;
  const size_t smem = std::max(sizeof(MergeSmem<V>), win_smem_bytes(2, sizeof(V)));
  if (!attr) {
    cudaFuncSetAttribute(rd_stage_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  return smem;
}

cudaError_t launch_rd_stage(const RdStageArgs& a, cudaStream_t s) {
  const int grid = a.grid > 0 ? std::min(a.grid, device_sm_count() * 4) : device_sm_count() * 4;
  SPARCML_PROF("rd_stage", s);
  if (a.f64) rd_stage_kernel<double><<<grid, kThreads, rd_stage_smem<double>(), s>>>(a);
  else rd_stage_kernel<float><<<grid, kThreads, rd_stage_smem<float>(), s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// split phase (§5.3.2): slice by partition, push every slice and its
// window-offset table into the owner's receive region over NVLink, then flag
// ===========================================================================
#ifndef SPARCML_PUSH_ITEMS
#define SPARCML_PUSH_ITEMS 4
#endif
constexpr int kPushItems = SPARCML_PUSH_ITEMS;   // pairs per thread in the split push

template <typename V>
__global__ void __launch_bounds__(kThreads) split_push_kernel(PushArgs a) {
  __shared__ uint64_t s_off[kMaxRanks + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t base = (uint64_t)blockIdx.x * kThreads * kPushItems;
  const uint64_t last = std::min<uint64_t>(a.n, base + (uint64_t)kThreads * kPushItems) - 1;
  const uint32_t part = (uint32_t)a.bnd[1];   // floor(N/P) (N < 2^32); owner(x) = min(x / part, P - 1)
  allow_dependents();
  // slice boundaries s_off[j] = first position with idx >= b_j: block 0 needs
  // all of them (counts, empty slices), the others only those of the owners
  // their element range touches (usually two searches)
  dbg_mark(a.ctl, 8);
  int j0 = 0, j1 = a.P;
  if (blockIdx.x != 0 && a.n > 0) {
    j0 = (int)std::min<uint32_t>(a.idx[base] / part, a.P - 1);
    j1 = (int)std::min<uint32_t>(a.idx[last] / part, a.P - 1) + 1;
  }
  for (int j = j0 + warp; j <= j1; j += kWarps) {
    uint64_t o;
    if (j == 0) o = 0;
    else if (j == a.P) o = a.n;
    else o = warp_lower_bound(a.idx, a.n, a.bnd[j]);
    if (lane == 0) s_off[j] = o;
  }
  __syncthreads();
  dbg_mark(a.ctl, 9);
#pragma unroll
  for (int i = 0; i < kPushItems; ++i) {
    const uint64_t e = base + (uint64_t)i * kThreads + tid;
    if (e < a.n) {
      const uint32_t x = a.idx[e];
      const V v = static_cast<const V*>(a.val)[e];
      const int j = (int)std::min<uint32_t>(x / part, a.P - 1);
      const uint64_t p = e - s_off[j];
      a.dst_idx[j][p] = x;
      static_cast<V*>(a.dst_val[j])[p] = v;
      // window-offset table (kTab positions per entry): win[w] = first slice
    // position whose table window >= w
      const uint64_t lo = a.bnd[j];
      const int64_t w = (int64_t)((x - lo) / kTab);
      const int64_t wprev = p == 0 ? -1 : (int64_t)((a.idx[e - 1] - lo) / kTab);
      for (int64_t q = wprev + 1; q <= w; ++q) a.dst_win[j][q] = (uint32_t)p;
      if (e + 1 == s_off[j + 1]) {   // last element of the slice
        const int64_t nwin = (int64_t)ceil_div(a.bnd[j + 1] - lo, kTab);
        for (int64_t q = w + 1; q <= nwin; ++q) a.dst_win[j][q] = (uint32_t)(p + 1);
      }
      if (a.validate) check_input(a.idx, e, a.n, a.N, x, v, &a.ctl->status);
    }
  }
  if (blockIdx.x == 0) {
    // empty slices: their whole table is zero
    for (int j = 0; j < a.P; ++j) {
      if (s_off[j + 1] != s_off[j]) continue;
      const uint64_t ntab = ceil_div(a.bnd[j + 1] - a.bnd[j], kTab);
      for (uint64_t q = tid; q <= ntab; q += kThreads) a.dst_win[j][q] = 0;
    }
    if (tid < a.P) {
      const uint64_t c = s_off[tid + 1] - s_off[tid];
      a.peer[tid]->slice_cnt[a.rank] = c;
      a.peer[tid]->k_in[a.rank] = a.n;
      a.peer[tid]->sig_in[a.rank] = sig_out(a.ctl, a.sig);
      a.ctl->slice_out[tid] = c;
    }
  }
  dbg_mark(a.ctl, 10);
  // gpu-scope arrival: a gpu-scope fence completes this block's NVLink stores
  // (they must be visible to every thread of this GPU, which reads the owner's
  // memory at the owner's L2); the last block then releases at system scope
  if (last_block<false>(&a.ctl->done_ctr[0]) && tid < a.P) {
    const uint32_t seq = a.ctl->seq;
    st_release_sys(&a.peer[tid]->src_done[a.rank], seq + 1);
  }
  dbg_mark(a.ctl, 11);
}

cudaError_t launch_split_push(const PushArgs& a, cudaStream_t s) {
  const uint64_t per = (uint64_t)kThreads * kPushItems;
  const uint64_t blocks = std::max<uint64_t>(1, (a.n + per - 1) / per);
  SPARCML_PROF("split_push", s);
  if (a.f64) split_push_kernel<double><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  else split_push_kernel<float><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// owner reduction, SSAR (§5.3.2): the P sorted slices of my
// partition are cut into tiles of ~kMT elements at window-table boundaries
// (table windows are kTab positions, so one tile holds < kMT + P*kTab
// elements).  A tile is staged in shared memory and reduced by the canonical
// tree (R-8) one height at a time: every node of that height merges its two
// sorted runs (left run first on equal keys, fl(left + right)) by rank
// arithmetic -- left element i goes to i + #right<key, right element j to
// j + #left<=key, a right duplicate dies -- then the tile is compacted.  Tiles
// are ticketed; a decoupled look-back gives each its output offset, so the
// partition result is written once, contiguous, with no grid-wide sync.
// ===========================================================================
constexpr int kMT = 512;                  // merge tile capacity beyond one table window
constexpr uint32_t kDead = 0xFFFFFFFFu;   // never an index: N <= 2^32 - 1

__host__ __device__ constexpr int mtile_cap(int P) { return kMT + kTab * P; }
__host__ __device__ constexpr size_t owner_merge_smem_bytes(int P, size_t vbytes = 4) {
  return (8 + 2 * vbytes) * (size_t)mtile_cap(P);   // xk, yk (u32) and xv, yv (values)
}


__device__ __forceinline__ uint32_t sm_lower_bound(const uint32_t* k, uint32_t n, uint32_t x) {
  uint32_t lo = 0;
  while (n > 0) {
    const uint32_t half = n >> 1;
    if (k[lo + half] < x) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

__device__ __forceinline__ uint32_t sm_upper_bound(const uint32_t* k, uint32_t n, uint32_t x) {
  uint32_t lo = 0;
  while (n > 0) {
    const uint32_t half = n >> 1;
    if (k[lo + half] <= x) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

// One lane per source waits for its slice; block 0 records k_sum and the
// algorithm decision (AUTO: sum k_i > delta -> DSAR, reading R-5).
__device__ __forceinline__ bool owner_prologue(const OwnerArgs& a, uint32_t seq, uint64_t* s_ks, uint32_t* s_dsar,
                                               uint64_t* s_sc = nullptr) {
  const int tid = threadIdx.x, P = a.P;
  Ctrl* ctl = a.ctl;
  if (tid < P) {
    bool ok = true;
    if (a.wait) ok = wait_flag_geq(&ctl->src_done[tid], seq + 1, ctl);
    if (ok && a.wait) check_sig(ctl, *(volatile uint64_t*)&ctl->sig_in[tid], a.sig);
    s_ks[tid] = ok ? *(volatile uint64_t*)&ctl->k_in[tid] : 0;   // a timed-out source counts as empty
    const uint64_t sc = ok ? *(volatile uint64_t*)&ctl->slice_cnt[tid] : 0;
    if (s_sc) s_sc[tid] = sc;
    if (blockIdx.x == 0) ctl->slice_rx[seq & 1][tid] = sc;   // this call's counts (the concat's header)
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t ks = 0;
    for (int i = 0; i < P; ++i) ks += s_ks[i];
    uint32_t dsar;
    if (a.host_dsar >= 0) dsar = (uint32_t)a.host_dsar;
    else if (a.algo == SPARCML_DSAR_SPLIT_ALLGATHER) dsar = 1;
    else if (a.algo == SPARCML_SSAR_SPLIT_ALLGATHER) dsar = 0;
    else dsar = ks > a.delta ? 1u : 0u;
    *s_dsar = dsar;
    if (blockIdx.x == 0) {
      ctl->dsar = dsar;
      ctl->k_sum = ks;
    }
  }
  __syncthreads();
  return *s_dsar != 0;
}

// count of run elements k[0..n) below x (x already +1 for "at most"):
// fixed halving steps from TOP (> any run length), branch-free so the
// searches of several elements interleave
template <uint32_t TOP>
__device__ __forceinline__ uint32_t run_rank(const uint32_t* k, uint32_t n, uint32_t x) {
  uint32_t lo = 0;
#pragma unroll
  for (uint32_t step = TOP; step; step >>= 1) {
    const uint32_t c = lo + step;
    if (c <= n && k[c - 1] < x) lo = c;
  }
  return lo;
}

__host__ __device__ constexpr uint32_t pow2_floor(uint32_t x) {
  uint32_t p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

// Shared-memory state of one merge tile.
template <int P>
struct MergeShared {
  uint32_t off[P + 1], len[P], dup[P], ta[P];
  uint8_t role[kMaxTreeH][P], part[kMaxTreeH][P];
  uint32_t wtot[kWarps];
  uint64_t excl;
};

// warp 0, lanes < P hold run lengths: offsets = exclusive prefix (off[P] = total)
template <int P>
__device__ __forceinline__ void runs_prefix(MergeShared<P>& m, uint32_t len) {
  const int lane = threadIdx.x & 31;
  uint32_t x = lane < P ? len : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane < P) {
    m.len[lane] = len;
    m.off[lane] = x - len;
  }
  if (lane == P - 1) m.off[P] = x;
}

// Reduce the elements of table windows [w0, w1) of the block's range (at
// most cap of them; s_c holds table entries, row = window, column = source).
// The result (sorted, unique, canonical-tree sums) is left in xk/xv, or, if
// oi != nullptr, written to oi/ov.  Returns its length.
// The P sources' slices: src.idx(s) / src.val(s) (OwnerArgs' peer arrays, or
// pointers staged in shared memory by the fused kernel).
struct OwnerSrc {
  const OwnerArgs& a;
  __device__ const uint32_t* idx(int s) const { return a.src_idx[s]; }
  __device__ const void* val(int s) const { return a.src_val[s]; }
};

// Stage the runs of table windows [w0, w1) (s_c: table entries, row = window,
// column = source) in shared memory, source-major (run s = slot s), all loads
// in flight; m.off / m.len / m.ta describe the runs.  Returns the element count.
template <int P, typename V, typename Src>
__device__ __forceinline__ uint32_t stage_runs(const Src& src, MergeShared<P>& m, const uint32_t* s_c, int w0, int w1,
                                               uint32_t* xk, V* xv) {
  constexpr int cap = mtile_cap(P);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    uint32_t len = 0;
    if (lane < P) {
      const uint32_t ea = s_c[w0 * P + lane];
      m.ta[lane] = ea;
      m.dup[lane] = 0;
      len = s_c[w1 * P + lane] - ea;
    }
    runs_prefix<P>(m, len);
  }
  __syncthreads();
  const uint32_t n = m.off[P];
  {
    constexpr int Q = (cap + kThreads - 1) / kThreads;
    uint32_t kk[Q];
    V vv[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const uint32_t u = q * kThreads + tid;
      if (u < n) {
        int s = 0;
#pragma unroll
        for (int j = 1; j < P; ++j) s += m.off[j] <= u ? 1 : 0;
        const uint32_t e = m.ta[s] + (u - m.off[s]);
        kk[q] = __ldcg(&src.idx(s)[e]);
        vv[q] = __ldcg(&static_cast<const V*>(src.val(s))[e]);
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const uint32_t u = q * kThreads + tid;
      if (u < n) {
        xk[u] = kk[q];
        xv[u] = vv[q];
      }
    }
  }
  __syncthreads();
  return n;
}

template <int P, typename V, typename Src>
__device__ uint32_t merge_subrange(const Src& src, int hmax_, int op, MergeShared<P>& m, const uint32_t* s_c, int w0,
                                   int w1, uint32_t* oi, V* ov_out, uint32_t* xk, V* xv, uint32_t* yk, V* yv) {
  constexpr int cap = mtile_cap(P);
  constexpr uint32_t kTop = pow2_floor(cap);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // (2) stage the runs
  uint32_t n = stage_runs<P, V>(src, m, s_c, w0, w1, xk, xv);
  // (3) canonical tree, one height per round
  const int hmax = hmax_ > 0 ? hmax_ : 1;
  uint32_t total = n;
  for (int h = 1; h <= hmax; ++h) {
    const uint8_t* role_h = m.role[h - 1];
    const uint8_t* part_h = m.part[h - 1];
    uint32_t off[P];
#pragma unroll
    for (int j = 0; j < P; ++j) off[j] = m.off[j];
    for (uint32_t b0 = 0; b0 < n; b0 += 2 * kThreads) {
      constexpr int Q = 2;
      uint32_t key[Q], rank[Q], qoff[Q], qlen[Q], pos0[Q];
      V v[Q];
      int role[Q], part[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const uint32_t u = b0 + q * kThreads + tid;
        int s = 0;
#pragma unroll
        for (int j = 1; j < P; ++j) s += off[j] <= u ? 1 : 0;
        const bool in = u < n;
        key[q] = in ? xk[u] : 0u;
        v[q] = in ? xv[u] : V(0);
        role[q] = in ? (int)role_h[s] : -1;
        const int pq = part_h[s];
        part[q] = pq;
        qoff[q] = m.off[pq];
        qlen[q] = role[q] > 0 ? m.len[pq] : 0u;
        pos0[q] = role[q] == 2 ? m.off[pq] + (u - off[s]) : u;   // right run lands in the left one's span
      }
#pragma unroll
      for (int q = 0; q < Q; ++q)   // left: #right < key ; right: #left <= key
        rank[q] = run_rank<kTop>(xk + qoff[q], qlen[q], key[q] + (role[q] == 2 ? 1u : 0u));
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (role[q] < 0) continue;
        uint32_t k = key[q];
        V val = v[q];
        const uint32_t pos = pos0[q] + rank[q];
        if (role[q] == 1) {   // left run (lower ranks): first on ties, fl(left + right)
          if (rank[q] < qlen[q] && xk[qoff[q] + rank[q]] == k) val = op_combine(op, val, xv[qoff[q] + rank[q]]);
        } else if (role[q] == 2) {   // right run: a key the left run holds was summed there
          if (rank[q] > 0 && xk[qoff[q] + rank[q] - 1] == k) {
            k = kDead;
            atomicAdd(&m.dup[part[q]], 1u);
          }
        }
        yk[pos] = k;
        yv[pos] = val;
      }
    }
    __syncthreads();
    // (4) compact y -> x (or, after the last height, -> the partition result)
    const uint32_t seg = (uint32_t)ceil_div(n, (uint64_t)kWarps * 32) * 32;
    const uint32_t u0 = warp * seg, u1 = std::min<uint32_t>(n, u0 + seg);
    uint32_t cnt = 0;
    for (uint32_t u = u0 + lane; u < u0 + seg; u += 32) {
      const bool alive = u < u1 && yk[u] != kDead;
      cnt += __popc(__ballot_sync(0xffffffffu, alive));
    }
    if (lane == 0) m.wtot[warp] = cnt;
    uint32_t nl = 0;
    if (warp == 0 && lane < P) {   // merged runs: new lengths
      const int r = role_h[lane];
      nl = r == 1 ? m.len[lane] + m.len[part_h[lane]] - m.dup[lane] : (r == 2 ? 0u : m.len[lane]);
    }
    __syncthreads();
    if (warp == 0) {
      runs_prefix<P>(m, nl);
      if (lane < P) m.dup[lane] = 0;
    }
    __syncthreads();
    total = m.off[P];
    const bool last = h == hmax;
    uint32_t base = 0;
    for (int w = 0; w < warp; ++w) base += m.wtot[w];
    uint32_t* ok = last && oi ? oi : xk;
    V* ov = last && oi ? ov_out : xv;
    for (uint32_t u = u0 + lane; u < u0 + seg; u += 32) {
      const uint32_t key = u < u1 ? yk[u] : kDead;
      const bool alive = key != kDead;
      const uint32_t mm = __ballot_sync(0xffffffffu, alive);
      if (alive) {
        const uint32_t pos = base + __popc(mm & ((1u << lane) - 1u));
        ok[pos] = key;
        ov[pos] = yv[u];
      }
      base += __popc(mm);
    }
    n = total;
    __syncthreads();
  }
  __syncthreads();
  return total;
}

constexpr int kTabSmem = 2048;   // table entries staged per chunk (general path)

// Cooperative: block b reduces table windows [b*W, (b+1)*W) of my partition.
// Common case -- the range holds at most one tile (cap elements): reduced in
// shared memory and kept there across the grid sync.  Otherwise the range is
// cut into pieces (< kMT + one window each) whose results are appended to the
// staging area at the range's input offset.  After one grid sync every block
// knows its output offset (sum of the block counts before it) and writes its
// result contiguously; the last block to finish flags the P sources.
template <int P, typename V>
__global__ void __launch_bounds__(kThreads) owner_merge_kernel(OwnerArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int cap = mtile_cap(P);
  uint32_t* xk = reinterpret_cast<uint32_t*>(smem);
  uint32_t* yk = xk + cap;
  V* xv = reinterpret_cast<V*>(yk + cap);   // 8-byte aligned: cap is even
  V* yv = xv + cap;
  V* const st_val = static_cast<V*>(a.st_val);
  V* const r_val = static_cast<V*>(a.r_val);
  __shared__ MergeShared<P> m;
  __shared__ uint64_t s_ks[kMaxRanks], s_sc[kMaxRanks];
  __shared__ uint32_t s_c[kTabSmem];                 // table entries of the current chunk
  __shared__ uint32_t s_dsar, s_scan[kWarps + 1];
  __shared__ uint64_t s_sum[kWarps + 1], s_excl;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  Ctrl* ctl = a.ctl;
  const uint32_t seq = ctl->seq;
  allow_dependents();
  dbg_mark(ctl, 0);
  for (int q = tid; q < kMaxTreeH * P; q += kThreads) {
    const int hh = q / P, sl = q - hh * P;
    m.role[hh][sl] = a.sched.role[hh][sl];
    m.part[hh][sl] = a.sched.part[hh][sl];
  }
  if (owner_prologue(a, seq, s_ks, &s_dsar, s_sc)) return;   // DSAR: the window kernel reduces
  dbg_mark(ctl, 1);
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t ntab = (uint32_t)ceil_div(a.hi - a.lo, kTab);
  const uint32_t W = (ntab + G - 1) / G;
  const uint32_t wa = std::min<uint32_t>(b * W, ntab), wb = std::min<uint32_t>(wa + W, ntab);
  bool in_smem = true;
  uint32_t cnt = 0;
  uint64_t ibase = 0;
  if (wa < wb) {
    if (tid < P) {
      s_c[tid] = __ldcg(&a.src_win[tid][wa]);
      s_c[P + tid] = __ldcg(&a.src_win[tid][wb]);
    }
    __syncthreads();
    uint32_t tot = 0;
#pragma unroll
    for (int src = 0; src < P; ++src) {
      tot += s_c[P + src] - s_c[src];
      ibase += s_c[src];
    }
    dbg_mark(ctl, 2);
    if (tot <= (uint32_t)cap) {
      cnt = merge_subrange<P, V>(OwnerSrc{a}, a.sched.hmax, a.op, m, s_c, 0, 1, nullptr, nullptr, xk, xv, yk, yv);
    } else {
      in_smem = false;
      const uint32_t wchunk = kTabSmem / P - 1;   // windows per chunk
      for (uint32_t cw = wa; cw < wb; cw += wchunk) {
        const int nw = (int)std::min<uint32_t>(wchunk, wb - cw);
        __syncthreads();
        for (int q = tid; q < (nw + 1) * P; q += kThreads) {
          const int w = q / P, src = q - w * P;
          s_c[q] = __ldcg(&a.src_win[src][cw + w]);
        }
        __syncthreads();
        // greedy maximal pieces of at most cap elements (one window always fits)
        for (int pos = 0; pos < nw;) {
          const int w = pos + tid;
          uint32_t c = 0;
          if (w < nw) {
#pragma unroll
            for (int src = 0; src < P; ++src) c += s_c[(w + 1) * P + src] - s_c[w * P + src];
          }
          uint32_t tsum;
          const uint32_t incl = block_exclusive_sum<uint32_t>(c, s_scan, &tsum) + c;
          const int take = __syncthreads_count(w < nw && incl <= (uint32_t)cap);
          cnt += merge_subrange<P, V>(OwnerSrc{a}, a.sched.hmax, a.op, m, s_c, pos, pos + take, a.st_idx + ibase + cnt, st_val + ibase + cnt, xk,
                                      xv, yk, yv);
          pos += take;
        }
      }
    }
  }
  uint32_t* blk32 = reinterpret_cast<uint32_t*>(a.blk);   // per-block counts (< 2^32 each)
  if (tid == 0) blk32[b] = cnt;
  dbg_mark(ctl, 3);
  grid.sync();
  dbg_mark(ctl, 4);
  // sum of the counts of blocks 0..b-1: one 16-byte load (4 counts) per thread per pass
  uint64_t v = 0;
  for (uint32_t j0 = 4 * tid; j0 < b; j0 += 4 * kThreads) {
    const uint4 q = __ldcg(reinterpret_cast<const uint4*>(blk32 + j0));
    v += (j0 < b ? q.x : 0u) + (j0 + 1 < b ? q.y : 0u) + (j0 + 2 < b ? q.z : 0u) + (j0 + 3 < b ? q.w : 0u);
  }
  uint64_t tot_before;
  block_exclusive_sum<uint64_t>(v, s_sum, &tot_before);
  if (tid == 0) s_excl = tot_before;
  __syncthreads();
  const uint64_t excl = s_excl;
  if (in_smem) {
    for (uint32_t i = tid; i < cnt; i += kThreads) {
      a.r_idx[excl + i] = xk[i];
      r_val[excl + i] = xv[i];
    }
  } else {
    for (uint32_t i = tid; i < cnt; i += kThreads) {
      a.r_idx[excl + i] = __ldcg(&a.st_idx[ibase + i]);
      r_val[excl + i] = __ldcg(&st_val[ibase + i]);
    }
  }
  dbg_mark(ctl, 5);
  // every block's writes are local: the grid barrier orders them (gpu scope)
  // before the last block's system-scope release to the P readers; K travels
  // with the flag, so readers need no remote load
  grid.sync();
  if (b == G - 1 && tid < P) {
    a.peer[tid]->owner_k[a.rank] = excl + cnt;
    st_release_sys(&a.peer[tid]->owner_done[a.rank], seq + 1);
  }
  dbg_mark(ctl, 6);
}

// ===========================================================================
// owner reduction, DSAR (§5.3.3 + §6): one block per 1024-position
// window of my partition (windows never straddle a QSGD bucket, B <= 1024).
// The P sources' elements of the window (located with the window-offset
// tables, or a binary search when P == 1) are scattered into per-source value
// rows, combined per position by the canonical tree (R-8), and the dense
// window is stored, or QSGD-encoded in place (Philox per element, the bucket
// max from a block reduction).  Every output lands at a fixed offset: no
// prefix, no grid-wide sync; the last block to finish flags the P readers.
// ===========================================================================
__host__ __device__ constexpr size_t dsar_smem_bytes(int P, size_t vbytes = 4) {
  return sizeof(uint32_t) * kWin + vbytes * kWin * (size_t)P;
}

// The canonical balanced rank-order tree (R-8): tree(lo, hi) = tree(lo, mid) +
// tree(mid, hi), mid = lo + (hi - lo) / 2, unrolled at compile time for P.
template <int OP, int LO, int HI, typename V>
__device__ __forceinline__ V canonical_tree(const V* v) {
  if constexpr (HI - LO == 1) {
    return v[LO];
  } else {
    constexpr int MID = LO + (HI - LO) / 2;
    return op_combine(OP, canonical_tree<OP, LO, MID>(v), canonical_tree<OP, MID, HI>(v));
  }
}

template <int P, typename V>
__global__ void __launch_bounds__(kThreads) dsar_owner_kernel(OwnerArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  V* vals = reinterpret_cast<V*>(smem + sizeof(uint32_t) * kWin);   // (the first kWin words: unused)
  V* const dense = static_cast<V*>(a.dense);
  __shared__ uint64_t s_ks[kMaxRanks];
  __shared__ uint32_t s_dsar, s_bmax[kWin / 8];
  __shared__ uint32_t s_e0[P], s_pre[P + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Ctrl* ctl = a.ctl;
  const uint32_t seq = ctl->seq;
  allow_dependents();
  if (!owner_prologue(a, seq, s_ks, &s_dsar)) return;   // SSAR: the merge kernel reduces
  const uint64_t nwin = ceil_div(a.hi - a.lo, kWin);
  const uint64_t ntab = ceil_div(a.hi - a.lo, kTab);
  // window w's [first element, count) per source, from the tables; loaded one
  // window ahead (warp 0, lane = source) so the loads overlap the current window
  auto tab_load = [&](uint64_t w, uint32_t& e0, uint32_t& e1) {
    if (lane < P) {
      e0 = __ldcg(&a.src_win[lane][std::min<uint64_t>(w * kTabPerWin, ntab)]);
      e1 = __ldcg(&a.src_win[lane][std::min<uint64_t>((w + 1) * kTabPerWin, ntab)]);
    }
  };
  uint32_t c0 = 0, c1 = 0, n0 = 0, n1 = 0;
  if (warp == 0 && blockIdx.x < nwin) tab_load(blockIdx.x, c0, c1);
  for (uint64_t w = blockIdx.x; w < nwin; w += gridDim.x) {
    const uint64_t wlo = a.lo + w * kWin;
    const int wn = (int)std::min<uint64_t>(kWin, a.hi - wlo);
    // (1) each source's element range in this window (and prefetch the next)
    if (warp == 0) {
      const uint32_t n = lane < P ? c1 - c0 : 0u;
      const uint32_t incl = warp_inclusive_sum<uint32_t>(n);
      if (lane < P) {
        s_e0[lane] = c0;
        s_pre[lane] = incl - n;
      }
      if (lane == P - 1) s_pre[P] = incl;
      if (w + gridDim.x < nwin) tab_load(w + gridDim.x, n0, n1);
    }
    // every source row starts at the operator's neutral element: an absent
    // operand then combines to the other one (fl(x + 0) = x up to the sign of
    // zero, which R-9 compares numerically; max(x, -inf) = x), so the tree
    // below needs no presence bits
    {
      const int p0 = tid * kWinPerThread;
      const V nv = op_neutral_v<V>(a.op);
#pragma unroll
      for (int s = 0; s < P; ++s)
#pragma unroll
        for (int q = 0; q < kWinPerThread; ++q) vals[s * kWin + p0 + q] = nv;
    }
    __syncthreads();
    // (2) scatter, every source at once, 4 element loads in flight per thread
    const uint32_t tot = s_pre[P];
    for (uint32_t b0 = 0; b0 < tot; b0 += 4 * kThreads) {
      uint32_t xi[4];
      V xv[4];
      int xs[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t u = b0 + q * kThreads + tid;
        xs[q] = -1;
        if (u < tot) {
          int s = 0;
#pragma unroll
          for (int j = 1; j < P; ++j) s += s_pre[j] <= u ? 1 : 0;
          const uint32_t e = s_e0[s] + (u - s_pre[s]);
          xi[q] = __ldcg(&a.src_idx[s][e]);
          xv[q] = __ldcg(&static_cast<const V*>(a.src_val[s])[e]);
          xs[q] = s;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (xs[q] >= 0) vals[xs[q] * kWin + (xi[q] - (uint32_t)wlo)] = xv[q];
    }
    __syncthreads();
    // (3) combine per position in the canonical tree order (R-8), in registers
    const int p0 = tid * kWinPerThread;
    V r[kWinPerThread];
#pragma unroll
    for (int q = 0; q < kWinPerThread; ++q) {
      V v[P];
#pragma unroll
      for (int s = 0; s < P; ++s) v[s] = vals[s * kWin + p0 + q];
      r[q] = a.op == 0 ? canonical_tree<0, 0, P>(v) : (a.op == 1 ? canonical_tree<1, 0, P>(v) : canonical_tree<2, 0, P>(v));
    }
    // (4) store: QSGD codes + scales, or dense
    const uint64_t e = w * kWin + p0;   // partition-relative
    bool coded = false;
    if constexpr (sizeof(V) == sizeof(float)) {   // QSGD is defined on fp32 values (the host rejects f64)
      if (a.bits) {
        const int rem = wn - p0;
        const int valid = rem < 0 ? 0 : (rem > 4 ? 4 : rem);
        qsgd_block_encode(r, valid, e, wlo + p0, a.bits, a.bucket, a.seed_lo, a.seed_hi, a.codes, a.scales, s_bmax,
                          a.qnorm);
        coded = true;
      }
    }
    if (!coded && p0 < wn) store4(dense + e, r, wn - p0);
    c0 = n0;
    c1 = n1;
    __syncthreads();   // vals / pres / s_pre reused by the next window
  }
  if (last_block<false>(&ctl->done_ctr[3]) && tid < a.P) st_release_sys(&a.peer[tid]->owner_done[a.rank], seq + 1);
}

using DsarFn = void (*)(OwnerArgs);
template <typename V, int... Ps>
struct DsarTable {
  static DsarFn get(int P) {
    DsarFn f = nullptr;
    ((P == Ps ? (f = dsar_owner_kernel<Ps, V>, 0) : 0), ...);
    return f;
  }
};
static DsarFn dsar_fn(int P, bool f64) {
  return f64 ? DsarTable<double, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::get(P)
             : DsarTable<float, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::get(P);
}

using OwnerMergeFn = void (*)(OwnerArgs);
template <typename V, int... Ps>
struct OwnerMergeTable {
  static OwnerMergeFn get(int P) {
    OwnerMergeFn f = nullptr;
    ((P == Ps ? (f = owner_merge_kernel<Ps, V>, 0) : 0), ...);
    return f;
  }
};
static OwnerMergeFn owner_merge_fn(int P, bool f64) {
  return f64 ? OwnerMergeTable<double, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::get(P)
             : OwnerMergeTable<float, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::get(P);
}

static int owner_merge_occupancy(int P, bool f64) {
  static int cache[2][kMaxRanks + 1] = {{0}};
  if (!cache[f64][P]) {
    const OwnerMergeFn f = owner_merge_fn(P, f64);
    const size_t smem = owner_merge_smem_bytes(P, f64 ? 8 : 4);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, kThreads, smem);
    cache[f64][P] = std::max(1, per);
  }
  return cache[f64][P];
}

cudaError_t launch_owner(const OwnerArgs& a, cudaStream_t s) {
  const bool f64 = a.f64 != 0;
  const size_t vb = f64 ? 8 : 4;
  if (a.host_dsar != 1) {   // SSAR (or undecided: the kernel exits if the device picks DSAR)
#ifndef SPARCML_OWNER_BPSM
#define SPARCML_OWNER_BPSM 0   // 0: as many blocks per SM as fit
#endif
    const int occ = owner_merge_occupancy(a.P, f64);
    const uint64_t G = (uint64_t)(SPARCML_OWNER_BPSM > 0 ? std::min(occ, SPARCML_OWNER_BPSM) : occ) * device_sm_count();
    OwnerArgs ac = a;
    void* args[] = {(void*)&ac};
    SPARCML_PROF("owner", s);
    cudaError_t e =
        a.pdl ? launch_pdl((const void*)owner_merge_fn(a.P, f64), dim3((unsigned)G), owner_merge_smem_bytes(a.P, vb),
                           s, args, true)
              : cudaLaunchCooperativeKernel((const void*)owner_merge_fn(a.P, f64), dim3((unsigned)G), dim3(kThreads),
                                            args, owner_merge_smem_bytes(a.P, vb), s);
    ++g_launches;
    if (e != cudaSuccess) return e;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (a.host_dsar != 0) {   // DSAR (or undecided: the kernel exits if the device picks SSAR)
    const DsarFn f = dsar_fn(a.P, f64);
    const size_t smem = dsar_smem_bytes(a.P, vb);
    static int occ[2][kMaxRanks + 1] = {{0}};
    if (!occ[f64][a.P]) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[f64][a.P], f, kThreads, smem);
      occ[f64][a.P] = std::max(1, occ[f64][a.P]);
    }
    const uint64_t nwin = (a.hi - a.lo + kWin - 1) / kWin;
    const uint64_t G = std::max<uint64_t>(1, std::min<uint64_t>(nwin, (uint64_t)occ[f64][a.P] * device_sm_count()));
    SPARCML_PROF("owner_dsar", s);
    if (a.pdl) {
      OwnerArgs ac = a;
      void* args[] = {(void*)&ac};
      const cudaError_t e = launch_pdl((const void*)f, dim3((unsigned)G), smem, s, args, false);
      if (e != cudaSuccess) return e;
    } else {
      f<<<(unsigned)G, kThreads, smem, s>>>(a);
    }
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}


// ===========================================================================
// fused split-allgather, SSAR (§5.3.2): ONE cooperative kernel per
// rank runs the three phases, ordered by arrival counters instead of kernel
// boundaries (the separate push / owner / concat kernels spent ~40% of the
// call in launch gaps and grid-wide syncs, profiles/r01_timeline_p4.log):
//  1. split: CTA b pushes its share of my stream, sliced by partition, into
//     every owner's receive region (+ window-offset tables), then adds one
//     arrival at each owner;
//  2. owner: once all G*P source CTAs have arrived, CTA b reduces its table
//     windows of my partition (canonical tree, R-8) into shared memory and
//     pushes the piece straight into every reader's staging area at a slot
//     that needs no prefix -- slot_b = ceil4(min(inputs before b, positions
//     before b)) + 4b is monotone with room for the piece -- plus a record
//     {count, slot}, then adds one arrival at each reader;
//  3. allgather: once all G*P owner CTAs have arrived, CTA b reads the P*G
//     records, and copies the pieces (j, b) of every owner j from its local
//     staging to its exact place in out (sparse concatenation), or densifies
//     them when K > delta; the last CTA writes the header.
// A rank starts call s+1 only after every owner's call-s pieces reached it,
// i.e. after every owner finished reading its receive regions: no buffer is
// reused early, and the counters need no reset.
// ===========================================================================
struct SmemSrc {
  const uint32_t* const* i;
  const void* const* v;
  __device__ const uint32_t* idx(int s) const { return i[s]; }
  __device__ const void* val(int s) const { return v[s]; }
};

__device__ __forceinline__ Ctrl* fz_ctl(const FusedArgs& a, int r) { return reinterpret_cast<Ctrl*>(a.base[r]); }
__device__ __forceinline__ uint32_t* fz_stage_idx(const FusedArgs& a, int reader, int owner) {
  return reinterpret_cast<uint32_t*>(a.base[reader] + a.fz_off + (uint64_t)owner * a.fz_bytes);
}
template <typename V>
__device__ __forceinline__ V* fz_stage_val(const FusedArgs& a, int reader, int owner) {
  return reinterpret_cast<V*>(a.base[reader] + a.fz_off + (uint64_t)owner * a.fz_bytes + 4 * a.fz_cap);
}
__device__ __forceinline__ uint64_t* fz_rec(const FusedArgs& a, int reader) {
  return reinterpret_cast<uint64_t*>(a.base[reader] + a.rec_off);
}
// table windows [wa, wb) of partition j reduced by CTA b (every rank computes the same split)
__device__ __forceinline__ void fz_range(const FusedArgs& a, int j, uint32_t b, uint32_t& wa, uint32_t& wb) {
  const uint32_t ntab = (uint32_t)ceil_div(a.bnd[j + 1] - a.bnd[j], kTab);
  const uint32_t W = (ntab + a.G - 1) / a.G;
  wa = std::min<uint32_t>(b * W, ntab);
  wb = std::min<uint32_t>(wa + W, ntab);
}

// Canonical tree (R-8) over the runs that hold a key: tree(lo, hi) =
// tree(lo, mid) (+) tree(mid, hi), a subtree without the key contributing
// nothing (the pairwise merges of the oracle skip absent operands).
template <int OP, int LO, int HI, typename V>
__device__ __forceinline__ bool present_tree(const V* v, uint32_t mask, V& out) {
  if constexpr (HI - LO == 1) {
    out = v[LO];
    return (mask >> LO) & 1u;
  } else {
    constexpr int MID = LO + (HI - LO) / 2;
    V a, b;
    const bool pa = present_tree<OP, LO, MID>(v, mask, a);
    const bool pb = present_tree<OP, MID, HI>(v, mask, b);
    out = (pa && pb) ? op_combine(OP, a, b) : (pa ? a : b);
    return pa || pb;
  }
}

// P-way merge of the staged runs (xk / xv, described by m) by rank, for a
// range that fits in shared memory.  Element (k, s) LEADS key k iff no run
// t < s holds k.  A leader's output slot is the number of leaders with a
// smaller key: sum over runs t of lower_bound_t(k) minus the non-leaders
// among those (a per-run prefix count, pre[]).  It combines the values of the
// runs holding k with present_tree.  Two passes of P-way searches, one block
// scan; no per-height merges.  Output (sorted, unique) to yk / yv; returns
// its length.  pre[] holds n + 1 entries.
// lower_bound of key x in each of the P runs, the P binary searches interleaved
// step by step (independent shared-memory chains, no branches)
template <int P, uint32_t TOP>
__device__ __forceinline__ void runs_lower_bound(const uint32_t* xk, const uint32_t (&off)[P],
                                                 const uint32_t (&len)[P], uint32_t x, uint32_t (&pos)[P]) {
#pragma unroll
  for (int t = 0; t < P; ++t) pos[t] = 0;
#pragma unroll
  for (uint32_t step = TOP; step; step >>= 1) {
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const uint32_t c = pos[t] + step;
      if (c <= len[t] && xk[off[t] + c - 1] < x) pos[t] = c;
    }
  }
}

template <int P, typename V>
__device__ uint32_t rank_merge(const MergeShared<P>& m, uint32_t n, const uint32_t* xk, const V* xv, uint32_t* pre,
                               uint32_t* yk, V* yv, int op, uint32_t* s_scan, Ctrl* dbg) {
  constexpr uint32_t kTop = pow2_floor(mtile_cap(P));
  const int tid = threadIdx.x;
  uint32_t off[P], len[P];
#pragma unroll
  for (int t = 0; t < P; ++t) {
    off[t] = m.off[t];
    len[t] = m.len[t];
  }
  // pass 1: non-leader flags
  for (uint32_t u = tid; u < n; u += kThreads) {
    int s = 0;
#pragma unroll
    for (int t = 1; t < P; ++t) s += off[t] <= u ? 1 : 0;
    const uint32_t k = xk[u];
    uint32_t pos[P];
    runs_lower_bound<P, kTop>(xk, off, len, k, pos);
    bool dup = false;
#pragma unroll
    for (int t = 0; t < P; ++t) dup |= t < s && pos[t] < len[t] && xk[off[t] + pos[t]] == k;
    pre[u] = dup ? 1u : 0u;
  }
  __syncthreads();
  // exclusive prefix of the flags (contiguous chunks per thread), pre[n] = total
  {
    const uint32_t C = (n + kThreads - 1) / kThreads;
    const uint32_t c0 = std::min<uint32_t>(n, tid * C), c1 = std::min<uint32_t>(n, c0 + C);
    uint32_t sum = 0;
    for (uint32_t u = c0; u < c1; ++u) sum += pre[u];
    uint32_t tot;
    uint32_t run = block_exclusive_sum<uint32_t>(sum, s_scan, &tot);
    for (uint32_t u = c0; u < c1; ++u) {
      const uint32_t f = pre[u];
      pre[u] = run;
      run += f;
    }
    if (tid == 0) pre[n] = tot;
  }
  __syncthreads();
  dbg_mark(dbg, 6);
  // pass 2: leaders place and combine
  for (uint32_t u = tid; u < n; u += kThreads) {
    if (pre[u + 1] != pre[u]) continue;   // not a leader
    int s = 0;
#pragma unroll
    for (int t = 1; t < P; ++t) s += off[t] <= u ? 1 : 0;
    const uint32_t k = xk[u];
    uint32_t pos[P];
    runs_lower_bound<P, kTop>(xk, off, len, k, pos);
    V v[P];
    uint32_t mask = 0, opos = 0;
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const uint32_t p = pos[t];
      const bool present = t >= s && p < len[t] && xk[off[t] + p] == k;   // t < s: absent (u leads)
      opos += p - (pre[off[t] + p] - pre[off[t]]);
      v[t] = present ? xv[off[t] + p] : V(0);
      mask |= present ? 1u << t : 0u;
    }
    V r;
    if (op == 0) present_tree<0, 0, P>(v, mask, r);
    else if (op == 1) present_tree<1, 0, P>(v, mask, r);
    else present_tree<2, 0, P>(v, mask, r);
    yk[opos] = k;
    yv[opos] = r;
  }
  __syncthreads();
  return n - pre[n];
}

__host__ __device__ constexpr size_t split_fused_smem_bytes(int P, size_t vbytes) {
  // xk, yk, pre (cap + 4) as u32; xv, yv as values
  return 4 * (size_t)mtile_cap(P) * 3 + 16 + 2 * vbytes * (size_t)mtile_cap(P);
}

template <int P, typename V>
__global__ void __launch_bounds__(kThreads) split_fused_kernel(FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int cap = mtile_cap(P);
  uint32_t* xk = reinterpret_cast<uint32_t*>(smem);
  uint32_t* yk = xk + cap;
  uint32_t* pre = yk + cap;                                 // cap + 4 entries
  V* xv = reinterpret_cast<V*>(pre + cap + 4);              // 16-byte aligned: cap % 4 == 0
  V* yv = xv + cap;
  __shared__ MergeShared<P> m;
  __shared__ uint64_t s_off[kMaxRanks + 1];
  __shared__ uint32_t s_c[kTabSmem];
  __shared__ uint32_t s_scan[kWarps + 1];
  __shared__ const uint32_t* s_sidx[P];
  __shared__ const void* s_sval[P];
  __shared__ uint32_t s_ok, s_last;
  __shared__ uint32_t s_tot[P], s_before[P], s_pu[P + 1], s_pc[P];
  __shared__ uint64_t s_pslot[P], s_po[P];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t G = (uint32_t)a.G;
  const int l = (int)(blockIdx.x / G);
  const uint32_t b = blockIdx.x - (uint32_t)l * G;
  if ((a.skip >> l) & 1u) return;
  const int r = a.rank0 + l;
  Ctrl* ctl = fz_ctl(a, r);
  const uint32_t calls = *(volatile uint32_t*)&ctl->fz_calls;
  const uint32_t target = (calls + 1u) * G;   // per counter: G arrivals per call (u32, wraps consistently)
  const uint32_t part = (uint32_t)a.bnd[1];   // N < 2^32: 32-bit owner arithmetic
  dbg_mark(ctl, 8);

  // ---- 1. split push: CTA b pushes elements [e0, e1) of my stream.  An
  // element keeps its STREAM index e in the owner's receive region, and the
  // window-offset tables hold stream indices (table[0] = the slice's first
  // element, table[ntab] = one past its last), so no CTA searches for the
  // partition boundaries: first / last elements of a slice are recognised
  // from their neighbours' owners, and so are empty slices.
  {
    const uint32_t* idx = a.idx[l];
    const V* val = static_cast<const V*>(a.val[l]);
    const uint64_t n = a.n[l];
    const uint64_t E = ceil_div(n, G);
    const uint64_t e0 = std::min<uint64_t>(n, (uint64_t)b * E), e1 = std::min<uint64_t>(n, e0 + E);
    if (tid == 0) s_ok = (b == 0 && n == 0) ? (1u << P) - 1u : 0u;   // owners with an empty slice
    __syncthreads();
    dbg_mark(ctl, 9);
    constexpr int kPI = 4;   // elements per thread per round, all loads in flight
    for (uint64_t eb = e0; eb < e1; eb += (uint64_t)kThreads * kPI) {
      uint32_t xs[kPI], xq[kPI], xn[kPI];
      V vs[kPI];
#pragma unroll
      for (int i = 0; i < kPI; ++i) {
        const uint64_t e = eb + (uint64_t)i * kThreads + tid;
        if (e < e1) {
          xs[i] = idx[e];
          vs[i] = val[e];
          xq[i] = e > 0 ? idx[e - 1] : 0u;
          xn[i] = e + 1 < n ? idx[e + 1] : 0u;
        }
      }
#pragma unroll
      for (int i = 0; i < kPI; ++i) {
        const uint64_t e = eb + (uint64_t)i * kThreads + tid;
        if (e >= e1) continue;
        const uint32_t x = xs[i];
        const int j = (int)std::min<uint32_t>(x / part, P - 1);
        const int jq = e > 0 ? (int)std::min<uint32_t>(xq[i] / part, P - 1) : -1;
        const int jn = e + 1 < n ? (int)std::min<uint32_t>(xn[i] / part, P - 1) : P;
        char* pb = a.base[j];
        uint32_t* di = reinterpret_cast<uint32_t*>(pb + a.recv_off + (uint64_t)r * a.region_bytes);
        di[e] = x;
        reinterpret_cast<V*>(di + a.cap_s)[e] = vs[i];
        // window-offset table: dw[w] = first stream index of the slice whose table window >= w
        uint32_t* dw = reinterpret_cast<uint32_t*>(pb + a.win_off + (uint64_t)r * a.win_bytes);
        const uint32_t lo = (uint32_t)a.bnd[j];
        const int64_t w = (int64_t)((x - lo) / kTab);
        const int64_t wprev = jq == j ? (int64_t)((xq[i] - lo) / kTab) : -1;
        for (int64_t q = wprev + 1; q <= w; ++q) dw[q] = (uint32_t)e;
        if (jn != j) {   // last element of the slice
          const int64_t nwin = (int64_t)ceil_div(a.bnd[j + 1] - lo, kTab);
          for (int64_t q = w + 1; q <= nwin; ++q) dw[q] = (uint32_t)(e + 1);
        }
        // owners strictly between my neighbours' and mine get nothing from me
        const uint32_t gap = ((jq + 1 < j) ? ((1u << j) - (1u << (jq + 1))) : 0u) |
                             ((jn > j + 1) ? ((1u << jn) - (1u << (j + 1))) : 0u);
        if (gap) atomicOr(&s_ok, gap);
        if (a.validate) check_input(idx, e, n, a.N, x, vs[i], &ctl->status);
      }
    }
    __syncthreads();
    const uint32_t empty = s_ok;
    for (int j = 0; j < P; ++j) {   // empty slices: a constant table (zero)
      if (!((empty >> j) & 1u)) continue;
      uint32_t* dw = reinterpret_cast<uint32_t*>(a.base[j] + a.win_off + (uint64_t)r * a.win_bytes);
      const uint64_t ntab = ceil_div(a.bnd[j + 1] - a.bnd[j], kTab);
      for (uint64_t q = tid; q <= ntab; q += kThreads) dw[q] = 0;
    }
    if (b == 0 && tid < P) {
      Ctrl* pc = fz_ctl(a, tid);
      pc->k_in[r] = n;
      pc->sig_in[r] = sig_out(ctl, a.sig[l]);
    }
    __syncthreads();
    dbg_mark(ctl, 11);
    if (tid < P) {   // release my stores, then arrive at owner tid (its counter for source r)
      fence_acq_rel_sys();
      red_add_sys(&fz_ctl(a, tid)->fz_push_arr[r * 32], 1u);
    }
    dbg_mark(ctl, 10);
  }

  // ---- 2. owner: reduce my table windows [wa, wb) once every source CTA arrived
  for (int q = tid; q < kMaxTreeH * P; q += kThreads) {
    const int hh = q / P, sl = q - hh * P;
    m.role[hh][sl] = a.sched.role[hh][sl];
    m.part[hh][sl] = a.sched.part[hh][sl];
  }
  if (tid < P) {
    s_sidx[tid] = reinterpret_cast<const uint32_t*>(a.base[r] + a.recv_off + (uint64_t)tid * a.region_bytes);
    s_sval[tid] = a.base[r] + a.recv_off + (uint64_t)tid * a.region_bytes + 4 * a.cap_s;
  }
  if (tid == 0) s_ok = 1;
  __syncthreads();
  if (tid < P && !wait_flag_geq(&ctl->fz_push_arr[tid * 32], target, ctl)) s_ok = 0;
  __syncthreads();
  const bool ok1 = s_ok != 0;
  dbg_mark(ctl, 1);
  const uint32_t* win0 = reinterpret_cast<const uint32_t*>(a.base[r] + a.win_off);
  const uint32_t ntab_r = (uint32_t)ceil_div(a.bnd[r + 1] - a.bnd[r], kTab);
  if (tid < P && ok1) {
    check_sig(ctl, *(volatile uint64_t*)&ctl->sig_in[tid], a.sig[l]);
    if (b == 0) {   // pairs received from source tid (the header's traffic)
      const uint32_t* wt = win0 + (uint64_t)tid * (a.win_bytes / 4);
      ctl->slice_rx[calls & 1u][tid] = __ldcg(&wt[ntab_r]) - __ldcg(&wt[0]);
    }
  }
  if (b == 0 && warp == 0) {
    uint64_t ks = (tid < P && ok1) ? *(volatile uint64_t*)&ctl->k_in[tid] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ks += __shfl_xor_sync(0xffffffffu, ks, o);
    if (lane == 0) {
      ctl->k_sum = ks;
      ctl->dsar = 0;
    }
  }
  uint32_t* const st_idx = reinterpret_cast<uint32_t*>(a.base[r] + a.stage_off);
  V* const st_val = reinterpret_cast<V*>(a.base[r] + a.stage_off + 4 * (uint64_t)P * a.cap_s);
  uint32_t wa, wb;
  fz_range(a, r, b, wa, wb);
  bool in_smem = true;
  uint32_t cnt = 0;
  uint64_t ibase = 0;
  if (ok1 && wa < wb) {
    if (tid < P) {   // (and the slice's first stream index: ibase counts elements)
      const uint32_t* wt = win0 + (uint64_t)tid * (a.win_bytes / 4);
      s_c[tid] = __ldcg(&wt[wa]);
      s_c[P + tid] = __ldcg(&wt[wb]);
      s_c[2 * P + tid] = __ldcg(&wt[0]);
    }
    __syncthreads();
    dbg_mark(ctl, 2);
    uint32_t tot = 0;
#pragma unroll
    for (int src = 0; src < P; ++src) {
      tot += s_c[P + src] - s_c[src];
      ibase += s_c[src] - s_c[2 * P + src];
    }
    const SmemSrc srcs{s_sidx, s_sval};
    if (tot <= (uint32_t)cap) {
      const uint32_t n = stage_runs<P, V>(srcs, m, s_c, 0, 1, xk, xv);
      dbg_mark(ctl, 0);
      cnt = rank_merge<P, V>(m, n, xk, xv, pre, yk, yv, a.op, s_scan, ctl);
    } else {
      in_smem = false;
      const uint32_t wchunk = kTabSmem / P - 1;   // windows per chunk
      for (uint32_t cw = wa; cw < wb; cw += wchunk) {
        const int nw = (int)std::min<uint32_t>(wchunk, wb - cw);
        __syncthreads();
        for (int q = tid; q < (nw + 1) * P; q += kThreads) {
          const int w = q / P, src = q - w * P;
          s_c[q] = __ldcg(&win0[(uint64_t)src * (a.win_bytes / 4) + cw + w]);
        }
        __syncthreads();
        for (int pos = 0; pos < nw;) {   // greedy maximal pieces of at most cap elements
          const int w = pos + tid;
          uint32_t c = 0;
          if (w < nw) {
#pragma unroll
            for (int src = 0; src < P; ++src) c += s_c[(w + 1) * P + src] - s_c[w * P + src];
          }
          uint32_t tsum;
          const uint32_t incl = block_exclusive_sum<uint32_t>(c, s_scan, &tsum) + c;
          const int take = __syncthreads_count(w < nw && incl <= (uint32_t)cap);
          cnt += merge_subrange<P, V>(srcs, a.sched.hmax, a.op, m, s_c, pos, pos + take, st_idx + ibase + cnt,
                                      st_val + ibase + cnt, xk, xv, yk, yv);
          pos += take;
        }
      }
    }
  }
  __syncthreads();
  dbg_mark(ctl, 3);
  // push the piece into every reader's staging area (mine last), then arrive
  {
    const uint64_t xb = std::min<uint64_t>(ibase, (uint64_t)wa * kTab);
    const uint64_t slot = ((xb + 3) & ~3ull) + 4ull * b;
    for (int i = 1; i <= P; ++i) {
      const int d = (r + i) % P;
      uint32_t* di = fz_stage_idx(a, d, r) + slot;
      V* dv = fz_stage_val<V>(a, d, r) + slot;
      if (in_smem) {   // 16-byte stores; the tail beyond cnt stays inside the slot
        for (uint32_t u = tid; 4 * u < cnt; u += kThreads) {
          reinterpret_cast<uint4*>(di)[u] = reinterpret_cast<const uint4*>(yk)[u];
          if constexpr (sizeof(V) == 4) {
            reinterpret_cast<float4*>(dv)[u] = reinterpret_cast<const float4*>(yv)[u];
          } else {
            reinterpret_cast<double2*>(dv)[2 * u] = reinterpret_cast<const double2*>(yv)[2 * u];
            reinterpret_cast<double2*>(dv)[2 * u + 1] = reinterpret_cast<const double2*>(yv)[2 * u + 1];
          }
        }
      } else {
        for (uint32_t u = tid; u < cnt; u += kThreads) {
          di[u] = __ldcg(st_idx + ibase + u);
          dv[u] = __ldcg(st_val + ibase + u);
        }
      }
      if (tid == 0) fz_rec(a, d)[(uint64_t)r * kFzMaxG + b] = (uint64_t)cnt | (slot << 32);
    }
    __syncthreads();
    dbg_mark(ctl, 4);
    if (tid < P) {   // arrive at reader tid (its counter for owner r)
      fence_acq_rel_sys();
      red_add_sys(&fz_ctl(a, tid)->fz_data_arr[r * 32], 1u);
    }
    dbg_mark(ctl, 5);
  }

  // ---- 3. allgather: pieces (j, b) of every owner j from my staging into out
  if (tid == 0) s_ok = 1;
  if (tid < P) {
    s_tot[tid] = 0;
    s_before[tid] = 0;
  }
  __syncthreads();
  if (tid < P && !wait_flag_geq(&ctl->fz_data_arr[tid * 32], target, ctl)) s_ok = 0;
  __syncthreads();
  const bool ok2 = s_ok != 0;
  dbg_mark(ctl, 14);
  const uint64_t* rec = fz_rec(a, r);
  if (ok2) {   // every owner's piece counts: all loads in flight, then one reduction per owner
    uint32_t t[P], bf[P];
#pragma unroll
    for (int j = 0; j < P; ++j) t[j] = bf[j] = 0;
    for (uint32_t q = tid; q < G; q += kThreads) {
      uint32_t c[P];
#pragma unroll
      for (int j = 0; j < P; ++j) c[j] = (uint32_t)__ldcg(rec + (uint64_t)j * kFzMaxG + q);
#pragma unroll
      for (int j = 0; j < P; ++j) {
        t[j] += c[j];
        bf[j] += q < b ? c[j] : 0u;
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const uint32_t tt = __reduce_add_sync(0xffffffffu, t[j]);
      const uint32_t bb = __reduce_add_sync(0xffffffffu, bf[j]);
      if (lane == 0) {
        atomicAdd(&s_tot[j], tt);
        atomicAdd(&s_before[j], bb);
      }
    }
  }
  __syncthreads();
  dbg_mark(ctl, 12);
  uint64_t K = 0;
  for (int j = 0; j < P; ++j) K += s_tot[j];
  const bool dense = K > a.delta;
  char* out = a.out[l];
  // CTA 0 writes the header now (its own phases produced k_sum and the slice
  // counts; every status bit but a late timeout is set by now)
  auto header_status = [&]() { return *(volatile uint32_t*)&ctl->status; };
  if (b == 0 && tid == 0) {
    uint64_t sent = 0, recv = 0;
    for (int j = 0; j < P; ++j) {
      if (j == r) continue;
      recv += pair_bytes<V>() * ctl->slice_rx[calls & 1u][j];
      recv += pair_bytes<V>() * s_tot[j];
    }
    sent += pair_bytes<V>() * (a.n[l] - ctl->slice_rx[calls & 1u][r]);   // my stream minus my own slice
    sent += (uint64_t)(P - 1) * pair_bytes<V>() * s_tot[r];
    write_header(reinterpret_cast<sparcml_header*>(out), dense ? SPARCML_REPR_DENSE : SPARCML_REPR_SPARSE,
                 dense ? a.N : K, a.N, ctl->k_sum, sent, recv, SPARCML_SSAR_SPLIT_ALLGATHER, header_status(),
                 dense ? (uint64_t)SPARCML_HEADER_BYTES : a.val_offset, hdr_magic<V>());
  }
  if (ok2 && !dense) {
    // my pieces (j, b): count, staging slot, output offset; units of 4 pairs
    if (tid == 0) {
      uint64_t pre_k = 0;
      s_pu[0] = 0;
      for (int j = 0; j < P; ++j) {
        const uint64_t rj = __ldcg(rec + (uint64_t)j * kFzMaxG + b);
        s_pslot[j] = rj >> 32;
        s_pc[j] = (uint32_t)rj;
        s_po[j] = pre_k + s_before[j];
        s_pu[j + 1] = s_pu[j] + (((uint32_t)rj + 3) >> 2);
        pre_k += s_tot[j];
      }
    }
    __syncthreads();
    uint32_t* oi = reinterpret_cast<uint32_t*>(out + SPARCML_HEADER_BYTES);
    V* ov = reinterpret_cast<V*>(out + a.val_offset);
    const uint32_t U = s_pu[P];
    constexpr int kU = 8;   // units per thread per round, all loads in flight
    for (uint32_t u0 = tid; u0 < U; u0 += kThreads * kU) {
      uint4 k4[kU];
      V v4[kU][4];
      int jj[kU];
#pragma unroll
      for (int x = 0; x < kU; ++x) {
        const uint32_t u = u0 + x * kThreads;
        jj[x] = -1;
        if (u >= U) continue;
        int j = 0;
        while (u >= s_pu[j + 1]) ++j;
        jj[x] = j;
        const uint64_t e = s_pslot[j] + 4ull * (u - s_pu[j]);
        k4[x] = __ldcg(reinterpret_cast<const uint4*>(fz_stage_idx(a, r, j) + e));
        load4(fz_stage_val<V>(a, r, j) + e, 4, v4[x]);
      }
#pragma unroll
      for (int x = 0; x < kU; ++x) {
        const int j = jj[x];
        if (j < 0) continue;
        const uint32_t u = u0 + x * kThreads;
        const uint32_t q = 4 * (u - s_pu[j]);
        const uint32_t c = std::min<uint32_t>(4u, s_pc[j] - q);
        const uint64_t o = s_po[j] + q;
        const uint32_t kk[4] = {k4[x].x, k4[x].y, k4[x].z, k4[x].w};
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i)
          if (i < c) {
            oi[o + i] = kk[i];
            ov[o + i] = v4[x][i];
          }
      }
    }
  } else if (ok2) {   // K > delta: owner j's positions of piece b, neutral where absent
    V* od = reinterpret_cast<V*>(out + SPARCML_HEADER_BYTES);
    const V nv = op_neutral_v<V>(a.op);
    for (int j = 0; j < P; ++j) {
      const uint64_t rj = __ldcg(rec + (uint64_t)j * kFzMaxG + b);
      const uint32_t c = (uint32_t)rj;
      const uint32_t* si = fz_stage_idx(a, r, j) + (rj >> 32);
      const V* sv = fz_stage_val<V>(a, r, j) + (rj >> 32);
      uint32_t pa, pz;
      fz_range(a, j, b, pa, pz);
      const uint64_t p0 = a.bnd[j] + (uint64_t)pa * kTab;
      const uint64_t p1 = std::min<uint64_t>(a.bnd[j + 1], a.bnd[j] + (uint64_t)pz * kTab);
      for (uint64_t p = p0 + tid; p < p1; p += kThreads) od[p] = nv;
      __syncthreads();
      for (uint32_t u = tid; u < c; u += kThreads) od[__ldcg(si + u)] = __ldcg(sv + u);
    }
  }
  // CTA 0 closes the call on this rank once its own copies are done: every
  // CTA of mine has read `calls` (their owner phases all arrived before my
  // data wait passed), and every status bit of the call but a late timeout is
  // in the header.  No ticket, so no CTA waits for the others' stores to drain.
  dbg_mark(ctl, 15);
  if (b == 0 && tid == 0) {
    ctl->status = 0;
    ctl->fz_calls = calls + 1;
    ctl->seq = ctl->seq + 1;   // the call is complete on this rank when the kernel is
  }
  dbg_mark(ctl, 13);
}

using FusedFn = void (*)(FusedArgs);
template <typename V, int... Ps>
struct FusedTable {
  static FusedFn get(int P) {
    FusedFn f = nullptr;
    ((P == Ps ? (f = split_fused_kernel<Ps, V>, 0) : 0), ...);
    return f;
  }
};
static FusedFn fused_fn(int P, bool f64) {
  return f64 ? FusedTable<double, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::get(P)
             : FusedTable<float, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::get(P);
}

// CTAs per rank: every CTA of the launch must be co-resident (they wait on
// each other's arrivals); one rank per GPU takes SPARCML_FUSED_BPSM (default
// 2) per SM, a loopback world splits the GPU's resident CTAs between its ranks.
int split_fused_grid(int P, bool f64, int nloc) {
  static int bpsm = -1;
  if (bpsm < 0) {
    const char* e = std::getenv("SPARCML_FUSED_BPSM");
    bpsm = e ? std::max(1, std::atoi(e)) : 1;   // A/B at P = 4 (cfg2): 1 per SM beats 2 and 3
  }
  if (P < 2 || P > kMaxRanks) return 0;
  static int occ[2][kMaxRanks + 1] = {{0}};
  if (!occ[f64][P]) {
    const FusedFn f = fused_fn(P, f64);
    const size_t smem = split_fused_smem_bytes(P, f64 ? 8 : 4);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, kThreads, smem);
    occ[f64][P] = std::max(per, 0) + 1;   // +1: 0 means "not computed"
  }
  const int per = occ[f64][P] - 1;
  int g = nloc == 1 ? std::min(per, bpsm) * device_sm_count() : per * device_sm_count() / nloc;
  return std::min(g, kFzMaxG);
}

cudaError_t launch_split_fused(const FusedArgs& a, cudaStream_t s) {
  const bool f64 = a.f64 != 0;
  FusedArgs ac = a;
  void* args[] = {(void*)&ac};
  SPARCML_PROF("split_fused", s);
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)fused_fn(a.P, f64), dim3((unsigned)(a.G * a.nloc)),
                                                    dim3(kThreads), args, split_fused_smem_bytes(a.P, f64 ? 8 : 4), s);
  ++g_launches;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ===========================================================================
// allgather phase (§5.3.2 P:757-758 / §5.3.3): pull every owner's
// partition result over NVLink straight into the caller's out (sparse
// concatenation, densification, or QSGD decode), then write the header
// ===========================================================================
// MODE 0: sparse result paths only (SSAR concat, K > delta densify); MODE 1:
// DSAR decode only.  Each instantiation returns at once unless the device's
// SSAR/DSAR decision is its case (separate register budgets).
template <int MODE, typename V>
__global__ void __launch_bounds__(kThreads) concat_kernel(ConcatArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t s_pref[kMaxRanks + 1];
  __shared__ uint64_t s_upref[kMaxRanks + 1];
  __shared__ uint32_t s_dsar;
  __shared__ WinSource<V> s_src[1];
  const int tid = threadIdx.x;
  Ctrl* ctl = a.ctl;
  const uint32_t seq = ctl->seq;
  __shared__ uint64_t s_k[kMaxRanks];
  dbg_mark(ctl, 12);
  // SSAR or DSAR: decided by this rank's own owner kernel earlier on this
  // stream.  The variant that is not the case returns before anything else:
  // when both are launched (host_dsar == -1) the one running second must not
  // wait for owner flags of a call the first has already completed (seq + 1).
  if (tid == 0) s_dsar = a.host_dsar >= 0 ? (uint32_t)a.host_dsar : *(volatile uint32_t*)&ctl->dsar;
  __syncthreads();
  const bool dsar = s_dsar != 0;
  if (dsar != (MODE == 1)) return;
  if (tid < a.P) {   // one lane per owner: wait for its flag, read its result size
    if (a.wait_owners) {
      const bool ok = wait_flag_geq(&ctl->owner_done[tid], seq + 1, ctl);
      s_k[tid] = ok ? *(volatile const uint64_t*)&ctl->owner_k[tid] : 0;   // stored by owner tid with its flag
    } else {
      s_k[tid] = *(volatile const uint64_t*)a.r_n[tid];
    }
  }
  __syncthreads();
  if (tid == 0) {
    s_pref[0] = 0;
    s_upref[0] = 0;
    for (int j = 0; j < a.P; ++j) {
      const uint64_t kj = s_dsar ? 0 : s_k[j];
      s_pref[j + 1] = s_pref[j] + kj;
      s_upref[j + 1] = s_upref[j] + ceil_div(kj, 4);
    }
  }
  __syncthreads();
  dbg_mark(ctl, 14);
  const uint64_t K = s_pref[a.P];
  V* out_dense = reinterpret_cast<V*>(a.out + SPARCML_HEADER_BYTES);
  uint32_t* out_idx = reinterpret_cast<uint32_t*>(a.out + SPARCML_HEADER_BYTES);
  V* out_val = reinterpret_cast<V*>(a.out + a.val_offset);
  const uint64_t gstride = (uint64_t)gridDim.x * kThreads;
  const uint64_t gtid = (uint64_t)blockIdx.x * kThreads + tid;
  bool dense_result = dsar;
  if (MODE == 1) {
    // decode partitions in warp units of 128 positions (partition-relative;
    // a partition's last unit may be short): lane l decodes positions
    // [e + 4l, e + 4l + 4) -- coalesced code loads and float4 stores
    __shared__ uint64_t s_units[kMaxRanks + 1];
    __shared__ float s_lvl[128];
    const uint32_t s = a.bits ? (1u << (a.bits - 1)) - 1u : 0u;
    if (tid == 0) {
      s_units[0] = 0;
      for (int j = 0; j < a.P; ++j) s_units[j + 1] = s_units[j] + ceil_div(a.bnd[j + 1] - a.bnd[j], 128);
    }
    // fl(level / s) for every level: the decode's one division, tabulated
    for (uint32_t l = tid; l <= s && a.bits; l += kThreads) s_lvl[l] = __fdiv_rn(__uint2float_rn(l), __uint2float_rn(s));
    __syncthreads();
    const int lane = tid & 31;
    const uint32_t lgB = 31u - __clz(a.bucket);
    const uint32_t mask = a.bits ? (1u << a.bits) - 1u : 0u;
    const uint64_t nunits = s_units[a.P];
    const uint64_t gw = gtid >> 5, nw = gstride >> 5;
    constexpr int U = 4;   // units per warp per iteration, all their loads in flight
    for (uint64_t u0 = gw; u0 < nunits; u0 += nw * U) {
      uint32_t word[U];
      float scl[U];   // a lane's 4 positions share one bucket (B >= 8, 4-aligned)
      V dv[U][4];
      int jj[U], cnt[U];
      uint64_t ee[U];
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const uint64_t u = u0 + (uint64_t)x * nw;
        cnt[x] = 0;
        jj[x] = 0;
        ee[x] = 0;
        if (u >= nunits) continue;
        int j = 0;
        while (u >= s_units[j + 1]) ++j;
        const uint64_t nj = a.bnd[j + 1] - a.bnd[j];
        const uint64_t e = (u - s_units[j]) * 128 + 4 * (uint64_t)lane;
        jj[x] = j;
        ee[x] = e;
        cnt[x] = e >= nj ? 0 : (int)((nj - e) < 4 ? (nj - e) : 4);
        if (cnt[x] == 0) continue;
        if (sizeof(V) == sizeof(float) && a.bits) {   // QSGD: fp32 only (the host rejects f64)
          const uint8_t* cp = a.r_codes[j] + (e * a.bits) / 8;
          uint32_t w;
          if (cnt[x] == 4 && a.bits == 4) w = *reinterpret_cast<const uint16_t*>(cp);
          else if (cnt[x] == 4 && a.bits == 8) w = *reinterpret_cast<const uint32_t*>(cp);
          else if (cnt[x] == 4 && a.bits == 2) w = *cp;
          else {
            w = 0;
            const int nbytes = (cnt[x] * a.bits + 7) / 8;
            for (int q = 0; q < nbytes; ++q) w |= (uint32_t)cp[q] << (8 * q);
          }
          word[x] = w;
          scl[x] = a.r_scales[j][e >> lgB];
        } else {
          load4(static_cast<const V*>(a.r_dense[j]) + e, cnt[x], dv[x]);
        }
      }
#pragma unroll
      for (int x = 0; x < U; ++x) {
        if (cnt[x] == 0) continue;
        V v[4];
        if (sizeof(V) == sizeof(float) && a.bits) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t code = (word[x] >> (i * a.bits)) & mask;
            const float mag = __fmul_rn(s_lvl[code & s], scl[x]);   // = qsgd_decode (reading R-16)
            v[i] = (code >> (a.bits - 1)) ? -mag : mag;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = dv[x][i];
        }
        store4(out_dense + a.bnd[jj[x]] + ee[x], v, cnt[x]);
      }
    }
  } else if (K <= a.delta) {
    // sparse concatenation: disjoint ranges, globally sorted by construction
    // (P:511-515).  Units of 4 pairs of one owner: 16-byte loads over NVLink.
    const uint64_t units = s_upref[a.P];
#ifndef SPARCML_CONCAT_U
#define SPARCML_CONCAT_U 4
#endif
    constexpr int U = SPARCML_CONCAT_U;   // units per thread per iteration: all their NVLink loads in flight
    for (uint64_t u0 = gtid; u0 < units; u0 += gstride * U) {
      uint4 ix[U];
      V vx[U][4];
      uint64_t oo[U];
      int cnt[U];   // pairs in the unit (4, or an owner's short last unit; 0 = none)
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const uint64_t u = u0 + (uint64_t)x * gstride;
        cnt[x] = 0;
        if (u >= units) continue;
        int j = 0;
        while (u >= s_upref[j + 1]) ++j;
        const uint64_t p = (u - s_upref[j]) * 4;
        const uint64_t kj = s_pref[j + 1] - s_pref[j];
        oo[x] = s_pref[j] + p;
        const int n = (int)std::min<uint64_t>(4, kj - p);
        if (n == 4) {
          ix[x] = *reinterpret_cast<const uint4*>(a.r_idx[j] + p);
        } else {
          const uint32_t* si = a.r_idx[j] + p;
          ix[x] = make_uint4(si[0], n > 1 ? si[1] : 0u, n > 2 ? si[2] : 0u, 0u);
        }
        load4(static_cast<const V*>(a.r_val[j]) + p, n, vx[x]);
        cnt[x] = n;
      }
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int n = cnt[x];
        if (n == 0) continue;
        const uint64_t o = oo[x];
        out_idx[o] = ix[x].x;
        out_val[o] = vx[x][0];
        if (n > 1) {
          out_idx[o + 1] = ix[x].y;
          out_val[o + 1] = vx[x][1];
        }
        if (n > 2) {
          out_idx[o + 2] = ix[x].z;
          out_val[o + 2] = vx[x][2];
        }
        if (n > 3) {
          out_idx[o + 3] = ix[x].w;
          out_val[o + 3] = vx[x][3];
        }
      }
    }
  } else {
    // K > delta cannot be stored sparse: densify partition by partition
    dense_result = true;
    TreeSched ts;
    ts.n = 0;
    WinOutput<V> wo = {};
    wo.mode = WIN_DENSE;
    wo.op = a.op;
    wo.dense = out_dense;
    wo.dense_base = 0;
    for (int j = 0; j < a.P; ++j) {
      if (tid == 0) {
        s_src[0].idx = a.r_idx[j];
        s_src[0].val = static_cast<const V*>(a.r_val[j]);
        s_src[0].n = s_pref[j + 1] - s_pref[j];
        s_src[0].dense = 0;
        s_src[0].dense_base = 0;
      }
      __syncthreads();
      const uint32_t nwin = (uint32_t)ceil_div(a.bnd[j + 1] - a.bnd[j], kWin);
      for (uint32_t w = blockIdx.x; w < nwin; w += gridDim.x)
        window_tile(s_src, 1, ts, a.bnd[j], a.bnd[j + 1], w, smem, a.status, 0, nwin, wo);
      __syncthreads();
    }
  }
  dbg_mark(ctl, 15);
  if (last_block<false>(&ctl->done_ctr[2]) && tid == 0) {
    // bytes this rank put on / took off NVLink (pull model counted at the owner)
    uint64_t sent = 0, recv = 0;
    for (int j = 0; j < a.P; ++j) {
      if (j == a.rank) continue;
      sent += pair_bytes<V>() * ctl->slice_out[j];
      recv += pair_bytes<V>() * ctl->slice_rx[seq & 1][j];
    }
    for (int j = 0; j < a.P; ++j) {
      uint64_t w;
      const uint64_t nj = a.bnd[j + 1] - a.bnd[j];
      if (dsar) w = a.bits ? (nj * a.bits + 7) / 8 + 4 * ceil_div(nj, a.bucket) : sizeof(V) * nj;
      else w = pair_bytes<V>() * (s_pref[j + 1] - s_pref[j]);
      if (j == a.rank) sent += (uint64_t)(a.P - 1) * w;
      else recv += w;
    }
    write_header(reinterpret_cast<sparcml_header*>(a.out), dense_result ? SPARCML_REPR_DENSE : SPARCML_REPR_SPARSE,
                 dense_result ? a.N : K, a.N, ctl->k_sum, sent, recv, dsar ? SPARCML_DSAR_SPLIT_ALLGATHER : a.algo,
                 ctl->status, dense_result ? (uint64_t)SPARCML_HEADER_BYTES : a.val_offset, hdr_magic<V>());
    ctl->status = 0;
    __threadfence();
    ctl->seq = seq + 1;   // the call is complete on this rank
  }
  dbg_mark(ctl, 13);
}

template <typename V>
static void launch_concat_t(const ConcatArgs& a, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = win_smem_bytes(1, sizeof(V));
  if (!attr) {
    cudaFuncSetAttribute(concat_kernel<0, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(concat_kernel<1, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  // two blocks per SM for the sparse concatenation (A/B at P = 2 and 4: 1 and
  // 2 blocks per SM beat 4; 2 beats 1 by ~2 us at P = 4), four for the dense decode
#ifndef SPARCML_CONCAT_BPSM
#define SPARCML_CONCAT_BPSM 2
#endif
  const int grid = device_sm_count() * (a.host_dsar == 0 ? SPARCML_CONCAT_BPSM : 4);
  ConcatArgs ac = a;
  void* args[] = {(void*)&ac};
  if (a.host_dsar != 1) {
    if (a.pdl) launch_pdl((const void*)concat_kernel<0, V>, dim3(grid), smem, s, args, false);
    else concat_kernel<0, V><<<grid, kThreads, smem, s>>>(a);
    ++g_launches;
  }
  if (a.host_dsar != 0) {
    if (a.pdl) launch_pdl((const void*)concat_kernel<1, V>, dim3(grid), smem, s, args, false);
    else concat_kernel<1, V><<<grid, kThreads, smem, s>>>(a);
    ++g_launches;
  }
}

cudaError_t launch_concat(const ConcatArgs& a, cudaStream_t s) {
  SPARCML_PROF("concat", s);
  if (a.f64) launch_concat_t<double>(a, s);
  else launch_concat_t<float>(a, s);
  return cudaGetLastError();
}

// ===========================================================================
// flag barrier over NVLink (one warp): sparcml_barrier
// ===========================================================================
__global__ void barrier_kernel(BarrierArgs a) {
  const int lane = threadIdx.x;
  uint32_t e = 0;
  if (lane == 0) {
    e = a.my->epoch + 1;
    a.my->epoch = e;
  }
  e = __shfl_sync(0xffffffffu, e, 0);
  fence_acq_rel_sys();
  if (!a.loopback && lane < a.P && lane != a.rank) {
    st_release_sys(a.peer_flags[lane], e);
    wait_flag_geq(&a.my->flags[lane], e, a.my);   // gives up after the comm's timeout (status bit)
  }
  __syncwarp();
  fence_acq_rel_sys();
}

cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s) {
  SPARCML_PROF("barrier", s);
  barrier_kernel<<<1, 32, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// P == 1: the collective is the identity on the stream (or its densified /
// QSGD-coded form); validate and fill the control block the concat reads.
template <typename V>
__global__ void __launch_bounds__(kThreads) p1_prep_kernel(P1PrepArgs a) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  if (a.validate || a.win) {
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < a.n; e += stride) {
      const uint32_t x = a.idx[e];
      if (a.validate) check_input(a.idx, e, a.n, a.N, x, static_cast<const V*>(a.val)[e], &a.ctl->status);
      if (a.win) {   // window-offset table of the one partition (as split_push builds for owners)
        const int64_t w = (int64_t)(x / kTab);
        const int64_t wprev = e == 0 ? -1 : (int64_t)(a.idx[e - 1] / kTab);
        for (int64_t q = wprev + 1; q <= w; ++q) a.win[q] = (uint32_t)e;
        if (e + 1 == a.n) {
          const int64_t ntab = (int64_t)ceil_div(a.N, kTab);
          for (int64_t q = w + 1; q <= ntab; ++q) a.win[q] = (uint32_t)a.n;
        }
      }
    }
    if (a.win && a.n == 0)
      for (uint64_t q = (uint64_t)blockIdx.x * kThreads + threadIdx.x; q <= ceil_div(a.N, kTab); q += stride) a.win[q] = 0;
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

// P == 1, sparse result (nnz <= delta): one kernel copies the input into out
// (16-byte vectors where aligned) and writes the header -- the whole call.
template <typename V>
__global__ void __launch_bounds__(kThreads) p1_sparse_kernel(P1PrepArgs a) {
  uint32_t* oi = reinterpret_cast<uint32_t*>(a.out + SPARCML_HEADER_BYTES);
  V* ov = reinterpret_cast<V*>(a.out + a.val_offset);
  const V* iv = static_cast<const V*>(a.val);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t gt = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(a.idx) | reinterpret_cast<uintptr_t>(a.val)) & 15u) == 0;
  if (!a.copy) {
    // in place: the payload is already there
  } else if (vec) {   // 16-byte units: 4 indices, 16 / sizeof(V) values
    constexpr uint64_t kv = 16 / sizeof(V);
    const uint64_t n4 = a.n / 4, nv = a.n / kv;
    for (uint64_t u = gt; u < n4; u += stride)
      reinterpret_cast<uint4*>(oi)[u] = ld_stream_u4(reinterpret_cast<const uint4*>(a.idx) + u);
    for (uint64_t u = gt; u < nv; u += stride)
      reinterpret_cast<uint4*>(ov)[u] = ld_stream_u4(reinterpret_cast<const uint4*>(iv) + u);
    for (uint64_t e = 4 * n4 + gt; e < a.n; e += stride) oi[e] = a.idx[e];
    for (uint64_t e = kv * nv + gt; e < a.n; e += stride) ov[e] = iv[e];
  } else {
    for (uint64_t e = gt; e < a.n; e += stride) {
      oi[e] = a.idx[e];
      ov[e] = iv[e];
    }
  }
  if (a.validate)
    for (uint64_t e = gt; e < a.n; e += stride) check_input(a.idx, e, a.n, a.N, a.idx[e], iv[e], &a.ctl->status);
  if (last_block<false>(&a.ctl->done_ctr[2]) && threadIdx.x == 0) {
    Ctrl* c = a.ctl;
    c->k_in[0] = a.n;
    c->slice_cnt[0] = a.n;
    c->slice_out[0] = a.n;
    c->owner_K = a.n;
    c->k_sum = a.n;
    c->dsar = 0;
    write_header(reinterpret_cast<sparcml_header*>(a.out), SPARCML_REPR_SPARSE, a.n, a.N, a.n, 0, 0, a.algo_used,
                 c->status, a.val_offset, hdr_magic<V>());
    c->status = 0;
    __threadfence();
    c->seq = c->seq + 1;   // the call is complete
  }
}

cudaError_t launch_p1_sparse(const P1PrepArgs& a, cudaStream_t s) {
  const uint64_t work = (a.copy || a.validate) ? a.n / 4 : 0;
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((work + kThreads - 1) / kThreads,
                                                                   (uint64_t)device_sm_count() * 4));
  SPARCML_PROF("p1_sparse", s);
  if (a.f64) p1_sparse_kernel<double><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  else p1_sparse_kernel<float><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_p1_prep(const P1PrepArgs& a, cudaStream_t s) {
  const uint64_t blocks = (a.validate || a.win)
                              ? std::max<uint64_t>(1, std::min<uint64_t>((a.n + kThreads - 1) / kThreads, 4096))
                              : 1;
  SPARCML_PROF("p1_prep", s);
  if (a.f64) p1_prep_kernel<double><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  else p1_prep_kernel<float><<<(unsigned)blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// layer-wise tensor fusion (NEXT row 1): concatenate per-layer streams with
// index offsets; locate layer ranges in a result
// ===========================================================================
__global__ void __launch_bounds__(kThreads) fuse_streams_kernel(FuseArgs a) {
  const uint64_t total = a.pre[a.L];
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (uint64_t)gridDim.x * kThreads) {
    int l = 0;
    while (e >= a.pre[l + 1]) ++l;
    const uint64_t i = e - a.pre[l];
    a.idx_out[e] = (uint32_t)(a.idx[l][i] + a.off[l]);
    a.val_out[e] = a.val[l][i];
  }
}

cudaError_t launch_fuse_streams(const FuseArgs& a, cudaStream_t s) {
  const uint64_t total = a.pre[a.L];
  const unsigned blocks =
      (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + kThreads - 1) / kThreads, (uint64_t)device_sm_count() * 8));
  fuse_streams_kernel<<<blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// one warp per layer boundary: lower bound of off[l] in the sparse result
__global__ void layer_ranges_kernel(const char* out, int L, LayerOffsets off, uint64_t* starts) {
  const sparcml_header* h = reinterpret_cast<const sparcml_header*>(out);
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (l > L) return;
  const bool dense = h->repr == SPARCML_REPR_DENSE;
  const uint64_t n = dense ? h->N : h->nnz;
  uint64_t r;
  if (l == L) r = n;
  else if (dense) r = off.v[l];
  else r = warp_lower_bound(reinterpret_cast<const uint32_t*>(out + SPARCML_HEADER_BYTES), n, off.v[l]);
  if ((threadIdx.x & 31) == 0) starts[l] = r;
}

cudaError_t launch_layer_ranges(const char* out, int L, const LayerOffsets& off, uint64_t* starts, cudaStream_t s) {
  const int warps = L + 1;
  layer_ranges_kernel<<<(warps + 7) / 8, 256, 0, s>>>(out, L, off, starts);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// sparse allgather for disjoint slices (§7 SCD; reading R-27):
// publish (local copy + announce to every peer), then one pull-concatenation
// ===========================================================================
// Published streams and their metadata alternate by call parity: a rank that
// has finished call s may publish s+1 (the other slot) while a slower peer
// still pulls s; it can publish s+2 (this slot again) only after every peer
// has published s+1, i.e. finished pulling s.
template <typename V>
__global__ void __launch_bounds__(kThreads) ag_publish_kernel(AgPublishArgs a) {
  const uint32_t seq = a.ctl->seq;
  const int par = seq & 1;
  uint32_t* my_idx = a.my_idx[par];
  V* my_val = static_cast<V*>(a.my_val[par]);
  for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < a.n; e += (uint64_t)gridDim.x * kThreads) {
    const uint32_t x = a.idx[e];
    const V v = static_cast<const V*>(a.val)[e];
    my_idx[e] = x;
    my_val[e] = v;
    if (a.validate) check_input(a.idx, e, a.n, a.N, x, v, &a.ctl->status);
  }
  if (last_block<false>(&a.ctl->done_ctr[0]) && threadIdx.x < a.P) {   // local copies only: gpu scope
    Ctrl* p = a.peer[threadIdx.x];
    p->ag_n[par][a.rank] = a.n;
    p->ag_first[par][a.rank] = a.n ? a.idx[0] : 0u;
    p->ag_last[par][a.rank] = a.n ? a.idx[a.n - 1] : 0u;
    p->ag_sig[par][a.rank] = sig_out(a.ctl, a.sig);
    st_release_sys(&p->ag_done[par][a.rank], seq + 1);
  }
}

cudaError_t launch_ag_publish(const AgPublishArgs& a, cudaStream_t s) {
  const unsigned blocks = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((a.n + kThreads - 1) / kThreads, (uint64_t)device_sm_count() * 4));
  SPARCML_PROF("ag_publish", s);
  if (a.f64) ag_publish_kernel<double><<<blocks, kThreads, 0, s>>>(a);
  else ag_publish_kernel<float><<<blocks, kThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

template <typename V>
__global__ void __launch_bounds__(kThreads) ag_gather_kernel(AgGatherArgs a) {
  __shared__ uint64_t s_n[kMaxRanks], s_pref[kMaxRanks + 1], s_upref[kMaxRanks + 1];
  __shared__ uint32_t s_first[kMaxRanks], s_last[kMaxRanks];
  __shared__ int s_ord[kMaxRanks], s_m;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  Ctrl* ctl = a.ctl;
  const uint32_t seq = ctl->seq;
  const int par = seq & 1;
  if (tid < a.P) {   // one lane per rank: its stream is published
    const bool ok = wait_flag_geq(&ctl->ag_done[par][tid], seq + 1, ctl);
    if (ok && blockIdx.x == 0) check_sig(ctl, *(volatile uint64_t*)&ctl->ag_sig[par][tid], a.sig);
    s_n[tid] = ok ? *(volatile uint64_t*)&ctl->ag_n[par][tid] : 0;
    s_first[tid] = *(volatile uint32_t*)&ctl->ag_first[par][tid];
    s_last[tid] = *(volatile uint32_t*)&ctl->ag_last[par][tid];
  }
  __syncthreads();
  if (tid == 0) {   // non-empty ranks in range order; the ranges must not overlap
    int m = 0;
    for (int r = 0; r < a.P; ++r) {
      if (s_n[r] == 0) continue;
      int i = m;
      while (i > 0 && s_first[s_ord[i - 1]] > s_first[r]) {
        s_ord[i] = s_ord[i - 1];
        --i;
      }
      s_ord[i] = r;
      ++m;
    }
    bool bad = false;
    for (int i = 0; i + 1 < m; ++i) bad |= s_last[s_ord[i]] >= s_first[s_ord[i + 1]];
    if (bad && blockIdx.x == 0) atomicOr(&ctl->status, 1u << SPARCML_ERR_INVALID_ARG);
    s_m = m;
    s_pref[0] = 0;
    s_upref[0] = 0;
    for (int i = 0; i < m; ++i) {
      s_pref[i + 1] = s_pref[i] + s_n[s_ord[i]];
      s_upref[i + 1] = s_upref[i] + ceil_div(s_n[s_ord[i]], 4);
    }
  }
  __syncthreads();
  const int m = s_m;
  const uint64_t K = s_pref[m];
  const bool dense = K > a.delta;
  const uint64_t gstride = (uint64_t)gridDim.x * kThreads;
  const uint64_t gtid = (uint64_t)blockIdx.x * kThreads + tid;
  if (!dense) {   // concatenation in range order, units of 4 pairs, four units' NVLink loads in flight
    uint32_t* out_idx = reinterpret_cast<uint32_t*>(a.out + SPARCML_HEADER_BYTES);
    V* out_val = reinterpret_cast<V*>(a.out + a.val_offset);
    const uint64_t units = s_upref[m];
    constexpr int U = 4;
    for (uint64_t u0 = gtid; u0 < units; u0 += gstride * U) {
      uint4 ix[U];
      V vx[U][4];
      uint64_t oo[U];
      int cnt[U];
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const uint64_t u = u0 + (uint64_t)x * gstride;
        cnt[x] = 0;
        if (u >= units) continue;
        int i = 0;
        while (u >= s_upref[i + 1]) ++i;
        const int r = s_ord[i];
        const uint64_t p = (u - s_upref[i]) * 4;
        const uint64_t nr = s_n[r];
        oo[x] = s_pref[i] + p;
        const int n = (int)std::min<uint64_t>(4, nr - p);
        if (n == 4) {
          ix[x] = *reinterpret_cast<const uint4*>(a.src_idx[par][r] + p);
        } else {
          const uint32_t* si = a.src_idx[par][r] + p;
          ix[x] = make_uint4(si[0], n > 1 ? si[1] : 0u, n > 2 ? si[2] : 0u, 0u);
        }
        load4(static_cast<const V*>(a.src_val[par][r]) + p, n, vx[x]);
        cnt[x] = n;
      }
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int n = cnt[x];
        if (n == 0) continue;
        const uint64_t o = oo[x];
        out_idx[o] = ix[x].x;
        out_val[o] = vx[x][0];
        if (n > 1) {
          out_idx[o + 1] = ix[x].y;
          out_val[o + 1] = vx[x][1];
        }
        if (n > 2) {
          out_idx[o + 2] = ix[x].z;
          out_val[o + 2] = vx[x][2];
        }
        if (n > 3) {
          out_idx[o + 3] = ix[x].w;
          out_val[o + 3] = vx[x][3];
        }
      }
    }
  } else {        // K > delta: zeros, then every value at its index
    V* d = reinterpret_cast<V*>(a.out + SPARCML_HEADER_BYTES);
    for (uint64_t e = gtid; e < a.N; e += gstride) d[e] = V(0);
    grid.sync();
    for (uint64_t e = gtid; e < K; e += gstride) {
      int i = 0;
      while (e >= s_pref[i + 1]) ++i;
      const int r = s_ord[i];
      const uint64_t q = e - s_pref[i];
      d[a.src_idx[par][r][q]] = static_cast<const V*>(a.src_val[par][r])[q];
    }
  }
  grid.sync();
  if (blockIdx.x == 0 && tid == 0) {
    const uint64_t mine = s_n[a.rank];
    write_header(reinterpret_cast<sparcml_header*>(a.out), dense ? SPARCML_REPR_DENSE : SPARCML_REPR_SPARSE,
                 dense ? a.N : K, a.N, K, pair_bytes<V>() * mine * (uint64_t)(a.P - 1), pair_bytes<V>() * (K - mine),
                 SPARCML_SPARSE_ALLGATHER, ctl->status, dense ? (uint64_t)SPARCML_HEADER_BYTES : a.val_offset,
                 hdr_magic<V>());
    ctl->status = 0;
    __threadfence();
    ctl->seq = seq + 1;   // the call is complete on this rank
  }
}

cudaError_t launch_ag_gather(const AgGatherArgs& a, cudaStream_t s) {
  static int occ[2] = {0, 0};
  const int f = a.f64 ? 1 : 0;
  const void* fn = a.f64 ? (const void*)ag_gather_kernel<double> : (const void*)ag_gather_kernel<float>;
  if (!occ[f]) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[f], fn, kThreads, 0);
    occ[f] = std::max(1, std::min(occ[f], 2));
  }
  AgGatherArgs ac = a;
  void* args[] = {(void*)&ac};
  SPARCML_PROF("ag_gather", s);
  const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(device_sm_count() * occ[f]), dim3(kThreads), args, 0, s);
  ++g_launches;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ===========================================================================
// Algorithm 1's update v <- v - g, g read from an allreduce result
// ===========================================================================
template <typename V>
__global__ void __launch_bounds__(kThreads) apply_update_kernel(V* v, const char* out) {
  const sparcml_header* h = reinterpret_cast<const sparcml_header*>(out);
  if (h->magic != hdr_magic<V>()) return;   // a result of the other value type
  const bool dense = h->repr == SPARCML_REPR_DENSE;
  const uint64_t n = dense ? h->N : h->nnz;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  if (dense) {
    const V* g = reinterpret_cast<const V*>(out + SPARCML_HEADER_BYTES);
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < n; e += stride) v[e] = v[e] - g[e];
  } else {
    const uint32_t* gi = reinterpret_cast<const uint32_t*>(out + SPARCML_HEADER_BYTES);
    const V* gv = reinterpret_cast<const V*>(out + h->val_offset);
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e < n; e += stride)
      v[gi[e]] = v[gi[e]] - gv[e];
  }
}

cudaError_t launch_apply_update(float* v, const char* out, cudaStream_t s) {
  SPARCML_PROF("apply_update", s);
  apply_update_kernel<float><<<device_sm_count() * 4, kThreads, 0, s>>>(v, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_apply_update_f64(double* v, const char* out, cudaStream_t s) {
  SPARCML_PROF("apply_update", s);
  apply_update_kernel<double><<<device_sm_count() * 4, kThreads, 0, s>>>(v, out);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace sparcml
