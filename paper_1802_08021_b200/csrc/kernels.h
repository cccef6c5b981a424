// kernels.h — launch interface between the host orchestrator (api.cu) and
// the kernels.  Plain structs passed by value as kernel parameters.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "tiles.cuh"

namespace sparcml {

// --------------------------------------------------------------- gating ----
// A kernel whose work depends on a device-side decision reads it from
// (*gate_ptr == gate_value); gate_ptr == nullptr means "always run".
struct Gate {
  const uint32_t* ptr;
  uint32_t value;
};

// -------------------------------------------------------- batched merges ---
struct MergeJob {
  const uint32_t* a_idx;
  const float* a_val;
  const uint64_t* a_n_dev;  // nullable: then a_n
  uint64_t a_n;
  const uint32_t* b_idx;
  const float* b_val;
  const uint64_t* b_n_dev;
  uint64_t b_n;
  MergeOutput out;
};

struct MergeJobsArgs {
  int njobs;
  MergeJob job[kMaxJobs];
  ScanCounters* ctr;
  TileStatus* status;
  Gate gate;
};

// ----------------------------------------------------------- window ------
struct WinSourceDesc {      // device-resolved at kernel start
  const uint32_t* idx;
  const float* val;
  const uint64_t* n_dev;    // nullable -> n
  uint64_t n;
  const uint32_t* dense_dev;  // nullable -> dense
  int dense;
  uint64_t dense_base;
};

struct WindowArgs {
  int nsrc;
  WinSourceDesc src[kMaxRanks];
  TreeSched sched;
  uint64_t lo, hi;
  WinOutput out;
  ScanCounters* ctr;
  TileStatus* status;
  Gate gate;
};

// ----------------------------------------------------- recursive doubling ---
// A "stream buffer": sparse idx at base, val at base + val_off; dense vals at base.
struct StreamBuf {
  char* base;
  uint64_t val_off;
};

struct RdStageArgs {
  // own stream (stage 1: the caller's input)
  const uint32_t* a_idx;
  const float* a_val;
  const uint64_t* a_n_dev;  // nullable -> a_n
  uint64_t a_n;
  const uint32_t* a_dense_dev;  // nullable -> sparse
  const uint64_t* a_ksum_dev;   // nullable -> a_n
  // partner stream, in my recv buffer
  StreamBuf b;
  const uint64_t* b_n_dev;
  const uint32_t* b_dense_dev;
  const uint64_t* b_ksum_dev;
  uint64_t N, delta;
  // output stream (cur buffer, or the caller's out payload)
  StreamBuf o;
  uint64_t* o_n_dev;
  uint32_t* o_dense_dev;
  uint64_t* o_ksum_dev;
  // optional mirror into the next partner's recv buffer
  StreamBuf m;
  uint64_t* m_n_dev;
  uint32_t* m_dense_dev;
  uint64_t* m_ksum_dev;
  Ctrl* ctl;            // my control block (bytes accounting, status)
  int stage;            // 1-based
  int last;
  sparcml_header* hdr;  // last stage only
  ScanCounters* ctr;
  TileStatus* status;
};

// Stage-1 push: my input -> partner's recv buffer (+counts).
struct RdPushArgs {
  const uint32_t* idx;
  const float* val;
  uint64_t n;
  StreamBuf dst;
  uint64_t* dst_n;
  uint32_t* dst_dense;
  uint64_t* dst_ksum;
  Ctrl* ctl;            // my control block
  uint64_t N;
  int validate;
};

// ---------------------------------------------------------- split phase ---
struct PushArgs {
  const uint32_t* idx;
  const float* val;
  uint64_t n;
  uint64_t N;
  int P, rank;
  uint64_t bnd[kMaxRanks + 1];
  uint32_t* dst_idx[kMaxRanks];    // owner j's receive region for source `rank`
  float* dst_val[kMaxRanks];
  uint64_t* dst_cnt[kMaxRanks];    // &owner_j.ctrl.slice_cnt[rank]
  uint64_t* dst_k[kMaxRanks];      // &peer_j.ctrl.k_in[rank]
  Ctrl* ctl;                       // my control block
  int validate;
};

// Owner decision (SSAR vs DSAR) evaluated at the start of the owner stage.
struct DecideArgs {
  const uint64_t* k_in;   // my Ctrl.k_in
  int P;
  int algo;               // sparcml_algo (2 or 3 forced; 0 auto)
  uint64_t delta;
  uint32_t* dsar_out;     // my Ctrl.dsar
  uint64_t* k_sum_out;    // my Ctrl.k_sum
};

struct ConcatArgs {
  int P, rank;
  uint64_t N, delta;
  uint64_t bnd[kMaxRanks + 1];
  // owner j's partial result (peer pointers)
  const uint32_t* r_idx[kMaxRanks];
  const float* r_val[kMaxRanks];
  const uint64_t* r_n[kMaxRanks];
  const uint8_t* r_codes[kMaxRanks];
  const float* r_scales[kMaxRanks];
  const float* r_dense[kMaxRanks];
  Ctrl* ctl;                       // my control block (dsar, k_sum, slice counts, status)
  int bits;
  uint32_t bucket;
  char* out;                       // caller's out (header + payload)
  uint64_t val_offset;
  uint32_t algo;
  ScanCounters* ctr;
  TileStatus* status;
};

struct BarrierArgs {
  Ctrl* my;
  uint32_t* peer_flags[kMaxRanks];  // &peer_p.ctrl.flags[rank]
  int P, rank;
  int first_in_call;
  int loopback;                     // no waiting (all ranks on one stream)
};

struct P1PrepArgs {                 // P == 1: validate and fill the control block
  const uint32_t* idx;
  const float* val;
  uint64_t n, N, delta;
  int algo;
  Ctrl* ctl;
  int validate;
};

// ----------------------------------------------------------- launchers -----
extern unsigned long long g_launches;   // kernels enqueued by this library

// RAII event bracket around one launch (no-op unless profiling is enabled)
class ProfScope {
 public:
  ProfScope(const char* name, cudaStream_t s);
  ~ProfScope();

 private:
  const char* name_;
  cudaStream_t s_;
  void* a_;
};
#define SPARCML_PROF(name, s) ::sparcml::ProfScope prof_scope_##__LINE__(name, s)

int device_sm_count();
cudaError_t launch_merge_jobs(const MergeJobsArgs& a, int grid_cap, cudaStream_t s);
cudaError_t launch_window(const WindowArgs& a, cudaStream_t s);
cudaError_t launch_rd_push(const RdPushArgs& a, cudaStream_t s);
cudaError_t launch_rd_stage(const RdStageArgs& a, cudaStream_t s);
cudaError_t launch_split_push(const PushArgs& a, cudaStream_t s);
cudaError_t launch_barrier_decide(const BarrierArgs& a, const DecideArgs& d, cudaStream_t s);
cudaError_t launch_concat(const ConcatArgs& a, cudaStream_t s);
cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s);
cudaError_t launch_p1_prep(const P1PrepArgs& a, cudaStream_t s);

// top-k / QSGD (kernels_topk.cu, kernels_qsgd.cu)
size_t topk_workspace_bytes(uint64_t N, uint64_t k);
cudaError_t launch_topk(const float* x, const float* grad, float alpha, int ef, float* x_out,
                        uint64_t N, uint64_t k, uint32_t* idx_out, float* val_out, float* residual,
                        void* ws, cudaStream_t s);
cudaError_t launch_quantize(const float* x, uint64_t n, int bits, uint32_t bucket, uint64_t seed,
                            uint64_t ctr_base, uint8_t* codes, float* scales, cudaStream_t s);
cudaError_t launch_dequantize(const uint8_t* codes, const float* scales, uint64_t n, int bits,
                              uint32_t bucket, float* out, cudaStream_t s);

}  // namespace sparcml
