// kernels.h — launch interface between the host orchestrator (api.cu) and
// the kernels.  Plain structs passed by value as kernel parameters.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "tiles.cuh"

namespace sparcml {

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
  MergeOutput<float> out;
};

struct MergeJobsArgs {   // stand-alone sparcml_merge_sum
  int njobs;
  MergeJob job[kMaxJobs];
  ScanCounters* ctr;
  TileStatus* status;
};

// ----------------------------------------------------------- window ------
// ----------------------------------------------------- recursive doubling ---
// A "stream buffer": sparse idx at base, val at base + val_off; dense vals at base.
struct StreamBuf {
  char* base;
  uint64_t val_off;
};

// Stage-1 push: my input -> stage-1 partner's receive buffer [par][1] (+ flag).
struct RdPushArgs {
  const uint32_t* idx;
  const void* val;           // float or double (f64)
  uint64_t n;
  StreamBuf dst[2];          // by call parity
  Ctrl* peer;                // the stage-1 partner's control block (or my fold partner's)
  Ctrl* ctl;                 // mine
  uint64_t N;
  int validate;
  int tgt;                   // receiving stage: 1, or 0 = fold into rank i (R-28)
  int f64;                   // values are double
  uint64_t sig;              // this rank's call signature (sent with the stream)
};

struct RdStageArgs {
  // own stream (stage 1: the caller's input)
  const uint32_t* a_idx;
  const void* a_val;
  uint64_t a_n;              // stage 1 only
  int a_from_cur;            // stages > 1: my cur[(t-1)%2]
  StreamBuf cur[2];          // my cur buffers
  StreamBuf b[2];            // my receive buffer [par][t]
  uint64_t N, delta;
  // output: cur[t%2] (or the caller's out payload at the last stage)
  StreamBuf o;
  int o_cur;                 // 1: o = cur[t % 2]
  // mirror into the next partner's receive buffer [par][t+1]
  StreamBuf m[2];
  Ctrl* mpeer;               // that partner's control block (nullptr at the last stage)
  Ctrl* ctl;                 // mine
  int stage;                 // 1-based; 0 = the fold step (R-28)
  int last;
  int fold;                  // this rank folded an extra rank in (and sends it the result)
  int op;                    // reduction operator (R-30)
  int grid;                  // blocks to launch (0: the default, enough for a dense window pass)
  sparcml_header* hdr;       // last stage only
  ScanCounters* ctr;
  TileStatus* status;
  int f64;
  uint64_t sig;              // this rank's call signature (checked, and mirrored on)
};

// Extra rank of a folded RD (R-28): wait for the result my fold partner
// mirrored into my buffer, copy it into the caller's out, write the header.
struct RdUnfoldArgs {
  StreamBuf src[2];          // my receive buffer [par][L+1]
  int stage;                 // L + 1
  Ctrl* ctl;
  char* out;
  uint64_t N, val_offset;
  int f64;
  uint64_t sig;
};

// ---------------------------------------------------------- split phase ---
struct PushArgs {
  const uint32_t* idx;
  const void* val;
  uint64_t n;
  uint64_t N;
  int P, rank;
  uint64_t bnd[kMaxRanks + 1];
  uint32_t* dst_idx[kMaxRanks];    // owner j's receive region for source `rank`
  void* dst_val[kMaxRanks];
  uint32_t* dst_win[kMaxRanks];    // owner j's window-offset table for source `rank` (ntab_j + 1)
  Ctrl* peer[kMaxRanks];           // every rank's control block
  Ctrl* ctl;                       // mine
  int validate;
  int f64;
  uint64_t sig;                    // this rank's call signature (sent with the slices)
};

struct OwnerArgs {
  int P, rank;
  int algo;                        // sparcml_algo (AUTO decides on the device)
  uint64_t delta;
  uint64_t lo, hi;                 // my partition
  const uint32_t* src_idx[kMaxRanks];
  const void* src_val[kMaxRanks];
  const uint32_t* src_win[kMaxRanks];
  TreeSched sched;
  // SSAR: compacted partition result
  uint32_t* r_idx;
  void* r_val;
  // DSAR: dense partition or QSGD codes + scales (fp32 only)
  void* dense;
  uint8_t* codes;
  float* scales;
  int bits;
  uint32_t bucket;
  uint32_t seed_lo, seed_hi;
  int host_dsar;                   // -1 device decides, else 0/1
  int wait;                        // 1: wait for the sources' flags (P > 1)
  int op;                          // reduction operator (R-30)
  int qnorm;                       // QSGD scale norm (R-16 / R-31)
  Ctrl* peer[kMaxRanks];
  Ctrl* ctl;
  // SSAR merge path: spill area for dense block ranges (P * cap_s pairs, SoA)
  // and per-block output counts
  uint32_t* st_idx;
  void* st_val;
  uint64_t* blk;
  int f64;
  int pdl;                         // launch as a programmatic dependent of the push (host_dsar known)
  uint64_t sig;                    // this rank's call signature (every source's must match)
};

struct ConcatArgs {
  int P, rank;
  uint64_t N, delta;
  uint64_t bnd[kMaxRanks + 1];
  // owner j's partition result (peer pointers)
  const uint32_t* r_idx[kMaxRanks];
  const void* r_val[kMaxRanks];
  const uint64_t* r_n[kMaxRanks];
  const uint8_t* r_codes[kMaxRanks];
  const float* r_scales[kMaxRanks];
  const void* r_dense[kMaxRanks];
  Ctrl* ctl;                       // mine (dsar, k_sum, slice counts, owner flags, status)
  int wait_owners;                 // 1: wait for owner_done flags (P > 1)
  int bits;
  uint32_t bucket;
  char* out;                       // caller's out (header + payload)
  uint64_t val_offset;
  uint32_t algo;
  TileStatus* status;
  int host_dsar;                   // -1: launch both concat variants (the device decides), else 0/1
  int op;                          // reduction operator (R-30): neutral fill when densifying
  int f64;
  int pdl;                         // launch as a programmatic dependent of the owner (host_dsar known)
};

// Fused split-allgather, SSAR (split_fused_kernel): one cooperative launch per
// rank (or one for all ranks of a loopback world) does the split push, the
// owner reduction and the allgather.  Addresses in peer workspaces follow the
// symmetric layout (api.cu Layout), so only the bases and offsets travel.
constexpr int kFzMaxG = 1024;        // CTAs per rank (record slots per owner)
struct FusedArgs {
  int P, nloc, G;                    // ranks; ranks served by this launch (1, or P on a loopback world); CTAs per rank
  int rank0;                         // rank of local slot 0
  uint32_t skip;                     // loopback failure injection: local ranks whose CTAs do nothing
  uint64_t N, delta, val_offset;
  uint64_t bnd[kMaxRanks + 1];       // partition bounds (floor(N/P), remainder on the last)
  char* base[kMaxRanks];             // every rank's workspace as mapped here
  uint64_t recv_off, region_bytes, cap_s, win_off, win_bytes, stage_off;   // layout (api.cu)
  uint64_t rec_off;                  // records {cnt, slot} of owner j's CTA b: u64 [j * kFzMaxG + b]
  uint64_t fz_off, fz_bytes, fz_cap; // staging for owner j's pieces: idx[fz_cap], val[fz_cap] at fz_off + j * fz_bytes
  const uint32_t* idx[kMaxRanks];    // per local rank: input stream, nnz, result buffer, call signature
  const void* val[kMaxRanks];
  uint64_t n[kMaxRanks];
  char* out[kMaxRanks];
  uint64_t sig[kMaxRanks];
  TreeSched sched;
  int op, validate, f64;
};

struct BarrierArgs {
  Ctrl* my;
  uint32_t* peer_flags[kMaxRanks];  // &peer_p.ctrl.flags[rank]
  int P, rank;
  int loopback;                     // no waiting (all ranks on one stream)
};

struct P1PrepArgs {                 // P == 1: validate, fill the control block, (DSAR) window table
  const uint32_t* idx;
  const void* val;
  uint64_t n, N, delta;
  int algo;
  Ctrl* ctl;
  int validate;
  uint32_t* win;                    // nullable: build the window-offset table (ntab + 1 entries)
  // p1_sparse_kernel only: the result is the input itself (sparse, nnz <= delta)
  char* out;
  uint64_t val_offset;
  uint32_t algo_used;
  int copy;                         // 0: the input already is out's payload (in place)
  int f64;
};

// ------------------------------------------------------ sparse allgather --
struct AgPublishArgs {
  const uint32_t* idx;
  const void* val;                 // float or double (f64)
  uint64_t n, N;
  int P, rank;
  uint32_t* my_idx[2];             // my published copy (my workspace), by call parity
  void* my_val[2];
  Ctrl* peer[kMaxRanks];
  Ctrl* ctl;
  int validate;
  int f64;
  uint64_t sig;
};
struct AgGatherArgs {
  int P, rank;
  uint64_t N, delta;
  const uint32_t* src_idx[2][kMaxRanks];   // every rank's published stream (peer pointers), by call parity
  const void* src_val[2][kMaxRanks];
  Ctrl* ctl;
  char* out;
  uint64_t val_offset;
  int f64;
  uint64_t sig;
};

// -------------------------------------------------- layer-wise fusion ------
constexpr int kMaxLayers = 64;      // layers per fused call (by value in the kernel parameters)
struct FuseArgs {
  int L;
  const uint32_t* idx[kMaxLayers];
  const float* val[kMaxLayers];
  uint64_t pre[kMaxLayers + 1];     // prefix of the layers' nnz
  uint64_t off[kMaxLayers];         // index offset of each layer
  uint32_t* idx_out;
  float* val_out;
};
struct LayerOffsets {
  uint64_t v[kMaxLayers + 1];
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
cudaError_t launch_rd_push(const RdPushArgs& a, cudaStream_t s);
cudaError_t launch_rd_stage(const RdStageArgs& a, cudaStream_t s);
cudaError_t launch_rd_unfold(const RdUnfoldArgs& a, cudaStream_t s);
cudaError_t launch_split_push(const PushArgs& a, cudaStream_t s);
cudaError_t launch_owner(const OwnerArgs& a, cudaStream_t s);   // host_dsar selects merge / window
int split_fused_grid(int P, bool f64, int nloc);                  // CTAs per rank (0: cannot run)
cudaError_t launch_split_fused(const FusedArgs& a, cudaStream_t s);
cudaError_t launch_concat(const ConcatArgs& a, cudaStream_t s);
cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s);
cudaError_t launch_p1_prep(const P1PrepArgs& a, cudaStream_t s);
cudaError_t launch_p1_sparse(const P1PrepArgs& a, cudaStream_t s);
cudaError_t launch_fuse_streams(const FuseArgs& a, cudaStream_t s);
cudaError_t launch_apply_update(float* v, const char* out, cudaStream_t s);
cudaError_t launch_apply_update_f64(double* v, const char* out, cudaStream_t s);
cudaError_t launch_ag_publish(const AgPublishArgs& a, cudaStream_t s);
cudaError_t launch_ag_gather(const AgGatherArgs& a, cudaStream_t s);
cudaError_t launch_layer_ranges(const char* out, int L, const LayerOffsets& off, uint64_t* starts, cudaStream_t s);

// top-k / QSGD (kernels_topk.cu, kernels_qsgd.cu)
size_t topk_workspace_bytes(uint64_t N, uint64_t k);
size_t topk_sample_positions(uint64_t N, uint64_t* pos, size_t cap);   // diagnostics (tests)
cudaError_t launch_topk(const float* x, const float* grad, float alpha, int ef, float* x_out,
                        uint64_t N, uint64_t k, uint32_t* idx_out, float* val_out, float* residual,
                        void* ws, cudaStream_t s);
// bucket = 128 * R, R in 1..8; dst = new eps (ef), residual (nullable) otherwise; ws nullable (status)
cudaError_t launch_topk_bucketed(const float* x, const float* grad, float alpha, int ef, float* dst, uint64_t N,
                                 uint64_t k, uint64_t bucket, uint32_t* idx_out, float* val_out, void* ws,
                                 cudaStream_t s);
cudaError_t launch_quantize(const float* x, uint64_t n, int bits, uint32_t bucket, uint64_t seed,
                            uint64_t ctr_base, uint8_t* codes, float* scales, cudaStream_t s, int norm = 0);
cudaError_t launch_dequantize(const uint8_t* codes, const float* scales, uint64_t n, int bits,
                              uint32_t bucket, float* out, cudaStream_t s);

}  // namespace sparcml
