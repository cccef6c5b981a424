// api.cu — the C ABI of include/sparcml.h: argument checks, the symmetric
// workspace and its CUDA-IPC mapping, and the host-side schedule of each
// collective (which kernels, barriers and buffers, in which order).  Every
// step of the method runs in the kernels; this file only enqueues them.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"

using namespace sparcml;

namespace sparcml {
cudaError_t topk_read_status(const void* ws, uint32_t* status, uint32_t* passes, cudaStream_t s);
}

namespace {

thread_local std::string g_last_error;

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

uint64_t half_cap(uint64_t N) {   // H = ceil4(floor(N/2)): sparse slots in a result
  return align_up(N / 2, 4);
}

// fp64 values: delta = floor(N*8/12) (P:488-491 with isize = 8)
uint64_t cap64(uint64_t N) { return align_up(N * 8 / 12, 4); }

// ---------------------------------------------------------------------------
// canonical tree over ranks (reading R-8): tree(lo,hi) = tree(lo,mid) + tree(mid,hi)
// ---------------------------------------------------------------------------
struct TreeNode {
  int lo, mid, hi, height, id;   // id: index of internal node (post-order)
  int left, right;               // child node ids, -1 for leaves (then leaf = lo / mid)
};

int build_tree(int lo, int hi, std::vector<TreeNode>& nodes) {   // returns node id or -1 (leaf)
  if (hi - lo == 1) return -1;
  const int mid = lo + (hi - lo) / 2;
  const int l = build_tree(lo, mid, nodes), r = build_tree(mid, hi, nodes);
  TreeNode n;
  n.lo = lo;
  n.mid = mid;
  n.hi = hi;
  n.left = l;
  n.right = r;
  n.height = 1 + std::max(l < 0 ? 0 : nodes[l].height, r < 0 ? 0 : nodes[r].height);
  n.id = (int)nodes.size();
  nodes.push_back(n);
  return n.id;
}

TreeSched make_sched(int P) {
  std::vector<TreeNode> nodes;
  build_tree(0, P, nodes);
  TreeSched ts = {};
  ts.n = (int)nodes.size();
  for (size_t i = 0; i < nodes.size(); ++i) {   // post-order: children before parents
    ts.dst[i] = (uint8_t)nodes[i].lo;
    ts.src[i] = (uint8_t)nodes[i].mid;
    ts.h[i] = (uint8_t)nodes[i].height;
    ts.hmax = std::max(ts.hmax, nodes[i].height);
    const int hh = nodes[i].height - 1;
    ts.role[hh][nodes[i].lo] = 1;
    ts.part[hh][nodes[i].lo] = (uint8_t)nodes[i].mid;
    ts.role[hh][nodes[i].mid] = 2;
    ts.part[hh][nodes[i].mid] = (uint8_t)nodes[i].lo;
  }
  return ts;
}

// ---------------------------------------------------------------------------
// symmetric workspace layout (identical on every rank)
// ---------------------------------------------------------------------------
struct Layout {
  int P, L;                 // ranks, recursive-doubling stages (0 if P is not a power of two)
  uint64_t max_N, max_nnz;
  uint64_t part_cap;        // largest partition (rounded to 64)
  uint64_t cap_s;           // pairs per receive region (one per source)
  uint64_t nwin;            // windows of the largest partition
  uint64_t ntab;            // window-offset table entries of the largest partition (kTab positions each)
  size_t status_off, n_status;
  size_t recv_off, region_bytes;
  size_t win_off, win_bytes;            // per-source window-offset tables (ntab + 1 each)
  size_t stage_off;                     // owner spill area: P * cap_s pairs (SoA)
  size_t blk_off;                       // owner per-block output counts
  size_t part_off, part_bytes, scales_off;
  size_t rd_off, rd_bytes, rd_val_off;  // cur[2] + recv[2 parities][L stages]
  size_t ag_off, ag_val_off, ag_bytes;  // sparse allgather: my published stream (max_nnz pairs) x 2 call parities
  size_t rec_off;                       // fused split-allgather: owner pieces' records (P x kFzMaxG)
  size_t fz_off, fz_bytes;              // ... and their staging, per owner
  uint64_t fz_cap;                      // pairs per owner's staging
  size_t total;
};

constexpr uint64_t kDefaultTimeoutNs = 10ull * 1000 * 1000 * 1000;   // flag waits give up after 10 s

Layout make_layout(int P, uint64_t max_N, uint64_t max_nnz) {
  Layout L;
  L.P = P;
  L.max_N = max_N;
  L.max_nnz = max_nnz;
  L.part_cap = align_up(max_N / P + P, 64);
  // pairs per receive region: the fused split push keeps each element's STREAM
  // index (up to max_nnz - 1), not its slice position; val[] 16-byte aligned
  L.cap_s = align_up(std::max<uint64_t>(max_nnz, 1), 4);
  L.nwin = (L.part_cap + kWin - 1) / kWin;
  L.ntab = (L.part_cap + kTab - 1) / kTab;
  size_t off = align_up(sizeof(Ctrl), 256);
  L.status_off = off;
  L.n_status = max_N / 1024 + 2 * max_nnz / kMergeTile + 2048;   // >= any stage grid (merge_span block counts)
  off = align_up(off + L.n_status * sizeof(TileStatus), 256);
  L.recv_off = off;
  // receive regions, spill area, partition result and RD buffers are sized
  // for 8-byte values (fp64 calls); fp32 calls use the same idx offsets
  L.region_bytes = align_up(12 * L.cap_s, 256);
  off += (size_t)P * L.region_bytes;
  L.win_off = off;
  L.win_bytes = align_up(4 * (L.ntab + 1), 256);
  off += (size_t)P * L.win_bytes;
  L.stage_off = off;
  off += align_up(12 * (size_t)P * L.cap_s, 256);
  L.blk_off = off;
  off += align_up(8 * 8192, 256);
  L.part_off = off;
  L.part_bytes = align_up(12 * L.part_cap + 256, 256);
  L.scales_off = off + align_up(L.part_cap + 16, 256);   // codes <= part_cap bytes (8 bits)
  off += L.part_bytes;
  L.L = 0;   // stages of recursive doubling over P' = the largest power of two <= P (R-28)
  while ((2 << L.L) <= P) ++L.L;
  L.rd_off = off;
  // sparse slots: stage outputs hold <= delta <= 2N/3 pairs (fp64; N/2 fp32),
  // the stage-1 push a whole input
  const uint64_t rd_pairs = std::max<uint64_t>(cap64(max_N), max_nnz);
  L.rd_val_off = align_up(4 * rd_pairs + 64, 256);
  L.rd_bytes = align_up(std::max<size_t>(L.rd_val_off + 8 * rd_pairs, 8 * max_N) + 256, 256);
  // cur x2 + recv[2 parities][stages 0..L+1] (0: fold in, L+1: result out, R-28)
  if (P > 1) off += (size_t)(2 + 2 * (L.L + 2)) * L.rd_bytes;
  L.ag_off = off;
  L.ag_val_off = align_up(4 * max_nnz, 256);
  L.ag_bytes = align_up(L.ag_val_off + 8 * max_nnz, 256);   // values up to 8 bytes (fp64)
  off += 2 * L.ag_bytes;
  // fused split-allgather: owner j's pieces land at slots <= min(its inputs,
  // its partition's positions) + 4 per CTA (split_fused_kernel)
  L.rec_off = off;
  off += align_up((size_t)P * kFzMaxG * 8, 256);
  L.fz_cap = align_up(std::min<uint64_t>((uint64_t)P * L.cap_s, L.part_cap + kTab) + 4 * (uint64_t)kFzMaxG + 4, 4);
  L.fz_off = off;
  L.fz_bytes = P > 1 ? align_up(12 * L.fz_cap, 256) : 0;
  off += (size_t)P * L.fz_bytes;
  L.total = align_up(off, 1 << 20);
  return L;
}

}  // namespace

struct sparcml_comm {
  int P = 1, rank = 0, device = 0;
  bool local = false, connected = false;
  Layout L;
  std::vector<char*> own;    // workspaces allocated here (local: P, ipc: 1)
  std::vector<char*> peer;   // every rank's workspace as seen from this process
  std::vector<bool> opened;  // peer[p] came from cudaIpcOpenMemHandle
  cudaIpcMemHandle_t handle;
  std::string err;
  uint64_t inject_skip = 0;  // loopback failure injection: ranks whose kernels are not launched
  uint64_t inject_sig = 0;   // r + 1: rank r calls with a perturbed signature
};

namespace {

sparcml_status fail(sparcml_comm* c, sparcml_status s, const std::string& msg) {
  g_last_error = msg;
  if (c) c->err = msg;
  return s;
}

sparcml_status cuda_fail(sparcml_comm* c, cudaError_t e, const char* what) {
  return fail(c, SPARCML_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(c, x)                                   \
  do {                                             \
    cudaError_t e_ = (x);                          \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #x); \
  } while (0)

inline Ctrl* ctrl_of(char* base) { return reinterpret_cast<Ctrl*>(base); }
inline TileStatus* status_of(const Layout& L, char* base) {
  return reinterpret_cast<TileStatus*>(base + L.status_off);
}
inline uint32_t* recv_idx(const Layout& L, char* base, int src) {
  return reinterpret_cast<uint32_t*>(base + L.recv_off + (size_t)src * L.region_bytes);
}
inline float* recv_val(const Layout& L, char* base, int src) {
  return reinterpret_cast<float*>(base + L.recv_off + (size_t)src * L.region_bytes + 4 * L.cap_s);
}
inline uint32_t* win_table(const Layout& L, char* base, int src) {
  return reinterpret_cast<uint32_t*>(base + L.win_off + (size_t)src * L.win_bytes);
}
inline StreamBuf rd_cur(const Layout& L, char* base, int i) {
  StreamBuf b;
  b.base = base + L.rd_off + (size_t)i * L.rd_bytes;
  b.val_off = L.rd_val_off;
  return b;
}
inline StreamBuf rd_recv(const Layout& L, char* base, int par, int t) {   // t = 0..L+1
  StreamBuf b;
  b.base = base + L.rd_off + (size_t)(2 + par * (L.L + 2) + t) * L.rd_bytes;
  b.val_off = L.rd_val_off;
  return b;
}

uint64_t effective_delta(uint64_t N, const sparcml_opts& o, int vbytes = 4) {
  // delta = floor(scale * N*isize/(c+isize)), c = 4: N/2 (fp32), 2N/3 (fp64);
  // never above the result capacity
  const uint64_t d =
      (uint64_t)std::floor((double)o.switch_scale * (double)N * vbytes / (double)(o.index_bytes + vbytes));
  return std::min<uint64_t>(d, vbytes == 8 ? N * 8 / 12 : N / 2);
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

// AUTO's recursive-doubling vs split-allgather crossover (RD for
// small data), MEASURED on this box by tools/auto_crossover.py
// (profiles/r02_auto_crossover_p2.log, _p4.log): the largest sum_i k_i * 8
// bytes at which recursive doubling still beat split-allgather, per P.  On 2
// and 4 B200 over NVSwitch it never did (N = 2^12 .. 2^24, densities 1/16 ..
// 1/256: split 35-82 us vs RD 39-94 us at P = 2, 37-139 vs 74-225 us at P = 4):
// every exchange is one hop, so RD's fewer alpha terms buy nothing and its
// log2(P) dependent stages cost more.  P = 8 is unmeasured and takes P = 4's
// entry.  0 = AUTO never picks RD.
constexpr uint64_t kRdMaxBytes[SPARCML_MAX_RANKS + 1] = {0};

bool auto_picks_rd(int P, uint64_t ksum_bytes) {
  if (!is_pow2(P) || P > SPARCML_MAX_RANKS) return false;
  const uint64_t lim = kRdMaxBytes[P];
  return lim > 0 && ksum_bytes <= lim;
}

// Programmatic dependent launch of the owner and concat kernels: opt-in
// (SPARCML_PDL=1).  Correct (same tests, stress), but measured slower: +1 us at
// P = 2 and +5 us at P = 4 per allreduce (profiles/r01_ab_pdl.log) -- the early
// blocks spin on flags on SMs the push / owner still needs.
bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("SPARCML_PDL");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

sparcml_status check_opts(sparcml_comm* c, const sparcml_opts& o) {
  if (o.index_bytes != 4) return fail(c, SPARCML_ERR_INVALID_ARG, "index_bytes must be 4 (u32 indices, P:931)");
  if (!(o.switch_scale > 0.0f) || o.switch_scale > 1.0f)
    return fail(c, SPARCML_ERR_INVALID_ARG, "switch_scale must be in (0, 1]");
  if (o.quant_bits != 0 && o.quant_bits != 2 && o.quant_bits != 4 && o.quant_bits != 8)
    return fail(c, SPARCML_ERR_INVALID_ARG, "quant_bits must be 0, 2, 4 or 8");
  if (o.quant_bits && (o.quant_bucket < 8 || o.quant_bucket > 1024 || (o.quant_bucket & (o.quant_bucket - 1))))
    return fail(c, SPARCML_ERR_INVALID_ARG, "quant_bucket must be a power of two in [8, 1024]");
  if (o.quant_norm != 0 && o.quant_norm != 1) return fail(c, SPARCML_ERR_INVALID_ARG, "quant_norm must be 0 or 1");
  if (o.algo < SPARCML_ALGO_AUTO || o.algo > SPARCML_DSAR_SPLIT_ALLGATHER)
    return fail(c, SPARCML_ERR_INVALID_ARG, "unknown algorithm");
  return SPARCML_OK;
}

// per-call parameters shared by all local ranks
struct CallCtx {
  uint64_t N, delta, val_offset;
  int f64;             // values are double
  sparcml_opts o;
  int algo;            // resolved: RD, SPLIT (SSAR/DSAR/AUTO decided below)
  int host_dsar;       // -1 unknown (device decides), 0/1 known
  int op;              // reduction operator (R-30)
  cudaStream_t s;
  uint64_t sig;        // call signature: every rank's must agree
};

// FNV-1a over the arguments every rank must pass identically
uint64_t call_signature(uint64_t N, int op, const sparcml_opts& o, int f64, int kind) {
  uint64_t h = 0xcbf29ce484222325ull;
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xFFu;
      h *= 0x100000001b3ull;
    }
  };
  uint32_t sc;
  std::memcpy(&sc, &o.switch_scale, 4);
  mix(N); mix((uint64_t)op); mix((uint64_t)o.algo); mix(sc); mix((uint64_t)o.index_bytes);
  mix((uint64_t)o.quant_bits); mix(o.quant_bucket); mix(o.seed); mix(o.k_sum_hint); mix((uint64_t)o.quant_norm);
  mix((uint64_t)f64); mix((uint64_t)kind);
  return h;
}

inline uint64_t rank_sig(const sparcml_comm* c, uint64_t sig, int r) {
  return c->inject_sig == (uint64_t)r + 1 ? sig ^ 0x9E3779B97F4A7C15ull : sig;
}
inline bool skipped(const sparcml_comm* c, int r) { return c->local && ((c->inject_skip >> r) & 1u); }

BarrierArgs barrier_args(sparcml_comm* c, int r) {
  BarrierArgs b = {};
  b.my = ctrl_of(c->peer[r]);
  b.P = c->P;
  b.rank = r;
  b.loopback = c->local ? 1 : 0;
  for (int p = 0; p < c->P; ++p) b.peer_flags[p] = &ctrl_of(c->peer[p])->flags[r];
  return b;
}

// ------------------------------------------------------------ RD schedule ---
// push (stage-1 partner) ; stage 1 .. L, each waiting for its partner's flag
sparcml_status run_rd(sparcml_comm* c, const std::vector<int>& R, const uint32_t* const* idx,
                      const void* const* val, const uint64_t* nnz, char* const* out, const CallCtx& cc) {
  const Layout& L = c->L;
  const int Lg = L.L;
  const int P2 = 1 << Lg, E = c->P - P2;   // R-28: extra ranks P2..P-1 fold into 0..E-1
  uint64_t max_in = L.max_nnz;             // bound on every rank's input (the comm's capacity)
  for (size_t i = 0; i < R.size(); ++i) max_in = std::max<uint64_t>(max_in, nnz[i]);
  auto pos = [&](int r) -> int {           // R's slot of rank r (loopback: every rank)
    if (skipped(c, r)) return -1;          // failure injection: a dead rank launches nothing
    for (size_t i = 0; i < R.size(); ++i)
      if (R[i] == r) return (int)i;
    return -1;
  };
  auto push = [&](int i, int r, int q, int tgt) -> sparcml_status {
    RdPushArgs a = {};
    a.idx = idx[i];
    a.val = val[i];
    a.n = nnz[i];
    a.dst[0] = rd_recv(L, c->peer[q], 0, tgt);
    a.dst[1] = rd_recv(L, c->peer[q], 1, tgt);
    a.peer = ctrl_of(c->peer[q]);
    a.ctl = ctrl_of(c->peer[r]);
    a.N = cc.N;
    a.validate = cc.o.validate;
    a.tgt = tgt;
    a.f64 = cc.f64;
    a.sig = rank_sig(c, cc.sig, r);
    CK(c, launch_rd_push(a, cc.s));
    return SPARCML_OK;
  };
  auto stage = [&](int i, int r, int t) -> sparcml_status {
    char* base = c->peer[r];
    const bool folded = r < E;
    RdStageArgs a = {};
    a.a_idx = idx[i];
    a.a_val = val[i];
    a.a_n = nnz[i];
    a.a_from_cur = t > 1 || (t == 1 && folded);
    a.cur[0] = rd_cur(L, base, 0);
    a.cur[1] = rd_cur(L, base, 1);
    a.b[0] = rd_recv(L, base, 0, t);
    a.b[1] = rd_recv(L, base, 1, t);
    a.N = cc.N;
    a.delta = cc.delta;
    a.fold = folded && t == Lg;
    a.op = cc.op;
    if (t == Lg) {
      a.o.base = out[i] + SPARCML_HEADER_BYTES;
      a.o.val_off = cc.val_offset - SPARCML_HEADER_BYTES;
      a.o_cur = 0;
      a.hdr = reinterpret_cast<sparcml_header*>(out[i]);
      a.last = 1;
    } else {
      a.o_cur = 1;
    }
    int q = -1;   // whose receive buffer [t+1] my output is mirrored into
    if (t < Lg) q = r ^ (1 << t);   // the next stage's partner (t = 0: the stage-1 partner)
    else if (folded) q = P2 + r;    // the result out to my extra rank
    if (q >= 0) {
      a.m[0] = rd_recv(L, c->peer[q], 0, t + 1);
      a.m[1] = rd_recv(L, c->peer[q], 1, t + 1);
      a.mpeer = ctrl_of(c->peer[q]);
    }
    a.ctl = ctrl_of(base);
    a.stage = t;
    // the stage's input is at most 2^t inputs of <= max_nnz pairs (t = 0: two); if
    // that cannot pass delta the output is sparse for sure: launch only the merge
    // tiles it can need instead of a grid sized for a dense window pass
    {
      const uint64_t ub = std::min<uint64_t>(cc.N, (uint64_t)max_in << (t == 0 ? 1 : t + (E > 0 ? 1 : 0)));
      a.grid = ub <= cc.delta ? (int)std::max<uint64_t>(1, (ub + kMergeTile - 1) / kMergeTile) : 0;
    }
    a.ctr = &ctrl_of(base)->scan[0];
    a.status = status_of(L, base);
    a.f64 = cc.f64;
    a.sig = rank_sig(c, cc.sig, r);
    CK(c, launch_rd_stage(a, cc.s));
    return SPARCML_OK;
  };
  sparcml_status st;
  // front: extra ranks push into their fold partner; the others push to their stage-1 partner
  for (int r = P2; r < c->P; ++r) {
    const int i = pos(r);
    if (i >= 0 && (st = push(i, r, r - P2, 0)) != SPARCML_OK) return st;
  }
  for (int r = E; r < P2; ++r) {
    const int i = pos(r);
    if (i >= 0 && (st = push(i, r, r ^ 1, 1)) != SPARCML_OK) return st;
  }
  for (int r = 0; r < E; ++r) {   // the fold step: sum the extra rank in, mirror to the stage-1 partner
    const int i = pos(r);
    if (i >= 0 && (st = stage(i, r, 0)) != SPARCML_OK) return st;
  }
  for (int t = 1; t <= Lg; ++t)
    for (int r = 0; r < P2; ++r) {
      const int i = pos(r);
      if (i >= 0 && (st = stage(i, r, t)) != SPARCML_OK) return st;
    }
  for (int r = P2; r < c->P; ++r) {   // end: the extra ranks take their partner's result
    const int i = pos(r);
    if (i < 0) continue;
    RdUnfoldArgs u = {};
    u.src[0] = rd_recv(L, c->peer[r], 0, Lg + 1);
    u.src[1] = rd_recv(L, c->peer[r], 1, Lg + 1);
    u.stage = Lg + 1;
    u.ctl = ctrl_of(c->peer[r]);
    u.out = out[i];
    u.N = cc.N;
    u.val_offset = cc.val_offset;
    u.f64 = cc.f64;
    u.sig = rank_sig(c, cc.sig, r);
    CK(c, launch_rd_unfold(u, cc.s));
  }
  return SPARCML_OK;
}

// --------------------------------------------------------- split schedule ---
// push (slices + window tables -> owners) ; owner reduction (waits for the P
// slices) ; pull-concat (waits for the P owners)
// SPARCML_FUSED=0 selects the three-kernel split path (push, owner, concat)
// even when SSAR is known on the host (A/B runs and its tests); read per call.
bool fused_enabled() {
  const char* e = std::getenv("SPARCML_FUSED");
  return !(e && e[0] == '0');
}

sparcml_status run_split(sparcml_comm* c, const std::vector<int>& R, const uint32_t* const* idx,
                         const void* const* val, const uint64_t* nnz, char* const* out, const CallCtx& cc) {
  const Layout& L = c->L;
  const int P = c->P;
  const uint64_t part = cc.N / P;
  uint64_t bnd[kMaxRanks + 1];
  for (int j = 0; j < P; ++j) bnd[j] = (uint64_t)j * part;
  bnd[P] = cc.N;
  // SSAR known on the host: one fused kernel does push, owner reduction and allgather
  const int nloc = (int)R.size();
  const int G = cc.host_dsar == 0 && fused_enabled() ? split_fused_grid(P, cc.f64 != 0, nloc) : 0;
  if (G > 0) {
    FusedArgs a = {};
    a.P = P;
    a.nloc = nloc;
    a.G = G;
    a.rank0 = R[0];
    a.N = cc.N;
    a.delta = cc.delta;
    a.val_offset = cc.val_offset;
    for (int j = 0; j <= P; ++j) a.bnd[j] = bnd[j];
    for (int j = 0; j < P; ++j) a.base[j] = c->peer[j];
    a.recv_off = L.recv_off;
    a.region_bytes = L.region_bytes;
    a.cap_s = L.cap_s;
    a.win_off = L.win_off;
    a.win_bytes = L.win_bytes;
    a.stage_off = L.stage_off;
    a.rec_off = L.rec_off;
    a.fz_off = L.fz_off;
    a.fz_bytes = L.fz_bytes;
    a.fz_cap = L.fz_cap;
    for (int i = 0; i < nloc; ++i) {
      a.idx[i] = idx[i];
      a.val[i] = val[i];
      a.n[i] = nnz[i];
      a.out[i] = out[i];
      a.sig[i] = rank_sig(c, cc.sig, R[i]);
      if (skipped(c, R[i])) a.skip |= 1u << i;
    }
    a.sched = make_sched(P);
    a.op = cc.op;
    a.validate = cc.o.validate;
    a.f64 = cc.f64;
    CK(c, launch_split_fused(a, cc.s));
    return SPARCML_OK;
  }
  for (size_t i = 0; i < R.size(); ++i) {
    const int r = R[i];
    if (skipped(c, r)) continue;
    PushArgs a = {};
    a.idx = idx[i];
    a.val = val[i];
    a.n = nnz[i];
    a.N = cc.N;
    a.P = P;
    a.rank = r;
    for (int j = 0; j <= P; ++j) a.bnd[j] = bnd[j];
    for (int j = 0; j < P; ++j) {
      a.dst_idx[j] = recv_idx(L, c->peer[j], r);
      a.dst_val[j] = recv_val(L, c->peer[j], r);
      a.dst_win[j] = win_table(L, c->peer[j], r);
      a.peer[j] = ctrl_of(c->peer[j]);
    }
    a.ctl = ctrl_of(c->peer[r]);
    a.validate = cc.o.validate;
    a.f64 = cc.f64;
    a.sig = rank_sig(c, cc.sig, r);
    CK(c, launch_split_push(a, cc.s));
  }
  const TreeSched ts = make_sched(P);
  for (size_t i = 0; i < R.size(); ++i) {
    const int r = R[i];
    if (skipped(c, r)) continue;
    char* base = c->peer[r];
    OwnerArgs w = {};
    w.P = P;
    w.rank = r;
    w.algo = cc.o.algo == SPARCML_SSAR_RECURSIVE_DOUBLE ? SPARCML_ALGO_AUTO : cc.o.algo;
    w.delta = cc.delta;
    w.lo = bnd[r];
    w.hi = bnd[r + 1];
    for (int s = 0; s < P; ++s) {
      w.src_idx[s] = recv_idx(L, base, s);
      w.src_val[s] = recv_val(L, base, s);
      w.src_win[s] = win_table(L, base, s);
      w.peer[s] = ctrl_of(c->peer[s]);
    }
    w.sched = ts;
    w.r_idx = reinterpret_cast<uint32_t*>(base + L.part_off);
    w.r_val = base + L.part_off + 4 * L.part_cap;
    w.dense = base + L.part_off;
    w.codes = reinterpret_cast<uint8_t*>(base + L.part_off);
    w.scales = reinterpret_cast<float*>(base + L.scales_off);
    w.bits = cc.o.quant_bits;
    w.bucket = cc.o.quant_bucket;
    w.seed_lo = (uint32_t)cc.o.seed;
    w.seed_hi = (uint32_t)(cc.o.seed >> 32);
    w.host_dsar = cc.host_dsar;
    w.wait = 1;
    w.op = cc.op;
    w.qnorm = cc.o.quant_norm;
    w.ctl = ctrl_of(base);
    w.st_idx = reinterpret_cast<uint32_t*>(base + L.stage_off);
    w.st_val = base + L.stage_off + 4 * (size_t)P * L.cap_s;
    w.blk = reinterpret_cast<uint64_t*>(base + L.blk_off);
    w.f64 = cc.f64;
    w.pdl = cc.host_dsar >= 0 && pdl_enabled() ? 1 : 0;   // one owner kernel: it may start during the push
    w.sig = rank_sig(c, cc.sig, r);
    CK(c, launch_owner(w, cc.s));
  }
  for (size_t i = 0; i < R.size(); ++i) {
    const int r = R[i];
    if (skipped(c, r)) continue;
    ConcatArgs a = {};
    a.P = P;
    a.rank = r;
    a.N = cc.N;
    a.delta = cc.delta;
    for (int j = 0; j <= P; ++j) a.bnd[j] = bnd[j];
    for (int j = 0; j < P; ++j) {
      char* pb = c->peer[j];
      a.r_idx[j] = reinterpret_cast<const uint32_t*>(pb + L.part_off);
      a.r_val[j] = pb + L.part_off + 4 * L.part_cap;
      a.r_n[j] = &ctrl_of(pb)->owner_K;
      a.r_codes[j] = reinterpret_cast<const uint8_t*>(pb + L.part_off);
      a.r_scales[j] = reinterpret_cast<const float*>(pb + L.scales_off);
      a.r_dense[j] = pb + L.part_off;
    }
    a.ctl = ctrl_of(c->peer[r]);
    a.wait_owners = 1;
    a.bits = cc.o.quant_bits;
    a.bucket = cc.o.quant_bucket ? cc.o.quant_bucket : 1024;
    a.out = out[i];
    a.val_offset = cc.val_offset;
    a.algo = SPARCML_SSAR_SPLIT_ALLGATHER;
    a.status = status_of(L, c->peer[r]);
    a.host_dsar = cc.host_dsar;
    a.op = cc.op;
    a.f64 = cc.f64;
    a.pdl = cc.host_dsar >= 0 && pdl_enabled() ? 1 : 0;
    CK(c, launch_concat(a, cc.s));
  }
  return SPARCML_OK;
}

// ------------------------------------------------------------- P == 1 ---
sparcml_status run_p1(sparcml_comm* c, const uint32_t* idx, const void* val, uint64_t n, char* out,
                      const CallCtx& cc) {
  const Layout& L = c->L;
  char* base = c->peer[0];
  Ctrl* my = ctrl_of(base);
  P1PrepArgs p = {};
  p.idx = idx;
  p.val = val;
  p.n = n;
  p.N = cc.N;
  p.delta = cc.delta;
  p.algo = cc.o.algo;
  p.ctl = my;
  p.validate = cc.o.validate;
  p.f64 = cc.f64;
  const bool dsar = cc.o.algo == SPARCML_DSAR_SPLIT_ALLGATHER || (cc.o.algo == SPARCML_ALGO_AUTO && n > cc.delta);
  const bool inplace = reinterpret_cast<const char*>(idx) == out + SPARCML_HEADER_BYTES &&
                       reinterpret_cast<const char*>(val) == out + cc.val_offset;
  if (!dsar && n <= cc.delta) {   // the result is the input: one copy kernel (or just the header) is the call
    p.out = out;
    p.val_offset = cc.val_offset;
    p.algo_used = cc.o.algo == SPARCML_ALGO_AUTO ? SPARCML_SSAR_SPLIT_ALLGATHER : cc.o.algo;
    p.copy = inplace ? 0 : 1;
    CK(c, launch_p1_sparse(p, cc.s));
    return SPARCML_OK;
  }
  if (inplace && !dsar)
    return fail(c, SPARCML_ERR_INVALID_ARG, "in-place input with nnz > delta under forced SSAR (the dense result overwrites it)");
  p.win = dsar ? win_table(L, base, 0) : nullptr;
  CK(c, launch_p1_prep(p, cc.s));
  ConcatArgs a = {};
  a.P = 1;
  a.rank = 0;
  a.N = cc.N;
  a.delta = cc.delta;
  a.bnd[0] = 0;
  a.bnd[1] = cc.N;
  a.r_idx[0] = idx;
  a.r_val[0] = val;
  a.r_n[0] = &my->owner_K;
  if (dsar) {   // densify (+ QSGD) the one partition with the DSAR owner kernel
    OwnerArgs w = {};
    w.P = 1;
    w.rank = 0;
    w.algo = SPARCML_DSAR_SPLIT_ALLGATHER;
    w.delta = cc.delta;
    w.lo = 0;
    w.hi = cc.N;
    w.src_idx[0] = idx;
    w.src_val[0] = val;
    w.src_win[0] = win_table(L, base, 0);   // built by p1_prep
    w.sched = make_sched(1);
    w.dense = base + L.part_off;
    w.codes = reinterpret_cast<uint8_t*>(base + L.part_off);
    w.scales = reinterpret_cast<float*>(base + L.scales_off);
    w.bits = cc.o.quant_bits;
    w.bucket = cc.o.quant_bucket;
    w.seed_lo = (uint32_t)cc.o.seed;
    w.seed_hi = (uint32_t)(cc.o.seed >> 32);
    w.f64 = cc.f64;
    w.host_dsar = 1;
    w.wait = 0;
    w.op = cc.op;
    w.qnorm = cc.o.quant_norm;
    w.peer[0] = my;
    w.ctl = my;
    CK(c, launch_owner(w, cc.s));
    a.r_codes[0] = reinterpret_cast<const uint8_t*>(base + L.part_off);
    a.r_scales[0] = reinterpret_cast<const float*>(base + L.scales_off);
    a.r_dense[0] = base + L.part_off;
  }
  a.ctl = my;
  a.wait_owners = 0;
  a.bits = cc.o.quant_bits;
  a.bucket = cc.o.quant_bucket ? cc.o.quant_bucket : 1024;
  a.out = out;
  a.val_offset = cc.val_offset;
  a.algo = cc.o.algo == SPARCML_ALGO_AUTO ? SPARCML_SSAR_SPLIT_ALLGATHER : cc.o.algo;
  a.status = status_of(L, base);
  a.host_dsar = dsar ? 1 : 0;
  a.op = cc.op;
  a.f64 = cc.f64;
  CK(c, launch_concat(a, cc.s));
  return SPARCML_OK;
}

sparcml_status allreduce_impl(sparcml_comm* c, const uint32_t* const* idx, const void* const* val,
                              const uint64_t* nnz, uint64_t N, sparcml_op op, const sparcml_opts* opts,
                              void* const* out, size_t out_bytes, void* stream, int f64 = 0) {
  if (!c) return fail(c, SPARCML_ERR_INVALID_ARG, "null communicator");
  if (!c->connected) return fail(c, SPARCML_ERR_STATE, "communicator not connected");
  if (op != SPARCML_OP_SUM && op != SPARCML_OP_MAX && op != SPARCML_OP_MIN)
    return fail(c, SPARCML_ERR_INVALID_ARG, "op must be SUM, MAX or MIN");
  if (N == 0 || N > c->L.max_N) return fail(c, SPARCML_ERR_INVALID_ARG, "N must be in [1, max_N]");
  if (N > 0xFFFFFFFFull) return fail(c, SPARCML_ERR_INVALID_ARG, "N must fit u32 indices");
  if ((uint64_t)c->P > N) return fail(c, SPARCML_ERR_INVALID_ARG, "N must be >= nranks");
  sparcml_opts o;
  sparcml_opts_default(&o);
  if (opts) o = *opts;
  sparcml_status st = check_opts(c, o);
  if (st != SPARCML_OK) return st;
  if (o.quant_bits && op != SPARCML_OP_SUM)
    return fail(c, SPARCML_ERR_INVALID_ARG, "QSGD (quant_bits) requires SPARCML_OP_SUM");
  if (f64 && o.quant_bits)
    return fail(c, SPARCML_ERR_INVALID_ARG, "QSGD (quant_bits) is defined on fp32 values only");
  if (out_bytes < (f64 ? sparcml_result_bytes_f64(N) : sparcml_result_bytes(N)))
    return fail(c, SPARCML_ERR_INVALID_ARG, "out_bytes < sparcml_result_bytes(N) (_f64 for double values)");
  const int nl = c->local ? c->P : 1;
  uint64_t ksum_host = 0;
  for (int i = 0; i < nl; ++i) {
    if (nnz[i] > c->L.max_nnz) return fail(c, SPARCML_ERR_INVALID_ARG, "nnz > max_nnz");
    if (nnz[i] > N) return fail(c, SPARCML_ERR_INVALID_ARG, "nnz > N");
    if (nnz[i] > 0 && (!idx[i] || !val[i])) return fail(c, SPARCML_ERR_INVALID_ARG, "null input with nnz > 0");
    if (!out[i]) return fail(c, SPARCML_ERR_INVALID_ARG, "null out");
    if ((reinterpret_cast<uintptr_t>(out[i]) & 15u) != 0) return fail(c, SPARCML_ERR_INVALID_ARG, "out must be 16-byte aligned");
    ksum_host += nnz[i];
  }
  CallCtx cc;
  cc.N = N;
  cc.o = o;
  cc.f64 = f64;
  cc.delta = effective_delta(N, o, f64 ? 8 : 4);
  cc.val_offset = f64 ? sparcml_result_val_offset_f64(N) : sparcml_result_val_offset(N);
  cc.op = (int)op;
  cc.s = static_cast<cudaStream_t>(stream);
  cc.sig = call_signature(N, (int)op, o, f64, 0);
  CK(c, cudaSetDevice(c->device));
  // algorithm: AUTO -> recursive doubling for small data (latency-bound,
  // P:635-650), split-allgather otherwise; RD needs P = 2^m
  int algo = o.algo;
  if (algo == SPARCML_ALGO_AUTO && c->P > 1) {
    // the data volume every rank agrees on: the exact sum (loopback), the hint, or the bound P*N
    const uint64_t ksum = c->local ? ksum_host : (o.k_sum_hint ? o.k_sum_hint : (uint64_t)c->P * N);
    algo = auto_picks_rd(c->P, 8 * ksum) ? SPARCML_SSAR_RECURSIVE_DOUBLE : SPARCML_ALGO_AUTO;
  }
  cc.algo = algo;
  if (algo == SPARCML_SSAR_RECURSIVE_DOUBLE && c->P > 1)
    for (int i = 0; i < nl; ++i)
      if (nnz[i] && reinterpret_cast<const char*>(idx[i]) == static_cast<const char*>(out[i]) + SPARCML_HEADER_BYTES)
        return fail(c, SPARCML_ERR_INVALID_ARG, "in-place input is not supported by recursive doubling");
  // SSAR/DSAR for split-allgather: forced, or AUTO by sum k_i > delta (R-5)
  if (algo == SPARCML_SSAR_SPLIT_ALLGATHER) cc.host_dsar = 0;
  else if (algo == SPARCML_DSAR_SPLIT_ALLGATHER) cc.host_dsar = 1;
  else if (c->local) cc.host_dsar = ksum_host > cc.delta ? 1 : 0;
  else if (o.k_sum_hint) cc.host_dsar = o.k_sum_hint > cc.delta ? 1 : 0;
  else cc.host_dsar = -1;
  if (c->P == 1) return run_p1(c, idx[0], val[0], nnz[0], static_cast<char*>(out[0]), cc);
  std::vector<int> R;
  if (c->local)
    for (int r = 0; r < c->P; ++r) R.push_back(r);
  else
    R.push_back(c->rank);
  char* const* outs = reinterpret_cast<char* const*>(out);
  if (algo == SPARCML_SSAR_RECURSIVE_DOUBLE) return run_rd(c, R, idx, val, nnz, outs, cc);
  return run_split(c, R, idx, val, nnz, outs, cc);
}

// ------------------------------------------------------ sparse allgather ---
sparcml_status allgather_impl(sparcml_comm* c, const uint32_t* const* idx, const void* const* val,
                              const uint64_t* nnz, uint64_t N, const sparcml_opts* opts, void* const* out,
                              size_t out_bytes, void* stream, int f64 = 0) {
  if (!c) return fail(c, SPARCML_ERR_INVALID_ARG, "null communicator");
  if (!c->connected) return fail(c, SPARCML_ERR_STATE, "communicator not connected");
  if (N == 0 || N > c->L.max_N) return fail(c, SPARCML_ERR_INVALID_ARG, "N must be in [1, max_N]");
  if (N > 0xFFFFFFFFull) return fail(c, SPARCML_ERR_INVALID_ARG, "N must fit u32 indices");
  sparcml_opts o;
  sparcml_opts_default(&o);
  if (opts) o = *opts;
  if (!(o.switch_scale > 0.0f) || o.switch_scale > 1.0f)
    return fail(c, SPARCML_ERR_INVALID_ARG, "switch_scale must be in (0, 1]");
  if (out_bytes < (f64 ? sparcml_result_bytes_f64(N) : sparcml_result_bytes(N)))
    return fail(c, SPARCML_ERR_INVALID_ARG, "out_bytes < sparcml_result_bytes(N) (_f64 for double values)");
  const int nl = c->local ? c->P : 1;
  for (int i = 0; i < nl; ++i) {
    if (nnz[i] > c->L.max_nnz) return fail(c, SPARCML_ERR_INVALID_ARG, "nnz > max_nnz");
    if (nnz[i] > N) return fail(c, SPARCML_ERR_INVALID_ARG, "nnz > N");
    if (nnz[i] > 0 && (!idx[i] || !val[i])) return fail(c, SPARCML_ERR_INVALID_ARG, "null input with nnz > 0");
    if (!out[i] || (reinterpret_cast<uintptr_t>(out[i]) & 15u) != 0)
      return fail(c, SPARCML_ERR_INVALID_ARG, "out must be non-null and 16-byte aligned");
  }
  const Layout& L = c->L;
  const int P = c->P;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(c, cudaSetDevice(c->device));
  std::vector<int> R;
  if (c->local)
    for (int r = 0; r < P; ++r) R.push_back(r);
  else
    R.push_back(c->rank);
  const uint64_t sig = call_signature(N, 0, o, f64, 1);
  for (size_t i = 0; i < R.size(); ++i) {
    const int r = R[i];
    if (skipped(c, r)) continue;
    AgPublishArgs a = {};
    a.idx = idx[i];
    a.val = val[i];
    a.n = nnz[i];
    a.N = N;
    a.P = P;
    a.rank = r;
    for (int q = 0; q < 2; ++q) {
      a.my_idx[q] = reinterpret_cast<uint32_t*>(c->peer[r] + L.ag_off + q * L.ag_bytes);
      a.my_val[q] = c->peer[r] + L.ag_off + q * L.ag_bytes + L.ag_val_off;
    }
    a.f64 = f64;
    a.sig = rank_sig(c, sig, r);
    for (int j = 0; j < P; ++j) a.peer[j] = ctrl_of(c->peer[j]);
    a.ctl = ctrl_of(c->peer[r]);
    a.validate = o.validate;
    CK(c, launch_ag_publish(a, s));
  }
  for (size_t i = 0; i < R.size(); ++i) {
    const int r = R[i];
    if (skipped(c, r)) continue;
    AgGatherArgs g = {};
    g.P = P;
    g.rank = r;
    g.N = N;
    g.delta = effective_delta(N, o, f64 ? 8 : 4);
    g.sig = rank_sig(c, sig, r);
    for (int q = 0; q < 2; ++q)
      for (int j = 0; j < P; ++j) {
        g.src_idx[q][j] = reinterpret_cast<const uint32_t*>(c->peer[j] + L.ag_off + q * L.ag_bytes);
        g.src_val[q][j] = c->peer[j] + L.ag_off + q * L.ag_bytes + L.ag_val_off;
      }
    g.ctl = ctrl_of(c->peer[r]);
    g.out = static_cast<char*>(out[i]);
    g.val_offset = f64 ? sparcml_result_val_offset_f64(N) : sparcml_result_val_offset(N);
    g.f64 = f64;
    CK(c, launch_ag_gather(g, s));
  }
  return SPARCML_OK;
}

sparcml_status alloc_ws(sparcml_comm* c, char** p) {
  cudaError_t e = cudaMalloc(p, c->L.total);
  if (e == cudaErrorMemoryAllocation) return fail(c, SPARCML_ERR_OOM, "workspace allocation failed");
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc");
  e = cudaMemset(*p, 0, c->L.total);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemset");
  const uint64_t t = kDefaultTimeoutNs;
  e = cudaMemcpy(*p + offsetof(Ctrl, timeout_ns), &t, sizeof(t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemcpy");
  return SPARCML_OK;
}

// the workspace descriptor exported after the IPC handle (connect checks it)
struct WsDesc {
  uint32_t magic, version;
  int32_t P, rank;
  uint64_t max_N, max_nnz, total;
  uint8_t pad[SPARCML_IPC_HANDLE_BYTES - 64 - 40];
};
static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
static_assert(sizeof(WsDesc) == SPARCML_IPC_HANDLE_BYTES - 64, "descriptor size");
constexpr uint32_t kDescMagic = 0x53445053u;   // "SPDS"


}  // namespace

// ===========================================================================
extern "C" {

const char* sparcml_version(void) { return "sparcml-b200 0.1 (sm_100a)"; }

const char* sparcml_status_string(sparcml_status s) {
  switch (s) {
    case SPARCML_OK: return "ok";
    case SPARCML_ERR_INVALID_ARG: return "invalid argument";
    case SPARCML_ERR_UNSORTED: return "input indices not strictly increasing or out of range";
    case SPARCML_ERR_NONFINITE: return "non-finite value";
    case SPARCML_ERR_MISMATCH: return "ranks disagree on a collective argument";
    case SPARCML_ERR_CUDA: return "CUDA error";
    case SPARCML_ERR_OOM: return "out of device memory";
    case SPARCML_ERR_STATE: return "communicator in the wrong state";
    case SPARCML_ERR_TIMEOUT: return "a peer did not arrive within the timeout (destroy the communicator)";
  }
  return "unknown status";
}

void sparcml_opts_default(sparcml_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->algo = SPARCML_ALGO_AUTO;
  o->switch_scale = 1.0f;
  o->index_bytes = 4;
  o->quant_bits = 0;
  o->quant_bucket = 1024;
  o->seed = 0;
  o->k_sum_hint = 0;
  o->validate = 0;
}

uint64_t sparcml_switch_threshold(uint64_t N, int isize, int c, float scale) {
  if (N == 0 || isize <= 0 || c <= 0 || !(scale > 0.0f)) return 0;
  return (uint64_t)std::floor((double)scale * (double)N * (double)isize / (double)(c + isize));
}

double sparcml_expected_nnz(uint64_t k, uint64_t N, int P) {
  if (N == 0 || P <= 0) return 0.0;
  const double d = std::min(1.0, (double)k / (double)N);
  if (d >= 1.0) return (double)N;
  return (double)N * -std::expm1((double)P * std::log1p(-d));   // N(1-(1-d)^P)
}

size_t sparcml_result_val_offset(uint64_t N) { return SPARCML_HEADER_BYTES + 4 * half_cap(N); }

size_t sparcml_result_bytes(uint64_t N) {
  return SPARCML_HEADER_BYTES + std::max<size_t>(4 * N, 8 * half_cap(N)) + 32;
}

size_t sparcml_result_val_offset_f64(uint64_t N) { return SPARCML_HEADER_BYTES + 4 * cap64(N); }

size_t sparcml_result_bytes_f64(uint64_t N) {
  return SPARCML_HEADER_BYTES + std::max<size_t>(8 * N, 12 * cap64(N)) + 32;
}

sparcml_status sparcml_comm_create(sparcml_comm** out, int nranks, int rank, int dev, uint64_t max_N,
                                   uint64_t max_nnz) {
  if (!out) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  if (nranks < 1 || nranks > SPARCML_MAX_RANKS || rank < 0 || rank >= nranks)
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bad nranks/rank");
  if (max_N == 0 || max_N > 0xFFFFFFFFull || max_nnz == 0)
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bad max_N / max_nnz");
  if (nranks > 8) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "IPC worlds span one 8-GPU box");
  sparcml_comm* c = new sparcml_comm();
  c->P = nranks;
  c->rank = rank;
  c->device = dev;
  c->L = make_layout(nranks, max_N, max_nnz);
  cudaError_t e = cudaSetDevice(dev);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(nullptr, e, "cudaSetDevice");
  }
  char* p = nullptr;
  sparcml_status st = alloc_ws(c, &p);
  if (st != SPARCML_OK) {
    delete c;
    return st;
  }
  c->own.push_back(p);
  c->peer.assign(nranks, nullptr);
  c->opened.assign(nranks, false);
  c->peer[rank] = p;
  if (nranks > 1) {
    e = cudaIpcGetMemHandle(&c->handle, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      delete c;
      return cuda_fail(nullptr, e, "cudaIpcGetMemHandle");
    }
  } else {
    c->connected = true;
  }
  *out = c;
  return SPARCML_OK;
}

sparcml_status sparcml_comm_export_handle(sparcml_comm* c, uint8_t* h) {
  if (!c || !h) return fail(c, SPARCML_ERR_INVALID_ARG, "null argument");
  if (c->local) return fail(c, SPARCML_ERR_STATE, "loopback worlds have no handle");
  std::memcpy(h, &c->handle, 64);
  WsDesc d = {};
  d.magic = kDescMagic;
  d.version = 1;
  d.P = c->P;
  d.rank = c->rank;
  d.max_N = c->L.max_N;
  d.max_nnz = c->L.max_nnz;
  d.total = c->L.total;
  std::memcpy(h + 64, &d, sizeof(d));
  return SPARCML_OK;
}

sparcml_status sparcml_comm_connect(sparcml_comm* c, const uint8_t* all) {
  if (!c || !all) return fail(c, SPARCML_ERR_INVALID_ARG, "null argument");
  if (c->local) return fail(c, SPARCML_ERR_STATE, "loopback worlds are connected at creation");
  if (c->connected) return SPARCML_OK;
  CK(c, cudaSetDevice(c->device));
  for (int p = 0; p < c->P; ++p) {   // every rank must have built the same layout
    WsDesc d;
    std::memcpy(&d, all + (size_t)p * SPARCML_IPC_HANDLE_BYTES + 64, sizeof(d));
    if (d.magic != kDescMagic || d.version != 1 || d.P != c->P || d.rank != p || d.max_N != c->L.max_N ||
        d.max_nnz != c->L.max_nnz || d.total != c->L.total)
      return fail(c, SPARCML_ERR_MISMATCH,
                  "rank " + std::to_string(p) + "'s workspace descriptor (nranks, rank, max_N, max_nnz, layout) "
                  "does not match this rank's: every rank must create the communicator with the same limits");
  }
  for (int p = 0; p < c->P; ++p) {
    if (p == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, all + (size_t)p * SPARCML_IPC_HANDLE_BYTES, 64);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaIpcOpenMemHandle");
    c->peer[p] = static_cast<char*>(ptr);
    c->opened[p] = true;
  }
  c->connected = true;
  return SPARCML_OK;
}

sparcml_status sparcml_comm_create_local(sparcml_comm** out, int nranks, int dev, uint64_t max_N,
                                         uint64_t max_nnz) {
  if (!out) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  if (nranks < 1 || nranks > SPARCML_MAX_RANKS) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bad nranks");
  if (max_N == 0 || max_N > 0xFFFFFFFFull || max_nnz == 0)
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bad max_N / max_nnz");
  sparcml_comm* c = new sparcml_comm();
  c->P = nranks;
  c->rank = -1;
  c->device = dev;
  c->local = true;
  c->L = make_layout(nranks, max_N, max_nnz);
  cudaError_t e = cudaSetDevice(dev);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(nullptr, e, "cudaSetDevice");
  }
  for (int r = 0; r < nranks; ++r) {
    char* p = nullptr;
    sparcml_status st = alloc_ws(c, &p);
    if (st != SPARCML_OK) {
      for (char* q : c->own) cudaFree(q);
      delete c;
      return st;
    }
    c->own.push_back(p);
  }
  c->peer = c->own;
  c->opened.assign(nranks, false);
  c->connected = true;
  *out = c;
  return SPARCML_OK;
}

sparcml_status sparcml_comm_set_timeout(sparcml_comm* c, uint64_t timeout_ms) {
  if (!c) return fail(c, SPARCML_ERR_INVALID_ARG, "null communicator");
  CK(c, cudaSetDevice(c->device));
  const uint64_t t = timeout_ms * 1000ull * 1000ull;
  for (char* p : c->own) CK(c, cudaMemcpy(p + offsetof(Ctrl, timeout_ns), &t, sizeof(t), cudaMemcpyHostToDevice));
  return SPARCML_OK;
}

sparcml_status sparcml_comm_inject(sparcml_comm* c, int what, uint64_t value) {
  if (!c) return fail(c, SPARCML_ERR_INVALID_ARG, "null communicator");
  if (!c->local) return fail(c, SPARCML_ERR_STATE, "failure injection is for loopback worlds");
  if (what == SPARCML_INJECT_SKIP_RANKS) c->inject_skip = value;
  else if (what == SPARCML_INJECT_PERTURB_SIG) c->inject_sig = value;
  else return fail(c, SPARCML_ERR_INVALID_ARG, "unknown injection");
  return SPARCML_OK;
}

sparcml_status sparcml_comm_destroy(sparcml_comm* c) {
  if (!c) return SPARCML_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int p = 0; p < (int)c->peer.size(); ++p)
    if (c->opened[p]) cudaIpcCloseMemHandle(c->peer[p]);
  for (char* q : c->own) cudaFree(q);
  delete c;
  return SPARCML_OK;
}

int sparcml_comm_nranks(const sparcml_comm* c) { return c ? c->P : 0; }
const void* sparcml_comm_workspace(const sparcml_comm* c, int rank) {
  if (!c || rank < 0 || rank >= (int)c->peer.size()) return nullptr;
  return c->peer[rank];
}
int sparcml_comm_rank(const sparcml_comm* c) { return c ? c->rank : -1; }
const char* sparcml_last_error(const sparcml_comm* c) {
  return c ? c->err.c_str() : g_last_error.c_str();
}

sparcml_status sparcml_sparse_allreduce_f64(sparcml_comm* c, const uint32_t* idx, const double* val, uint64_t nnz,
                                            uint64_t N, sparcml_op op, const sparcml_opts* opts, void* out,
                                            size_t out_bytes, void* stream) {
  if (c && c->local) return fail(c, SPARCML_ERR_STATE, "use sparcml_sparse_allreduce_local_f64 on a loopback world");
  const void* v = val;
  return allreduce_impl(c, &idx, &v, &nnz, N, op, opts, &out, out_bytes, stream, 1);
}

sparcml_status sparcml_sparse_allreduce_local_f64(sparcml_comm* c, const uint32_t* const* idx,
                                                  const double* const* val, const uint64_t* nnz, uint64_t N,
                                                  sparcml_op op, const sparcml_opts* opts, void* const* out,
                                                  size_t out_bytes, void* stream) {
  if (!c || !idx || !val || !nnz || !out) return fail(c, SPARCML_ERR_INVALID_ARG, "null argument");
  if (!c->local) return fail(c, SPARCML_ERR_STATE, "not a loopback world");
  std::vector<const void*> v(val, val + c->P);
  return allreduce_impl(c, idx, v.data(), nnz, N, op, opts, out, out_bytes, stream, 1);
}

sparcml_status sparcml_sparse_allreduce(sparcml_comm* c, const uint32_t* idx, const float* val, uint64_t nnz,
                                        uint64_t N, sparcml_op op, const sparcml_opts* opts, void* out,
                                        size_t out_bytes, void* stream) {
  if (c && c->local) return fail(c, SPARCML_ERR_STATE, "use sparcml_sparse_allreduce_local on a loopback world");
  const void* v = val;
  return allreduce_impl(c, &idx, &v, &nnz, N, op, opts, &out, out_bytes, stream);
}

sparcml_status sparcml_sparse_allreduce_local(sparcml_comm* c, const uint32_t* const* idx, const float* const* val,
                                              const uint64_t* nnz, uint64_t N, sparcml_op op,
                                              const sparcml_opts* opts, void* const* out, size_t out_bytes,
                                              void* stream) {
  if (!c || !idx || !val || !nnz || !out) return fail(c, SPARCML_ERR_INVALID_ARG, "null argument");
  if (!c->local) return fail(c, SPARCML_ERR_STATE, "not a loopback world");
  std::vector<const void*> v(val, val + c->P);
  return allreduce_impl(c, idx, v.data(), nnz, N, op, opts, out, out_bytes, stream);
}

sparcml_status sparcml_sparse_allgather(sparcml_comm* c, const uint32_t* idx, const float* val, uint64_t nnz,
                                        uint64_t N, const sparcml_opts* opts, void* out, size_t out_bytes,
                                        void* stream) {
  if (c && c->local) return fail(c, SPARCML_ERR_STATE, "use sparcml_sparse_allgather_local on a loopback world");
  const void* v = val;
  return allgather_impl(c, &idx, &v, &nnz, N, opts, &out, out_bytes, stream);
}

sparcml_status sparcml_sparse_allgather_local(sparcml_comm* c, const uint32_t* const* idx, const float* const* val,
                                              const uint64_t* nnz, uint64_t N, const sparcml_opts* opts,
                                              void* const* out, size_t out_bytes, void* stream) {
  if (!c || !idx || !val || !nnz || !out) return fail(c, SPARCML_ERR_INVALID_ARG, "null argument");
  if (!c->local) return fail(c, SPARCML_ERR_STATE, "not a loopback world");
  std::vector<const void*> v(val, val + c->P);
  return allgather_impl(c, idx, v.data(), nnz, N, opts, out, out_bytes, stream);
}

sparcml_status sparcml_sparse_allgather_f64(sparcml_comm* c, const uint32_t* idx, const double* val, uint64_t nnz,
                                        uint64_t N, const sparcml_opts* opts, void* out, size_t out_bytes,
                                        void* stream) {
  if (c && c->local) return fail(c, SPARCML_ERR_STATE, "use sparcml_sparse_allgather_local_f64 on a loopback world");
  const void* v = val;
  return allgather_impl(c, &idx, &v, &nnz, N, opts, &out, out_bytes, stream, 1);
}

sparcml_status sparcml_sparse_allgather_local_f64(sparcml_comm* c, const uint32_t* const* idx, const double* const* val,
                                              const uint64_t* nnz, uint64_t N, const sparcml_opts* opts,
                                              void* const* out, size_t out_bytes, void* stream) {
  if (!c || !idx || !val || !nnz || !out) return fail(c, SPARCML_ERR_INVALID_ARG, "null argument");
  if (!c->local) return fail(c, SPARCML_ERR_STATE, "not a loopback world");
  std::vector<const void*> v(val, val + c->P);
  return allgather_impl(c, idx, v.data(), nnz, N, opts, out, out_bytes, stream, 1);
}

sparcml_status sparcml_barrier(sparcml_comm* c, void* stream) {
  if (!c) return fail(c, SPARCML_ERR_INVALID_ARG, "null communicator");
  if (!c->connected) return fail(c, SPARCML_ERR_STATE, "communicator not connected");
  CK(c, cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->local) {
    for (int r = 0; r < c->P; ++r) CK(c, launch_barrier(barrier_args(c, r), s));
  } else if (c->P > 1) {
    CK(c, launch_barrier(barrier_args(c, c->rank), s));
  }
  return SPARCML_OK;
}

sparcml_status sparcml_read_header(const void* out, sparcml_header* h, void* stream) {
  if (!out || !h) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(nullptr, cudaMemcpyAsync(h, out, sizeof(sparcml_header), cudaMemcpyDeviceToHost, s));
  CK(nullptr, cudaStreamSynchronize(s));
  return SPARCML_OK;
}

size_t sparcml_ops_workspace_bytes(uint64_t max_elems) {
  return 256 + (max_elems / kMergeTile + 4) * sizeof(TileStatus);
}

sparcml_status sparcml_ops_workspace_init(void* ws, size_t bytes, void* stream) {
  if (!ws) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null workspace");
  CK(nullptr, cudaMemsetAsync(ws, 0, bytes, static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

sparcml_status sparcml_merge_sum(const uint32_t* ia, const float* va, uint64_t na, const uint32_t* ib,
                                 const float* vb, uint64_t nb, uint32_t* io, float* vo, uint64_t* n_out,
                                 void* ws, size_t ws_bytes, void* stream) {
  if (!n_out || !ws) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  if ((na && (!ia || !va)) || (nb && (!ib || !vb)) || ((na + nb) && (!io || !vo)))
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null stream with nonzero length");
  if (ws_bytes < sparcml_ops_workspace_bytes(na + nb)) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "workspace too small");
  MergeJobsArgs m = {};
  m.njobs = 1;
  m.job[0].a_idx = ia;
  m.job[0].a_val = va;
  m.job[0].a_n = na;
  m.job[0].b_idx = ib;
  m.job[0].b_val = vb;
  m.job[0].b_n = nb;
  m.job[0].out.idx = io;
  m.job[0].out.val = vo;
  m.job[0].out.n = n_out;
  m.ctr = static_cast<ScanCounters*>(ws);
  m.status = reinterpret_cast<TileStatus*>(static_cast<char*>(ws) + 256);
  const int tiles = (int)std::min<uint64_t>((na + nb + kMergeTile - 1) / kMergeTile, 1u << 20);
  CK(nullptr, launch_merge_jobs(m, std::max(1, tiles), static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

size_t sparcml_topk_workspace_bytes(uint64_t N, uint64_t k) { return topk_workspace_bytes(N, k); }

size_t sparcml_topk_sample_positions(uint64_t N, uint64_t* pos_host, size_t cap) {
  return topk_sample_positions(N, pos_host, pos_host ? cap : 0);
}

static sparcml_status topk_common(const float* x, const float* grad, float alpha, int ef, float* xout, uint64_t N,
                                  uint64_t k, uint64_t bucket, uint32_t* io, float* vo, float* resid, void* ws,
                                  size_t ws_bytes, void* stream) {
  if (N == 0 || k == 0) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "N and k must be positive");
  if (N > 0xFFFFFFFFull) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "N must fit u32 indices");
  if (bucket != 0 && (bucket % 128 != 0 || bucket > 1024))
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bucket must be 0 (global) or a multiple of 128 up to 1024");
  if (!x || !io || !vo || (ef && !grad)) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  auto mis = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0; };
  if (mis(x) || (grad && mis(grad)) || (resid && mis(resid)))
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "vectors must be 16-byte aligned");
  if (bucket != 0) {   // bucketed (§7): no workspace needed; ws (optional) receives the status
    if (ws && ws_bytes < sizeof(uint64_t) * 64)
      return fail(nullptr, SPARCML_ERR_INVALID_ARG, "workspace too small");
    if (resid == x) resid = const_cast<float*>(x);
    CK(nullptr, launch_topk_bucketed(x, grad, alpha, ef, ef ? xout : resid, N, k, bucket, io, vo, ws,
                                     static_cast<cudaStream_t>(stream)));
    return SPARCML_OK;
  }
  if (k < N && (!ws || ws_bytes < topk_workspace_bytes(N, k)))
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "workspace too small");
  CK(nullptr, launch_topk(x, grad, alpha, ef, xout, N, k, io, vo, resid, ws, static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

sparcml_status sparcml_topk_sparsify(const float* x, uint64_t N, uint64_t k, uint64_t bucket, uint32_t* io,
                                     float* vo, float* resid, void* ws, size_t ws_bytes, void* stream) {
  return topk_common(x, nullptr, 0.0f, 0, nullptr, N, k, bucket, io, vo, resid, ws, ws_bytes, stream);
}

sparcml_status sparcml_ef_topk(float* eps, const float* grad, float alpha, uint64_t N, uint64_t k, uint64_t bucket,
                               uint32_t* io, float* vo, void* ws, size_t ws_bytes, void* stream) {
  return topk_common(eps, grad, alpha, 1, eps, N, k, bucket, io, vo, nullptr, ws, ws_bytes, stream);
}

sparcml_status sparcml_fuse_streams(int L, const uint32_t* const* idx, const float* const* val, const uint64_t* nnz,
                                    const uint64_t* off, uint32_t* idx_out, float* val_out, void* stream) {
  if (L <= 0 || L > kMaxLayers || !idx || !val || !nnz || !off)
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "need 1..64 layers and non-null arrays");
  FuseArgs a = {};
  a.L = L;
  a.pre[0] = 0;
  for (int l = 0; l < L; ++l) {
    if (l > 0 && off[l] < off[l - 1]) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "layer offsets must not decrease");
    if (nnz[l] > 0xFFFFFFFFull || off[l] > 0xFFFFFFFFull)
      return fail(nullptr, SPARCML_ERR_INVALID_ARG, "layer counts and offsets must fit u32 indices");
    if (nnz[l] && (!idx[l] || !val[l])) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null layer stream");
    a.idx[l] = idx[l];
    a.val[l] = val[l];
    a.off[l] = off[l];
    a.pre[l + 1] = a.pre[l] + nnz[l];
  }
  if (a.pre[L] && (!idx_out || !val_out)) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null output");
  a.idx_out = idx_out;
  a.val_out = val_out;
  if (a.pre[L] == 0) return SPARCML_OK;
  CK(nullptr, launch_fuse_streams(a, static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

sparcml_status sparcml_apply_update(float* v, const void* out, void* stream) {
  if (!v || !out) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  CK(nullptr, launch_apply_update(v, static_cast<const char*>(out), static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

sparcml_status sparcml_apply_update_f64(double* v, const void* out, void* stream) {
  if (!v || !out) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  CK(nullptr, launch_apply_update_f64(v, static_cast<const char*>(out), static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

sparcml_status sparcml_layer_ranges(const void* out, int L, const uint64_t* off, uint64_t* starts, void* stream) {
  if (!out || !off || !starts || L <= 0 || L > kMaxLayers)
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "need 1..64 layers and non-null arguments");
  LayerOffsets o = {};
  for (int l = 0; l < L; ++l) {
    if (l > 0 && off[l] < off[l - 1]) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "layer offsets must not decrease");
    o.v[l] = off[l];
  }
  CK(nullptr, launch_layer_ranges(static_cast<const char*>(out), L, o, starts, static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

sparcml_status sparcml_topk_status(const void* ws, uint32_t* status, uint32_t* passes, void* stream) {
  if (!ws || !status || !passes) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  CK(nullptr, topk_read_status(ws, status, passes, static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

sparcml_status sparcml_quantized_size(uint64_t n, int bits, uint32_t bucket, size_t* cb, size_t* ns) {
  if (!cb || !ns || (bits != 2 && bits != 4 && bits != 8) || bucket == 0)
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bad quantizer arguments");
  *cb = (size_t)((n * (uint64_t)bits + 7) / 8);
  *ns = (size_t)((n + bucket - 1) / bucket);
  return SPARCML_OK;
}

sparcml_status sparcml_quantize_norm(const float* x, uint64_t n, int bits, uint32_t bucket, int norm, uint64_t seed,
                                     uint64_t ctr_base, uint8_t* codes, float* scales, void* stream) {
  if ((bits != 2 && bits != 4 && bits != 8) || bucket < 8 || bucket > 1024 || (bucket & (bucket - 1)))
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bits in {2,4,8}, bucket a power of two in [8,1024]");
  if (norm != 0 && norm != 1) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "norm must be 0 (max) or 1 (l2)");
  if (n == 0) return SPARCML_OK;
  if (!x || !codes || !scales) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(codes) & 3u) != 0) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "codes must be 4-byte aligned");
  CK(nullptr, launch_quantize(x, n, bits, bucket, seed, ctr_base, codes, scales, static_cast<cudaStream_t>(stream), norm));
  return SPARCML_OK;
}

sparcml_status sparcml_quantize(const float* x, uint64_t n, int bits, uint32_t bucket, uint64_t seed,
                                uint64_t ctr_base, uint8_t* codes, float* scales, void* stream) {
  return sparcml_quantize_norm(x, n, bits, bucket, 0, seed, ctr_base, codes, scales, stream);
}

sparcml_status sparcml_dequantize(const uint8_t* codes, const float* scales, uint64_t n, int bits, uint32_t bucket,
                                  float* out, void* stream) {
  if ((bits != 2 && bits != 4 && bits != 8) || bucket < 8 || (bucket & 7))
    return fail(nullptr, SPARCML_ERR_INVALID_ARG, "bits in {2,4,8}, bucket a multiple of 8");
  if (n == 0) return SPARCML_OK;
  if (!codes || !scales || !out) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(codes) & 7u) != 0) return fail(nullptr, SPARCML_ERR_INVALID_ARG, "codes must be 8-byte aligned");
  CK(nullptr, launch_dequantize(codes, scales, n, bits, bucket, out, static_cast<cudaStream_t>(stream)));
  return SPARCML_OK;
}

uint64_t sparcml_kernel_launches(void) { return (uint64_t)g_launches; }

}  // extern "C"
