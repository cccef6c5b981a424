/*
 * sparcml.h — C ABI of the B200-native SparCML hot path (arXiv 1802.08021).
 *
 * libsparcml.so (paper_1802_08021_b200/libsparcml.so) exports exactly the
 * functions declared here.  Signatures carry only plain pointers and sizes.
 * Citations: "P:n" = PAPER.md line n (section in brackets).
 *
 * Conventions (apply to every call unless stated):
 *  - Pointers are DEVICE pointers unless the name ends in _host.
 *  - `stream` is a cudaStream_t passed as void*; NULL means the legacy default
 *    stream.  Every device call is stream-ordered and returns as soon as the
 *    work is enqueued; outputs are valid once `stream` reaches that point.
 *  - Return value is a sparcml_status; the library never throws, never
 *    aborts and never synchronises the device except where stated.
 *    Argument errors are reported before anything is enqueued.
 *    Device-detected errors (unsorted input, non-finite values) are written
 *    to the result header's `status` field (sparcml_header.status).
 *  - Sparse streams are struct-of-arrays: idx[n] (uint32, strictly
 *    increasing, every index < N) and val[n] (float32,
 *    P:470-471).  Inputs are read-only and must stay valid until `stream`
 *    passes the call; outputs must not alias inputs unless stated.
 *  - There is no CPU fallback: a call that cannot run on the GPU fails.
 */
#ifndef SPARCML_H
#define SPARCML_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define SPARCML_MAX_RANKS 16          /* one 8-GPU box; 16 for loopback worlds */
#define SPARCML_HEADER_BYTES 64       /* result header at out[0]              */
#define SPARCML_IPC_HANDLE_BYTES 128  /* cudaIpcMemHandle_t + workspace descriptor */
#define SPARCML_HEADER_MAGIC 0x4D435053u /* "SPCM" little-endian              */
#define SPARCML_HEADER_MAGIC_F64 0x44435053u /* "SPCD": a result of the _f64 calls (double values) */

typedef enum {
  SPARCML_OK = 0,
  SPARCML_ERR_INVALID_ARG = 1,  /* bad size, null pointer, unsupported option */
  SPARCML_ERR_UNSORTED = 2,     /* input indices not strictly increasing or >= N */
  SPARCML_ERR_NONFINITE = 3,    /* NaN/Inf value where the method needs finite */
  SPARCML_ERR_MISMATCH = 4,     /* ranks disagree on a collective argument: the
                                   call signature (N, op, algo, options, value
                                   type) travels with every exchange and a rank
                                   receiving another one reports this in its
                                   header; connect reports mismatched limits */
  SPARCML_ERR_CUDA = 5,         /* a CUDA runtime call failed (see last_error) */
  SPARCML_ERR_OOM = 7,          /* device allocation failed                    */
  SPARCML_ERR_STATE = 8,        /* communicator not connected / wrong mode     */
  SPARCML_ERR_TIMEOUT = 9       /* a peer's flag did not arrive within the comm's
                                   timeout (dead, hung or mismatched rank); the
                                   call completed without it, its result is
                                   undefined and the communicator must be
                                   destroyed (device-reported, header.status) */
} sparcml_status;

/* Reduction operator (§5: "arbitrary coordinate-wise associative
 * reduction operations for which a neutral element can be defined"; reading
 * R-30).  Dense results hold the neutral element where no rank has an entry:
 * 0 (SUM), -inf (MAX), +inf (MIN).  QSGD (quant_bits) requires SUM. */
typedef enum { SPARCML_OP_SUM = 0, SPARCML_OP_MAX = 1, SPARCML_OP_MIN = 2 } sparcml_op;

/* Allreduce algorithms (§5.3).  AUTO: recursive doubling only
 * while sum_i k_i * 8 bytes stays under the crossover measured on this box
 * (the paper's small-data rule; on 2 and 4 B200 over
 * NVSwitch split-allgather won at every size measured, so AUTO picks it),
 * otherwise split-allgather; inside split-allgather SSAR vs DSAR follows the
 * dense-switch rule (R-5). */
typedef enum {
  SPARCML_ALGO_AUTO = 0,
  SPARCML_SSAR_RECURSIVE_DOUBLE = 1,   /* §5.3.1                 */
  SPARCML_SSAR_SPLIT_ALLGATHER = 2,    /* §5.3.2                 */
  SPARCML_DSAR_SPLIT_ALLGATHER = 3,    /* §5.3.3 P:782-832 (+ §6 QSGD)     */
  SPARCML_SPARSE_ALLGATHER = 4         /* header algo_used of sparcml_sparse_allgather (§7 SCD) */
} sparcml_algo;

/* Representation flag "at the beginning of each vector". */
typedef enum { SPARCML_REPR_SPARSE = 0, SPARCML_REPR_DENSE = 1 } sparcml_repr;

typedef struct {
  sparcml_algo algo;      /* default AUTO                                          */
  float switch_scale;     /* delta multiplier, default 1 ("should be even smaller") */
  int index_bytes;        /* c in delta = N*isize/(c+isize); must be 4 (u32) */
  int quant_bits;         /* 0 = off; 2, 4 or 8: QSGD in DSAR phase 2 only (§6) */
  uint32_t quant_bucket;  /* B, default 1024; a power of two in [8, 1024]     */
  uint64_t seed;          /* Philox key for QSGD                                    */
  uint64_t k_sum_hint;    /* 0 = unknown; else the exact sum of all ranks' nnz: lets
                             the host pick SSAR/DSAR without launching both paths   */
  int validate;           /* 1: check sorted/unique/< N and finiteness on device    */
  int quant_norm;         /* QSGD bucket scale: 0 max |v| (R-16), 1 l2 norm (R-31)   */
} sparcml_opts;

/* Result header, 64 bytes at out[0] (device).  The payload follows it:
 *   dense:  val[N] float at byte SPARCML_HEADER_BYTES
 *   sparse: idx[nnz] uint32 at byte SPARCML_HEADER_BYTES and val[nnz] float at
 *           byte val_offset (fixed for a given N: the buffer is laid out for
 *           the largest sparse result, delta = N/2 pairs).        */
typedef struct {
  uint32_t magic;        /* SPARCML_HEADER_MAGIC                                */
  uint32_t repr;         /* sparcml_repr                                        */
  uint64_t nnz;          /* sparse: K = |union H_i| exactly; dense: N           */
  uint64_t N;
  uint64_t k_sum;        /* sum over ranks of the input nnz                     */
  uint64_t bytes_sent;   /* payload bytes this rank put on NVLink               */
  uint64_t bytes_recv;   /* payload bytes this rank received                    */
  uint32_t algo_used;    /* sparcml_algo actually run                           */
  uint32_t status;       /* 0, or a sparcml_status detected on the device       */
  uint64_t val_offset;   /* byte offset of val[] from the start of out          */
} sparcml_header;

/* ----------------------------- utilities ------------------------------- */

const char* sparcml_version(void);
const char* sparcml_status_string(sparcml_status s);
void sparcml_opts_default(sparcml_opts* opts_host);

/* delta = floor(scale * N*isize/(c+isize)) (§5.1).  Sparse is kept
 * while nnz <= delta. */
uint64_t sparcml_switch_threshold(uint64_t N, int isize, int c, float scale);

/* E[K] = N(1-(1-k/N)^P) for uniform supports (App. B). */
double sparcml_expected_nnz(uint64_t k, uint64_t N, int P);

/* Bytes `out` must provide for an allreduce over dimension N:
 * 64 + max(4N, 8*H) + 32 with H = ceil4(floor(N/2)). */
size_t sparcml_result_bytes(uint64_t N);

/* Byte offset of val[] for a sparse result of dimension N. */
size_t sparcml_result_val_offset(uint64_t N);

/* The same for double values (the _f64 calls): delta = floor(N*8/12)
 * (P:488-491 with isize = 8), H64 = ceil4(floor(2N/3)) sparse slots:
 * 64 + max(8N, 12*H64) + 32 bytes, val[] (double) at 64 + 4*H64. */
size_t sparcml_result_bytes_f64(uint64_t N);
size_t sparcml_result_val_offset_f64(uint64_t N);

/* ---------------------------- communicator ----------------------------- */

typedef struct sparcml_comm sparcml_comm;

/* One rank per process (the production mode).  Allocates the rank's
 * symmetric workspace on `cuda_device`, sized for dimensions <= max_N and
 * per-rank nnz <= max_nnz.  Then every rank exports its handle, the caller
 * gathers the nranks handles in rank order (any host transport; the Python
 * binding uses torch.distributed) and passes them to sparcml_comm_connect,
 * which maps the peers' workspaces over NVLink (CUDA IPC).  A handle is the
 * CUDA IPC handle (64 B) followed by a descriptor of the workspace layout
 * (nranks, rank, max_N, max_nnz, layout size): connect returns
 * SPARCML_ERR_MISMATCH, mapping nothing, unless every peer's descriptor matches
 * this rank's (ranks built with different limits would address each other's
 * memory at different offsets). */
sparcml_status sparcml_comm_create(sparcml_comm** comm_out_host, int nranks, int rank,
                                   int cuda_device, uint64_t max_N, uint64_t max_nnz);
sparcml_status sparcml_comm_export_handle(sparcml_comm* comm,
                                          uint8_t* handle_host /* SPARCML_IPC_HANDLE_BYTES */);
sparcml_status sparcml_comm_connect(sparcml_comm* comm,
                                    const uint8_t* all_handles_host /* nranks*SPARCML_IPC_HANDLE_BYTES, rank order */);

/* Failure handling ("watchdog").  Every wait of a collective
 * for a peer's flag gives up after timeout_ms (default 10000; 0 = wait
 * forever): the call then completes with header.status = SPARCML_ERR_TIMEOUT
 * on the ranks that waited, instead of hanging every GPU of the world.  After a
 * timeout the communicator's flag protocol is out of step: destroy it.
 * Synchronous (writes the value into the workspaces this process owns). */
sparcml_status sparcml_comm_set_timeout(sparcml_comm* comm, uint64_t timeout_ms);

/* Failure injection for tests, loopback worlds only:
 *   what = SPARCML_INJECT_SKIP_RANKS: value = bit mask of ranks whose kernels
 *          are not launched (dead ranks; the others must time out);
 *   what = SPARCML_INJECT_PERTURB_SIG: value = r + 1 makes rank r call with a
 *          different signature (N/op/algo/options; the others must report
 *          SPARCML_ERR_MISMATCH), 0 = off.                                  */
#define SPARCML_INJECT_SKIP_RANKS 1
#define SPARCML_INJECT_PERTURB_SIG 2
sparcml_status sparcml_comm_inject(sparcml_comm* comm, int what, uint64_t value);

/* Loopback world: all nranks ranks live in this process on one device and
 * run the same kernels and exchanges through local memory.  Used for tests
 * and single-GPU emulation.  Collectives are issued with the *_local calls. */
sparcml_status sparcml_comm_create_local(sparcml_comm** comm_out_host, int nranks,
                                         int cuda_device, uint64_t max_N, uint64_t max_nnz);

sparcml_status sparcml_comm_destroy(sparcml_comm* comm);
int sparcml_comm_nranks(const sparcml_comm* comm);
/* Diagnostics: device pointer of rank `rank`'s symmetric workspace (its
 * control block first) as seen from this process; NULL if unknown. */
const void* sparcml_comm_workspace(const sparcml_comm* comm, int rank);
int sparcml_comm_rank(const sparcml_comm* comm);   /* -1 for a loopback world */
const char* sparcml_last_error(const sparcml_comm* comm);  /* NULL comm: global */

/* ---------------------------- allreduce -------------------------------- */

/* Sparse allreduce (§5.3 problem statement P:576-579): every rank passes its
 * stream (idx, val, nnz) over dimension N; after the call `out` on every rank
 * holds x = sum_i x_i with index set exactly the union of the H_i (explicit
 * zeros kept), sparse or dense per the dense-switch rule
 * (P:501-527).  Collective: all ranks call with the same N, op and opts in
 * the same order.  `out` (out_bytes >= sparcml_result_bytes(N)) is fully
 * written (header + payload).  In place: the input may BE the sparse payload
 * slots of `out` (idx == out + 64, val == out + sparcml_result_val_offset(N),
 * e.g. written there by the top-k); a one-rank call then only writes the
 * header.  In-place is supported by split-allgather (every rank's input is
 * consumed before its result is written) but not by recursive doubling, nor
 * for one rank with nnz > delta under forced SSAR (SPARCML_ERR_INVALID_ARG).
 * Any other overlap of inputs and `out` is undefined.  Never
 * synchronises the host; read the header after the stream passes.
 * Errors: N == 0, N > max_N, nnz > max_nnz, null pointers with nnz > 0,
 * unsupported opts -> SPARCML_ERR_INVALID_ARG; loopback comm ->
 * SPARCML_ERR_STATE. */
sparcml_status sparcml_sparse_allreduce(sparcml_comm* comm, const uint32_t* idx, const float* val,
                                        uint64_t nnz, uint64_t N, sparcml_op op,
                                        const sparcml_opts* opts_host /* NULL = defaults */,
                                        void* out, size_t out_bytes, void* stream);

/* Loopback-world allreduce: arrays of nranks per-rank inputs/outputs (host
 * arrays of device pointers).  Same semantics as above for every rank. */
sparcml_status sparcml_sparse_allreduce_local(sparcml_comm* comm,
                                              const uint32_t* const* idx_host,
                                              const float* const* val_host,
                                              const uint64_t* nnz_host, uint64_t N, sparcml_op op,
                                              const sparcml_opts* opts_host,
                                              void* const* out_host, size_t out_bytes, void* stream);

/* The sparse allreduce with fp64 values: the paper's streams carry "single
 * or double precision floating point values" (§5.1).  Identical to
 * the calls above with val[] double, every combine one fp64 rounding in the
 * same canonical order, a pair = 12 bytes (so delta = floor(N*8/12)),
 * the result laid out per sparcml_result_*_f64 with header magic
 * SPARCML_HEADER_MAGIC_F64 and double payload values.  All algorithms and
 * operators; QSGD (quant_bits != 0) is fp32-only -> SPARCML_ERR_INVALID_ARG. */
sparcml_status sparcml_sparse_allreduce_f64(sparcml_comm* comm, const uint32_t* idx, const double* val,
                                            uint64_t nnz, uint64_t N, sparcml_op op,
                                            const sparcml_opts* opts_host, void* out, size_t out_bytes,
                                            void* stream);
sparcml_status sparcml_sparse_allreduce_local_f64(sparcml_comm* comm, const uint32_t* const* idx_host,
                                                  const double* const* val_host, const uint64_t* nnz_host,
                                                  uint64_t N, sparcml_op op, const sparcml_opts* opts_host,
                                                  void* const* out_host, size_t out_bytes, void* stream);

/* Device-side barrier of all ranks (one warp per rank spinning on flags its
 * peers store over NVLink).  Stream-ordered, no host synchronisation;
 * collective like the allreduce.  On a loopback world it only orders. */
sparcml_status sparcml_barrier(sparcml_comm* comm, void* stream);

/* Sparse allgather for disjoint slices (§7 SCD: "the values
 * calculated by each node lie in different slices of the entire model vector
 * ... a sparse allgather"; reading R-27).  Precondition: the index ranges
 * [first, last] of the non-empty ranks are pairwise disjoint (any rank
 * order).  `out` on every rank receives their union -- the streams
 * concatenated in range order (K = sum nnz), dense when K > delta -- with
 * header algo_used = SPARCML_SPARSE_ALLGATHER.  One exchange: each rank
 * publishes its stream in its own workspace and flags every peer; every rank
 * pulls the P streams over NVLink.  Overlapping ranges: header status
 * SPARCML_ERR_INVALID_ARG, payload undefined.  opts: only switch_scale and
 * validate are used (NULL = defaults).  Errors as sparcml_sparse_allreduce. */
sparcml_status sparcml_sparse_allgather(sparcml_comm* comm, const uint32_t* idx, const float* val,
                                        uint64_t nnz, uint64_t N, const sparcml_opts* opts_host,
                                        void* out, size_t out_bytes, void* stream);
sparcml_status sparcml_sparse_allgather_local(sparcml_comm* comm, const uint32_t* const* idx_host,
                                              const float* const* val_host, const uint64_t* nnz_host,
                                              uint64_t N, const sparcml_opts* opts_host,
                                              void* const* out_host, size_t out_bytes, void* stream);
/* The same with fp64 values: result laid out per
 * sparcml_result_*_f64 (magic SPARCML_HEADER_MAGIC_F64), dense when
 * K > floor(N*8/12), header byte counts at 12 bytes per pair. */
sparcml_status sparcml_sparse_allgather_f64(sparcml_comm* comm, const uint32_t* idx, const double* val,
                                            uint64_t nnz, uint64_t N, const sparcml_opts* opts_host,
                                            void* out, size_t out_bytes, void* stream);
sparcml_status sparcml_sparse_allgather_local_f64(sparcml_comm* comm, const uint32_t* const* idx_host,
                                                  const double* const* val_host, const uint64_t* nnz_host,
                                                  uint64_t N, const sparcml_opts* opts_host,
                                                  void* const* out_host, size_t out_bytes, void* stream);

/* Algorithm 1's update ("v_t <- v_{t-1} - g_t"): v[j] -= g[j] for the
 * allreduce result g in `out` (sparse: its pairs; dense: all N values),
 * read from the device header -- no host synchronisation.  v: N floats
 * (N = the result's N).  fp32 results only: a result whose header magic is
 * not SPARCML_HEADER_MAGIC (e.g. an _f64 result) leaves v unchanged.
 * Errors: null arguments -> SPARCML_ERR_INVALID_ARG. */
sparcml_status sparcml_apply_update(float* v, const void* out, void* stream);
/* The same for an _f64 result (v: N doubles, one fp64 rounding per element);
 * a result that is not fp64 (magic != SPARCML_HEADER_MAGIC_F64) leaves v unchanged. */
sparcml_status sparcml_apply_update_f64(double* v, const void* out, void* stream);

/* ---------------------- layer-wise tensor fusion ------------------------ */
/* (the paper's deployment mode: "communication is
 * done layer-wise using non-blocking calls".)  A model's L layers
 * (dimensions N_l) are laid end to end: layer l owns global indices
 * [off_l, off_l + N_l), off_0 = 0, off_{l+1} = off_l + N_l.  Fusing the L
 * per-layer streams is a concatenation with index offsets -- the result is
 * one sorted stream over N = sum N_l that one allreduce reduces; the
 * allreduce result splits back into layers by index range.  Values are
 * unchanged (the summation tree is over ranks, R-8), so per-layer results
 * equal per-layer allreduces; only the dense switch sees the fused N.  All
 * calls are stream-ordered and graph-capturable ("non-blocking": the host
 * never waits; order work across streams with CUDA events). */

/* idx_out[n_0 + ... + n_{l-1} + i] = idx_l[i] + off_l, val likewise, for the
 * L layers (host arrays of L device pointers / counts / offsets).  idx_l
 * strictly increasing < N_l (so the output is strictly increasing when the
 * offsets are).  Errors: L <= 0, null arrays, decreasing offsets, a count
 * above 2^32 -> SPARCML_ERR_INVALID_ARG. */
sparcml_status sparcml_fuse_streams(int L, const uint32_t* const* idx_host, const float* const* val_host,
                                    const uint64_t* nnz_host, const uint64_t* off_host,
                                    uint32_t* idx_out, float* val_out, void* stream);

/* Layer ranges of an allreduce result: starts_dev[l] (device, L+1 entries
 * of uint64) = first payload position of layer l -- for a sparse result the
 * lower bound of off_l in the result's sorted indices, for a dense one off_l
 * itself; starts_dev[L] = nnz (sparse) or N (dense).  Layer l's entries are
 * [starts[l], starts[l+1]) of the payload (idx at 64, val at val_offset). */
sparcml_status sparcml_layer_ranges(const void* out, int L, const uint64_t* off_host, uint64_t* starts_dev,
                                    void* stream);

/* Synchronous helper: copies the 64-byte header at out[0] to the host
 * (cudaMemcpyAsync on `stream` + stream synchronize). */
sparcml_status sparcml_read_header(const void* out, sparcml_header* hdr_host, void* stream);

/* ------------------------------ stream ops ----------------------------- */

/* Workspace for the stand-alone stream ops below: size, and one-time zero
 * initialisation of a fresh allocation (stream-ordered memset). */
size_t sparcml_ops_workspace_bytes(uint64_t max_elems);
sparcml_status sparcml_ops_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* Union-merge-with-sum of two sparse streams (§5.1 "Efficient Summation",
 * both sparse, overlapping indices; no dense switch).  io/vo hold
 * na+nb pairs; *n_out_dev receives the output count (device uint64). */
sparcml_status sparcml_merge_sum(const uint32_t* ia, const float* va, uint64_t na,
                                 const uint32_t* ib, const float* vb, uint64_t nb,
                                 uint32_t* io, float* vo, uint64_t* n_out_dev,
                                 void* ws, size_t ws_bytes, void* stream);

/* ------------------------------- top-k --------------------------------- */

/* Top-k by magnitude (§2.2): the m = min(k, N) coordinates with the
 * largest |x_j|, ties to the lower index; written sorted by index to
 * idx_out[m], val_out[m] (= x_j).  residual (nullable, may alias x) receives
 * x with the selected coordinates zeroed (acc - TopK(acc)).
 * bucket = 0: global top-k.  bucket > 0 (a multiple of 128, at most 1024):
 * bucketed top-k (§7; reading R-26) -- the same rule in
 * every bucket [bB, min((b+1)B, N)) with k per bucket; m = sum_b min(k,|b|)
 * entries, buckets in order (sorted overall); ws may then be NULL (it only
 * receives the status).  Requires finite x (NaN/Inf are reported through
 * sparcml_topk_status).  ws from sparcml_topk_workspace_bytes, zero-initialised
 * once with sparcml_ops_workspace_init; one workspace serves any N up to the
 * size it was made for.  The workspace carries state between calls: the
 * global top-k remembers the k-th magnitude m it found, and the next call with
 * the same (N, k, EF or not) starts its candidate threshold at m(1 - 1/64)
 * instead of sampling (the warm start).  The result never
 * depends on it -- a wrong guess costs one more filter pass (passes == 2) --
 * so use one workspace per vector (e.g. per layer's eps) to keep the guesses
 * good.  Calls on one workspace must be stream-ordered (not concurrent). */
size_t sparcml_topk_workspace_bytes(uint64_t N, uint64_t k);
sparcml_status sparcml_topk_sparsify(const float* x, uint64_t N, uint64_t k, uint64_t bucket,
                                     uint32_t* idx_out, float* val_out, float* residual,
                                     void* ws, size_t ws_bytes, void* stream);

/* Error-feedback top-k, Algorithm 1: acc = fmaf(alpha, grad, eps)
 * (one rounding), (idx, val) = TopK(acc), eps <- acc - TopK(acc), in place.
 * bucket as in sparcml_topk_sparsify. */
sparcml_status sparcml_ef_topk(float* eps, const float* grad, float alpha, uint64_t N,
                               uint64_t k, uint64_t bucket, uint32_t* idx_out, float* val_out,
                               void* ws, size_t ws_bytes, void* stream);

/* Diagnostics: the positions of the float4 granules the global top-k samples
 * (4 values each) to set its candidate threshold on the current device, for a
 * vector of N values; writes min(count, cap) of them to pos_host and returns
 * the count (0 when N < 65536: no sampling).  The selection never depends on
 * them for correctness -- an input that defeats the sample takes the exact
 * re-filter path (passes == 2); tests use this to build such an input.  (A
 * call that starts warm samples only when its warm threshold misses.) */
size_t sparcml_topk_sample_positions(uint64_t N, uint64_t* pos_host, size_t cap);

/* Synchronous: device status of the last top-k run on `ws` (0 or
 * SPARCML_ERR_NONFINITE) and how many filter passes it needed (1; +1 for each
 * re-filter: a warm-start miss re-filters from a sample, a sample miss with
 * threshold 0). */
sparcml_status sparcml_topk_status(const void* ws, uint32_t* status_host, uint32_t* passes_host,
                                   void* stream);

/* -------------------------------- QSGD --------------------------------- */

/* Sizes of a QSGD encoding of n values (§6): ceil(n*bits/8) code
 * bytes and ceil(n/bucket) fp32 scales. */
sparcml_status sparcml_quantized_size(uint64_t n, int bits, uint32_t bucket,
                                      size_t* code_bytes_host, size_t* n_scales_host);

/* Stochastic bucketed quantization (§6, R-16): per bucket
 * of `bucket` consecutive values scale = max|v|; level = min(s, floor(fl(
 * fl(fl(|v|/scale)*s) + u))) with s = 2^(bits-1)-1 and u from Philox4x32-10
 * (key = seed, counter = ctr_base + element index); code = sign<<(bits-1) |
 * level packed little-endian.  bits in {2,4,8}; bucket a power of two in
 * [8, 1024]; codes 4-byte aligned. */
sparcml_status sparcml_quantize(const float* x, uint64_t n, int bits, uint32_t bucket,
                                uint64_t seed, uint64_t ctr_base, uint8_t* codes, float* scales,
                                void* stream);

/* v = +-fl(fl(level/s) * scale). */
/* sparcml_quantize with the bucket scale chosen by `norm`: 0 max |v| (R-16),
 * 1 the l2 norm by a balanced pairwise tree in index order (R-31; bucket a
 * power of two in [8, 1024]). */
sparcml_status sparcml_quantize_norm(const float* x, uint64_t n, int bits, uint32_t bucket, int norm,
                                     uint64_t seed, uint64_t ctr_base, uint8_t* codes, float* scales,
                                     void* stream);

sparcml_status sparcml_dequantize(const uint8_t* codes, const float* scales, uint64_t n, int bits,
                                  uint32_t bucket, float* out, void* stream);

/* ------------------------------ telemetry ------------------------------ */

/* Number of kernels this process has enqueued through the library since
 * load (the bench's gpu_launches count). */
uint64_t sparcml_kernel_launches(void);

/* Per-kernel timing for the bench's roofline.  While enabled, every launch of
 * a kernel class ("topk", "topk_bucketed", "split_push", "owner", "owner_dsar",
 * "concat", "rd_push", "rd_stage", "ag_publish", "ag_gather", "merge", "barrier",
 * ...) is bracketed by CUDA events on its stream.
 * sparcml_profile_read synchronises those events and returns the launch
 * count and the summed duration in milliseconds. */
void sparcml_profile_enable(int on);
void sparcml_profile_only(const char* kernel_name /* NULL: every class */);
void sparcml_profile_reset(void);
sparcml_status sparcml_profile_read(const char* kernel_name, uint64_t* launches_host,
                                    double* total_ms_host);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* SPARCML_H */
