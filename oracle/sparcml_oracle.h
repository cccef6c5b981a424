/*
 * sparcml_oracle.h — plain, slow, single-threaded CPU ORACLE for the SparCML
 * (arXiv 1802.08021) sparse-allreduce hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product (libsparcml.so, include/sparcml.h) never includes, links or
 * calls anything under oracle/, and this file includes nothing from it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section named beside
 * it); "S:n" = SPEC.md line n.  Readings of silent/garbled passages are
 * numbered R-* and listed in DESIGN.md §3.
 *
 * Representation: a stream is either
 *   sparse: n strictly increasing u32 indices < N with one fp32 value each, or
 *   dense:  N fp32 values.
 * Index type u32.  Values: the paper works "with single or double
 * precision".  The collective simulators (or_merge_sum ..
 * or_sparse_allgather, the functions taking `or_val`) are compiled twice:
 * liboracle.so with or_val = float (BASELINE.json's fp32, computed in fp32
 * exactly as the method would) and liboracle_f64.so with or_val = double
 * (-DOR_VAL=double; every combine in fp64, pair = 12 bytes on the wire, QSGD
 * not defined).  or_brute_force (the fp32 definition, additionally summed in
 * fp64), top-k and QSGD are fp32 in both builds.
 *
 * Parity pins: see tests/test_oracle_*.py.  Every function below is pinned;
 * none is "parity unpinned".
 */
#ifndef SPARCML_ORACLE_H
#define SPARCML_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#ifndef OR_VAL
#define OR_VAL float
#endif
typedef OR_VAL or_val;   /* value type of the collective simulators (float or double) */

/* sizeof(or_val) of this build: 4 (liboracle.so) or 8 (liboracle_f64.so). */
int or_val_bytes(void);

/* Dense-switch threshold δ = floor(scale * N*isize/(c+isize))  (§5.1 P:488-491,
 * symbol garbled to "0.0 cm"; reading R-1).  Sparse allowed while nnz <= δ. */
uint64_t or_switch_threshold(uint64_t N, int isize, int c, double scale);

/* Two-pointer union merge with fp32 sum of two sparse streams (§5.1
 * "Efficient Summation", overlapping case, both sparse, no switch).
 * Output buffers must hold na+nb pairs.  Returns the output count. */
uint64_t or_merge_sum(const uint32_t* ia, const or_val* va, uint64_t na,
                      const uint32_t* ib, const or_val* vb, uint64_t nb,
                      uint32_t* io, or_val* vo);

/* One stream summation u1+u2 with the paper's four cases:
 * both sparse & na+nb <= delta -> sparse union merge; both sparse & na+nb > delta
 * -> dense (upper-bound rule P:520-527); sparse+dense -> scatter-accumulate
 * into the dense copy (reading R-12); dense+dense -> elementwise add
 * (P:530).  dense flags in/out; out_idx unused when the result is dense.
 * out_val must hold max(N, na+nb) floats, out_idx na+nb.  Returns out count
 * (N if dense). */
uint64_t or_stream_sum(uint64_t N, uint64_t delta,
                       int a_dense, const uint32_t* ia, const or_val* va, uint64_t na,
                       int b_dense, const uint32_t* ib, const or_val* vb, uint64_t nb,
                       int* out_dense, uint32_t* out_idx, or_val* out_val);

/* THE DEFINITION (§5.3 problem statement P:576-579; union index set P:459-461):
 * result[j] = sum_i x_i[j] over ranks holding j.  Inputs: P streams
 * concatenated, rank i at [off[i], off[i+1]).  Outputs (each length N):
 *   mask[j]  = 1 iff j in the union of supports,
 *   d64[j]   = fp64 sum in rank order,
 *   f32[j]   = fp32 sequential sum in rank order,
 *   abs64[j] = fp64 sum of |x_i[j]| (for tolerance derivation).
 * Returns K = |union of H_i|. */
uint64_t or_brute_force(int P, uint64_t N, const uint32_t* idx, const float* val,
                        const uint64_t* off, uint8_t* mask, double* d64,
                        float* f32, double* abs64);

/* Reduction operator of the simulators below (§5: any
 * coordinate-wise associative operation with a neutral element): 0 SUM
 * (neutral 0), 1 MAX (-inf), 2 MIN (+inf); SUM until set.  The neutral
 * element fills dense results.  QSGD requires SUM.  Returns 0 or -1. */
int or_set_op(int op);

/* The definition for the current operator: mask = union of the index sets,
 * f32[j] = the operator over the ranks holding j (rank order), the neutral
 * element elsewhere.  Returns K. */
uint64_t or_brute_force_op(int P, uint64_t N, const uint32_t* idx, const or_val* val,
                           const uint64_t* off, uint8_t* mask, or_val* f32);

/* Per-rank accounting of one simulated collective (the SPEC's TraceRecord,
 * S:172-179, reduced to what the tests check). */
typedef struct {
  uint64_t bytes_sent;    /* payload bytes this rank sent over all stages   */
  uint64_t bytes_recv;    /* payload bytes this rank received               */
  uint64_t msgs_sent;     /* point-to-point messages this rank sent         */
  uint64_t pairs_sent;    /* sparse (idx,val) pairs sent (dense words excl.) */
  uint64_t stage_nnz[8];  /* RD: stream size after stage t (N once dense)   */
  int      stage_dense[8];/* RD: representation after stage t              */
} or_rank_stats;

/* SSAR_Recursive_double (§5.3.1, Fig. fig:ssar_rec_dbl).
 * P <= 256.  When P is not a power of two (App. A P:1331 "add two
 * additional steps in front and at the end ... to reduce the number of
 * participating nodes to the nearest lower power of two"; reading R-28): with
 * P' the largest power of two <= P, extra rank P'+i first sends its stream
 * to rank i, which sums it in (dense switch applies), recursive doubling
 * runs over ranks 0..P'-1, and rank i finally sends its result to P'+i.
 * Stage t=1..log2 P': rank r exchanges its whole
 * current stream with r XOR 2^(t-1) (0-based reading of the figure's
 * p1<->p2, p1<->p3, p1<->p5; reading R-10) and sums with or_stream_sum using
 * delta (dense switch inside the sum; once dense stays dense).
 * Every new stream is computed from the old ones before any is replaced.
 * Outputs for rank r (r < n_out): out_dense[r], out_n[r], out_idx + r*N,
 * out_val + r*N (capacity N each).  stats: P entries (nullable).
 * Returns 0, or -1 on bad arguments. */
int or_ssar_recursive_double(int P, uint64_t N, uint64_t delta,
                             const uint32_t* idx, const or_val* val, const uint64_t* off,
                             int n_out, int* out_dense, uint64_t* out_n,
                             uint32_t* out_idx, or_val* out_val, or_rank_stats* stats);

/* Canonical balanced tree over ranks lo..hi-1 (reading R-8): hi-lo==1 -> x_lo,
 * else sum(tree(lo,mid), tree(mid,hi)) with mid = lo + (hi-lo)/2, absent
 * operands passing the present one through.  For P a power of two this is
 * exactly the order recursive doubling produces. */

/* Algorithm selector (§5.3; AUTO reading R-5). */
enum { OR_ALGO_AUTO = 0, OR_ALGO_SSAR_RD = 1, OR_ALGO_SSAR_SPLIT = 2, OR_ALGO_DSAR_SPLIT = 3 };

/* SSAR_Split_allgather / DSAR_Split_allgather (§5.3.2, §5.3.3
 * P:782-832, §6).  Any P >= 1.  Partition j = [j*floor(N/P),
 * (j+1)*floor(N/P)), last takes the remainder (App. A).
 *  phase 1: rank i sends slice_ij to owner j (P-1 messages);
 *  owner j reduces its P slices with the canonical tree of or_stream_sum
 *    (sparse; partition-local);
 *  decision: algo SSAR/DSAR forced, AUTO -> DSAR iff sum_i k_i > delta;
 *  SSAR phase 2: concatenating allgather; the
 *    concatenation switches to dense if K > delta;
 *  DSAR phase 2: each R_j densified over its partition; if quant_bits>0 it is
 *    QSGD-encoded with or_qsgd_quantize(ctr_base = partition start) and every
 *    rank, the owner included, adopts the decoded partition (§6 P:849-851,
 *    reading R-16); then a dense allgather.
 * Outputs as for or_ssar_recursive_double; *dsar_used set to 1 if the DSAR
 * path ran.  Returns 0, -1 on bad args. */
int or_split_allgather(int P, uint64_t N, uint64_t delta, int algo,
                       int quant_bits, uint32_t bucket, uint64_t seed,
                       const uint32_t* idx, const or_val* val, const uint64_t* off,
                       int n_out, int* out_dense, uint64_t* out_n,
                       uint32_t* out_idx, or_val* out_val, or_rank_stats* stats,
                       int* dsar_used);

/* Sparse allgather for disjoint slices (§7 SCD: "the values
 * calculated by each node lie in different slices of the entire model
 * vector ... the runtime of a sparse allgather"; reading R-27): every rank
 * contributes a sorted stream whose index RANGE [first, last] is disjoint
 * from every other non-empty rank's; the result on every rank is the union,
 * i.e. the streams concatenated in the order of their ranges -- no
 * arithmetic.  K = sum n_i; K > delta is stored dense.  Per-rank
 * accounting: rank r receives 8 n_i from every i != r and sends 8 n_r to
 * each of the P-1 others.  Returns 0, or -2 if two non-empty ranges overlap
 * (the precondition fails), -1 on bad arguments.  Outputs as in
 * or_split_allgather (all ranks get the same result). */
int or_sparse_allgather(int P, uint64_t N, uint64_t delta, const uint32_t* idx, const or_val* val,
                        const uint64_t* off, int n_out, int* out_dense, uint64_t* out_n,
                        uint32_t* out_idx, or_val* out_val, or_rank_stats* stats);

/* Top-k by magnitude (§2.2; Algorithm 1).  Orders every
 * coordinate by (|x_j| descending, j ascending) — ties to the lower index,
 * reading R-18 — keeps the first m = min(k, N), emits them sorted by j with
 * val = x_j.  residual (nullable, may alias x): x with the selected
 * coordinates set to 0 (acc - TopK(acc)).  Returns m.
 * Precondition: finite x. */
uint64_t or_topk(const float* x, uint64_t N, uint64_t k,
                 uint32_t* idx_out, float* val_out, float* residual);

/* Error-feedback top-k (Algorithm 1 lines "acc" and "epsilon"):
 * acc_j = fmaf(alpha, g_j, eps_j) (one rounding, reading R-19);
 * (idx,val) = TopK(acc); eps <- acc with the selected coordinates zeroed. */
uint64_t or_ef_topk(float* eps, const float* grad, float alpha, uint64_t N,
                    uint64_t k, uint32_t* idx_out, float* val_out);

/* Bucketed top-k (§7 P:1106-1107 "select k entries from every bucket of 512
 * consecutive elements"; "split into groups of 512 consecutive
 * coordinates, out of which we select the 4 largest ones ... saving the rest
 * locally"): the or_topk rule applied independently to every bucket
 * [bB, min((b+1)B, N)), reading R-26.  Output: buckets in order, each bucket's
 * min(k, |bucket|) entries sorted by index, so the whole output is sorted.
 * residual as in or_topk.  Returns m = sum_b min(k, |bucket b|). */
uint64_t or_topk_bucketed(const float* x, uint64_t N, uint64_t k, uint64_t B,
                          uint32_t* idx_out, float* val_out, float* residual);

/* Error feedback with bucketed selection (Algorithm 1 with the §7 selector):
 * acc = fmaf(alpha, g, eps); (idx, val) = bucketed TopK(acc); eps <- acc - TopK(acc). */
uint64_t or_ef_topk_bucketed(float* eps, const float* grad, float alpha, uint64_t N,
                             uint64_t k, uint64_t B, uint32_t* idx_out, float* val_out);

/* Philox4x32-10 block (Salmon et al. SC'11 / Random123; reading R-16 RNG). */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* The uniform u in [0,1) QSGD draws for global element counter c:
 * ctr = (c>>2 low32, c>>2 high32, 0, 0), key = (seed low32, seed high32),
 * u = (word[c & 3] >> 8) * 2^-24. */
float or_qsgd_uniform(uint64_t seed, uint64_t c);

/* QSGD bucketed stochastic quantization (§6; reading R-16):
 * bucket = B consecutive entries (last may be short), scale = max|v|,
 * s = 2^(bits-1)-1 levels, level = min(s, floor(fl(fl(fl(|v|/scale)*s) + u)))
 * (0 if scale == 0), code = (v<0 && level>0) << (bits-1) | level, packed
 * little-endian: element e at byte e*bits/8, bit (e % (8/bits))*bits.
 * codes: ceil(n*bits/8) bytes, scales: ceil(n/B) floats.  bits in {2,4,8}. */
/* QSGD scale norm for or_qsgd_quantize and the DSAR simulator (§6
 * mentions max- and l2-normalised variants; reading R-31): 0 max |v| (R-16,
 * default), 1 l2 = sqrtf of the balanced pairwise tree of fl(v*v) over the
 * bucket's B slots in index order (B a power of two).  Returns 0 or -1. */
int or_set_qsgd_norm(int norm);

int or_qsgd_quantize(const float* x, uint64_t n, int bits, uint32_t B,
                     uint64_t seed, uint64_t ctr_base, uint8_t* codes, float* scales);

/* Decode: v = +-fl(fl(level/s) * scale). */
int or_qsgd_dequantize(const uint8_t* codes, const float* scales, uint64_t n,
                       int bits, uint32_t B, float* out);

/* Algorithm 1's model update v <- v - g ("v_{t+1} = v_t - g_t"):
 * g is an allreduce result, dense (N values) or sparse (n strictly
 * increasing indices with one value each; absent coordinates are the neutral
 * 0 and leave v unchanged).  Every touched coordinate is one or_val
 * round-to-nearest subtraction fl(v_j - g_j).  Returns 0, or -1 on a sparse
 * index >= N. */
int or_apply_update(or_val* v, uint64_t N, int dense, uint64_t n,
                    const uint32_t* idx, const or_val* val);

/* E[K] for uniform supports (App. B), the paper's
 * inclusion-exclusion sum N * sum_{i=1..P} (-1)^(i-1) C(P,i) (k/N)^i,
 * evaluated term by term in long double. */
double or_expected_nnz(uint64_t k, uint64_t N, int P);

#ifdef __cplusplus
}
#endif
#endif
