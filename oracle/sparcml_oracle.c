/*
 * sparcml_oracle.c — plain, slow, single-threaded CPU oracle (TEST
 * INFRASTRUCTURE; see sparcml_oracle.h for the contract and citations).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (oracle/build.py).
 * -ffp-contract=off keeps every fp32 expression as written: one rounding per
 * operation, no FMA contraction, except the explicit fmaf of Algorithm 1.
 *
 * Deliberately unoptimised: every loop follows the paper's wording in order.
 */
#include "sparcml_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* §5.1 sparse streams                                                        */
/* ------------------------------------------------------------------------- */

uint64_t or_switch_threshold(uint64_t N, int isize, int c, double scale) {
  /* sparse transmits nnz*(c+isize) bytes, dense N*isize bytes, so
   * sparse only pays while nnz <= N*isize/(c+isize).  P:493-494: "in practice
   * [it] should be even smaller" -> user scale (default 1). */
  if (N == 0 || isize <= 0 || c <= 0) return 0;
  long double d = (long double)N * (long double)isize / (long double)(c + isize);
  d *= (long double)scale;
  if (d < 0) return 0;
  return (uint64_t)floorl(d);
}

/* Reduction operator for the collective simulators (§5: "arbitrary
 * coordinate-wise associative reduction operations for which a neutral
 * element can be defined"): 0 SUM (neutral 0), 1 MAX (neutral -inf),
 * 2 MIN (neutral +inf).  Set with or_set_op; SUM by default. */
static int g_op = 0;

/* value and pair sizes on the wire: 4 / 8 bytes (fp32), 8 / 12 bytes (fp64) */
#define VB ((uint64_t)sizeof(or_val))
#define PB ((uint64_t)(4 + sizeof(or_val)))

int or_val_bytes(void) { return (int)sizeof(or_val); }

int or_set_op(int op) {
  if (op < 0 || op > 2) return -1;
  g_op = op;
  return 0;
}

static or_val op_combine(or_val a, or_val b) {
  if (g_op == 1) return a > b ? a : b;
  if (g_op == 2) return a < b ? a : b;
  return a + b;
}

static or_val op_neutral(void) {
  if (g_op == 1) return -INFINITY;
  if (g_op == 2) return INFINITY;
  return 0;
}

uint64_t or_merge_sum(const uint32_t* ia, const or_val* va, uint64_t na,
                      const uint32_t* ib, const or_val* vb, uint64_t nb,
                      uint32_t* io, or_val* vo) {
  /* P:516-527, overlapping indices, both sparse: union of the index sets,
   * values summed where the indices coincide.  Cancellation is ignored: an
   * index present in either input is present in the output even if the sum
   * is zero. */
  uint64_t i = 0, j = 0, o = 0;
  while (i < na && j < nb) {
    if (ia[i] < ib[j]) {
      io[o] = ia[i]; vo[o] = va[i]; i++;
    } else if (ib[j] < ia[i]) {
      io[o] = ib[j]; vo[o] = vb[j]; j++;
    } else {
      io[o] = ia[i]; vo[o] = op_combine(va[i], vb[j]); i++; j++;
    }
    o++;
  }
  while (i < na) { io[o] = ia[i]; vo[o] = va[i]; i++; o++; }
  while (j < nb) { io[o] = ib[j]; vo[o] = vb[j]; j++; o++; }
  return o;
}

uint64_t or_stream_sum(uint64_t N, uint64_t delta,
                       int a_dense, const uint32_t* ia, const or_val* va, uint64_t na,
                       int b_dense, const uint32_t* ib, const or_val* vb, uint64_t nb,
                       int* out_dense, uint32_t* out_idx, or_val* out_val) {
  uint64_t j;
  if (!a_dense && !b_dense) {
    /* upper-bound |H1|+|H2|; if bigger than delta switch to dense. */
    if (na + nb > delta) {
      for (j = 0; j < N; j++) out_val[j] = op_neutral();   /* neutral element */
      for (j = 0; j < na; j++) out_val[ia[j]] = op_combine(out_val[ia[j]], va[j]);
      for (j = 0; j < nb; j++) out_val[ib[j]] = op_combine(out_val[ib[j]], vb[j]);
      *out_dense = 1;
      return N;
    }
    *out_dense = 0;
    return or_merge_sum(ia, va, na, ib, vb, nb, out_idx, out_val);
  }
  if (a_dense && b_dense) {
    /* dense + dense -> elementwise (vectorised in the paper) sum. */
    for (j = 0; j < N; j++) out_val[j] = op_combine(va[j], vb[j]);
    *out_dense = 1;
    return N;
  }
  /* one dense, one sparse: iterate over the sparse pairs and
   * "set" (accumulate, reading R-12) the value at that position. */
  {
    const or_val* dv = a_dense ? va : vb;
    const uint32_t* si = a_dense ? ib : ia;
    const or_val* sv = a_dense ? vb : va;
    uint64_t sn = a_dense ? nb : na;
    for (j = 0; j < N; j++) out_val[j] = dv[j];
    for (j = 0; j < sn; j++) out_val[si[j]] = op_combine(out_val[si[j]], sv[j]);
  }
  *out_dense = 1;
  return N;
}

uint64_t or_brute_force_op(int P, uint64_t N, const uint32_t* idx, const or_val* val,
                           const uint64_t* off, uint8_t* mask, or_val* f32) {
  /* The definition for any operator: every index of the union, reduced over
   * the ranks that hold it (rank order; MAX and MIN are order-free). */
  uint64_t j, K = 0;
  int i;
  for (j = 0; j < N; j++) { mask[j] = 0; f32[j] = op_neutral(); }
  for (i = 0; i < P; i++)
    for (j = off[i]; j < off[i + 1]; j++) {
      const uint32_t x = idx[j];
      f32[x] = mask[x] ? op_combine(f32[x], val[j]) : val[j];
      mask[x] = 1;
    }
  for (j = 0; j < N; j++) K += mask[j];
  return K;
}

uint64_t or_brute_force(int P, uint64_t N, const uint32_t* idx, const float* val,
                        const uint64_t* off, uint8_t* mask, double* d64,
                        float* f32, double* abs64) {
  /* The plain definition: densify every rank's vector and add. */
  uint64_t j, K = 0;
  int i;
  for (j = 0; j < N; j++) { mask[j] = 0; d64[j] = 0.0; f32[j] = 0.0f; abs64[j] = 0.0; }
  for (i = 0; i < P; i++) {
    for (j = off[i]; j < off[i + 1]; j++) {
      uint32_t x = idx[j];
      mask[x] = 1;
      d64[x] += (double)val[j];
      f32[x] = f32[x] + val[j];
      abs64[x] += fabs((double)val[j]);
    }
  }
  for (j = 0; j < N; j++) K += mask[j];
  return K;
}

/* ------------------------------------------------------------------------- */
/* simulated streams                                                          */
/* ------------------------------------------------------------------------- */

typedef struct {
  int dense;
  uint64_t n;     /* pairs if sparse, N if dense */
  uint32_t* idx;  /* sparse only */
  or_val* val;
} strm;

static void strm_free(strm* s) { free(s->idx); free(s->val); s->idx = NULL; s->val = NULL; }

static int strm_copy_in(strm* s, const uint32_t* idx, const or_val* val, uint64_t n) {
  s->dense = 0; s->n = n;
  s->idx = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  s->val = (or_val*)malloc((n ? n : 1) * sizeof(or_val));
  if (!s->idx || !s->val) return -1;
  memcpy(s->idx, idx, n * sizeof(uint32_t));
  memcpy(s->val, val, n * sizeof(or_val));
  return 0;
}

/* r = a + b via or_stream_sum; allocates r. */
static int strm_sum(uint64_t N, uint64_t delta, const strm* a, const strm* b, strm* r) {
  uint64_t cap_pairs = a->n + b->n;
  uint64_t cap_vals = cap_pairs > N ? cap_pairs : N;
  r->idx = (uint32_t*)malloc((cap_pairs ? cap_pairs : 1) * sizeof(uint32_t));
  r->val = (or_val*)malloc((cap_vals ? cap_vals : 1) * sizeof(or_val));
  if (!r->idx || !r->val) return -1;
  r->n = or_stream_sum(N, delta, a->dense, a->idx, a->val, a->n,
                       b->dense, b->idx, b->val, b->n, &r->dense, r->idx, r->val);
  return 0;
}

static uint64_t strm_bytes(const strm* s) {
  /* payload bytes on the wire: PB per (u32, value) pair, VB per dense word */
  return s->dense ? VB * s->n : PB * s->n;
}

static void strm_out(const strm* s, uint64_t N, int r, int* out_dense, uint64_t* out_n,
                     uint32_t* out_idx, or_val* out_val) {
  out_dense[r] = s->dense;
  out_n[r] = s->n;
  if (s->dense) {
    memcpy(out_val + (uint64_t)r * N, s->val, N * sizeof(or_val));
  } else {
    memcpy(out_idx + (uint64_t)r * N, s->idx, s->n * sizeof(uint32_t));
    memcpy(out_val + (uint64_t)r * N, s->val, s->n * sizeof(or_val));
  }
}

/* ------------------------------------------------------------------------- */
/* §5.3.1 SSAR_Recursive_double                                               */
/* ------------------------------------------------------------------------- */

int or_ssar_recursive_double(int P, uint64_t N, uint64_t delta,
                             const uint32_t* idx, const or_val* val, const uint64_t* off,
                             int n_out, int* out_dense, uint64_t* out_n,
                             uint32_t* out_idx, or_val* out_val, or_rank_stats* stats) {
  int r, t, L = 0, P2 = 1, e;
  strm *cur, *nxt;
  if (P < 1 || P > 256) return -1;
  while (P2 * 2 <= P) P2 *= 2;   /* nearest lower power of two (App. A) */
  e = P - P2;                     /* extra ranks, folded into ranks 0..e-1 (reading R-28) */
  while ((1 << L) < P2) L++;
  cur = (strm*)calloc((size_t)P, sizeof(strm));
  nxt = (strm*)calloc((size_t)P, sizeof(strm));
  if (!cur || !nxt) return -1;
  if (stats) memset(stats, 0, (size_t)P * sizeof(or_rank_stats));
  for (r = 0; r < P; r++)
    if (strm_copy_in(&cur[r], idx + off[r], val + off[r], off[r + 1] - off[r])) return -1;

  /* front step: extra rank P2+i sends its stream to rank i, which sums it in */
  for (r = 0; r < e; r++) {
    const int x = P2 + r;
    if (stats) {
      stats[x].bytes_sent += strm_bytes(&cur[x]);
      stats[x].msgs_sent += 1;
      if (!cur[x].dense) stats[x].pairs_sent += cur[x].n;
      stats[r].bytes_recv += strm_bytes(&cur[x]);
    }
    if (strm_sum(N, delta, &cur[r], &cur[x], &nxt[r])) return -1;
    strm_free(&cur[r]);
    cur[r] = nxt[r];
    memset(&nxt[r], 0, sizeof(strm));
  }

  for (t = 1; t <= L; t++) {
    int d = 1 << (t - 1);     /* distance 2^(t-1) */
    for (r = 0; r < P2; r++) {
      int q = r ^ d;
      /* rank r sends its whole current stream to q and receives q's */
      if (stats) {
        stats[r].bytes_sent += strm_bytes(&cur[r]);
        stats[r].bytes_recv += strm_bytes(&cur[q]);
        stats[r].msgs_sent += 1;
        if (!cur[r].dense) stats[r].pairs_sent += cur[r].n;
      }
      if (strm_sum(N, delta, &cur[r], &cur[q], &nxt[r])) return -1;
      if (stats && t <= 8) {
        stats[r].stage_nnz[t - 1] = nxt[r].n;
        stats[r].stage_dense[t - 1] = nxt[r].dense;
      }
    }
    for (r = 0; r < P2; r++) { strm_free(&cur[r]); cur[r] = nxt[r]; memset(&nxt[r], 0, sizeof(strm)); }
  }
  /* end step: rank i sends the result to extra rank P2+i */
  for (r = 0; r < e; r++) {
    const int x = P2 + r;
    if (stats) {
      stats[r].bytes_sent += strm_bytes(&cur[r]);
      stats[r].msgs_sent += 1;
      if (!cur[r].dense) stats[r].pairs_sent += cur[r].n;
      stats[x].bytes_recv += strm_bytes(&cur[r]);
    }
    strm_free(&cur[x]);
    if (cur[r].dense) {
      memset(&cur[x], 0, sizeof(strm));
      cur[x].dense = 1;
      cur[x].n = N;
      cur[x].val = (or_val*)malloc((N ? N : 1) * sizeof(or_val));
      if (!cur[x].val) return -1;
      memcpy(cur[x].val, cur[r].val, N * sizeof(or_val));
    } else if (strm_copy_in(&cur[x], cur[r].idx, cur[r].val, cur[r].n)) {
      return -1;
    }
  }
  for (r = 0; r < P && r < n_out; r++) strm_out(&cur[r], N, r, out_dense, out_n, out_idx, out_val);
  for (r = 0; r < P; r++) strm_free(&cur[r]);
  free(cur); free(nxt);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* §5.3.2 / §5.3.3 split-allgather                                             */
/* ------------------------------------------------------------------------- */

/* first position in idx[0..n) with idx >= key */
static uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint64_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if ((uint64_t)a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* canonical balanced tree over slices lo..hi-1 (reading R-8), all sparse */
static int tree_reduce(strm* slices, int lo, int hi, uint64_t part_n, strm* out) {
  strm a, b;
  int mid;
  if (hi - lo == 1) {
    return strm_copy_in(out, slices[lo].idx, slices[lo].val, slices[lo].n);
  }
  mid = lo + (hi - lo) / 2;
  memset(&a, 0, sizeof a); memset(&b, 0, sizeof b);
  if (tree_reduce(slices, lo, mid, part_n, &a)) return -1;
  if (tree_reduce(slices, mid, hi, part_n, &b)) return -1;
  /* partition-local sum; the partition result can never exceed the partition,
   * so no switch here (delta = infinity) */
  if (strm_sum(part_n, UINT64_MAX, &a, &b, out)) return -1;
  strm_free(&a); strm_free(&b);
  return 0;
}

int or_split_allgather(int P, uint64_t N, uint64_t delta, int algo,
                       int quant_bits, uint32_t bucket, uint64_t seed,
                       const uint32_t* idx, const or_val* val, const uint64_t* off,
                       int n_out, int* out_dense, uint64_t* out_n,
                       uint32_t* out_idx, or_val* out_val, or_rank_stats* stats,
                       int* dsar_used) {
  int i, j, r;
  uint64_t part, ksum = 0, K = 0, e;
  uint64_t* bnd;           /* partition boundaries b_0..b_P */
  strm* slices;            /* slices[j*P + i] = rank i's entries in partition j */
  strm* R;                 /* owner results */
  int dsar;
  if (P < 1 || N < (uint64_t)P) return -1;
  if (quant_bits != 0 && quant_bits != 2 && quant_bits != 4 && quant_bits != 8) return -1;
  if (quant_bits && bucket == 0) return -1;
  if (quant_bits && g_op != 0) return -1;   /* QSGD needs the 0 neutral element (max-norm scale) */
  if (quant_bits && sizeof(or_val) != sizeof(float)) return -1;   /* QSGD is defined on fp32 values here */
  part = N / (uint64_t)P;                         /* floor(N/P), App. A */
  bnd = (uint64_t*)malloc(((size_t)P + 1) * sizeof(uint64_t));
  slices = (strm*)calloc((size_t)P * (size_t)P, sizeof(strm));
  R = (strm*)calloc((size_t)P, sizeof(strm));
  if (!bnd || !slices || !R) return -1;
  for (j = 0; j < P; j++) bnd[j] = (uint64_t)j * part;
  bnd[P] = N;                                     /* last rank: the remainder */
  if (stats) memset(stats, 0, (size_t)P * sizeof(or_rank_stats));

  /* phase 1 (split): each rank slices its stream by partition and sends
   * slice_ij directly to owner j */
  for (i = 0; i < P; i++) {
    const uint32_t* ii = idx + off[i];
    const or_val* vv = val + off[i];
    uint64_t n = off[i + 1] - off[i];
    ksum += n;
    for (j = 0; j < P; j++) {
      uint64_t s0 = lower_bound_u32(ii, n, bnd[j]);
      uint64_t s1 = lower_bound_u32(ii, n, bnd[j + 1]);
      strm* s = &slices[(size_t)j * P + i];
      uint64_t t;
      if (strm_copy_in(s, ii + s0, vv + s0, s1 - s0)) return -1;
      for (t = 0; t < s->n; t++) s->idx[t] -= (uint32_t)bnd[j];  /* partition-local */
      if (stats && j != i) {
        stats[i].bytes_sent += PB * s->n;
        stats[i].pairs_sent += s->n;
        stats[i].msgs_sent += 1;
        stats[j].bytes_recv += PB * s->n;
      }
    }
  }
  /* each owner reduces the slices it received (canonical tree, R-8) */
  for (j = 0; j < P; j++) {
    if (tree_reduce(&slices[(size_t)j * P], 0, P, bnd[j + 1] - bnd[j], &R[j])) return -1;
    K += R[j].n;
  }

  /* SSAR vs DSAR: forced, or AUTO by the upper bound sum k_i > delta (R-5) */
  if (algo == OR_ALGO_DSAR_SPLIT) dsar = 1;
  else if (algo == OR_ALGO_SSAR_SPLIT) dsar = 0;
  else dsar = ksum > delta;
  if (dsar_used) *dsar_used = dsar;

  if (!dsar) {
    /* phase 2: concatenating sparse allgather; disjoint ranges
     * make the sum a concatenation.  If K > delta the
     * concatenation cannot be stored sparse and is densified. */
    strm res;
    memset(&res, 0, sizeof res);
    if (stats) {
      for (r = 0; r < P; r++)
        for (j = 0; j < P; j++)
          if (j != r) {
            stats[j].bytes_sent += PB * R[j].n; stats[j].pairs_sent += R[j].n;
            stats[j].msgs_sent += 1; stats[r].bytes_recv += PB * R[j].n;
          }
    }
    if (K > delta) {
      res.dense = 1; res.n = N;
      res.val = (or_val*)malloc((N ? N : 1) * sizeof(or_val));
      if (!res.val) return -1;
      for (e = 0; e < N; e++) res.val[e] = op_neutral();
      for (j = 0; j < P; j++)
        for (e = 0; e < R[j].n; e++) res.val[bnd[j] + R[j].idx[e]] = R[j].val[e];
    } else {
      uint64_t o = 0;
      res.dense = 0; res.n = K;
      res.idx = (uint32_t*)malloc((K ? K : 1) * sizeof(uint32_t));
      res.val = (or_val*)malloc((K ? K : 1) * sizeof(or_val));
      if (!res.idx || !res.val) return -1;
      for (j = 0; j < P; j++)
        for (e = 0; e < R[j].n; e++) {
          res.idx[o] = (uint32_t)(bnd[j] + R[j].idx[e]);
          res.val[o] = R[j].val[e];
          o++;
        }
    }
    for (r = 0; r < P && r < n_out; r++) strm_out(&res, N, r, out_dense, out_n, out_idx, out_val);
    strm_free(&res);
  } else {
    /* DSAR: owner switches its reduced split to dense (neutral fill 0),
     * optionally QSGD-encodes it (§6), then dense allgather. */
    or_val* dense = (or_val*)malloc((N ? N : 1) * sizeof(or_val));
    if (!dense) return -1;
    for (e = 0; e < N; e++) dense[e] = op_neutral();
    for (j = 0; j < P; j++) {
      uint64_t nj = bnd[j + 1] - bnd[j];
      or_val* Dj = dense + bnd[j];
      uint64_t wire;
      for (e = 0; e < R[j].n; e++) Dj[R[j].idx[e]] = R[j].val[e];
      if (quant_bits) {   /* fp32 build only (checked above) */
        uint64_t cb = (nj * (uint64_t)quant_bits + 7) / 8;
        uint64_t ns = (nj + bucket - 1) / bucket;
        uint8_t* codes = (uint8_t*)malloc(cb ? cb : 1);
        float* scales = (float*)malloc((ns ? ns : 1) * sizeof(float));
        if (!codes || !scales) return -1;
        or_qsgd_quantize((const float*)Dj, nj, quant_bits, bucket, seed, bnd[j], codes, scales);
        or_qsgd_dequantize(codes, scales, nj, quant_bits, bucket, (float*)Dj);
        free(codes); free(scales);
        wire = cb + 4 * ns;
      } else {
        wire = VB * nj;
      }
      if (stats)
        for (r = 0; r < P; r++)
          if (r != j) {
            stats[j].bytes_sent += wire; stats[j].msgs_sent += 1;
            stats[r].bytes_recv += wire;
          }
    }
    for (r = 0; r < P && r < n_out; r++) {
      out_dense[r] = 1; out_n[r] = N;
      memcpy(out_val + (uint64_t)r * N, dense, N * sizeof(or_val));
    }
    free(dense);
  }
  for (j = 0; j < P * P; j++) strm_free(&slices[j]);
  for (j = 0; j < P; j++) strm_free(&R[j]);
  free(slices); free(R); free(bnd);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* §2.2 / Algorithm 1: top-k and error feedback                               */
/* ------------------------------------------------------------------------- */

typedef struct { float mag; uint32_t j; } kv;

static int cmp_mag_desc_idx_asc(const void* pa, const void* pb) {
  const kv* a = (const kv*)pa;
  const kv* b = (const kv*)pb;
  if (a->mag > b->mag) return -1;
  if (a->mag < b->mag) return 1;
  if (a->j < b->j) return -1;   /* ties: lower index first (R-18) */
  if (a->j > b->j) return 1;
  return 0;
}

static int cmp_u32(const void* pa, const void* pb) {
  uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  return (a > b) - (a < b);
}

int or_sparse_allgather(int P, uint64_t N, uint64_t delta, const uint32_t* idx, const or_val* val,
                        const uint64_t* off, int n_out, int* out_dense, uint64_t* out_n,
                        uint32_t* out_idx, or_val* out_val, or_rank_stats* stats) {
  int r, i, j, order[256], m = 0;
  uint64_t K = 0, e, pos;
  if (P < 1 || P > 256 || N == 0 || n_out < 0 || n_out > P) return -1;
  /* non-empty ranks ordered by their first index (insertion sort, P <= 256) */
  for (r = 0; r < P; r++) {
    const uint64_t n = off[r + 1] - off[r];
    K += n;
    if (n == 0) continue;
    for (i = m; i > 0 && idx[off[order[i - 1]]] > idx[off[r]]; i--) order[i] = order[i - 1];
    order[i] = r;
    m++;
  }
  /* the precondition: consecutive ranges do not overlap */
  for (i = 0; i + 1 < m; i++) {
    const int a = order[i], b = order[i + 1];
    if (idx[off[a + 1] - 1] >= idx[off[b]]) return -2;
  }
  for (r = 0; r < n_out; r++) {
    uint32_t* oi = out_idx + (uint64_t)r * N;
    or_val* ov = out_val + (uint64_t)r * N;
    if (K > delta) {   /* dense result: zeros, then every value at its index */
      out_dense[r] = 1;
      out_n[r] = N;
      for (e = 0; e < N; e++) ov[e] = 0;
      for (j = 0; j < m; j++)
        for (e = off[order[j]]; e < off[order[j] + 1]; e++) ov[idx[e]] = val[e];
    } else {           /* sparse: the concatenation in range order */
      out_dense[r] = 0;
      out_n[r] = K;
      pos = 0;
      for (j = 0; j < m; j++)
        for (e = off[order[j]]; e < off[order[j] + 1]; e++, pos++) {
          oi[pos] = idx[e];
          ov[pos] = val[e];
        }
    }
  }
  if (stats)
    for (r = 0; r < P; r++) {
      const uint64_t n = off[r + 1] - off[r];
      memset(&stats[r], 0, sizeof(stats[r]));
      stats[r].bytes_sent = PB * n * (uint64_t)(P - 1);
      stats[r].bytes_recv = PB * (K - n);
      stats[r].msgs_sent = (uint64_t)(P - 1);
      stats[r].pairs_sent = n * (uint64_t)(P - 1);
    }
  return 0;
}

uint64_t or_topk(const float* x, uint64_t N, uint64_t k,
                 uint32_t* idx_out, float* val_out, float* residual) {
  /* "communicates only the k largest (by magnitude) components" */
  uint64_t m = k < N ? k : N, j;
  kv* all = (kv*)malloc((N ? N : 1) * sizeof(kv));
  if (!all) return 0;
  for (j = 0; j < N; j++) { all[j].mag = fabsf(x[j]); all[j].j = (uint32_t)j; }
  qsort(all, N, sizeof(kv), cmp_mag_desc_idx_asc);           /* brute force: full sort */
  for (j = 0; j < m; j++) idx_out[j] = all[j].j;
  qsort(idx_out, m, sizeof(uint32_t), cmp_u32);               /* emit in index order */
  for (j = 0; j < m; j++) val_out[j] = x[idx_out[j]];
  if (residual) {
    if (residual != x) memcpy(residual, x, N * sizeof(float));
    for (j = 0; j < m; j++) residual[idx_out[j]] = 0.0f;      /* acc - TopK(acc) */
  }
  free(all);
  return m;
}

uint64_t or_ef_topk(float* eps, const float* grad, float alpha, uint64_t N,
                    uint64_t k, uint32_t* idx_out, float* val_out) {
  uint64_t j;
  for (j = 0; j < N; j++) eps[j] = fmaf(alpha, grad[j], eps[j]);  /* acc */
  return or_topk(eps, N, k, idx_out, val_out, eps);              /* eps <- acc - TopK(acc) */
}

uint64_t or_topk_bucketed(const float* x, uint64_t N, uint64_t k, uint64_t B,
                          uint32_t* idx_out, float* val_out, float* residual) {
  /* every bucket of B consecutive coordinates selects its own top k */
  uint64_t m = 0, b0, j;
  if (residual && residual != x) memcpy(residual, x, N * sizeof(float));
  for (b0 = 0; b0 < N; b0 += B) {
    const uint64_t n = (N - b0 < B) ? N - b0 : B;
    const uint64_t mb = or_topk(x + b0, n, k, idx_out + m, val_out + m, NULL);
    for (j = 0; j < mb; j++) {
      idx_out[m + j] += (uint32_t)b0;                     /* bucket-relative -> global index */
      if (residual) residual[idx_out[m + j]] = 0.0f;      /* the rest is saved locally */
    }
    m += mb;
  }
  return m;
}

uint64_t or_ef_topk_bucketed(float* eps, const float* grad, float alpha, uint64_t N,
                             uint64_t k, uint64_t B, uint32_t* idx_out, float* val_out) {
  uint64_t j;
  for (j = 0; j < N; j++) eps[j] = fmaf(alpha, grad[j], eps[j]);   /* acc */
  return or_topk_bucketed(eps, N, k, B, idx_out, val_out, eps);
}

/* ------------------------------------------------------------------------- */
/* §6 QSGD low-precision encoding                                             */
/* ------------------------------------------------------------------------- */

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  /* Philox4x32 with 10 rounds, constants of Salmon et al. (Random123). */
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  int round;
  for (round = 0; round < 10; round++) {
    uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;   /* key bump between rounds (unused after the last) */
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

float or_qsgd_uniform(uint64_t seed, uint64_t c) {
  uint32_t ctr[4], key[2], w[4];
  uint64_t blk = c >> 2;
  ctr[0] = (uint32_t)blk; ctr[1] = (uint32_t)(blk >> 32); ctr[2] = 0; ctr[3] = 0;
  key[0] = (uint32_t)seed; key[1] = (uint32_t)(seed >> 32);
  or_philox4x32_10(ctr, key, w);
  return (float)(w[c & 3] >> 8) * (1.0f / 16777216.0f);   /* exact: 24-bit / 2^24 */
}

static int g_qnorm = 0;   /* 0: max-norm scale (R-16); 1: l2-norm scale (R-31) */

int or_set_qsgd_norm(int norm) {
  if (norm != 0 && norm != 1) return -1;
  g_qnorm = norm;
  return 0;
}

/* l2 scale of one bucket (R-31): squares fl(v*v), summed by the balanced
 * pairwise tree over the bucket's B slots in index order (slots past a
 * ragged end hold +0), then the correctly rounded square root. */
static float l2_scale(const float* v, uint64_t m, uint32_t B) {
  float* t = (float*)malloc((size_t)B * sizeof(float));
  uint32_t len, i;
  float r;
  if (!t) return 0.0f;
  for (i = 0; i < B; i++) t[i] = i < m ? v[i] * v[i] : 0.0f;
  for (len = B; len > 1; len /= 2)
    for (i = 0; i < len / 2; i++) t[i] = t[2 * i] + t[2 * i + 1];
  r = sqrtf(t[0]);
  free(t);
  return r;
}

int or_qsgd_quantize(const float* x, uint64_t n, int bits, uint32_t B,
                     uint64_t seed, uint64_t ctr_base, uint8_t* codes, float* scales) {
  uint64_t b0, e, nb;
  uint32_t s;
  int per_byte;
  if (bits != 2 && bits != 4 && bits != 8) return -1;
  if (B == 0) return -1;
  if (g_qnorm && (B & (B - 1))) return -1;   /* the l2 tree needs a power-of-two bucket */
  s = (1u << (bits - 1)) - 1u;            /* levels per sign: 1, 7, 127 */
  per_byte = 8 / bits;
  nb = (n * (uint64_t)bits + 7) / 8;
  for (e = 0; e < nb; e++) codes[e] = 0;
  for (b0 = 0; b0 < n; b0 += B) {
    uint64_t m = (n - b0) < B ? (n - b0) : B;
    float scale = 0.0f;
    if (g_qnorm) {
      scale = l2_scale(x + b0, m, B);
    } else {
      for (e = 0; e < m; e++) {              /* full-precision per-bucket scale */
        float a = fabsf(x[b0 + e]);
        if (a > scale) scale = a;
      }
    }
    scales[b0 / B] = scale;
    for (e = 0; e < m; e++) {
      uint64_t g = b0 + e;
      float v = x[g];
      uint32_t level = 0, code, neg;
      if (scale != 0.0f) {
        float u = or_qsgd_uniform(seed, ctr_base + g);
        float r = fabsf(v) / scale;
        float t = r * (float)s;
        float f = floorf(t + u);         /* stochastic rounding (unbiased) */
        level = (uint32_t)f;
        if (level > s) level = s;
      }
      neg = (v < 0.0f && level > 0) ? 1u : 0u;
      code = (neg << (bits - 1)) | level;
      codes[g / (uint64_t)per_byte] |= (uint8_t)(code << ((g % (uint64_t)per_byte) * (uint64_t)bits));
    }
  }
  return 0;
}

int or_qsgd_dequantize(const uint8_t* codes, const float* scales, uint64_t n,
                       int bits, uint32_t B, float* out) {
  uint64_t g;
  uint32_t s, mask;
  int per_byte;
  if (bits != 2 && bits != 4 && bits != 8) return -1;
  if (B == 0) return -1;
  s = (1u << (bits - 1)) - 1u;
  mask = (1u << bits) - 1u;
  per_byte = 8 / bits;
  for (g = 0; g < n; g++) {
    uint32_t code = (codes[g / (uint64_t)per_byte] >> ((g % (uint64_t)per_byte) * (uint64_t)bits)) & mask;
    uint32_t level = code & s;
    uint32_t neg = code >> (bits - 1);
    float mag = ((float)level / (float)s) * scales[g / B];
    out[g] = neg ? -mag : mag;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1, last line: v <- v - g                                 */
/* ------------------------------------------------------------------------- */

int or_apply_update(or_val* v, uint64_t N, int dense, uint64_t n,
                    const uint32_t* idx, const or_val* val) {
  uint64_t e;
  if (dense) {
    for (e = 0; e < N; e++) v[e] = v[e] - val[e];
    return 0;
  }
  for (e = 0; e < n; e++) {
    if (idx[e] >= N) return -1;
    v[idx[e]] = v[idx[e]] - val[e];
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* App. B: expected result size for uniform supports                          */
/* ------------------------------------------------------------------------- */

double or_expected_nnz(uint64_t k, uint64_t N, int P) {
  /* E[K] = N * sum_{i=1}^{P} (-1)^{i-1} C(P,i) (k/N)^i */
  long double d = (long double)k / (long double)N, sum = 0.0L, binom = 1.0L, pw = 1.0L;
  int i;
  for (i = 1; i <= P; i++) {
    binom = binom * (long double)(P - i + 1) / (long double)i;   /* C(P,i) */
    pw *= d;
    sum += ((i & 1) ? 1.0L : -1.0L) * binom * pw;
  }
  return (double)((long double)N * sum);
}
