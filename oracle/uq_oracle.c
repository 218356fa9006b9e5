/*
 * uq_oracle.c -- plain, slow, obviously-correct CPU oracle for the EVP ternary
 * search path of arXiv 2506.00528 ("Ultra-Quantisation: Efficient Embedding
 * Search via 1.58-bit Encodings").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_2506_00528_b200/) never includes, links or calls it, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Citations: "P:NNN" = /root/reference/PAPER.md line NNN (section given);
 * readings of ambiguous passages are numbered R1..R12 in DESIGN.md.
 *
 * Written in the paper's order and notation; no blocking, fusion or reordering
 * beyond what the definitions state.  OpenMP is used only to run independent
 * rows / queries in parallel (each row's / query's arithmetic is untouched).
 *
 * Pins: every function here is pinned in tests/test_oracle.py against values
 * the paper prints (Table 3, Fig. 2), closed forms, brute-force enumeration and
 * invariants.  Nothing here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Plane size of the packed code: 16 * ceil(d/128) bytes per plane (R6). */
int64_t orc_plane_bytes(int32_t d) { return 16 * (((int64_t)d + 127) / 128); }
int64_t orc_code_bytes(int32_t d) { return 2 * orc_plane_bytes(d); }

/* ------------------------------------------------------------------------ */
/* Encode: nearest {x,d} EVP vertex.  P:189-196 (Sec. 2.4):                   */
/*   1. find the x largest absolute elements in the vector                    */
/*   2. assign 1 to every positive element within this set, -1 to negative    */
/*   3. assign 0 to all other elements                                        */
/* Ties in |u_i| go to the lower index (R1); a selected exact zero maps to 0  */
/* (R2); -0.0 is zero (R3).  Values arrive as doubles: f32/f16 widen exactly. */
/* ------------------------------------------------------------------------ */
typedef struct { double mag; int32_t idx; } orc_mag_t;

static int cmp_mag_desc_idx_asc(const void* a, const void* b) {
  const orc_mag_t* x = (const orc_mag_t*)a;
  const orc_mag_t* y = (const orc_mag_t*)b;
  if (x->mag > y->mag) return -1;
  if (x->mag < y->mag) return 1;
  /* equal magnitude: lower index first (R1) */
  return (x->idx < y->idx) ? -1 : (x->idx > y->idx) ? 1 : 0;
}

static void encode_row(const double* u, int32_t d, int32_t x, int8_t* v) {
  orc_mag_t* m = (orc_mag_t*)malloc(sizeof(orc_mag_t) * (size_t)d);
  for (int32_t i = 0; i < d; ++i) { m[i].mag = fabs(u[i]); m[i].idx = i; }
  /* step 1: the x largest |u_i| (sort by |u| desc, index asc; take x) */
  qsort(m, (size_t)d, sizeof(orc_mag_t), cmp_mag_desc_idx_asc);
  /* step 3: all other elements 0 */
  for (int32_t i = 0; i < d; ++i) v[i] = 0;
  /* step 2: sign of each selected element */
  for (int32_t r = 0; r < x; ++r) {
    int32_t i = m[r].idx;
    v[i] = (int8_t)((u[i] > 0.0) - (u[i] < 0.0));
  }
  free(m);
}

/* u: [n][ld] doubles (row-major), v: [n][d] int8 ternary */
void orc_encode(const double* u, int64_t n, int32_t d, int64_t ld, int32_t x, int8_t* v) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t r = 0; r < n; ++r) encode_row(u + r * ld, d, x, v + r * (int64_t)d);
}

/* ------------------------------------------------------------------------ */
/* Pack: P:379 (Sec. 5.1.2) "binary vectors v+ and v- ... constructed by      */
/* simply mapping the position of the values 1 and -1".  Bit i lives in byte  */
/* i/8, bit i%8 (LSB first); pos plane then neg plane; pad bits are 0 (R6).   */
/* ------------------------------------------------------------------------ */
void orc_pack(const int8_t* v, int64_t n, int32_t d, uint8_t* codes) {
  const int64_t pb = orc_plane_bytes(d), cb = 2 * pb;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    uint8_t* pos = codes + r * cb;
    uint8_t* neg = pos + pb;
    memset(pos, 0, (size_t)cb);
    for (int32_t i = 0; i < d; ++i) {
      int8_t e = v[r * (int64_t)d + i];
      if (e == 1) pos[i / 8] |= (uint8_t)(1u << (i % 8));
      if (e == -1) neg[i / 8] |= (uint8_t)(1u << (i % 8));
    }
  }
}

/* Inverse of pack; a position with both bits set is reported as 2 (invalid). */
void orc_unpack(const uint8_t* codes, int64_t n, int32_t d, int8_t* v) {
  const int64_t pb = orc_plane_bytes(d), cb = 2 * pb;
  for (int64_t r = 0; r < n; ++r) {
    const uint8_t* pos = codes + r * cb;
    const uint8_t* neg = pos + pb;
    for (int32_t i = 0; i < d; ++i) {
      int p = (pos[i / 8] >> (i % 8)) & 1, q = (neg[i / 8] >> (i % 8)) & 1;
      v[r * (int64_t)d + i] = (int8_t)((p && q) ? 2 : (p - q));
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Scalar products.                                                          */
/* ------------------------------------------------------------------------ */
/* Plain ternary scalar product sum_i a_i b_i (Sec. 2.6). */
int32_t orc_dot_naive(const int8_t* a, const int8_t* b, int32_t d) {
  int32_t s = 0;
  for (int32_t i = 0; i < d; ++i) s += (int32_t)a[i] * (int32_t)b[i];
  return s;
}

/* bsp(v,w) = number of set bits of v AND w  (Sec. 5.1.2), counted one
   64-bit word at a time with the compiler's population-count primitive
   (__builtin_popcountll = the number of set bits of a word).  Planes are whole
   16-byte units (R6), so nbytes is a multiple of 8. */
static int32_t bsp(const uint8_t* v, const uint8_t* w, int64_t nbytes) {
  int32_t c = 0;
  for (int64_t j = 0; j < nbytes; j += 8) {
    uint64_t a, b;
    memcpy(&a, v + j, 8);
    memcpy(&b, w + j, 8);
    c += __builtin_popcountll(a & b);
  }
  return c;
}

/* b2sp(v,w) = (bsp(v+,w+) + bsp(v-,w-)) - (bsp(v+,w-) + bsp(v-,w+)) */
int32_t orc_b2sp(const uint8_t* cv, const uint8_t* cw, int32_t d) {
  const int64_t pb = orc_plane_bytes(d);
  const uint8_t *vp = cv, *vn = cv + pb, *wp = cw, *wn = cw + pb;
  return (bsp(vp, wp, pb) + bsp(vn, wn, pb)) - (bsp(vp, wn, pb) + bsp(vn, wp, pb));
}

/* Dense Delta matrix out[q][r] = b2sp(query q, db row r). */
void orc_scores(const uint8_t* qc, int64_t nq, const uint8_t* dc, int64_t n, int32_t d,
                int32_t* out) {
  const int64_t cb = orc_code_bytes(d);
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nq; ++q)
    for (int64_t r = 0; r < n; ++r) out[q * n + r] = orc_b2sp(qc + q * cb, dc + r * cb, d);
}

/* ------------------------------------------------------------------------ */
/* Exhaustive kNN in the proxy space (Sec. 1.1; Sec. 5.3.1):       */
/* Delta against every row; order by (Delta desc, id asc) (R7, R8); keep k;   */
/* pad with (INT32_MIN, -1) when n < k (R9).                                   */
/* ------------------------------------------------------------------------ */
typedef struct { int32_t s; int64_t id; } orc_cand_t;

static int cmp_cand(const void* a, const void* b) {
  const orc_cand_t* x = (const orc_cand_t*)a;
  const orc_cand_t* y = (const orc_cand_t*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  return (x->id < y->id) ? -1 : (x->id > y->id) ? 1 : 0;
}

/* one query: Delta against every row (rows in parallel: each row's
   arithmetic is untouched), then the plain sort, then the first k */
static void knn_one(const uint8_t* q, const uint8_t* dc, int64_t n, int32_t d, int32_t k, int64_t id_base,
                    int rows_parallel, int32_t* out_s, int64_t* out_id) {
  const int64_t cb = orc_code_bytes(d);
  orc_cand_t* c = (orc_cand_t*)malloc(sizeof(orc_cand_t) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(static) if (rows_parallel)
  for (int64_t r = 0; r < n; ++r) {
    c[r].s = orc_b2sp(q, dc + r * cb, d);
    c[r].id = id_base + r;
  }
  qsort(c, (size_t)n, sizeof(orc_cand_t), cmp_cand);
  for (int32_t j = 0; j < k; ++j) {
    out_s[j] = (j < n) ? c[j].s : INT32_MIN;
    out_id[j] = (j < n) ? c[j].id : -1;
  }
  free(c);
}

/* threads of the OpenMP loops (1 without OpenMP) */
static int orc_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_knn(const uint8_t* qc, int64_t nq, const uint8_t* dc, int64_t n, int32_t d, int32_t k,
             int64_t id_base, int32_t* out_s, int64_t* out_id) {
  const int64_t cb = orc_code_bytes(d);
  if (nq >= orc_threads()) {
    /* many queries: one query per thread */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nq; ++q) knn_one(qc + q * cb, dc, n, d, k, id_base, 0, out_s + q * k, out_id + q * k);
  } else {
    /* few queries over many rows (full-size sampled checks): rows in parallel */
    for (int64_t q = 0; q < nq; ++q) knn_one(qc + q * cb, dc, n, d, k, id_base, 1, out_s + q * k, out_id + q * k);
  }
}

/* ------------------------------------------------------------------------ */
/* Single-operand translation (Sec. 6.1): only the database is      */
/* ternary; the query stays in the original space "quantised to 8-bit         */
/* integers", and the scalar product is the masked addition of P:379          */
/* (Sec. 5.1.2): add q_i where v_i^+ = 1, subtract q_i where v_i^- = 1.        */
/* Quantisation (R15; the paper names no scheme): per vector, scale =         */
/* 127 / max_i |u_i| and q_i = round-half-even(u_i * scale), both in fp32      */
/* arithmetic; an all-zero vector maps to zeros.                               */
/* ------------------------------------------------------------------------ */
void orc_quantize_i8(const float* u, int64_t n, int32_t d, int8_t* out) {
  for (int64_t r = 0; r < n; ++r) {
    const float* row = u + r * d;
    float m = 0.0f;
    for (int32_t i = 0; i < d; ++i) {
      const float a = fabsf(row[i]);
      if (a > m) m = a;
    }
    const float scale = (m > 0.0f) ? 127.0f / m : 0.0f;
    for (int32_t i = 0; i < d; ++i) {
      float q = rintf(row[i] * scale);
      if (q > 127.0f) q = 127.0f;
      if (q < -127.0f) q = -127.0f;
      out[r * d + i] = (int8_t)q;
    }
  }
}

/* masked addition of one int8 query against one packed ternary row */
static int32_t masked_add(const int8_t* q, const uint8_t* code, int32_t d) {
  const int64_t pb = orc_plane_bytes(d);
  int32_t s = 0;
  for (int32_t i = 0; i < d; ++i) {
    const int pos = (code[i / 8] >> (i % 8)) & 1;
    const int neg = (code[pb + i / 8] >> (i % 8)) & 1;
    if (pos) s += q[i];
    if (neg) s -= q[i];
  }
  return s;
}

static void knn_asym_one(const int8_t* q, const uint8_t* dc, int64_t n, int32_t d, int32_t k, int64_t id_base,
                         int rows_parallel, int32_t* out_s, int64_t* out_id) {
  const int64_t cb = orc_code_bytes(d);
  orc_cand_t* c = (orc_cand_t*)malloc(sizeof(orc_cand_t) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(static) if (rows_parallel)
  for (int64_t r = 0; r < n; ++r) {
    c[r].s = masked_add(q, dc + r * cb, d);
    c[r].id = id_base + r;
  }
  qsort(c, (size_t)n, sizeof(orc_cand_t), cmp_cand);
  for (int32_t j = 0; j < k; ++j) {
    out_s[j] = (j < n) ? c[j].s : INT32_MIN;
    out_id[j] = (j < n) ? c[j].id : -1;
  }
  free(c);
}

/* Exhaustive kNN by masked addition: order (score desc, id asc), keep k, pad. */
void orc_knn_asym(const int8_t* q8, int64_t nq, const uint8_t* dc, int64_t n, int32_t d, int32_t k,
                  int64_t id_base, int32_t* out_s, int64_t* out_id) {
  if (nq >= orc_threads()) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nq; ++q) knn_asym_one(q8 + q * d, dc, n, d, k, id_base, 0, out_s + q * k, out_id + q * k);
  } else {
    for (int64_t q = 0; q < nq; ++q) knn_asym_one(q8 + q * d, dc, n, d, k, id_base, 1, out_s + q * k, out_id + q * k);
  }
}

/* ------------------------------------------------------------------------ */
/* Cosine ground truth in fp64 (Sec. 1.1; R12): normalise each row,  */
/* cos = <q^, u^>; order by (cos desc, id asc); keep k.                        */
/* ------------------------------------------------------------------------ */
typedef struct { double s; int64_t id; } orc_fcand_t;

static int cmp_fcand(const void* a, const void* b) {
  const orc_fcand_t* x = (const orc_fcand_t*)a;
  const orc_fcand_t* y = (const orc_fcand_t*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  return (x->id < y->id) ? -1 : (x->id > y->id) ? 1 : 0;
}

static double norm2(const double* a, int32_t d) {
  double s = 0.0;
  for (int32_t i = 0; i < d; ++i) s += a[i] * a[i];
  return sqrt(s);
}

void orc_cosine_knn(const double* qv, int64_t nq, const double* dv, int64_t n, int32_t d,
                    int32_t k, double* out_s, int64_t* out_id) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nq; ++q) {
    orc_fcand_t* c = (orc_fcand_t*)malloc(sizeof(orc_fcand_t) * (size_t)(n > 0 ? n : 1));
    const double* a = qv + q * d;
    double na = norm2(a, d);
    for (int64_t r = 0; r < n; ++r) {
      const double* b = dv + r * d;
      double nb = norm2(b, d), dot = 0.0;
      for (int32_t i = 0; i < d; ++i) dot += (a[i] / na) * (b[i] / nb);
      c[r].s = dot;
      c[r].id = r;
    }
    qsort(c, (size_t)n, sizeof(orc_fcand_t), cmp_fcand);
    for (int32_t j = 0; j < k; ++j) {
      out_s[q * k + j] = (j < n) ? c[j].s : -INFINITY;
      out_id[q * k + j] = (j < n) ? c[j].id : -1;
    }
    free(c);
  }
}

/* ------------------------------------------------------------------------ */
/* k@n re-rank (Sec. 5.3): the candidates of the approximate       */
/* search are "reordered with respect to the original space, with the best k */
/* then selected" -- fp64 cosine of each candidate, (cos desc, id asc), top k. */
/* ------------------------------------------------------------------------ */
void orc_rerank(const double* qv, int64_t nq, const double* dv, int64_t n, int32_t d,
                const int64_t* cand, int32_t n_cand, int32_t k, double* out_s, int64_t* out_id) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nq; ++q) {
    orc_fcand_t* c = (orc_fcand_t*)malloc(sizeof(orc_fcand_t) * (size_t)n_cand);
    const double* a = qv + q * d;
    const double na = norm2(a, d);
    int32_t m = 0;
    for (int32_t j = 0; j < n_cand; ++j) {
      const int64_t id = cand[q * n_cand + j];
      if (id < 0 || id >= n) continue;
      const double* b = dv + id * d;
      const double nb = norm2(b, d);
      double dot = 0.0;
      for (int32_t i = 0; i < d; ++i) dot += (a[i] / na) * (b[i] / nb);
      c[m].s = dot;
      c[m].id = id;
      ++m;
    }
    qsort(c, (size_t)m, sizeof(orc_fcand_t), cmp_fcand);
    for (int32_t j = 0; j < k; ++j) {
      out_s[q * k + j] = (j < m) ? c[j].s : -INFINITY;
      out_id[q * k + j] = (j < m) ? c[j].id : -1;
    }
    free(c);
  }
}

/* Rows whose code is not a valid packed ternary vector: a position set in both
 * planes (pos AND neg != 0, the invariant of P:369-372), or a set pad bit (R6). */
int64_t orc_check_codes(const uint8_t* codes, int64_t n, int32_t d) {
  const int64_t pb = orc_plane_bytes(d), cb = 2 * pb;
  int64_t bad = 0;
  for (int64_t r = 0; r < n; ++r) {
    const uint8_t* pos = codes + r * cb;
    const uint8_t* neg = pos + pb;
    int is_bad = 0;
    for (int64_t i = 0; i < pb * 8; ++i) {
      int p = (pos[i / 8] >> (i % 8)) & 1, q = (neg[i / 8] >> (i % 8)) & 1;
      if (p && q) is_bad = 1;
      if (i >= d && (p || q)) is_bad = 1;
    }
    bad += is_bad;
  }
  return bad;
}

/* ------------------------------------------------------------------------ */
/* Timing harness only (not arithmetic): worker threads of the OpenMP loops. */
/* ------------------------------------------------------------------------ */
int orc_set_threads(int n) {
#ifdef _OPENMP
  int prev = omp_get_max_threads();
  if (n > 0) omp_set_num_threads(n);
  return prev;
#else
  (void)n;
  return 1;
#endif
}
