/*
 * uq.h -- C ABI of libuq.so: B200 (sm_100a) brute-force kNN over {x,d} EVP
 * ternary codes (arXiv 2506.00528, "Ultra-Quantisation: Efficient Embedding
 * Search via 1.58-bit Encodings").  Citations: P:NNN = PAPER.md line.
 *
 * Conventions (all entry points):
 *  - Every pointer is a CUDA DEVICE pointer unless marked "host".  The caller
 *    owns every buffer; the library allocates nothing and keeps no state beyond
 *    cached device attributes, so calls are thread-safe and reentrant.
 *  - Every call is stream-ordered and asynchronous on `stream` (0 = legacy
 *    default stream).  Device faults surface at the caller's next sync.
 *  - Argument checks are synchronous and return before any launch:
 *      UQ_ERR_INVALID_ARG  null pointer with a non-empty extent, n/nq < 0,
 *                          d < 1, x outside [1,d], k < 1, ld < d,
 *                          misaligned pointer (codes: 16 B; u: element size);
 *      UQ_ERR_UNSUPPORTED  beyond compiled limits: d > UQ_MAX_D, k > UQ_MAX_K,
 *                          n >= 2^32-1 rows in one call;
 *      UQ_ERR_WORKSPACE    workspace smaller than uq_search_workspace();
 *      UQ_ERR_CUDA         a launch / attribute call failed.
 *  - Preconditions NOT checked: inputs are finite; codes are valid (pos AND
 *    neg = 0, pad bits 0) -- uq_check_codes() verifies them on demand.
 *
 * Code layout (one row = code_bytes = 2 * plane_bytes bytes, 16-B aligned):
 *    [ pos plane : plane_bytes ][ neg plane : plane_bytes ],
 *    plane_bytes = 16 * ceil(d / 128);  bit i of a plane is bit (i % 8) of
 *    byte (i / 8) (LSB first); pos bit i <=> v_i = +1, neg bit i <=> v_i = -1
 *    (the v+ / v- planes of P:357); bits i >= d are 0.
 *
 * Ranking: Delta = b2sp(q, r), the integer ternary scalar product;
 * larger is more similar (negative scalar product ~ l2 distance).  Ties
 * in Delta go to the lower id.  Results are sorted best first.
 */
#ifndef UQ_H_
#define UQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* uq_stream_t; /* == cudaStream_t */

typedef enum {
  UQ_OK = 0,
  UQ_ERR_INVALID_ARG = 1,
  UQ_ERR_UNSUPPORTED = 2,
  UQ_ERR_CUDA = 3,
  UQ_ERR_WORKSPACE = 4
} uq_status;

typedef enum { UQ_F32 = 0, UQ_F16 = 1, UQ_BF16 = 2 } uq_dtype;

/* Scan engine selection for uq_search_ex (uq_search uses UQ_ALGO_AUTO). */
typedef enum {
  UQ_ALGO_AUTO = 0,    /* tensor path for large query batches, popcount otherwise */
  UQ_ALGO_POPC = 1,    /* LOP3 + POPC scan on CUDA cores                          */
  UQ_ALGO_TCGEN05 = 2, /* int8 tcgen05 GEMM (UTCIMMA) with fused top-k            */
  UQ_ALGO_TC_FP4 = 3   /* E2M1 tcgen05 GEMM on CTA pairs (kind::mxf4, UTCOMMA):
                          ternary values are exact in E2M1, scales fixed at 2^0,
                          f32 accumulation of |Delta| <= 2048 is exact; d <= 1536 */
} uq_algo;

#define UQ_MAX_D 2048
#define UQ_MAX_K 1024

/* Bytes of one packed code row: 2 * 16 * ceil(d/128).  0 if d < 1. */
size_t uq_code_bytes(int32_t d);

/* Static string for a status code (never NULL). */
const char* uq_status_str(uq_status s);

/* Library version string, e.g. "uq 0.1 sm_100a". */
const char* uq_version(void);

/*
 * uq_encode -- nearest {x,d} EVP vertex of each row, packed.
 *   u      [n][ld_elems] row-major, element type dt (f32 / f16 / bf16).
 *          Encoded on raw values (no normalisation: the top-x order is scale
 *          invariant), comparing |u_i| exactly (IEEE abs bits).
 *   x      number of non-zeros, 1 <= x <= d.  Ties in |u_i| go to the
 *          lower index i; a selected exact zero (or -0.0) encodes as 0.
 *   codes  [n][uq_code_bytes(d)] output, 16-B aligned.
 */
uq_status uq_encode(const void* u, uq_dtype dt, int64_t n, int32_t d, int64_t ld_elems,
                    int32_t x, uint8_t* codes, uq_stream_t stream);

/*
 * uq_scores -- dense Delta matrix (test/debug): out[q][r] = b2sp(qcodes[q],
 * dbcodes[r]), int32, row-major [nq][n].
 */
uq_status uq_scores(const uint8_t* qcodes, int64_t nq, const uint8_t* dbcodes, int64_t n,
                    int32_t d, int32_t* out, uq_stream_t stream);

/*
 * uq_search_workspace -- bytes of device workspace uq_search needs for this
 * shape on the CURRENT device (*bytes is a host pointer).  Sizing helper of
 * uq_search (P:61 / P:480); the workspace holds the per-CTA top-k stream
 * buffers, the per-chunk candidate lists of the merge and the threshold
 * seed, never results.  Errors as uq_search's
 * synchronous checks; UQ_ERR_UNSUPPORTED if no engine runs the shape.
 */
uq_status uq_search_workspace(int64_t nq, int64_t n, int32_t d, int32_t k, size_t* bytes);
uq_status uq_search_workspace_ex(int64_t nq, int64_t n, int32_t d, int32_t k, uq_algo algo,
                                 size_t* bytes);

/*
 * uq_search_resolve -- which scan engine uq_search_ex(algo) runs for this shape
 * on the CURRENT device (*resolved is a host pointer; UQ_ALGO_POPC,
 * UQ_ALGO_TCGEN05 or UQ_ALGO_TC_FP4).  UQ_ERR_UNSUPPORTED if `algo` cannot run this shape.
 */
uq_status uq_search_resolve(int64_t nq, int64_t n, int32_t d, int32_t k, uq_algo algo,
                            uq_algo* resolved);

/*
 * uq_search -- exhaustive kNN in the proxy space (P:61 problem statement;
 * P:480 "exhaustive queries over the whole data").  For every query q: Delta
 * against every row r of dbcodes, keep the k best under (Delta desc, id asc),
 * write them best first:
 *   out_scores [nq][k] int32 Delta,   out_ids [nq][k] int64 id = id_base + r.
 * If n < k the tail of each row is (INT32_MIN, -1).  The result is unique
 * (total order), hence identical for every engine, launch shape and sharding.
 *   workspace  device scratch of >= uq_search_workspace() bytes, 256-B aligned.
 */
uq_status uq_search(const uint8_t* qcodes, int64_t nq, const uint8_t* dbcodes, int64_t n,
                    int32_t d, int32_t k, int64_t id_base, int32_t* out_scores,
                    int64_t* out_ids, void* workspace, size_t workspace_bytes,
                    uq_stream_t stream);
uq_status uq_search_ex(const uint8_t* qcodes, int64_t nq, const uint8_t* dbcodes, int64_t n,
                       int32_t d, int32_t k, int64_t id_base, int32_t* out_scores,
                       int64_t* out_ids, void* workspace, size_t workspace_bytes, uq_algo algo,
                       uq_stream_t stream);

/*
 * E2M1 index (an acceleration structure for UQ_ALGO_TC_FP4, not a new code
 * format): the database codes expanded once to the E2M1 operand of the pair
 * engine (4 bits per dim), each 120-row half tile stored as the kernel's
 * shared-memory stage image, rows padded with zeros to whole 240-row tiles.
 * With it a pipeline stage is one bulk copy (cp.async.bulk) instead of a
 * 2-bit -> E2M1 expansion by the producer warps; results are identical.
 *   uq_f4_index_bytes(n, d)                   size of the index (host call)
 *   uq_build_f4_index(dbcodes, n, d, index)   fills it (device buffers, 16-B aligned)
 *   uq_search_f4x(..., dbcodes, index, index_bytes, ...)
 *                                             uq_search_ex(UQ_ALGO_TC_FP4) reading the
 *                                             index (dbcodes still serves the
 *                                             workspace plan; d <= 1536)
 * index_bytes must equal uq_f4_index_bytes(n, d): an index built for another
 * row count is rejected synchronously (UQ_ERR_INVALID_ARG) instead of being
 * read out of bounds.  Other errors as uq_search_ex; UQ_ERR_UNSUPPORTED for
 * d > 1536.
 */
size_t uq_f4_index_bytes(int64_t n, int32_t d);
uq_status uq_build_f4_index(const uint8_t* dbcodes, int64_t n, int32_t d, uint8_t* index,
                            uq_stream_t stream);
uq_status uq_search_f4x(const uint8_t* qcodes, int64_t nq, const uint8_t* dbcodes, const uint8_t* index,
                        size_t index_bytes, int64_t n, int32_t d, int32_t k, int64_t id_base, int32_t* out_scores,
                        int64_t* out_ids, void* workspace, size_t workspace_bytes, uq_stream_t stream);

/*
 * int8 index: the same acceleration structure for the int8 pair engine (8
 * bits per dim, 128-row half tiles as its stage image, rows padded to 256),
 * used by single-operand search.  d <= 1024.
 *   uq_i8_index_bytes(n, d), uq_build_i8_index(dbcodes, n, d, index)
 *   uq_search_asym_x(..., index, index_bytes, ...)   uq_search_asym reading the
 *                           index; index_bytes must equal uq_i8_index_bytes(n, d)
 *                           (else UQ_ERR_INVALID_ARG)
 */
size_t uq_i8_index_bytes(int64_t n, int32_t d);
uq_status uq_build_i8_index(const uint8_t* dbcodes, int64_t n, int32_t d, uint8_t* index,
                            uq_stream_t stream);
uq_status uq_search_asym_x(const int8_t* q8, int64_t nq, int64_t ldq, const uint8_t* dbcodes,
                           const uint8_t* index, size_t index_bytes, int64_t n, int32_t d, int32_t k, int64_t id_base,
                           int32_t* out_scores, int64_t* out_ids, void* workspace,
                           size_t workspace_bytes, uq_stream_t stream);

/*
 * uq_merge_topk -- merge g sorted-or-unsorted candidate lists per query (e.g.
 * the per-GPU results of a sharded search after an allgather) into the k best
 * under (score desc, id asc):
 *   scores [g][nq][k] int32, ids [g][nq][k] int64 (entries with id < 0 are
 *   padding and ignored; ids must be < 2^32 - 1 and distinct per query),
 *   out_scores / out_ids [nq][k], best first, padded with (INT32_MIN, -1).
 * Exact because the global top-k is a subset of the union of shard top-k's.
 */
uq_status uq_merge_topk(const int32_t* scores, const int64_t* ids, int32_t g, int64_t nq,
                        int32_t k, int32_t* out_scores, int64_t* out_ids, uq_stream_t stream);

/*
 * uq_merge_topk_ptrs -- uq_merge_topk over g lists given by base pointers:
 * score_ptrs / id_ptrs are DEVICE arrays of g device pointers, list r being
 * scores [nq][k] int32 / ids [nq][k] int64 at score_ptrs[r] / id_ptrs[r].  The
 * pointers may be peer-mapped buffers of other GPUs (CUDA IPC / symmetric
 * memory over NVLink): the exchange step of the G-GPU search then is this one
 * kernel reading every rank's lists directly, with no staging allgather.
 * Same ordering, padding and errors as uq_merge_topk.
 */
uq_status uq_merge_topk_ptrs(const int32_t* const* score_ptrs, const int64_t* const* id_ptrs, int32_t g,
                             int64_t nq, int32_t k, int32_t* out_scores, int64_t* out_ids,
                             uq_stream_t stream);

/*
 * uq_check_codes -- count rows that are not valid packed ternary codes.  A
 * code is an EVP vertex component-wise in {-1, 0, 1}, stored as the
 * two bit planes v+ / v- of P:357 and P:379 ("positive and negative elements"
 * of Table 3), so no position can be set in both planes; bits past
 * d are the plane padding (reading R6 of DESIGN.md) and must be 0,
 * which keeps b2sp padding-independent.  A row is counted if some
 * position is set in both planes (pos AND neg != 0) or a pad bit (i >= d) is
 * set.  *bad_rows is a DEVICE uint64 scalar that the call overwrites.  The
 * search kernels assume valid codes (their 2-popcount identity needs
 * pos AND neg = 0); this call is the on-demand check of that precondition.
 * Errors: UQ_ERR_INVALID_ARG for n < 0, d < 1, a null bad_rows, or null /
 * misaligned codes with n > 0; UQ_ERR_UNSUPPORTED for d > UQ_MAX_D.
 */
uq_status uq_check_codes(const uint8_t* codes, int64_t n, int32_t d,
                         unsigned long long* bad_rows, uq_stream_t stream);

/*
 * uq_quantize_i8 -- query quantisation for single-operand search (P:507-509:
 * queries "quantised to 8-bit integers"; the scheme is reading R15 of
 * DESIGN.md): per row, scale = 127 / max_i |u_i| and out_i =
 * round-half-even(u_i * scale) in IEEE fp32, clamped to [-127, 127]; an
 * all-zero row maps to zeros.
 *   u   [n][ld] f32 / f16 / bf16 (element type dt), ld >= d
 *   out [n][ldo] int8, ldo >= d; columns >= d are not written.
 * Errors: UQ_ERR_INVALID_ARG for bad sizes / null pointers / misalignment,
 * UQ_ERR_UNSUPPORTED for d > UQ_MAX_D.
 */
uq_status uq_quantize_i8(const void* u, uq_dtype dt, int64_t n, int32_t d, int64_t ld, int8_t* out,
                         int64_t ldo, uq_stream_t stream);

/*
 * uq_search_asym -- single-operand exhaustive kNN (Sec. 6.1): only
 * the database is ternary; each query is an int8 vector q (e.g. from
 * uq_quantize_i8) and the score of row v is the masked addition of P:379,
 * S = sum_{v_i = +1} q_i - sum_{v_i = -1} q_i (an exact int32, |S| <= 127 d).
 * Results as uq_search: (S desc, id asc), ids = id_base + row, padding
 * (INT32_MIN, -1).
 *   q8 [nq][ldq] int8 (device), ldq >= d; dbcodes [n][code_bytes(d)] (16-B
 *   aligned); workspace >= uq_search_asym_workspace() bytes, 256-B aligned.
 * Runs on the int8 tcgen05 CTA-pair engine (the queries are the A operand)
 * with the same verified optimistic seeding as uq_search: d <= 1024,
 * otherwise UQ_ERR_UNSUPPORTED.  Other errors as uq_search.
 */
uq_status uq_search_asym_workspace(int64_t nq, int64_t n, int32_t d, int32_t k, size_t* bytes);
uq_status uq_search_asym(const int8_t* q8, int64_t nq, int64_t ldq, const uint8_t* dbcodes, int64_t n,
                         int32_t d, int32_t k, int64_t id_base, int32_t* out_scores, int64_t* out_ids,
                         void* workspace, size_t workspace_bytes, uq_stream_t stream);

/*
 * uq_rerank -- k@n: re-rank proxy-space candidates in the original space
 * (Sec. 5.3: "n > k results are found from the approximate search,
 * which are then reordered with respect to the original space, with the best k
 * then selected").  For query i the candidates cand[i][0..n_cand) (database
 * row ids, e.g. uq_search's ids with k = n_cand; ids < 0 or >= n are skipped;
 * ids must be distinct) are scored by cosine similarity of the float vectors and the
 * best k kept, ordered by (cos desc, id asc).
 *   q       [nq][ldq] query vectors, element type dt (f32 / f16 / bf16)
 *   db      [n][ld] database vectors, same dt (the vectors the codes came from)
 *   cand    [nq][n_cand] int64, 1 <= n_cand <= UQ_MAX_K
 *   out_cos [nq][k] f32 cosines (fp32 arithmetic; padding -inf), out_ids
 *           [nq][k] int64 (padding -1), 1 <= k <= n_cand.
 * Errors: UQ_ERR_INVALID_ARG for bad sizes / null pointers / misaligned
 * vectors, UQ_ERR_UNSUPPORTED for d > UQ_MAX_D, n_cand > UQ_MAX_K or
 * n >= 2^32 - 1.  Fewer than k valid candidates pad the tail.
 */
uq_status uq_rerank(const void* q, uq_dtype dt, int64_t nq, int64_t ldq, const void* db, int64_t n,
                    int64_t ld, int32_t d, const int64_t* cand, int32_t n_cand, int32_t k,
                    float* out_cos, int64_t* out_ids, uq_stream_t stream);

/*
 * Device-side timing of the scan kernels (the dominant kernel of uq_search), for
 * roofline accounting.  While enabled on a host thread, each scan launch issued
 * from that thread is bracketed by CUDA events on its stream.  collect() waits
 * for the recorded events, returns the summed kernel time (*scan_ms, host) and
 * the number of timed launches (*launches, host), and resets the record.
 */
uq_status uq_timing_enable(int32_t on);
uq_status uq_timing_collect(double* scan_ms, int64_t* launches);
/*
 * uq_timing_collect_ex -- as uq_timing_collect, split by launch kind: index 0 =
 * main scans (every database row), index 1 = threshold-seeding scans over a
 * strided sample.  scan_ms[2], launches[2] and delta_evals[2] (host arrays)
 * receive the summed kernel time, the launch count and the summed Delta
 * evaluations (nq x rows) of each kind.  Resets the record.
 */
uq_status uq_timing_collect_ex(double* scan_ms, int64_t* launches, double* delta_evals);

/*
 * uq_last_launches -- number of kernels the most recent uq_* call on this
 * host thread enqueued (for launch accounting in benchmarks).
 */
int32_t uq_last_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* UQ_H_ */
