// internal.h -- launch plans and launchers shared between the C-ABI layer
// (api.cu) and the kernel translation units.  Product path only.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/uq.h"

// Timing ablations and cycle accounting of the tensor scans (tools/ only).
// The product library is built WITHOUT UQ_PROFILE: UQ_DBG(p) is the constant 0,
// every ablation / profiling branch is compiled out, and no environment
// variable can change a result.  `python paper_2506_00528_b200/build.py
// --profile` builds libuq_prof.so with them for tools/tc2_prof.py.
#ifdef UQ_PROFILE
#define UQ_DBG(p) ((p).dbg)
#else
#define UQ_DBG(p) 0
#endif

namespace uq {

// env UQ_TC_ABLATE in profile builds, 0 otherwise
int tc_ablate_flags();

void note_launch(int n = 1);

// Phi^-1(p) (rational approximation; steering heuristics only, never a result)
float inv_norm_cdf(double p);

cudaError_t launch_encode(const void* u, uq_dtype dt, int64_t n, int32_t d, int64_t ld, int32_t x,
                          uint8_t* codes, int sms, cudaStream_t st);
cudaError_t launch_scores(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                          int32_t* out, cudaStream_t st);
cudaError_t launch_check_codes(const uint8_t* codes, int64_t n, int32_t d, unsigned long long* bad,
                               int sms, cudaStream_t st);
cudaError_t launch_merge_keys(const uint64_t* keys, int64_t lists, int64_t nq, int32_t kin, int32_t k,
                              int64_t id_base, int32_t* out_s, int64_t* out_id, cudaStream_t st,
                              const int32_t* counts = nullptr, const int32_t* only = nullptr,
                              const int32_t* any = nullptr, void* scratch = nullptr, size_t scratch_bytes = 0);
// bytes of workspace for the two-level merge of a search with nq queries (0: single level)
size_t merge_scratch_bytes(int64_t nq, int32_t k);
cudaError_t launch_rerank(const void* q, uq_dtype dt, int64_t nq, int64_t ldq, const void* db, int64_t n,
                          int64_t ld, int32_t d, const int64_t* cand, int32_t n_cand, int32_t k, float* out_cos,
                          int64_t* out_ids, cudaStream_t st);
cudaError_t launch_merge_si(const int32_t* scores, const int64_t* ids, int64_t lists, int64_t nq,
                            int32_t k, int32_t* out_s, int64_t* out_id, cudaStream_t st);
cudaError_t launch_merge_ptrs(const int32_t* const* score_ptrs, const int64_t* const* id_ptrs, int64_t lists,
                              int64_t nq, int32_t k, int32_t* out_s, int64_t* out_id, cudaStream_t st);

// Popcount scan (scan_popc.cu).
struct PopcPlan {
  int32_t qt, n_qtiles, cap, grid, smem;
  int32_t stages;   // > 0: the TMA-fed kernel with this many ring stages (one CTA per SM)
  int64_t L, n_chunks;
  size_t buf_bytes, part_bytes;
};
PopcPlan plan_popc(int64_t nq, int64_t n, int32_t d, int32_t k, int sms);
cudaError_t launch_scan_popc(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                             int32_t k, const PopcPlan& pl, uint32_t* bufs, uint64_t* part,
                             const int32_t* thr0, int32_t thr0_stride, int64_t row_stride,
                             cudaStream_t st, int32_t* part_cnt = nullptr);

// Tensor-core scan (scan_tc.cu).
struct TcPlan {
  bool ok;
  int32_t grid, smem, n_qtiles, cap, stages;
  int32_t s_lo, r_hi;   // query tile t is split into s_lo + (t < r_hi) DB chunks
  int64_t n_items;
  int64_t n_chunks;     // lists per query for the merge (= max chunks per tile)
  size_t buf_bytes, part_bytes;
};
TcPlan plan_tc(int64_t nq, int64_t n, int32_t d, int32_t k, int sms);
cudaError_t launch_scan_tc(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                           int32_t k, const TcPlan& pl, uint32_t* bufs, uint64_t* part,
                           const int32_t* thr0, int32_t thr0_stride, int64_t row_stride,
                           cudaStream_t st);

// Tensor-core scan on CTA pairs (scan_tc2.cu), used for query batches > 128;
// op: operand kind, 0 = int8 (kind::i8), 1 = E2M1 (kind::mxf4, f32 accumulate).
// sbound: bound on |score| (d for ternary queries; 127 d for int8 queries)
TcPlan plan_tc2(int64_t nq, int64_t n, int32_t d, int32_t k, int sms, int op, int32_t sbound = 0);
cudaError_t tc2_prof_read(unsigned long long* out48);
TcPlan plan_tc2_hist(int64_t nq, int64_t n, int32_t d, int32_t k, int sms, int op);
// Seeding: histogram scan over rows {i * row_stride : i < n}, then per query
// thr[q] = the largest bin edge with at least `need` sampled rows at or above
// it (INT32_MIN if none).  need = k: an exact lower bound on D_k; need < k: an
// optimistic bound, checked after the main scan by launch_seed_verify.
cudaError_t launch_seed_tc2_hist(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                                 int32_t k, int32_t need, int64_t row_stride, uint32_t* ghist, uint32_t* qbase,
                                 int32_t* thr, int sms, int op, cudaStream_t st, const int8_t* q8 = nullptr,
                                 int64_t ldq8 = 0, const uint8_t* dbx = nullptr, size_t dbx_bytes = 0);
// After a search with optimistic seeds: fail[q] = 1 iff q was filtered
// (thr[q] != INT32_MIN) and fewer than k rows passed (its k-th result is
// padding); *any |= 1 if some query failed (*any must be zero on entry).
cudaError_t launch_seed_verify(const int64_t* out_ids, int64_t nq, int32_t k, const int32_t* thr, int32_t* fail,
                               int32_t* any, cudaStream_t st);
// qfail / any_fail (optional, the seed fallback pass): the launch is a no-op
// unless *any_fail, and only pair tiles holding a query with qfail[q] run.
cudaError_t launch_scan_tc2(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                            int32_t k, const TcPlan& pl, uint32_t* bufs, uint64_t* part, int32_t* part_cnt,
                            const int32_t* thr0, int32_t thr0_stride, int64_t row_stride, int op,
                            cudaStream_t st, const int32_t* qfail = nullptr, const int32_t* any_fail = nullptr,
                            const int8_t* q8 = nullptr, int64_t ldq8 = 0, const uint8_t* dbx = nullptr,
                            size_t dbx_bytes = 0);
// E2M1 index (uq_build_f4_index): rows padded to whole 240-row pair tiles
size_t f4_index_bytes(int64_t n, int32_t d);
size_t i8_index_bytes(int64_t n, int32_t d);
cudaError_t launch_build_i8_index(const uint8_t* codes, int64_t n, int32_t d, uint8_t* index, cudaStream_t st);
cudaError_t launch_build_f4_index(const uint8_t* codes, int64_t n, int32_t d, uint8_t* index, cudaStream_t st);
// int8 query quantisation (R15): per row scale 127 / max|u| (fp32), round half even
cudaError_t launch_quantize_i8(const void* u, uq_dtype dt, int64_t n, int32_t d, int64_t ld, int8_t* out,
                               int64_t ldo, cudaStream_t st);

}  // namespace uq
