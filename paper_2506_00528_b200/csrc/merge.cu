// merge.cu -- final per-query top-k over candidate lists.
//
// Used (a) after a scan, over the per-chunk lists of 64-bit global keys, and
// (b) by uq_merge_topk over G shard results (score, id) after an allgather.
// Exactness: the global top-k under a total order is a subset of the union of
// the per-list top-k's, so selecting the k largest keys of the union is exact.
//
// One CTA per query: (1) T = k-th largest key by bisection over the 64 key
// bits with block-wide counts; (2) gather the <= k keys >= T into shared
// memory; (3) bitonic sort descending; (4) write (score, id) best first,
// padding with (INT32_MIN, -1).
#include "common.cuh"
#include "internal.h"

namespace uq {

constexpr int kMergeThreads = 256;

struct MergeParams {
  // source (a): keys [lists][nq][k]; source (b): scores/ids [lists][nq][k]
  const uint64_t* keys;
  const int32_t* scores;
  const int64_t* ids;
  int64_t lists;
  int64_t nq;
  int32_t kin;      // entries per list per query
  int32_t k;        // output k
  int64_t id_base;  // added to rows of source (a)
  int32_t* out_s;
  int64_t* out_id;
  int32_t stage_cap;  // candidates staged in shared memory if C <= stage_cap
};

template <bool FROM_SI>
__device__ __forceinline__ uint64_t cand_key(const MergeParams& p, int64_t q, int64_t i) {
  const int64_t l = i / p.kin, e = i % p.kin;
  const size_t off = ((size_t)l * p.nq + q) * p.kin + e;
  if (FROM_SI) return global_key(p.scores[off], p.ids[off]);
  return p.keys[off];
}

__device__ __forceinline__ unsigned block_sum(unsigned v, unsigned* s_acc) {
  v = __reduce_add_sync(kFull, v);
  if ((threadIdx.x & 31) == 0) atomicAdd(s_acc, v);
  __syncthreads();
  const unsigned tot = *s_acc;
  __syncthreads();
  if (threadIdx.x == 0) *s_acc = 0;
  __syncthreads();
  return tot;
}

template <bool FROM_SI>
__global__ void __launch_bounds__(kMergeThreads) merge_kernel(MergeParams p) {
  extern __shared__ uint64_t smem_u64[];
  __shared__ unsigned s_acc;
  __shared__ int s_nsel;
  const int64_t q = blockIdx.x;
  const int64_t C = p.lists * p.kin;
  const int P = 1 << bitlen((unsigned)(p.k - 1 > 0 ? p.k - 1 : 1));  // pow2 >= k (>= 2)
  uint64_t* s_sel = smem_u64;          // [P]
  uint64_t* s_cand = smem_u64 + P;     // [stage_cap] (if staged)
  const bool staged = C <= p.stage_cap;
  if (threadIdx.x == 0) { s_acc = 0; s_nsel = 0; }
  if (staged)
    for (int64_t i = threadIdx.x; i < C; i += kMergeThreads) s_cand[i] = cand_key<FROM_SI>(p, q, i);
  __syncthreads();
  auto get = [&](int64_t i) -> uint64_t { return staged ? s_cand[i] : cand_key<FROM_SI>(p, q, i); };

  // (1) T = k-th largest key (max T with #{key >= T} >= k)
  uint64_t T = 0;
  for (int b = 63; b >= 0; --b) {
    const uint64_t cand = T | (1ull << b);
    unsigned c = 0;
    for (int64_t i = threadIdx.x; i < C; i += kMergeThreads) c += get(i) >= cand ? 1u : 0u;
    const unsigned tot = block_sum(c, &s_acc);
    if (tot >= (unsigned)p.k) {
      T = cand;
      if (tot == (unsigned)p.k) break;
    }
  }
  if (T == 0) T = 1;  // fewer than k valid candidates: take every valid one
  // (2) gather
  for (int i = threadIdx.x; i < P; i += kMergeThreads) s_sel[i] = 0ull;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < C; i += kMergeThreads) {
    const uint64_t key = get(i);
    if (key >= T) {
      const int pos = atomicAdd(&s_nsel, 1);
      if (pos < P) s_sel[pos] = key;
    }
  }
  __syncthreads();
  // (3) bitonic sort, descending
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += kMergeThreads) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & size) == 0);
          const uint64_t a = s_sel[i], b = s_sel[j];
          if (desc ? (a < b) : (a > b)) { s_sel[i] = b; s_sel[j] = a; }
        }
      }
      __syncthreads();
    }
  }
  // (4) write
  for (int i = threadIdx.x; i < p.k; i += kMergeThreads) {
    const uint64_t key = s_sel[i];
    const size_t o = (size_t)q * p.k + i;
    if (key == 0) {
      p.out_s[o] = INT32_MIN;
      p.out_id[o] = -1;
    } else {
      p.out_s[o] = key_score(key);
      p.out_id[o] = (FROM_SI ? 0 : p.id_base) + key_row(key);
    }
  }
}

static int merge_smem(int32_t k, int64_t C, int32_t* stage_cap) {
  const int P = 1 << bitlen((unsigned)(k - 1 > 0 ? k - 1 : 1));
  const int64_t budget = 96 * 1024 / 8 - P;  // keys that fit beside s_sel
  *stage_cap = (int32_t)(C <= budget ? C : 0);
  return (int)((P + *stage_cap) * 8);
}

static cudaError_t launch_merge_common(MergeParams p, bool from_si, cudaStream_t st) {
  if (p.nq <= 0) return cudaSuccess;
  const int smem = merge_smem(p.k, p.lists * p.kin, &p.stage_cap);
  if (from_si) {
    cudaError_t e = cudaFuncSetAttribute(merge_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    merge_kernel<true><<<(unsigned)p.nq, kMergeThreads, smem, st>>>(p);
  } else {
    cudaError_t e = cudaFuncSetAttribute(merge_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    merge_kernel<false><<<(unsigned)p.nq, kMergeThreads, smem, st>>>(p);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_merge_keys(const uint64_t* keys, int64_t lists, int64_t nq, int32_t kin, int32_t k,
                              int64_t id_base, int32_t* out_s, int64_t* out_id, cudaStream_t st) {
  MergeParams p{keys, nullptr, nullptr, lists, nq, kin, k, id_base, out_s, out_id, 0};
  return launch_merge_common(p, false, st);
}

cudaError_t launch_merge_si(const int32_t* scores, const int64_t* ids, int64_t lists, int64_t nq,
                            int32_t k, int32_t* out_s, int64_t* out_id, cudaStream_t st) {
  MergeParams p{nullptr, scores, ids, lists, nq, k, k, 0, out_s, out_id, 0};
  return launch_merge_common(p, true, st);
}

}  // namespace uq
