// merge.cu -- final per-query top-k over candidate lists.
//
// Used (a) after a scan, over the per-chunk lists of 64-bit global keys, and
// (b) by uq_merge_topk over G shard results (score, id) after an allgather.
// Exactness: the global top-k under a total order is a subset of the union of
// the per-list top-k's, so selecting the k largest keys of the union is exact.
//
// One CTA per query: (1) T = k-th largest valid key by an MSB-first radix
// select (8-bit digits, shared-memory histogram per digit, starting at the
// highest bit in which the candidates differ, early exit once a whole digit
// bucket is taken); (2) gather the <= k keys >= T into shared memory; (3) rank
// each selected key by counting the larger ones (keys are unique) and write
// (score, id) at its rank, padding with (INT32_MIN, -1).
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace uq {

constexpr int kMergeThreads = 256;
constexpr int kMergeWarps = kMergeThreads / 32;
constexpr int kMergeMaxLists = 2048;   // counted lists gathered compactly up to this many

struct MergeParams {
  // source (a): keys [lists][nq][k]; source (b): scores/ids [lists][nq][k]
  const uint64_t* keys;
  const int32_t* scores;
  const int64_t* ids;
  int64_t lists;
  int64_t nq;
  int32_t kin;      // entries per list per query
  int32_t k;        // output k
  int64_t id_base;  // added to every output row (source (a): the shard's first row; (b): 0, or the
                    // shard's first row at level 2 of a two-level merge, whose level 1 keeps local rows)
  int32_t* out_s;
  int64_t* out_id;
  int32_t stage_cap;  // candidates staged in shared memory if C <= stage_cap
  const int32_t* counts;  // source (a), optional: valid entries per list [lists][nq] (rest unread, empty)
  const int32_t* only;    // optional: merge only queries q with only[q] != 0 (seed fallback pass)
  const int32_t* any;     // optional: the whole launch is a no-op unless *any != 0
  // source (b) through per-list base pointers (peer-mapped buffers of other
  // GPUs: the merge reads every rank's [nq][k] lists directly over NVLink)
  const int32_t* const* score_ptrs;
  const int64_t* const* id_ptrs;
  // two-level merge (few queries, many lists): CTA (q, y) merges lists
  // [y*lpg, (y+1)*lpg) of source (a) into slot y of out_s / out_id [G][nq][k]
  int64_t lpg;
};

template <bool FROM_SI>
__device__ __forceinline__ uint64_t cand_key(const MergeParams& p, int64_t q, int64_t i) {
  const int64_t l = i / p.kin, e = i % p.kin;
  const size_t off = ((size_t)l * p.nq + q) * p.kin + e;
  if (FROM_SI) {
    if (p.score_ptrs != nullptr) {
      const size_t o = (size_t)q * p.kin + e;
      return global_key(p.score_ptrs[l][o], p.id_ptrs[l][o]);
    }
    return global_key(p.scores[off], p.ids[off]);
  }
  if (p.counts != nullptr && e >= p.counts[(size_t)l * p.nq + q]) return 0ull;
  return p.keys[off];
}

// (key >> r) with r in [0, 64]
__device__ __forceinline__ uint64_t shr64(uint64_t v, int r) { return r >= 64 ? 0ull : (v >> r); }

template <bool FROM_SI>
__global__ void __launch_bounds__(kMergeThreads) merge_kernel(MergeParams p) {
  extern __shared__ uint64_t smem_u64[];
  __shared__ unsigned s_hist[256];
  __shared__ unsigned long long s_and[kMergeWarps], s_or[kMergeWarps];
  __shared__ unsigned s_cnt[kMergeWarps];
  __shared__ int s_nsel;
  __shared__ int s_b, s_above, s_inb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = blockIdx.x;
  if ((p.any != nullptr && *p.any == 0) || (p.only != nullptr && p.only[q] == 0)) return;
  if (!FROM_SI && p.lpg > 0) {
    const int64_t l0 = (int64_t)blockIdx.y * p.lpg;
    p.lists = min(p.lpg, p.lists - l0);
    p.keys += l0 * p.nq * p.kin;
    if (p.counts != nullptr) p.counts += l0 * p.nq;
    p.out_s += (size_t)blockIdx.y * p.nq * p.k;
    p.out_id += (size_t)blockIdx.y * p.nq * p.k;
  }
  __shared__ int s_off[kMergeMaxLists + 1];
  int64_t C = p.lists * p.kin;
  const int P = 1 << bitlen((unsigned)(p.k - 1 > 0 ? p.k - 1 : 1));  // pow2 >= k (>= 2)
  uint64_t* s_sel = smem_u64;          // [P]
  uint64_t* s_cand = smem_u64 + P;     // [stage_cap] (if staged)
  bool staged = C <= p.stage_cap;
  bool compact = false;
  // counted lists: gather only the valid entries, contiguously, into SMEM
  if (!FROM_SI && p.counts != nullptr && p.lists <= kMergeMaxLists) {
    if (warp == 0) {
      int base = 0;
      for (int64_t l0 = 0; l0 < p.lists; l0 += 32) {
        const int64_t l = l0 + lane;
        const int c = (l < p.lists) ? min(p.counts[(size_t)l * p.nq + q], p.kin) : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += t;
        }
        if (l < p.lists) s_off[l] = base + incl - c;
        base += __shfl_sync(kFull, incl, 31);
      }
      if (lane == 0) s_off[p.lists] = base;
    }
    __syncthreads();
    const int total = s_off[p.lists];
    if (total <= p.stage_cap) {
      for (int64_t l = warp; l < p.lists; l += kMergeWarps) {
        const int o = s_off[l], c = s_off[l + 1] - o;
        const uint64_t* src = p.keys + ((size_t)l * p.nq + q) * p.kin;
        UQ_ASSERT(o + c <= p.stage_cap);
        for (int e = lane; e < c; e += 32) s_cand[o + e] = src[e];
      }
      C = total;
      staged = true;
      compact = true;
      __syncthreads();
    }
  }
  // stage + common bits of the valid (non-zero) keys
  uint64_t a_and = ~0ull, a_or = 0ull;
  unsigned nv = 0;
  for (int64_t i = threadIdx.x; i < C; i += kMergeThreads) {
    const uint64_t key = compact ? s_cand[i] : cand_key<FROM_SI>(p, q, i);
    if (staged && !compact) s_cand[i] = key;
    if (key != 0ull) { a_and &= key; a_or |= key; ++nv; }
  }
  a_and = __reduce_and_sync(kFull, (unsigned)a_and) | ((uint64_t)__reduce_and_sync(kFull, (unsigned)(a_and >> 32)) << 32);
  a_or = __reduce_or_sync(kFull, (unsigned)a_or) | ((uint64_t)__reduce_or_sync(kFull, (unsigned)(a_or >> 32)) << 32);
  nv = __reduce_add_sync(kFull, nv);
  if (lane == 0) { s_and[warp] = a_and; s_or[warp] = a_or; s_cnt[warp] = nv; }
  if (threadIdx.x == 0) s_nsel = 0;
  __syncthreads();
  uint64_t all_and = ~0ull, all_or = 0ull;
  unsigned nvalid = 0;
#pragma unroll
  for (int w = 0; w < kMergeWarps; ++w) { all_and &= s_and[w]; all_or |= s_or[w]; nvalid += s_cnt[w]; }
  auto get = [&](int64_t i) -> uint64_t { return staged ? s_cand[i] : cand_key<FROM_SI>(p, q, i); };

  // (1) T = k-th largest valid key
  uint64_t T = 1ull;  // fewer than k valid candidates: take every valid one
  if (nvalid > (unsigned)p.k) {
    const uint64_t diff = all_and ^ all_or;      // != 0: keys are unique
    int r = 64 - __clzll((long long)diff);       // bits [r, 64) are common to every valid key
    uint64_t prefix = (r >= 64) ? 0ull : (all_and >> r) << r;
    int krem = p.k;
    while (r > 0) {
      const int w = r < 8 ? r : 8;
      const int sh = r - w;
      const unsigned dmask = (1u << w) - 1u;
      s_hist[threadIdx.x] = 0u;
      __syncthreads();
      const uint64_t hi = shr64(prefix, r);
      // warp-aggregated: candidates concentrate in a few digits (seeded scans
      // keep only scores near D_k), so lanes with equal digits add once
      // (MATCH + POPC) instead of serialising on one shared-memory word
      for (int64_t b = (int64_t)warp * 32; b < C; b += kMergeThreads) {
        const int64_t i = b + lane;
        const uint64_t key = i < C ? get(i) : 0ull;
        const bool in = key != 0ull && shr64(key, r) == hi;
        const unsigned bin = in ? ((unsigned)(key >> sh) & dmask) : 0xffffffffu;
        const unsigned peers = __match_any_sync(kFull, bin);
        if (in && (peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&s_hist[bin], (unsigned)__popc(peers));
      }
      __syncthreads();
      if (warp == 0) {
        // lane l owns bins [248 - 8l, 255 - 8l] (descending digit order)
        unsigned c[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { c[j] = s_hist[255 - 8 * lane - j]; sum += c[j]; }
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned t = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += t;
        }
        unsigned above = incl - sum;  // keys in bins of higher-numbered lanes' ranges (larger digits)
        const bool mine = above < (unsigned)krem && incl >= (unsigned)krem;
        if (mine) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (above < (unsigned)krem && above + c[j] >= (unsigned)krem) {
              s_b = 255 - 8 * lane - j;
              s_above = (int)above;
              s_inb = (int)c[j];
            }
            above += c[j];
          }
        }
      }
      __syncthreads();
      const int b = s_b;
      krem -= s_above;
      prefix |= (uint64_t)b << sh;
      r = sh;
      if (krem == s_inb) break;  // the whole bucket is taken: T = its smallest possible key
      __syncthreads();           // s_hist / s_b reused by the next digit
    }
    T = prefix;
  }
  // (2) gather the keys >= T (exactly min(k, nvalid): keys are unique)
  for (int64_t b = (int64_t)warp * 32; b < C; b += kMergeThreads) {   // one atomic per warp
    const int64_t i = b + lane;
    const uint64_t key = i < C ? get(i) : 0ull;
    const bool take = key != 0ull && key >= T;
    const unsigned m = __ballot_sync(kFull, take);
    int base = 0;
    if (lane == 0 && m != 0u) base = atomicAdd(&s_nsel, __popc(m));
    base = __shfl_sync(kFull, base, 0);
    const int pos = base + __popc(m & ((1u << lane) - 1u));
    if (take && pos < P) s_sel[pos] = key;
  }
  __syncthreads();
  const int nsel = s_nsel < p.k ? s_nsel : p.k;
  // (3) rank by counting (distinct keys) and write best first
  for (int i = threadIdx.x; i < nsel; i += kMergeThreads) {
    const uint64_t key = s_sel[i];
    int rank = 0;
    for (int j = 0; j < nsel; ++j) rank += (s_sel[j] > key) ? 1 : 0;
    const size_t o = (size_t)q * p.k + rank;
    p.out_s[o] = key_score(key);
    p.out_id[o] = p.id_base + key_row(key);
  }
  for (int i = nsel + threadIdx.x; i < p.k; i += kMergeThreads) {
    const size_t o = (size_t)q * p.k + i;
    p.out_s[o] = INT32_MIN;
    p.out_id[o] = -1;
  }
}

static int merge_smem(int32_t k, int64_t C, int32_t* stage_cap, int64_t bytes) {
  const int P = 1 << bitlen((unsigned)(k - 1 > 0 ? k - 1 : 1));
  const int64_t budget = bytes / 8 - P;  // keys staged beside s_sel
  *stage_cap = (int32_t)(C <= budget ? C : budget);   // lists larger than this are read from global
  return (int)((P + *stage_cap) * 8);
}

// smem_bytes: staging budget (48 KB: 4 CTAs per SM; a few-query merge with one
// CTA per query takes most of an SM's shared memory instead)
static cudaError_t launch_merge_common(MergeParams p, bool from_si, cudaStream_t st, unsigned groups = 1,
                                       int64_t smem_bytes = 48 * 1024) {
  if (p.nq <= 0) return cudaSuccess;
  const int64_t lists_per_cta = (!from_si && p.lpg > 0) ? p.lpg : p.lists;
  const int smem = merge_smem(p.k, lists_per_cta * p.kin, &p.stage_cap, smem_bytes);
  const dim3 grid((unsigned)p.nq, groups);
  if (from_si) {
    cudaError_t e = cudaFuncSetAttribute(merge_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    merge_kernel<true><<<grid, kMergeThreads, smem, st>>>(p);
  } else {
    cudaError_t e = cudaFuncSetAttribute(merge_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    merge_kernel<false><<<grid, kMergeThreads, smem, st>>>(p);
  }
  note_launch();
  return cudaGetLastError();
}

static int merge_sms() {
  static const int sms = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    return v;
  }();
  return sms;
}

// Scratch for the two-level merge: G x nq x k (score, id) pairs, G*nq <= 2 SMs.
size_t merge_scratch_bytes(int64_t nq, int32_t k) {
  const int sms = merge_sms();
  if (nq * 2 >= sms) return 0;
  return (size_t)2 * sms * k * 12 + 1024;
}

cudaError_t launch_merge_keys(const uint64_t* keys, int64_t lists, int64_t nq, int32_t kin, int32_t k,
                              int64_t id_base, int32_t* out_s, int64_t* out_id, cudaStream_t st,
                              const int32_t* counts, const int32_t* only, const int32_t* any, void* scratch,
                              size_t scratch_bytes) {
  MergeParams p{keys, nullptr, nullptr, lists, nq, kin, k, id_base, out_s, out_id, 0, counts, only, any, nullptr,
                nullptr, 0};
  // Few queries over many candidate lists: one CTA per query would select
  // among lists * kin keys alone (c2, Q = 1, k = 100, popcount engine: 44k
  // keys, ~0.3 ms).  Split the lists over G ~ sqrt(lists) CTAs per query
  // (G * nq <= 2 SMs), each keeping its k best, then merge the G partials.
  const int sms = merge_sms();
  if (scratch != nullptr && nq * 2 < sms && lists >= 8 && lists * kin > 4096) {
    // G ~ sqrt(lists): both levels select among ~sqrt(lists) * kin keys
    int64_t g = 1;
    while (g * g < lists) ++g;
    g = std::min<int64_t>(g, (2 * sms + nq - 1) / nq);
    const int64_t lpg = (lists + g - 1) / g;
    g = (lists + lpg - 1) / lpg;
    if ((size_t)g * nq * k * 12 + 256 <= scratch_bytes && g > 1) {
      int32_t* ss = reinterpret_cast<int32_t*>(scratch);
      int64_t* si = reinterpret_cast<int64_t*>(
          (reinterpret_cast<uintptr_t>(ss + (size_t)g * nq * k) + 255) & ~(uintptr_t)255);
      MergeParams p1 = p;
      p1.out_s = ss;
      p1.out_id = si;
      p1.lpg = lpg;
      p1.id_base = 0;   // level 1 keeps local rows (< 2^32 - 1): global_key() repacks them at level 2
      cudaError_t e = launch_merge_common(p1, false, st, (unsigned)g);
      if (e != cudaSuccess) return e;
      MergeParams p2{nullptr, ss, si, g, nq, k, k, id_base, out_s, out_id, 0, nullptr, only, any, nullptr, nullptr, 0};
      return launch_merge_common(p2, true, st);
    }
  }
  return launch_merge_common(p, false, st);
}

cudaError_t launch_merge_si(const int32_t* scores, const int64_t* ids, int64_t lists, int64_t nq,
                            int32_t k, int32_t* out_s, int64_t* out_id, cudaStream_t st) {
  MergeParams p{nullptr, scores, ids, lists, nq, k, k, 0, out_s, out_id, 0, nullptr, nullptr, nullptr, nullptr,
                nullptr, 0};
  return launch_merge_common(p, true, st);
}

cudaError_t launch_merge_ptrs(const int32_t* const* score_ptrs, const int64_t* const* id_ptrs, int64_t lists,
                              int64_t nq, int32_t k, int32_t* out_s, int64_t* out_id, cudaStream_t st) {
  MergeParams p{nullptr, nullptr, nullptr, lists, nq, k, k, 0, out_s, out_id, 0, nullptr, nullptr, nullptr,
                score_ptrs, id_ptrs, 0};
  return launch_merge_common(p, true, st);
}

}  // namespace uq
