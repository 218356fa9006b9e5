// rerank.cu -- k@n: exact re-ranking of proxy-space candidates.
//
// P:414-416 (Sec. 5.3, "Hypothesis 2: Search"): "to achieve a kNN search, often
// n > k results are found from the approximate search, which are then
// reordered with respect to the original space, with the best k then
// selected".  For each query the n candidates of the ternary search (ids from
// uq_search with k = n) are scored by cosine similarity on the float vectors
// (on unit vectors l2 order = cosine order) and the best k are kept,
// ordered by (cos desc, id asc).  After this step recall@k equals the paper's
// k@n (the fraction of the k true neighbours among the n candidates).
//
// One CTA per query: the query row is staged in SMEM as fp32, each warp scores
// candidates (16-byte gathers of the candidate row, fp32 FMA dot product and
// squared norm, warp reduction), then a bitonic sort of 64-bit keys
// (order-preserving cos bits << 32 | ~id) in SMEM selects the top k.  fp32
// arithmetic: cosines agree with the fp64 oracle within 1e-5 relative (tests).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"

namespace uq {

constexpr int kRrThreads = 256;
constexpr int kRrWarps = kRrThreads / 32;

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// float -> uint32 whose unsigned order is the float order (finite values)
__device__ __forceinline__ uint32_t ord_f32(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

template <typename T>
__global__ void __launch_bounds__(kRrThreads) rerank_kernel(const T* __restrict__ q, int64_t ldq,
                                                            const T* __restrict__ db, int64_t n, int64_t ld,
                                                            int32_t d, const int64_t* __restrict__ cand,
                                                            int32_t n_cand, int32_t pow2, int32_t k,
                                                            float* __restrict__ out_cos,
                                                            int64_t* __restrict__ out_ids) {
  extern __shared__ uint8_t smem_raw[];
  float* s_q = reinterpret_cast<float*>(smem_raw);                      // [d]
  uint64_t* s_key = reinterpret_cast<uint64_t*>(s_q + ((d + 1) & ~1));   // [pow2]
  __shared__ float s_red[kRrWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t qi = blockIdx.x;
  const T* qr = q + qi * ldq;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += kRrThreads) {
    const float v = to_f32<T>(qr[i]);
    s_q[i] = v;
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
  if (lane == 0) s_red[warp] = ss;
  for (int i = threadIdx.x; i < pow2; i += kRrThreads) s_key[i] = 0ull;   // 0 = empty (sorts last)
  __syncthreads();
  float qn2 = 0.f;
#pragma unroll
  for (int w = 0; w < kRrWarps; ++w) qn2 += s_red[w];

  // score the candidates: one warp per candidate row; rows whose length and
  // stride are multiples of 16 B are read with 16-B loads, all of a lane's
  // loads of a row issued before its arithmetic (one memory round trip per row)
  const int64_t* cq = cand + qi * (int64_t)n_cand;
  constexpr int E = 16 / sizeof(T);   // elements per 16-B vector
  const bool vec = (d % E) == 0 && (ld % E) == 0 && ((uintptr_t)db % 16) == 0;
  for (int c = warp; c < n_cand; c += kRrWarps) {
    const int64_t id = cq[c];
    if (id < 0 || id >= n) continue;   // padding from uq_search (n < k) or foreign ids
    const T* ur = db + id * ld;
    float dot = 0.f, un2 = 0.f;
    if (vec) {
      const uint4* ur4 = reinterpret_cast<const uint4*>(ur);
      const int nv = d / E;
      for (int v0 = lane; v0 < nv; v0 += 32 * 4) {
        uint4 buf[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int v = v0 + 32 * j;
          buf[j] = v < nv ? __ldg(ur4 + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int v = v0 + 32 * j;
          if (v < nv) {
            const T* e = reinterpret_cast<const T*>(&buf[j]);
            const float4* q4 = reinterpret_cast<const float4*>(s_q + v * E);   // 16-B SMEM reads
#pragma unroll
            for (int t4 = 0; t4 < E / 4; ++t4) {
              const float4 qv = q4[t4];
              const float qq[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float u = to_f32<T>(e[4 * t4 + t]);
                dot = fmaf(qq[t], u, dot);
                un2 = fmaf(u, u, un2);
              }
            }
          }
        }
      }
    } else {
      for (int i = lane; i < d; i += 32) {
        const float u = to_f32<T>(ur[i]);
        dot = fmaf(s_q[i], u, dot);
        un2 = fmaf(u, u, un2);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dot += __shfl_xor_sync(kFull, dot, o);
      un2 += __shfl_xor_sync(kFull, un2, o);
    }
    if (lane == 0) {
      const float den = sqrtf(qn2) * sqrtf(un2);
      const float cs = den > 0.f ? dot / den : 0.f;
      s_key[c] = ((uint64_t)ord_f32(cs) << 32) | (uint64_t)(0xffffffffu - (uint32_t)id);
    }
  }
  __syncthreads();
  // bitonic sort, descending
  for (int size = 2; size <= pow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < pow2; i += kRrThreads) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & size) == 0);
          const uint64_t a = s_key[i], b = s_key[j];
          if (desc ? (a < b) : (a > b)) { s_key[i] = b; s_key[j] = a; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < k; i += kRrThreads) {
    const uint64_t key = (i < pow2) ? s_key[i] : 0ull;
    const size_t o = (size_t)qi * k + i;
    if (key == 0ull) {
      out_cos[o] = -INFINITY;
      out_ids[o] = -1;
    } else {
      out_cos[o] = unord_f32((uint32_t)(key >> 32));
      out_ids[o] = (int64_t)(0xffffffffu - (uint32_t)key);
    }
  }
}

template <typename T>
static cudaError_t launch_rerank_t(const void* q, int64_t nq, int64_t ldq, const void* db, int64_t n, int64_t ld,
                                   int32_t d, const int64_t* cand, int32_t n_cand, int32_t k, float* out_cos,
                                   int64_t* out_ids, cudaStream_t st) {
  const int pow2 = 1 << bitlen((unsigned)(n_cand > 1 ? n_cand - 1 : 1));
  const int smem = (int)(((d + 1) & ~1) * sizeof(float) + (size_t)pow2 * 8);
  auto kern = rerank_kernel<T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)nq, kRrThreads, smem, st>>>((const T*)q, ldq, (const T*)db, n, ld, d, cand, n_cand, pow2, k,
                                              out_cos, out_ids);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_rerank(const void* q, uq_dtype dt, int64_t nq, int64_t ldq, const void* db, int64_t n,
                          int64_t ld, int32_t d, const int64_t* cand, int32_t n_cand, int32_t k, float* out_cos,
                          int64_t* out_ids, cudaStream_t st) {
  switch (dt) {
    case UQ_F32: return launch_rerank_t<float>(q, nq, ldq, db, n, ld, d, cand, n_cand, k, out_cos, out_ids, st);
    case UQ_F16: return launch_rerank_t<__half>(q, nq, ldq, db, n, ld, d, cand, n_cand, k, out_cos, out_ids, st);
    case UQ_BF16:
      return launch_rerank_t<__nv_bfloat16>(q, nq, ldq, db, n, ld, d, cand, n_cand, k, out_cos, out_ids, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace uq
