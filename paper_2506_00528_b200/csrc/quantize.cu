// quantize.cu -- int8 query quantisation for single-operand search.
//
// P:507-509 (Sec. 6.1, "Single-operand translation"): the ternary database
// can be compared with queries kept "in the original floating-point space, or
// the same space quantised to 8-bit integers", through the masked addition of
// P:379.  The paper names no quantisation scheme; reading R15:
// per vector, scale = 127 / max_i |u_i| and q_i = round-half-even(u_i * scale),
// both in IEEE fp32 (explicit __fdiv_rn / __fmul_rn, so the result does not
// depend on compiler contraction), clamped to [-127, 127]; an all-zero vector
// maps to zeros.  One warp per row: a max-reduction over |u| (exact), then one
// pass writing the codes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"

namespace uq {

template <typename T> __device__ __forceinline__ float qz_f32(T v);
template <> __device__ __forceinline__ float qz_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float qz_f32<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float qz_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__global__ void __launch_bounds__(256) quantize_i8_kernel(const T* __restrict__ u, int64_t n, int32_t d, int64_t ld,
                                                          int8_t* __restrict__ out, int64_t ldo) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const T* ur = u + row * ld;
  float m = 0.f;
  for (int i = lane; i < d; i += 32) m = fmaxf(m, fabsf(qz_f32<T>(ur[i])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  const float scale = m > 0.f ? __fdiv_rn(127.0f, m) : 0.f;
  int8_t* orow = out + row * ldo;
  for (int i = lane; i < d; i += 32) {
    float q = rintf(__fmul_rn(qz_f32<T>(ur[i]), scale));
    q = fminf(fmaxf(q, -127.f), 127.f);
    orow[i] = (int8_t)(int)q;
  }
}

template <typename T>
static cudaError_t launch_q(const void* u, int64_t n, int32_t d, int64_t ld, int8_t* out, int64_t ldo,
                            cudaStream_t st) {
  quantize_i8_kernel<T><<<(unsigned)((n + 7) / 8), 256, 0, st>>>((const T*)u, n, d, ld, out, ldo);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_quantize_i8(const void* u, uq_dtype dt, int64_t n, int32_t d, int64_t ld, int8_t* out,
                               int64_t ldo, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  switch (dt) {
    case UQ_F32: return launch_q<float>(u, n, d, ld, out, ldo, st);
    case UQ_F16: return launch_q<__half>(u, n, d, ld, out, ldo, st);
    case UQ_BF16: return launch_q<__nv_bfloat16>(u, n, d, ld, out, ldo, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace uq
