// encode.cu -- nearest {x,d} EVP vertex + 2-plane pack, one warp per row.
//
// P:189-196 (Sec. 2.4): "find the x largest absolute elements ... assign 1 to
// every positive element within this set, and -1 to every negative element ...
// assign 0 to all other elements"; P:379 (Sec. 5.1.2): v+ / v- bit planes.
//
// Exactness: |u_i| is compared as the IEEE abs-bit pattern (an unsigned integer
// whose order equals the order of |u_i| for finite values), so the selection is
// integer-exact and FTZ-independent; signs come from the sign bit of non-zero
// magnitudes (-0.0 and selected zeros encode as 0, R2/R3).  No
// normalisation: scaling does not change the top-x order (R5).
//
// Per row (warp): lane l holds VEC = 16/sizeof(T) consecutive elements of each
// 32*VEC-element chunk.  T* = the x-th largest key is found by bisection on the
// key bits with warp-wide counts (REDUX); keys > T* are selected, keys == T*
// are taken in index order until x are selected (lowest index wins, R1).
// Bits are assembled with warp shuffles into 32-bit plane words and stored.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"

namespace uq {

template <typename T> struct ElemBits;
template <> struct ElemBits<float> {
  static constexpr int kKeyBits = 31;
  __device__ static uint32_t raw(const float* p) { return __float_as_uint(*p); }
  __device__ static uint32_t abs_bits(uint32_t r) { return r & 0x7fffffffu; }
  __device__ static uint32_t sign(uint32_t r) { return r >> 31; }
};
template <> struct ElemBits<__half> {
  static constexpr int kKeyBits = 15;
  __device__ static uint32_t raw(const __half* p) { return (uint32_t)__half_as_ushort(*p); }
  __device__ static uint32_t abs_bits(uint32_t r) { return r & 0x7fffu; }
  __device__ static uint32_t sign(uint32_t r) { return (r >> 15) & 1u; }
};
template <> struct ElemBits<__nv_bfloat16> {
  static constexpr int kKeyBits = 15;
  __device__ static uint32_t raw(const __nv_bfloat16* p) { return (uint32_t)__bfloat16_as_ushort(*p); }
  __device__ static uint32_t abs_bits(uint32_t r) { return r & 0x7fffu; }
  __device__ static uint32_t sign(uint32_t r) { return (r >> 15) & 1u; }
};

constexpr int kEncWarps = 8;

// NCH: chunks of 32*VEC elements per row (compile-time so keys live in registers).
template <typename T, int NCH, bool VECLOAD>
__global__ void __launch_bounds__(kEncWarps * 32)
encode_kernel(const T* __restrict__ u, int64_t n, int32_t d, int64_t ld, int32_t x,
              uint8_t* __restrict__ codes) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int E = NCH * VEC;        // elements per lane
  constexpr int G = 32 / VEC;         // lanes per 32-bit plane word
  using EB = ElemBits<T>;
  const int lane = threadIdx.x & 31;
  const int64_t pw = plane_bytes(d) / 4;      // 32-bit words per plane
  const int64_t cb = code_bytes(d);
  const int64_t warp_global = (int64_t)blockIdx.x * kEncWarps + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kEncWarps;

  for (int64_t row = warp_global; row < n; row += nwarps) {
    const T* src = u + row * ld;
    uint32_t key[E];
    uint32_t sgn = 0, sgn2 = 0;   // sign bits of this lane's elements (E <= 64)
    // ---- load (element e of lane: chunk e/VEC, offset e%VEC) ----
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int i0 = j * 32 * VEC + lane * VEC;
      if (VECLOAD && i0 + VEC <= d) {
        uint4 w = __ldg(reinterpret_cast<const uint4*>(src + i0));
        const T* tv = reinterpret_cast<const T*>(&w);
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          uint32_t r = EB::raw(tv + c);
          key[j * VEC + c] = EB::abs_bits(r);
          const int e = j * VEC + c;
          if (e < 32) sgn |= EB::sign(r) << e; else sgn2 |= EB::sign(r) << (e - 32);
        }
      } else {
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          uint32_t r = 0;
          if (i0 + c < d) r = EB::raw(src + i0 + c);
          key[j * VEC + c] = EB::abs_bits(r);
          const int e = j * VEC + c;
          if (e < 32) sgn |= EB::sign(r) << e; else sgn2 |= EB::sign(r) << (e - 32);
        }
      }
    }
    // ---- T* = x-th largest key (bisection, warp counts) ----
    uint32_t Tk = 0;
    bool exact = false;   // true: exactly x keys are >= Tk (no tie resolution)
#pragma unroll 1
    for (int b = EB::kKeyBits - 1; b >= 0; --b) {
      const uint32_t cand = Tk | (1u << b);
      int c = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) c += (key[e] >= cand) ? 1 : 0;
      const unsigned tot = __reduce_add_sync(kFull, (unsigned)c);
      if (tot >= (unsigned)x) {
        Tk = cand;
        if (tot == (unsigned)x) { exact = true; break; }
      }
    }
    // ---- selection mask (bit e of sel/sel2) ----
    uint32_t sel = 0, sel2 = 0;
    if (exact || Tk == 0) {
      // exact: keys >= Tk are precisely the x largest.  Tk == 0: fewer than x
      // non-zero magnitudes -> every non-zero is selected; selected zeros
      // would encode as 0 anyway (R2), so they need no bit.
      const uint32_t lo = (Tk == 0) ? 1u : Tk;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t s = (key[e] >= lo) ? 1u : 0u;
        if (e < 32) sel |= s << e; else sel2 |= s << (e - 32);
      }
    } else {
      int cgt = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) cgt += (key[e] > Tk) ? 1 : 0;
      const int gt = (int)__reduce_add_sync(kFull, (unsigned)cgt);
      int need = x - gt;            // how many keys == Tk to take, in index order
      // index order: chunk j, then lane, then c
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        int eq = 0;
#pragma unroll
        for (int c = 0; c < VEC; ++c) eq += (key[j * VEC + c] == Tk) ? 1 : 0;
        // exclusive warp prefix of eq
        int incl = eq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += t;
        }
        int rank = incl - eq;
        const int total = __shfl_sync(kFull, incl, 31);
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          const int e = j * VEC + c;
          uint32_t s = 0;
          if (key[e] > Tk) s = 1;
          else if (key[e] == Tk) { s = (rank < need) ? 1u : 0u; ++rank; }
          if (e < 32) sel |= s << e; else sel2 |= s << (e - 32);
        }
        need -= total;
      }
    }
    // ---- pack: pos bit = selected & non-zero & sign 0; neg = ... & sign 1 ----
    uint8_t* dst = codes + row * cb;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      uint32_t pbits = 0, nbits = 0;
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        const int e = j * VEC + c;
        const uint32_t s = (e < 32) ? (sel >> e) & 1u : (sel2 >> (e - 32)) & 1u;
        const uint32_t g = (e < 32) ? (sgn >> e) & 1u : (sgn2 >> (e - 32)) & 1u;
        const uint32_t nz = key[e] != 0 ? 1u : 0u;
        pbits |= (s & nz & (g ^ 1u)) << c;
        nbits |= (s & nz & g) << c;
      }
      // lane l's VEC bits sit at bit VEC*(l % G) of plane word (chunk word l / G)
      uint32_t pwv = pbits << (VEC * (lane % G));
      uint32_t nwv = nbits << (VEC * (lane % G));
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        pwv |= __shfl_xor_sync(kFull, pwv, o);
        nwv |= __shfl_xor_sync(kFull, nwv, o);
      }
      // lanes t < VEC take pos word t, lanes VEC+t take neg word t (from lane t*G)
      const int t = lane % VEC;
      const uint32_t pword = __shfl_sync(kFull, pwv, t * G);
      const uint32_t nword = __shfl_sync(kFull, nwv, t * G);
      const int64_t wi = (int64_t)j * VEC + t;
      if (lane < 2 * VEC && wi < pw) {
        uint32_t* out = reinterpret_cast<uint32_t*>(dst + (lane < VEC ? 0 : pw * 4));
        out[wi] = (lane < VEC) ? pword : nword;
      }
    }
    // plane words beyond the last full chunk (only when pw > NCH*VEC words): zero
    for (int64_t wi = (int64_t)NCH * VEC + lane; wi < pw; wi += 32) {
      reinterpret_cast<uint32_t*>(dst)[wi] = 0u;
      reinterpret_cast<uint32_t*>(dst + pw * 4)[wi] = 0u;
    }
  }
}

template <typename T, int NCH>
static cudaError_t launch_encode_nch(const void* u, int64_t n, int32_t d, int64_t ld, int32_t x,
                                     uint8_t* codes, bool vec, int sms, cudaStream_t st) {
  int64_t blocks = (n + kEncWarps - 1) / kEncWarps;
  int64_t cap = (int64_t)sms * 16;  // grid-stride beyond ~16 CTAs per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (vec)
    encode_kernel<T, NCH, true><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
        (const T*)u, n, d, ld, x, codes);
  else
    encode_kernel<T, NCH, false><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
        (const T*)u, n, d, ld, x, codes);
  note_launch();
  return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_encode_t(const void* u, int64_t n, int32_t d, int64_t ld, int32_t x,
                                   uint8_t* codes, bool vec, int sms, cudaStream_t st) {
  constexpr int VEC = 16 / sizeof(T);
  const int nch = (d + 32 * VEC - 1) / (32 * VEC);
  switch (nch) {
#define UQ_ENC_CASE(N) \
  case N: return launch_encode_nch<T, N>(u, n, d, ld, x, codes, vec, sms, st);
    UQ_ENC_CASE(1) UQ_ENC_CASE(2) UQ_ENC_CASE(3) UQ_ENC_CASE(4)
    UQ_ENC_CASE(5) UQ_ENC_CASE(6) UQ_ENC_CASE(7) UQ_ENC_CASE(8)
#undef UQ_ENC_CASE
    default: break;
  }
  if constexpr (VEC == 4) {
    switch (nch) {
#define UQ_ENC_CASE(N) \
  case N: return launch_encode_nch<T, N>(u, n, d, ld, x, codes, vec, sms, st);
      UQ_ENC_CASE(9) UQ_ENC_CASE(10) UQ_ENC_CASE(11) UQ_ENC_CASE(12)
      UQ_ENC_CASE(13) UQ_ENC_CASE(14) UQ_ENC_CASE(15) UQ_ENC_CASE(16)
#undef UQ_ENC_CASE
      default: break;
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_encode(const void* u, uq_dtype dt, int64_t n, int32_t d, int64_t ld, int32_t x,
                          uint8_t* codes, int sms, cudaStream_t st) {
  const size_t es = (dt == UQ_F32) ? 4 : 2;
  const bool vec = ((uintptr_t)u % 16 == 0) && ((ld * (int64_t)es) % 16 == 0);
  switch (dt) {
    case UQ_F32: return launch_encode_t<float>(u, n, d, ld, x, codes, vec, sms, st);
    case UQ_F16: return launch_encode_t<__half>(u, n, d, ld, x, codes, vec, sms, st);
    case UQ_BF16: return launch_encode_t<__nv_bfloat16>(u, n, d, ld, x, codes, vec, sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace uq
