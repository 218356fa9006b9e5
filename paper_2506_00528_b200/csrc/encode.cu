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
// 32*VEC-element chunk.  T* = the x-th largest key is found by a bracketed
// search on count(key >= c) (warp totals by REDUX):
//   1. probes: a float estimate t of |u|_(x) (row RMS x a per-warp ratio that
//      starts at the Gaussian quantile z = Phi^-1(1 - x/2d) and then tracks the
//      previous row's T*/RMS), counted at t(1 -/+ delta) in one fused pass;
//   2. interpolation passes inside the bracket [lo, hi) (value-space secant,
//      every third pass a key-space bisection, so the key range at least halves
//      every three passes and the search ends in <= 3*31 passes whatever the
//      data), until count(>= c) == x or hi == lo + 1.
// The probes only steer the search: T* is exact for any input.  fp16 rows count
// two keys per instruction (HSET2 on |u| half pairs, exact small-integer HADD2).
// Keys > T* are selected, keys == T* are taken in index order until x are
// selected (lowest index wins, R1).  Bits are assembled with warp shuffles into
// 32-bit plane words and stored.  The next row's loads are issued before the
// current row is packed, and rows further ahead are prefetched into L2.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace uq {

template <typename T> struct ElemBits;
template <> struct ElemBits<float> {
  static constexpr uint32_t kKeyEnd = 0x80000000u;  // keys are < kKeyEnd
  __device__ static uint32_t abs_bits(uint32_t r) { return r & 0x7fffffffu; }
  __device__ static uint32_t sign(uint32_t r) { return r >> 31; }
  __device__ static float key2f(uint32_t k) { return __uint_as_float(k); }
  __device__ static uint32_t f2key(float v) { return __float_as_uint(v) & 0x7fffffffu; }
};
template <> struct ElemBits<__half> {
  static constexpr uint32_t kKeyEnd = 0x8000u;
  __device__ static uint32_t abs_bits(uint32_t r) { return r & 0x7fffu; }
  __device__ static uint32_t sign(uint32_t r) { return (r >> 15) & 1u; }
  __device__ static float key2f(uint32_t k) { return __half2float(__ushort_as_half((unsigned short)k)); }
  __device__ static uint32_t f2key(float v) { return (uint32_t)__half_as_ushort(__float2half_rz(v)) & 0x7fffu; }
};
template <> struct ElemBits<__nv_bfloat16> {
  static constexpr uint32_t kKeyEnd = 0x8000u;
  __device__ static uint32_t abs_bits(uint32_t r) { return r & 0x7fffu; }
  __device__ static uint32_t sign(uint32_t r) { return (r >> 15) & 1u; }
  __device__ static float key2f(uint32_t k) { return __bfloat162float(__ushort_as_bfloat16((unsigned short)k)); }
  __device__ static uint32_t f2key(float v) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rz(v)) & 0x7fffu;
  }
};

constexpr int kEncWarps = 8;
constexpr float kProbeDelta = 0.08f;
constexpr int kMaxCodeBytes = 2 * 16 * ((UQ_MAX_D + 127) / 128);

// element c of a raw 16-byte word as its IEEE bit pattern
template <typename T>
__device__ __forceinline__ uint32_t raw_elem(const uint4& w, int c) {
  const uint32_t wd = (c * (int)sizeof(T) / 4 == 0) ? w.x : (c * (int)sizeof(T) / 4 == 1) ? w.y
                      : (c * (int)sizeof(T) / 4 == 2) ? w.z : w.w;
  if (sizeof(T) == 4) return wd;
  return (c & 1) ? (wd >> 16) : (wd & 0xffffu);
}

// one 32*VEC-element chunk of a row into a raw 16-byte word per lane
template <typename T, bool VECLOAD>
__device__ __forceinline__ uint4 load_chunk(const T* src, int i0, int d) {
  constexpr int VEC = 16 / sizeof(T);
  if (VECLOAD && i0 + VEC <= d) return __ldg(reinterpret_cast<const uint4*>(src + i0));
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  const unsigned short* s16 = reinterpret_cast<const unsigned short*>(src);
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
#pragma unroll
  for (int c = 0; c < VEC; ++c) {
    if (i0 + c < d) {
      if (sizeof(T) == 4) w[c] = __ldg(s32 + i0 + c);
      else w[c / 2] |= (uint32_t)__ldg(s16 + i0 + c) << (16 * (c & 1));
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// count of keys >= c in this lane (generic).  Keys and c are < 2^31, so
// (k - c) >> 31 is 1 exactly when k < c: two instructions per key (IADD +
// LEA.HI) into four independent accumulators (no serial select chain).
// acc + ((k - c) >> 31), kept arithmetic (IADD + LEA.HI) through inline PTX
__device__ __forceinline__ unsigned add_lt(unsigned acc, uint32_t k, uint32_t c) {
  unsigned r;
  asm("{\n\t.reg .u32 t;\n\tsub.u32 t, %1, %2;\n\tshr.u32 t, t, 31;\n\tadd.u32 %0, %3, t;\n\t}"
      : "=r"(r) : "r"(k), "r"(c), "r"(acc));
  return r;
}

template <typename T, int E, int NCH>
struct Counter {
  static constexpr int VEC = 16 / sizeof(T);
  __device__ static unsigned ge(const uint4 (&raw)[NCH], uint32_t c) {
    unsigned a[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int e = 0; e < E; ++e) a[e & 3] = add_lt(a[e & 3], raw_elem<T>(raw[e / VEC], e % VEC), c);
    return (unsigned)E - (a[0] + a[1] + a[2] + a[3]);
  }
  __device__ static void ge2(const uint4 (&raw)[NCH], uint32_t c1, uint32_t c2, unsigned& n1, unsigned& n2) {
    unsigned a[2] = {0u, 0u}, b[2] = {0u, 0u};
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t k = raw_elem<T>(raw[e / VEC], e % VEC);
      a[e & 1] = add_lt(a[e & 1], k, c1);
      b[e & 1] = add_lt(b[e & 1], k, c2);
    }
    n1 = (unsigned)E - (a[0] + a[1]);
    n2 = (unsigned)E - (b[0] + b[1]);
  }
};
// fp16: |u| half pairs straight from the raw words (HSET2 gives 1.0 / 0.0 per
// half; the per-half sums stay <= 2*NCH*2, exact in fp16)
template <int E, int NCH>
struct Counter<__half, E, NCH> {
  __device__ static __half2 absw(uint32_t w) {  // w: sign-cleared half pair
    return *reinterpret_cast<const __half2*>(&w);
  }
  __device__ static unsigned total(__half2 acc) {
    return (unsigned)(__low2float(acc) + __high2float(acc));
  }
  __device__ static unsigned ge(const uint4 (&raw)[NCH], uint32_t c) {
    const __half h = __ushort_as_half((unsigned short)c);
    const __half2 cc = __halves2half2(h, h);
    __half2 acc = __float2half2_rn(0.f);
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      acc = __hadd2(acc, __hge2(absw(raw[j].x), cc));
      acc = __hadd2(acc, __hge2(absw(raw[j].y), cc));
      acc = __hadd2(acc, __hge2(absw(raw[j].z), cc));
      acc = __hadd2(acc, __hge2(absw(raw[j].w), cc));
    }
    return total(acc);
  }
  __device__ static void ge2(const uint4 (&raw)[NCH], uint32_t c1, uint32_t c2, unsigned& n1, unsigned& n2) {
    const __half h1 = __ushort_as_half((unsigned short)c1), h2 = __ushort_as_half((unsigned short)c2);
    const __half2 cc1 = __halves2half2(h1, h1), cc2 = __halves2half2(h2, h2);
    __half2 a1 = __float2half2_rn(0.f), a2 = a1;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __half2 a = absw(w[i]);
        a1 = __hadd2(a1, __hge2(a, cc1));
        a2 = __hadd2(a2, __hge2(a, cc2));
      }
    }
    n1 = total(a1);
    n2 = total(a2);
  }
};

#define KEY(e) raw_elem<T>(raw[(e) / VEC], (e) % VEC)

// Four words of 16-bit lanes with flags in bits 15 and 31 -> 8 bits, bit
// 2i + h = flag of half h of word i (PRMT gathers the flag bytes, one multiply
// moves bits 7/15/23/31 to 28..31 without carries).
__device__ __forceinline__ uint32_t flags16_to_bits8(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
  const uint32_t t01 = __byte_perm(w0, w1, 0x7531);
  const uint32_t t23 = __byte_perm(w2, w3, 0x7531);
  const uint32_t n01 = ((t01 & 0x80808080u) * 0x00204081u) >> 28;
  const uint32_t n23 = ((t23 & 0x80808080u) * 0x00204081u) >> 28;
  return n01 | (n23 << 4);
}
__device__ __forceinline__ __half2 as_h2(uint32_t w) { return *reinterpret_cast<const __half2*>(&w); }

// NCH: chunks of 32*VEC elements per row (compile-time so keys live in registers).
template <typename T, int NCH, bool VECLOAD>
__global__ void __launch_bounds__(kEncWarps * 32)
encode_kernel(const T* __restrict__ u, int64_t n, int32_t d, int64_t ld, int32_t x, float z0,
              uint8_t* __restrict__ codes) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int E = NCH * VEC;        // elements per lane
  constexpr int NS = (sizeof(T) == 4) ? NCH : (NCH < 2 ? NCH : 2);  // chunks used for the RMS
  using EB = ElemBits<T>;
  using CNT = Counter<T, E, NCH>;
  const int lane = threadIdx.x & 31;
  const int64_t pw = plane_bytes(d) / 4;      // 32-bit words per plane
  const int64_t cb = code_bytes(d);
  const int64_t warp_global = (int64_t)blockIdx.x * kEncWarps + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kEncWarps;
  const float inv_ns = 1.0f / (float)min(d, 32 * VEC * NS);
  __shared__ __align__(16) uint8_t s_codes[kEncWarps][kMaxCodeBytes];
  uint8_t* const s_code = s_codes[threadIdx.x >> 5];
  float ratio = z0;   // T* / RMS, learned from the previous row of this warp

  uint4 raw[NCH];
  if (warp_global < n) {
#pragma unroll
    for (int j = 0; j < NCH; ++j) raw[j] = load_chunk<T, VECLOAD>(u + warp_global * ld, j * 32 * VEC + lane * VEC, d);
  }
  // L2 prefetch (one bulk-prefetch instruction per row, no registers) of the
  // row this warp processes two iterations ahead
  const uint32_t pf_bytes = VECLOAD ? ((uint32_t)(d * (int)sizeof(T)) & ~15u) : 0u;
  auto prefetch = [&](int64_t r) {
    if (VECLOAD && lane == 0 && r < n && pf_bytes > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + r * ld), "r"(pf_bytes) : "memory");
  };
  prefetch(warp_global + nwarps);
  for (int64_t row = warp_global; row < n; row += nwarps) {
    const int64_t nrow = row + nwarps;
    prefetch(row + 2 * nwarps);
    // ---- keys, sign bits, RMS estimate (element e of lane: chunk e/VEC, offset e%VEC) ----
    uint64_t sgnm = 0;   // sign bits of this lane's elements (bit e; E <= 64)
    float ss = 0.f;
    if constexpr (std::is_same<T, __half>::value) {
      // sign flags are bits 15/31 of each word; RMS from HFMA2 on pre-scaled
      // halves (an estimate: overflow only degrades the probes)
      __half2 acc = __float2half2_rn(0.f);
      const __half2 sc = __float2half2_rn(0.015625f);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        sgnm |= (uint64_t)flags16_to_bits8(raw[j].x, raw[j].y, raw[j].z, raw[j].w) << (8 * j);
        if (j < NS) {
          const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const __half2 h = __hmul2(as_h2(w[i]), sc);
            acc = __hfma2(h, h, acc);
          }
        }
        raw[j].x &= 0x7fff7fffu; raw[j].y &= 0x7fff7fffu; raw[j].z &= 0x7fff7fffu; raw[j].w &= 0x7fff7fffu;
      }
      ss = (__low2float(acc) + __high2float(acc)) * 4096.f;
    } else {
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          const uint32_t r = raw_elem<T>(raw[j], c);
          const int e = j * VEC + c;
          if (EB::sign(r)) sgnm |= 1ull << e;
          if (j < NS) {
            const float v = EB::key2f(EB::abs_bits(r));
            ss = fmaf(v, v, ss);
          }
        }
        // keys in place: clear the sign bits
        constexpr uint32_t m = (sizeof(T) == 4) ? 0x7fffffffu : 0x7fff7fffu;
        raw[j].x &= m; raw[j].y &= m; raw[j].z &= m; raw[j].w &= m;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
    ss *= inv_ns;
    const float rms = (ss > 0.f) ? ss * rsqrtf(ss) : 0.f;   // estimate only

    // ---- T* = x-th largest key ----
    uint32_t lo = 0u, hi = EB::kKeyEnd;        // count(>= lo) >= x > count(>= hi)
    unsigned clo = 32u * E, chi = 0u;
    uint32_t Tk = 0u;
    bool exact = false;                        // true: exactly x keys are >= Tk
    auto update = [&](uint32_t c, unsigned cnt) {
      if (cnt == (unsigned)x) { Tk = c; exact = true; }
      else if (cnt > (unsigned)x) { if (c > lo) { lo = c; clo = cnt; } }
      else if (c < hi) { hi = c; chi = cnt; }
    };
    {
      const float t = rms * ratio;
      uint32_t p1 = EB::f2key(t * (1.f - kProbeDelta)), p2 = EB::f2key(t * (1.f + kProbeDelta));
      p1 = min(max(p1, 1u), EB::kKeyEnd - 2u);
      p2 = min(max(p2, p1 + 1u), EB::kKeyEnd - 1u);
      unsigned n1, n2;
      CNT::ge2(raw, p1, p2, n1, n2);
      n1 = __reduce_add_sync(kFull, n1);
      n2 = __reduce_add_sync(kFull, n2);
      update(p1, n1);
      if (!exact) update(p2, n2);
    }
    unsigned phase = 0;   // every third pass bisects the key range (guaranteed progress)
#pragma unroll 1
    while (!exact && hi - lo > 1u) {
      const float vl = EB::key2f(lo), vh = EB::key2f(hi);
      const float f = __fdividef((float)(clo - (unsigned)x) + 0.5f, (float)(clo - chi));
      const uint32_t ci = min(max(EB::f2key(fmaf(f, vh - vl, vl)), lo + 1u), hi - 1u);
      const bool bis = (hi == EB::kKeyEnd) || phase == 2u;
      phase = (phase == 2u) ? 0u : phase + 1u;
      const uint32_t c = bis ? lo + ((hi - lo) >> 1) : ci;   // lo < c < hi
      const unsigned cnt = __reduce_add_sync(kFull, CNT::ge(raw, c));
      exact = cnt == (unsigned)x;
      const bool up = cnt > (unsigned)x;
      Tk = c;
      lo = up ? c : lo;
      clo = up ? cnt : clo;
      hi = up ? hi : c;
      chi = up ? chi : cnt;
    }
    if (!exact) { Tk = lo; exact = (clo == (unsigned)x); }
    if (Tk != 0u && rms > 0.f) {
      const float rn = __fdividef(EB::key2f(Tk), rms);
      if (rn > 0.f && rn < 1e30f) ratio = rn;
    }

    // ---- selection mask (bit e): selected keys are >= max(Tk, 1), so non-zero ----
    uint64_t selm = 0;
    if (exact || Tk == 0) {
      // exact: keys >= Tk are precisely the x largest.  Tk == 0: fewer than x
      // non-zero magnitudes -> every non-zero is selected; selected zeros
      // would encode as 0 anyway (R2), so they need no bit.
      const uint32_t lo_sel = (Tk == 0) ? 1u : Tk;
      if constexpr (std::is_same<T, __half>::value) {
        const __half hs = __ushort_as_half((unsigned short)lo_sel);
        const __half2 t2 = __halves2half2(hs, hs);
#pragma unroll
        for (int j = 0; j < NCH; ++j)
          selm |= (uint64_t)flags16_to_bits8(__hge2_mask(as_h2(raw[j].x), t2), __hge2_mask(as_h2(raw[j].y), t2),
                                             __hge2_mask(as_h2(raw[j].z), t2), __hge2_mask(as_h2(raw[j].w), t2))
                  << (8 * j);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (KEY(e) >= lo_sel) selm |= 1ull << e;
      }
    } else {
      int cgt = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) cgt += (KEY(e) > Tk) ? 1 : 0;
      const int gt = (int)__reduce_add_sync(kFull, (unsigned)cgt);
      int need = x - gt;            // how many keys == Tk to take, in index order
      // index order: chunk j, then lane, then c
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        int eq = 0;
#pragma unroll
        for (int c = 0; c < VEC; ++c) eq += (KEY(j * VEC + c) == Tk) ? 1 : 0;
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
          const uint32_t k = KEY(e);
          bool s = k > Tk;
          if (k == Tk) { s = rank < need; ++rank; }
          if (s) selm |= 1ull << e;
        }
        need -= total;
      }
    }
    // ---- pack: pos bit = selected & sign 0; neg = selected & sign 1 ----
    // Each lane's bits of chunk j are plane bits [128 j + VEC l, +VEC): bytes
    // are assembled in this warp's shared-memory code buffer (fp32: two lanes'
    // nibbles per byte, one shuffle), then copied out with 16-byte stores.
    const uint64_t posm = selm & ~sgnm, negm = selm & sgnm;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      constexpr uint32_t vmask = (1u << VEC) - 1u;
      const uint32_t pb_ = (uint32_t)(posm >> (j * VEC)) & vmask;
      const uint32_t nb_ = (uint32_t)(negm >> (j * VEC)) & vmask;
      uint32_t byte_idx;
      uint32_t v;
      bool wr;
      if (VEC == 4) {
        const uint32_t pq = pb_ | (nb_ << 8);
        const uint32_t partner = __shfl_down_sync(kFull, pq, 1);
        v = pq | (partner << 4);                 // bits 0-7: pos byte, 8-15: neg byte
        byte_idx = (uint32_t)j * 16u + (uint32_t)(lane >> 1);
        wr = (lane & 1) == 0;
      } else {
        v = pb_ | (nb_ << 8);
        byte_idx = (uint32_t)j * 32u + (uint32_t)lane;
        wr = true;
      }
      if (wr && byte_idx < (uint32_t)(pw * 4)) {
        s_code[byte_idx] = (uint8_t)v;
        s_code[pw * 4 + byte_idx] = (uint8_t)(v >> 8);
      }
    }
    __syncwarp();
    {
      uint4* dst = reinterpret_cast<uint4*>(codes + row * cb);
      const uint4* src = reinterpret_cast<const uint4*>(s_code);
      for (int i = lane; i < (int)(cb / 16); i += 32) dst[i] = src[i];
    }
    __syncwarp();
    if (nrow < n) {
#pragma unroll
      for (int j = 0; j < NCH; ++j) raw[j] = load_chunk<T, VECLOAD>(u + nrow * ld, j * 32 * VEC + lane * VEC, d);
    }
  }
}

// Phi^-1(p) for p in (0, 1) (Acklam's rational approximation; only steers the
// probes of the search, never decides a bit)
float inv_norm_cdf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549671010415733e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double dd[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                              3.754408661907416e+00};
  if (p <= 0.0) p = 1e-12;
  if (p >= 1.0) p = 1.0 - 1e-12;
  const double pl = 0.02425;
  double q, r;
  if (p < pl) {
    q = sqrt(-2 * log(p));
    return (float)((((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
                   ((((dd[0] * q + dd[1]) * q + dd[2]) * q + dd[3]) * q + 1));
  }
  if (p > 1 - pl) {
    q = sqrt(-2 * log(1 - p));
    return (float)(-(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
                   ((((dd[0] * q + dd[1]) * q + dd[2]) * q + dd[3]) * q + 1));
  }
  q = p - 0.5;
  r = q * q;
  return (float)((((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
                 (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1));
}

template <typename T, int NCH>
static cudaError_t launch_encode_nch(const void* u, int64_t n, int32_t d, int64_t ld, int32_t x,
                                     uint8_t* codes, bool vec, int sms, cudaStream_t st) {
  int64_t blocks = (n + kEncWarps - 1) / kEncWarps;
  int64_t cap = (int64_t)sms * 16;  // grid-stride beyond ~16 CTAs per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // |u|_(x) of d i.i.d. N(0, s^2) draws ~ s * Phi^-1(1 - x / 2d)
  float z0 = inv_norm_cdf(1.0 - ((double)x - 0.5) / (2.0 * (double)d));
  if (!(z0 > 1e-3f)) z0 = 1e-3f;
  if (vec)
    encode_kernel<T, NCH, true><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
        (const T*)u, n, d, ld, x, z0, codes);
  else
    encode_kernel<T, NCH, false><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
        (const T*)u, n, d, ld, x, z0, codes);
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
