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
// f32 runs steps 1-2 first on COARSE keys -- the top 16 bits of two keys per
// word (a bf16 truncation), compared as f16 patterns by HSET2 and counted by
// HADD2, half the instructions of a 32-bit key pass; coarse(a) > coarse(b)
// implies key(a) > key(b), so the coarse bracket is a key bracket -- and only
// the last one-coarse-value bracket (a few keys) with full 32-bit keys.
// The probes only steer the search: T* is exact for any input.  fp16 rows count
// two keys per instruction (HSET2 on |u| half pairs, exact small-integer HADD2).
// Keys > T* are selected, keys == T* are taken in index order until x are
// selected (lowest index wins, R1).  Bits are assembled with warp shuffles into
// 32-bit plane words and stored.  The next row's loads are issued before the
// current row is packed, and rows further ahead are prefetched into L2.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
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

__device__ __forceinline__ __half2 as_h2(uint32_t w) { return *reinterpret_cast<const __half2*>(&w); }
__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<const uint32_t*>(&h); }

// 1/v (MUFU.RCP; steering arithmetic only, never decides a bit)
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// f32 coarse keys (two 15-bit patterns per word, compared as f16): count >= c
template <int NW>
__device__ __forceinline__ unsigned coarse_ge(const uint32_t (&cw)[NW], uint32_t c) {
  const __half2 cc = as_h2(c | (c << 16));
  __half2 a0 = __float2half2_rn(0.f), a1 = a0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const __half2 w = as_h2(cw[i]);
    if (i & 1) a1 = __hadd2(a1, __hge2(w, cc));
    else a0 = __hadd2(a0, __hge2(w, cc));
  }
  const __half2 a = __hadd2(a0, a1);
  return (unsigned)(__low2float(a) + __high2float(a));
}
template <int NW>
__device__ __forceinline__ void coarse_ge2(const uint32_t (&cw)[NW], uint32_t c1, uint32_t c2, unsigned& n1,
                                           unsigned& n2) {
  const __half2 cc1 = as_h2(c1 | (c1 << 16)), cc2 = as_h2(c2 | (c2 << 16));
  __half2 a1 = __float2half2_rn(0.f), a2 = a1;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const __half2 w = as_h2(cw[i]);
    a1 = __hadd2(a1, __hge2(w, cc1));
    a2 = __hadd2(a2, __hge2(w, cc2));
  }
  n1 = (unsigned)(__low2float(a1) + __high2float(a1));
  n2 = (unsigned)(__low2float(a2) + __high2float(a2));
}

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
// NCH: chunks of 32*VEC elements per row (compile-time so keys live in registers).
template <typename T, int NCH, bool VECLOAD>
__global__ void __launch_bounds__(kEncWarps * 32, (sizeof(T) == 4 && NCH > 8) ? 2 : 3)
encode_kernel(const T* __restrict__ u, int64_t n, int32_t d, int64_t ld, int32_t x, float z0, float delta,
              uint8_t* __restrict__ codes) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int E = NCH * VEC;        // elements per lane
  constexpr int NS = (sizeof(T) == 4) ? (NCH < 2 ? NCH : NCH / 2) : (NCH < 2 ? NCH : 2);  // chunks used for the RMS
  constexpr bool F32 = sizeof(T) == 4;
  constexpr int NWC = F32 ? E / 2 : 1;   // f32: coarse words (top 16 bits of two keys each)
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
    } else if constexpr (!F32) {
      // bf16: sign flags as f16 (bits 15/31 of each word); RMS from the halves widened to f32
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        sgnm |= (uint64_t)flags16_to_bits8(raw[j].x, raw[j].y, raw[j].z, raw[j].w) << (8 * j);
        if (j < NS) {
          const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xffff0000u);
            ss = fmaf(lo, lo, fmaf(hi, hi, ss));
          }
        }
        raw[j].x &= 0x7fff7fffu; raw[j].y &= 0x7fff7fffu; raw[j].z &= 0x7fff7fffu; raw[j].w &= 0x7fff7fffu;
      }
    } else {
      // f32: sign bits shifted in by funnel shifts (one SHF per element, last
      // element first so that bit e ends up at position e)
      uint32_t sg[2] = {0u, 0u};
#pragma unroll
      for (int e = E - 1; e >= 0; --e) {
        const uint32_t r = raw_elem<T>(raw[e / VEC], e % VEC);
        sg[e >> 5] = __funnelshift_l(r, sg[e >> 5], 1);
      }
      sgnm = (uint64_t)sg[0] | ((uint64_t)sg[1] << 32);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        if (j < NS) {
          ss = fmaf(__uint_as_float(raw[j].x), __uint_as_float(raw[j].x), ss);
          ss = fmaf(__uint_as_float(raw[j].y), __uint_as_float(raw[j].y), ss);
          ss = fmaf(__uint_as_float(raw[j].z), __uint_as_float(raw[j].z), ss);
          ss = fmaf(__uint_as_float(raw[j].w), __uint_as_float(raw[j].w), ss);
        }
        raw[j].x &= 0x7fffffffu; raw[j].y &= 0x7fffffffu; raw[j].z &= 0x7fffffffu; raw[j].w &= 0x7fffffffu;
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
    if constexpr (F32) {
      // Coarse phase: the top 16 bits of two keys per word (a bf16 truncation),
      // compared as f16 patterns (for non-negative patterns the f16 order is the
      // integer order; >= 0x7C00 -- |u| >= 2^121 -- clamped to 0x7BFF by HMNMX2),
      // counted two keys per HSET2 + HADD2: half the cost of a full-key pass.
      // coarse(a) > coarse(b) => key(a) > key(b), so the coarse bracket is a key
      // bracket: [lo_c << 16, hi_c << 16).  It ends exact (exactly x keys have
      // coarse >= Tc, i.e. key >= Tc << 16) or one coarse value wide (its few
      // keys are then resolved by full-key passes below).
      uint32_t cw[NWC];
      const __half2 cmax = as_h2(0x7bff7bffu);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        cw[2 * j] = h2_bits(__hmin2(as_h2(__byte_perm(raw[j].x, raw[j].y, 0x7632)), cmax));
        cw[2 * j + 1] = h2_bits(__hmin2(as_h2(__byte_perm(raw[j].z, raw[j].w, 0x7632)), cmax));
      }
      uint32_t lc = 0u, hc = 0x7c00u;
      const float t = rms * ratio;
      uint32_t p1 = (__float_as_uint(t * (1.f - delta)) >> 16) & 0x7fffu;
      uint32_t p2 = (__float_as_uint(t * (1.f + delta)) >> 16) & 0x7fffu;
      p1 = min(max(p1, 1u), 0x7bfeu);
      p2 = min(max(p2, p1 + 1u), 0x7bffu);
      unsigned n1, n2;
      coarse_ge2<NWC>(cw, p1, p2, n1, n2);
      n1 = __reduce_add_sync(kFull, n1);
      n2 = __reduce_add_sync(kFull, n2);
      auto cupd = [&](uint32_t c, unsigned cnt) {
        if (exact) return;
        if (cnt == (unsigned)x) { Tk = c << 16; exact = true; }
        else if (cnt > (unsigned)x) { if (c > lc) { lc = c; clo = cnt; } }
        else if (c < hc) { hc = c; chi = cnt; }
      };
      cupd(p1, n1);
      cupd(p2, n2);
      unsigned cph = 0;
#pragma unroll 1
      while (!exact && hc - lc > 1u) {
        const float vl = __uint_as_float(lc << 16), vh = __uint_as_float(hc << 16);
        const float f = ((float)(clo - (unsigned)x) + 0.5f) * rcp_approx((float)(clo - chi));
        const uint32_t ci = min(max((__float_as_uint(fmaf(f, vh - vl, vl)) >> 16) & 0x7fffu, lc + 1u), hc - 1u);
        const bool bis = (hc == 0x7c00u) || cph == 2u;
        cph = (cph == 2u) ? 0u : cph + 1u;
        const uint32_t c = bis ? lc + ((hc - lc) >> 1) : ci;
        const unsigned cnt = __reduce_add_sync(kFull, coarse_ge<NWC>(cw, c));
        exact = cnt == (unsigned)x;
        const bool up = cnt > (unsigned)x;
        Tk = c << 16;
        lc = up ? c : lc;
        clo = up ? cnt : clo;
        hc = up ? hc : c;
        chi = up ? chi : cnt;
      }
      // full-key bracket (the clamped top coarse value reaches the end of the key range)
      lo = lc << 16;
      hi = (hc == 0x7c00u) ? EB::kKeyEnd : (hc << 16);
      if (hc == 0x7c00u) chi = 0u;
    } else {
      const float t = rms * ratio;
      uint32_t p1 = EB::f2key(t * (1.f - delta)), p2 = EB::f2key(t * (1.f + delta));
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
      const float f = ((float)(clo - (unsigned)x) + 0.5f) * rcp_approx((float)(clo - chi));
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
      } else if constexpr (F32) {
        // bit = (key >= lo_sel) = sign of (lo_sel - 1 - key) (both < 2^31), shifted in
        uint32_t sl[2] = {0u, 0u};
#pragma unroll
        for (int e = E - 1; e >= 0; --e) sl[e >> 5] = __funnelshift_l(lo_sel - 1u - KEY(e), sl[e >> 5], 1);
        selm = (uint64_t)sl[0] | ((uint64_t)sl[1] << 32);
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
      UQ_ASSERT(!wr || byte_idx >= (uint32_t)(pw * 4) || pw * 8 <= kMaxCodeBytes);
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

// ---------------------------------------------------------------------------
// fp16 rows: a leaner kernel for the same search (c5's DB encode).  The generic
// kernel spent ~716 warp instructions per d=768 row, ALU-pipe bound (ncu:
// issue 76%, ALU 72%; profiles/r02/enc_f16_*).  Here:
//  * the raw words keep their signs; |u| comes from the HSET2 operand modifier
//    (no sign-clearing pass, no separate sign mask);
//  * a count pass is 2 instructions per two keys (HSET2.BF + HADD2) plus 3 for
//    the warp total: the per-half sums start at 512 so lo + hi = 1024 + n is an
//    f16 whose low bits are n (HADD2 + LOP3 + REDUX, no float conversions);
//  * the interpolation runs in key space (integer keys are piecewise linear in
//    |u|) and the forced bisections start only after 4 interpolated passes;
//    T*/RMS is tracked as an average over the warp's rows (measured in a
//    simulator of this search on c5 rows: 4.08 -> 3.42 passes per row);
//  * selected bits come straight from signed compares (u >= T: +1, u <= -T:
//    -1), assembled by LOP3 from the HSET2 masks, and each lane stores its
//    plane bytes directly (one 32-byte sector per warp store).
// Exactness is as in the generic kernel: every decision is an exact compare
// of f16 magnitudes (HSET2 is exact on f16, subnormals included).
__device__ __forceinline__ __half2 h2(uint32_t w) { return *reinterpret_cast<const __half2*>(&w); }

// Warp total of count(|u| >= c) over this lane's NW half pairs, BIASED by
// kF16Bias: each lane's half sums start at 512, so lo + hi = 1024 + n is an f16
// whose bit pattern is 0x6400 + n (n <= 2*NW < 1024: exact).  The search
// compares biased counts with x + kF16Bias and never unbiases them.
constexpr uint32_t kF16Bias = 32u * 0x6400u;
// (|w| >= c) per half as 1.0 / 0.0 (HSET2.BF with the |.| operand modifier).  One
// asm block so the compiler cannot hoist the loop-invariant |w| out of the
// search loop into 12 extra registers and 12 extra instructions per row.
__device__ __forceinline__ uint32_t hge_abs_bf(uint32_t w, uint32_t c2) {
  uint32_t r;
  asm("{\n\t.reg .b32 a;\n\tabs.f16x2 a, %1;\n\tset.ge.f16x2.f16x2 %0, a, %2;\n\t}" : "=r"(r) : "r"(w), "r"(c2));
  return r;
}
// warp sum (REDUX) without the compiler's divergent-warp fallback path
__device__ __forceinline__ unsigned redux_add(unsigned v) {
  unsigned r;
  asm("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
template <int NW, bool ABS = true>
__device__ __forceinline__ unsigned f16_count_ge(const uint32_t (&w)[NW], uint32_t c2) {  // c2 = c | c << 16
  const __half2 cc = h2(c2);
  __half2 acc = h2(0x60006000u);  // (512, 512)
#pragma unroll
  for (int i = 0; i < NW; ++i) acc = __hadd2(acc, ABS ? h2(hge_abs_bf(w[i], c2)) : __hge2(h2(w[i]), cc));
  const __half s = __hadd(__low2half(acc), __high2half(acc));
  return redux_add((unsigned)__half_as_ushort(s));
}
__device__ __forceinline__ uint32_t dup16(uint32_t c) { return __byte_perm(c, 0u, 0x1010); }

// 8 flags (bit 2k + h = half h of m_k, from HSET2 masks 0xffff/0) -> low byte
__device__ __forceinline__ uint32_t mask8(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  uint32_t t = m0 & 0x00020001u;
  t |= m1 & 0x00080004u;
  t |= m2 & 0x00200010u;
  t |= m3 & 0x00800040u;
  return t | (t >> 16);   // bits 0..7 (upper bits: don't care, stored as a byte)
}

// 8 flags as HSET2.BF halves (1.0 / 0.0; b_k = elements 2k, 2k+1) -> 0x6400 + byte
// in the low 16 bits: weighted sums on the FP16 pipe (HFMA2), exact small
// integers, the 1024.0 bias puts the byte in the low 8 bits of the f16 pattern
__device__ __forceinline__ uint32_t bits8_bf(__half2 b0, __half2 b1, __half2 b2, __half2 b3) {
  __half2 acc = h2(0x00006400u);                     // (1024, 0)
  acc = __hfma2(b0, h2(0x40003c00u), acc);           // (1, 2)
  acc = __hfma2(b1, h2(0x48004400u), acc);           // (4, 8)
  acc = __hfma2(b2, h2(0x50004c00u), acc);           // (16, 32)
  acc = __hfma2(b3, h2(0x58005400u), acc);           // (64, 128)
  return (uint32_t)__half_as_ushort(__hadd(__low2half(acc), __high2half(acc)));
}

__device__ __forceinline__ float rsqrt_approx(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// FULL: 16-byte aligned rows with d == 256 * NCH (every chunk a full vector
// load, plane bytes = 32 * NCH): no per-chunk bounds.
// Search steering of the fp16 kernel (never decides a bit): the interpolation
// aims a quarter element above the x-th count and T*/scale is averaged with
// weight 0.15 -- a simulator of this search on c5 rows: 4.98 -> 4.79 count
// passes per row against the round-2 0.5 / 0.3.
#ifndef UQ_ENC16_OFF
#define UQ_ENC16_OFF 0.25f
#endif
#ifndef UQ_ENC16_EMA
#define UQ_ENC16_EMA 0.15f
#endif
#ifndef UQ_ENC16_ONEPROBE
#define UQ_ENC16_ONEPROBE 1
#endif
#ifndef UQ_ENC16_SLOPE_EMA
#define UQ_ENC16_SLOPE_EMA 0.05f
#endif
#ifndef UQ_ENC16_REDUX_SCALE
#define UQ_ENC16_REDUX_SCALE 1
#endif
template <int NCH, bool VECLOAD, bool FULL>
__global__ void __launch_bounds__(kEncWarps * 32, NCH <= 4 ? 6 : 3)
encode_f16_kernel(const __half* __restrict__ u, int64_t n, int32_t d, int64_t ld, int32_t x, float z0, float delta,
                  float slope0, uint8_t* __restrict__ codes) {
  constexpr int NW = 4 * NCH;                 // half pairs per lane
  constexpr int NS = NCH < 2 ? NCH : 2;       // chunks sampled for the RMS
  constexpr uint32_t kEnd = 0x7c01u;          // finite keys are < kEnd (inf / NaN: precondition, R4)
  const int lane = threadIdx.x & 31;
  const int64_t pb = FULL ? 32 * NCH : plane_bytes(d);
  const int64_t cb = 2 * pb;
  const int64_t warp_global = (int64_t)blockIdx.x * kEncWarps + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kEncWarps;
  const float inv_ns = 1.0f / (float)min(d, 256 * NS);
  const unsigned xb = (unsigned)x + kF16Bias;
  const int64_t ustep = nwarps * ld, cstep = nwarps * cb;
  float ratio = z0;   // T* / RMS, averaged over this warp's rows
  float slope = slope0;   // keys per unit of count near T*, averaged over this warp's rows
  auto load_row = [&](const __half* src, uint4 (&r)[NCH]) {
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      if constexpr (FULL) r[j] = __ldg(reinterpret_cast<const uint4*>(src + j * 256 + lane * 8));
      else r[j] = load_chunk<__half, VECLOAD>(src, j * 256 + lane * 8, d);
    }
  };
  // L2 prefetch of the row two iterations ahead: one 128-byte line per lane
  const bool pf_lane = VECLOAD && lane * 64 < d;
  // The row is loaded at the top of its iteration (no register double buffer:
  // 40 registers, six CTAs = 48 warps per SM; the L2 prefetch two rows ahead
  // covers the latency).  Measured against a register double buffer (54-59
  // registers, 32 warps): 3447 vs 3401 GB/s on c5 rows.
  uint4 raw[NCH];
  const __half* up = u + warp_global * ld;
  uint8_t* cp = codes + warp_global * cb;
  for (int64_t row = warp_global; row < n; row += nwarps, up += ustep, cp += cstep) {
    if (pf_lane && row + 2 * nwarps < n)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(up + 2 * ustep + lane * 64) : "memory");
    load_row(up, raw);
    uint32_t w[NW];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      w[4 * j] = raw[j].x; w[4 * j + 1] = raw[j].y; w[4 * j + 2] = raw[j].z; w[4 * j + 3] = raw[j].w;
    }
    // ---- scale estimate: mean |u| (HFMA2 of |u| * 2^-6; steering only) ----
    float ss;
    {
      __half2 acc = __float2half2_rn(0.f);
      const __half2 sc = __float2half2_rn(0.015625f);
#pragma unroll
      for (int i = 0; i < 4 * NS; ++i) acc = __hfma2(__habs2(h2(w[i])), sc, acc);
      ss = (__low2float(acc) + __high2float(acc)) * 64.f;
    }
#if UQ_ENC16_REDUX_SCALE
    // warp sum as one REDUX of 2^-10 fixed point (clamped so 32 lanes cannot
    // overflow; steering only): 3 instructions instead of 5 shuffles + 5 adds
    const float rms = (float)(int)redux_add((unsigned)min(__float2int_rn(ss * 1024.f), 1 << 26)) *
                      (inv_ns * (1.f / 1024.f));
#else
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
    const float rms = ss * inv_ns;
#endif

    // ---- T* = x-th largest key: count(>= lo) >= x > count(>= hi) (counts biased) ----
    uint32_t lo = 0u, hi = kEnd, Tk = 0u;
    unsigned clo = 256u * NCH + kF16Bias, chi = kF16Bias;
    bool exact = false;
#if UQ_ENC16_ONEPROBE
    // one probe at the predicted T*, then a step by the warp's learned count
    // slope straight at the x-th count (a simulator of this search on c5 rows:
    // 4.82 -> 4.05 count passes per row against two probes at t(1 -/+ delta))
    uint32_t p1;
    unsigned n1;
    {
      const float t = rms * ratio;
      p1 = min(max((uint32_t)__half_as_ushort(__float2half_rn(t)) & 0x7fffu, 1u), 0x7bffu);
      n1 = f16_count_ge<NW>(w, dup16(p1));
      float islope = slope;
      uint32_t c = p1;
      if (n1 == xb) { Tk = p1; exact = true; }
      else {
        const bool up1 = n1 > xb;
        lo = up1 ? p1 : 0u; clo = up1 ? n1 : clo;
        hi = up1 ? kEnd : p1; chi = up1 ? chi : n1;
        // n1 - xb > 0: T* above p1; the step lands inside (lo, hi)
        c = (uint32_t)((int)p1 + __float2int_rn((float)(int)(n1 - xb) * slope));
        c = (int)c <= (int)lo ? lo + 1u : min(c, hi - 1u);
      }
      unsigned sec = 6u;   // interpolated passes before the forced bisections start
#pragma unroll 1
      while (!exact) {
        const unsigned cnt = f16_count_ge<NW>(w, dup16(c));
        exact = cnt == xb;
        const bool up_ = cnt > xb;
        Tk = c;
        lo = up_ ? c : lo;
        clo = up_ ? cnt : clo;
        hi = up_ ? hi : c;
        chi = up_ ? chi : cnt;
        if (exact || hi - lo <= 1u) break;
        if (hi == kEnd || lo == 0u) {
          // T* still outside the bracket: step past its one end by the
          // learned slope, doubling each time the step falls short
          const uint32_t s = (uint32_t)(((float)(hi == kEnd ? clo - xb : xb - chi) + 0.5f) * islope) + 1u;
          c = hi == kEnd ? lo + s : (hi > s ? hi - s : 0u);
          c = min(max(c, lo + 1u), hi - 1u);
          islope *= 2.f;
        } else if (sec == 0u) {
          c = lo + ((hi - lo) >> 1);                 // guaranteed progress
          sec = 1u;
        } else {
          const float f = ((float)(clo - xb) + UQ_ENC16_OFF) * rcp_approx((float)(clo - chi));
          c = lo + (uint32_t)(f * (float)(hi - lo));
          c = min(max(c, lo + 1u), hi - 1u);
          --sec;
        }
      }
    }
#else
    float islope;
    {
      const float t = rms * ratio;
      // both probes in one packed conversion; clamped to [1, 0x7bff] per half
      const uint32_t pp = __vminu2(__vmaxu2(h2_bits(__floats2half2_rn(t * (1.f - delta), t * (1.f + delta))) & 0x7fff7fffu,
                                            0x00010001u), 0x7bff7bffu);
      const uint32_t p1 = pp & 0xffffu;
      const uint32_t p2 = max(pp >> 16, p1 + 1u);
      const unsigned n1 = f16_count_ge<NW>(w, dup16(p1));
      const unsigned n2 = f16_count_ge<NW>(w, dup16(p2));
      // keys per unit of count between the probes (extrapolation when T* is
      // outside them)
      islope = (float)(p2 - p1) * rcp_approx((float)max(n1 - n2, 1u));
      // n1 >= n2 (p1 < p2)
      if (n1 == xb) { Tk = p1; exact = true; }
      else if (n2 == xb) { Tk = p2; exact = true; }
      else if (n2 > xb) { lo = p2; clo = n2; }
      else if (n1 > xb) { lo = p1; clo = n1; hi = p2; chi = n2; }
      else { hi = p1; chi = n1; }
    }
    unsigned sec = 6u;   // interpolated passes before the forced bisections start
#pragma unroll 1
    while (!exact && hi - lo > 1u) {
      uint32_t c;
      if (hi == kEnd || lo == 0u) {
        // T* outside the probes: step past the nearer one by the probes'
        // slope (doubling each time the step falls short)
        const uint32_t s = (uint32_t)(((float)(hi == kEnd ? clo - xb : xb - chi) + 0.5f) * islope) + 1u;
        c = hi == kEnd ? lo + s : (hi > s ? hi - s : 0u);
        c = min(max(c, lo + 1u), hi - 1u);
        islope *= 2.f;
      } else if (sec == 0u) {
        c = lo + ((hi - lo) >> 1);                 // guaranteed progress
        sec = 1u;
      } else {
        const float f = ((float)(clo - xb) + UQ_ENC16_OFF) * rcp_approx((float)(clo - chi));
        c = lo + (uint32_t)(f * (float)(hi - lo));
        c = min(max(c, lo + 1u), hi - 1u);
        --sec;
      }
      const unsigned cnt = f16_count_ge<NW>(w, dup16(c));
      exact = cnt == xb;
      const bool up_ = cnt > xb;
      Tk = c;
      lo = up_ ? c : lo;
      clo = up_ ? cnt : clo;
      hi = up_ ? hi : c;
      chi = up_ ? chi : cnt;
    }
#endif
    if (!exact) { Tk = lo; exact = (clo == xb); }
    if (Tk != 0u && rms > 0.f) {
      const float rn = __fdividef(ElemBits<__half>::key2f(Tk), rms);
      if (rn > 0.f && rn < 1e30f) ratio = fmaf(UQ_ENC16_EMA, rn - ratio, ratio);
    }
#if UQ_ENC16_ONEPROBE
    if (n1 != xb) {   // observed keys per count between the probe and T*
      const float so = (float)abs((int)Tk - (int)p1) * rcp_approx((float)abs((int)(n1 - xb)));
      slope = fmaf(UQ_ENC16_SLOPE_EMA, min(so, 4096.f) - slope, slope);
    }
#endif

    // ---- plane bytes: +1 where u >= T, -1 where u <= -T (T >= 1: zeros never) ----
    uint32_t posb[NCH], negb[NCH];
    if (exact || Tk == 0u) {
      // exact: the keys >= Tk are the x largest.  Tk == 0: fewer than x
      // non-zero magnitudes -> every non-zero is selected (R2).
      const uint32_t ts = (Tk == 0u) ? 1u : Tk;
      const __half2 tp = h2(dup16(ts)), tn = h2(dup16(ts | 0x8000u));
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        posb[j] = bits8_bf(__hge2(h2(w[4 * j]), tp), __hge2(h2(w[4 * j + 1]), tp),
                           __hge2(h2(w[4 * j + 2]), tp), __hge2(h2(w[4 * j + 3]), tp));
        negb[j] = bits8_bf(__hle2(h2(w[4 * j]), tn), __hle2(h2(w[4 * j + 1]), tn),
                           __hle2(h2(w[4 * j + 2]), tn), __hle2(h2(w[4 * j + 3]), tn));
      }
    } else {
      // ties at T* (count(>= T) = clo > x > chi = count(> T)): keys > T plus
      // the first x - chi keys == T in index order (chunk, lane, element; R1)
      const __half2 tp = h2(dup16(Tk)), tn = h2(dup16(Tk | 0x8000u));
      int need = (int)(xb - chi);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const uint32_t gp = mask8(__hgt2_mask(h2(w[4 * j]), tp), __hgt2_mask(h2(w[4 * j + 1]), tp),
                                  __hgt2_mask(h2(w[4 * j + 2]), tp), __hgt2_mask(h2(w[4 * j + 3]), tp)) & 0xffu;
        const uint32_t gn = mask8(__hlt2_mask(h2(w[4 * j]), tn), __hlt2_mask(h2(w[4 * j + 1]), tn),
                                  __hlt2_mask(h2(w[4 * j + 2]), tn), __hlt2_mask(h2(w[4 * j + 3]), tn)) & 0xffu;
        const uint32_t ep = mask8(__heq2_mask(h2(w[4 * j]), tp), __heq2_mask(h2(w[4 * j + 1]), tp),
                                  __heq2_mask(h2(w[4 * j + 2]), tp), __heq2_mask(h2(w[4 * j + 3]), tp)) & 0xffu;
        const uint32_t en = mask8(__heq2_mask(h2(w[4 * j]), tn), __heq2_mask(h2(w[4 * j + 1]), tn),
                                  __heq2_mask(h2(w[4 * j + 2]), tn), __heq2_mask(h2(w[4 * j + 3]), tn)) & 0xffu;
        uint32_t eq = ep | en;
        const int ce = __popc(eq);
        int incl = ce;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int tv = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += tv;
        }
        const int take = min(max(need - (incl - ce), 0), ce);   // keep the lowest `take` bits of eq
        while (__popc(eq) > take) eq &= ~(0x80000000u >> __clz(eq));
        need -= __shfl_sync(kFull, incl, 31);
        posb[j] = gp | (eq & ep);
        negb[j] = gn | (eq & en);
      }
    }
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int64_t bi = 32 * j + lane;
      if (FULL || bi < pb) {
        cp[bi] = (uint8_t)posb[j];
        cp[pb + bi] = (uint8_t)negb[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fp16 rows, large n: R rows per warp iteration (a BATCH), the same exact
// search as encode_f16_kernel with its CONTROL run lane-parallel.  The search
// above spends ~75 warp instructions per count pass of which 26 count; the
// rest -- bracket update, interpolation, clamps, branches -- is warp-uniform
// scalar work.  Here lane r (< R) owns the search state of the batch's row r:
// one round is, for every row still searching, {broadcast its threshold (one
// SHFL), count over the row (the same biased HSET2/HADD2 sums + REDUX), keep
// the count in lane r}, then ONE lane-parallel bracket update / next
// threshold for all R rows at once.  A warp cannot hold R rows in registers,
// so the batch is staged in shared memory by cp.async (16 B per lane per
// chunk, each lane reads back only what it staged itself: no barriers, no bank
// conflicts) and each pass re-reads its row with NCH LDS.128.  T*/scale and the
// count slope are learned per lane (each lane sees every R-th row of the warp).
// Every decision is the same exact f16 compare as above: identical bytes.
#ifndef UQ_ENC16_BATCH
#define UQ_ENC16_BATCH 0
#endif
#ifndef UQ_ENC16_BATCH_R
#define UQ_ENC16_BATCH_R 8
#endif
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
  return v;
}

template <int NCH, int R>
__global__ void __launch_bounds__(kEncWarps * 32, R >= 8 ? 2 : 4)
encode_f16_batch_kernel(const __half* __restrict__ u, int64_t n, int64_t ld, int32_t x, float z0, float slope0,
                        uint8_t* __restrict__ codes) {
  extern __shared__ __align__(16) uint8_t enc_smem[];
  constexpr int NW = 4 * NCH;
  constexpr int NS = NCH < 2 ? NCH : 2;
  constexpr uint32_t kEnd = 0x7c01u;
  constexpr int64_t pb = 32 * NCH, cb = 2 * pb;
  constexpr uint32_t kRowBytes = 512u * NCH;
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (int64_t)blockIdx.x * kEncWarps + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kEncWarps;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(enc_smem) + (threadIdx.x >> 5) * (R * kRowBytes) + lane * 16;
  const float inv_ns = 1.0f / (float)(256 * NS);
  const unsigned xb = (unsigned)x + kF16Bias;
  float ratio = z0, slope = slope0;   // per lane: learned over the rows this lane owns
  const int64_t nbatch = (n + R - 1) / R;
  for (int64_t b = warp_global; b < nbatch; b += nwarps) {
    const int64_t row0 = b * R;
    const int nr = (int)min((int64_t)R, n - row0);
    const __half* ub = u + row0 * ld;
    // L2 prefetch of this warp's next batch, one 128-byte line per lane and step
    if (b + nwarps < nbatch) {
      const __half* un = ub + nwarps * R * ld;
      const int nrn = (int)min((int64_t)R, n - (row0 + nwarps * R));
#pragma unroll
      for (int t = 0; t < (R * NCH * 4 + 31) / 32; ++t) {
        const int li = t * 32 + lane, pr = li / (NCH * 4), pl = li % (NCH * 4);
        if (pr < nrn) asm volatile("prefetch.global.L2 [%0];" ::"l"(un + pr * ld + pl * 64) : "memory");
      }
    }
    // ---- stage the batch: lane l keeps 16 B of every 512-B chunk ----
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nr) {
#pragma unroll
        for (int j = 0; j < NCH; ++j) cp_async16(sbase + r * kRowBytes + j * 512, ub + r * ld + j * 256 + lane * 8);
      }
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");

    // ---- row scales: mean |u| over the first NS chunks (steering only) ----
    int ssi = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nr) {
        __half2 acc = __float2half2_rn(0.f);
        const __half2 sc = __float2half2_rn(0.015625f);
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          const uint4 v = lds128(sbase + r * kRowBytes + j * 512);
          acc = __hfma2(__habs2(h2(v.x)), sc, acc);
          acc = __hfma2(__habs2(h2(v.y)), sc, acc);
          acc = __hfma2(__habs2(h2(v.z)), sc, acc);
          acc = __hfma2(__habs2(h2(v.w)), sc, acc);
        }
        const float ss = (__low2float(acc) + __high2float(acc)) * 64.f;
        const int tot = (int)redux_add((unsigned)min(__float2int_rn(ss * 1024.f), 1 << 26));
        if (lane == r) ssi = tot;
      }
    }
    const float rms = (float)ssi * (inv_ns * (1.f / 1024.f));

    // ---- lane r: search state of row r ----
    const bool owner = lane < nr;
    uint32_t lo = 0u, hi = kEnd, Tk = 0u;
    unsigned clo = 256u * NCH + kF16Bias, chi = kF16Bias;
    bool exact = false, done = !owner;
    const uint32_t p1 =
        min(max((uint32_t)__half_as_ushort(__float2half_rn(rms * ratio)) & 0x7fffu, 1u), 0x7bffu);
    uint32_t c = p1;
    unsigned n1 = xb, sec = 6u;
    float islope = slope;
    bool first = true;
    unsigned act = __ballot_sync(kFull, !done);
    while (act != 0u) {
      unsigned cnt = 0u;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (act & (1u << r)) {
          const uint32_t c2 = dup16(__shfl_sync(kFull, c, r));
          uint32_t w[NW];
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            const uint4 v = lds128(sbase + r * kRowBytes + j * 512);
            w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
          }
          const unsigned cr = f16_count_ge<NW>(w, c2);
          if (lane == r) cnt = cr;
        }
      }
      if (!done) {
        if (first) {
          // the probe at the predicted T*, then a step by the learned slope
          n1 = cnt;
          if (n1 == xb) { Tk = p1; exact = true; done = true; }
          else {
            const bool up1 = n1 > xb;
            lo = up1 ? p1 : 0u; clo = up1 ? n1 : clo;
            hi = up1 ? kEnd : p1; chi = up1 ? chi : n1;
            c = (uint32_t)((int)p1 + __float2int_rn((float)(int)(n1 - xb) * slope));
            c = (int)c <= (int)lo ? lo + 1u : min(c, hi - 1u);
          }
        } else {
          exact = cnt == xb;
          const bool up_ = cnt > xb;
          Tk = c;
          lo = up_ ? c : lo;
          clo = up_ ? cnt : clo;
          hi = up_ ? hi : c;
          chi = up_ ? chi : cnt;
          if (exact || hi - lo <= 1u) done = true;
          else if (hi == kEnd || lo == 0u) {
            const uint32_t s = (uint32_t)(((float)(hi == kEnd ? clo - xb : xb - chi) + 0.5f) * islope) + 1u;
            c = hi == kEnd ? lo + s : (hi > s ? hi - s : 0u);
            c = min(max(c, lo + 1u), hi - 1u);
            islope *= 2.f;
          } else if (sec == 0u) {
            c = lo + ((hi - lo) >> 1);
            sec = 1u;
          } else {
            const float f = ((float)(clo - xb) + UQ_ENC16_OFF) * rcp_approx((float)(clo - chi));
            c = lo + (uint32_t)(f * (float)(hi - lo));
            c = min(max(c, lo + 1u), hi - 1u);
            --sec;
          }
        }
      }
      first = false;
      act = __ballot_sync(kFull, !done);
    }
    if (owner) {
      if (!exact) { Tk = lo; exact = (clo == xb); }
      if (Tk != 0u && rms > 0.f) {
        const float rn = __fdividef(ElemBits<__half>::key2f(Tk), rms);
        if (rn > 0.f && rn < 1e30f) ratio = fmaf(UQ_ENC16_EMA, rn - ratio, ratio);
      }
      if (n1 != xb) {
        const float so = (float)abs((int)Tk - (int)p1) * rcp_approx((float)abs((int)(n1 - xb)));
        slope = fmaf(UQ_ENC16_SLOPE_EMA, min(so, 4096.f) - slope, slope);
      }
    }

    // ---- plane bytes, row by row ----
    const uint32_t tkx = Tk | (exact ? 0x80000000u : 0u);
    uint8_t* cp = codes + row0 * cb;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nr) {
        const uint32_t tr = __shfl_sync(kFull, tkx, r);
        const uint32_t Tr = tr & 0x7fffffffu;
        uint32_t w[NW];
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const uint4 v = lds128(sbase + r * kRowBytes + j * 512);
          w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
        }
        uint32_t posb[NCH], negb[NCH];
        if ((tr >> 31) != 0u || Tr == 0u) {
          const uint32_t ts = (Tr == 0u) ? 1u : Tr;
          const __half2 tp = h2(dup16(ts)), tn = h2(dup16(ts | 0x8000u));
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            posb[j] = bits8_bf(__hge2(h2(w[4 * j]), tp), __hge2(h2(w[4 * j + 1]), tp),
                               __hge2(h2(w[4 * j + 2]), tp), __hge2(h2(w[4 * j + 3]), tp));
            negb[j] = bits8_bf(__hle2(h2(w[4 * j]), tn), __hle2(h2(w[4 * j + 1]), tn),
                               __hle2(h2(w[4 * j + 2]), tn), __hle2(h2(w[4 * j + 3]), tn));
          }
        } else {
          // ties at T*: keys > T plus the first x - count(> T) keys == T in index order (R1)
          const __half2 tp = h2(dup16(Tr)), tn = h2(dup16(Tr | 0x8000u));
          int need = (int)(xb - __shfl_sync(kFull, chi, r));
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            const uint32_t gp = mask8(__hgt2_mask(h2(w[4 * j]), tp), __hgt2_mask(h2(w[4 * j + 1]), tp),
                                      __hgt2_mask(h2(w[4 * j + 2]), tp), __hgt2_mask(h2(w[4 * j + 3]), tp)) & 0xffu;
            const uint32_t gn = mask8(__hlt2_mask(h2(w[4 * j]), tn), __hlt2_mask(h2(w[4 * j + 1]), tn),
                                      __hlt2_mask(h2(w[4 * j + 2]), tn), __hlt2_mask(h2(w[4 * j + 3]), tn)) & 0xffu;
            const uint32_t ep = mask8(__heq2_mask(h2(w[4 * j]), tp), __heq2_mask(h2(w[4 * j + 1]), tp),
                                      __heq2_mask(h2(w[4 * j + 2]), tp), __heq2_mask(h2(w[4 * j + 3]), tp)) & 0xffu;
            const uint32_t en = mask8(__heq2_mask(h2(w[4 * j]), tn), __heq2_mask(h2(w[4 * j + 1]), tn),
                                      __heq2_mask(h2(w[4 * j + 2]), tn), __heq2_mask(h2(w[4 * j + 3]), tn)) & 0xffu;
            uint32_t eq = ep | en;
            const int ce = __popc(eq);
            int incl = ce;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int tv = __shfl_up_sync(kFull, incl, o);
              if (lane >= o) incl += tv;
            }
            const int take = min(max(need - (incl - ce), 0), ce);
            while (__popc(eq) > take) eq &= ~(0x80000000u >> __clz(eq));
            need -= __shfl_sync(kFull, incl, 31);
            posb[j] = gp | (eq & ep);
            negb[j] = gn | (eq & en);
          }
        }
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          cp[r * cb + 32 * j + lane] = (uint8_t)posb[j];
          cp[r * cb + pb + 32 * j + lane] = (uint8_t)negb[j];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// f32 rows (c2-c4 DB encodes): the f16 kernel's structure on the f32 search.
// The generic kernel spent ~850 warp instructions per d=768 row (ncu: ALU pipe
// 78%, issue 77%; profiles/r02/enc_f32_*).  Here:
//  * raw words keep their signs; the coarse keys (top 16 bits of |u|, compared
//    as f16 patterns, clamped below the f16 inf pattern) come from one PRMT +
//    HMNMX2(|.|) per two elements;
//  * the coarse search is the f16 kernel's (biased HSET2/HADD2 counts,
//    key-space interpolation, slope extrapolation when T* is outside the
//    probes); coarse(a) > coarse(b) => key(a) > key(b), so it brackets T*
//    exactly, and only a one-coarse-value bracket (a few elements) goes to
//    full 32-bit counts (abs keys built once, on demand);
//  * selection by signed integer compares of the raw bits (u >= T as int32:
//    +1; u >= T | 2^31 as uint32: -1), one nibble per plane per chunk;
//  * lane pairs swap nibbles with one shuffle per chunk; even lanes store the
//    + plane byte, odd lanes the - plane byte (one store per chunk per warp).
template <int NCH, bool VECLOAD, bool FULL>
__global__ void __launch_bounds__(kEncWarps * 32, NCH > 8 ? 2 : 3)
encode_f32_kernel(const float* __restrict__ u, int64_t n, int32_t d, int64_t ld, int32_t x, float z0, float delta,
                  float slope0, uint8_t* __restrict__ codes) {
  constexpr int E = 4 * NCH;                  // elements per lane
  constexpr int NWC = 2 * NCH;                // coarse half pairs per lane
  constexpr int NS = NCH < 2 ? NCH : NCH / 2; // chunks sampled for the RMS
  constexpr uint32_t kCEnd = 0x7c00u;         // coarse keys are <= 0x7bff
  const int lane = threadIdx.x & 31;
  const int64_t pb = FULL ? 16 * NCH : plane_bytes(d);
  const int64_t cb = 2 * pb;
  const int64_t warp_global = (int64_t)blockIdx.x * kEncWarps + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kEncWarps;
  const float inv_ns = 1.0f / (float)min(d, 128 * NS);
  const unsigned xb = (unsigned)x + kF16Bias;
  const int64_t ustep = nwarps * ld, cstep = nwarps * cb;
  float ratio = z0;   // T* / RMS, averaged over this warp's rows
  float slope = slope0;   // coarse keys per unit of count near T*, averaged over this warp's rows
  auto load_row = [&](const float* src, uint4 (&r)[NCH]) {
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      if constexpr (FULL) r[j] = __ldg(reinterpret_cast<const uint4*>(src + j * 128 + lane * 4));
      else r[j] = load_chunk<float, VECLOAD>(src, j * 128 + lane * 4, d);
    }
  };
  const bool pf_lane = VECLOAD && lane * 32 < d;   // one 128-byte line per lane

  uint4 raw[NCH];
  const float* up = u + warp_global * ld;
  uint8_t* cp = codes + warp_global * cb;
  if (warp_global < n) load_row(up, raw);
  for (int64_t row = warp_global; row < n; row += nwarps, up += ustep, cp += cstep) {
    if (pf_lane && row + 2 * nwarps < n)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(up + 2 * ustep + lane * 32) : "memory");
    uint32_t r[E];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      r[4 * j] = raw[j].x; r[4 * j + 1] = raw[j].y; r[4 * j + 2] = raw[j].z; r[4 * j + 3] = raw[j].w;
    }
    // ---- RMS estimate (FFMA; steering only) ----
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 4 * NS; ++i) ss = fmaf(__uint_as_float(r[i]), __uint_as_float(r[i]), ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
    ss *= inv_ns;
    const float rms = (ss > 0.f) ? ss * rsqrt_approx(ss) : 0.f;

    // ---- coarse keys: u rounded toward zero to f16 (one F2FP per two elements;
    // RZ never overflows to inf).  |coarse(u)| >= c <=> |u| >= f16 value c, so
    // a coarse threshold c is the full-key threshold f32bits(c). ----
    uint32_t cw[NWC];
#pragma unroll
    for (int i = 0; i < NWC; ++i)
      cw[i] = h2_bits(__halves2half2(__float2half_rz(__uint_as_float(r[2 * i])),
                                     __float2half_rz(__uint_as_float(r[2 * i + 1]))));

    // ---- coarse search: count(>= lo) >= x > count(>= hi) (biased counts) ----
    uint32_t lo = 0u, hi = kCEnd, Tk = 0u;
    unsigned clo = 128u * NCH + kF16Bias, chi = kF16Bias;
    bool exact = false;
#if UQ_ENC16_ONEPROBE
    // one probe at the predicted T*, then a step by the warp's learned slope
    // (as the f16 kernel)
    uint32_t p1;
    unsigned n1;
    {
      p1 = min(max((uint32_t)__half_as_ushort(__float2half_rn(rms * ratio)) & 0x7fffu, 1u), 0x7bffu);
      n1 = f16_count_ge<NWC>(cw, dup16(p1));
      float islope = slope;
      uint32_t c = p1;
      if (n1 == xb) { Tk = p1; exact = true; }
      else {
        const bool up1 = n1 > xb;
        lo = up1 ? p1 : 0u; clo = up1 ? n1 : clo;
        hi = up1 ? kCEnd : p1; chi = up1 ? chi : n1;
        c = (uint32_t)((int)p1 + __float2int_rn((float)(int)(n1 - xb) * slope));
        c = (int)c <= (int)lo ? lo + 1u : min(c, hi - 1u);
      }
      unsigned sec = 6u;
#pragma unroll 1
      while (!exact) {
        const unsigned cnt = f16_count_ge<NWC>(cw, dup16(c));
        exact = cnt == xb;
        const bool up_ = cnt > xb;
        Tk = c;
        lo = up_ ? c : lo;
        clo = up_ ? cnt : clo;
        hi = up_ ? hi : c;
        chi = up_ ? chi : cnt;
        if (exact || hi - lo <= 1u) break;
        if (hi == kCEnd || lo == 0u) {
          const uint32_t s = (uint32_t)(((float)(hi == kCEnd ? clo - xb : xb - chi) + 0.5f) * islope) + 1u;
          c = hi == kCEnd ? lo + s : (hi > s ? hi - s : 0u);
          c = min(max(c, lo + 1u), hi - 1u);
          islope *= 2.f;
        } else if (sec == 0u) {
          c = lo + ((hi - lo) >> 1);
          sec = 1u;
        } else {
          const float f = ((float)(clo - xb) + 0.5f) * rcp_approx((float)(clo - chi));
          c = lo + (uint32_t)(f * (float)(hi - lo));
          c = min(max(c, lo + 1u), hi - 1u);
          --sec;
        }
      }
      // coarse keys per count between the probe and the coarse result
      // (steering only)
      if (n1 != xb) {
        const float so = (float)abs((int)Tk - (int)p1) * rcp_approx((float)abs((int)(n1 - xb)));
        slope = fmaf(UQ_ENC16_SLOPE_EMA, min(so, 4096.f) - slope, slope);
      }
    }
#else
    float islope;
    {
      const float t = rms * ratio;
      const uint32_t pp = __vminu2(__vmaxu2(h2_bits(__floats2half2_rn(t * (1.f - delta), t * (1.f + delta))) & 0x7fff7fffu,
                                            0x00010001u), 0x7bff7bffu);
      const uint32_t p1 = pp & 0xffffu;
      const uint32_t p2 = max(pp >> 16, p1 + 1u);
      const unsigned n1 = f16_count_ge<NWC>(cw, dup16(p1));
      const unsigned n2 = f16_count_ge<NWC>(cw, dup16(p2));
      islope = (float)(p2 - p1) * rcp_approx((float)max(n1 - n2, 1u));
      if (n1 == xb) { Tk = p1; exact = true; }
      else if (n2 == xb) { Tk = p2; exact = true; }
      else if (n2 > xb) { lo = p2; clo = n2; }
      else if (n1 > xb) { lo = p1; clo = n1; hi = p2; chi = n2; }
      else { hi = p1; chi = n1; }
    }
    {
      unsigned sec = 6u;
#pragma unroll 1
      while (!exact && hi - lo > 1u) {
        uint32_t c;
        if (hi == kCEnd || lo == 0u) {
          const uint32_t s = (uint32_t)(((float)(hi == kCEnd ? clo - xb : xb - chi) + 0.5f) * islope) + 1u;
          c = hi == kCEnd ? lo + s : (hi > s ? hi - s : 0u);
          c = min(max(c, lo + 1u), hi - 1u);
          islope *= 2.f;
        } else if (sec == 0u) {
          c = lo + ((hi - lo) >> 1);
          sec = 1u;
        } else {
          const float f = ((float)(clo - xb) + 0.5f) * rcp_approx((float)(clo - chi));
          c = lo + (uint32_t)(f * (float)(hi - lo));
          c = min(max(c, lo + 1u), hi - 1u);
          --sec;
        }
        const unsigned cnt = f16_count_ge<NWC>(cw, dup16(c));
        exact = cnt == xb;
        const bool up_ = cnt > xb;
        Tk = c;
        lo = up_ ? c : lo;
        clo = up_ ? cnt : clo;
        hi = up_ ? hi : c;
        chi = up_ ? chi : cnt;
      }
    }
    #endif
    auto c2key = [](uint32_t c) { return __float_as_uint(__half2float(__ushort_as_half((unsigned short)c))); };
    if (exact) {
      Tk = c2key(Tk);                 // keys >= f32(Tc) <=> coarse >= Tc: exactly x of them
    } else {
      // ---- full keys inside one coarse value: [f32(lc), f32(hc)) ----
      const unsigned xu = (unsigned)x;
      uint32_t flo = c2key(lo), fhi = (hi == kCEnd) ? 0x80000000u : c2key(hi);
      unsigned fclo = clo - kF16Bias, fchi = (hi == kCEnd) ? 0u : chi - kF16Bias;
      uint32_t kk[E];
#pragma unroll
      for (int e = 0; e < E; ++e) kk[e] = r[e] & 0x7fffffffu;
      unsigned sec = 3u;
#pragma unroll 1
      while (!exact && fhi - flo > 1u) {
        uint32_t c;
        if (sec == 0u || fhi == 0x80000000u) {
          c = flo + ((fhi - flo) >> 1);
          sec = 1u;
        } else {
          const float f = ((float)(fclo - xu) + 0.5f) * rcp_approx((float)(fclo - fchi));
          c = flo + (uint32_t)(f * (float)(fhi - flo));
          c = min(max(c, flo + 1u), fhi - 1u);
          --sec;
        }
        unsigned a0 = 0u, a1 = 0u;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          a0 = add_lt(a0, kk[e], c);
          a1 = add_lt(a1, kk[e + 1], c);
        }
        const unsigned cnt = __reduce_add_sync(kFull, (unsigned)E - a0 - a1);
        exact = cnt == xu;
        const bool up_ = cnt > xu;
        Tk = c;
        flo = up_ ? c : flo;
        fclo = up_ ? cnt : fclo;
        fhi = up_ ? fhi : c;
        fchi = up_ ? fchi : cnt;
      }
      if (!exact) { Tk = flo; exact = (fclo == xu); chi = fchi; }
    }
    if (Tk != 0u && rms > 0.f) {
      const float rn = __fdividef(__uint_as_float(Tk), rms);
      if (rn > 0.f && rn < 1e30f) ratio = fmaf(0.3f, rn - ratio, ratio);
    }

    // ---- nibbles (bits 0-3: +1 where u >= T; bits 4-7: -1 where u <= -T) ----
    uint32_t nib[NCH];
    // step(u >= T) = sat((u - Tp) * S) with Tp the float below T and S = 1 /
    // ulp(Tp) (a power of two; Tp * S is Tp's integer significand, exact):
    // 0 for u <= Tp, >= 1 before saturation for u >= T (one FFMA rounding).
    // Nibble bytes are weighted sums 2^23 + sum step * 2^c (exact), whose low
    // byte is the bit pattern: FMA-pipe work instead of ALU compares.  Needs
    // Tp normal with biased exponent >= 23 (S <= 2^127); else integer compares.
    const uint32_t tpb = ((Tk == 0u) ? 1u : Tk) - 1u;
    const uint32_t tpe = tpb >> 23;
    if ((exact || Tk == 0u) && tpe >= 23u && tpe <= 254u) {
      const float S = __uint_as_float((277u - tpe) << 23);
      const float nts = -__uint_as_float(tpb) * S;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        float acc = 8388608.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float v = __uint_as_float(r[4 * j + c]);
          acc = fmaf(__saturatef(fmaf(v, S, nts)), (float)(1 << c), acc);
          acc = fmaf(__saturatef(fmaf(-v, S, nts)), (float)(16 << c), acc);
        }
        nib[j] = __float_as_uint(acc);   // low byte: + bits 0-3, - bits 4-7
      }
    } else if (exact || Tk == 0u) {
      const int32_t ti = (int32_t)((Tk == 0u) ? 1u : Tk);
      const uint32_t tn = (uint32_t)ti | 0x80000000u;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        uint32_t v = 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          v |= ((int32_t)r[4 * j + c] >= ti ? 1u : 0u) << c;
          v |= (r[4 * j + c] >= tn ? 1u : 0u) << (4 + c);
        }
        nib[j] = v;
      }
    } else {
      // ties at T (count(> T) = chi < x < count(>= T)): keys > T plus the
      // first x - chi keys == T in index order (chunk, lane, element; R1)
      const int32_t ti = (int32_t)Tk;
      const uint32_t tn = Tk | 0x80000000u;
      int need = (int)((unsigned)x - chi);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        uint32_t g = 0u, eq = 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t v = r[4 * j + c];
          g |= ((int32_t)v > ti ? 1u : 0u) << c;
          g |= (v > tn ? 1u : 0u) << (4 + c);
          eq |= (v == (uint32_t)ti ? 1u : 0u) << c;
          eq |= (v == tn ? 1u : 0u) << (4 + c);
        }
        uint32_t e4 = (eq | (eq >> 4)) & 0xfu;      // positions with |u| == T
        const int ce = __popc(e4);
        int incl = ce;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int tv = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += tv;
        }
        const int take = min(max(need - (incl - ce), 0), ce);
        while (__popc(e4) > take) e4 &= ~(0x80000000u >> __clz(e4));
        need -= __shfl_sync(kFull, incl, 31);
        nib[j] = g | (eq & (e4 | (e4 << 4)));
      }
    }
    // ---- store: lane pairs swap nibbles; even lanes write +, odd lanes - ----
    {
      const bool odd = lane & 1;
      uint8_t* dst = cp + (odd ? pb : 0) + (lane >> 1);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const uint32_t o = __shfl_xor_sync(kFull, nib[j], 1);
        const uint32_t b = odd ? ((o >> 4) & 0xfu) | (nib[j] & 0xf0u) : (nib[j] & 0xfu) | ((o & 0xfu) << 4);
        if (FULL || 16 * j + (lane >> 1) < pb) dst[16 * j] = (uint8_t)b;
      }
    }
    if (row + nwarps < n) load_row(up + ustep, raw);
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
  // probe half-width: the probes bracket T* unless the predicted T* / RMS
  // ratio is off by more than delta (steering only; UQ_ENC_DELTA overrides).
  // Measured optimum (tools/enc_bench.py over delta in 0.02-0.30,
  // profiles/r02/enc_delta_scan.txt): 0.12 for f32 (coarse phase), 0.08 for
  // 16-bit keys.
  static const float delta_env = [] {
    const char* e = getenv("UQ_ENC_DELTA");
    return e ? (float)atof(e) : 0.f;
  }();
  const float delta = delta_env > 0.f ? delta_env : (sizeof(T) == 4 ? 0.03f : std::is_same<T, __half>::value ? 0.03f : 0.08f);
  // initial f16 keys per unit of count near T* for d half-normal magnitudes
  // of scale s: count density 2 d phi(z) / s per unit value, ~T* 2^-10.5 per
  // key (f16 ulp) at T* = s z -> 2^10.5 / (2 d phi(z) z); learned per warp
  // (the f16 search and the f32 coarse search)
  const double phz = std::exp(-0.5 * (double)z0 * (double)z0) * 0.3989422804014327;
  const float slope0 = (float)std::min(4096.0, std::max(0.25, 1448.15468787 / (2.0 * d * phz * (double)z0)));
  if constexpr (std::is_same<T, __half>::value) {
    z0 *= 1.2533141f;   // the f16 kernel steers by mean |u| = s * sqrt(2 / pi) for N(0, s^2)
#if UQ_ENC16_BATCH
    if constexpr (NCH <= 4) {
      // large n: the batched kernel (R rows per warp iteration, lane-parallel
      // search control); small n keeps one row per warp (more warps in flight)
      constexpr int R = NCH <= 3 ? UQ_ENC16_BATCH_R : (UQ_ENC16_BATCH_R < 4 ? UQ_ENC16_BATCH_R : 4);
      constexpr int kSmem = kEncWarps * R * 512 * NCH;
      constexpr int kCtas = R >= 8 ? 2 : 4;
      if (vec && d == 256 * NCH && n >= (int64_t)sms * kCtas * kEncWarps * R) {
        static const cudaError_t attr = cudaFuncSetAttribute(encode_f16_batch_kernel<NCH, R>,
                                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (attr != cudaSuccess) return attr;
        const int64_t nb = (n + R - 1) / R;
        const int64_t bl = std::min<int64_t>((nb + kEncWarps - 1) / kEncWarps, (int64_t)sms * kCtas);
        encode_f16_batch_kernel<NCH, R><<<(unsigned)bl, kEncWarps * 32, kSmem, st>>>(
            (const __half*)u, n, ld, x, z0, slope0, codes);
        note_launch();
        return cudaGetLastError();
      }
    }
#endif
    if (vec && d == 256 * NCH)
      encode_f16_kernel<NCH, true, true><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
          (const __half*)u, n, d, ld, x, z0, delta, slope0, codes);
    else if (vec)
      encode_f16_kernel<NCH, true, false><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
          (const __half*)u, n, d, ld, x, z0, delta, slope0, codes);
    else
      encode_f16_kernel<NCH, false, false><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
          (const __half*)u, n, d, ld, x, z0, delta, slope0, codes);
    note_launch();
    return cudaGetLastError();
  }
  if constexpr (std::is_same<T, float>::value) {
    if (vec && d == 128 * NCH)
      encode_f32_kernel<NCH, true, true><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
          (const float*)u, n, d, ld, x, z0, delta, slope0, codes);
    else if (vec)
      encode_f32_kernel<NCH, true, false><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
          (const float*)u, n, d, ld, x, z0, delta, slope0, codes);
    else
      encode_f32_kernel<NCH, false, false><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
          (const float*)u, n, d, ld, x, z0, delta, slope0, codes);
    note_launch();
    return cudaGetLastError();
  }
  if (vec)
    encode_kernel<T, NCH, true><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
        (const T*)u, n, d, ld, x, z0, delta, codes);
  else
    encode_kernel<T, NCH, false><<<(unsigned)blocks, kEncWarps * 32, 0, st>>>(
        (const T*)u, n, d, ld, x, z0, delta, codes);
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
