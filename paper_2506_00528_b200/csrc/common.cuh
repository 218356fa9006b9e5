// common.cuh -- shared device/host helpers of libuq (product path; shares
// nothing with oracle/).  Citations: P:NNN = PAPER.md line.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/uq.h"

// Device-side bounds checks of the CHECKED build (libuq_checked.so, built
// with -DUQ_CHECKED by `build.py --checked`; tools/sanitize.py runs every
// engine against it).  compute-sanitizer is not available on the GPU pool, so
// these asserts stand in for its memcheck on the accesses that matter: stream
// buffer appends, candidate-list writes, bulk-copy sources inside the index,
// shared-memory code buffers.  The product library compiles them out.
#ifdef UQ_CHECKED
#include <cstdio>
#define UQ_ASSERT(c)                                                                 \
  do {                                                                               \
    if (!(c)) {                                                                      \
      printf("UQ_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                     \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define UQ_ASSERT(c) \
  do {               \
  } while (0)
#endif

namespace uq {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// plane_bytes = 16 * ceil(d/128): 128-bit plane granularity (R6).
__host__ __device__ inline int64_t plane_bytes(int32_t d) { return 16 * (((int64_t)d + 127) / 128); }
__host__ __device__ inline int64_t code_bytes(int32_t d) { return 2 * plane_bytes(d); }
__host__ __device__ inline int blocks128(int32_t d) { return (d + 127) / 128; }

// ---------------------------------------------------------------------------
// Keys.  The ranking order is (Delta desc, id asc) (R7, R8); both
// key forms below are unsigned integers whose natural order IS that order, and
// 0 is reserved for "no entry".
//
// Local 32-bit key (inside one scan chunk of < 2^rb rows):
//     key = ((Delta + d + 1) << rb) | (2^rb - 1 - local_row),  sb + rb = 32,
//     sb = bit length of 2d+1, so Delta + d + 1 in [1, 2d+1] never collides
//     with 0.  Unique per row.
// Global 64-bit key (across chunks / GPUs, row < 2^32 - 1):
//     key = ((uint32(Delta) ^ 0x80000000) << 32) | (0xFFFFFFFF - row).
// ---------------------------------------------------------------------------
struct KeyFmt {
  int32_t off;    // d + 1
  int32_t rb;     // row bits
  uint32_t rmask; // 2^rb - 1
};

__host__ __device__ inline int bitlen(uint32_t v) {
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

inline KeyFmt make_keyfmt(int32_t d) {
  KeyFmt f;
  f.off = d + 1;
  f.rb = 32 - bitlen((uint32_t)(2 * d + 1));
  f.rmask = (f.rb >= 32) ? 0xffffffffu : ((1u << f.rb) - 1u);
  return f;
}

__device__ __forceinline__ uint32_t local_key(const KeyFmt& f, int32_t delta, uint32_t local_row) {
  return ((uint32_t)(delta + f.off) << f.rb) | (f.rmask - local_row);
}

// base[i] = v where p, as one predicated store (no branch, no reconvergence);
// the address is one wide multiply-add of the 32-bit index
__device__ __forceinline__ void st_global_if(uint32_t* base, uint32_t i, uint32_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\t.reg .u64 a;\n\tsetp.ne.u32 q, %3, 0;\n\t"
               "mad.wide.u32 a, %1, 4, %0;\n\t@q st.global.u32 [a], %2;\n\t}"
               ::"l"(base), "r"(i), "r"(v), "r"((uint32_t)p) : "memory");
}

// *ptr += v where p, one predicated global reduction (no branch)
__device__ __forceinline__ void red_global_add_if(uint32_t* ptr, uint32_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.global.add.u32 [%0], %1;\n\t}"
               ::"l"(ptr), "r"(v), "r"((uint32_t)p) : "memory");
}
// shared [addr] += v where p, one predicated reduction (no branch)
__device__ __forceinline__ void red_shared_add_if(uint32_t addr, uint32_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}"
               ::"r"(addr), "r"(v), "r"((uint32_t)p) : "memory");
}

__device__ __forceinline__ uint64_t global_key_from_local(const KeyFmt& f, uint32_t lk, uint64_t chunk_start) {
  if (lk == 0) return 0ull;
  int32_t delta = (int32_t)(lk >> f.rb) - f.off;
  uint64_t row = chunk_start + (uint64_t)(f.rmask - (lk & f.rmask));
  return ((uint64_t)((uint32_t)delta ^ 0x80000000u) << 32) | (uint64_t)(0xffffffffu - (uint32_t)row);
}

__device__ __forceinline__ uint64_t global_key(int32_t score, int64_t id) {
  if (id < 0) return 0ull;
  return ((uint64_t)((uint32_t)score ^ 0x80000000u) << 32) | (uint64_t)(0xffffffffu - (uint32_t)id);
}

__device__ __forceinline__ int32_t key_score(uint64_t k) { return (int32_t)((uint32_t)(k >> 32) ^ 0x80000000u); }
__device__ __forceinline__ int64_t key_row(uint64_t k) { return (int64_t)(0xffffffffu - (uint32_t)k); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// Warp-cooperative "stream" selector.  A stream is a candidate buffer of
// 32-bit local keys in global memory plus a threshold: a new key enters only
// if it beats the k-th best key retained so far (everything while fewer than
// k are retained).  A key that does not can never reach the stream's final
// top-k, because k distinct better keys already exist.
//
// A rebuild cuts a buffer of cnt > k keys back to exactly its k best.  The
// whole warp cooperates (all 32 lanes converged); the keys are loaded into
// registers once (lane l holds buffer entries l, l+32, ...), so the selection
// costs no memory round trips beyond one load and one store per key.
// ---------------------------------------------------------------------------
template <int MAXR>
__device__ __forceinline__ void stream_load(const uint32_t* buf, int cnt, int lane, uint32_t (&r)[MAXR]) {
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    const int idx = i * kWarp + lane;
    r[i] = (idx < cnt) ? buf[idx] : 0u;
  }
}

// General stream (keys appended in any row order): T = k-th largest key by
// bisection over the 32 key bits; keep the keys >= T (exactly k: keys are
// unique).  Returns the smallest retained key (the new threshold: pass iff
// key > thr).
template <int MAXR>
__device__ uint32_t stream_rebuild_regs(uint32_t* buf, int cnt, int k, int lane) {
  uint32_t r[MAXR];
  stream_load<MAXR>(buf, cnt, lane, r);
  uint32_t T = 0;
#pragma unroll 1
  for (int b = 31; b >= 0; --b) {
    const uint32_t cand = T | (1u << b);
    unsigned c = 0;
#pragma unroll
    for (int i = 0; i < MAXR; ++i) c += (r[i] >= cand) ? 1u : 0u;
    const unsigned tot = __reduce_add_sync(kFull, c);
    if (tot >= (unsigned)k) {
      T = cand;
      if (tot == (unsigned)k) break;  // exactly k keys >= cand: a valid cut
    }
  }
  int w = 0;
  uint32_t kmin = 0xffffffffu;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    const bool keep = (i * kWarp + lane < cnt) && r[i] >= T;
    const unsigned bal = __ballot_sync(kFull, keep);
    if (keep) {
      buf[w + __popc(bal & lanemask_lt())] = r[i];
      kmin = min(kmin, r[i]);
    }
    w += __popc(bal);
  }
  __syncwarp();
  return __reduce_min_sync(kFull, kmin);
}

// Ordered stream (one producer appending rows in increasing order, e.g. one
// query per thread scanning its chunk front to back): the buffer order is the
// row order, so among equal Delta the earlier entries win.  D = k-th largest
// Delta field (key >> rb) by bisection over the sb field bits; keep every key
// with field > D plus the first (k - #{field > D}) keys with field == D.
// Returns D: later keys pass iff their field > D (equal Delta, larger row).
template <int MAXR>
__device__ uint32_t ordered_rebuild_regs(uint32_t* buf, int cnt, int k, int lane, int rb) {
  uint32_t r[MAXR];
  stream_load<MAXR>(buf, cnt, lane, r);
  const int sb = 32 - rb;
  uint32_t D = 0;
#pragma unroll 1
  for (int b = sb - 1; b >= 0; --b) {
    const uint32_t cand = D | (1u << b);
    unsigned c = 0;
#pragma unroll
    for (int i = 0; i < MAXR; ++i) c += ((r[i] >> rb) >= cand) ? 1u : 0u;
    const unsigned tot = __reduce_add_sync(kFull, c);
    if (tot >= (unsigned)k) {
      D = cand;
      if (tot == (unsigned)k) break;
    }
  }
  unsigned gt = 0;
#pragma unroll
  for (int i = 0; i < MAXR; ++i) gt += ((r[i] >> rb) > D) ? 1u : 0u;
  const int m = k - (int)__reduce_add_sync(kFull, gt);  // entries with field == D to keep
  int w = 0, eq_seen = 0;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    const bool in = i * kWarp + lane < cnt;
    const uint32_t f = r[i] >> rb;
    const bool eq = in && f == D;
    const unsigned beq = __ballot_sync(kFull, eq);
    const bool keep = in && (f > D || (eq && eq_seen + __popc(beq & lanemask_lt()) < m));
    eq_seen += __popc(beq);
    const unsigned bal = __ballot_sync(kFull, keep);
    if (keep) buf[w + __popc(bal & lanemask_lt())] = r[i];
    w += __popc(bal);
  }
  __syncwarp();
  return D;
}

#define UQ_REBUILD_DISPATCH(FN, ...)                          \
  do {                                                        \
    UQ_ASSERT(cnt <= 48 * kWarp);                             \
    if (cnt <= 8 * kWarp) return FN<8>(__VA_ARGS__);          \
    if (cnt <= 16 * kWarp) return FN<16>(__VA_ARGS__);        \
    if (cnt <= 24 * kWarp) return FN<24>(__VA_ARGS__);        \
    if (cnt <= 32 * kWarp) return FN<32>(__VA_ARGS__);        \
    return FN<48>(__VA_ARGS__);                               \
  } while (0)

// cnt <= 48*32 = 1536 (= UQ_MAX_K + 2*256 buffer capacity)
__device__ __forceinline__ uint32_t stream_rebuild(uint32_t* buf, int cnt, int k, int lane) {
  UQ_REBUILD_DISPATCH(stream_rebuild_regs, buf, cnt, k, lane);
}
__device__ __forceinline__ uint32_t ordered_rebuild(uint32_t* buf, int cnt, int k, int lane, int rb) {
  UQ_REBUILD_DISPATCH(ordered_rebuild_regs, buf, cnt, k, lane, rb);
}
// Out-of-line form for kernels whose hot loops must stay small in the
// instruction cache (the five inlined MAXR variants are ~5k SASS instructions;
// the call is rare: about one cut per stream)
static __device__ __noinline__ uint32_t ordered_rebuild_call(uint32_t* buf, int cnt, int k, int lane, int rb) {
  UQ_REBUILD_DISPATCH(ordered_rebuild_regs, buf, cnt, k, lane, rb);
}

}  // namespace uq
