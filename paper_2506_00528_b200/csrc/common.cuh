// common.cuh -- shared device/host helpers of libuq (product path; shares
// nothing with oracle/).  Citations: P:NNN = PAPER.md line.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/uq.h"

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
// 32-bit local keys in global memory plus a threshold `thr`: a new key enters
// only if key > thr, where thr is the k-th largest key retained so far (0
// while fewer than k keys exist).  A key <= thr can never reach the stream's
// final top-k because k distinct larger keys are already retained.
//
// rebuild(): the whole warp (all 32 lanes, converged) finds T = k-th largest
// of the cnt buffered keys by bisection over the 32 key bits, then compacts the
// keys >= T (exactly k of them: keys are unique) to the buffer front.  Returns
// the new threshold; the new count is min(cnt, k).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t warp_count_ge(const uint32_t* buf, int cnt, uint32_t t, int lane) {
  int c = 0;
  for (int i = lane; i < cnt; i += kWarp) c += (buf[i] >= t) ? 1 : 0;
  return __reduce_add_sync(kFull, (unsigned)c);
}

__device__ inline uint32_t stream_rebuild(uint32_t* buf, int cnt, int k, int lane) {
  if (cnt <= k) return 0u;  // fewer than k candidates: keep all, accept everything
  uint32_t T = 0;
  for (int b = 31; b >= 0; --b) {
    uint32_t cand = T | (1u << b);
    uint32_t c = warp_count_ge(buf, cnt, cand, lane);
    if (c >= (uint32_t)k) {
      T = cand;
      if (c == (uint32_t)k) break;  // exactly k keys >= cand: cand is a valid cut
    }
  }
  // compact keys >= T to the front (write index <= read index: in-place safe)
  int w = 0;
  uint32_t kmin = 0xffffffffu;
  for (int base = 0; base < cnt; base += kWarp) {
    int i = base + lane;
    uint32_t key = (i < cnt) ? buf[i] : 0u;
    bool keep = (i < cnt) && key >= T;
    unsigned bal = __ballot_sync(kFull, keep);
    __syncwarp();
    if (keep) {
      buf[w + __popc(bal & lanemask_lt())] = key;
      kmin = min(kmin, key);
    }
    w += __popc(bal);
    __syncwarp();
  }
  // w == k here.  Threshold for future keys: the smallest retained key.
  return __reduce_min_sync(kFull, kmin);
}

}  // namespace uq
