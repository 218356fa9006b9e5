// scan_popc.cu -- Delta scan on CUDA cores (LOP3 + POPC) with fused per-query
// top-k streams.
//
// Delta = b2sp(q, r) = (bsp(q+,r+) + bsp(q-,r-)) - (bsp(q+,r-) + bsp(q-,r+))
// (Sec. 5.1.2).  For valid codes (pos AND neg = 0) the identity
//     m = q+ | q-,  t = m & (r+ | r-),  u = t & (q- ^ r-),
//     Delta = popc(t) - 2 popc(u)
// holds word by word (t marks positions non-zero in both, u those whose signs
// differ), so each 32 dims cost 2 LOP3 + 2 POPC + adds instead of 4 AND + 4
// POPC.  Precondition documented in uq.h; uq_check_codes() verifies it.
//
// Layout: CTA = 8 warps; a work item = (query tile of <= QT_MAX queries,
// DB chunk of L rows).  The query tile sits in shared memory as (m, q-)
// planes and is read with warp-uniform (broadcast) LDS.128; each lane holds
// one DB row (both planes) in registers, so one DB row load serves every query
// of the tile.  Per query the CTA keeps one stream (common.cuh): candidates
// key > thr[q] are appended (warp-aggregated atomics on a shared counter) to a
// global-memory buffer; after every 256-row stage the buffers that exceed
// k + 256 entries are cut back to exactly k by one warp each.
#include <cuda.h>          // CUtensorMap (the encoder is fetched through the runtime: no -lcuda)
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace uq {

constexpr int kScanWarps = 8;
constexpr int kScanThreads = kScanWarps * 32;
constexpr int kStageRows = kScanThreads;  // one row per thread per stage
// stages between stream checks: up to 4, fewer for large k so that a buffer
// (k + (check + 1) stages of keys) stays within the stream cut's 1536 keys
static int popc_check(int32_t k) {
  const int c = (1536 - k) / kStageRows - 1;
  return c < 1 ? 1 : (c > 4 ? 4 : c);
}

struct PopcParams {
  const uint8_t* q;
  int64_t nq;
  const uint8_t* db;
  int64_t n;
  int32_t d;
  int32_t k;
  KeyFmt kf;
  int32_t qt;        // queries per tile
  int32_t n_qtiles;  // QT
  int64_t n_chunks;  // S
  int64_t L;         // rows per chunk (multiple of kStageRows)
  int32_t cap;       // stream buffer capacity (k + 2*kStageRows)
  uint32_t* bufs;    // [gridDim.x][qt][cap]
  uint64_t* part;    // [S][nq][k] global keys
  const int32_t* thr0;  // optional per-query seed D_k: rows with Delta < thr0[q * thr0_stride] cannot matter
  int32_t thr0_stride;
  int64_t row_stride;   // DB row r of this scan is row r * row_stride of dbcodes
  int32_t check;        // stages between stream checks (popc_check)
  int32_t* part_cnt;    // optional [S][nq]: valid entries per published list (the rest is left unwritten)
};

// Delta of this lane's DB row (dm = r+ | r-, dn = r-) against every query of
// the tile (broadcast LDS of the query planes), then the stream append: keys
// above the query's threshold are appended (warp-aggregated shared counter).
template <int NB>
__device__ __forceinline__ void popc_stage_queries(const PopcParams& p, const uint4 (&dm)[NB], const uint4 (&dn)[NB],
                                                   bool valid, int64_t lr, int nqt, const uint4* s_qm,
                                                   const uint4* s_qn, const uint32_t* s_thr, int* s_cnt,
                                                   uint32_t* mybufs, int lane) {
#pragma unroll 1
  for (int j = 0; j < nqt; ++j) {
    int a = 0, u2 = 0;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint4 m = s_qm[j * NB + b];
      const uint4 qn = s_qn[j * NB + b];
      uint32_t tt, uu;
      tt = m.x & dm[b].x; uu = tt & (qn.x ^ dn[b].x); a += __popc(tt); u2 += __popc(uu);
      tt = m.y & dm[b].y; uu = tt & (qn.y ^ dn[b].y); a += __popc(tt); u2 += __popc(uu);
      tt = m.z & dm[b].z; uu = tt & (qn.z ^ dn[b].z); a += __popc(tt); u2 += __popc(uu);
      tt = m.w & dm[b].w; uu = tt & (qn.w ^ dn[b].w); a += __popc(tt); u2 += __popc(uu);
    }
    const int delta = a - 2 * u2;
    const uint32_t key = valid ? local_key(p.kf, delta, (uint32_t)lr) : 0u;
    const bool pass = key > s_thr[j];
    const unsigned bal = __ballot_sync(kFull, pass);
    if (bal) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&s_cnt[j], __popc(bal));
      base = __shfl_sync(kFull, base, 0);
      UQ_ASSERT(!pass || base + __popc(bal) <= p.cap);
      if (pass) mybufs[(size_t)j * p.cap + base + __popc(bal & lanemask_lt())] = key;
    }
  }
}

// OCC: resident CTAs per SM the registers are capped for.  Few-query tiles
// (the HBM-bound case, e.g. Q = 1) keep fewer values live and gain from a
// third CTA's extra loads in flight; many-query tiles (POPC-bound) do not.
template <int NB, int OCC>
__global__ void __launch_bounds__(kScanThreads, OCC) scan_popc_kernel(PopcParams p) {
  extern __shared__ uint4 smem_u4[];
  uint4* s_qm = smem_u4;                              // [qt][NB]  q+ | q-
  uint4* s_qn = smem_u4 + (size_t)p.qt * NB;          // [qt][NB]  q-
  uint32_t* s_thr = reinterpret_cast<uint32_t*>(smem_u4 + 2 * (size_t)p.qt * NB);
  int* s_cnt = reinterpret_cast<int*>(s_thr + p.qt);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pb = (int64_t)NB * 16, cb = 2 * pb;
  uint32_t* mybufs = p.bufs + (size_t)blockIdx.x * p.qt * p.cap;
  const int64_t n_items = (int64_t)p.n_qtiles * p.n_chunks;

  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int t = (int)(item % p.n_qtiles);
    const int64_t c = item / p.n_qtiles;
    const int64_t q0 = (int64_t)t * p.qt;
    const int nqt = (int)(p.nq - q0 < (int64_t)p.qt ? p.nq - q0 : (int64_t)p.qt);
    const int64_t row0 = c * p.L;
    const int64_t rows = (p.n - row0 < p.L) ? p.n - row0 : p.L;

    __syncthreads();  // previous item fully done with shared state
    for (int i = threadIdx.x; i < nqt * NB; i += kScanThreads) {
      const uint8_t* qr = p.q + (q0 + i / NB) * cb + (i % NB) * 16;
      const uint4 a = *reinterpret_cast<const uint4*>(qr);
      const uint4 b = *reinterpret_cast<const uint4*>(qr + pb);
      s_qm[i] = make_uint4(a.x | b.x, a.y | b.y, a.z | b.z, a.w | b.w);
      s_qn[i] = b;
    }
    for (int j = threadIdx.x; j < nqt; j += kScanThreads) {
      uint32_t t0 = 0u;  // key > t0  <=>  Delta >= D_k (t0 has all row bits set)
      if (p.thr0) {
        const int32_t dk = p.thr0[(q0 + j) * p.thr0_stride];
        if (dk != INT32_MIN && dk - 1 + p.kf.off >= 0) t0 = ((uint32_t)(dk - 1 + p.kf.off) << p.kf.rb) | p.kf.rmask;
      }
      s_thr[j] = t0;
      s_cnt[j] = 0;
    }
    __syncthreads();

    for (int64_t s0 = 0; s0 < rows; s0 += kStageRows) {
      const int64_t lr = s0 + warp * 32 + lane;  // local row inside the chunk
      const bool valid = lr < rows;
      // dm = r+ | r- and dn = r- of this lane's row, in registers
      uint4 dm[NB], dn[NB];
      if (valid) {
        const uint8_t* rr = p.db + (row0 + lr) * p.row_stride * cb;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const uint4 dp = __ldg(reinterpret_cast<const uint4*>(rr) + b);
          dn[b] = __ldg(reinterpret_cast<const uint4*>(rr + pb) + b);
          dm[b] = make_uint4(dp.x | dn[b].x, dp.y | dn[b].y, dp.z | dn[b].z, dp.w | dn[b].w);
        }
      } else {
#pragma unroll
        for (int b = 0; b < NB; ++b) { dm[b] = make_uint4(0, 0, 0, 0); dn[b] = dm[b]; }
      }

      popc_stage_queries<NB>(p, dm, dn, valid, lr, nqt, s_qm, s_qn, s_thr, s_cnt, mybufs, lane);
      // streams are checked (and cut back to k) every p.check stages: the
      // buffers hold k + (check + 1) stages of keys, and the stages in
      // between run without CTA barriers
      if ((s0 / kStageRows) % p.check == p.check - 1 || s0 + kStageRows >= rows) {
        __syncthreads();
        for (int j = warp; j < nqt; j += kScanWarps) {
          const int cnt = s_cnt[j];
          if (cnt > p.k + kStageRows) {
            const uint32_t thr = stream_rebuild(mybufs + (size_t)j * p.cap, cnt, p.k, lane);
            if (lane == 0) { s_thr[j] = thr; s_cnt[j] = p.k; }
          }
        }
        __syncthreads();
      }
    }
    // finalize: cut each stream to k and publish its global keys
    for (int j = warp; j < nqt; j += kScanWarps) {
      int cnt = s_cnt[j];
      uint32_t* buf = mybufs + (size_t)j * p.cap;
      if (cnt > p.k) { stream_rebuild(buf, cnt, p.k, lane); cnt = p.k; }
      uint64_t* out = p.part + ((size_t)c * p.nq + (q0 + j)) * p.k;
      const int wr = p.part_cnt != nullptr ? cnt : p.k;   // counted lists: no zero padding
      for (int i = lane; i < wr; i += 32)
        out[i] = (i < cnt) ? global_key_from_local(p.kf, buf[i], (uint64_t)row0) : 0ull;
      if (p.part_cnt != nullptr && lane == 0) p.part_cnt[(size_t)c * p.nq + (q0 + j)] = cnt;
    }
  }
}


// ---------------------------------------------------------------------------
// TMA-fed variant (north star item 3: "database codes streamed through TMA
// double buffering"; the paper stresses that loading the codes through the
// memory hierarchy is what bounds the scan).  One CTA per SM: warp 8
// is the producer -- one lane issues, per 256-row stage, NBOX 2-D TMA loads
// (cp.async.bulk.tensor, box = 64 B of a row x 256 rows, 64B swizzle) into a
// ring of `stages` shared-memory stages, each completing on the stage's
// `full` mbarrier (transaction count); warps 0-7 consume: thread t reads row t
// of the stage with conflict-free LDS.128 (the swizzle spreads the 16-B
// chunks of 8 consecutive rows over all banks), releases the stage on its
// `empty` mbarrier, and runs the same Delta + stream code as scan_popc_kernel.
// The row stride of strided (seeding) scans is folded into the tensor map's
// row pitch.  The DB stream never passes through registers before it is
// needed, and `stages` x 256 rows stay in flight per SM.
// ---------------------------------------------------------------------------
constexpr int kTmaBox = 64;                         // bytes of a row per box (= the 64B swizzle span)
constexpr int kTmaThreads = kScanThreads + 32;      // 8 consumer warps + the producer warp
template <int NB>
struct PopcTmaGeo {
  static constexpr int NBOX = (2 * NB * 16 + kTmaBox - 1) / kTmaBox;   // boxes per row
  static constexpr int BOX_BYTES = kStageRows * kTmaBox;               // 16 KB
  static constexpr int STAGE = NBOX * BOX_BYTES;
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t x, int32_t y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

template <int NB>
__global__ void __launch_bounds__(kTmaThreads, 1)
scan_popc_tma_kernel(const __grid_constant__ CUtensorMap tmap, PopcParams p, int stages) {
  using Geo = PopcTmaGeo<NB>;
  using namespace ::uq::tc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)stages * Geo::STAGE);
  uint64_t* empty = full + stages;
  uint4* s_qm = reinterpret_cast<uint4*>(empty + stages + 2);          // [qt][NB]  q+ | q-
  uint4* s_qn = s_qm + (size_t)p.qt * NB;                              // [qt][NB]  q-
  uint32_t* s_thr = reinterpret_cast<uint32_t*>(s_qn + (size_t)p.qt * NB);
  int* s_cnt = reinterpret_cast<int*>(s_thr + p.qt);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_items = (int64_t)p.n_qtiles * p.n_chunks;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), kScanWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kScanWarps) {
    // ======== producer: one lane streams every stage of this CTA's items ========
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      int s = 0;
      uint32_t ph = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int64_t row0 = (item / p.n_qtiles) * p.L;
        const int64_t rows = (p.n - row0 < p.L) ? p.n - row0 : p.L;
        for (int64_t s0 = 0; s0 < rows; s0 += kStageRows) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1u);
          const uint32_t bar = smem_u32(&full[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)Geo::STAGE)
                       : "memory");
          const uint32_t dst = smem_u32(ring + (size_t)s * Geo::STAGE);
#pragma unroll
          for (int j = 0; j < Geo::NBOX; ++j)
            tma_load_2d(dst + (uint32_t)(j * Geo::BOX_BYTES), &tmap, j * kTmaBox, (int32_t)(row0 + s0), bar);
          if (++s == stages) { s = 0; ph ^= 1u; }
        }
      }
    }
    return;
  }

  // ======== consumers: warps 0-7, thread t = row t of every stage ========
  const int t = threadIdx.x;
  uint32_t* mybufs = p.bufs + (size_t)blockIdx.x * p.qt * p.cap;
  // row t's 16-B chunk c of box j sits at t*64 + ((c ^ ((t >> 1) & 3)) << 4)
  // (64B swizzle: address bits [4,6) ^= bits [7,9))
  const uint32_t swz = (uint32_t)((t >> 1) & 3);
  int s = 0;
  uint32_t ph = 0;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int qtile = (int)(item % p.n_qtiles);
    const int64_t c = item / p.n_qtiles;
    const int64_t q0 = (int64_t)qtile * p.qt;
    const int nqt = (int)(p.nq - q0 < (int64_t)p.qt ? p.nq - q0 : (int64_t)p.qt);
    const int64_t row0 = c * p.L;
    const int64_t rows = (p.n - row0 < p.L) ? p.n - row0 : p.L;
    const int64_t pb = (int64_t)NB * 16, cb = 2 * pb;

    named_bar_sync(1, kScanThreads);  // previous item fully done with shared state
    for (int i = t; i < nqt * NB; i += kScanThreads) {
      const uint8_t* qr = p.q + (q0 + i / NB) * cb + (i % NB) * 16;
      const uint4 a = *reinterpret_cast<const uint4*>(qr);
      const uint4 b = *reinterpret_cast<const uint4*>(qr + pb);
      s_qm[i] = make_uint4(a.x | b.x, a.y | b.y, a.z | b.z, a.w | b.w);
      s_qn[i] = b;
    }
    for (int j = t; j < nqt; j += kScanThreads) {
      uint32_t t0 = 0u;
      if (p.thr0) {
        const int32_t dk = p.thr0[(q0 + j) * p.thr0_stride];
        if (dk != INT32_MIN && dk - 1 + p.kf.off >= 0) t0 = ((uint32_t)(dk - 1 + p.kf.off) << p.kf.rb) | p.kf.rmask;
      }
      s_thr[j] = t0;
      s_cnt[j] = 0;
    }
    named_bar_sync(1, kScanThreads);

    for (int64_t s0 = 0; s0 < rows; s0 += kStageRows) {
      const int64_t lr = s0 + t;
      const bool valid = lr < rows;
      mbar_wait(smem_u32(&full[s]), ph);
      const uint8_t* st = ring + (size_t)s * Geo::STAGE + (size_t)t * kTmaBox;
      uint4 u[2 * NB];
#pragma unroll
      for (int j = 0; j < Geo::NBOX; ++j)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          if (4 * j + cc < 2 * NB)
            u[4 * j + cc] = *reinterpret_cast<const uint4*>(st + (size_t)j * Geo::BOX_BYTES + ((cc ^ swz) << 4));
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[s]));   // the stage's bytes are in registers
      if (++s == stages) { s = 0; ph ^= 1u; }
      uint4 dm[NB], dn[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        dn[b] = u[NB + b];
        dm[b] = make_uint4(u[b].x | dn[b].x, u[b].y | dn[b].y, u[b].z | dn[b].z, u[b].w | dn[b].w);
      }
      popc_stage_queries<NB>(p, dm, dn, valid, lr, nqt, s_qm, s_qn, s_thr, s_cnt, mybufs, lane);
      if ((s0 / kStageRows) % p.check == p.check - 1 || s0 + kStageRows >= rows) {
        named_bar_sync(1, kScanThreads);
        for (int j = warp; j < nqt; j += kScanWarps) {
          const int cnt = s_cnt[j];
          if (cnt > p.k + kStageRows) {
            const uint32_t thr = stream_rebuild(mybufs + (size_t)j * p.cap, cnt, p.k, lane);
            if (lane == 0) { s_thr[j] = thr; s_cnt[j] = p.k; }
          }
        }
        named_bar_sync(1, kScanThreads);
      }
    }
    for (int j = warp; j < nqt; j += kScanWarps) {
      int cnt = s_cnt[j];
      uint32_t* buf = mybufs + (size_t)j * p.cap;
      if (cnt > p.k) { stream_rebuild(buf, cnt, p.k, lane); cnt = p.k; }
      uint64_t* out = p.part + ((size_t)c * p.nq + (q0 + j)) * p.k;
      const int wr = p.part_cnt != nullptr ? cnt : p.k;   // counted lists: no zero padding
      for (int i = lane; i < wr; i += 32)
        out[i] = (i < cnt) ? global_key_from_local(p.kf, buf[i], (uint64_t)row0) : 0ull;
      if (p.part_cnt != nullptr && lane == 0) p.part_cnt[(size_t)c * p.nq + (q0 + j)] = cnt;
    }
  }
}

// ---------------------------------------------------------------------------
static int popc_occ(int NB, int qt) { return (NB <= 6 && qt <= 8) ? 3 : (NB <= 10 ? 2 : 1); }

// TMA ring depth for the one-CTA-per-SM TMA variant: as many 256-row stages
// as fit (at most 4) beside the query tile; 0 = use the LDG kernel.  The TMA
// kernel serves the HBM-bound regime (tiles of <= 8 queries: c5 Q = 1 streams
// 9.6 GB at 6.9 TB/s vs 5.1 TB/s with per-thread LDG); POPC-bound tiles (more
// queries per DB row) keep the LDG kernel, whose 2-3 CTAs per SM issue more
// POPC than 8 consumer warps (c2, Q = 1000: 11.9 vs 20.6 ms); d > 1536 leaves
// room for fewer than two stages.  UQ_POPC_LDG=1 forces the LDG kernel
// (measurement knob; both kernels return identical results).
static int popc_tma_stages(int NB, int qt, int64_t n) {
  static const bool ldg = [] {
    const char* e = getenv("UQ_POPC_LDG");
    return e != nullptr && atoi(e) != 0;
  }();
  if (ldg || qt > 8 || NB > 12 || n >= ((int64_t)1 << 31)) return 0;   // TMA row coordinates are int32
  const int stage = ((2 * NB * 16 + kTmaBox - 1) / kTmaBox) * kStageRows * kTmaBox;
  const int fixed = 1024 + 2 * qt * NB * 16 + qt * 8 + 2 * 4 * 8 + 16;
  int st = (227 * 1024 - fixed) / stage;
  if (st > 4) st = 4;
  return st >= 2 ? st : 0;
}

PopcPlan plan_popc(int64_t nq, int64_t n, int32_t d, int32_t k, int sms) {
  PopcPlan pl{};
  const int NB = blocks128(d);
  pl.qt = (int32_t)(nq < 64 ? (nq > 0 ? nq : 1) : 64);
  pl.n_qtiles = (int32_t)((nq + pl.qt - 1) / pl.qt);
  pl.cap = k + (popc_check(k) + 1) * kStageRows;
  pl.stages = popc_tma_stages(NB, pl.qt, n);
  // resident CTAs: one per SM for the TMA kernel, else the LDG kernel's launch bounds
  const int grid_max = pl.stages > 0 ? sms : sms * popc_occ(NB, pl.qt);
  const KeyFmt kf = make_keyfmt(d);
  const int64_t lmax = ((int64_t)kf.rmask + 1) / kStageRows * kStageRows;
  int64_t s_des = (2 * (int64_t)grid_max + pl.n_qtiles - 1) / (pl.n_qtiles > 0 ? pl.n_qtiles : 1);
  if (s_des < 1) s_des = 1;
  int64_t L = (n + s_des - 1) / s_des;
  L = (L + kStageRows - 1) / kStageRows * kStageRows;
  if (L < kStageRows) L = kStageRows;
  if (L > lmax) L = lmax;
  pl.L = L;
  pl.n_chunks = (n + L - 1) / L;
  const int64_t items = (int64_t)pl.n_qtiles * pl.n_chunks;
  pl.grid = (int32_t)(items < grid_max ? (items > 0 ? items : 1) : grid_max);
  pl.smem = (int32_t)(2 * (size_t)pl.qt * NB * 16 + (size_t)pl.qt * 8);
  if (pl.stages > 0)
    pl.smem += 1024 + pl.stages * (((2 * NB * 16 + kTmaBox - 1) / kTmaBox) * kStageRows * kTmaBox) +
               (2 * pl.stages + 2) * 8;
  pl.buf_bytes = (size_t)pl.grid * pl.qt * pl.cap * 4;
  pl.part_bytes = (size_t)pl.n_chunks * nq * k * 8;
  return pl;
}

template <int NB, int OCC>
static cudaError_t launch_popc_occ(const PopcParams& p, const PopcPlan& pl, cudaStream_t st) {
  auto kern = scan_popc_kernel<NB, OCC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return e;
  kern<<<pl.grid, kScanThreads, pl.smem, st>>>(p);
  note_launch();
  return cudaGetLastError();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

template <int NB>
static cudaError_t launch_popc_tma(const PopcParams& p, const PopcPlan& pl, cudaStream_t st) {
  if constexpr (NB > 12) {
    return cudaErrorInvalidValue;
  } else {
    auto enc = tensor_map_encoder();
    if (enc == nullptr) return cudaErrorNotSupported;
    // 2-D view of the scanned rows: dim0 = the code_bytes of a row, dim1 = the
    // n scan rows, pitch code_bytes * row_stride; box = 64 B x 256 rows
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)(2 * NB * 16), (cuuint64_t)p.n};
    const cuuint64_t strides[1] = {(cuuint64_t)(2 * NB * 16) * (cuuint64_t)p.row_stride};
    const cuuint32_t box[2] = {(cuuint32_t)kTmaBox, (cuuint32_t)kStageRows};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(p.db), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    auto kern = scan_popc_tma_kernel<NB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
    if (e != cudaSuccess) return e;
    kern<<<pl.grid, kTmaThreads, pl.smem, st>>>(map, p, pl.stages);
    note_launch();
    return cudaGetLastError();
  }
}

template <int NB>
static cudaError_t launch_popc_nb(const PopcParams& p, const PopcPlan& pl, cudaStream_t st) {
  if (pl.stages > 0) return launch_popc_tma<NB>(p, pl, st);
  const int occ = popc_occ(NB, pl.qt);
  if (NB <= 6 && occ == 3) return launch_popc_occ<NB, (NB <= 6 ? 3 : 2)>(p, pl, st);
  return launch_popc_occ<NB, (NB <= 10 ? 2 : 1)>(p, pl, st);
}

cudaError_t launch_scan_popc(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                             int32_t k, const PopcPlan& pl, uint32_t* bufs, uint64_t* part,
                             const int32_t* thr0, int32_t thr0_stride, int64_t row_stride,
                             cudaStream_t st, int32_t* part_cnt) {
  PopcParams p{q, nq, db, n, d, k, make_keyfmt(d), pl.qt, pl.n_qtiles, pl.n_chunks, pl.L, pl.cap,
               bufs, part, thr0, thr0_stride, row_stride, popc_check(k), part_cnt};
  switch (blocks128(d)) {
#define UQ_POPC_CASE(N) \
  case N: return launch_popc_nb<N>(p, pl, st);
    UQ_POPC_CASE(1) UQ_POPC_CASE(2) UQ_POPC_CASE(3) UQ_POPC_CASE(4)
    UQ_POPC_CASE(5) UQ_POPC_CASE(6) UQ_POPC_CASE(7) UQ_POPC_CASE(8)
    UQ_POPC_CASE(9) UQ_POPC_CASE(10) UQ_POPC_CASE(11) UQ_POPC_CASE(12)
    UQ_POPC_CASE(13) UQ_POPC_CASE(14) UQ_POPC_CASE(15) UQ_POPC_CASE(16)
#undef UQ_POPC_CASE
    default: break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace uq
