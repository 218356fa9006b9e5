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
#include "common.cuh"
#include "internal.h"

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
};

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
          if (pass) mybufs[(size_t)j * p.cap + base + __popc(bal & lanemask_lt())] = key;
        }
      }
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
      for (int i = lane; i < p.k; i += 32)
        out[i] = (i < cnt) ? global_key_from_local(p.kf, buf[i], (uint64_t)row0) : 0ull;
    }
  }
}

// ---------------------------------------------------------------------------
static int popc_occ(int NB, int qt) { return (NB <= 6 && qt <= 8) ? 3 : (NB <= 10 ? 2 : 1); }

PopcPlan plan_popc(int64_t nq, int64_t n, int32_t d, int32_t k, int sms) {
  PopcPlan pl{};
  const int NB = blocks128(d);
  pl.qt = (int32_t)(nq < 64 ? (nq > 0 ? nq : 1) : 64);
  pl.n_qtiles = (int32_t)((nq + pl.qt - 1) / pl.qt);
  pl.cap = k + (popc_check(k) + 1) * kStageRows;
  const int grid_max = sms * popc_occ(NB, pl.qt);   // resident CTAs (launch bounds)
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

template <int NB>
static cudaError_t launch_popc_nb(const PopcParams& p, const PopcPlan& pl, cudaStream_t st) {
  const int occ = popc_occ(NB, pl.qt);
  if (NB <= 6 && occ == 3) return launch_popc_occ<NB, (NB <= 6 ? 3 : 2)>(p, pl, st);
  return launch_popc_occ<NB, (NB <= 10 ? 2 : 1)>(p, pl, st);
}

cudaError_t launch_scan_popc(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                             int32_t k, const PopcPlan& pl, uint32_t* bufs, uint64_t* part,
                             const int32_t* thr0, int32_t thr0_stride, int64_t row_stride,
                             cudaStream_t st) {
  PopcParams p{q, nq, db, n, d, k, make_keyfmt(d), pl.qt, pl.n_qtiles, pl.n_chunks, pl.L, pl.cap,
               bufs, part, thr0, thr0_stride, row_stride, popc_check(k)};
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
