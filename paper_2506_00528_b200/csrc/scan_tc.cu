// scan_tc.cu -- Delta as an int8 GEMM on the 5th-generation tensor cores
// (tcgen05.mma.kind::i8 -> SASS UTCIMMA), fused with the per-query top-k.
//
// Delta(q, r) = sum_i v_q[i] * v_r[i] with v in {-1,0,1} (the scalar
// product of two ternary vertices; P:385-389 compute the same integer with
// bit operations).  Written as T_q (Q x K, int8) . T_db^T (K x N, int8) with
// s32 accumulation it is exact by construction.
//
// CTA (one per SM, persistent over work items = (128-query tile, DB chunk)):
//   warps 0-6  producers: thread t owns DB row t of the current 224-row tile;
//              loads its 2-bit planes once per tile (LDG.128) and expands one
//              128-dim block per pipeline stage to int8 in shared memory
//              (UMMA K-major, no-swizzle canonical layout).
//   warp 7     MMA issuer (one lane) + TMEM owner (512 columns = two 128x224
//              s32 accumulators at column 0 and 256, double-buffered).
//   warps 8-11 epilogue: TMEM lane = query; tcgen05.ld 32 accumulator columns
//              (= 32 DB rows) at a time and run the per-query top-k stream
//              (threshold filter, append, warp-cooperative cut back to k).
//   The query tile (A operand, 128 x 128*NB int8) stays resident in SMEM for
//   the whole work item.
//
// K permutation: inside every 32-dim group the K slot 4b+j holds dim 8j+b
// (b = 0..7, j = 0..3), for both operands, so that one output word is
// ((p >> b) & 0x01010101) + 255 * ((n >> b) & 0x01010101): two shifts, two
// masks and one IMAD per 4 dims.  A common permutation of K leaves every dot
// product unchanged.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace uq {
namespace tc {

constexpr int BM = 128;              // queries per tile (UMMA M, TMEM lanes)
constexpr int KB = 128;              // K bytes (= dims) per pipeline stage
constexpr int kAccStride = 256;      // TMEM column offset of the second accumulator
constexpr uint32_t kTmemCols = 512;
constexpr int kBnWide = 224;         // DB rows per tile (UMMA N) for d <= 1024
constexpr int kBnNarrow = 64;        // d in (1024, 1536]: the 192 KB query tile leaves room for 8 KB stages only

// Per-N layout: one producer thread per DB row of the tile; warp kMmaWarp
// issues the MMAs; four epilogue warps start at a multiple of 4 (warp % 4 =
// TMEM lane quarter).  N = 224: 12 warps (168 registers); N = 64: 8 warps.
template <int BN>
struct Cfg {
  static constexpr int kProdWarps = BN / 32;
  static constexpr int kMmaWarp = kProdWarps;
  static constexpr int kEpiWarp0 = (kProdWarps + 1 + 3) / 4 * 4;
  static constexpr int kThreads = (kEpiWarp0 + 4) * 32;
  static constexpr int kStageBytes = BN * KB;
};

struct Params {
  const uint8_t* q;
  int64_t nq;
  const uint8_t* db;
  int64_t n;
  int32_t d;
  int32_t k;
  KeyFmt kf;
  int32_t n_qtiles;   // QT
  // Work items: query tile t is split into S_t DB chunks, S_t = s_lo + (t < r_hi)
  // (the first r_hi tiles get one more chunk); items are numbered tile-major.
  int32_t s_lo, r_hi, s_max;
  int64_t n_items;
  int32_t cap;
  int32_t stages;
  uint32_t* bufs;    // [gridDim.x][BM][cap]
  uint64_t* part;    // [s_max][nq][k]
  const int32_t* thr0;  // optional per-query seed D_k: rows with Delta < thr0[q * thr0_stride] cannot matter
  int32_t thr0_stride;
  int64_t row_stride;   // DB row r of this scan is row r * row_stride of dbcodes
  int32_t dbg;       // timing ablation (env UQ_TC_ABLATE): 1 = no expansion, 2 = no epilogue work, 4 = no DB loads
};

struct Item {
  int t;             // query tile
  int c;             // chunk index inside the tile
  int s_t;           // chunks of this tile
  int64_t row0, rows;
};

template <int BN>
__device__ __forceinline__ Item decode_item(const Params& p, int64_t i, int64_t n) {
  Item it;
  const int64_t big = (int64_t)p.r_hi * (p.s_lo + 1);
  if (i < big) {
    it.t = (int)(i / (p.s_lo + 1));
    it.c = (int)(i % (p.s_lo + 1));
    it.s_t = p.s_lo + 1;
  } else {
    const int64_t j = i - big;
    it.t = p.r_hi + (int)(j / p.s_lo);
    it.c = (int)(j % p.s_lo);
    it.s_t = p.s_lo;
  }
  int64_t L = (n + it.s_t - 1) / it.s_t;
  L = (L + BN - 1) / BN * BN;
  it.row0 = (int64_t)it.c * L;
  it.rows = n - it.row0;
  if (it.rows > L) it.rows = L;
  if (it.rows < 0) it.rows = 0;
  return it;
}

// ---------------------------------------------------------------------------
template <int NB, int BN>
__global__ void __launch_bounds__(Cfg<BN>::kThreads, 1) scan_tc_kernel(Params p) {
  constexpr int kProdWarps = Cfg<BN>::kProdWarps, kMmaWarp = Cfg<BN>::kMmaWarp, kEpiWarp0 = Cfg<BN>::kEpiWarp0;
  constexpr int kThreads = Cfg<BN>::kThreads, kStageBytes = Cfg<BN>::kStageBytes;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int KTOT = NB * KB;                 // K bytes of the A tile
  constexpr uint32_t A_LBO = BM * 16;           // 2048: next 16-B K chunk
  constexpr uint32_t B_LBO = BN * 16;           // next 16-B K chunk of B
  constexpr uint32_t SBO = 128;                 // next 8-row group
  uint8_t* sA = smem;                                        // [KTOT/16][BM/8][8][16]
  uint8_t* sB = smem + (size_t)BM * KTOT;                    // stages x [8][BN/8][8][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)p.stages * kStageBytes);
  uint64_t* full = bars;                  // [stages]  producers -> MMA (count 256)
  uint64_t* empty = bars + p.stages;      // [stages]  MMA commit -> producers
  uint64_t* tfull = bars + 2 * p.stages;  // [2]       MMA commit -> epilogue
  uint64_t* tempty = tfull + 2;           // [2]       epilogue (128) -> MMA
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pb = (int64_t)NB * 16, cb = 2 * pb;
  const int S = p.stages;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), kProdWarps * 32);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 4 * 32);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(smem_u32(s_tmem), kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  // pipeline state (persists across work items)
  int stage = 0;
  uint32_t sphase = 0;
  int acc = 0;
  uint32_t aphase = 0;

  // epilogue stream state (one stream per query = per epilogue thread)
  const int eq = (warp - kEpiWarp0) * 32 + lane;  // query row inside the tile (epilogue only)
  uint32_t* my_buf = p.bufs + ((size_t)blockIdx.x * BM + (eq >= 0 ? eq : 0)) * p.cap;

  for (int64_t item = blockIdx.x; item < p.n_items; item += gridDim.x) {
    const Item it = decode_item<BN>(p, item, p.n);
    const int64_t q0 = (int64_t)it.t * BM;
    const int64_t row0 = it.row0;
    const int64_t rows = it.rows;
    const int ntiles = (int)((rows + BN - 1) / BN);

    // ---- A tile: expand the 128 query codes (all threads) ----
    __syncthreads();
    for (int u = threadIdx.x; u < BM * NB; u += kThreads) {
      const int r = u / NB, kb = u % NB;
      uint4 qp = make_uint4(0, 0, 0, 0), qn = qp;
      if (q0 + r < p.nq) {
        const uint8_t* src = p.q + (q0 + r) * cb + kb * 16;
        qp = *reinterpret_cast<const uint4*>(src);
        qn = *reinterpret_cast<const uint4*>(src + pb);
      }
      uint8_t* dst = sA + (size_t)(kb * 8) * A_LBO + (r >> 3) * SBO + (r & 7) * 16;
      expand_block_store(qp, qn, dst, A_LBO);
    }
    fence_proxy_async();
    __syncthreads();

    if (warp < kProdWarps) {
      // ================= producers =================
      const int r = threadIdx.x;  // row inside the tile
      // Register ring: block kb of the next tile is loaded right after block kb
      // of the current tile has been expanded, so every load has a whole tile
      // of pipeline time to land.
      uint4 dp[NB], dn[NB];
      auto load_block = [&](int tile, int kb, uint4& a, uint4& b) {
        const int64_t lr = (int64_t)tile * BN + r;
        if (tile < ntiles && lr < rows && !(UQ_DBG(p) & 4)) {
          const uint8_t* src = p.db + (row0 + lr) * p.row_stride * cb;
          a = __ldg(reinterpret_cast<const uint4*>(src) + kb);
          b = __ldg(reinterpret_cast<const uint4*>(src + pb) + kb);
        } else {
          a = make_uint4(0, 0, 0, 0);
          b = a;
        }
      };
#pragma unroll
      for (int kb = 0; kb < NB; ++kb) load_block(0, kb, dp[kb], dn[kb]);
      for (int tile = 0; tile < ntiles; ++tile) {
#pragma unroll
        for (int kb = 0; kb < NB; ++kb) {
          mbar_wait(smem_u32(&empty[stage]), sphase ^ 1u);
          uint8_t* dst = sB + (size_t)stage * kStageBytes + (r >> 3) * SBO + (r & 7) * 16;
          if (!(UQ_DBG(p) & 1)) expand_block_store(dp[kb], dn[kb], dst, B_LBO);
          fence_proxy_async();
          mbar_arrive(smem_u32(&full[stage]));
          if (++stage == S) { stage = 0; sphase ^= 1u; }
          load_block(tile + 1, kb, dp[kb], dn[kb]);
        }
      }
    } else if (warp == kMmaWarp) {
      // ================= MMA issuer =================
      // warp-uniform loop (descriptors in uniform registers), one elected lane
      // issues each tcgen05 instruction
      constexpr uint32_t idesc = idesc_i8(BM, BN);
      const uint64_t a_desc0 = smem_desc(smem_u32(sA), A_LBO, SBO);
      const uint64_t b_desc0 = smem_desc(smem_u32(sB), B_LBO, SBO);
      for (int tile = 0; tile < ntiles; ++tile) {
        mbar_wait(smem_u32(&tempty[acc]), aphase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kAccStride);
#pragma unroll 1
        for (int kb = 0; kb < NB; ++kb) {
          mbar_wait(smem_u32(&full[stage]), sphase);
          tc_fence_after();
          const uint64_t b_stage = b_desc0 + (uint64_t)(((uint32_t)stage * kStageBytes) >> 4);
          const uint64_t a_blk = a_desc0 + (uint64_t)(((uint32_t)(kb * 8) * A_LBO) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < KB / 32; ++ks) {
              const uint64_t ad = a_blk + (uint64_t)(((uint32_t)(ks * 2) * A_LBO) >> 4);
              const uint64_t bd = b_stage + (uint64_t)(((uint32_t)(ks * 2) * B_LBO) >> 4);
              mma_i8(d_tmem, ad, bd, idesc, (kb | ks) != 0 ? 1u : 0u);
            }
            mma_commit(smem_u32(&empty[stage]));
            if (kb == NB - 1) mma_commit(smem_u32(&tfull[acc]));
          }
          __syncwarp();
          if (++stage == S) { stage = 0; sphase ^= 1u; }
        }
        if (++acc == 2) { acc = 0; aphase ^= 1u; }
      }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
      // ================= epilogue: per-query top-k streams =================
      const int quarter = warp - kEpiWarp0;  // == warp % 4: TMEM lanes 32*quarter..
      int cnt = 0;
      // Delta threshold: a score passes iff Delta > thrd (never for the
      // padding lanes past the last query)
      int thrd = q0 + eq < p.nq ? INT32_MIN : INT32_MAX;
      if (p.thr0 && q0 + eq < p.nq) {
        const int32_t dk = p.thr0[(q0 + eq) * p.thr0_stride];
        if (dk != INT32_MIN) thrd = dk - 1;  // pass iff Delta >= D_k
      }
      for (int tile = 0; tile < ntiles; ++tile) {
        mbar_wait(smem_u32(&tfull[acc]), aphase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * kAccStride);
        const int64_t lr0 = (int64_t)tile * BN;
        const int ncols = (rows - lr0 < BN) ? (int)(rows - lr0) : BN;
#pragma unroll 1
        for (int c0 = 0; c0 < ((UQ_DBG(p) & 2) ? 0 : BN); c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + (uint32_t)c0, v);
          if (ncols - c0 < 32) {  // ragged tail (warp-uniform): mask columns past the chunk
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j >= ncols) v[j] = 0x80000000u;
          }
          // 4-score maxima, one vote for the whole 32-score row; then, per
          // 4-score chunk some lane needs, a register-only append (rows stay
          // in increasing order)
          int cm[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            cm[i] = max(__vimax3_s32((int)v[4 * i], (int)v[4 * i + 1], (int)v[4 * i + 2]), (int)v[4 * i + 3]);
          const int mx = __vimax3_s32(__vimax3_s32(cm[0], cm[1], cm[2]), __vimax3_s32(cm[3], cm[4], cm[5]),
                                      max(cm[6], cm[7]));
          if (__any_sync(kFull, mx > thrd)) {
            const uint32_t rb0 = (uint32_t)(lr0 + c0);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (__any_sync(kFull, cm[i] > thrd)) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int sc = (int)v[4 * i + j];
                  UQ_ASSERT(!(sc > thrd) || cnt < p.cap);
                  if (sc > thrd) my_buf[cnt++] = local_key(p.kf, sc, rb0 + (uint32_t)(4 * i + j));
                }
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty[acc]));
        if (++acc == 2) { acc = 0; aphase ^= 1u; }
        // cut streams that grew beyond k + BN back to k (warp-cooperative)
        __syncwarp();
        unsigned need = __ballot_sync(kFull, cnt > p.k + BN);
        while (need) {
          const int L = __ffs(need) - 1;
          need &= need - 1;
          const int cL = __shfl_sync(kFull, cnt, L);
          uint32_t* bL = p.bufs + ((size_t)blockIdx.x * BM + quarter * 32 + L) * p.cap;
          const uint32_t D = ordered_rebuild(bL, cL, p.k, lane, p.kf.rb);
          if (lane == L) {
            cnt = p.k;
            thrd = max(thrd, (int)D - p.kf.off);
          }
        }
      }
      // finalize: cut to k, publish global keys (warp copies each lane's list)
      __syncwarp();
      unsigned need = __ballot_sync(kFull, cnt > p.k);
      while (need) {
        const int L = __ffs(need) - 1;
        need &= need - 1;
        const int cL = __shfl_sync(kFull, cnt, L);
        uint32_t* bL = p.bufs + ((size_t)blockIdx.x * BM + quarter * 32 + L) * p.cap;
        ordered_rebuild(bL, cL, p.k, lane, p.kf.rb);
        if (lane == L) cnt = p.k;
      }
      __syncwarp();
      for (int L = 0; L < 32; ++L) {
        const int64_t qi = q0 + quarter * 32 + L;
        const int cL = __shfl_sync(kFull, cnt, L);
        if (qi >= p.nq) continue;
        const uint32_t* bL = p.bufs + ((size_t)blockIdx.x * BM + quarter * 32 + L) * p.cap;
        uint64_t* out = p.part + ((size_t)it.c * p.nq + qi) * p.k;
        for (int i = lane; i < p.k; i += 32)
          out[i] = (i < cL) ? global_key_from_local(p.kf, bL[i], (uint64_t)row0) : 0ull;
        // tiles with fewer chunks than s_max: the last chunk zero-fills the unused lists
        if (it.c == it.s_t - 1)
          for (int c2 = it.s_t; c2 < p.s_max; ++c2) {
            uint64_t* z = p.part + ((size_t)c2 * p.nq + qi) * p.k;
            for (int i = lane; i < p.k; i += 32) z[i] = 0ull;
          }
      }
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

}  // namespace tc

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int tc_bn(int NB) { return NB <= 8 ? tc::kBnWide : tc::kBnNarrow; }

static int tc_stages(int NB) {
  const int a_bytes = tc::BM * NB * tc::KB;
  const int stage_bytes = tc_bn(NB) * tc::KB;
  const int budget = 227 * 1024 - a_bytes - 1024;
  int s = budget / stage_bytes;
  if (s > 4) s = 4;
  return s;
}

// Work split: every SM gets one (query tile, DB chunk) item when the query
// tiles do not cover the SMs: tile t gets s_lo or s_lo + 1 chunks so that the
// item count equals the SM count.  Chunks are bounded by the local-key row
// field (2^rb rows) and kept >= 4 tiles long.  d <= 1024 runs N = 224 tiles,
// 1024 < d <= 1536 N = 64 (the resident query tile takes 192 KB of SMEM).
TcPlan plan_tc(int64_t nq, int64_t n, int32_t d, int32_t k, int sms) {
  TcPlan pl{};
  const int NB = blocks128(d);
  pl.ok = false;
  if (NB > 12 || nq < 1 || n < 1) return pl;
  const int BN = tc_bn(NB);
  pl.stages = tc_stages(NB);
  if (pl.stages < 2) return pl;
  pl.ok = true;
  pl.n_qtiles = (int32_t)((nq + tc::BM - 1) / tc::BM);
  pl.cap = k + 2 * BN;
  const KeyFmt kf = make_keyfmt(d);
  const int64_t lmax = ((int64_t)kf.rmask + 1) / BN * BN;
  const int64_t s_min = (n + lmax - 1) / lmax;                  // key-format bound
  int64_t s_cap = (n + 4 * BN - 1) / (4 * BN);                  // >= 4 tiles per chunk
  if (s_cap < s_min) s_cap = s_min;
  const int64_t QT = pl.n_qtiles;
  if (QT * s_min >= sms) {
    pl.s_lo = (int32_t)s_min;
    pl.r_hi = 0;
  } else {
    int64_t lo = sms / QT, hi = sms % QT;
    if (lo >= s_cap) { lo = s_cap; hi = 0; }
    pl.s_lo = (int32_t)lo;
    pl.r_hi = (int32_t)hi;
  }
  pl.n_chunks = pl.s_lo + (pl.r_hi > 0 ? 1 : 0);
  pl.n_items = QT * pl.s_lo + pl.r_hi;
  pl.grid = (int32_t)(pl.n_items < sms ? pl.n_items : sms);
  pl.smem = tc::BM * NB * tc::KB + pl.stages * BN * tc::KB + (2 * pl.stages + 4) * 8 + 16;
  pl.buf_bytes = (size_t)pl.grid * tc::BM * pl.cap * 4;
  pl.part_bytes = (size_t)pl.n_chunks * nq * k * 8;
  return pl;
}

template <int NB, int BN>
static cudaError_t launch_tc_nb(const tc::Params& p, const TcPlan& pl, cudaStream_t st) {
  auto kern = tc::scan_tc_kernel<NB, BN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return e;
  kern<<<pl.grid, tc::Cfg<BN>::kThreads, pl.smem, st>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_scan_tc(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                           int32_t k, const TcPlan& pl, uint32_t* bufs, uint64_t* part,
                           const int32_t* thr0, int32_t thr0_stride, int64_t row_stride,
                           cudaStream_t st) {
  const int NB = blocks128(d);
  const int dbg = tc_ablate_flags();
  tc::Params p{q, nq, db, n, d, k, make_keyfmt(d), pl.n_qtiles, pl.s_lo, pl.r_hi,
               (int32_t)pl.n_chunks, pl.n_items, pl.cap, pl.stages, bufs, part, thr0, thr0_stride,
               row_stride, dbg};
  constexpr int W = tc::kBnWide, R = tc::kBnNarrow;
  switch (NB) {
    case 1: return launch_tc_nb<1, W>(p, pl, st);
    case 2: return launch_tc_nb<2, W>(p, pl, st);
    case 3: return launch_tc_nb<3, W>(p, pl, st);
    case 4: return launch_tc_nb<4, W>(p, pl, st);
    case 5: return launch_tc_nb<5, W>(p, pl, st);
    case 6: return launch_tc_nb<6, W>(p, pl, st);
    case 7: return launch_tc_nb<7, W>(p, pl, st);
    case 8: return launch_tc_nb<8, W>(p, pl, st);
    case 9: return launch_tc_nb<9, R>(p, pl, st);
    case 10: return launch_tc_nb<10, R>(p, pl, st);
    case 11: return launch_tc_nb<11, R>(p, pl, st);
    case 12: return launch_tc_nb<12, R>(p, pl, st);
    default: break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace uq
