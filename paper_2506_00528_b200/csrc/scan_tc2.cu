// scan_tc2.cu -- Delta as an int8 GEMM on CTA pairs (tcgen05.mma.cta_group::2
// .kind::i8 -> UTCIMMA.2CTA), fused with the per-query top-k.
//
// Same contraction as scan_tc.cu (Delta = T_q . T_db^T over {-1,0,1}, s32,
// exact; P:209-216 / P:385-389) on a 2-CTA cluster: the pair computes a
// 256-query x 256-row tile.  CTA r of the pair
//   * keeps its own 128 queries resident in SMEM (A, 128 x 128*NB int8),
//   * expands only rows [128 r, 128 r + 128) of each 256-row DB tile (its half
//     of B), so each SM expands half as many DB rows per unit of MMA work as
//     the one-CTA kernel -- the expansion is the per-SM instruction bottleneck,
//   * holds the 128 x 256 s32 accumulator of its own queries in TMEM (two
//     buffers) and runs their epilogue in its epilogue warps.
// A pipeline stage carries 256 dims (two 128-dim blocks, 8 MMAs of K=32): the
// per-stage barrier round trip (producers of both CTAs -> leader `full`, MMA
// commit -> both CTAs' `empty`) costs about as much as four MMAs, so 8 MMAs per
// stage keep the tensor pipe busy (tools/mma_bench.cu replica: 4 MMAs/stage
// 3.2 POPS, 8 MMAs/stage 4.4 POPS at N = 192).
//
// Two epilogue modes:
//   kTopK  per-query top-k streams (threshold filter in registers, append to
//          a per-stream buffer, warp-cooperative cut back to k), lists of
//          64-bit global keys per (chunk, column half) for the merge kernel;
//   kHist  threshold seeding: per-query histogram of Delta >= F_q in 128 bins
//          of width 2^hs_q spanning [F_q, nnz(q)] (shared-memory atomics,
//          flushed to a global [nq][128] histogram; F_q ~ 2-3 sigma of
//          unrelated-code Delta filters most scores first).  At least
//          sum_{b' >= b} hist[b'] sampled rows have Delta >= F_q + (b << hs_q).
//
// Warps: 0-3 producers (one thread per DB row of this CTA's 128-row half; the
// int8 expansion is bound by the integer ALU pipe of each SM sub-partition, so
// one producer warp per sub-partition), warp 3 of the leader also issues the
// MMAs, 4-11 epilogue in two sets of four (warp % 4 = TMEM lane quarter; set h
// reads accumulator columns [128 h, 128 h + 128)).  12 warps = 3 per SM
// sub-partition, whose 16K-register file allows 168 registers per thread.
// Measured alternatives: a dedicated 13th issuer warp caps registers at 128
// and the producers slow down more than the issue gains (0.76 vs 0.65 ms on
// c2); and TMEM epilogue warps must form whole aligned warpgroups (warps
// 5..12 read the wrong lanes, 8..15 are correct).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace uq {
namespace tc2 {

using namespace ::uq::tc;

constexpr int BM = 128;               // queries per CTA (pair M = 256)
constexpr int kProdWarps = 4;         // warps 0-3
constexpr int kMmaWarp = 3;           // warp 3: also MMA issuer (leader) + TMEM owner
constexpr int kEpiWarp0 = 4;          // warps 4..11 (warp % 4 = TMEM lane quarter)
constexpr uint32_t kTmemCols = 512;   // two accumulators (+ the f4 scale factors)
constexpr int kOpI8 = 0, kOpF4 = 1;   // operand kind: int8 (kind::i8) / E2M1 (kind::mxf4)

// Tile geometry per operand kind.
//   i8: N = 256 rows per pair tile (128 per CTA), 128 B of SMEM per row per
//       128-dim block, two 256-column s32 accumulators fill TMEM;
//   f4: N = 240 (120 per CTA): two 240-column f32 accumulators leave TMEM
//       columns [480, 512) for the (constant) scale factors; 64 B per row per
//       block, so a stage of 3-4 blocks (384-512 dims) still carries 6-8 MMAs.
#ifndef UQ_F4_MAX_BPS
#define UQ_F4_MAX_BPS 8
#endif
constexpr int kF4MaxBps = UQ_F4_MAX_BPS;   // f4: at most this many 128-dim blocks per stage
#ifndef UQ_F4_MAX_BPS_WIDE
#define UQ_F4_MAX_BPS_WIDE 4
#endif
constexpr int kF4MaxBpsWide = UQ_F4_MAX_BPS_WIDE;   // the same for d > 1024
constexpr int i8_max_bps(int NB) {
  // two stages beside the resident query tile and the seeding histogram (32 KB)
  const int fit = (227 * 1024 - 128 * NB * 128 - 32 * 1024 - 2048) / (2 * 128 * 128);
  return fit < 4 ? (fit < 1 ? 1 : fit) : 4;
}
template <int OP> struct Geo {
  static constexpr int BN = OP == kOpF4 ? 240 : 256;   // UMMA N
  static constexpr int BH = BN / 2;                    // DB rows expanded per CTA
  static constexpr int RB = OP == kOpF4 ? 64 : 128;    // SMEM bytes per row per 128-dim block
  static constexpr int CPB = RB / 16;                  // 16-B K chunks per block
  static constexpr int MPB = RB / 32;                  // MMAs per block (32 B of K each)
  static constexpr int ACC = BN;                       // TMEM column of the second accumulator
  static constexpr uint32_t SF_COL = 480;              // f4 scale factors: columns [480, 512)
  // epilogue warp sets (4 warps each, warp % 4 = TMEM lane quarter), each owning
  // CW columns of a tile: 2 sets = 12 warps = 3 per SMSP -> 168 registers.
  // f4 histogram mode (seeding; light epilogue, no stream buffers) uses 3 sets
  // (16 warps, 128 registers) to hide more TMEM-load / vote latency: measured
  // 155k vs 190k cycles per item on c2; the top-k epilogue spills at 128.
  static constexpr int sets(int mode) { return (OP == kOpF4 && mode == 1) ? 3 : 2; }
  static constexpr int threads(int mode) { return (kProdWarps + 4 * sets(mode)) * 32; }
  static constexpr int cw(int mode) { return BN / sets(mode); }
  static constexpr int bps(int NB) {                   // 128-dim blocks per pipeline stage
    // at most mx blocks per stage, split evenly over the fewest stages; int8:
    // mx <= 4 and two stages must fit beside the resident query tile
    // f4, d > 1024: the 96 KB query tile leaves room for only two 6-block
    // stages, i.e. half a tile in flight, and the MMA waited on `full` 54% of
    // the time on c4 (tools/tc2_prof.py); 4-block stages keep 4 in flight
    const int mx = OP == kOpI8 ? i8_max_bps(NB) : (NB > 8 ? kF4MaxBpsWide : kF4MaxBps);
    return NB <= mx ? NB : (NB + (NB + mx - 1) / mx - 1) / ((NB + mx - 1) / mx);
  }
  static constexpr int stage_bytes(int NB) { return bps(NB) * BH * RB; }
};
#ifndef UQ_EPI_PIPE
#define UQ_EPI_PIPE 1
#endif
constexpr bool kEpiPipe = UQ_EPI_PIPE != 0;   // index-fed top-k epilogue: pipelined TMEM loads
constexpr int kF4Bias = 0x4B400000;   // f32 bits of 1.5 * 2^23: (float)(v) + 1.5*2^23 has bits kF4Bias + v
// Seeding histogram: 256 bins where shared memory allows (E2M1, d <= 768: a
// finer bound, fewer main-scan candidates), else 128; two u16 counts per word,
// [bins/2 words][128 queries].  The global histogram is always [nq][256].
constexpr int kHistBinsMax = 256;
constexpr int hist_bins(int OP, int NB) { return (OP == kOpF4 && NB <= 6) ? 256 : 128; }
constexpr int hist_bytes(int OP, int NB) { return (hist_bins(OP, NB) / 2) * BM * 4; }
constexpr int kModeTopK = 0, kModeHist = 1;

struct Params {
  const uint8_t* q;
  int64_t nq;
  const uint8_t* db;
  int64_t n;
  int32_t d;
  int32_t k;
  KeyFmt kf;
  int32_t n_qtiles;     // pair tiles of 256 queries
  int32_t s_lo, r_hi, s_max;
  int64_t n_items;
  int32_t cap;
  int32_t stages;
  uint32_t* bufs;       // [gridDim.x][SETS*BM][cap]
  uint64_t* part;       // [s_max*SETS][nq][cap] (top-k mode)
  int32_t* part_cnt;    // [s_max*SETS][nq] valid entries of each list
  const int32_t* thr0;  // optional per-query seed D_k (rows with Delta < D_k cannot matter)
  int32_t thr0_stride;
  int64_t row_stride;
  uint32_t* ghist;      // kHist: [nq][kHistBinsMax]
  float zfloor;         // kHist: only Delta >= F = zfloor * nnz(q) / sqrt(d) is counted
  uint32_t* qbase;      // kHist: per query (hs << 16) | F, bin = (Delta - F) >> hs
  float topsig;         // kHist: bins span [F, min(bound, F + topsig * sigma)]
  const int32_t* qfail; // top-k, optional (seed fallback pass): run only pair tiles with a failed query
  const int32_t* any_fail;  // optional: the launch is a no-op unless *any_fail
  const int8_t* q8;     // optional (int8 engine): int8 queries [nq][ldq8] instead of ternary codes
  int64_t ldq8;
  const uint8_t* dbx;   // optional (E2M1 engine): pre-expanded index (uq_build_f4_index), stages by bulk copy
  size_t dbx_bytes;     // its size (checked builds assert every bulk copy lies inside it; 0 = unknown)
  int32_t dbg;          // timing ablation (env UQ_TC_ABLATE): 1 no expansion, 2 no epilogue work, 4 no DB loads,
                        // 8 cycle accounting, 16 no producer proxy fence
};

// Cycle accounting (ablation/profiling only: dbg & 8), read by uq_tc2_prof:
// 0 MMA item loop, 1 MMA wait tempty, 2 MMA wait full, 3 producer loop, 4
// producer wait empty, 5 epilogue loop, 6 epilogue wait tfull, 7 epilogue
// TMEM load + filter, 8 epilogue rebuilds, 9 epilogue publish, 10 items,
// 11 CTA setup, 12 CTA item loop, 13 CTA teardown, 14 CTAs (thread 0 of each),
// 15 appended candidates, 16 in-loop stream cuts, 17 streams cut at the end.
__device__ unsigned long long g_prof[48];   // [0, 24): top-k mode, [24, 48): histogram mode
__device__ __forceinline__ long long clk() { return clock64(); }
#define PROF_ON ((UQ_DBG(p) & 8) != 0)
#define PROF_ADD(i, v) do { if (PROF_ON && lane == 0) atomicAdd(&g_prof[(i) + (MODE == kModeHist ? 24 : 0)], (unsigned long long)(v)); } while (0)

struct Item {
  int t, c, s_t;
  int64_t row0, rows;
};

template <int BN>
__device__ __forceinline__ Item decode_item(const Params& p, int64_t i) {
  Item it;
  const int64_t big = (int64_t)p.r_hi * (p.s_lo + 1);
  if (i < big) {
    it.t = (int)(i / (p.s_lo + 1));
    it.c = (int)(i % (p.s_lo + 1));
    it.s_t = p.s_lo + 1;
  } else if (p.r_hi == 0) {
    // uniform chunking (more items than pairs): consecutive items -- the ones
    // running concurrently on consecutive pairs -- take the same DB chunk for
    // different query tiles, so each chunk is fetched from DRAM about once and
    // re-read from L2 (query-tile-major order streamed the database once per
    // query tile: 786 MB of DRAM reads for 192 MB of codes on c2 with int8 queries)
    it.t = (int)(i % p.n_qtiles);
    it.c = (int)(i / p.n_qtiles);
    it.s_t = p.s_lo;
  } else {
    const int64_t j = i - big;
    it.t = p.r_hi + (int)(j / p.s_lo);
    it.c = (int)(j % p.s_lo);
    it.s_t = p.s_lo;
  }
  int64_t L = (p.n + it.s_t - 1) / it.s_t;
  L = (L + BN - 1) / BN * BN;
  it.row0 = (int64_t)it.c * L;
  it.rows = p.n - it.row0;
  if (it.rows > L) it.rows = L;
  if (it.rows < 0) it.rows = 0;
  return it;
}

// kHist: add this thread's histogram column (query `qi`) to the global one and clear it
template <int HB>
__device__ __forceinline__ void hist_flush(uint32_t* s_hist, int col, uint32_t* g) {
#pragma unroll 4
  for (int w = 0; w < HB / 2; ++w) {
    // the flush runs between two named barriers of every set of this
    // quarter: plain load + store, and predicated global reductions for the
    // (few) non-zero bins instead of a divergent branch per bin
    uint32_t* cell = s_hist + w * BM + col;
    const uint32_t v = *cell;
    *cell = 0u;
    if (g != nullptr) {   // (timing ablation UQ_TC_ABLATE & 64 passes g = nullptr)
      red_global_add_if(g + 2 * w, v & 0xffffu, (v & 0xffffu) != 0u);
      red_global_add_if(g + 2 * w + 1, v >> 16, (v >> 16) != 0u);
    }
  }
}

// XM: the stages come from the pre-expanded index by bulk copy (p.dbx set);
// its instantiation carries no producer expansion code, which keeps the hot
// loops of the MMA issuer and the epilogue small in the instruction cache.
template <int NB, int MODE, int OP, bool XM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Geo<OP>::threads(MODE), 1) scan_tc2_kernel(Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  using G = Geo<OP>;
  constexpr int BN = G::BN, BH = G::BH;
  constexpr int kHistBins = hist_bins(OP, NB);
  constexpr int kHistBytes = hist_bytes(OP, NB);
  constexpr int kHistLog = kHistBins == 256 ? 8 : 7;
  constexpr int kEpiSets = G::sets(MODE);
  constexpr int kThreads = G::threads(MODE);
  constexpr int kBlkPerStage = G::bps(NB);
  constexpr int kStageBytes = G::stage_bytes(NB);
  constexpr int kAccStride = G::ACC;
  constexpr int NST = (NB + kBlkPerStage - 1) / kBlkPerStage;  // stages per tile
  constexpr uint32_t A_LBO = BM * 16;   // next 16-B K chunk of A (128 rows)
  constexpr uint32_t B_LBO = BH * 16;   // next 16-B K chunk of this CTA's B half
  constexpr uint32_t SBO = 128;         // next 8-row group
  // scores: i8 accumulators are s32.  f4 accumulators are f32 holding exact
  // integers; a warp whose thresholds t are all >= 0 compares the raw f32
  // bits as int32 (for t >= 0, v > t as floats <=> bits(v) > bits(t) as
  // int32: negative floats and -0.0 have negative bit patterns), otherwise it
  // first adds 1.5*2^23 (bits kF4Bias + v, one FADD per score).
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)BM * NB * G::RB;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(sB + (size_t)p.stages * kStageBytes);  // kHist only
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(s_hist) + (MODE == kModeHist ? kHistBytes : 0));
  uint64_t* full = bars;                   // [stages] (leader): 2 CTAs x producer warps
  uint64_t* empty = bars + p.stages;       // [stages] (each CTA): MMA commit
  uint64_t* tfull = bars + 2 * p.stages;   // [2] (each CTA): MMA commit
  uint64_t* tempty = tfull + 2;            // [2] (leader): 2 CTAs x 4 epilogue warps per set
  uint64_t* loaded = tempty + 2;           // [stages] (each CTA): bulk-copy transaction barriers (dbx mode)
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(loaded + p.stages);
  constexpr bool xmode = XM;

  // seed fallback pass with nothing to redo: every thread of both CTAs leaves
  if (p.any_fail != nullptr && *p.any_fail == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t_entry = PROF_ON ? clk() : 0;
  const uint32_t cr = cluster_ctarank();
  const bool leader = cr == 0;
  const int64_t pb = (int64_t)NB * 16, cb = 2 * pb;
  const int S = p.stages;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), xmode ? 2 : 2 * kProdWarps);   // dbx: one forwarder per CTA
      mbar_init(smem_u32(&empty[s]), 1);
      mbar_init(smem_u32(&loaded[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 2 * 4 * kEpiSets);
    }
    fence_barrier_init();
  }
  if (MODE == kModeHist)
    for (int i = threadIdx.x; i < kHistBytes / 4; i += kThreads) s_hist[i] = 0u;
  if (warp == kMmaWarp) tmem_alloc2(smem_u32(s_tmem), kTmemCols);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  if (OP == kOpF4 && warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
    // UE8M0 scale factors = 2^0 (0x7F) in every byte of columns [480, 512): the
    // MMA's SFA / SFB reads fall inside, whatever their layout
    const uint32_t ta = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + G::SF_COL;
    tmem_fill16(ta, 0x7F7F7F7Fu);
    tmem_fill16(ta + 16u, 0x7F7F7F7Fu);
    tc_fence_before();   // ordered before the MMAs by the item's cluster_sync below
  }
  const long long t_setup = PROF_ON ? clk() : 0;
  if (threadIdx.x == 0) PROF_ADD(11, t_setup - t_entry);

  int stage = 0;            // producers: next stage to fill
  uint32_t sphase = 0;
  int acc = 0;              // accumulator buffer (issuer and epilogue each track it)
  uint32_t aphase = 0;

  for (int64_t item = pair; item < p.n_items; item += npairs) {
    const Item it = decode_item<BN>(p, item);
    const int64_t q0 = (int64_t)it.t * (2 * BM) + (int64_t)cr * BM;  // this CTA's queries
    const int64_t row0 = it.row0;
    const int64_t rows = it.rows;
    const int ntiles = (int)((rows + BN - 1) / BN);

    if (p.qfail != nullptr) {
      // fallback pass: skip pair tiles without a failed query (both CTAs test
      // the same 256 queries, so both skip or both run)
      int f = 0;
      for (int i = threadIdx.x; i < 2 * BM; i += kThreads) {
        const int64_t qq = (int64_t)it.t * (2 * BM) + i;
        if (qq < p.nq && p.qfail[qq] != 0) f = 1;
      }
      if (!__syncthreads_or(f)) continue;
    }
    // ---- A: this CTA's 128 query codes, expanded (all threads) ----
    cluster_sync();  // previous item retired in both CTAs (A is read by the pair's MMAs)
    if (OP == kOpI8 && p.q8 != nullptr) {
      // single-operand search: A = the int8 queries themselves, in
      // the K permutation of the DB expansion (chunk 2w + hb, byte 4 bb + j of
      // a 128-dim block <-> dim 32 w + 8 j + bb + 4 hb), zero past d
      for (int u = threadIdx.x; u < BM * NB * 8; u += kThreads) {
        const int r = u / (NB * 8), kb = (u / 8) % NB, c = u % 8;
        const int w = c >> 1, hb = c & 1;
        uint32_t sw[8];
        const int64_t qq = q0 + r;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          uint32_t word = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int dim = kb * 128 + 32 * w + 4 * t + e;
            const uint32_t b = (qq < p.nq && dim < p.d) ? (uint8_t)p.q8[qq * p.ldq8 + dim] : 0u;
            word |= b << (8 * e);
          }
          sw[t] = word;
        }
        uint32_t o[4];
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          uint32_t word = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) word |= ((sw[2 * j + hb] >> (8 * bb)) & 0xffu) << (8 * j);
          o[bb] = word;
        }
        st_shared_v4(smem_u32(sA + (size_t)(kb * G::CPB + c) * A_LBO + (r >> 3) * SBO + (r & 7) * 16), o[0], o[1],
                     o[2], o[3]);
      }
    } else
    for (int u = threadIdx.x; u < BM * NB; u += kThreads) {
      const int r = u / NB, kb = u % NB;
      uint4 qp = make_uint4(0, 0, 0, 0), qn = qp;
      if (q0 + r < p.nq) {
        const uint8_t* src = p.q + (q0 + r) * cb + kb * 16;
        qp = *reinterpret_cast<const uint4*>(src);
        qn = *reinterpret_cast<const uint4*>(src + pb);
      }
      uint8_t* dst = sA + (size_t)(kb * G::CPB) * A_LBO + (r >> 3) * SBO + (r & 7) * 16;
      if (OP == kOpF4) expand_block_store_f4(qp, qn, dst, A_LBO);
      else expand_block_store(qp, qn, dst, A_LBO);
    }
    fence_proxy_async();
    cluster_sync();  // both CTAs' A tiles are in place before the leader issues

    if (warp < kProdWarps && xmode) {
      // ======= pre-expanded index: a stage is one bulk copy of its SMEM image =======
      // The index stores each 120-row half tile as the K-major stage layout of
      // this kernel (block kb, chunk c, row group, row: uq_build_f4_index), so
      // the bytes of blocks [ks*bps, ks*bps+bps) of a half tile are contiguous.
      // Warp 0 lane 0 issues the copies (transaction-counted on loaded[stage]),
      // warp 1 lane 0 forwards their completion to the pair's full barrier,
      // warp 3 of the leader issues the MMAs.
      const uint32_t full_dst = mapa(smem_u32(&full[0]), 0);
      constexpr uint32_t kHalfTileBytes = (uint32_t)NB * G::CPB * BH * 16;
      auto half_tile = [&](int tile) -> int64_t {   // global half-tile index of (tile, this CTA)
        // the same scan-row -> database-row map as the producers' sample_row:
        // histogram mode takes whole BN-row blocks, one in every row_stride;
        // top-k mode rows (row0 + sr) * row_stride (row_stride is 1 whenever an
        // index is read in top-k mode).  row0 and tile offsets are multiples of BH.
        const int64_t sr = row0 + (int64_t)tile * BN + (int64_t)cr * BH;
        const int64_t row = MODE == kModeHist ? (sr / BN) * (BN * p.row_stride) + sr % BN : sr * p.row_stride;
        return row / BH;
      };
      if (warp == 0 && lane == 0) {
        for (int tile = 0; tile < ntiles; ++tile) {
          const uint8_t* img = p.dbx + (size_t)half_tile(tile) * kHalfTileBytes;
          for (int ks = 0; ks < NST; ++ks) {
            const int nb = (ks + 1) * kBlkPerStage <= NB ? kBlkPerStage : NB - ks * kBlkPerStage;
            const uint32_t bytes = (uint32_t)nb * G::CPB * BH * 16;
            UQ_ASSERT(p.dbx_bytes == 0 || (size_t)half_tile(tile) * kHalfTileBytes +
                                              (size_t)ks * kBlkPerStage * G::CPB * BH * 16 + bytes <= p.dbx_bytes);
            mbar_wait(smem_u32(&empty[stage]), sphase ^ 1u);
            const uint32_t bar = smem_u32(&loaded[stage]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sB + (size_t)stage * kStageBytes)),
                "l"(img + (size_t)ks * kBlkPerStage * G::CPB * BH * 16), "r"(bytes), "r"(bar)
                : "memory");
            if (++stage == S) { stage = 0; sphase ^= 1u; }
          }
        }
      } else if (warp == 1 && lane == 0) {
        for (int tile = 0; tile < ntiles; ++tile)
          for (int ks = 0; ks < NST; ++ks) {
            mbar_wait(smem_u32(&loaded[stage]), sphase);
            mbar_arrive_cluster(full_dst + (uint32_t)stage * 8u);
            if (++stage == S) { stage = 0; sphase ^= 1u; }
          }
      } else if (leader && warp == kMmaWarp) {
        constexpr uint32_t idesc = OP == kOpF4 ? idesc_mxf4(2 * BM, BN) : idesc_i8(2 * BM, BN);
        const uint32_t sf_tmem = tmem_base + G::SF_COL;
        const uint64_t a_desc0 = smem_desc(smem_u32(sA), A_LBO, SBO);
        const uint64_t b_desc0 = smem_desc(smem_u32(sB), B_LBO, SBO);
        long long t_loop = PROF_ON ? clk() : 0, t_we = 0, t_wf = 0;
        for (int tile = 0; tile < ntiles; ++tile) {
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kAccStride);
          for (int ks = 0; ks < NST; ++ks) {
            long long t1 = PROF_ON ? clk() : 0;
            if (ks == 0) mbar_wait_cluster(smem_u32(&tempty[acc]), aphase ^ 1u);
            long long t2 = PROF_ON ? clk() : 0;
            if (PROF_ON) t_we += t2 - t1;
            mbar_wait_cluster(smem_u32(&full[stage]), sphase);
            if (PROF_ON) t_wf += clk() - t2;
            tc_fence_after();
            const uint64_t b_stage = b_desc0 + (uint64_t)(((uint32_t)stage * kStageBytes) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int bb = 0; bb < kBlkPerStage; ++bb) {
                const int kb = ks * kBlkPerStage + bb;
                if (kb < NB) {
#pragma unroll
                  for (int kk = 0; kk < G::MPB; ++kk) {
                    const uint64_t ad = a_desc0 + (uint64_t)(((uint32_t)(kb * G::CPB + kk * 2) * A_LBO) >> 4);
                    const uint64_t bd = b_stage + (uint64_t)(((uint32_t)(bb * G::CPB + kk * 2) * B_LBO) >> 4);
                    if (OP == kOpF4) mma2_f4(d_tmem, ad, bd, idesc, sf_tmem, sf_tmem, (kb | kk) != 0 ? 1u : 0u);
                    else mma2_i8(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                  }
                }
              }
              mma2_commit_mc(smem_u32(&empty[stage]), 0x3);
              if (ks == NST - 1) mma2_commit_mc(smem_u32(&tfull[acc]), 0x3);
            }
            __syncwarp();
            if (++stage == S) { stage = 0; sphase ^= 1u; }
          }
          if (++acc == 2) { acc = 0; aphase ^= 1u; }
        }
        PROF_ADD(0, clk() - t_loop);
        PROF_ADD(1, t_we);
        PROF_ADD(2, t_wf);
        PROF_ADD(10, 1);
      }
    } else if (warp < kProdWarps) {
      if constexpr (!XM) {
      // ================= producers: rows [cr*BH, cr*BH+BH) of each tile =================
      // Warp kMmaWarp of the leader CTA is also the MMA issuer: after writing
      // its rows of a stage it waits for the pair's `full` barrier and issues
      // the stage's 8 MMAs (warp-uniform loop, one elected lane), so every SM
      // sub-partition carries one producer warp and the issue costs only a few
      // uniform-datapath instructions per stage.
      const bool issuer = leader && warp == kMmaWarp;
      const int r = threadIdx.x;
      const uint32_t full_dst = mapa(smem_u32(&full[0]), 0);  // leader's full[0]
      uint4 dp[NB], dn[NB];
      // scan row -> database row: row_stride-strided rows (top-k mode), or in
      // histogram mode whole BN-row blocks, one in every row_stride (the
      // seeding sample stays spread over the database, and each block is
      // contiguous for the L2 prefetch)
      auto sample_row = [&](int64_t sr) -> int64_t {
        if (MODE == kModeHist) return (sr / BN) * (BN * p.row_stride) + sr % BN;
        return sr * p.row_stride;
      };
      // this thread's DB row of a tile (nullptr past the data), computed once
      // per tile: the per-block loads then cost no address arithmetic
      auto row_src = [&](int tile) -> const uint8_t* {
        const int64_t lr = (int64_t)tile * BN + (int64_t)cr * BH + r;
        if (tile < ntiles && lr < rows && r < BH && !(UQ_DBG(p) & 4)) return p.db + sample_row(row0 + lr) * cb;
        return nullptr;
      };
      auto load_block = [&](const uint8_t* src, int kb, uint4& a, uint4& b) {
        if (src != nullptr) {
          a = __ldg(reinterpret_cast<const uint4*>(src) + kb);
          b = __ldg(reinterpret_cast<const uint4*>(src + pb) + kb);
        } else {
          a = make_uint4(0, 0, 0, 0);
          b = a;
        }
      };
      {
        const uint8_t* src0 = row_src(0);
#pragma unroll
        for (int kb = 0; kb < NB; ++kb) load_block(src0, kb, dp[kb], dn[kb]);
      }
      long long t_loop = PROF_ON ? clk() : 0, t_wait = 0, t_we = 0, t_wf = 0;
      // L2 prefetch of this warp's 32 rows two tiles ahead (contiguous rows only):
      // the register ring hides one tile of latency, L2 covers the rest
      auto prefetch_rows = [&](int tile) {
        const int64_t lr = (int64_t)tile * BN + (int64_t)cr * BH + (r & ~31);
        if ((MODE == kModeHist || p.row_stride == 1) && lane == 0 && tile < ntiles && lr < rows &&
            (r & ~31) < BH) {
          int64_t nr = (rows - lr < 32) ? rows - lr : 32;   // 32 rows stay inside one BN-row block
          if (nr > BH - (r & ~31)) nr = BH - (r & ~31);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.db + sample_row(row0 + lr) * cb),
                       "r"((uint32_t)(nr * cb)) : "memory");
        }
      };
      constexpr uint32_t idesc = OP == kOpF4 ? idesc_mxf4(2 * BM, BN) : idesc_i8(2 * BM, BN);
      const uint32_t sf_tmem = tmem_base + G::SF_COL;
      const uint64_t a_desc0 = smem_desc(smem_u32(sA), A_LBO, SBO);
      const uint64_t b_desc0 = smem_desc(smem_u32(sB), B_LBO, SBO);
      prefetch_rows(1);
      for (int tile = 0; tile < ntiles; ++tile) {
        prefetch_rows(tile + 2);
        const uint8_t* nsrc = row_src(tile + 1);
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kAccStride);
#pragma unroll
        for (int ks = 0; ks < NST; ++ks) {
          long long t0 = PROF_ON ? clk() : 0;
          mbar_wait(smem_u32(&empty[stage]), sphase ^ 1u);
          if (PROF_ON) t_wait += clk() - t0;
          uint8_t* sdst = sB + (size_t)stage * kStageBytes + (r >> 3) * SBO + (r & 7) * 16;
#pragma unroll
          for (int bb = 0; bb < kBlkPerStage; ++bb) {
            const int kb = ks * kBlkPerStage + bb;
            if (kb < NB) {
              if (!(UQ_DBG(p) & 1) && r < BH && !(issuer && (UQ_DBG(p) & 512))) {   // (512: ablation, issuer skips its rows)
                if (OP == kOpF4)
                  expand_block_store_f4(dp[kb], dn[kb], sdst + (size_t)(bb * G::CPB) * B_LBO, B_LBO, !(UQ_DBG(p) & 32));
                else
                  expand_block_store(dp[kb], dn[kb], sdst + (size_t)(bb * G::CPB) * B_LBO, B_LBO, !(UQ_DBG(p) & 32));
              }
              load_block(nsrc, kb, dp[kb], dn[kb]);
            }
          }
          if (!(UQ_DBG(p) & 16)) fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(full_dst + (uint32_t)stage * 8u);
          if (issuer) {
            if (ks == 0) {
              long long t1 = PROF_ON ? clk() : 0;
              mbar_wait_cluster(smem_u32(&tempty[acc]), aphase ^ 1u);  // accumulator drained (both CTAs)
              if (PROF_ON) t_we += clk() - t1;
            }
            long long t2 = PROF_ON ? clk() : 0;
            mbar_wait_cluster(smem_u32(&full[stage]), sphase);       // all rows of the stage written
            tc_fence_after();
            if (PROF_ON) t_wf += clk() - t2;
            const uint64_t b_stage = b_desc0 + (uint64_t)(((uint32_t)stage * kStageBytes) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int bb = 0; bb < kBlkPerStage; ++bb) {
                const int kb = ks * kBlkPerStage + bb;
                if (kb < NB) {
#pragma unroll
                  for (int kk = 0; kk < G::MPB; ++kk) {
                    const uint64_t ad = a_desc0 + (uint64_t)(((uint32_t)(kb * G::CPB + kk * 2) * A_LBO) >> 4);
                    const uint64_t bd = b_stage + (uint64_t)(((uint32_t)(bb * G::CPB + kk * 2) * B_LBO) >> 4);
                    if (OP == kOpF4) mma2_f4(d_tmem, ad, bd, idesc, sf_tmem, sf_tmem, (kb | kk) != 0 ? 1u : 0u);
                    else mma2_i8(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                  }
                }
              }
              mma2_commit_mc(smem_u32(&empty[stage]), 0x3);
              if (ks == NST - 1) mma2_commit_mc(smem_u32(&tfull[acc]), 0x3);
            }
            __syncwarp();
          }
          if (++stage == S) { stage = 0; sphase ^= 1u; }
        }
        if (++acc == 2) { acc = 0; aphase ^= 1u; }
      }
      PROF_ADD(3, clk() - t_loop);
      PROF_ADD(4, t_wait);
      if (issuer) {
        PROF_ADD(0, clk() - t_loop);
        PROF_ADD(1, t_we);
        PROF_ADD(2, t_wf);
        PROF_ADD(10, 1);
      }
      }  // !XM
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4 * kEpiSets) {
      // ================= epilogue =================
      // set h handles accumulator columns [h*BN/2, (h+1)*BN/2) of every tile, so
      // each query has kEpiSets streams, each seeing its rows in increasing order
      const int ew = warp - kEpiWarp0;
      const int quarter = ew & 3;             // == warp % 4: TMEM lane quarter
      const int h = ew >> 2;                  // column half
      const int col = quarter * 32 + lane;    // this thread's query inside the CTA tile
      const int64_t qme = q0 + col;
      const uint32_t tempty_dst = mapa(smem_u32(&tempty[0]), 0);  // leader's tempty[0]
      constexpr int CW = G::cw(MODE);         // columns per set per tile
      if (MODE == kModeHist) {
        // Only Delta >= F enters the histogram, F = z nnz(q) / sqrt(d) (z standard
        // deviations of Delta against unrelated codes, z chosen on the host so
        // that ~4k unrelated sample rows still clear it): the count above any
        // bin edge stays a lower bound, and almost every score costs one compare.
        int floor_m1 = 0x7fffffff;
        int top = 0;   // bound on any score of this query: nnz(q) (ternary) or sum |q_i| (int8)
        if (qme < p.nq) {
          if (OP == kOpI8 && p.q8 != nullptr) {
            // int8 query (single-operand search): unrelated rows' scores have
            // sigma ~ |q|_2 sqrt(x/d); x/d = 1/2 assumed for the floor (only
            // the seed's efficiency depends on it)
            int64_t s2 = 0;
            for (int i = 0; i < p.d; ++i) {
              const int v = p.q8[qme * p.ldq8 + i];
              s2 += v * v;
              top += v < 0 ? -v : v;
            }
            const float sigma = sqrtf(0.5f * (float)s2);
            floor_m1 = max(0, (int)(p.zfloor * sigma)) - 1;
            // bins up to 32 sigma above the floor (sum |q_i| is a far looser
            // bound; higher scores land in the last bin, which keeps every
            // "count >= edge" a valid lower bound)
            top = min(top, floor_m1 + 1 + (int)(p.topsig * sigma) + 1);
          } else {
            const uint8_t* qc = p.q + qme * cb;
            for (int b = 0; b < NB; ++b) {
              const uint4 a = *reinterpret_cast<const uint4*>(qc + b * 16);
              const uint4 c = *reinterpret_cast<const uint4*>(qc + pb + b * 16);
              top += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(c.x) + __popc(c.y) +
                     __popc(c.z) + __popc(c.w);
            }
            const float sigma = (float)top * rsqrtf((float)p.d);
            floor_m1 = max(0, (int)(p.zfloor * sigma)) - 1;
            top = min(top, floor_m1 + 1 + (int)(p.topsig * sigma) + 1);
          }
        }
        // bins of width 2^hs_q from F = floor_m1 + 1 up to top >= any score
        int hs_q = 0;
        if (qme < p.nq) {
          const int range = max(top - floor_m1, 1);   // scores in [F, top]: range values
          hs_q = range > kHistBins ? 32 - __clz(range - 1) - kHistLog : 0;
          if (h == 0) p.qbase[qme] = ((uint32_t)hs_q << 16) | (uint32_t)(floor_m1 + 1);
        }
        const bool raw = OP == kOpF4 && __all_sync(kFull, floor_m1 >= 0);
        const int fl = OP != kOpF4 ? floor_m1 : raw ? __float_as_int((float)floor_m1) : min(floor_m1, 4096) + kF4Bias;
        const uint32_t pad = (OP == kOpF4 && !raw) ? 0u : 0x80000000u;
        for (int tile = 0; tile < ntiles; ++tile) {
          mbar_wait(smem_u32(&tfull[acc]), aphase);
          tc_fence_after();
          const uint32_t tbase =
              tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * kAccStride) + (uint32_t)(h * CW);
          const int64_t lr0 = (int64_t)tile * BN + h * CW;
          const int ncols = (rows - lr0 < CW) ? (int)(rows - lr0) : CW;
#pragma unroll 1
          for (int c0 = 0; c0 < ((UQ_DBG(p) & 2) ? 0 : CW); c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + (uint32_t)c0, v);
            if (OP == kOpF4 && !raw) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + 12582912.0f);
            }
            // 4-score maxima, one vote for the whole 32-score row; then, per
            // 4-score chunk some lane needs, a register-only append
            int cm[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              cm[i] = max(__vimax3_s32((int)v[4 * i], (int)v[4 * i + 1], (int)v[4 * i + 2]), (int)v[4 * i + 3]);
            if (ncols - c0 < 32) {
              // columns past the tile: whole 4-groups masked at the maxima (f4's
              // 120-column sets end on a group boundary), element-wise only in a
              // database's partial last group
              const int rem = ncols - c0;
              if (rem & 3) {   // rare: a database's partial last group
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (j >= rem) v[j] = pad;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  cm[i] = max(__vimax3_s32((int)v[4 * i], (int)v[4 * i + 1], (int)v[4 * i + 2]), (int)v[4 * i + 3]);
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) cm[i] = 4 * i >= rem ? (int)pad : cm[i];   // selects, no branches
            }
            const int mx = __vimax3_s32(__vimax3_s32(cm[0], cm[1], cm[2]), __vimax3_s32(cm[3], cm[4], cm[5]),
                                        max(cm[6], cm[7]));
            if (__any_sync(kFull, mx > fl)) {
              // predicated histogram increments, no branch per score (as the
              // top-k appends): Delta from one FADD whose addend is 1.5 * 2^23
              // on raw tiles and 0 on biased ones
              const float fadd = raw ? 12582912.0f : 0.0f;
              const uint32_t hbase = smem_u32(s_hist) + 4u * (uint32_t)col;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (__any_sync(kFull, cm[i] > fl)) {
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const int sc = (int)v[4 * i + j];
                    const int dv = OP != kOpF4 ? sc : __float_as_int(__int_as_float(sc) + fadd) - kF4Bias;
                    const uint32_t b = min((uint32_t)(dv - floor_m1 - 1) >> hs_q, (uint32_t)(kHistBins - 1));
                    red_shared_add_if(hbase + (b >> 1) * (4u * BM), (b & 1u) ? 0x10000u : 1u, sc > fl);
                  }
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_dst + (uint32_t)acc * 8u);
          if (++acc == 2) { acc = 0; aphase ^= 1u; }
          // u16 counters: flush every 128 tiles (128 * 256 rows < 65536 per query)
          if ((tile & 127) == 127) {
            named_bar_sync(1 + quarter, 32 * kEpiSets);  // all sets' warps of this quarter
            if (h == 0) hist_flush<kHistBins>(s_hist, col, qme < p.nq ? p.ghist + (size_t)qme * kHistBinsMax : nullptr);
            named_bar_sync(1 + quarter, 32 * kEpiSets);
          }
        }
        named_bar_sync(1 + quarter, 32 * kEpiSets);
        const long long tf0 = (UQ_DBG(p) & 8) ? clk() : 0;
        if (h == 0) hist_flush<kHistBins>(s_hist, col, (qme < p.nq && !(UQ_DBG(p) & 64)) ? p.ghist + (size_t)qme * kHistBinsMax : nullptr);
        named_bar_sync(1 + quarter, 32 * kEpiSets);
        if ((UQ_DBG(p) & 8) && lane == 0 && h == 0) atomicAdd(&g_prof[18], (unsigned long long)(clk() - tf0));
        if ((UQ_DBG(p) & 8) && lane == 0 && h == 0) atomicAdd(&g_prof[19], 1ull);
      } else {
        const int sidx = h * BM + quarter * 32; // first stream of this warp
        uint32_t* const wbufs = p.bufs + ((size_t)blockIdx.x * kEpiSets * BM + sidx) * p.cap;
        uint32_t* const my_buf = wbufs + (size_t)lane * p.cap;
        int cnt = 0;
        unsigned n_app = 0, n_reb = 0;   // cycle accounting only: appended keys, in-loop cuts
        // a score passes iff Delta > thrd; lanes past the last query (the
        // zero-padded rows of a partial query tile) never pass -- with
        // INT32_MIN they appended every score of every tile (c3's last tile
        // holds 16 queries and 240 padding lanes) and cut their buffers
        // constantly, stretching those items
        int thrd = qme < p.nq ? INT32_MIN : (1 << 24);   // 2^24 > |score| (<= 127 d)
        if (p.thr0 && qme < p.nq) {
          const int32_t dk = p.thr0[qme * p.thr0_stride];
          if (dk != INT32_MIN) thrd = dk - 1;
        }

        long long t_loop = PROF_ON ? clk() : 0, t_w = 0, t_f = 0, t_r = 0;
        for (int tile = 0; tile < ntiles; ++tile) {
          long long t0 = PROF_ON ? clk() : 0;
          mbar_wait(smem_u32(&tfull[acc]), aphase);
          tc_fence_after();
          long long t1 = PROF_ON ? clk() : 0;
          if (PROF_ON) t_w += t1 - t0;
          const uint32_t tbase =
              tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * kAccStride) + (uint32_t)(h * CW);
          const int64_t lr0 = (int64_t)tile * BN + h * CW;  // local row of this set's column 0
          // f4 compare form for this tile (biased form: |Delta| <= 2048, so max(thrd, -4096) loses nothing)
          const bool raw = OP == kOpF4 && __all_sync(kFull, thrd >= 0);
          const int thb = OP != kOpF4 ? thrd : raw ? __float_as_int((float)thrd) : max(thrd, -4096) + kF4Bias;
          const uint32_t pad = (OP == kOpF4 && !raw) ? 0u : 0x80000000u;
          const int ncols = (rows - lr0 < CW) ? (int)(rows - lr0) : CW;
          // one 32-column group of scores (v: columns c0 .. c0 + 31 of this set)
          auto process = [&](uint32_t (&v)[32], const int c0) {
            if (OP == kOpF4 && !raw) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + 12582912.0f);
            }
            // 4-score maxima, one vote for the whole 32-score row; then, per
            // 4-score chunk some lane needs, a register-only append
            int cm[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              cm[i] = max(__vimax3_s32((int)v[4 * i], (int)v[4 * i + 1], (int)v[4 * i + 2]), (int)v[4 * i + 3]);
            if (ncols - c0 < 32) {
              // columns past the tile: whole 4-groups masked at the maxima (f4's
              // 120-column sets end on a group boundary), element-wise only in a
              // database's partial last group
              const int rem = ncols - c0;
              if (rem & 3) {   // rare: a database's partial last group
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (j >= rem) v[j] = pad;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  cm[i] = max(__vimax3_s32((int)v[4 * i], (int)v[4 * i + 1], (int)v[4 * i + 2]), (int)v[4 * i + 3]);
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) cm[i] = 4 * i >= rem ? (int)pad : cm[i];   // selects, no branches
            }
            const int mx = __vimax3_s32(__vimax3_s32(cm[0], cm[1], cm[2]), __vimax3_s32(cm[3], cm[4], cm[5]),
                                        max(cm[6], cm[7]));
            if (__any_sync(kFull, mx > thb)) {
              // key = ((Delta + off) << rb) | (rmask - local row), written as
              // (s << rb) + kb0 - (4i + j): s = the score as an integer
              // pattern (int8: Delta; f32: kF4Bias + Delta, from one FADD
              // whose addend is 1.5 * 2^23 on raw tiles and 0 on biased ones,
              // which already hold that pattern), kb0 folds the pattern bias,
              // off and the row term (shifts distribute over + mod 2^32; the
              // row term stays below 2^rb, so + is the |)
              const uint32_t kb0 = ((uint32_t)(OP != kOpF4 ? p.kf.off : p.kf.off - kF4Bias) << p.kf.rb) +
                                   (p.kf.rmask - (uint32_t)(lr0 + c0));
              const float fadd = raw ? 12582912.0f : 0.0f;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (__any_sync(kFull, cm[i] > thb)) {
                  // predicated appends, no branches: the 4 keys are built
                  // unconditionally and stored where the score passes (a
                  // divergent branch per score cost ~67 instructions and four
                  // reconvergence regions per chunk; with k = 100 about half of
                  // the 32-score groups of a warp take this path)
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const int sc = (int)v[4 * i + j];
                    const bool pj = sc > thb;
                    const uint32_t sp = OP != kOpF4 ? (uint32_t)sc : __float_as_uint(__int_as_float(sc) + fadd);
                    const uint32_t key = (sp << p.kf.rb) + (kb0 - (uint32_t)(4 * i + j));
                    UQ_ASSERT(!pj || cnt < p.cap);
                    st_global_if(my_buf, (uint32_t)cnt, key, pj);
                    cnt += pj ? 1 : 0;
                    if (PROF_ON) n_app += pj ? 1u : 0u;
                  }
                }
              }
            }
          };
          auto release = [&]() {   // this warp is done reading the accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_dst + (uint32_t)acc * 8u);
          };
          if constexpr (XM && kEpiPipe) {
            // software-pipelined: the TMEM load of group g + 1 is in flight while
            // group g is filtered, and the accumulator is released as soon as
            // its last group has been loaded (index-fed kernels only: without
            // the producer code the two inlined bodies fit the instruction cache)
            constexpr int NG = (CW + 31) / 32;
            uint32_t va[32], vb[32];
            tmem_ld32_nowait(tbase, va);
#pragma unroll 1
            for (int g = 0; g < NG; g += 2) {
              tmem_wait_ld_dep(va);
              const bool hb = g + 1 < NG;
              if (hb) tmem_ld32_nowait(tbase + (uint32_t)(32 * (g + 1)), vb);
              else release();
              process(va, 32 * g);
              if (hb) {
                tmem_wait_ld_dep(vb);
                if (g + 2 < NG) tmem_ld32_nowait(tbase + (uint32_t)(32 * (g + 2)), va);
                else release();
                process(vb, 32 * (g + 1));
              }
            }
          } else {
#pragma unroll 1
            for (int c0 = 0; c0 < ((UQ_DBG(p) & 2) ? 0 : CW); c0 += 32) {
              uint32_t v[32];
              tmem_ld32(tbase + (uint32_t)c0, v);
              process(v, c0);
            }
            release();
          }
          if (++acc == 2) { acc = 0; aphase ^= 1u; }
          long long t2 = PROF_ON ? clk() : 0;
          if (PROF_ON) t_f += t2 - t1;
          unsigned need = __ballot_sync(kFull, cnt > p.k + CW);
          while (need) {
            const int L = __ffs(need) - 1;
            need &= need - 1;
            const int cL = __shfl_sync(kFull, cnt, L);
            const uint32_t D = ordered_rebuild_call(wbufs + (size_t)L * p.cap, cL, p.k, lane, p.kf.rb);
            if (lane == L) {
              cnt = p.k;
              thrd = max(thrd, (int)D - p.kf.off);
              ++n_reb;
            }
          }
          if (PROF_ON) t_r += clk() - t2;
        }
        long long t_pub = PROF_ON ? clk() : 0;
        if (PROF_ON) {
          const unsigned a = __reduce_add_sync(kFull, n_app), rb = __reduce_add_sync(kFull, n_reb);
          const unsigned fin = __popc(__ballot_sync(kFull, cnt > p.k));
          PROF_ADD(15, a);
          PROF_ADD(16, rb);
          PROF_ADD(17, fin);
        }
        PROF_ADD(5, t_pub - t_loop);
        PROF_ADD(6, t_w);
        PROF_ADD(7, t_f);
        PROF_ADD(8, t_r);
        // finalize: publish each stream's candidates as list (chunk, set), all
        // cnt <= cap of them -- a superset of the stream's top-k, so the merge
        // stays exact, without the warp-serial cut of every stream to k (with
        // k = 10 nearly every stream needed one: 85 us of c5's kernel tail)
        __syncwarp();
        // publish: 8 streams x 4 entries per lane per round, all loads issued
        // before the stores (a stream-at-a-time loop serialised ~100 L2 round
        // trips per warp: 25 us of every work item's tail on c2)
        {
          const int64_t qi = q0 + quarter * 32 + lane;   // this lane's stream: its list's count
          if (qi < p.nq) p.part_cnt[(size_t)(it.c * kEpiSets + h) * p.nq + qi] = cnt;   // entries past it are never read
        }
        const int cmax = (int)__reduce_max_sync(kFull, (unsigned)cnt);   // rounds past it would move nothing
        for (int L0 = 0; L0 < 32; L0 += 8) {
          for (int i0 = 0; i0 < cmax; i0 += 128) {
            uint32_t t[8][4];
            int cLs[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              cLs[u] = __shfl_sync(kFull, cnt, L0 + u);
              const uint32_t* bL = wbufs + (size_t)(L0 + u) * p.cap;
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                const int i = i0 + 32 * v + lane;
                t[u][v] = (i < cLs[u]) ? bL[i] : 0u;
              }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int64_t qi = q0 + quarter * 32 + L0 + u;
              if (qi >= p.nq) continue;
              const size_t list = (size_t)(it.c * kEpiSets + h) * p.nq + qi;
              uint64_t* out = p.part + list * p.cap;
              const int cv = cLs[u];
              UQ_ASSERT(cv <= p.cap && it.c < p.s_max);
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                const int i = i0 + 32 * v + lane;
                if (i < cv) out[i] = global_key_from_local(p.kf, t[u][v], (uint64_t)row0);
              }
            }
          }
        }
        if (it.c == it.s_t - 1) {   // tiles with fewer chunks than s_max: the unused lists are empty
          const int64_t qi = q0 + quarter * 32 + lane;
          if (qi < p.nq)
            for (int c2 = it.s_t; c2 < p.s_max; ++c2) p.part_cnt[(size_t)(c2 * kEpiSets + h) * p.nq + qi] = 0;
        }
        PROF_ADD(9, clk() - t_pub);
      }
    }
  }
  const long long t_items = PROF_ON ? clk() : 0;
  if (threadIdx.x == 0) PROF_ADD(12, t_items - t_setup);
  tc_fence_before();
  cluster_sync();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, kTmemCols);
  }
  if (threadIdx.x == 0) PROF_ADD(13, clk() - t_items);
  if (threadIdx.x == 0) PROF_ADD(14, 1);
}

// kHist -> per-query seed: thr[q] = F_q + (b << hs_q) for the largest bin b with
// sum_{b' >= b} hist[q][b'] >= need (at least `need` sampled rows have Delta >=
// that edge), INT32_MIN if fewer than need sampled rows were counted.  One warp
// per query (lane l: bins 4l .. 4l+3); clears the histogram.
__global__ void thr_from_hist_kernel(uint32_t* ghist, int64_t nq, int32_t k, const uint32_t* qbase, int32_t* thr) {
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  // lane l: bins 8l .. 8l+7
  uint4* g = reinterpret_cast<uint4*>(ghist + (size_t)q * kHistBinsMax) + 2 * lane;
  const uint4 h0 = g[0], h1 = g[1];
  g[0] = make_uint4(0u, 0u, 0u, 0u);
  g[1] = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t hb[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
  uint32_t tot = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) tot += hb[j];
  uint32_t suf = tot;  // sum over lanes >= lane
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_down_sync(kFull, suf, o);
    if (lane + o < 32) suf += t;
  }
  // suffix sums of this lane's bins: s[j] = sum of bins >= 8 lane + j
  uint32_t sj[8];
  uint32_t run = suf - tot;
#pragma unroll
  for (int j = 7; j >= 0; --j) {
    run += hb[j];
    sj[j] = run;
  }
  const unsigned ok = __ballot_sync(kFull, sj[0] >= (uint32_t)k);
  if (ok == 0u) {
    if (lane == 0) thr[q] = INT32_MIN;
    return;
  }
  const int L = 31 - __clz(ok);
  if (lane == L) {
    int j = 0;
#pragma unroll
    for (int jj = 1; jj < 8; ++jj)
      if (sj[jj] >= (uint32_t)k) j = jj;
    const uint32_t qb = qbase[q];
    thr[q] = (int32_t)(qb & 0xffffu) + ((8 * L + j) << (qb >> 16));
  }
}

// E2M1 index: every 120-row half tile stored as the pair kernel's K-major
// stage image -- [NB blocks][4 chunks][15 row groups][8 rows][16 B], chunk c of
// block kb = expand_word_f4 of plane word 4 kb + c -- rows padded with zeros to
// whole 240-row pair tiles.  One thread per (row, block).
__global__ void build_f4_index_kernel(const uint8_t* __restrict__ codes, int64_t n, int64_t n_pad, int NB,
                                      uint8_t* __restrict__ index) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pad * NB) return;
  const int64_t r = t / NB;
  const int kb = (int)(t % NB);
  const int64_t pb = (int64_t)NB * 16;
  uint4 pw = make_uint4(0, 0, 0, 0), nw = pw;
  if (r < n) {
    pw = *reinterpret_cast<const uint4*>(codes + r * 2 * pb + kb * 16);
    nw = *reinterpret_cast<const uint4*>(codes + r * 2 * pb + pb + kb * 16);
  }
  const uint32_t pp[4] = {pw.x, pw.y, pw.z, pw.w}, nn[4] = {nw.x, nw.y, nw.z, nw.w};
  constexpr int HT = 120;
  const int64_t h = r / HT;
  const int j = (int)(r % HT);
  uint8_t* base = index + (size_t)h * NB * 4 * HT * 16 + (size_t)kb * 4 * HT * 16 + (j >> 3) * 128 + (j & 7) * 16;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t o[4];
    ::uq::tc::expand_word_f4(pp[c], nn[c], o);
    *reinterpret_cast<uint4*>(base + (size_t)c * HT * 16) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// int8 index (single-operand search / the int8 engine): each 128-row half tile
// as the int8 pair kernel's stage image -- [NB][8 chunks][16 row groups][8
// rows][16 B], chunk 2w + h of block kb = bytes 16h.. of expand_word(word 4kb+w)
// -- rows padded with zeros to whole 256-row tiles.
__global__ void build_i8_index_kernel(const uint8_t* __restrict__ codes, int64_t n, int64_t n_pad, int NB,
                                      uint8_t* __restrict__ index) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pad * NB) return;
  const int64_t r = t / NB;
  const int kb = (int)(t % NB);
  const int64_t pb = (int64_t)NB * 16;
  uint4 pw = make_uint4(0, 0, 0, 0), nw = pw;
  if (r < n) {
    pw = *reinterpret_cast<const uint4*>(codes + r * 2 * pb + kb * 16);
    nw = *reinterpret_cast<const uint4*>(codes + r * 2 * pb + pb + kb * 16);
  }
  const uint32_t pp[4] = {pw.x, pw.y, pw.z, pw.w}, nn[4] = {nw.x, nw.y, nw.z, nw.w};
  constexpr int HT = 128;
  const int64_t h = r / HT;
  const int j = (int)(r % HT);
  uint8_t* base = index + (size_t)h * NB * 8 * HT * 16 + (size_t)kb * 8 * HT * 16 + (j >> 3) * 128 + (j & 7) * 16;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t o[8];
    ::uq::tc::expand_word(pp[w], nn[w], o);
    *reinterpret_cast<uint4*>(base + (size_t)(2 * w) * HT * 16) = make_uint4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<uint4*>(base + (size_t)(2 * w + 1) * HT * 16) = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

}  // namespace tc2

size_t i8_index_bytes(int64_t n, int32_t d) {
  const int64_t n_pad = (n + 255) / 256 * 256;
  return (size_t)n_pad * blocks128(d) * 128;
}

cudaError_t launch_build_i8_index(const uint8_t* codes, int64_t n, int32_t d, uint8_t* index, cudaStream_t st) {
  const int NB = blocks128(d);
  const int64_t n_pad = (n + 255) / 256 * 256;
  const int64_t threads = n_pad * NB;
  if (threads == 0) return cudaSuccess;
  tc2::build_i8_index_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(codes, n, n_pad, NB, index);
  note_launch();
  return cudaGetLastError();
}

size_t f4_index_bytes(int64_t n, int32_t d) {
  const int64_t n_pad = (n + 239) / 240 * 240;
  return (size_t)n_pad * blocks128(d) * 64;
}

cudaError_t launch_build_f4_index(const uint8_t* codes, int64_t n, int32_t d, uint8_t* index, cudaStream_t st) {
  const int NB = blocks128(d);
  const int64_t n_pad = (n + 239) / 240 * 240;
  const int64_t threads = n_pad * NB;
  if (threads == 0) return cudaSuccess;
  tc2::build_f4_index_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(codes, n, n_pad, NB, index);
  note_launch();
  return cudaGetLastError();
}

namespace tc2 {

// fail[q] = the query was filtered by a seed and its k-th result is padding
// (fewer than k rows passed the optimistic bound): it must be searched again
__global__ void seed_verify_kernel(const int64_t* out_ids, int64_t nq, int32_t k, const int32_t* thr, int32_t* fail,
                                   int32_t* any) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const bool f = thr[q] != INT32_MIN && out_ids[q * k + (k - 1)] < 0;
  fail[q] = f ? 1 : 0;
  if (f) atomicOr(any, 1);
}

}  // namespace tc2

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
template <int OP>
static int tc2_stages(int NB, int mode) {
  const int a_bytes = tc2::BM * NB * tc2::Geo<OP>::RB;
  const int budget = 227 * 1024 - a_bytes - (mode == tc2::kModeHist ? tc2::hist_bytes(OP, NB) : 0) - 2048;
  int s = budget / tc2::Geo<OP>::stage_bytes(NB);
  if (s > 6) s = 6;
  return s;
}
static int tc2_max_nb(int op) { return op == tc2::kOpF4 ? 12 : 8; }


// Pairs: the query set is cut into 256-query pair tiles; each of the SMs/2
// pairs gets one (pair tile, DB chunk) item when the tiles do not cover them.
template <int OP>
static TcPlan plan_tc2_mode(int64_t nq, int64_t n, int32_t d, int32_t k, int sms, int mode, int32_t sbound) {
  using G = tc2::Geo<OP>;
  TcPlan pl{};
  const int NB = blocks128(d);
  pl.ok = false;
  if (NB > tc2_max_nb(OP) || nq < 1 || n < 1) return pl;
  pl.stages = tc2_stages<OP>(NB, mode);
  if (pl.stages < 2) return pl;
  pl.ok = true;
  const int npairs = sms / 2;
  pl.n_qtiles = (int32_t)((nq + 2 * tc2::BM - 1) / (2 * tc2::BM));
  pl.cap = k + 2 * G::cw(mode);
  const KeyFmt kf = make_keyfmt(sbound);   // |score| <= sbound (d; 127 d for int8 queries)
  const int64_t lmax = ((int64_t)kf.rmask + 1) / G::BN * G::BN;
  const int64_t s_min = (n + lmax - 1) / lmax;
  int64_t s_cap = (n + 4 * G::BN - 1) / (4 * G::BN);
  if (s_cap < s_min) s_cap = s_min;
  const int64_t QT = pl.n_qtiles;
  if (QT * s_min >= npairs) {
    // more items than pairs (items are dealt to pairs round robin): choose the
    // chunk count s in [s_min, 4 s_min] minimising the busiest pair's work,
    // ceil(QT s / npairs) items of ~n/s rows plus a fixed per-item cost (query
    // tile expansion, pipeline drain, publish: ~8 tiles) -- e.g. c5 Q=1024:
    // 4 x 48 items on 74 pairs leave the busiest pair 3 items for 2.6 on
    // average; 4 x 55 items are dealt 2.97 : 3
    int64_t best_s = s_min;
    double best = 1e300;
    for (int64_t sc = s_min; sc <= std::min<int64_t>(4 * s_min, s_cap); ++sc) {
      const double per_item = (double)((n + sc - 1) / sc) + 8.0 * G::BN;
      const double cost = (double)((QT * sc + npairs - 1) / npairs) * per_item;
      if (cost < best * 0.999) { best = cost; best_s = sc; }
    }
    pl.s_lo = (int32_t)best_s;
    pl.r_hi = 0;
  } else {
    int64_t lo = npairs / QT, hi = npairs % QT;
    if (lo >= s_cap) { lo = s_cap; hi = 0; }
    // uniform chunking (the remainder pairs idle) when that idles <= 5% of the
    // pairs: it enables the chunk-major item order, under which the pairs that
    // share a DB chunk are adjacent -- c2: DRAM reads 371 -> 217 MB for 192 MB
    // of codes (the query-tile-major order put each chunk's readers on both
    // dies), for ~1% more scan time (2 of 74 pairs idle)
    if (hi * 20 <= npairs) hi = 0;
    // cost of that plan: one round, its largest items (n / lo rows) plus the
    // fixed per-item cost.  Uniform chunking over several rounds can beat it
    // when the query tiles are a large fraction of the pairs: c3's seeding
    // scan (40 tiles, 74 pairs) gave 34 tiles half-size items and left the 6
    // full-size ones as the critical path
    double best = (double)((n + lo - 1) / lo) + 8.0 * G::BN;
    int64_t best_s = -1;
    for (int64_t sc = lo + 1; sc <= std::min<int64_t>(4 * (lo + 1), s_cap); ++sc) {
      const double per_item = (double)((n + sc - 1) / sc) + 8.0 * G::BN;
      const double cost = (double)((QT * sc + npairs - 1) / npairs) * per_item;
      if (cost < best * 0.97) { best = cost; best_s = sc; }
    }
    pl.s_lo = (int32_t)(best_s > 0 ? best_s : lo);
    pl.r_hi = (int32_t)(best_s > 0 ? 0 : hi);
  }
  const int32_t s_max = pl.s_lo + (pl.r_hi > 0 ? 1 : 0);
  pl.n_chunks = (int64_t)s_max * G::sets(mode);  // lists per query for the merge
  pl.n_items = QT * pl.s_lo + pl.r_hi;
  const int64_t pairs = pl.n_items < npairs ? pl.n_items : npairs;
  pl.grid = (int32_t)(2 * pairs);
  pl.smem = 1024 + tc2::BM * NB * G::RB + pl.stages * G::stage_bytes(NB) +
            (mode == tc2::kModeHist ? tc2::hist_bytes(OP, NB) : 0) + (3 * pl.stages + 4) * 8 + 16;
  pl.buf_bytes = (mode == tc2::kModeHist) ? 0 : (size_t)pl.grid * G::sets(mode) * tc2::BM * pl.cap * 4;
  pl.part_bytes = (mode == tc2::kModeHist) ? 0 : (size_t)pl.n_chunks * nq * pl.cap * 8;
  return pl;
}

TcPlan plan_tc2(int64_t nq, int64_t n, int32_t d, int32_t k, int sms, int op, int32_t sbound) {
  if (sbound <= 0) sbound = d;
  return op == tc2::kOpF4 ? plan_tc2_mode<tc2::kOpF4>(nq, n, d, k, sms, tc2::kModeTopK, sbound)
                          : plan_tc2_mode<tc2::kOpI8>(nq, n, d, k, sms, tc2::kModeTopK, sbound);
}
TcPlan plan_tc2_hist(int64_t nq, int64_t n, int32_t d, int32_t k, int sms, int op) {
  return op == tc2::kOpF4 ? plan_tc2_mode<tc2::kOpF4>(nq, n, d, k, sms, tc2::kModeHist, d)
                          : plan_tc2_mode<tc2::kOpI8>(nq, n, d, k, sms, tc2::kModeHist, d);
}

template <int NB, int MODE, int OP>
static cudaError_t launch_tc2_nb(const tc2::Params& p, const TcPlan& pl, cudaStream_t st) {
  auto kern = p.dbx != nullptr ? tc2::scan_tc2_kernel<NB, MODE, OP, true> : tc2::scan_tc2_kernel<NB, MODE, OP, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return e;
  kern<<<pl.grid, tc2::Geo<OP>::threads(MODE), pl.smem, st>>>(p);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess && getenv("UQ_DEBUG"))
    fprintf(stderr, "scan_tc2_kernel<%d,%d,%d> launch (grid %d, smem %d): %s\n", NB, MODE, OP, pl.grid, pl.smem,
            cudaGetErrorString(e));
  return e;
}

template <int MODE, int OP>
static cudaError_t launch_tc2_op(const tc2::Params& p, const TcPlan& pl, int NB, cudaStream_t st) {
  switch (NB) {
    case 1: return launch_tc2_nb<1, MODE, OP>(p, pl, st);
    case 2: return launch_tc2_nb<2, MODE, OP>(p, pl, st);
    case 3: return launch_tc2_nb<3, MODE, OP>(p, pl, st);
    case 4: return launch_tc2_nb<4, MODE, OP>(p, pl, st);
    case 5: return launch_tc2_nb<5, MODE, OP>(p, pl, st);
    case 6: return launch_tc2_nb<6, MODE, OP>(p, pl, st);
    case 7: return launch_tc2_nb<7, MODE, OP>(p, pl, st);
    case 8: return launch_tc2_nb<8, MODE, OP>(p, pl, st);
    default: break;
  }
  if (OP == tc2::kOpF4) {
    switch (NB) {
      case 9: return launch_tc2_nb<9, MODE, tc2::kOpF4>(p, pl, st);
      case 10: return launch_tc2_nb<10, MODE, tc2::kOpF4>(p, pl, st);
      case 11: return launch_tc2_nb<11, MODE, tc2::kOpF4>(p, pl, st);
      case 12: return launch_tc2_nb<12, MODE, tc2::kOpF4>(p, pl, st);
      default: break;
    }
  }
  return cudaErrorInvalidValue;
}
template <int MODE>
static cudaError_t launch_tc2_mode(const tc2::Params& p, const TcPlan& pl, int NB, int op, cudaStream_t st) {
  return op == tc2::kOpF4 ? launch_tc2_op<MODE, tc2::kOpF4>(p, pl, NB, st)
                          : launch_tc2_op<MODE, tc2::kOpI8>(p, pl, NB, st);
}

int tc_ablate_flags() {
#ifdef UQ_PROFILE
  static const int dbg = [] {
    const char* e = getenv("UQ_TC_ABLATE");
    return e ? atoi(e) : 0;
  }();
  return dbg;
#else
  return 0;
#endif
}
static int tc2_dbg() { return tc_ablate_flags(); }

// profiling counters (dbg & 8): copy out and reset
cudaError_t tc2_prof_read(unsigned long long* out48) {
  cudaError_t e = cudaMemcpyFromSymbol(out48, tc2::g_prof, 48 * sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  static const unsigned long long z[48] = {0};
  return cudaMemcpyToSymbol(tc2::g_prof, z, sizeof(z));
}

cudaError_t launch_scan_tc2(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                            int32_t k, const TcPlan& pl, uint32_t* bufs, uint64_t* part, int32_t* part_cnt,
                            const int32_t* thr0, int32_t thr0_stride, int64_t row_stride, int op,
                            cudaStream_t st, const int32_t* qfail, const int32_t* any_fail, const int8_t* q8,
                            int64_t ldq8, const uint8_t* dbx, size_t dbx_bytes) {
  if (q8 != nullptr && op != tc2::kOpI8) return cudaErrorInvalidValue;
  // an index is read by whole contiguous half tiles: top-k scans of an
  // index are over every row (strided top-k scans only seed the other engines)
  if (dbx != nullptr && row_stride != 1) return cudaErrorInvalidValue;
  tc2::Params p{q, nq, db, n, d, k, make_keyfmt(q8 ? 127 * d : d), pl.n_qtiles, pl.s_lo, pl.r_hi,
                (int32_t)(pl.s_lo + (pl.r_hi > 0 ? 1 : 0)), pl.n_items, pl.cap, pl.stages, bufs, part, part_cnt, thr0,
                thr0_stride, row_stride, nullptr, 0.f, nullptr, 0.f, qfail, any_fail, q8, ldq8, dbx, dbx_bytes,
                tc2_dbg()};
  return launch_tc2_mode<tc2::kModeTopK>(p, pl, blocks128(d), op, st);
}

// Threshold seeding over rows {i * row_stride : i < n}: histogram scan, then
// thr[q] (stride 1) from the histogram.  ghist: [nq][128] u32, zero on entry
// (left zero on exit).
cudaError_t launch_seed_tc2_hist(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                                 int32_t k, int32_t need, int64_t row_stride, uint32_t* ghist, uint32_t* qbase,
                                 int32_t* thr, int sms, int op, cudaStream_t st, const int8_t* q8, int64_t ldq8,
                                 const uint8_t* dbx, size_t dbx_bytes) {
  if (q8 != nullptr && op != tc2::kOpI8) return cudaErrorInvalidValue;
  const TcPlan pl = plan_tc2_hist(nq, n, d, k, sms, op);
  if (!pl.ok) return cudaErrorInvalidValue;
  // floor: about 4 * need of the n sampled unrelated rows exceed it (Gaussian
  // tail), z in [0, 4]; only the rows above the final bound matter, so a
  // higher floor just skips counting (and the SMEM atomics of) the bulk
  double ptail = 4.0 * (double)need / (double)(n > 0 ? n : 1);
  if (ptail > 0.5) ptail = 0.5;
  float z = inv_norm_cdf(1.0 - ptail);
  // histogram bins span [F, min(score bound, F + 32 sigma)] (measured: narrower
  // caps clamp c2's D_k into the last bin; sum |q_i| is far too loose for int8 queries)
  const float topsig = 32.f;
  z = z < 0.f ? 0.f : (z > 4.f ? 4.f : z);
  tc2::Params p{q, nq, db, n, d, k, make_keyfmt(d), pl.n_qtiles, pl.s_lo, pl.r_hi,
                (int32_t)(pl.s_lo + (pl.r_hi > 0 ? 1 : 0)), pl.n_items, pl.cap, pl.stages, nullptr, nullptr, nullptr,
                nullptr, 0, row_stride, ghist, z, qbase, topsig, nullptr, nullptr, q8, ldq8, dbx, dbx_bytes,
                tc2_dbg()};
  cudaError_t e = launch_tc2_mode<tc2::kModeHist>(p, pl, blocks128(d), op, st);
  if (e != cudaSuccess) return e;
  tc2::thr_from_hist_kernel<<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(ghist, nq, need, qbase, thr);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_seed_verify(const int64_t* out_ids, int64_t nq, int32_t k, const int32_t* thr, int32_t* fail,
                               int32_t* any, cudaStream_t st) {
  tc2::seed_verify_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(out_ids, nq, k, thr, fail, any);
  note_launch();
  return cudaGetLastError();
}

}  // namespace uq
