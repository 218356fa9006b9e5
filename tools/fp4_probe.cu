// fp4_probe.cu -- feasibility probe (measurement tool, not part of libuq):
// can the ternary Delta contraction run on tcgen05.mma.cta_group::2.kind::mxf4
// (E2M1 operands, UE8M0 block-32 scale factors fixed at 2^0, f32 accumulate),
// and how fast is it against kind::i8 on the same 256 x N pair tile?
//   1. exactness: random ternary A/B as E2M1 nibbles (+1 = 0x2, -1 = 0xA,
//      0 = 0x0), one K = 256 sweep, D compared with the integer dot product
//      computed on the host; the run with scale bytes 0x80 (2^1) must give 4x;
//   2. throughput: back-to-back pair MMAs (leader thread), M = 256, N = 256 /
//      192, K = 64 (fp4) vs K = 32 (i8), cycles per MMA -> ops/s per GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp4_probe tools/fp4_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_f4(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t sfa, uint32_t sfb,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_mc(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
}

constexpr int KBYTES = 128;   // bytes of K per row in SMEM (fp4: 256 elements, i8: 128)

// KIND 0: mxf4, 1: i8.  gA: [256][KBYTES] (rows 128 r.. of CTA r), gB: [N][KBYTES]
// (rows N/2 r.. of CTA r); out: [256][N] (float for mxf4, int for i8) when iters == 0,
// else cycles of `iters` K-sweeps.
template <int KIND, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const uint8_t* gA, const uint8_t* gB, uint32_t sf_byte, int iters, uint32_t* out,
          unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  uint32_t cr;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  constexpr int BH = N / 2;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * KBYTES;
  // K-major no-swizzle core matrices: row r, 16-B chunk c at c*rows*16 + (r/8)*128 + (r%8)*16
  for (int i = threadIdx.x; i < 128 * (KBYTES / 16); i += blockDim.x) {
    const int r = i / (KBYTES / 16), c = i % (KBYTES / 16);
    *reinterpret_cast<uint4*>(sA + c * 128 * 16 + (r >> 3) * 128 + (r & 7) * 16) =
        *reinterpret_cast<const uint4*>(gA + (size_t)(128 * cr + r) * KBYTES + c * 16);
  }
  for (int i = threadIdx.x; i < BH * (KBYTES / 16); i += blockDim.x) {
    const int r = i / (KBYTES / 16), c = i % (KBYTES / 16);
    *reinterpret_cast<uint4*>(sB + c * BH * 16 + (r >> 3) * 128 + (r & 7) * 16) =
        *reinterpret_cast<const uint4*>(gB + (size_t)(BH * cr + r) * KBYTES + c * 16);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cl_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const int warp = threadIdx.x >> 5;
  // scale factors: columns [256, 288) of every lane = sf_byte
  {
    const uint32_t v = sf_byte * 0x01010101u;
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 256u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(ta),
        "r"(v)
        : "memory");
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(ta + 16u),
        "r"(v)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cl_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  constexpr int KSTEP = 32;                     // bytes of K per MMA (fp4: 64 elements, i8: 32)
  constexpr int NMMA = KBYTES / KSTEP;
  const uint32_t sf = tmem + 256u;
  long long t0 = clock64();
  if (cr == 0 && threadIdx.x == 0) {
    const int reps = iters > 0 ? iters : 1;
    for (int it = 0; it < reps; ++it) {
#pragma unroll
      for (int ks = 0; ks < NMMA; ++ks) {
        const uint64_t ad = desc(smem_u32(sA) + ks * 2 * 128 * 16, 128 * 16, 128);
        const uint64_t bd = desc(smem_u32(sB) + ks * 2 * BH * 16, BH * 16, 128);
        const uint32_t acc = (it | ks) != 0;
        if (KIND == 0) mma_f4(tmem, ad, bd, idesc_mxf4(256, N), sf, sf, acc);
        else mma_i8(tmem, ad, bd, idesc_i8(256, N), acc);
      }
    }
    commit_mc(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t1 = clock64();
  if (iters > 0) {
    if (cr == 0 && threadIdx.x == 0) cycles[blockIdx.x >> 1] = (unsigned long long)(t1 - t0);
  } else {
    // D: lane = query row (128 per CTA), column = B row
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\ttcgen05.wait::ld.sync.aligned;"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0)
                   : "memory");
      for (int j = 0; j < 8; ++j) out[(size_t)(128 * cr + row) * N + c0 + j] = v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cl_sync();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

static uint32_t rng_state = 12345u;
static uint32_t rnd() {
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 17;
  rng_state ^= rng_state << 5;
  return rng_state;
}
// ternary value of nibble / byte
static int tern_f4(uint8_t nib) { return nib == 0x2 ? 1 : nib == 0xA ? -1 : 0; }

template <int KIND, int N>
static int check(float scale_expect, uint32_t sf_byte) {
  std::vector<uint8_t> A(256 * KBYTES), B(N * KBYTES);
  auto fill = [&](std::vector<uint8_t>& v) {
    for (auto& b : v) {
      if (KIND == 0) {
        uint8_t lo = (uint8_t)(rnd() % 3), hi = (uint8_t)(rnd() % 3);
        const uint8_t m[3] = {0x0, 0x2, 0xA};
        b = (uint8_t)(m[lo] | (m[hi] << 4));
      } else {
        const int8_t m[3] = {0, 1, -1};
        b = (uint8_t)m[rnd() % 3];
      }
    }
  };
  fill(A);
  fill(B);
  uint8_t *dA, *dB;
  uint32_t* dO;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dO, 256 * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  const int smem = 1024 + 128 * KBYTES + (N / 2) * KBYTES;
  cudaFuncSetAttribute(probe<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<KIND, N><<<2, 128, smem>>>(dA, dB, sf_byte, 0, dO, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"check\": \"%s N=%d\", \"error\": \"%s\"}\n", KIND == 0 ? "mxf4" : "i8", N, cudaGetErrorString(e));
    return 1;
  }
  std::vector<uint32_t> O(256 * N);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0, nz = 0;
  double maxabs = 0;
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < N; ++j) {
      long ref = 0;
      for (int b = 0; b < KBYTES; ++b) {
        const uint8_t x = A[(size_t)i * KBYTES + b], y = B[(size_t)j * KBYTES + b];
        if (KIND == 0) ref += tern_f4(x & 15) * tern_f4(y & 15) + tern_f4(x >> 4) * tern_f4(y >> 4);
        else ref += (long)(int8_t)x * (int8_t)y;
      }
      double got;
      if (KIND == 0) { float f; memcpy(&f, &O[(size_t)i * N + j], 4); got = f; }
      else got = (double)(int32_t)O[(size_t)i * N + j];
      if (got != scale_expect * (double)ref) ++bad;
      if (ref != 0) ++nz;
      if (std::abs((double)ref) > maxabs) maxabs = std::abs((double)ref);
    }
  printf("{\"check\": \"%s N=%d sf=0x%02x\", \"mismatches\": %ld, \"nonzero_refs\": %ld, \"max_abs_ref\": %.0f}\n",
         KIND == 0 ? "mxf4" : "i8", N, sf_byte, bad, nz, maxabs);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  return bad != 0;
}

template <int KIND, int N>
static void tput(int sms) {
  std::vector<uint8_t> A(256 * KBYTES, 0x22), B(N * KBYTES, 0x22);
  uint8_t *dA, *dB;
  unsigned long long* dc;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dc, sizeof(unsigned long long) * sms);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  const int smem = 1024 + 128 * KBYTES + (N / 2) * KBYTES;
  cudaFuncSetAttribute(probe<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  probe<KIND, N><<<sms, 128, smem>>>(dA, dB, 0x7f, 100, nullptr, dc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<KIND, N><<<sms, 128, smem>>>(dA, dB, 0x7f, iters, nullptr, dc);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> c(sms / 2);
  cudaMemcpy(c.data(), dc, 8 * (sms / 2), cudaMemcpyDeviceToHost);
  unsigned long long cmax = 0;
  for (auto v : c) cmax = v > cmax ? v : cmax;
  const double nmma = (double)iters * (KBYTES / 32);
  const double kel = KIND == 0 ? 64 : 32;
  const double ops = 2.0 * 256 * N * kel * nmma * (sms / 2);
  printf("{\"tput\": \"%s N=%d\", \"err\": \"%s\", \"cycles_per_mma\": %.1f, \"ms\": %.3f, \"tops\": %.1f}\n",
         KIND == 0 ? "mxf4" : "i8", N, cudaGetErrorString(e), (double)cmax / nmma, ms, ops / (ms * 1e-3) / 1e12);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sms &= ~1;
  int bad = 0;
  bad |= check<1, 256>(1.f, 0x7f);
  bad |= check<0, 256>(1.f, 0x7f);
  bad |= check<0, 256>(4.f, 0x80);
  bad |= check<0, 192>(1.f, 0x7f);
  tput<1, 256>(sms);
  tput<0, 256>(sms);
  tput<0, 192>(sms);
  tput<0, 128>(sms);
  return bad;
}
