// mma_bench.cu -- tcgen05.mma.kind::i8 throughput microbenchmark (measurement
// tool, not part of libuq): one CTA per SM, one thread issues back-to-back
// M=128 x N x K=32 MMAs from shared memory into TMEM, for the no-swizzle and
// the 128B-swizzle K-major layouts.  Prints one JSON line per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

template <int N, int LAYOUT>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  // A: 128 x 128 B, B: N x 128 B (one 128-B K block each); zero-filled
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * 128;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u * (i & 1), 0, 0x01010101u, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint64_t ad, bd;
        if (LAYOUT == 0) {  // no swizzle: core matrices 8x16B; K chunk stride = rows*16
          ad = desc(smem_u32(sA) + ks * 2 * 128 * 16, 128 * 16, 128, 0);
          bd = desc(smem_u32(sB) + ks * 2 * N * 16, N * 16, 128, 0);
        } else {            // 128B swizzle: 8-row atoms of 1024 B; K step = +32 B
          ad = desc(smem_u32(sA) + ks * 32, 16, 1024, 2);
          bd = desc(smem_u32(sB) + ks * 32, 16, 1024, 2);
        }
        uint32_t acc = (it | ks) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      if ((it & 15) == 15) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar)), "r"(phase));
        }
        phase ^= 1;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int N, int LAYOUT>
static void run(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(mma_kernel<N, LAYOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  mma_kernel<N, LAYOUT><<<sms, 128, smem>>>(16, cyc);
  cudaMemset(cyc, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  mma_kernel<N, LAYOUT><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double macs = (double)sms * iters * 4 * 128.0 * N * 32;
  const double cyc_per_mma = (double)c / sms / (iters * 4.0);
  printf("{\"variant\": \"%s\", \"N\": %d, \"err\": \"%s\", \"ms\": %.3f, \"tops\": %.1f, "
         "\"cycles_per_mma\": %.1f, \"macs_per_clk_sm\": %.0f}\n",
         name, N, cudaGetErrorString(cudaGetLastError()), ms, 2 * macs / (ms * 1e-3) / 1e12, cyc_per_mma,
         128.0 * N * 32 / cyc_per_mma);
  cudaFree(cyc);
}

// 2-CTA variant: cluster of 2, M=256 (128 per CTA), N (N/2 rows of B per CTA), leader issues.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  uint32_t cr;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * 128;
  for (int i = threadIdx.x; i < (128 + N / 2) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u * (i & 1), 0, 0x01010101u, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0 && cr == 0) {
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint64_t ad = desc(smem_u32(sA) + ks * 2 * 128 * 16, 128 * 16, 128, 0);
        uint64_t bd = desc(smem_u32(sB) + ks * 2 * (N / 2) * 16, (N / 2) * 16, 128, 0);
        uint32_t acc = (it | ks) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      if ((it & 15) == 15) {
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"((uint16_t)1));
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar)), "r"(phase));
        }
        phase ^= 1;
      }
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int N>
static void run2(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = (128 + N / 2) * 128 + 1024;
  cudaFuncSetAttribute(mma2_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  const int grid = sms / 2 * 2;
  mma2_kernel<N><<<grid, 128, smem>>>(16, cyc);
  cudaMemset(cyc, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  mma2_kernel<N><<<grid, 128, smem>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double macs = (double)(grid / 2) * iters * 4 * 256.0 * N * 32;
  printf("{\"variant\": \"%s\", \"N\": %d, \"err\": \"%s\", \"ms\": %.3f, \"tops\": %.1f}\n", name, N,
         cudaGetErrorString(cudaGetLastError()), ms, 2 * macs / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
}


// Pipelined 2-CTA replica of scan_tc2's MMA structure without data work:
// S stages; per stage the leader waits full[s] (arrivals from one producer warp
// in each CTA), issues KPS MMAs (M=256, N, K=32), commits to empty[s] in both
// CTAs; producers wait empty[s] and re-arrive.  ACC=1 adds the per-tile
// accumulator handshake (tfull / tempty with one epilogue warp per CTA).
__device__ __forceinline__ bool tryw(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint32_t mapa0(uint32_t a) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  return r;
}
template <int N, int S, int KPS, int ACC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma3_kernel(int tiles, int ktiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t full[S], empty[S], tfull[2], tempty[2];
  uint32_t cr;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * 128;
  for (int i = threadIdx.x; i < (128 + N / 2) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u * (i & 1), 0, 0x01010101u, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    for (int a = 0; a < 2; ++a) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull[a])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&tempty[a])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = tiles * ktiles;  // stages
  if (warp == 1) {        // producer: one warp per CTA
    int st = 0; uint32_t ph = 0;
    const uint32_t fdst = mapa0(smem_u32(&full[0]));
    for (int i = 0; i < total; ++i) {
      while (!tryw(smem_u32(&empty[st]), ph ^ 1u)) {}
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(fdst + 8u * st) : "memory");
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  } else if (warp == 0 && cr == 0) {   // MMA issuer
    if (lane == 0) {
      int st = 0; uint32_t ph = 0; int acc = 0; uint32_t aph = 0;
      for (int t = 0; t < tiles; ++t) {
        if (ACC) { while (!tryw(smem_u32(&tempty[acc]), aph ^ 1u)) {} asm volatile("tcgen05.fence::after_thread_sync;"); }
        for (int kt = 0; kt < ktiles; ++kt) {
          while (!tryw(smem_u32(&full[st]), ph)) {}
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int ks = 0; ks < KPS; ++ks) {
            uint64_t ad = desc(smem_u32(sA) + (ks & 3) * 2 * 128 * 16, 128 * 16, 128, 0);
            uint64_t bd = desc(smem_u32(sB) + (ks & 3) * 2 * (N / 2) * 16, (N / 2) * 16, 128, 0);
            uint32_t a = (kt | ks) ? 1u : 0u;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (ACC ? acc * 256 : 0)),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(a));
          }
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       ::"r"(smem_u32(&empty[st])), "h"((uint16_t)3));
          if (++st == S) { st = 0; ph ^= 1u; }
        }
        if (ACC) asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                              ::"r"(smem_u32(&tfull[acc])), "h"((uint16_t)3));
        if (++acc == 2) { acc = 0; aph ^= 1u; }
      }
    }
    __syncwarp();
  } else if (warp == 2 && ACC) {       // epilogue stand-in: release each accumulator
    int acc = 0; uint32_t aph = 0;
    const uint32_t tdst = mapa0(smem_u32(&tempty[0]));
    for (int t = 0; t < tiles; ++t) {
      while (!tryw(smem_u32(&tfull[acc]), aph)) {}
      asm volatile("tcgen05.fence::after_thread_sync;");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tdst + 8u * acc) : "memory");
      if (++acc == 2) { acc = 0; aph ^= 1u; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int S, int KPS, int ACC>
static void run3(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = (128 + N / 2) * 128 + 1024;
  cudaFuncSetAttribute(mma3_kernel<N, S, KPS, ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = sms / 2 * 2;
  const int ktiles = 24 / KPS, tiles = 600;   // K = 768 per tile
  mma3_kernel<N, S, KPS, ACC><<<grid, 128, smem>>>(4, ktiles);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  mma3_kernel<N, S, KPS, ACC><<<grid, 128, smem>>>(tiles, ktiles);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double macs = (double)(grid / 2) * tiles * 768.0 * 256.0 * N;
  printf("{\"variant\": \"%s\", \"N\": %d, \"S\": %d, \"mma_per_stage\": %d, \"acc_handshake\": %d, \"err\": \"%s\", \"ms\": %.3f, \"tops\": %.1f}\n",
         name, N, S, KPS, ACC, cudaGetErrorString(cudaGetLastError()), ms, 2 * macs / (ms * 1e-3) / 1e12);
}

int main() {
  run3<192, 8, 4, 0>("pipe");
  run3<192, 8, 4, 1>("pipe");
  run3<192, 8, 8, 1>("pipe");
  run3<192, 4, 8, 1>("pipe");
  run3<192, 8, 2, 1>("pipe");
  run3<256, 8, 4, 1>("pipe");

  run2<256>("2cta_noswizzle");
  run2<224>("2cta_noswizzle");
  run2<192>("2cta_noswizzle");
  run2<128>("2cta_noswizzle");
  run<224, 0>("noswizzle");
  run<224, 2>("sw128");
  run<256, 0>("noswizzle");
  run<256, 2>("sw128");
  run<128, 2>("sw128");
  return 0;
}
