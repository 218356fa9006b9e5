// expand_bench.cu -- throughput of the 2-bit -> int8 operand expansion
// (tc_common.cuh expand_block_store) alone (measurement tool, not part of
// libuq): WPS warps per SM sub-partition each expand 128-dim blocks of
// register-resident plane words into shared memory in a loop.  Prints cycles
// per block per warp and per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/expand_bench tools/expand_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2506_00528_b200/csrc/tc_common.cuh"

using namespace uq::tc;

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) expand_kernel(int iters, const uint4* seed, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int t = threadIdx.x;
  uint4 p = seed[t & 31], n = seed[32 + (t & 31)];
  n.x &= ~p.x; n.y &= ~p.y; n.z &= ~p.z; n.w &= ~p.w;
  uint8_t* base = smem + (t >> 3) * 128 + (t & 7) * 16;
  const uint32_t stride = WARPS * 32 * 16;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    expand_block_store(p, n, base, stride);
    p.x = p.x * 1664525u + 1013904223u;   // keep the inputs live and changing
    n.x = (n.x ^ (n.x >> 7)) & ~p.x;
  }
  __syncthreads();
  long long t1 = clock64();
  if (t == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
}

template <int WARPS>
static void run(int sms, const uint4* seed, unsigned long long* cyc) {
  const int iters = 4096;
  const int smem = WARPS * 32 * 16 * 8;
  cudaFuncSetAttribute(expand_kernel<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(cyc, 0, 8);
  expand_kernel<WARPS><<<sms, WARPS * 32, smem>>>(iters, seed, cyc);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double cyc_per_cta = (double)c / sms;
  printf("{\"warps_per_sm\": %d, \"warps_per_smsp\": %.2f, \"err\": \"%s\", \"cycles_per_block_per_warp\": %.1f, "
         "\"blocks_per_kcycle_per_sm\": %.2f}\n",
         WARPS, WARPS / 4.0, cudaGetErrorString(cudaGetLastError()), cyc_per_cta / iters,
         1000.0 * WARPS * iters / cyc_per_cta);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* seed;
  unsigned long long* cyc;
  cudaMalloc(&seed, 64 * sizeof(uint4));
  cudaMalloc(&cyc, 8);
  uint4 h[64];
  for (int i = 0; i < 64; ++i) h[i] = make_uint4(0x9e3779b9u * (i + 1), 0x85ebca6bu * (i + 3), 0xc2b2ae35u * (i + 5), 0x27d4eb2fu * (i + 7));
  cudaMemcpy(seed, h, sizeof(h), cudaMemcpyHostToDevice);
  run<4>(sms, seed, cyc);
  run<8>(sms, seed, cyc);
  run<12>(sms, seed, cyc);
  run<16>(sms, seed, cyc);
  return 0;
}
