// peaks.cu -- microbenchmark of the CUDA-core pipes the popcount scan uses
// (POPC, LOP3) on the GPU at hand; prints one JSON line.  Measurement tool for
// the "alu" roofline, not part of libuq.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void popc_kernel(unsigned* out, unsigned seed) {
  unsigned v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = seed * (threadIdx.x + 1) + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = __popc(v[c]) ^ (v[c] + i);  // POPC + LOP3/IADD chain
  }
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void popc_only_kernel(unsigned* out, unsigned seed) {
  unsigned v[kChains], acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) { v[c] = seed * (threadIdx.x + 1) + c; acc[c] = 0; }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      v[c] = v[c] * 0x9E3779B1u + (unsigned)c;  // IMAD (fma pipe): independent data per chain
      acc[c] += __popc(v[c]);                   // POPC + IADD (alu pipe)
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void lop3_kernel(unsigned* out, unsigned seed) {
  unsigned a[kChains], b = seed ^ threadIdx.x, c = seed + threadIdx.x;
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = seed * (threadIdx.x + 3) + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = (a[k] & b) ^ (c | a[k]);  // one LOP3
  }
  unsigned s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s ^= a[k];
  if (s == 0x12345678u) out[0] = s;
}

template <typename K>
static double time_kernel(K kern, int sms, int ops_per_iter_chain, double* per_clk_sm, int clk_khz) {
  unsigned* out;
  cudaMalloc(&out, 4);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, threads>>>(out, 1);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 1 + r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = 5.0 * blocks * threads * (double)kIters * kChains * ops_per_iter_chain;
  const double rate = ops / (ms * 1e-3);
  *per_clk_sm = rate / (sms * (clk_khz * 1e3));
  cudaFree(out);
  return rate;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max boost)
  double p1, p2, p3;
  double r1 = time_kernel(popc_only_kernel, sms, 1, &p1, clk);
  double r2 = time_kernel(popc_kernel, sms, 1, &p2, clk);
  double r3 = time_kernel(lop3_kernel, sms, 1, &p3, clk);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"popc_per_s\": %.4e, \"popc_per_clk_sm_at_attr_clock\": %.2f, "
         "\"popc_chain_per_s\": %.4e, \"lop3_per_s\": %.4e, \"lop3_per_clk_sm_at_attr_clock\": %.2f}\n",
         sms, clk, r1, p1, r2, r3, p3);
  return 0;
}
