// scores.cu -- dense Delta matrix (test/debug entry point uq_scores) and the
// code-validity check uq_check_codes.
//
// uq_scores evaluates the paper's b2sp literally:
//   (bsp(q+,r+) + bsp(q-,r-)) - (bsp(q+,r-) + bsp(q-,r+)),  bsp = popc(AND)
// so it is also correct on invalid codes (it does not use the 2-popcount
// identity of the scan kernels).
#include "common.cuh"
#include "internal.h"

namespace uq {

__global__ void __launch_bounds__(128) scores_kernel(const uint8_t* __restrict__ q, int64_t nq,
                                                     const uint8_t* __restrict__ db, int64_t n,
                                                     int32_t d, int32_t* __restrict__ out) {
  extern __shared__ uint4 s_q[];
  const int NB = blocks128(d);
  const int64_t pb = plane_bytes(d), cb = 2 * pb;
  const int64_t qi = blockIdx.y;
  for (int i = threadIdx.x; i < 2 * NB; i += blockDim.x)
    s_q[i] = reinterpret_cast<const uint4*>(q + qi * cb)[i];
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint4* rp = reinterpret_cast<const uint4*>(db + r * cb);
  const uint4* rn = reinterpret_cast<const uint4*>(db + r * cb + pb);
  int s = 0;
  for (int b = 0; b < NB; ++b) {
    const uint4 a = s_q[b], an = s_q[NB + b], x = __ldg(rp + b), xn = __ldg(rn + b);
    s += __popc(a.x & x.x) + __popc(a.y & x.y) + __popc(a.z & x.z) + __popc(a.w & x.w);
    s += __popc(an.x & xn.x) + __popc(an.y & xn.y) + __popc(an.z & xn.z) + __popc(an.w & xn.w);
    s -= __popc(a.x & xn.x) + __popc(a.y & xn.y) + __popc(a.z & xn.z) + __popc(a.w & xn.w);
    s -= __popc(an.x & x.x) + __popc(an.y & x.y) + __popc(an.z & x.z) + __popc(an.w & x.w);
  }
  out[qi * n + r] = s;
}

cudaError_t launch_scores(const uint8_t* q, int64_t nq, const uint8_t* db, int64_t n, int32_t d,
                          int32_t* out, cudaStream_t st) {
  if (nq == 0 || n == 0) return cudaSuccess;
  for (int64_t q0 = 0; q0 < nq; q0 += 65535) {
    const int64_t qn = (nq - q0 < 65535) ? nq - q0 : 65535;
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)qn);
    scores_kernel<<<grid, 128, 2 * blocks128(d) * 16, st>>>(q + q0 * code_bytes(d), qn, db, n, d,
                                                            out + q0 * n);
    note_launch();
  }
  return cudaGetLastError();
}

// Invalid row: a position in both planes, or a set bit at index >= d.
__global__ void check_codes_kernel(const uint8_t* __restrict__ codes, int64_t n, int32_t d,
                                   unsigned long long* bad) {
  const int NB = blocks128(d);
  const int64_t pb = plane_bytes(d), cb = 2 * pb;
  unsigned long long local = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(codes + r * cb);
    const uint32_t* m = reinterpret_cast<const uint32_t*>(codes + r * cb + pb);
    uint32_t viol = 0;
    for (int w = 0; w < NB * 4; ++w) {
      uint32_t both = p[w] & m[w];
      uint32_t any = p[w] | m[w];
      const int lo = w * 32;
      uint32_t padmask = (lo >= d) ? 0xffffffffu : (d - lo >= 32 ? 0u : (0xffffffffu << (d - lo)));
      viol |= both | (any & padmask);
    }
    local += viol ? 1ull : 0ull;
  }
  local = __reduce_add_sync(kFull, (unsigned)local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}

cudaError_t launch_check_codes(const uint8_t* codes, int64_t n, int32_t d, unsigned long long* bad,
                               int sms, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  check_codes_kernel<<<(unsigned)blocks, 256, 0, st>>>(codes, n, d, bad);
  note_launch();
  return cudaGetLastError();
}

}  // namespace uq
