// Microbenchmark: register-resident GF(2^128) multiply throughput on sm_100a (clk/product/SM).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1803_11301_b200/csrc/gf128.cuh"  // from tools/microbench/
using namespace fpm;
template <int CH>
__global__ void __launch_bounds__(256) prep_kernel(uint4* out, int iters, uint4 w0) {
  const GfPrep p = gf_prep(make_uint4(w0.x ^ threadIdx.x, w0.y, w0.z, w0.w));
  uint4 v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = make_uint4(threadIdx.x * 7 + c, c, blockIdx.x, 1);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = gf_mul_prep(p, v[c]);
  uint4 r = v[0];
#pragma unroll
  for (int c = 1; c < CH; ++c) r = x4(r, v[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int CH>
__global__ void __launch_bounds__(256) gen_kernel(uint4* out, int iters, uint4 w0) {
  uint4 w = make_uint4(w0.x ^ threadIdx.x, w0.y, w0.z, w0.w);
  uint4 v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = make_uint4(threadIdx.x * 7 + c, c, blockIdx.x, 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = gf_mul(w, v[c]);
    w.x += 1;
  }
  uint4 r = v[0];
#pragma unroll
  for (int c = 1; c < CH; ++c) r = x4(r, v[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <class K>
void run(const char* name, K k, int ctas_per_sm, int ch) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* out; cudaMalloc(&out, (size_t)sms * ctas_per_sm * 256 * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  k<<<sms * ctas_per_sm, 256>>>(out, 10, make_uint4(1, 2, 3, 4));
  cudaEventRecord(e0);
  k<<<sms * ctas_per_sm, 256>>>(out, iters, make_uint4(1, 2, 3, 4));
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double prods = (double)sms * ctas_per_sm * 256 * iters * ch;
  printf("%-10s ch=%d warps/SM=%2d: %.3f ms  %.2f clk/product/SM (at %.0f MHz)  %s\n", name, ch, ctas_per_sm * 8, ms,
         (ms * 1e-3 * clk * 1e3) / (prods / sms), clk / 1e3, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}
int main() {
  for (int c : {1, 2, 4}) {
    run("prep", prep_kernel<1>, c, 1);
    run("prep", prep_kernel<2>, c, 2);
    run("generic", gen_kernel<1>, c, 1);
    run("generic", gen_kernel<2>, c, 2);
  }
  return 0;
}
