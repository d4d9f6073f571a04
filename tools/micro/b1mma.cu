// Microbenchmark: legacy warp-level mma.sync throughput on sm_100a (b1 and.popc, s8).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void b1_kernel(unsigned* out, int iters) {
  unsigned a0 = threadIdx.x * 0x9E3779B9u, a1 = a0 ^ 0x1234567u, a2 = a0 * 3u, a3 = a1 * 5u;
  unsigned b0 = a0 ^ 0xdeadbeefu, b1 = a1 ^ 0x5555u;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[q][0]), "+r"(c[q][1]), "+r"(c[q][2]), "+r"(c[q][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0 + q), "r"(b1));
  }
  int s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void s8_kernel(unsigned* out, int iters) {
  unsigned a0 = threadIdx.x * 0x9E3779B9u, a1 = a0 ^ 0x1234567u, a2 = a0 * 3u, a3 = a1 * 5u;
  unsigned b0 = a0 ^ 0xdeadbeefu, b1 = a1 ^ 0x5555u;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[q][0]), "+r"(c[q][1]), "+r"(c[q][2]), "+r"(c[q][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0 + q), "r"(b1));
  }
  int s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 4096;
    for (int k = 0; k < 2; ++k) {
      b1_kernel<<<sms, 32 * warps>>>(out, 16);
      cudaEventRecord(e0);
      if (k == 0) b1_kernel<<<sms, 32 * warps>>>(out, iters); else s8_kernel<<<sms, 32 * warps>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double mmas = (double)sms * warps * iters * 8;
      printf("%s warps/SM=%d: %.3f ms, %.3f mma/clk/SM (at 1.9 GHz), err=%s\n", k ? "s8 m16n8k32" : "b1 m16n8k256", warps, ms,
             mmas / sms / (ms * 1e-3 * 1.9e9), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
