// Microbenchmark: per-SM throughput of IMAD.WIDE.U32, IMAD (32-bit), LOP3 on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void __launch_bounds__(256) k(uint32_t* out, int iters, uint32_t s) {
  uint32_t a[8], b[8];
  uint64_t acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * (j + 3) ^ s; b[j] = a[j] * 0x9E3779B9u; acc[j] = j; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (OP == 0) acc[j] = (uint64_t)(uint32_t)acc[j] * b[(j + r) & 7] + acc[j];                     // IMAD.WIDE
        if (OP == 1) acc[j] = (uint32_t)acc[j] * a[(j + r) & 7] + b[j];                        // IMAD
        if (OP == 2) { uint32_t x = (uint32_t)acc[j]; asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(a[(j + r) & 7]), "r"(b[j])); acc[j] = x; }  // LOP3
      }
  }
  uint32_t r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= (uint32_t)acc[j] ^ (uint32_t)(acc[j] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int OP>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, sms * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  k<OP><<<sms * 8, 256>>>(out, 10, 1);
  cudaEventRecord(e0);
  k<OP><<<sms * 8, 256>>>(out, iters, 1);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ops = (double)sms * 8 * 256 * iters * 32;
  printf("%-10s %.3f ms  %.1f thread-ops/clk/SM\n", name, ms, ops / sms / (ms * 1e-3 * clk * 1e3));
}
int main() { run<0>("IMAD.WIDE"); run<1>("IMAD"); run<2>("LOP3"); return 0; }
