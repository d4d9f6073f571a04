// dram_pattern.cu -- HBM efficiency of the access shapes a column-block basis conversion would use:
// an array viewed as 2^16 rows x 8 KiB; segment g = (column block cb = g >> 16, row d = g & 0xFFFF)
// of S bytes at d * 8 KiB + cb * S, so consecutive segments walk DOWN a column (stride 8 KiB).
// Reports GB/s (read + write bytes) for S = 32..512 against a coalesced copy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint64_t kRows = 1 << 16, kRowBytes = 8192, kBytes = kRows * kRowBytes;  // 512 MiB

template <int S, bool STRIDED_READ, bool STRIDED_WRITE>
__global__ void seg_copy(const uint4* __restrict__ src, uint4* __restrict__ dst) {
  constexpr int V = S / 16;  // uint4 per segment
  const uint64_t nvec = kBytes / 16;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nvec; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = k / V, v = k % V;
    const uint64_t cb = g >> 16, d = g & 0xFFFF;
    const uint64_t strided = (d * kRowBytes + cb * S) / 16 + v;
    const uint4 x = src[STRIDED_READ ? strided : k];
    dst[STRIDED_WRITE ? strided : k] = x;
  }
}

template <int S, bool R, bool W>
void run(const char* name, uint4* a, uint4* b, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) seg_copy<S, R, W><<<sms * 8, 256>>>(a, b);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) seg_copy<S, R, W><<<sms * 8, 256>>>(a, b);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-28s S=%4d  %8.1f GB/s\n", name, S, 2.0 * kBytes * reps / (ms * 1e-3) / 1e9);
}

int main() {
  uint4 *a, *b;
  cudaMalloc(&a, kBytes);
  cudaMalloc(&b, kBytes);
  cudaMemset(a, 1, kBytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<512, false, false>("coalesced copy", a, b, sms);
  run<32, true, false>("strided read, linear write", a, b, sms);
  run<64, true, false>("strided read, linear write", a, b, sms);
  run<128, true, false>("strided read, linear write", a, b, sms);
  run<256, true, false>("strided read, linear write", a, b, sms);
  run<32, false, true>("linear read, strided write", a, b, sms);
  run<64, false, true>("linear read, strided write", a, b, sms);
  run<128, false, true>("linear read, strided write", a, b, sms);
  run<32, true, true>("strided both", a, b, sms);
  run<128, true, true>("strided both", a, b, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
