// Microbenchmarks that decide the GF(2^128) multiply strategy on B200 (sm_100a).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o ubench ubench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

struct U128 { uint64_t lo, hi; };

// ---------------- host reference: bit-serial mod x^128+x^7+x^2+x+1 -------------
static U128 host_mul(U128 a, U128 b) {
  U128 acc{0, 0};
  for (int i = 127; i >= 0; --i) {
    uint64_t carry = acc.hi >> 63;
    acc.hi = (acc.hi << 1) | (acc.lo >> 63);
    acc.lo <<= 1;
    if (carry) acc.lo ^= 0x87;
    uint64_t bit = i >= 64 ? (b.hi >> (i - 64)) & 1 : (b.lo >> i) & 1;
    if (bit) { acc.lo ^= a.lo; acc.hi ^= a.hi; }
  }
  return acc;
}

// ---------------- device: clmul32 via integer multiply with 4-bit holes ---------
__device__ __forceinline__ uint64_t clmul32(uint32_t a, uint32_t b) {
  const uint32_t m = 0x11111111u;
  uint32_t a0 = a & m, a1 = a & (m << 1), a2 = a & (m << 2), a3 = a & (m << 3);
  uint32_t b0 = b & m, b1 = b & (m << 1), b2 = b & (m << 2), b3 = b & (m << 3);
  uint64_t r0 = (uint64_t)a0 * b0 ^ (uint64_t)a1 * b3 ^ (uint64_t)a2 * b2 ^ (uint64_t)a3 * b1;
  uint64_t r1 = (uint64_t)a0 * b1 ^ (uint64_t)a1 * b0 ^ (uint64_t)a2 * b3 ^ (uint64_t)a3 * b2;
  uint64_t r2 = (uint64_t)a0 * b2 ^ (uint64_t)a1 * b1 ^ (uint64_t)a2 * b0 ^ (uint64_t)a3 * b3;
  uint64_t r3 = (uint64_t)a0 * b3 ^ (uint64_t)a1 * b2 ^ (uint64_t)a2 * b1 ^ (uint64_t)a3 * b0;
  const uint64_t M = 0x1111111111111111ull;
  return (r0 & M) | (r1 & (M << 1)) | (r2 & (M << 2)) | (r3 & (M << 3));
}

__device__ __forceinline__ void clmul64(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
  uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  uint64_t p0 = clmul32(a0, b0), p2 = clmul32(a1, b1), p1 = clmul32(a0 ^ a1, b0 ^ b1) ^ p0 ^ p2;
  lo = p0 ^ (p1 << 32);
  hi = p2 ^ (p1 >> 32);
}

__device__ __forceinline__ uint4 gfmul_imad(uint4 a, uint4 b) {
  uint64_t al = a.x | ((uint64_t)a.y << 32), ah = a.z | ((uint64_t)a.w << 32);
  uint64_t bl = b.x | ((uint64_t)b.y << 32), bh = b.z | ((uint64_t)b.w << 32);
  uint64_t c0l, c0h, c2l, c2h, c1l, c1h;
  clmul64(al, bl, c0l, c0h);
  clmul64(ah, bh, c2l, c2h);
  clmul64(al ^ ah, bl ^ bh, c1l, c1h);
  c1l ^= c0l ^ c2l; c1h ^= c0h ^ c2h;
  // 256-bit product: [c0l, c0h^c1l, c2l^c1h, c2h]
  uint64_t r0 = c0l, r1 = c0h ^ c1l, r2 = c2l ^ c1h, r3 = c2h;
  // reduce hi = (r2,r3) mod x^128 + x^7 + x^2 + x + 1
  uint64_t o = (r3 >> 63) ^ (r3 >> 62) ^ (r3 >> 57);
  r2 ^= o;
  r1 ^= r3 ^ (r3 << 1) ^ (r3 << 2) ^ (r3 << 7) ^ (r2 >> 63) ^ (r2 >> 62) ^ (r2 >> 57);
  r0 ^= r2 ^ (r2 << 1) ^ (r2 << 2) ^ (r2 << 7);
  return make_uint4((uint32_t)r0, (uint32_t)(r0 >> 32), (uint32_t)r1, (uint32_t)(r1 >> 32));
}

// bit-serial (shift/mask) for contrast
__device__ __forceinline__ uint4 gfmul_serial(uint4 a, uint4 b) {
  uint64_t al = a.x | ((uint64_t)a.y << 32), ah = a.z | ((uint64_t)a.w << 32);
  uint64_t bl = b.x | ((uint64_t)b.y << 32), bh = b.z | ((uint64_t)b.w << 32);
  uint64_t zl = 0, zh = 0;
#pragma unroll 8
  for (int i = 127; i >= 0; --i) {
    uint64_t carry = zh >> 63;
    zh = (zh << 1) | (zl >> 63);
    zl = (zl << 1) ^ (0x87 & (0 - carry));
    uint64_t bit = ((i >= 64 ? bh >> (i - 64) : bl >> i) & 1);
    uint64_t mk = 0 - bit;
    zl ^= al & mk; zh ^= ah & mk;
  }
  return make_uint4((uint32_t)zl, (uint32_t)(zl >> 32), (uint32_t)zh, (uint32_t)(zh >> 32));
}

// ---------------- throughput kernels ------------------------------------------
__global__ void k_lop3(uint32_t* out, int iters, uint32_t s) {
  uint32_t a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * (k + 1) ^ s;
  uint32_t b = s * 3, c = s * 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
  }
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) r ^= a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_imadw(uint64_t* out, int iters, uint32_t s) {
  uint64_t a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * (k + 1) ^ s;
  uint32_t b = s * 3 | 1, c = s * 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[k]) : "r"(b), "r"(c ^ k));
  }
  uint64_t r = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) r ^= a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int KIND>
__global__ void k_gfmul(const uint4* __restrict__ in, const uint4* __restrict__ tw, uint4* out, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint4 x = in[i];
  uint4 w = tw[i & 1023];
  for (int it = 0; it < iters; ++it) {
    uint4 p = KIND == 0 ? gfmul_imad(w, x) : gfmul_serial(w, x);
    x.x ^= p.x; x.y ^= p.y; x.z ^= p.z; x.w ^= p.w;   // butterfly-like dependence
  }
  out[i] = x;
}

// M4R: 16 chunks x 256 entries x 16 B = 64 KiB table of w * (byte << 8c)
__global__ void k_m4r(const uint4* __restrict__ in, const uint4* __restrict__ table_g, uint4* out, int n, int iters) {
  extern __shared__ uint4 tab[];
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) tab[e] = table_g[e];
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint4 x = in[i];
  for (int it = 0; it < iters; ++it) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      uint32_t byte = __byte_perm(w4[c >> 2], 0, 0x4440 + (c & 3));
      uint4 t = tab[c * 256 + byte];
      acc.x ^= t.x; acc.y ^= t.y; acc.z ^= t.z; acc.w ^= t.w;
    }
    x.x ^= acc.x; x.y ^= acc.y; x.z ^= acc.z; x.w ^= acc.w;
  }
  out[i] = x;
}

// 4-bit M4R with 8-way bank-group replication: lane uses copy (lane & 7)
__global__ void k_m4r4(const uint4* __restrict__ in, const uint4* __restrict__ table_g, uint4* out, int n, int iters) {
  extern __shared__ uint4 tab[];  // 512 entries x 8 copies
  for (int e = threadIdx.x; e < 512 * 8; e += blockDim.x) tab[e] = table_g[e >> 3];
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cp = threadIdx.x & 7;
  uint4 x = in[i];
  for (int it = 0; it < iters; ++it) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      uint32_t nib = (w4[c >> 3] >> (4 * (c & 7))) & 15;
      uint4 t = tab[((c * 16 + nib) << 3) + cp];
      acc.x ^= t.x; acc.y ^= t.y; acc.z ^= t.z; acc.w ^= t.w;
    }
    x.x ^= acc.x; x.y ^= acc.y; x.z ^= acc.z; x.w ^= acc.w;
  }
  out[i] = x;
}

__global__ void k_mma_b1(int* out, int iters, uint32_t s) {
  uint32_t a0 = threadIdx.x * 7 ^ s, a1 = threadIdx.x * 13 ^ s, b0 = s ^ threadIdx.x;
  int c[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m16n8k128.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
        : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3]) : "r"(a0 + k), "r"(a1), "r"(b0));
  }
  int r = 0;
  for (int k = 0; k < 4; ++k) r ^= c[k][0] ^ c[k][1] ^ c[k][2] ^ c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float t; cudaEventElapsedTime(&t, a, b); return t; }

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int sms = pr.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s sms=%d clock=%d MHz\n", pr.name, sms, clk_khz / 1000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  const int nthreads = threads * blocks;
  void* scratch; CK(cudaMalloc(&scratch, (size_t)nthreads * 64));

  { // LOP3
    int iters = 20000;
    k_lop3<<<blocks, threads>>>((uint32_t*)scratch, 100, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_lop3<<<blocks, threads>>>((uint32_t*)scratch, iters, 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ops = (double)nthreads * iters * 8; double ms = time_ms(e0, e1);
    printf("LOP3: %.3f ms  %.2f Tops/s  %.1f ops/clk/SM(at %d MHz)\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz/1000);
  }
  { // IMAD.WIDE
    int iters = 20000;
    k_imadw<<<blocks, threads>>>((uint64_t*)scratch, 100, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_imadw<<<blocks, threads>>>((uint64_t*)scratch, iters, 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ops = (double)nthreads * iters * 8; double ms = time_ms(e0, e1);
    printf("IMAD.WIDE: %.3f ms  %.2f Tops/s  %.1f ops/clk/SM\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk_khz * 1e3));
  }
  { // b1 mma (emulated on sm_100a)
    int iters = 2000;
    k_mma_b1<<<blocks, threads>>>((int*)scratch, 10, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_mma_b1<<<blocks, threads>>>((int*)scratch, iters, 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double mmas = (double)nthreads / 32 * iters * 4; double ms = time_ms(e0, e1);
    printf("mma.b1 m16n8k128: %.3f ms  %.2f G mma/s  %.3f mma/clk/SM  (=%.1f T bitMAC/s)\n", ms, mmas / ms / 1e6,
           mmas / (ms * 1e-3) / sms / (clk_khz * 1e3), mmas * 16384 / ms / 1e9);
  }
  // GF mult correctness + throughput
  const int n = nthreads;
  std::mt19937_64 rng(42);
  std::vector<U128> hin(n), htw(1024);
  for (auto& v : hin) v = {rng(), rng()};
  for (auto& v : htw) v = {rng(), rng()};
  uint4 *din, *dtw, *dout, *dtab;
  CK(cudaMalloc(&din, n * 16)); CK(cudaMalloc(&dtw, 1024 * 16)); CK(cudaMalloc(&dout, n * 16)); CK(cudaMalloc(&dtab, 4096 * 16));
  CK(cudaMemcpy(din, hin.data(), n * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtw, htw.data(), 1024 * 16, cudaMemcpyHostToDevice));
  for (int kind = 0; kind < 2; ++kind) {
    auto launch = [&](int iters) {
      if (kind == 0) k_gfmul<0><<<(n + 255) / 256, 256>>>(din, dtw, dout, n, iters);
      else k_gfmul<1><<<(n + 255) / 256, 256>>>(din, dtw, dout, n, iters);
    };
    launch(1); CK(cudaDeviceSynchronize());
    std::vector<U128> hout(n); CK(cudaMemcpy(hout.data(), dout, n * 16, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < 4096; ++i) {
      U128 p = host_mul(htw[i & 1023], hin[i]);
      U128 want{hin[i].lo ^ p.lo, hin[i].hi ^ p.hi};
      if (want.lo != hout[i].lo || want.hi != hout[i].hi) ++bad;
    }
    int iters = kind == 0 ? 200 : 20;
    cudaEventRecord(e0); launch(iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ms = time_ms(e0, e1), muls = (double)n * iters;
    printf("gfmul %s: bad=%d  %.3f ms  %.2f G mul/s  %.2f clk/mul/SM\n", kind == 0 ? "imad-karatsuba" : "bit-serial", bad, ms,
           muls / ms / 1e6, (ms * 1e-3) * sms * (clk_khz * 1e3) / muls);
  }
  { // M4R 8-bit table
    std::vector<U128> tab(4096);
    U128 w = htw[0];
    for (int c = 0; c < 16; ++c)
      for (int v = 0; v < 256; ++v) {
        U128 x{0, 0};
        int pos = 8 * c;
        for (int b = 0; b < 8; ++b) if (v >> b & 1) { int k = pos + b; if (k < 64) x.lo |= 1ull << k; else x.hi |= 1ull << (k - 64); }
        tab[c * 256 + v] = host_mul(w, x);
      }
    CK(cudaMemcpy(dtab, tab.data(), 4096 * 16, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_m4r, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    k_m4r<<<(n + 255) / 256, 256, 65536>>>(din, dtab, dout, n, 1); CK(cudaDeviceSynchronize());
    std::vector<U128> hout(n); CK(cudaMemcpy(hout.data(), dout, n * 16, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < 4096; ++i) { U128 p = host_mul(w, hin[i]); if ((hin[i].lo ^ p.lo) != hout[i].lo || (hin[i].hi ^ p.hi) != hout[i].hi) ++bad; }
    int iters = 200;
    cudaEventRecord(e0); k_m4r<<<(n + 255) / 256, 256, 65536>>>(din, dtab, dout, n, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ms = time_ms(e0, e1), muls = (double)n * iters;
    printf("gfmul m4r-8bit smem: bad=%d  %.3f ms  %.2f G mul/s  %.2f clk/mul/SM\n", bad, ms, muls / ms / 1e6, (ms * 1e-3) * sms * (clk_khz * 1e3) / muls);
    // 4-bit replicated
    std::vector<U128> tab4(512);
    for (int c = 0; c < 32; ++c)
      for (int v = 0; v < 16; ++v) {
        U128 x{0, 0};
        for (int b = 0; b < 4; ++b) if (v >> b & 1) { int k = 4 * c + b; if (k < 64) x.lo |= 1ull << k; else x.hi |= 1ull << (k - 64); }
        tab4[c * 16 + v] = host_mul(w, x);
      }
    CK(cudaMemcpy(dtab, tab4.data(), 512 * 16, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_m4r4, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    k_m4r4<<<(n + 255) / 256, 256, 65536>>>(din, dtab, dout, n, 1); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hout.data(), dout, n * 16, cudaMemcpyDeviceToHost));
    bad = 0;
    for (int i = 0; i < 4096; ++i) { U128 p = host_mul(w, hin[i]); if ((hin[i].lo ^ p.lo) != hout[i].lo || (hin[i].hi ^ p.hi) != hout[i].hi) ++bad; }
    cudaEventRecord(e0); k_m4r4<<<(n + 255) / 256, 256, 65536>>>(din, dtab, dout, n, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    ms = time_ms(e0, e1);
    printf("gfmul m4r-4bit x8 smem: bad=%d  %.3f ms  %.2f G mul/s  %.2f clk/mul/SM\n", bad, ms, muls / ms / 1e6, (ms * 1e-3) * sms * (clk_khz * 1e3) / muls);
  }
  { // HBM copy
    size_t bytes = (size_t)2 << 30; void *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    cudaMemset(a, 1, bytes); cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0); cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ms = time_ms(e0, e1); printf("D2D copy 2GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
  }
  return 0;
}
