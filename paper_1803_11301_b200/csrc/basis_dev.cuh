// basis_dev.cuh -- device helpers for the basis-conversion fold passes (shared by k_basis.cu and
// k_batch.cu).  Pass semantics: proj/src/basis_convert.cpp:34-46 (see k_basis.cu).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "fpm_tables.h"

namespace fpm {

constexpr int kMaxTilePasses = 64;

struct PassList {
  int n;
  uint32_t S[kMaxTilePasses], D[kMaxTilePasses], m1[kMaxTilePasses], m2[kMaxTilePasses];
};

__device__ __forceinline__ uint32_t range_mask(int64_t lo, int64_t hi) {  // bits [lo, hi) of a word
  if (lo < 0) lo = 0;
  if (hi > 32) hi = 32;
  if (hi <= lo) return 0u;
  const uint32_t upper = hi == 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u);
  return upper & ~((1u << lo) - 1u);
}

template <class Src>
__device__ __forceinline__ uint32_t get32(Src src, uint64_t nwords, uint64_t pos) {
  const uint64_t i = pos >> 5;
  const uint32_t s = (uint32_t)(pos & 31);
  const uint32_t lo = i < nwords ? src[i] : 0u;
  if (!s) return lo;
  const uint32_t hi = i + 1 < nwords ? src[i + 1] : 0u;
  return __funnelshift_r(lo, hi, s);
}

// New value of word wi for pass (S, D) restricted to span-local target region [rlo, rhi).
template <class Src>
__device__ __forceinline__ uint32_t fold_word(Src src, uint64_t nwords, uint64_t wi, uint64_t S, uint64_t D,
                                              bool inverse, uint64_t rlo, uint64_t rhi) {
  const uint32_t old = src[wi];
  const uint64_t P = wi << 5;
  const uint64_t base = P & ~(S - 1);
  const int64_t p = (int64_t)(P - base);
  const uint32_t tmask = range_mask((int64_t)rlo - p, (int64_t)rhi - p);
  if (!tmask) return old;
  uint32_t v = get32(src, nwords, P + D) & tmask;
  if (!inverse) {
    const uint32_t m2 = tmask & range_mask(-1, (int64_t)S - 2 * (int64_t)D - p);
    if (m2) v ^= get32(src, nwords, P + 2 * D) & m2;
  }
  return old ^ v;
}

// Applies pl's passes to a tile of `words` 32-bit words held in shared buffer a (b is scratch of the
// same size).  Returns the buffer holding the result.  All threads of the CTA must call it.
__device__ __forceinline__ uint32_t* smem_passes(uint32_t* a, uint32_t* b, int words, const PassList& pl,
                                                 bool inverse) {
  for (int k = 0; k < pl.n; ++k) {
    const uint32_t S = pl.S[k], D = pl.D[k];
    if (S <= 32) {  // in-word pass (the reference's TailOp masks, basis_convert.cpp:186-238)
      const uint32_t m1 = pl.m1[k], m2 = pl.m2[k];
      for (int i = threadIdx.x; i < words; i += blockDim.x) {
        const uint32_t x = a[i];
        b[i] = x ^ ((x & m1) >> D) ^ ((x & m2) >> (2 * D));
      }
    } else {
      for (int i = threadIdx.x; i < words; i += blockDim.x)
        b[i] = fold_word(a, (uint64_t)words, (uint64_t)i, S, D, inverse, S / 2 - D, S - D);
    }
    __syncthreads();
    uint32_t* t = a;
    a = b;
    b = t;
  }
  return a;
}

// Host: fills a PassList for `passes` (in application order).
inline uint32_t host_span_mask(uint32_t S, uint32_t lo, uint32_t hi) {
  const uint32_t unit = (hi - lo >= 32) ? 0xFFFFFFFFu : (((1u << (hi - lo)) - 1u) << lo);
  uint32_t m = 0;
  for (uint32_t pos = 0; pos + S <= 32; pos += S) m |= unit << pos;
  return m;
}

inline PassList make_passlist(const std::vector<Pass>& passes, bool inverse) {
  PassList pl{};
  if (passes.size() > (size_t)kMaxTilePasses) throw std::runtime_error("basis_cvt: tile schedule too long");
  pl.n = (int)passes.size();
  for (int k = 0; k < pl.n; ++k) {
    const uint32_t S = (uint32_t)passes[k].span, D = (uint32_t)passes[k].shift;
    pl.S[k] = S;
    pl.D[k] = D;
    pl.m1[k] = S <= 32 ? host_span_mask(S, S / 2, S) : 0u;
    pl.m2[k] = (S <= 32 && !inverse) ? host_span_mask(S, S / 2 + D, S) : 0u;
  }
  return pl;
}

}  // namespace fpm
