// fpm_multi.cu -- fp_polymul over several GPUs from ONE process (the C-ABI's fpm_polymul_multi):
// the product sharded over P logical ranks as SURVEY.md 8(e) describes, with every cross-rank step a
// direct peer-memory access over NVLink (cudaDeviceEnablePeerAccess) ordered by CUDA events -- no
// host barrier, no staging copy.  A device may appear several times in the rank list (logical ranks
// on one GPU: the same code path with local "peer" pointers; that is how the tests run it).
//
// Rank g owns evaluation-vector elements [g m, (g+1) m), m = n_p / P:
//   forward conversion  operand a on rank 0, operand b on rank 1 (split by operand, not replicated)
//   encode              rank g encodes ITS columns straight from the converting rank's memory
//   top log2 P layers   fft_pair_kernel per layer: reads the partner's half from the partner's memory,
//                       writes this rank's other ping-pong buffer (bfly_pair_device with `out`)
//   local layers        the coset sub-FFTs, pointwise product, inverse local layers (tower fast path:
//                       radix-4 passes + fused tower tile pass, as fpm_shard_local_product_dev)
//   decode              rank g writes its columns of the 128-row product matrix into the converting
//                       ranks' arrays (peer stores)
//   inverse conversion  2^33-bit products: the two independent 2^32-bit blocks on ranks 0 and 1, the
//                       top pass fused into rank 0's block reading rank 1's final block (peer loads);
//                       smaller products: the whole array on rank 0
// Reference path replaced: fp_polymul -> run_pipeline<gf128> (proj/src/polymul.cpp:78-135, 223-239).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fpmul_b200.h"
#include "fpm_internal.h"

namespace fpm {
namespace {

struct DevScope {
  int prev = -1;
  explicit DevScope(int dev) {
    FPM_CUDA(cudaGetDevice(&prev));
    if (dev != prev) FPM_CUDA(cudaSetDevice(dev));
  }
  ~DevScope() { if (prev >= 0) cudaSetDevice(prev); }
};

// A pool buffer owned by one rank (allocated and freed on the rank's device and stream).
struct RankBuf {
  void* p = nullptr;
  int dev = 0;
  cudaStream_t s = nullptr;
  RankBuf() = default;
  RankBuf(const RankBuf&) = delete;
  RankBuf& operator=(const RankBuf&) = delete;
  void alloc(int d, cudaStream_t st, size_t bytes) {
    dev = d;
    s = st;
    DevScope g(dev);
    p = pool_alloc(bytes, s);
  }
  void release() {
    if (!p) return;
    int prev;
    if (cudaGetDevice(&prev) == cudaSuccess) {
      cudaSetDevice(dev);
      pool_free(p, s);
      cudaSetDevice(prev);
    }
    p = nullptr;
  }
  ~RankBuf() { release(); }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

struct Rank {
  int dev = 0;
  cudaStream_t s = nullptr;
  cudaEvent_t ev = nullptr;  // re-recorded after each step other ranks wait for
  RankBuf buf[4];            // ping-pong element buffers: a0, a1, b0, b1 (m elements each)
  Rank() = default;
  Rank(const Rank&) = delete;
  Rank& operator=(const Rank&) = delete;
  ~Rank() {  // also on an exception: drain the stream (it may still copy into the caller's buffer)
    if (s) {
      int prev;
      if (cudaGetDevice(&prev) == cudaSuccess) {
        cudaSetDevice(dev);
        cudaStreamSynchronize(s);
        for (auto& b : buf) b.release();
        if (ev) cudaEventDestroy(ev);
        cudaStreamDestroy(s);
        cudaSetDevice(prev);
      }
    }
  }
};

void enable_peer_access(const std::vector<int>& devs) {
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int ok = 0;
      FPM_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
      if (!ok) throw Error(kCuda, "fpm_polymul_multi: device " + std::to_string(a) + " cannot access device " +
                                      std::to_string(b) + " (no P2P / NVLink path)");
      DevScope g(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else FPM_CUDA(e);
    }
}

// FPM_SHARD_CVT=0: keep the conversions on ranks 0 and 1 at every P (the split by operand / block only).
bool sharded_conversion_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPM_SHARD_CVT");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

U128 twiddle(unsigned i, uint64_t b, U128 base) {  // C2P((base >> i) ^ 2b), butterfly.cpp:45-49
  U128 c;
  c.lo = i == 0 ? base.lo : (i < 64 ? (base.lo >> i) | (base.hi << (64 - i)) : base.hi >> (i - 64));
  c.hi = i == 0 ? base.hi : (i < 64 ? base.hi >> i : 0);
  c.lo ^= b << 1;
  c.hi ^= b >> 63;
  return host_cantor_to_poly(field_tables(), c);
}

}  // namespace

void polymul_multi(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c,
                   const std::vector<int>& devices) {
  const int P = (int)devices.size();
  if (P < 2 || (P & (P - 1)) || P > 64) throw Error(kInvalid, "fpm_polymul_multi: the rank count must be a power of two in [2, 64]");
  fpm_plan plan{};
  if (fpm_plan_mul(a_bits, b_bits, FPM_FIELD_GF128, &plan) != FPM_OK) throw Error(kInvalid, fpm_last_error());
  const unsigned l = plan.l, lgP = (unsigned)__builtin_ctz((unsigned)P);
  const uint64_t n = plan.n_bits, n_p = plan.n_p, m = n_p / P;
  if (m < 1024) throw Error(kInvalid, "fpm_polymul_multi: every rank needs >= 1024 elements (product too small for " +
                                          std::to_string(P) + " ranks)");
  const unsigned lp = l - lgP;
  const bool tower = fpm_shard_tower(lp) != 0;
  const U128 base = partition_base(l);
  std::vector<int> distinct(devices);
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  enable_peer_access(distinct);

  std::vector<Rank> R(P);
  for (int g = 0; g < P; ++g) {
    R[g].dev = devices[g];
    DevScope d(R[g].dev);
    FPM_CUDA(cudaStreamCreateWithFlags(&R[g].s, cudaStreamNonBlocking));
    FPM_CUDA(cudaEventCreateWithFlags(&R[g].ev, cudaEventDisableTiming));
    for (auto& bb : R[g].buf) bb.alloc(R[g].dev, R[g].s, m * 16);
  }
  auto mark = [&](int g) {
    DevScope d(R[g].dev);
    FPM_CUDA(cudaEventRecord(R[g].ev, R[g].s));
  };
  auto wait_all = [&](int g) {  // rank g's stream after every rank's last marked step
    for (int h = 0; h < P; ++h)
      if (h != g) FPM_CUDA(cudaStreamWaitEvent(R[g].s, R[h].ev, 0));
  };
  auto wait_one = [&](int g, int h) { if (h != g) FPM_CUDA(cudaStreamWaitEvent(R[g].s, R[h].ev, 0)); };
  auto wait_group = [&](int g, int q_per) {  // rank g's stream after its group's (g / q_per) last marks
    for (int h = g - g % q_per; h < g - g % q_per + q_per; ++h) wait_one(g, h);
  };

  // ---- forward conversions.  P >= 4 with 2^32-bit operands (a 2^33-bit product): each operand on Q =
  // P/2 ranks, phase by phase (sharded_forward); otherwise a on rank 0, b on rank 1 (n/2-bit arrays,
  // zero-padded).
  const uint64_t half_words = n / 128;
  const int Q = P / 2;
  auto pow2_at_least = [](size_t v) {
    size_t c = 32;
    while (c < v) c <<= 1;
    return c;
  };
  const bool shard_cvt = sharded_conversion_enabled() && P >= 4 && Q <= 4 && n == (uint64_t{1} << 33) &&
                         pow2_at_least(a_bits) == (uint64_t{1} << 32) && pow2_at_least(b_bits) == (uint64_t{1} << 32);
  std::vector<RankBuf> X(P), side(P);
  const uint64_t* xs[2] = {a, b};
  const size_t xb[2] = {a_bits, b_bits};
  RankPtrs owners[2] = {};  // per operand: the replicas holding its converted columns
  int nowners = 1;
  if (shard_cvt) {
    nowners = Q;
    for (int k = 0; k < 2; ++k) {
      for (int q = 0; q < Q; ++q) owners[k].p[q] = nullptr;
      for (int q = 0; q < Q; ++q) {
        const int g = k * Q + q;
        Rank& r = R[g];
        DevScope d(r.dev);
        X[g].alloc(r.dev, r.s, half_words * 8);
        side[g].alloc(r.dev, r.s, 256 * 2048 * sizeof(uint32_t));
        owners[k].p[q] = X[g].as<uint32_t>();
        // upload this rank's quarter of the chunks (its own PCIe link), zero beyond the operand
        const uint64_t qw = half_words / Q, w0 = (uint64_t)q * qw;
        const uint64_t wtot = (xb[k] + 63) / 64;
        const uint64_t have = wtot > w0 ? std::min(qw, wtot - w0) : 0;
        if (have) FPM_CUDA(cudaMemcpyAsync(X[g].as<uint64_t>() + w0, xs[k] + w0, have * 8, cudaMemcpyHostToDevice, r.s));
        if (have < qw) FPM_CUDA(cudaMemsetAsync(X[g].as<uint64_t>() + w0 + have, 0, (qw - have) * 8, r.s));
        if (xb[k] % 64 && wtot - 1 >= w0 && wtot - 1 < w0 + qw) {  // bits >= the operand length must be zero
          uint64_t last = 0;
          std::memcpy(&last, xs[k] + wtot - 1, 8);
          last &= (uint64_t{1} << (xb[k] % 64)) - 1;
          FPM_CUDA(cudaMemcpyAsync(X[g].as<uint64_t>() + wtot - 1, &last, 8, cudaMemcpyHostToDevice, r.s));
          FPM_CUDA(cudaStreamSynchronize(r.s));  // `last` lives on this stack frame
        }
        mark(g);
      }
    }
    // every phase: all ranks of a group run their share, then each pulls what it owns next
    auto phase = [&](auto&& fn) {
      for (int g = 0; g < P; ++g) {
        DevScope d(R[g].dev);
        wait_group(g, Q);
        fn(g / Q, g % Q, R[g].s);
      }
      for (int g = 0; g < P; ++g) mark(g);
    };
    auto regather = [&](int from, int to) {
      phase([&](int k, int q, cudaStream_t st) { b32_regather(owners[k].p[q], owners[k], from, to, q, Q, st); });
    };
    regather(kDistChunk, kDistWindow);
    phase([&](int k, int q, cudaStream_t st) {  // L1_outer over this rank's windows
      b32_l1_outer(owners[k].p[q], owners[k].p[q], side[k * Q + q].as<uint32_t>(), false, q, Q, st);
    });
    regather(kDistWindow, kDistChunk);
    phase([&](int k, int q, cudaStream_t st) {  // L1_outer's fix-up, L1_inner + T_r on this rank's chunks
      const uint32_t c0 = (uint32_t)(q * (256 / Q)), c1 = c0 + 256 / Q;
      b32_l1_outer_fix(owners[k].p[q], side[k * Q + Q - 1].as<uint32_t>(), false, c0, c1, st);
      b32_rows(owners[k].p[q] + (uint64_t)c0 * 256 * 2048, (uint64_t)(c1 - c0) * 256, false, st);
    });
    regather(kDistChunk, kDistColumn);
    phase([&](int k, int q, cudaStream_t st) { b32_cols(owners[k].p[q], false, q, Q, st); });  // T_d
  } else {
    for (int k = 0; k < 2; ++k) {
      Rank& r = R[k];
      DevScope d(r.dev);
      X[k].alloc(r.dev, r.s, half_words * 8);
      const uint64_t w = (xb[k] + 63) / 64;
      FPM_CUDA(cudaMemcpyAsync(X[k].p, xs[k], w * 8, cudaMemcpyHostToDevice, r.s));
      if (w < half_words) FPM_CUDA(cudaMemsetAsync(X[k].as<uint64_t>() + w, 0, (half_words - w) * 8, r.s));
      if (xb[k] % 64) {  // bits >= the operand length must be zero
        uint64_t last = 0;
        std::memcpy(&last, xs[k] + w - 1, 8);
        last &= (uint64_t{1} << (xb[k] % 64)) - 1;
        FPM_CUDA(cudaMemcpyAsync(X[k].as<uint64_t>() + w - 1, &last, 8, cudaMemcpyHostToDevice, r.s));
        FPM_CUDA(cudaStreamSynchronize(r.s));  // `last` lives on this stack frame
      }
      basis_cvt_device(X[k].as<uint32_t>(), pow2_at_least(xb[k]), xb[k], false, r.s);
      mark(k);
      owners[k].p[0] = X[k].as<uint32_t>();
    }
  }
  // ---- encode: every rank its own columns, read from the converting ranks' memory
  for (int g = 0; g < P; ++g) {
    Rank& r = R[g];
    DevScope d(r.dev);
    wait_all(g);
    for (int k = 0; k < 2; ++k)
      encode_cols_owners(owners[k], nowners, l, (uint64_t)g * m, m, r.buf[2 * k].as<uint4>(), 64, r.s, tower);
  }
  for (int g = 0; g < P; ++g) mark(g);
  int cur[2] = {0, 0};
  // ---- exchanged top layers (forward: i = l-1 .. lp; inverse: lp .. l-1)
  auto exchanged = [&](int k, unsigned i, bool inverse) {
    for (int g = 0; g < P; ++g) {
      Rank& r = R[g];
      DevScope d(r.dev);
      wait_all(g);
      const int partner = g ^ (1 << (i - lp));
      const int side = (g >> (i - lp)) & 1;
      const uint64_t blk = ((uint64_t)g * m) >> (i + 1);
      const U128 w = twiddle(i, blk, base);
      bfly_pair_device(R[g].buf[2 * k + cur[k]].as<uint4>(), R[partner].buf[2 * k + cur[k]].as<uint4>(), m, w, side,
                       inverse, r.s, tower, R[g].buf[2 * k + 1 - cur[k]].as<uint4>());
    }
    for (int g = 0; g < P; ++g) mark(g);
    cur[k] ^= 1;
  };
  for (int k = 0; k < 2; ++k)
    for (unsigned i = l; i-- > lp;) exchanged(k, i, false);
  // ---- local layers of both operands, pointwise product, local inverse layers (per rank)
  for (int g = 0; g < P; ++g) {
    Rank& r = R[g];
    DevScope d(r.dev);
    uint4* ea = r.buf[cur[0]].as<uint4>();
    uint4* eb = r.buf[2 + cur[1]].as<uint4>();
    U128 cb = base;  // coset base e_{l+64} ^ g m
    cb.lo ^= (uint64_t)g * m;
    if (tower) {
      const TwiddleSrc tw = make_twiddle_src(r.dev, lp, cb);
      const unsigned T = pipeline_tile_log2(lp);
      butterfly_top_device(ea, lp, T, false, tw, r.s, true, eb);  // both operands per launch
      butterfly_tile_tower_device(ea, eb, lp, T, tw, r.s);
      butterfly_top_device(eb, lp, T, true, tw, r.s, true);
    } else {
      butterfly_device(ea, lp, cb, false, r.s);
      butterfly_device(eb, lp, cb, false, r.s);
      pointwise_device(ea, eb, eb, m, r.s);
      butterfly_device(eb, lp, cb, true, r.s);
    }
  }
  for (int g = 0; g < P; ++g) mark(g);
  for (unsigned i = lp; i < l; ++i) exchanged(1, i, true);
  const uint64_t out_bits = a_bits + b_bits - 1, out_words = (out_bits + 63) / 64;
  if (shard_cvt) {
    // ---- sharded inverse: the lower 2^32-bit block on ranks [0, Q), the upper on [Q, 2Q), in the
    // operands' replicas (free once every rank's encode has read them: the exchanged layers already
    // ordered every rank after every encode).  Decode writes each column into its owner's replica.
    RankPtrs Yb[2] = {owners[0], owners[1]};
    for (int g = 0; g < P; ++g) {
      Rank& r = R[g];
      DevScope d(r.dev);
      wait_all(g);
      decode_cols_owners(r.buf[2 + cur[1]].as<uint4>(), m, (uint64_t)g * m, n_p, Yb[0], Yb[1], Q, r.s, tower);
    }
    for (int g = 0; g < P; ++g) mark(g);
    auto phase = [&](bool all, auto&& fn) {
      for (int g = 0; g < 2 * Q; ++g) {
        DevScope d(R[g].dev);
        if (all) wait_all(g);
        else wait_group(g, Q);
        fn(g / Q, g % Q, R[g].s);
      }
      for (int g = 0; g < P; ++g) mark(g);
    };
    auto regather = [&](bool all, int from, int to) {
      phase(all, [&](int k, int q, cudaStream_t st) { b32_regather(Yb[k].p[q], Yb[k], from, to, q, Q, st); });
    };
    phase(true, [&](int k, int q, cudaStream_t st) { b32_cols(Yb[k].p[q], true, q, Q, st); });  // T_d^-1
    regather(false, kDistColumn, kDistChunk);
    phase(false, [&](int k, int q, cudaStream_t st) {  // T_r^-1 + L1_inner^-1 on this rank's chunks
      const uint64_t c0 = (uint64_t)q * (256 / Q);
      b32_rows(Yb[k].p[q] + c0 * 256 * 2048, (uint64_t)(256 / Q) * 256, true, st);
    });
    regather(false, kDistChunk, kDistWindow);
    phase(false, [&](int k, int q, cudaStream_t st) {  // L1_outer^-1 over this rank's windows
      b32_l1_outer(Yb[k].p[q], Yb[k].p[q], side[k * Q + q].as<uint32_t>(), true, q, Q, st);
    });
    phase(false, [&](int k, int q, cudaStream_t st) {  // its fix-up: the chunks' first words (rank 0's windows)
      if (q == 0) b32_l1_outer_fix(Yb[k].p[0], side[k * Q + Q - 1].as<uint32_t>(), true, 0, 256, st);
    });
    // the 2^33-bit array's single top pass: lower block bit b ^= upper bit b - 1 (b in [1, 2^32)),
    // then the upper block's bit 0 ^= its last bit
    phase(true, [&](int k, int q, cudaStream_t st) {
      if (k == 0) b32_top_pass(Yb[0].p[q], Yb[1], q, Q, st);
    });
    phase(true, [&](int k, int q, cudaStream_t st) {
      if (k == 1 && q == 0) b32_top_bit_fix(Yb[1].p[0], Yb[1].p[Q - 1], st);
    });
    regather(true, kDistWindow, kDistChunk);
    // each rank copies its chunks out over its own PCIe link
    for (int g = 0; g < 2 * Q; ++g) {
      Rank& r = R[g];
      DevScope d(r.dev);
      const int k = g / Q, q = g % Q;
      const uint64_t per = (uint64_t{1} << 26) / Q, w0 = (uint64_t)k * (uint64_t{1} << 26) + (uint64_t)q * per;
      const uint64_t w1 = std::min(out_words, w0 + per);
      if (w0 < w1)
        FPM_CUDA(cudaMemcpyAsync(c + w0, reinterpret_cast<const uint64_t*>(Yb[k].p[q]) + (w0 - (uint64_t)k * (uint64_t{1} << 26)),
                                 (w1 - w0) * 8, cudaMemcpyDeviceToHost, r.s));
    }
  } else {
    // ---- decode into the converting ranks' product arrays
    const bool blocks = n == (uint64_t{1} << 33);  // two independent 2^32-bit blocks (+ the top pass)
    RankBuf Y[2];
    if (blocks) {
      Y[0].alloc(R[0].dev, R[0].s, n / 16);
      Y[1].alloc(R[1].dev, R[1].s, n / 16);
    } else {
      Y[0].alloc(R[0].dev, R[0].s, n / 8);
    }
    mark(0);
    mark(1);
    uint32_t* lo = Y[0].as<uint32_t>();
    uint32_t* hi = blocks ? Y[1].as<uint32_t>() : lo + 64 * (n_p / 32);
    for (int g = 0; g < P; ++g) {
      Rank& r = R[g];
      DevScope d(r.dev);
      wait_one(g, 0);
      wait_one(g, 1);
      decode_cols_split_device(r.buf[2 + cur[1]].as<uint4>(), m, (uint64_t)g * m, n_p, lo, hi, r.s, tower);
    }
    for (int g = 0; g < P; ++g) mark(g);
    if (blocks) {
      const uint64_t bw = (uint64_t{1} << 32) / 64;  // 64-bit words per block
      {
        DevScope d(R[1].dev);
        wait_all(1);
        basis_cvt_device(Y[1].as<uint32_t>(), uint64_t{1} << 32, uint64_t{1} << 32, true, R[1].s);
        mark(1);
      }
      {
        DevScope d(R[0].dev);
        wait_all(0);
        basis_cvt_block32_inverse(Y[0].as<uint32_t>(), Y[1].as<uint32_t>(), R[0].s);
        mark(0);
        FPM_CUDA(cudaMemcpyAsync(c, Y[0].p, std::min(bw, out_words) * 8, cudaMemcpyDeviceToHost, R[0].s));
      }
      {
        DevScope d(R[1].dev);
        wait_one(1, 0);
        top_bit_fix_device(Y[1].as<uint32_t>(), R[1].s);
        if (out_words > bw) FPM_CUDA(cudaMemcpyAsync(c + bw, Y[1].p, (out_words - bw) * 8, cudaMemcpyDeviceToHost, R[1].s));
      }
    } else {
      DevScope d(R[0].dev);
      wait_all(0);
      basis_cvt_device(lo, n, n, true, R[0].s);
      FPM_CUDA(cudaMemcpyAsync(c, Y[0].p, out_words * 8, cudaMemcpyDeviceToHost, R[0].s));
    }
  }
  for (int g = 0; g < P; ++g) {
    DevScope d(R[g].dev);
    FPM_CUDA(cudaStreamSynchronize(R[g].s));
  }
  if (out_bits % 64) c[out_words - 1] &= (uint64_t{1} << (out_bits % 64)) - 1;
}

}  // namespace fpm

using namespace fpm;

extern "C" fpm_status fpm_polymul_multi(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits,
                                        uint64_t* c, int field, const int* devices, int n_devices) {
  return fpm_guard([&] {
    if (!a_bits || !b_bits) return;
    if (!a || !b || !c || !devices) throw Error(kInvalid, "fpm_polymul_multi: null argument");
    fpm_plan p{};
    if (fpm_plan_mul(a_bits, b_bits, field, &p) != FPM_OK) throw Error(kInvalid, fpm_last_error());
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(kCuda, "no CUDA device available (the B200 path has no CPU fallback)");
    for (int g = 0; g < n_devices; ++g)
      if (devices[g] < 0 || devices[g] >= ndev) throw Error(kInvalid, "fpm_polymul_multi: device ordinal out of range");
    if (n_devices == 1) {  // one rank: the single-GPU pipeline
      const fpm_status st = fpm_polymul(a, a_bits, b, b_bits, c, field, devices[0], nullptr);
      if (st != FPM_OK) throw Error(st, fpm_last_error());
      return;
    }
    polymul_multi(a, a_bits, b, b_bits, c, std::vector<int>(devices, devices + n_devices));
  });
}

extern "C" fpm_status fpm_polymul_n(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c,
                                    int field, int n_gpus) {
  std::vector<int> devs(n_gpus > 0 ? n_gpus : 0);
  for (int g = 0; g < n_gpus; ++g) devs[g] = g;
  if (n_gpus < 1) return fpm_guard([&] { throw Error(kInvalid, "fpm_polymul_n: n_gpus must be >= 1"); });
  return fpm_polymul_multi(a, a_bits, b, b_bits, c, field, devs.data(), n_gpus);
}
