// fpm_capi.cu -- the C-ABI (include/fpmul_b200.h): device tables, the fp_polymul pipeline and
// the stage entry points.  The pipeline follows run_pipeline<gf128> (proj/src/polymul.cpp:78-135):
//
//   per operand X in (a, b):  load+zero-pad -> basis_cvt -> encode -> forward butterflies
//   pointwise -> inverse butterflies -> decode -> i_basis_cvt -> trim (polymul.cpp:237)
//
// B200 specifics: everything stays in HBM (inputs are read once, the product written once); the
// bottom 12 butterfly layers run on 64 KiB shared-memory tiles and the pointwise product is fused
// between operand b's last forward tile layers and the first inverse tile layers; products with
// n <= 2^17 bits run whole inside one CTA (k_batch.cu).  There is no CPU fallback: without a
// device every entry point returns FPM_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <tuple>
#include <exception>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "../../include/fpmul_b200.h"
#include "fpm_internal.h"
#include "gf128.cuh"

namespace fpm {
namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

template <class Fn>
fpm_status guard(Fn&& fn) {
  try {
    fn();
    return FPM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    // a failed runtime call also stays behind as the thread's "last error": clear it, or the next
    // call's launch check (cudaGetLastError) would report this call's failure as its own
    if (e.code == kCuda) cudaGetLastError();
    return (fpm_status)e.code;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return FPM_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FPM_ECUDA;
  }
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw Error(kCuda, std::string("no CUDA device available (the B200 path has no CPU fallback): ") +
                           (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
}

inline uint4 to4(U128 v) { return make_uint4((uint32_t)v.lo, (uint32_t)(v.lo >> 32), (uint32_t)v.hi, (uint32_t)(v.hi >> 32)); }

// ------------------------------------------------------------------ small helper kernels
// dst[0 .. dst_words) <- src bits [0, src_bits), zero above.
__global__ void load_operand_kernel(uint64_t* __restrict__ dst, uint64_t dst_words, const uint64_t* __restrict__ src,
                                    uint64_t src_bits) {
  pdl_wait();
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < dst_words; k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = 0;
    if (k * 64 < src_bits) {
      v = src[k];
      if (src_bits - k * 64 < 64) v &= (((uint64_t)1) << (src_bits - k * 64)) - 1;
    }
    dst[k] = v;
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void store_product_kernel(uint64_t* __restrict__ dst, const uint64_t* __restrict__ src, uint64_t out_bits,
                                     uint64_t k0, uint64_t k1) {
  pdl_wait();
  const uint64_t words = (out_bits + 63) / 64;
  for (uint64_t k = k0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < k1; k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = src[k];
    if (k == words - 1 && (out_bits & 63)) v &= (((uint64_t)1) << (out_bits & 63)) - 1;
    dst[k] = v;
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

int grid_1d(uint64_t n, int per_sm = 16) {
  int dev, sms;
  FPM_CUDA(cudaGetDevice(&dev));
  FPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t g = std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * per_sm);
  return (int)(g ? g : 1);
}

// ------------------------------------------------------------------ plan (polymul.cpp:187-219)
unsigned log2_ceil(size_t n) {
  unsigned l = 0;
  while (((size_t)1 << l) < n) ++l;
  return l;
}
bool field_supports(unsigned m, size_t n_bits) {  // polymul.cpp:45-49
  if (n_bits < m) return false;
  const unsigned l = log2_ceil(n_bits) - log2_ceil(m);
  return l < m / 2 && l + 1 < m / 2;
}
fpm_plan plan_mul(size_t a_bits, size_t b_bits, int field) {
  if (a_bits == 0 || b_bits == 0) throw Error(kInvalid, "plan_mul: input lengths must be positive");
  const size_t mx = a_bits > b_bits ? a_bits : b_bits;
  if (mx > ((size_t)1 << 62)) throw Error(kInvalid, "plan_mul: input length out of range");
  size_t n = (size_t)1 << log2_ceil(2 * mx);
  unsigned m = 0;
  if (field == FPM_FIELD_GF64) m = 64;
  else if (field == FPM_FIELD_GF128) m = 128;
  else if (field == FPM_FIELD_AUTO) m = field_supports(64, n < 64 ? 64 : n) ? 64 : 128;
  else throw Error(kInvalid, "plan_mul: unknown field choice");
  if (n < m) n = m;
  if (!field_supports(m, n)) throw Error(kInvalid, "plan_mul: length exceeds the field's supported bound");
  fpm_plan p{};
  p.n_bits = n;
  p.log2_n = log2_ceil(n);
  p.field_degree = m;
  p.log2_field_degree = m == 64 ? 6 : 7;
  p.l = p.log2_n - p.log2_field_degree;
  p.n_p = (uint64_t)1 << p.l;
  return p;
}

// ------------------------------------------------------------------ stage timing
struct StageClock {
  cudaStream_t s;
  double* out;
  std::vector<std::pair<int, cudaEvent_t>> marks;
  StageClock(cudaStream_t st, double* o) : s(st), out(o) {}
  void mark(int stage) {  // stage = index the interval ending at the NEXT mark belongs to
    if (!out) return;
    cudaEvent_t e;
    FPM_CUDA(cudaEventCreate(&e));
    FPM_CUDA(cudaEventRecord(e, s));
    marks.emplace_back(stage, e);
  }
  void finish() {
    if (!out) return;
    mark(-1);
    FPM_CUDA(cudaEventSynchronize(marks.back().second));
    for (size_t k = 0; k + 1 < marks.size(); ++k) {
      float ms = 0;
      FPM_CUDA(cudaEventElapsedTime(&ms, marks[k].second, marks[k + 1].second));
      if (marks[k].first >= 0) out[marks[k].first] += ms * 1e-3;
    }
    for (auto& m : marks) cudaEventDestroy(m.second);
    marks.clear();
  }
};
enum { kStBasis = 0, kStEncode, kStBfly, kStPointwise, kStIBfly, kStDecode, kStIBasis };


// Host-buffer pipelining for fpm_polymul: the compute stream waits for operand k's upload only
// right before operand k is first read (operand b's copy overlaps operand a's transforms), and
// product words are copied to h_out on the d2h stream as soon as the inverse basis conversion has
// finished them (the upper half overlaps the lower half's conversion at 2^33 bits).
struct HostIO {
  cudaEvent_t ready[2] = {nullptr, nullptr};
  uint64_t* h_out = nullptr;
  cudaStream_t d2h = nullptr;
  // no other host-buffer call in flight on this device: the GPU idles while operand b is uploaded,
  // and part of operand a's tile layers runs in that window (with concurrent callers the window is
  // another caller's compute time, and the split pass would only add table builds)
  bool alone = true;
};

// Field plumbing of run_pipeline<F> (polymul.cpp:78-135) for the two fields built on the GPU.
struct Gf128Ops {
  using E = uint4;
  static constexpr int kM = 128;
  using Tw = TwiddleSrc;
  static constexpr int kLiveRows = 64;  // rows >= m/2 of a padded operand are zero
  static Tw twiddles(int dev, unsigned l) { return make_twiddle_src(dev, l, partition_base(l)); }
  static unsigned tile_log2(unsigned l) { return pipeline_tile_log2(l); }
  // The fused pass on tower-representation tiles (tower.cuh); then encode, the top passes and
  // decode work in R as well.
  static bool tower(unsigned T) { return pipeline_tower(T); }
  static void encode(const uint32_t* p, unsigned l, E* ev, cudaStream_t s, bool r) {
    encode_device_rows(p, l, ev, kLiveRows, s, r);
  }
  static void decode(const E* ev, unsigned l, uint32_t* p, cudaStream_t s, bool r) { decode_device(ev, l, p, s, r); }
  static void top(E* ev, unsigned l, unsigned T, bool inv, const Tw& tw, cudaStream_t s, bool r, E* ev2 = nullptr) {
    butterfly_top_device(ev, l, T, inv, tw, s, r, ev2);
  }
  static void tile(E* ev, unsigned l, unsigned T, bool inv, const Tw& tw, cudaStream_t s) {
    butterfly_tile_device(ev, l, T, inv, tw, s);
  }
  static void fused(const E* ea, E* eb, unsigned l, unsigned T, const Tw& tw, cudaStream_t s) {
    butterfly_tile_fused_device(ea, eb, l, T, tw, s);
  }
  // both operands' tile layers in the fused pass (no separate tile pass of operand a)
  static bool fuse_ab(unsigned T) { return pipeline_fuses_operands(T); }
  static void fused2(const E* ea, E* eb, unsigned l, unsigned T, const Tw& tw, cudaStream_t s, bool r,
                     uint64_t pre_tiles = 0) {
    if (r) butterfly_tile_tower_device(ea, eb, l, T, tw, s, 0, pre_tiles);
    else butterfly_tile_fused2_device(ea, eb, l, T, tw, s);
  }
  // Host-buffer products: part of operand a's tile layers ahead of the fused pass (returns the
  // number of tiles done), in the window before operand b has arrived.
  static uint64_t pre_pass(E* ea, unsigned l, unsigned T, const Tw& tw, cudaStream_t s, bool r) {
    const uint64_t k = r ? tower_pre_tiles(l, T) : 0;
    butterfly_tile_tower_pre_device(ea, l, T, tw, k, s);
    return k;
  }
};
struct Gf64Ops {
  using E = uint2;
  static constexpr int kM = 64;
  using Tw = TwiddleSrc64;
  static constexpr int kLiveRows = 32;
  static Tw twiddles(int dev, unsigned l) { return make_twiddle_src64(dev, l, partition_base64(l)); }
  static unsigned tile_log2(unsigned l) { return pipeline64_tile_log2(l); }
  static bool tower(unsigned T) { return tile64_fused2_enabled(T) && tile64_tower_enabled(T); }
  static void encode(const uint32_t* p, unsigned l, E* ev, cudaStream_t s, bool r) {
    encode64_device(p, l, ev, kLiveRows, s, r);
  }
  static void decode(const E* ev, unsigned l, uint32_t* p, cudaStream_t s, bool r) { decode64_device(ev, l, p, s, r); }
  static void top(E* ev, unsigned l, unsigned T, bool inv, const Tw& tw, cudaStream_t s, bool r, E* ev2 = nullptr) {
    butterfly64_top_device(ev, l, T, inv, tw, s, r, ev2);
  }
  static void tile(E* ev, unsigned l, unsigned T, bool inv, const Tw& tw, cudaStream_t s) {
    butterfly64_tile_device(ev, l, T, inv, tw, s);
  }
  static void fused(const E* ea, E* eb, unsigned l, unsigned T, const Tw& tw, cudaStream_t s) {
    butterfly64_tile_fused_device(ea, eb, l, T, tw, s);
  }
  static bool fuse_ab(unsigned T) { return tile64_fused2_enabled(T); }
  static void fused2(const E* ea, E* eb, unsigned l, unsigned T, const Tw& tw, cudaStream_t s, bool r,
                     uint64_t pre_tiles = 0) {
    if (r) butterfly64_tile_tower_device(ea, eb, l, T, tw, s, pre_tiles);
    else butterfly64_tile_fused2_device(ea, eb, l, T, tw, s);
  }
  static uint64_t pre_pass(E* ea, unsigned l, unsigned T, const Tw& tw, cudaStream_t s, bool r) {
    const uint64_t k = r ? tower64_pre_tiles(l, T) : 0;
    butterfly64_tile_tower_pre_device(ea, l, T, tw, k, s);
    return k;
  }
};

// fp_polymul on device buffers.  field: FPM_FIELD_GF128, FPM_FIELD_GF64, or FPM_FIELD_AUTO (the
// reference's plan_mul choice: GF(2^64) whenever it supports the size, polymul.cpp:203-205).
// Products are field-independent; the field only selects the transform.
template <class F>
void run_pipeline(const uint64_t* d_a, size_t a_bits, const uint64_t* d_b, size_t b_bits, uint64_t* d_c,
                  const fpm_plan& p, cudaStream_t s, double* stages, const HostIO* io) {
  using E = typename F::E;
  const size_t out_bits = a_bits + b_bits - 1;
  const uint64_t out_words = (out_bits + 63) / 64;
  StageClock clk(s, stages);
  auto wait_operand = [&](int k) {
    if (io && io->ready[k]) FPM_CUDA(cudaStreamWaitEvent(s, io->ready[k], 0));
  };
  auto copy_out = [&](uint64_t w0, uint64_t w1) {  // 64-bit words of d_c, final on s
    if (!io || !io->h_out || w0 >= w1) return;
    cudaEvent_t e;
    FPM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    FPM_CUDA(cudaEventRecord(e, s));
    FPM_CUDA(cudaStreamWaitEvent(io->d2h, e, 0));
    FPM_CUDA(cudaEventDestroy(e));  // released once the wait is satisfied
    FPM_CUDA(cudaMemcpyAsync(io->h_out + w0, d_c + w0, (w1 - w0) * 8, cudaMemcpyDeviceToHost, io->d2h));
  };
  if (p.n_bits <= ((size_t)1 << 17)) {  // whole product in one CTA (the same product in any field)
    wait_operand(0);
    wait_operand(1);
    clk.mark(kStPointwise);
    polymul_batch_device(d_a, a_bits, 0, d_b, b_bits, 0, d_c, 0, 1, s);
    clk.finish();
    copy_out(0, out_words);
    return;
  }
  const unsigned l = p.l, T = F::tile_log2(l);
  const bool fuse_ab = T > 0 && F::fuse_ab(T);
  const bool rep = fuse_ab && F::tower(T);  // EvalVecs in the tower representation
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const typename F::Tw tw = F::twiddles(dev, l);
  const size_t n = p.n_bits, n_p = p.n_p;
  // The n-bit work array: the product buffer itself when it spans exactly n bits (equal-length
  // power-of-two operands: out_bits = n - 1), else a scratch array trimmed into d_c at the end.
  const bool in_place = out_words * 64 == n;
  DevBuf P(in_place ? 0 : n / 8, s), EA(n_p * sizeof(E), s), EB(n_p * sizeof(E), s);
  uint64_t* const work = in_place ? d_c : P.as<uint64_t>();
  uint32_t* const work32 = reinterpret_cast<uint32_t*>(work);
  uint64_t* const work_base = work;
  const cudaStream_t run_stream = s;
  const uint64_t* xs[2] = {d_a, d_b};
  const size_t xbits[2] = {a_bits, b_bits};
  E* es[2] = {EA.as<E>(), EB.as<E>()};
  // Device-resident operands: both conversions first, then the top passes of both EvalVecs in one
  // launch per layer pair (one set of twiddle tables per CTA for both).  Host-buffer calls keep
  // operand a's transforms ahead of operand b's upload.
  const bool joint_top = !io;
  // Device-resident products: operand b converts on a second stream beside operand
  // a (into the upper half of the n-bit work array, its own scratch); the top passes join them.
  static const unsigned conc_min_log2 = [] {  // FPM_CONC_MIN_LOG2: smallest n (log2) that forks
    const char* e = std::getenv("FPM_CONC_MIN_LOG2");
    return e ? (unsigned)std::atoi(e) : 18u;
  }();
  const bool conc = joint_top && n >= ((size_t)1 << conc_min_log2) && concurrent_blocks_enabled();
  cudaStream_t sb = s;
  std::optional<Ev> fork, joined;  // (released on every exit path)
  if (conc) {
    sb = side_stream(dev);
    fork.emplace();
    joined.emplace();
    clk.mark(kStBasis);
    FPM_CUDA(cudaEventRecord(fork->e, s));
    FPM_CUDA(cudaStreamWaitEvent(sb, fork->e, 0));
  }
  uint64_t pre_tiles = 0;  // operand a's tiles whose forward tile layers ran ahead (host-buffer calls)
  for (int k = 0; k < 2; ++k) {
    wait_operand(k);
    if (!conc) clk.mark(kStBasis);
    const cudaStream_t s = conc && k == 1 ? sb : run_stream;  // (shadows the pipeline stream for operand b)
    uint64_t* const work = conc && k == 1 ? work_base + n / 128 : work_base;
    uint32_t* const work32 = reinterpret_cast<uint32_t*>(work);
    const uint64_t half_words = n / 128;  // n/2 bits in uint64 words
    size_t count = (size_t)1 << log2_ceil(xbits[k]);
    if (count < 32) count = 32;
    // a 2^32-bit conversion's last step also encodes (GF(2^128): the converted bits never reach HBM)
    EncodeSink sink{es[k], rep, F::kM};
    const bool fused = count == n / 2 && basis_cvt_can_encode(count, rep);
    if (xbits[k] == n / 2 && count == n / 2 && count >= ((size_t)1 << 17) && count <= ((size_t)1 << 32)) {
      // the operand fills the conversion exactly: convert straight from the caller's buffer
      basis_cvt_device(work32, count, xbits[k], false, s, nullptr, reinterpret_cast<const uint32_t*>(xs[k]),
                       fused ? &sink : nullptr);
    } else {
      launch_k(load_operand_kernel, dim3(grid_1d(half_words)), dim3(256), 0, s, work, half_words, xs[k], xbits[k]);
      FPM_LAUNCH_CHECK();
      basis_cvt_device(work32, count, xbits[k], false, s, nullptr, nullptr, fused ? &sink : nullptr);
    }
    if (!conc) clk.mark(kStEncode);
    if (!fused) F::encode(work32, l, es[k], s, rep);
    if (joint_top) continue;
    clk.mark(kStBfly);
    F::top(es[k], l, T, false, tw, s, rep);
    if (k == 0 && !fuse_ab) F::tile(es[k], l, T, false, tw, s);
    if (k == 0 && fuse_ab && io->alone) pre_tiles = F::pre_pass(es[0], l, T, tw, s, rep);
  }
  if (conc) {
    FPM_CUDA(cudaEventRecord(joined->e, sb));
    FPM_CUDA(cudaStreamWaitEvent(s, joined->e, 0));
    clk.mark(kStEncode);
  }
  if (joint_top) {
    clk.mark(kStBfly);
    F::top(es[0], l, T, false, tw, s, rep, es[1]);
    if (!fuse_ab) F::tile(es[0], l, T, false, tw, s);
  }
  clk.mark(kStPointwise);  // + operand b's (and a's) bottom T forward and the bottom T inverse layers (fused)
  if (fuse_ab) F::fused2(EA.as<E>(), EB.as<E>(), l, T, tw, s, rep, pre_tiles);
  else F::fused(EA.as<E>(), EB.as<E>(), l, T, tw, s);
  clk.mark(kStIBfly);
  F::top(EB.as<E>(), l, T, true, tw, s, rep);
  clk.mark(kStDecode);
  // a 2^33-bit product's decode runs inside the inverse conversion's first step (GF(2^128))
  const bool fused_dec = basis_cvt_can_decode(n);
  DecodeSource dsrc{EB.p, rep, F::kM};
  if (!fused_dec) F::decode(EB.as<E>(), l, work32, s, rep);
  clk.mark(kStIBasis);
  // Each finished range of the product is trimmed into d_c (and copied out) right away.
  const FinalFn on_final = [&](uint64_t w0, uint64_t w1) {  // 32-bit word range of P
    // 64-bit word q holds 32-bit words 2q, 2q+1: rounding both ends up keeps the reported ranges a
    // partition and only ever copies a word once both of its halves are final.
    const uint64_t q0 = std::min<uint64_t>((w0 + 1) / 2, out_words), q1 = std::min<uint64_t>((w1 + 1) / 2, out_words);
    if (q0 >= q1) return;
    if (!in_place) {  // (in place, bit n-1 is the product's, which is zero: deg < out_bits)
      launch_k(store_product_kernel, dim3(grid_1d(q1 - q0)), dim3(256), 0, s, d_c, work, out_bits, q0, q1);
      FPM_LAUNCH_CHECK();
    }
    copy_out(q0, q1);
  };
  basis_cvt_device(work32, n, n, true, s, &on_final, nullptr, nullptr, fused_dec ? &dsrc : nullptr, !io);
  clk.finish();
}

// karatsuba_mul (polymul.cpp:268-282) on device buffers: the word product of the masked operands,
// trimmed to a_bits + b_bits - 1 bits.
void karatsuba_device(const uint64_t* d_a, size_t a_bits, const uint64_t* d_b, size_t b_bits, uint64_t* d_c,
                      cudaStream_t s) {
  const uint64_t wa = (a_bits + 63) / 64, wb = (b_bits + 63) / 64;
  const size_t out_bits = a_bits + b_bits - 1;
  DevBuf X(wa * 8, s), Y(wb * 8, s), P((wa + wb) * 8, s);
  launch_k(load_operand_kernel, dim3(grid_1d(wa)), dim3(256), 0, s, X.as<uint64_t>(), wa, d_a, a_bits);
  FPM_LAUNCH_CHECK();
  launch_k(load_operand_kernel, dim3(grid_1d(wb)), dim3(256), 0, s, Y.as<uint64_t>(), wb, d_b, b_bits);
  FPM_LAUNCH_CHECK();
  clmul_words_device(X.as<uint64_t>(), wa, Y.as<uint64_t>(), wb, P.as<uint64_t>(), s);
  const uint64_t out_words = (out_bits + 63) / 64;
  launch_k(store_product_kernel, dim3(grid_1d(out_words)), dim3(256), 0, s, d_c, P.as<uint64_t>(), out_bits, 0, out_words);
  FPM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ CUDA graphs for repeated products
// A product of n <= 2^26 bits is tens of short kernels: launch-bound.  Device-buffer calls
// (fpm_polymul_dev without stage timing) replay a CUDA graph of the whole pipeline, captured on the
// second call with the same buffers and shape (the first call runs eagerly: it uploads the device
// tables and sets kernel attributes, which capture cannot).  Per-call scratch comes from graph
// memory nodes.  FPM_GRAPHS=0 disables it.
struct GraphKey {
  const void* a;
  size_t a_bits;
  const void* b;
  size_t b_bits;
  void* c;
  unsigned m;
  bool operator<(const GraphKey& o) const {
    return std::tie(a, a_bits, b, b_bits, c, m) < std::tie(o.a, o.a_bits, o.b, o.b_bits, o.c, o.m);
  }
};
bool graph_eligible(const fpm_plan& p) {
  static const bool on = [] {
    const char* e = std::getenv("FPM_GRAPHS");
    return !(e && std::string(e) == "0");
  }();
  return on && p.n_bits <= ((uint64_t)1 << 26);
}
template <class Run>
void launch_graph(const GraphKey& key, cudaStream_t s, Run&& run) {
  struct Entry {
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
    uint64_t kernels = 0;  // kernel nodes: fpm_launch_count() counts them at every replay
  };
  static std::mutex mu;
  static std::map<std::pair<int, GraphKey>, Entry> cache;
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;
  bool capture = false;
  {
    std::lock_guard<std::mutex> lock(mu);
    Entry& e = cache[{dev, key}];
    exec = e.exec;
    kernels = e.kernels;
    if (!exec) capture = ++e.seen >= 2 && cache.size() <= 64;  // first sighting: run eagerly
  }
  if (exec) {
    FPM_CUDA(cudaGraphLaunch(exec, s));
    g_launches.fetch_add(kernels, std::memory_order_relaxed);
    return;
  }
  if (!capture) {
    run(s);
    return;
  }
  // Capture on a private stream (capture executes nothing, and the caller's stream may be the
  // legacy default stream, which cannot capture); the graph is then launched on the caller's stream.
  static cudaStream_t cap_streams[64] = {};
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!cap_streams[dev]) FPM_CUDA(cudaStreamCreateWithFlags(&cap_streams[dev], cudaStreamNonBlocking));
  }
  const cudaStream_t cs = cap_streams[dev];
  cudaGraph_t g = nullptr;
  const uint64_t n0 = g_launches.load();
  FPM_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  try {
    run(cs);
  } catch (...) {
    cudaStreamEndCapture(cs, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  FPM_CUDA(cudaStreamEndCapture(cs, &g));
  kernels = g_launches.load() - n0;  // captured, not executed (single-threaded capture assumed for the count)
  g_launches.fetch_sub(kernels, std::memory_order_relaxed);
  cudaGraphExec_t made = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&made, g, 0);
  cudaGraphDestroy(g);
  FPM_CUDA(ie);
  {
    std::lock_guard<std::mutex> lock(mu);
    Entry& e = cache[{dev, key}];
    if (e.exec) {  // another thread won the race
      cudaGraphExecDestroy(made);
      made = e.exec;
    } else {
      e.exec = made;
      e.kernels = kernels;
    }
  }
  FPM_CUDA(cudaGraphLaunch(made, s));
  g_launches.fetch_add(kernels, std::memory_order_relaxed);
}

void polymul_device(const uint64_t* d_a, size_t a_bits, const uint64_t* d_b, size_t b_bits, uint64_t* d_c,
                    int field, cudaStream_t s, double* stages, const HostIO* io = nullptr) {
  if (!a_bits || !b_bits) return;
  if (field == FPM_FIELD_AUTO && std::max(a_bits, b_bits) < kFftThresholdBits) {
    // the reference's auto-mode bypass (polymul.cpp:226-231): short inputs take karatsuba_mul
    if (io && io->ready[0]) FPM_CUDA(cudaStreamWaitEvent(s, io->ready[0], 0));
    if (io && io->ready[1]) FPM_CUDA(cudaStreamWaitEvent(s, io->ready[1], 0));
    StageClock clk(s, stages);
    clk.mark(kStPointwise);
    karatsuba_device(d_a, a_bits, d_b, b_bits, d_c, s);
    clk.finish();
    if (io && io->h_out) {
      const uint64_t out_words = (a_bits + b_bits - 1 + 63) / 64;
      cudaEvent_t done;
      FPM_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      FPM_CUDA(cudaEventRecord(done, s));
      FPM_CUDA(cudaStreamWaitEvent(io->d2h, done, 0));
      FPM_CUDA(cudaEventDestroy(done));  // released once the wait is satisfied
      FPM_CUDA(cudaMemcpyAsync(io->h_out, d_c, out_words * 8, cudaMemcpyDeviceToHost, io->d2h));
    }
    return;
  }
  const fpm_plan p = plan_mul(a_bits, b_bits, field);  // validates the field and the size bound
  auto run = [&](cudaStream_t st) {
    if (p.field_degree == 64) run_pipeline<Gf64Ops>(d_a, a_bits, d_b, b_bits, d_c, p, st, stages, io);
    else run_pipeline<Gf128Ops>(d_a, a_bits, d_b, b_bits, d_c, p, st, stages, io);
  };
  if (!stages && !io && graph_eligible(p)) {
    launch_graph(GraphKey{d_a, a_bits, d_b, b_bits, d_c, p.field_degree}, s, run);
    return;
  }
  run(s);
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    require_device();
    FPM_CUDA(cudaGetDevice(&prev));
    if (dev != prev) FPM_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

cudaStream_t host_stream(int dev) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (!streams[dev]) FPM_CUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
  return streams[dev];
}

cudaStream_t copy_stream(int dev, int which) {
  static std::mutex mu;
  static cudaStream_t streams[64][2] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (!streams[dev][which]) FPM_CUDA(cudaStreamCreateWithFlags(&streams[dev][which], cudaStreamNonBlocking));
  return streams[dev][which];
}

// Stream sets for concurrent host-buffer callers of fpm_polymul: each call leases one set (pipeline
// stream + upload + download stream), so that one caller's PCIe copies overlap another caller's
// kernels instead of queueing behind them.  Set 0 is host_stream / copy_stream; a fifth concurrent
// caller waits for a set.
struct StreamLease {
  static constexpr int kSets = 4;
  struct Pool {
    std::mutex mu;
    std::condition_variable cv;
    bool busy[kSets] = {};
    cudaStream_t st[kSets][3] = {};
    std::chrono::steady_clock::time_point last_overlap{};  // last time two leases were held at once
  };
  static Pool& pool(int dev) {
    static Pool pools[64];
    return pools[dev & 63];
  }
  Pool& p;
  int k = -1;
  cudaStream_t s = nullptr, h2d = nullptr, d2h = nullptr;
  explicit StreamLease(int dev) : p(pool(dev)) {
    std::unique_lock<std::mutex> lock(p.mu);
    p.cv.wait(lock, [&] {
      for (int i = 0; i < kSets; ++i)
        if (!p.busy[i]) return true;
      return false;
    });
    for (int i = 0; i < kSets && k < 0; ++i)
      if (!p.busy[i]) k = i;
    if (k == 0) {
      p.st[0][0] = host_stream(dev), p.st[0][1] = copy_stream(dev, 0), p.st[0][2] = copy_stream(dev, 1);
    } else {
      for (int j = 0; j < 3; ++j)
        if (!p.st[k][j]) FPM_CUDA(cudaStreamCreateWithFlags(&p.st[k][j], cudaStreamNonBlocking));
    }
    p.busy[k] = true;
    s = p.st[k][0], h2d = p.st[k][1], d2h = p.st[k][2];
    if (held() > 1) p.last_overlap = std::chrono::steady_clock::now();
  }
  ~StreamLease() {
    {
      std::lock_guard<std::mutex> lock(p.mu);
      p.busy[k] = false;
    }
    p.cv.notify_one();
  }
  int held() const {  // (p.mu held) leases on this device, this one included
    int n = 0;
    for (int i = 0; i < kSets; ++i) n += p.busy[i] ? 1 : 0;
    return n;
  }
  // No other host-buffer call on this device now or within the last second (concurrent callers
  // start their calls at different times: one of them may find the device momentarily free).
  bool alone() {
    std::lock_guard<std::mutex> lock(p.mu);
    return held() == 1 && std::chrono::steady_clock::now() - p.last_overlap > std::chrono::seconds(1);
  }
  StreamLease(const StreamLease&) = delete;
  StreamLease& operator=(const StreamLease&) = delete;
};


}  // namespace

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void set_last_error(const char* msg) { g_err = msg; }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPM_PDL");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

namespace {
cudaMemPool_t library_pool(int dev) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (dev < 0 || dev >= 64) throw Error(kInvalid, "device ordinal out of range");
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    FPM_CUDA(cudaMemPoolCreate(&pools[dev], &props));
    uint64_t thr = UINT64_MAX;  // keep freed memory cached across calls (per-call GiB scratch)
    FPM_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
    // Concurrent callers allocate on their own streams.  By default the pool may satisfy caller B's
    // allocation with memory whose free is still PENDING on caller A's stream, making B's stream
    // wait for A's pipeline to reach that free: the two products then run one after the other
    // (measured: two callers 49-50 ms per 2^33-bit product in most runs but 75-150 ms in one of
    // three).  Without internal dependencies an allocation only reuses memory that is already free
    // (or whose free the allocating stream already follows by an event); otherwise the pool grows.
    int off = 0;
    FPM_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolReuseAllowInternalDependencies, &off));
  }
  return pools[dev];
}
}  // namespace

void* pool_alloc(size_t bytes, cudaStream_t s) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  void* p = nullptr;
  FPM_CUDA(cudaMallocFromPoolAsync(&p, bytes, library_pool(dev), s));
  return p;
}

void pool_free(void* p, cudaStream_t s) { cudaFreeAsync(p, s); }

void trim_pool(int dev) { FPM_CUDA(cudaMemPoolTrimTo(library_pool(dev), 0)); }

const DeviceTables& device_tables(int dev) {
  static std::mutex mu;
  static DeviceTables tabs[64];
  static bool have[64];
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) throw Error(kInvalid, "device ordinal out of range");
  if (have[dev]) return tabs[dev];
  const FieldTables& ft = field_tables();
  std::vector<uint4> cantor(128), rows(128), inv(128), c2p(4 * 512);
  for (int i = 0; i < 128; ++i) { cantor[i] = to4(ft.cantor[i]); rows[i] = to4(ft.enc_rows[i]); inv[i] = to4(ft.inv_rows[i]); }
  // rotated 8-bit tables (gf128.cuh m8 layout): entry (c, v) at (c >> 3) * 2048 + v * 8 + (c & 7)
  // tower representation (fpm_tables.h): encode writes R(x*E); decode reads R, i.e. its row k is
  // the decode of e_k = poly(R basis vector k)
  const TowerTables& tt = tower_tables();
  std::vector<uint4> to_r(128), to_poly(128);
  U128 enc_rows_r[128], inv_rows_r[128];
  for (int k = 0; k < 128; ++k) {
    to_r[k] = to4(tt.to_r[k]);
    to_poly[k] = to4(tt.to_poly[k]);
    enc_rows_r[k] = host_to_r(ft.enc_rows[k]);
    U128 d;
    for (int m = 0; m < 128; ++m)
      if ((m < 64 ? tt.to_poly[k].lo >> m : tt.to_poly[k].hi >> (m - 64)) & 1) {
        d.lo ^= ft.inv_rows[m].lo;
        d.hi ^= ft.inv_rows[m].hi;
      }
    inv_rows_r[k] = d;
  }
  std::vector<uint4> enc8(kM8Uint4), dec8(kM8Uint4), enc8r(kM8Uint4), dec8r(kM8Uint4);
  auto m8_entries = [](std::vector<uint4>& tab, const U128* rows) {
    for (int c = 0; c < 16; ++c)
      for (int v = 0; v < 256; ++v) {
        U128 e;
        for (int j = 0; j < 8; ++j)
          if (v >> j & 1) { e.lo ^= rows[8 * c + j].lo; e.hi ^= rows[8 * c + j].hi; }
        tab[(c >> 3) * 2048 + v * 8 + (c & 7)] = to4(e);
      }
  };
  m8_entries(enc8, ft.enc_rows);
  m8_entries(dec8, ft.inv_rows);
  m8_entries(enc8r, enc_rows_r);
  m8_entries(dec8r, inv_rows_r);
  std::vector<uint2> dec_half[2] = {std::vector<uint2>(4096), std::vector<uint2>(4096)};
  for (int c = 0; c < 16; ++c)
    for (int v = 0; v < 256; ++v) {
      U128 e;
      for (int j = 0; j < 8; ++j)
        if (v >> j & 1) { e.lo ^= inv_rows_r[8 * c + j].lo; e.hi ^= inv_rows_r[8 * c + j].hi; }
      dec_half[0][v * 16 + c] = make_uint2((uint32_t)e.lo, (uint32_t)(e.lo >> 32));
      dec_half[1][v * 16 + c] = make_uint2((uint32_t)e.hi, (uint32_t)(e.hi >> 32));
    }
  for (int part = 0; part < 4; ++part)
    for (int e = 0; e < 512; ++e) {
      U128 acc;
      for (int k = 0; k < 9; ++k)
        if (e >> k & 1) {
          const int idx = 9 * part + k + 1;  // C2P(2 * (e << 9 part)): Cantor bit 9p+k+1
          acc.lo ^= ft.cantor[idx].lo;
          acc.hi ^= ft.cantor[idx].hi;
        }
      c2p[part * 512 + e] = to4(acc);
    }
  // GF(2^64): G8 tables (gf64.cuh: entry (c, v) copy h at v*16 + 8h + c), C2P tables, rows
  const FieldTables& f64 = field_tables64();
  auto u2 = [](uint64_t v) { return make_uint2((uint32_t)v, (uint32_t)(v >> 32)); };
  std::vector<uint2> enc64(4096), dec64(4096), c2p64(4 * 512), rows64(64), inv64(64);
  for (int c = 0; c < 8; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t e = 0, d = 0;
      for (int j = 0; j < 8; ++j)
        if (v >> j & 1) { e ^= f64.enc_rows[8 * c + j].lo; d ^= f64.inv_rows[8 * c + j].lo; }
      for (int h = 0; h < 2; ++h) {
        enc64[v * 16 + 8 * h + c] = u2(e);
        dec64[v * 16 + 8 * h + c] = u2(d);
      }
    }
  for (int part = 0; part < 4; ++part)
    for (int e = 0; e < 512; ++e) {
      uint64_t acc = 0;
      for (int k = 0; k < 9; ++k)
        if (e >> k & 1) {
          const int idx = 9 * part + k + 1;
          if (idx < 64) acc ^= f64.cantor[idx].lo;
        }
      c2p64[part * 512 + e] = u2(acc);
    }
  for (int j = 0; j < 64; ++j) { rows64[j] = u2(f64.enc_rows[j].lo); inv64[j] = u2(f64.inv_rows[j].lo); }
  // GF(2^64) tower representation: encode writes R, decode reads R (cf. the GF(2^128) tables)
  const TowerTables& t64 = tower_tables64();
  std::vector<uint2> to_r64(64), to_poly64(64), enc64r(4096), dec64r(4096);
  uint64_t enc_r[64], inv_r[64];
  for (int k = 0; k < 64; ++k) {
    to_r64[k] = u2(t64.to_r[k].lo);
    to_poly64[k] = u2(t64.to_poly[k].lo);
    uint64_t e = 0, d = 0;
    for (int m = 0; m < 64; ++m) {
      if (f64.enc_rows[k].lo >> m & 1) e ^= t64.to_r[m].lo;
      if (t64.to_poly[k].lo >> m & 1) d ^= f64.inv_rows[m].lo;
    }
    enc_r[k] = e;
    inv_r[k] = d;
  }
  for (int c = 0; c < 8; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t e = 0, d = 0;
      for (int j = 0; j < 8; ++j)
        if (v >> j & 1) { e ^= enc_r[8 * c + j]; d ^= inv_r[8 * c + j]; }
      for (int h = 0; h < 2; ++h) {
        enc64r[v * 16 + 8 * h + c] = u2(e);
        dec64r[v * 16 + 8 * h + c] = u2(d);
      }
    }
  int prev;
  FPM_CUDA(cudaGetDevice(&prev));
  FPM_CUDA(cudaSetDevice(dev));
  DeviceTables t;
  auto up = [](uint4** dst, const std::vector<uint4>& v) {
    FPM_CUDA(cudaMalloc(dst, v.size() * sizeof(uint4)));
    FPM_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  };
  up(&t.cantor, cantor); up(&t.enc_rows, rows); up(&t.inv_rows, inv);
  up(&t.c2p, c2p);
  up(&t.enc_m8, enc8); up(&t.dec_m8, dec8);
  up(&t.to_r, to_r); up(&t.to_poly, to_poly); up(&t.enc_m8r, enc8r); up(&t.dec_m8r, dec8r);
  auto up2 = [](uint2** dst, const std::vector<uint2>& v) {
    FPM_CUDA(cudaMalloc(dst, v.size() * sizeof(uint2)));
    FPM_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(uint2), cudaMemcpyHostToDevice));
  };
  up2(&t.dec_half_r[0], dec_half[0]);
  up2(&t.dec_half_r[1], dec_half[1]);
  up2(&t.enc_g8, enc64); up2(&t.dec_g8, dec64); up2(&t.c2p64, c2p64); up2(&t.rows64, rows64); up2(&t.inv64, inv64);
  up2(&t.to_r64, to_r64); up2(&t.to_poly64, to_poly64); up2(&t.enc_g8r, enc64r); up2(&t.dec_g8r, dec64r);
  FPM_CUDA(cudaSetDevice(prev));
  tabs[dev] = t;
  have[dev] = true;
  return tabs[dev];
}

}  // namespace fpm

namespace fpm {
namespace {
template <class Fn>
fpm_status host_call(int device, Fn&& fn) {
  return guard([&] {
    DeviceGuard g(device);
    cudaStream_t s = host_stream(device);
    fn(s);
    FPM_CUDA(cudaStreamSynchronize(s));
  });
}
}  // namespace
}  // namespace fpm

using namespace fpm;

namespace fpm {
namespace {
RankPtrs rank_ptrs(const uint64_t* const* p, int Q) {
  if (!p || Q < 1 || Q > 4 || (Q & (Q - 1))) throw Error(kInvalid, "sharded conversion: 1, 2 or 4 replicas");
  RankPtrs r{};
  for (int q = 0; q < Q; ++q) {
    if (!p[q]) throw Error(kInvalid, "sharded conversion: null replica pointer");
    r.p[q] = reinterpret_cast<uint32_t*>(const_cast<uint64_t*>(p[q]));
  }
  return r;
}
void check_q(int q, int Q) {
  if (Q < 2 || Q > 4 || (Q & (Q - 1)) || q < 0 || q >= Q) throw Error(kInvalid, "sharded conversion: 2 or 4 ranks, 0 <= q < Q");
}
}  // namespace
}  // namespace fpm

namespace fpm {
namespace {
// Host-buffer calls of small products (<= 2^22 bits) stage through persistent device buffers, so that the device-resident pipeline between the copies replays a captured CUDA graph
// (its key includes the buffer addresses): config 1 / 3 with host buffers are launch-bound otherwise.
// One staging set per device, taken with try_lock (a concurrent call uses the general path).
struct SmallStage {
  std::mutex mu;
  uint64_t* a = nullptr;
  uint64_t* b = nullptr;
  uint64_t* c = nullptr;
  size_t wa = 0, wb = 0, wc = 0;
};
SmallStage& small_stage(int dev) {
  static SmallStage st[64];
  return st[dev & 63];
}
void grow(uint64_t*& p, size_t& have, size_t want) {
  if (have >= want) return;
  if (p) FPM_CUDA(cudaFree(p));
  p = nullptr;
  have = 0;
  FPM_CUDA(cudaMalloc(&p, want * 8));
  have = want;
}
}  // namespace
}  // namespace fpm

extern "C" {

const char* fpm_last_error(void) { return g_err.c_str(); }
const char* fpm_version(void) { return "fpmul_b200 0.1 (sm_100a)"; }

unsigned fpm_fft_tile_log2(unsigned l) { return fpm::pipeline_tile_log2(l); }
int fpm_pipeline_fuses_operands(unsigned l) {
  const unsigned T = fpm::pipeline_tile_log2(l);
  return l >= 18 && T > 0 && fpm::pipeline_fuses_operands(T) ? 1 : 0;
}
int fpm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
uint64_t fpm_launch_count(int reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

fpm_status fpm_test_flip_encode_table(int device) {
  return guard([&] {
    DeviceGuard g(device);
    flip_encode_tables(device, host_stream(device));
  });
}

fpm_status fpm_trim_pool(int device) {
  return guard([&] {
    require_device();
    trim_pool(device);
  });
}

fpm_status fpm_reserve_pool(int device, size_t bytes) {
  return guard([&] {
    DeviceGuard g(device);
    if (!bytes) return;
    cudaStream_t s = host_stream(device);
    // blocks of at most 1 GiB (the size class of the large per-product buffers), all live at once,
    // then freed: they stay cached in the pool (release threshold: never)
    std::vector<std::unique_ptr<DevBuf>> blocks;
    for (size_t left = bytes; left;) {
      const size_t b = std::min<size_t>(left, (size_t)1 << 30);
      blocks.emplace_back(new DevBuf(b, s));
      left -= b;
    }
    blocks.clear();
    FPM_CUDA(cudaStreamSynchronize(s));
  });
}

fpm_status fpm_random_bitpoly(size_t n_bits, uint64_t seed, uint64_t* out) {
  return guard([&] {
    if (n_bits && !out) throw Error(kInvalid, "random_bitpoly: null output");
    std::mt19937_64 rng(seed);  // bitpoly.cpp:19-24: one draw per word, excess bits cleared
    const size_t words = (n_bits + 63) / 64;
    for (size_t i = 0; i < words; ++i) out[i] = rng();
    if (n_bits % 64) out[words - 1] &= (((uint64_t)1) << (n_bits % 64)) - 1;
  });
}

fpm_status fpm_plan_mul(size_t a_bits, size_t b_bits, int field, fpm_plan* out) {
  return guard([&] {
    if (!out) throw Error(kInvalid, "plan_mul: null output");
    *out = plan_mul(a_bits, b_bits, field);
  });
}

fpm_status fpm_tables128(uint64_t* cantor, uint64_t* rows, uint64_t* inv_rows) {
  return guard([&] {
    const FieldTables& t = field_tables();
    for (int i = 0; i < 128; ++i) {
      if (cantor) { cantor[2 * i] = t.cantor[i].lo; cantor[2 * i + 1] = t.cantor[i].hi; }
      if (rows) { rows[2 * i] = t.enc_rows[i].lo; rows[2 * i + 1] = t.enc_rows[i].hi; }
      if (inv_rows) { inv_rows[2 * i] = t.inv_rows[i].lo; inv_rows[2 * i + 1] = t.inv_rows[i].hi; }
    }
  });
}

fpm_status fpm_tower_tables(int field_degree, uint64_t* t, uint64_t* to_poly, uint64_t* to_r, uint8_t* tau) {
  return guard([&] {
    if (field_degree != 128 && field_degree != 64) throw Error(kInvalid, "tower tables: field degree must be 128 or 64");
    const TowerTables& tt = field_degree == 128 ? tower_tables() : tower_tables64();
    if (t) { t[0] = tt.t.lo; t[1] = tt.t.hi; }
    for (int k = 0; k < field_degree; ++k) {
      if (to_poly) { to_poly[2 * k] = tt.to_poly[k].lo; to_poly[2 * k + 1] = tt.to_poly[k].hi; }
      if (to_r) { to_r[2 * k] = tt.to_r[k].lo; to_r[2 * k + 1] = tt.to_r[k].hi; }
    }
    if (tau)
      for (int b = 0; b < 8; ++b) tau[b] = tt.tau[b];
  });
}

fpm_status fpm_polymul_dev(const uint64_t* d_a, size_t a_bits, const uint64_t* d_b, size_t b_bits, uint64_t* d_c,
                           int field, void* stream, double* stage_seconds) {
  return guard([&] {
    require_device();
    polymul_device(d_a, a_bits, d_b, b_bits, d_c, field, (cudaStream_t)stream, stage_seconds);
  });
}


fpm_status fpm_polymul(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c, int field,
                       int device, double* stage_seconds) {
  return guard([&] {
    if (!a_bits || !b_bits) return;
    const fpm_plan plan = plan_mul(a_bits, b_bits, field);
    DeviceGuard g(device);
    cudaStream_t s = host_stream(device);
    const size_t wa = (a_bits + 63) / 64, wb = (b_bits + 63) / 64, wc = (a_bits + b_bits - 1 + 63) / 64;
    static const bool staged = [] {
      const char* e = std::getenv("FPM_SMALL_STAGE");
      return !(e && std::string(e) == "0");
    }();
    // (up to 2^22-bit products: larger ones gain more from overlapping the copies with the pipeline --
    // config 3 with host buffers: 0.65 ms overlapped vs 0.74 staged; config 1: 0.176 -> 0.160 ms)
    if (staged && !stage_seconds && graph_eligible(plan) && plan.n_bits <= ((size_t)1 << 22)) {
      SmallStage& st = small_stage(device);
      std::unique_lock<std::mutex> lk(st.mu, std::try_to_lock);
      if (lk.owns_lock()) {
        FPM_CUDA(cudaStreamSynchronize(s));  // (buffers may be reallocated below)
        grow(st.a, st.wa, wa);
        grow(st.b, st.wb, wb);
        grow(st.c, st.wc, wc);
        FPM_CUDA(cudaMemcpyAsync(st.a, a, wa * 8, cudaMemcpyHostToDevice, s));
        FPM_CUDA(cudaMemcpyAsync(st.b, b, wb * 8, cudaMemcpyHostToDevice, s));
        polymul_device(st.a, a_bits, st.b, b_bits, st.c, field, s, nullptr);
        FPM_CUDA(cudaMemcpyAsync(c, st.c, wc * 8, cudaMemcpyDeviceToHost, s));
        FPM_CUDA(cudaStreamSynchronize(s));
        return;
      }
    }
    // concurrent callers: own pipeline / copy streams per call (declared before the buffers: they
    // are freed on the leased stream and the stream is synchronized before the lease ends)
    StreamLease lease(device);
    s = lease.s;
    cudaStream_t h2d = lease.h2d, d2h = lease.d2h;
    DevBuf A(wa * 8, s), B(wb * 8, s), C(wc * 8, s);
    // On an exception (e.g. an allocation failure inside the pipeline) the buffers above are freed
    // while the copy streams may still read or write them: drain both copy streams first (this
    // guard is destroyed before the DevBufs).
    struct DrainOnUnwind {
      cudaStream_t a, b;
      int pending = std::uncaught_exceptions();
      ~DrainOnUnwind() {
        if (std::uncaught_exceptions() > pending) {
          cudaStreamSynchronize(a);
          cudaStreamSynchronize(b);
        }
      }
    } drain{h2d, d2h};
    Ev allocated, ready_a, ready_b, copied;
    FPM_CUDA(cudaEventRecord(allocated.e, s));  // stream-ordered allocations visible to the copy streams
    FPM_CUDA(cudaStreamWaitEvent(h2d, allocated.e, 0));
    FPM_CUDA(cudaStreamWaitEvent(d2h, allocated.e, 0));
    FPM_CUDA(cudaMemcpyAsync(A.p, a, wa * 8, cudaMemcpyHostToDevice, h2d));
    FPM_CUDA(cudaEventRecord(ready_a.e, h2d));
    FPM_CUDA(cudaMemcpyAsync(B.p, b, wb * 8, cudaMemcpyHostToDevice, h2d));
    FPM_CUDA(cudaEventRecord(ready_b.e, h2d));
    HostIO io;
    io.ready[0] = ready_a.e;
    io.ready[1] = ready_b.e;
    io.h_out = c;
    io.d2h = d2h;
    io.alone = lease.alone();
    polymul_device(A.as<uint64_t>(), a_bits, B.as<uint64_t>(), b_bits, C.as<uint64_t>(), field, s, stage_seconds, &io);
    FPM_CUDA(cudaEventRecord(copied.e, d2h));
    FPM_CUDA(cudaStreamWaitEvent(s, copied.e, 0));  // frees below are ordered after the copies
    FPM_CUDA(cudaStreamSynchronize(s));
  });
}

fpm_status fpm_polymul_batch_dev(const uint64_t* d_a, size_t a_bits, size_t a_stride_words, const uint64_t* d_b,
                                 size_t b_bits, size_t b_stride_words, uint64_t* d_c, size_t c_stride_words,
                                 size_t count, void* stream) {
  return guard([&] {
    require_device();
    if (!a_bits || !b_bits || !count) return;
    polymul_batch_device(d_a, a_bits, a_stride_words, d_b, b_bits, b_stride_words, d_c, c_stride_words, count,
                         (cudaStream_t)stream);
  });
}

fpm_status fpm_polymul_batch(const uint64_t* a, size_t a_bits, size_t a_stride_words, const uint64_t* b, size_t b_bits,
                             size_t b_stride_words, uint64_t* c, size_t c_stride_words, size_t count, int device) {
  return guard([&] {
    if (!a_bits || !b_bits || !count) return;
    if (!a || !b || !c) throw Error(kInvalid, "polymul_batch: null buffer");
    const size_t wa = (a_bits + 63) / 64, wb = (b_bits + 63) / 64, wc = (a_bits + b_bits - 1 + 63) / 64;
    if (a_stride_words < wa || b_stride_words < wb || c_stride_words < wc)
      throw Error(kInvalid, "polymul_batch: a stride is shorter than its operand / product");
    DeviceGuard g(device);
    cudaStream_t s = host_stream(device), h2d = copy_stream(device, 0), d2h = copy_stream(device, 1);
    // chunks of >= 64 products (the tower batch path), at most 8 of them; three device slots
    const size_t chunk = std::max<size_t>(64, (count + 7) / 8);
    const size_t nchunks = (count + chunk - 1) / chunk;
    constexpr int kSlots = 3;
    DevBuf A(kSlots * chunk * wa * 8, s), B(kSlots * chunk * wb * 8, s), Cb(kSlots * chunk * wc * 8, s);
    struct DrainOnUnwind {
      cudaStream_t a, b, c;
      int pending = std::uncaught_exceptions();
      ~DrainOnUnwind() {
        if (std::uncaught_exceptions() > pending) {
          cudaStreamSynchronize(a);
          cudaStreamSynchronize(b);
          cudaStreamSynchronize(c);
        }
      }
    } drain{h2d, d2h, s};
    Ev allocated;
    FPM_CUDA(cudaEventRecord(allocated.e, s));
    FPM_CUDA(cudaStreamWaitEvent(h2d, allocated.e, 0));
    FPM_CUDA(cudaStreamWaitEvent(d2h, allocated.e, 0));
    std::vector<Ev> in(nchunks), done(nchunks), out(nchunks);
    for (size_t k = 0; k < nchunks; ++k) {
      const size_t p0 = k * chunk, cnt = std::min(chunk, count - p0), slot = k % kSlots;
      uint64_t* da = A.as<uint64_t>() + slot * chunk * wa;
      uint64_t* db = B.as<uint64_t>() + slot * chunk * wb;
      uint64_t* dc = Cb.as<uint64_t>() + slot * chunk * wc;
      if (k >= kSlots) FPM_CUDA(cudaStreamWaitEvent(h2d, done[k - kSlots].e, 0));  // slot's inputs consumed
      FPM_CUDA(cudaMemcpy2DAsync(da, wa * 8, a + p0 * a_stride_words, a_stride_words * 8, wa * 8, cnt,
                                 cudaMemcpyHostToDevice, h2d));
      FPM_CUDA(cudaMemcpy2DAsync(db, wb * 8, b + p0 * b_stride_words, b_stride_words * 8, wb * 8, cnt,
                                 cudaMemcpyHostToDevice, h2d));
      FPM_CUDA(cudaEventRecord(in[k].e, h2d));
      FPM_CUDA(cudaStreamWaitEvent(s, in[k].e, 0));
      if (k >= kSlots) FPM_CUDA(cudaStreamWaitEvent(s, out[k - kSlots].e, 0));  // slot's products copied out
      polymul_batch_device(da, a_bits, wa, db, b_bits, wb, dc, wc, cnt, s);
      FPM_CUDA(cudaEventRecord(done[k].e, s));
      FPM_CUDA(cudaStreamWaitEvent(d2h, done[k].e, 0));
      FPM_CUDA(cudaMemcpy2DAsync(c + p0 * c_stride_words, c_stride_words * 8, dc, wc * 8, wc * 8, cnt,
                                 cudaMemcpyDeviceToHost, d2h));
      FPM_CUDA(cudaEventRecord(out[k].e, d2h));
    }
    FPM_CUDA(cudaStreamWaitEvent(s, out[nchunks - 1].e, 0));  // frees below after the last copy
    FPM_CUDA(cudaStreamSynchronize(s));
  });
}

fpm_status fpm_clmul_words_dev(const uint64_t* d_a, size_t wa, const uint64_t* d_b, size_t wb, uint64_t* d_out,
                               void* stream) {
  return guard([&] {
    require_device();
    clmul_words_device(d_a, wa, d_b, wb, d_out, (cudaStream_t)stream);
  });
}

fpm_status fpm_karatsuba_mul(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c,
                             int device) {
  return guard([&] {
    if (!a_bits || !b_bits) return;
    DeviceGuard g(device);
    cudaStream_t s = host_stream(device);
    const size_t wa = (a_bits + 63) / 64, wb = (b_bits + 63) / 64, wc = (a_bits + b_bits - 1 + 63) / 64;
    DevBuf A(wa * 8, s), B(wb * 8, s), C(wc * 8, s);
    FPM_CUDA(cudaMemcpyAsync(A.p, a, wa * 8, cudaMemcpyHostToDevice, s));
    FPM_CUDA(cudaMemcpyAsync(B.p, b, wb * 8, cudaMemcpyHostToDevice, s));
    karatsuba_device(A.as<uint64_t>(), a_bits, B.as<uint64_t>(), b_bits, C.as<uint64_t>(), s);
    FPM_CUDA(cudaMemcpyAsync(c, C.p, wc * 8, cudaMemcpyDeviceToHost, s));
    FPM_CUDA(cudaStreamSynchronize(s));
  });
}

fpm_status fpm_basis_cvt_dev(uint64_t* d_w, size_t n_bits, size_t content_bits, void* stream) {
  return guard([&] {
    require_device();
    if (n_bits == 0 || (n_bits & (n_bits - 1))) throw Error(kInvalid, "basis_cvt: length must be a power of two");
    if (n_bits <= 2) return;  // identity (basis_convert.cpp:280)
    basis_cvt_device(reinterpret_cast<uint32_t*>(d_w), n_bits, content_bits ? std::min(content_bits, n_bits) : 1,
                     false, (cudaStream_t)stream);
  });
}

fpm_status fpm_i_basis_cvt_dev(uint64_t* d_w, size_t n_bits, void* stream) {
  return guard([&] {
    require_device();
    if (n_bits == 0 || (n_bits & (n_bits - 1))) throw Error(kInvalid, "basis_cvt: length must be a power of two");
    if (n_bits <= 2) return;
    basis_cvt_device(reinterpret_cast<uint32_t*>(d_w), n_bits, n_bits, true, (cudaStream_t)stream);
  });
}

fpm_status fpm_encode_dev(const uint64_t* d_poly, unsigned l, uint64_t* d_ev, void* stream) {
  return guard([&] {
    require_device();
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    encode_device(reinterpret_cast<const uint32_t*>(d_poly), l, reinterpret_cast<uint4*>(d_ev), (cudaStream_t)stream);
  });
}

fpm_status fpm_decode_dev(const uint64_t* d_ev, unsigned l, uint64_t* d_poly, void* stream) {
  return guard([&] {
    require_device();
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    decode_device(reinterpret_cast<const uint4*>(d_ev), l, reinterpret_cast<uint32_t*>(d_poly), (cudaStream_t)stream);
  });
}

fpm_status fpm_butterfly_dev(uint64_t* d_ev, unsigned l, int inverse, void* stream) {
  return guard([&] {
    require_device();
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    if (l == 0) return;
    butterfly_device(reinterpret_cast<uint4*>(d_ev), l, partition_base(l), inverse != 0, (cudaStream_t)stream);
  });
}

fpm_status fpm_lch_butterfly_dev(uint64_t* d_ev, unsigned l, const uint64_t* base, int inverse, void* stream) {
  return guard([&] {
    require_device();
    if (l > 64) throw Error(kInvalid, "lch_butterfly: at most 64 layers");
    if (l == 0) return;
    if (!base) throw Error(kInvalid, "lch_butterfly: null base");
    U128 b;
    b.lo = base[0];
    b.hi = base[1];
    butterfly_device(reinterpret_cast<uint4*>(d_ev), l, b, inverse != 0, (cudaStream_t)stream);
  });
}

fpm_status fpm_encode_cols_dev(const uint64_t* d_poly, unsigned l, size_t col0, size_t ncols, int rows_live,
                               uint64_t* d_ev, void* stream) {
  return guard([&] {
    require_device();
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    encode_cols_device(reinterpret_cast<const uint32_t*>(d_poly), l, col0, ncols, reinterpret_cast<uint4*>(d_ev),
                       rows_live == 64 ? 64 : 128, (cudaStream_t)stream);
  });
}

fpm_status fpm_decode_cols_dev(const uint64_t* d_ev, size_t ncols, uint64_t* d_slice, void* stream) {
  return guard([&] {
    require_device();
    decode_cols_device(reinterpret_cast<const uint4*>(d_ev), ncols, reinterpret_cast<uint32_t*>(d_slice),
                       (cudaStream_t)stream);
  });
}

int fpm_shard_tower(unsigned l) {
  const unsigned T = pipeline_tile_log2(l);
  return l >= 18 && l < 64 && pipeline_tower(T) ? 1 : 0;
}

fpm_status fpm_encode_cols_r_dev(const uint64_t* d_poly, unsigned l, size_t col0, size_t ncols, int rows_live,
                                 uint64_t* d_ev, void* stream) {
  return guard([&] {
    require_device();
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    encode_cols_device(reinterpret_cast<const uint32_t*>(d_poly), l, col0, ncols, reinterpret_cast<uint4*>(d_ev),
                       rows_live == 64 ? 64 : 128, (cudaStream_t)stream, true);
  });
}

fpm_status fpm_decode_cols_r_dev(const uint64_t* d_ev, size_t ncols, uint64_t* d_slice, void* stream) {
  return guard([&] {
    require_device();
    decode_cols_device(reinterpret_cast<const uint4*>(d_ev), ncols, reinterpret_cast<uint32_t*>(d_slice),
                       (cudaStream_t)stream, true);
  });
}

fpm_status fpm_bfly_pair_r_dev(uint64_t* d_mine, const uint64_t* d_theirs, size_t n, const uint64_t* w, int side,
                               int inverse, void* stream) {
  return guard([&] {
    require_device();
    if (!w || (side != 0 && side != 1)) throw Error(kInvalid, "bfly_pair: bad twiddle or side");
    U128 t;
    t.lo = w[0];
    t.hi = w[1];
    bfly_pair_device(reinterpret_cast<uint4*>(d_mine), reinterpret_cast<const uint4*>(d_theirs), n, t, side,
                     inverse != 0, (cudaStream_t)stream, true);
  });
}

fpm_status fpm_bfly_pair_peer_dev(const uint64_t* d_mine, const uint64_t* d_theirs, uint64_t* d_out, size_t n,
                                  const uint64_t* w, int side, int inverse, int tower, void* stream) {
  return guard([&] {
    require_device();
    if (!w || (side != 0 && side != 1)) throw Error(kInvalid, "bfly_pair: bad twiddle or side");
    if (d_out == d_mine || d_out == d_theirs) throw Error(kInvalid, "bfly_pair_peer: the output must be a third buffer");
    U128 t;
    t.lo = w[0];
    t.hi = w[1];
    bfly_pair_device(const_cast<uint4*>(reinterpret_cast<const uint4*>(d_mine)), reinterpret_cast<const uint4*>(d_theirs),
                     n, t, side, inverse != 0, (cudaStream_t)stream, tower != 0, reinterpret_cast<uint4*>(d_out));
  });
}

fpm_status fpm_ipc_alloc(size_t bytes, void** d_ptr, uint8_t* handle) {
  return guard([&] {
    require_device();
    if (!d_ptr || !handle || !bytes) throw Error(kInvalid, "ipc_alloc: null argument or size");
    FPM_CUDA(cudaMalloc(d_ptr, bytes));
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, *d_ptr);
    if (e != cudaSuccess) {
      cudaFree(*d_ptr);
      *d_ptr = nullptr;
      throw Error(kCuda, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    }
    static_assert(sizeof(h) == FPM_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
  });
}

fpm_status fpm_ipc_open(const uint8_t* handle, void** d_peer) {
  return guard([&] {
    require_device();
    if (!handle || !d_peer) throw Error(kInvalid, "ipc_open: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    FPM_CUDA(cudaIpcOpenMemHandle(d_peer, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

fpm_status fpm_ipc_close(void* d_peer) {
  return guard([&] { FPM_CUDA(cudaIpcCloseMemHandle(d_peer)); });
}

fpm_status fpm_ipc_free(void* d_ptr) {
  return guard([&] { FPM_CUDA(cudaFree(d_ptr)); });
}

fpm_status fpm_shard_local_product_dev(uint64_t* d_ea, uint64_t* d_eb, unsigned l, const uint64_t* base,
                                       void* stream) {
  return guard([&] {
    require_device();
    if (!base) throw Error(kInvalid, "local product: null base");
    if (!fpm_shard_tower(l)) throw Error(kInvalid, "local product: the coset needs 2^18 or more elements");
    int dev;
    FPM_CUDA(cudaGetDevice(&dev));
    U128 b;
    b.lo = base[0];
    b.hi = base[1];
    const TwiddleSrc tw = make_twiddle_src(dev, l, b);
    const unsigned T = pipeline_tile_log2(l);
    const cudaStream_t s = (cudaStream_t)stream;
    uint4* ea = reinterpret_cast<uint4*>(d_ea);
    uint4* eb = reinterpret_cast<uint4*>(d_eb);
    butterfly_top_device(ea, l, T, false, tw, s, true, eb);  // both operands per launch
    butterfly_tile_tower_device(ea, eb, l, T, tw, s);
    butterfly_top_device(eb, l, T, true, tw, s, true);
  });
}

fpm_status fpm_decode_cols_split_dev(const uint64_t* d_ev, size_t ncols, size_t col0, size_t row_bits, uint64_t* d_lo,
                                     uint64_t* d_hi, int tower, void* stream) {
  return guard([&] {
    require_device();
    if (!d_ev || !d_lo || !d_hi) throw Error(kInvalid, "decode_cols_split: null pointer");
    decode_cols_split_device(reinterpret_cast<const uint4*>(d_ev), ncols, col0, row_bits, reinterpret_cast<uint32_t*>(d_lo),
                             reinterpret_cast<uint32_t*>(d_hi), (cudaStream_t)stream, tower != 0);
  });
}

fpm_status fpm_i_basis_cvt_block32_dev(uint64_t* d_lo, const uint64_t* d_top, void* stream) {
  return guard([&] {
    require_device();
    if (!d_lo) throw Error(kInvalid, "i_basis_cvt_block32: null block");
    basis_cvt_block32_inverse(reinterpret_cast<uint32_t*>(d_lo), reinterpret_cast<const uint32_t*>(d_top),
                              (cudaStream_t)stream);
  });
}

fpm_status fpm_top_bit_fix_dev(uint64_t* d_hi, void* stream) {
  return guard([&] {
    require_device();
    if (!d_hi) throw Error(kInvalid, "top_bit_fix: null block");
    top_bit_fix_device(reinterpret_cast<uint32_t*>(d_hi), (cudaStream_t)stream);
  });
}

fpm_status fpm_load_operand_dev(uint64_t* d_dst, size_t dst_words, const uint64_t* d_src, size_t src_bits, void* stream) {
  return guard([&] {
    require_device();
    if (!dst_words) return;
    launch_k(load_operand_kernel, dim3(grid_1d(dst_words)), dim3(256), 0, (cudaStream_t)stream, d_dst, dst_words, d_src, src_bits);
    FPM_LAUNCH_CHECK();
  });
}


fpm_status fpm_b32_regather_dev(uint64_t* d_w, const uint64_t* const* d_srcs, int from, int to, int q, int Q, void* stream) {
  return guard([&] {
    require_device();
    check_q(q, Q);
    if (!d_w || from < 0 || from > 2 || to < 0 || to > 2 || from == to) throw Error(kInvalid, "regather: bad arguments");
    b32_regather(reinterpret_cast<uint32_t*>(d_w), rank_ptrs(d_srcs, Q), from, to, q, Q, (cudaStream_t)stream);
  });
}

fpm_status fpm_b32_l1_outer_dev(uint64_t* d_w, uint64_t* d_side, int inverse, int q, int Q, void* stream) {
  return guard([&] {
    require_device();
    check_q(q, Q);
    if (!d_w || !d_side) throw Error(kInvalid, "b32_l1_outer: null pointer");
    b32_l1_outer(reinterpret_cast<const uint32_t*>(d_w), reinterpret_cast<uint32_t*>(d_w), reinterpret_cast<uint32_t*>(d_side),
                 inverse != 0, q, Q, (cudaStream_t)stream);
  });
}

fpm_status fpm_b32_l1_outer_fix_dev(uint64_t* d_w, const uint64_t* d_side, int inverse, unsigned e_lo, unsigned e_hi,
                                    void* stream) {
  return guard([&] {
    require_device();
    if (!d_w || !d_side || e_lo > e_hi || e_hi > 256) throw Error(kInvalid, "b32_l1_outer_fix: bad arguments");
    b32_l1_outer_fix(reinterpret_cast<uint32_t*>(d_w), reinterpret_cast<const uint32_t*>(d_side), inverse != 0, e_lo, e_hi,
                     (cudaStream_t)stream);
  });
}

fpm_status fpm_b32_rows_dev(uint64_t* d_rows, size_t rows, int inverse, void* stream) {
  return guard([&] {
    require_device();
    if (!d_rows || !rows || rows % 256 || rows > 65536) throw Error(kInvalid, "b32_rows: whole chunks of 256 rows");
    b32_rows(reinterpret_cast<uint32_t*>(d_rows), rows, inverse != 0, (cudaStream_t)stream);
  });
}

fpm_status fpm_b32_cols_dev(uint64_t* d_w, int inverse, int q, int Q, void* stream) {
  return guard([&] {
    require_device();
    check_q(q, Q);
    if (!d_w) throw Error(kInvalid, "b32_cols: null block");
    b32_cols(reinterpret_cast<uint32_t*>(d_w), inverse != 0, q, Q, (cudaStream_t)stream);
  });
}

fpm_status fpm_b32_top_pass_dev(uint64_t* d_lo, const uint64_t* const* d_his, int q, int Q, void* stream) {
  return guard([&] {
    require_device();
    check_q(q, Q);
    if (!d_lo) throw Error(kInvalid, "b32_top_pass: null block");
    b32_top_pass(reinterpret_cast<uint32_t*>(d_lo), rank_ptrs(d_his, Q), q, Q, (cudaStream_t)stream);
  });
}

fpm_status fpm_b32_top_bit_fix_dev(uint64_t* d_hi0, const uint64_t* d_hi_last, void* stream) {
  return guard([&] {
    require_device();
    if (!d_hi0 || !d_hi_last) throw Error(kInvalid, "b32_top_bit_fix: null pointer");
    b32_top_bit_fix(reinterpret_cast<uint32_t*>(d_hi0), reinterpret_cast<const uint32_t*>(d_hi_last), (cudaStream_t)stream);
  });
}

fpm_status fpm_encode_cols_owners_dev(const uint64_t* const* d_polys, int Q, unsigned l, size_t col0, size_t ncols,
                                      int rows_live, uint64_t* d_ev, int tower, void* stream) {
  return guard([&] {
    require_device();
    if (!d_ev) throw Error(kInvalid, "encode_cols_owners: null output");
    if (rows_live != 64 && rows_live != 128) throw Error(kInvalid, "encode_cols_owners: rows_live must be 64 or 128");
    encode_cols_owners(rank_ptrs(d_polys, Q), Q, l, col0, ncols, reinterpret_cast<uint4*>(d_ev), rows_live,
                       (cudaStream_t)stream, tower != 0);
  });
}

fpm_status fpm_decode_cols_owners_dev(const uint64_t* d_ev, size_t ncols, size_t col0, size_t row_bits,
                                      const uint64_t* const* d_los, const uint64_t* const* d_his, int Q, int tower,
                                      void* stream) {
  return guard([&] {
    require_device();
    if (!d_ev) throw Error(kInvalid, "decode_cols_owners: null input");
    decode_cols_owners(reinterpret_cast<const uint4*>(d_ev), ncols, col0, row_bits, rank_ptrs(d_los, Q), rank_ptrs(d_his, Q), Q,
                       (cudaStream_t)stream, tower != 0);
  });
}

fpm_status fpm_copy_dev(void* d_dst, const void* d_src, size_t bytes, void* stream) {
  return guard([&] {
    require_device();
    if (bytes) FPM_CUDA(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  });
}

fpm_status fpm_bfly_pair_dev(uint64_t* d_mine, const uint64_t* d_theirs, size_t n, const uint64_t* w, int side,
                             int inverse, void* stream) {
  return guard([&] {
    require_device();
    if (!w || (side != 0 && side != 1)) throw Error(kInvalid, "bfly_pair: bad twiddle or side");
    U128 t;
    t.lo = w[0];
    t.hi = w[1];
    bfly_pair_device(reinterpret_cast<uint4*>(d_mine), reinterpret_cast<const uint4*>(d_theirs), n, t, side,
                     inverse != 0, (cudaStream_t)stream);
  });
}

fpm_status fpm_twiddle128(unsigned i, uint64_t b, const uint64_t* base, uint64_t* out) {
  return guard([&] {
    if (!base || !out || i >= 128) throw Error(kInvalid, "twiddle: bad arguments");
    U128 c;  // (base >> i) ^ 2b
    c.lo = i == 0 ? base[0] : (i < 64 ? (base[0] >> i) | (base[1] << (64 - i)) : base[1] >> (i - 64));
    c.hi = i == 0 ? base[1] : (i < 64 ? base[1] >> i : 0);
    c.lo ^= b << 1;
    c.hi ^= b >> 63;
    const U128 p = host_cantor_to_poly(field_tables(), c);
    out[0] = p.lo;
    out[1] = p.hi;
  });
}

fpm_status fpm_pointwise_dev(const uint64_t* d_u, const uint64_t* d_v, uint64_t* d_out, size_t n, void* stream) {
  return guard([&] {
    require_device();
    pointwise_device(reinterpret_cast<const uint4*>(d_u), reinterpret_cast<const uint4*>(d_v),
                     reinterpret_cast<uint4*>(d_out), n, (cudaStream_t)stream);
  });
}

// ---- host wrappers

fpm_status fpm_basis_cvt(uint64_t* w, size_t n_bits, size_t content_bits, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (n_bits == 0 || (n_bits & (n_bits - 1))) throw Error(kInvalid, "basis_cvt: length must be a power of two");
    if (n_bits <= 2) return;
    const size_t bytes = (n_bits + 63) / 64 * 8;
    DevBuf W(bytes, s);
    FPM_CUDA(cudaMemcpyAsync(W.p, w, bytes, cudaMemcpyHostToDevice, s));
    basis_cvt_device(W.as<uint32_t>(), n_bits, content_bits ? std::min(content_bits, n_bits) : 1, false, s);
    FPM_CUDA(cudaMemcpyAsync(w, W.p, bytes, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_i_basis_cvt(uint64_t* w, size_t n_bits, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (n_bits == 0 || (n_bits & (n_bits - 1))) throw Error(kInvalid, "basis_cvt: length must be a power of two");
    if (n_bits <= 2) return;
    const size_t bytes = (n_bits + 63) / 64 * 8;
    DevBuf W(bytes, s);
    FPM_CUDA(cudaMemcpyAsync(W.p, w, bytes, cudaMemcpyHostToDevice, s));
    basis_cvt_device(W.as<uint32_t>(), n_bits, n_bits, true, s);
    FPM_CUDA(cudaMemcpyAsync(w, W.p, bytes, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_encode(const uint64_t* poly, unsigned l, uint64_t* ev, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    const size_t pb = ((size_t)128 << l) / 8, eb = ((size_t)16 << l);
    DevBuf P(pb, s), E(eb, s);
    FPM_CUDA(cudaMemcpyAsync(P.p, poly, pb, cudaMemcpyHostToDevice, s));
    encode_device(P.as<uint32_t>(), l, E.as<uint4>(), s);
    FPM_CUDA(cudaMemcpyAsync(ev, E.p, eb, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_decode(const uint64_t* ev, unsigned l, uint64_t* poly, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    const size_t pb = ((size_t)128 << l) / 8, eb = ((size_t)16 << l);
    DevBuf P(pb, s), E(eb, s);
    FPM_CUDA(cudaMemcpyAsync(E.p, ev, eb, cudaMemcpyHostToDevice, s));
    decode_device(E.as<uint4>(), l, P.as<uint32_t>(), s);
    FPM_CUDA(cudaMemcpyAsync(poly, P.p, pb, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_lch_butterfly(uint64_t* ev, unsigned l, const uint64_t* base, int inverse, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (l > 64) throw Error(kInvalid, "lch_butterfly: at most 64 layers");
    if (l == 0) return;
    if (!base) throw Error(kInvalid, "lch_butterfly: null base");
    U128 b;
    b.lo = base[0];
    b.hi = base[1];
    const size_t eb = ((size_t)16 << l);
    DevBuf E(eb, s);
    FPM_CUDA(cudaMemcpyAsync(E.p, ev, eb, cudaMemcpyHostToDevice, s));
    butterfly_device(E.as<uint4>(), l, b, inverse != 0, s);
    FPM_CUDA(cudaMemcpyAsync(ev, E.p, eb, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_butterfly(uint64_t* ev, unsigned l, int inverse, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (l >= 64) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
    if (l == 0) return;
    const size_t eb = ((size_t)16 << l);
    DevBuf E(eb, s);
    FPM_CUDA(cudaMemcpyAsync(E.p, ev, eb, cudaMemcpyHostToDevice, s));
    butterfly_device(E.as<uint4>(), l, partition_base(l), inverse != 0, s);
    FPM_CUDA(cudaMemcpyAsync(ev, E.p, eb, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_pointwise(const uint64_t* u, const uint64_t* v, uint64_t* out, size_t n, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (!n) return;
    DevBuf U(n * 16, s), V(n * 16, s);
    FPM_CUDA(cudaMemcpyAsync(U.p, u, n * 16, cudaMemcpyHostToDevice, s));
    FPM_CUDA(cudaMemcpyAsync(V.p, v, n * 16, cudaMemcpyHostToDevice, s));
    pointwise_device(U.as<uint4>(), V.as<uint4>(), U.as<uint4>(), n, s);
    FPM_CUDA(cudaMemcpyAsync(out, U.p, n * 16, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_gf128_mul(const uint64_t* a, const uint64_t* b, uint64_t* out, size_t n, int device) {
  return fpm_pointwise(a, b, out, n, device);
}

// ---- GF(2^64) stages
fpm_status fpm_tables64(uint64_t* cantor, uint64_t* rows, uint64_t* inv_rows) {
  return guard([&] {
    const FieldTables& t = field_tables64();
    for (int i = 0; i < 64; ++i) {
      if (cantor) cantor[i] = t.cantor[i].lo;
      if (rows) rows[i] = t.enc_rows[i].lo;
      if (inv_rows) inv_rows[i] = t.inv_rows[i].lo;
    }
  });
}

static void check_l64(unsigned l) {
  if (l >= 32) throw Error(kInvalid, "PartitionSpec: l must satisfy l < m/2");
}

fpm_status fpm_encode64_dev(const uint64_t* d_poly, unsigned l, uint64_t* d_ev, void* stream) {
  return guard([&] {
    require_device();
    check_l64(l);
    encode64_device(reinterpret_cast<const uint32_t*>(d_poly), l, reinterpret_cast<uint2*>(d_ev), 64,
                    (cudaStream_t)stream);
  });
}

fpm_status fpm_decode64_dev(const uint64_t* d_ev, unsigned l, uint64_t* d_poly, void* stream) {
  return guard([&] {
    require_device();
    check_l64(l);
    decode64_device(reinterpret_cast<const uint2*>(d_ev), l, reinterpret_cast<uint32_t*>(d_poly), (cudaStream_t)stream);
  });
}

fpm_status fpm_lch_butterfly64_dev(uint64_t* d_ev, unsigned l, uint64_t base, int inverse, void* stream) {
  return guard([&] {
    require_device();
    if (l > 63) throw Error(kInvalid, "lch_butterfly: at most 63 layers");
    if (l == 0) return;
    butterfly64_device(reinterpret_cast<uint2*>(d_ev), l, base, inverse != 0, (cudaStream_t)stream);
  });
}

fpm_status fpm_pointwise64_dev(const uint64_t* d_u, const uint64_t* d_v, uint64_t* d_out, size_t n, void* stream) {
  return guard([&] {
    require_device();
    pointwise64_device(reinterpret_cast<const uint2*>(d_u), reinterpret_cast<const uint2*>(d_v),
                       reinterpret_cast<uint2*>(d_out), n, (cudaStream_t)stream);
  });
}

fpm_status fpm_encode64(const uint64_t* poly, unsigned l, uint64_t* ev, int device) {
  return host_call(device, [&](cudaStream_t s) {
    check_l64(l);
    const size_t pb = ((size_t)64 << l) / 8, eb = ((size_t)8 << l);
    DevBuf P(pb < 8 ? 8 : pb, s), E(eb, s);
    FPM_CUDA(cudaMemcpyAsync(P.p, poly, (pb + 7) / 8 * 8, cudaMemcpyHostToDevice, s));
    encode64_device(P.as<uint32_t>(), l, E.as<uint2>(), 64, s);
    FPM_CUDA(cudaMemcpyAsync(ev, E.p, eb, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_decode64(const uint64_t* ev, unsigned l, uint64_t* poly, int device) {
  return host_call(device, [&](cudaStream_t s) {
    check_l64(l);
    const size_t pb = ((size_t)64 << l) / 8, eb = ((size_t)8 << l);
    DevBuf P(pb < 8 ? 8 : pb, s), E(eb, s);
    FPM_CUDA(cudaMemcpyAsync(E.p, ev, eb, cudaMemcpyHostToDevice, s));
    FPM_CUDA(cudaMemsetAsync(P.p, 0, pb < 8 ? 8 : pb, s));
    decode64_device(E.as<uint2>(), l, P.as<uint32_t>(), s);
    FPM_CUDA(cudaMemcpyAsync(poly, P.p, (pb + 7) / 8 * 8, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_lch_butterfly64(uint64_t* ev, unsigned l, uint64_t base, int inverse, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (l > 63) throw Error(kInvalid, "lch_butterfly: at most 63 layers");
    if (l == 0) return;
    const size_t eb = ((size_t)8 << l);
    DevBuf E(eb, s);
    FPM_CUDA(cudaMemcpyAsync(E.p, ev, eb, cudaMemcpyHostToDevice, s));
    butterfly64_device(E.as<uint2>(), l, base, inverse != 0, s);
    FPM_CUDA(cudaMemcpyAsync(ev, E.p, eb, cudaMemcpyDeviceToHost, s));
  });
}

fpm_status fpm_pointwise64(const uint64_t* u, const uint64_t* v, uint64_t* out, size_t n, int device) {
  return host_call(device, [&](cudaStream_t s) {
    if (!n) return;
    DevBuf U(n * 8, s), V(n * 8, s);
    FPM_CUDA(cudaMemcpyAsync(U.p, u, n * 8, cudaMemcpyHostToDevice, s));
    FPM_CUDA(cudaMemcpyAsync(V.p, v, n * 8, cudaMemcpyHostToDevice, s));
    pointwise64_device(U.as<uint2>(), V.as<uint2>(), U.as<uint2>(), n, s);
    FPM_CUDA(cudaMemcpyAsync(out, U.p, n * 8, cudaMemcpyDeviceToHost, s));
  });
}

}  // extern "C"
