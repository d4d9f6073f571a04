// fpm_internal.h -- shared host-side declarations of the CUDA library (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>

#include "fpm_tables.h"

namespace fpm {

// Status codes of the C-ABI (include/fpmul_b200.h).
enum Status : int { kOk = 0, kInvalid = 1, kCuda = 2, kNoMem = 3 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FPM_CUDA(x)                                                                            \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw ::fpm::Error(e_ == cudaErrorMemoryAllocation ? ::fpm::kNoMem : ::fpm::kCuda,        \
                         std::string(#x) + ": " + cudaGetErrorString(e_));                     \
  } while (0)
// C-ABI error plumbing: runs fn, maps exceptions to status codes and the thread-local
// fpm_last_error() message.
void set_last_error(const char* msg);
template <class Fn>
int fpm_guard_impl(Fn&& fn) {
  try {
    fn();
    return kOk;
  } catch (const Error& e) {
    set_last_error(e.what());
    if (e.code == kCuda) cudaGetLastError();  // (clear the runtime's own last-error slot, as guard() in fpm_capi.cu)
    return e.code;
  } catch (const std::bad_alloc& e) {
    set_last_error(e.what());
    return kNoMem;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return kCuda;
  }
}
#define fpm_guard(...) ((fpm_status)::fpm::fpm_guard_impl(__VA_ARGS__))

// Every kernel launch of the library goes through this check; it also feeds fpm_launch_count().
void note_launch();
#define FPM_LAUNCH_CHECK()             \
  do {                                 \
    ::fpm::note_launch();              \
    FPM_CUDA(cudaGetLastError());      \
  } while (0)

// Stream-ordered scratch from the library's own per-device memory pool (never the device's default
// pool, so the host application's allocator and cudaMallocAsync users are unaffected).  Freed pool
// memory stays cached for the next call (reentrant per-call scratch at GiB scale); fpm_trim_pool
// returns it to the driver.
void* pool_alloc(size_t bytes, cudaStream_t s);
void pool_free(void* p, cudaStream_t s);
void trim_pool(int dev);
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  DevBuf(size_t bytes, cudaStream_t st) : s(st) { if (bytes) p = pool_alloc(bytes, st); }
  ~DevBuf() { if (p) pool_free(p, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// A timing-disabled event released on every exit path (destroying an event with waits still pending
// is allowed: the waits complete and the event is freed afterwards).
struct Ev {
  cudaEvent_t e = nullptr;
  Ev() { FPM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~Ev() { if (e) cudaEventDestroy(e); }
  Ev(const Ev&) = delete;
  Ev& operator=(const Ev&) = delete;
};

// Programmatic dependent launch (sm_90+).  Every library kernel begins with pdl_wait() (the
// previous kernel of its stream has completed and its writes are visible -- nothing is read before
// it) and pdl_trigger() (the stream's next kernel may be scheduled now; its CTAs park at their own
// pdl_wait), and every launch goes through launch_k with the programmatic-serialization attribute:
// back-to-back kernels overlap their launch latency instead of leaving a gap (graphs keep the edges
// as programmatic dependencies).  FPM_PDL=0 launches without the attribute (plain serialization).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
bool pdl_enabled();
template <class... KArgs, class... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);  // errors: FPM_LAUNCH_CHECK
}

// Runs an initialisation (e.g. cudaFuncSetAttribute of a kernel's dynamic shared memory) once per
// device: kernel attributes belong to a device context, so a process driving several GPUs must set
// them on each one.  Thread-safe; devices 0..63.
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  template <class Fn>
  void run(Fn&& fn) {
    int dev = 0;
    FPM_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = uint64_t{1} << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    fn();
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
};

// Grid of a persistent (grid-stride) kernel: as many CTAs as are co-resident on the device
// (occupancy query for the actual threads / dynamic shared memory), capped at the work items --
// a grid that is not a multiple of the resident slots leaves a half-empty last wave.
template <class K>
int resident_grid(K kernel, int threads, size_t smem, uint64_t work) {
  int dev = 0, sms = 0, per_sm = 0;
  FPM_CUDA(cudaGetDevice(&dev));
  FPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  FPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  if (per_sm < 1) per_sm = 1;
  const uint64_t g = (uint64_t)sms * per_sm;
  return (int)(work < g ? (work ? work : 1) : g);
}

// Per-device immutable tables (uploaded once, lazily, under a mutex -- the reference's
// thread-safe singletons CantorField::get / EncodeMatrix::get, cantor.cpp:136-140).
struct DeviceTables {
  uint4* cantor = nullptr;    // 128 x v_i
  uint4* enc_rows = nullptr;  // 128 x r_j
  uint4* inv_rows = nullptr;  // 128 rows of E^{-1}
  uint4* enc_m8 = nullptr;    // rotated 8-bit tables (gf128.cuh m8 layout) of x*E
  uint4* dec_m8 = nullptr;    // ... of x*E^{-1}
  uint4* c2p = nullptr;       // 4 x 512: part p entry e = C2P(2 * (e << 9p))
  // Tower representation R (fpm_tables.h TowerTables), used inside the product pipeline's FFT:
  uint4* to_r = nullptr;      // 128 x R(x^k): rows of the poly -> R map
  uint4* to_poly = nullptr;   // 128 x e_k in poly: rows of the R -> poly map
  uint4* enc_m8r = nullptr;   // M8 tables of x -> R(x*E)
  uint4* dec_m8r = nullptr;   // M8 tables of x_R -> poly(x)*E^{-1}
  // the same split by output half (h = 0: product rows 0..63, the lower 2^32-bit block of a 2^33-bit
  // product; h = 1: rows 64..127, the upper block): entry (byte v, byte index c < 16) at v * 16 + c,
  // 8 bytes each -- sixteen lanes rotated over the sixteen c read distinct banks with LDS.64
  uint2* dec_half_r[2] = {nullptr, nullptr};
  // GF(2^64) (run_pipeline<gf64>): G8 tables (gf64.cuh layout) of x*E and x*E^{-1}, C2P tables
  uint2* enc_g8 = nullptr;
  uint2* dec_g8 = nullptr;
  uint2* c2p64 = nullptr;     // 4 x 512, as c2p
  uint2* rows64 = nullptr;    // 64 x r_j
  uint2* inv64 = nullptr;     // 64 rows of E^{-1}
  // GF(2^64) tower representation (fpm_tables.h tower_tables64): as the GF(2^128) fields above
  uint2* to_r64 = nullptr;
  uint2* to_poly64 = nullptr;
  uint2* enc_g8r = nullptr;
  uint2* dec_g8r = nullptr;
};

void flip_encode_tables(int dev, cudaStream_t s);  // fault-injection test hook (k_codec.cu)

// Twiddle generator inputs (passed by value as a kernel parameter):
//   w(i, b) = C2P((base >> i) ^ 2b) = layer[i] ^ C2P(2b)      (butterfly.cpp:45-49; C2P is linear)
// layer[i] = C2P(base >> i); the pipeline's base is e_{l+64} (encode.cpp:47) so layer[i] = v_{l+64-i}.
constexpr int kMaxLayers = 64;
struct TwiddleSrc {
  const uint4* c2p;          // device: 4 x 512 C2P(2 * (e << 9p)) tables
  const uint4* to_r;         // device: DeviceTables::to_r (tower-representation table rows)
  const uint4* to_poly;      // device: DeviceTables::to_poly
  uint64_t tau;              // TowerTables::tau, byte b = R(v_{b+1}) (subfield twiddle parts)
  uint4 layer[kMaxLayers];   // C2P(base >> i)
};
// Host: twiddle source for plan_butterflies(l, base) (base in Cantor coordinates).
TwiddleSrc make_twiddle_src(int device, unsigned l, U128 base);
struct TwiddleSrc64 {
  const uint2* c2p;
  const uint2* to_r;     // DeviceTables::to_r64
  const uint2* to_poly;  // DeviceTables::to_poly64
  uint64_t tau;          // tower_tables64().tau
  uint2 layer[kMaxLayers];
};
TwiddleSrc64 make_twiddle_src64(int device, unsigned l, uint64_t base);
inline uint64_t partition_base64(unsigned l) { return uint64_t{1} << (l + 32); }  // e_{l+32}
inline U128 partition_base(unsigned l) {  // make_partition_spec<gf128>(l).base = e_{l+64}
  U128 b;
  if (l + 64 < 64) b.lo = uint64_t{1} << (l + 64); else b.hi = uint64_t{1} << (l + 64 - 64);
  return b;
}

const DeviceTables& device_tables(int device);

// Basis conversion (k_basis.cu).  w: n_bits/32 uint32 words on the device, in place.
// live_bits: forward only; bits >= live_bits are zero on entry (zero-tail skip).
// on_final (inverse only, may be null): called with word ranges [w0, w1) of w (32-bit words) as soon
// as the work enqueued on s so far leaves them final, so callers can start copying them out while
// the rest of the conversion runs; every word is reported exactly once.
using FinalFn = std::function<void(uint64_t w0, uint64_t w1)>;
// src (forward, 2^17..2^32 bits only; may be null): the unconverted array is read from src and the
// result written to w (w's prior contents are ignored).
// enc (forward 2^32-bit conversions only, basis_cvt_can_encode): the conversion's last step writes
// the GF(2^128) encode of the converted operand (64 live partition rows, l = 26) to enc->ev instead
// of the converted bits (w is then scratch on exit).
struct EncodeSink {
  void* ev;    // 2^26 uint4 (m = 128) or 2^27 uint2 (m = 64) elements
  bool tower;  // elements in the tower representation R (the product pipeline's FFT)
  int m = 128; // field degree
};
bool basis_cvt_can_encode(size_t n_bits, bool tower);
// dec (inverse 2^33-bit conversions only, basis_cvt_can_decode): the GF(2^128) decode of dec->ev
// (2^26 elements) is the conversion's input -- fused into its first step; w's contents on entry are
// ignored.
struct DecodeSource {
  const void* ev;
  bool tower;
  int m = 128;
};
bool basis_cvt_can_decode(size_t n_bits);
void conv_rows_batch16(uint32_t* data, uint64_t nwords, bool inv, cudaStream_t s);
// config-2 batches in the tower representation (k_codec.cu): 2^16-bit operands / 2^17-bit products
void encode_batch_r(const uint32_t* polys, uint64_t count, uint64_t stride_words, uint4* ev, cudaStream_t s);
void decode_batch_r(const uint4* ev, uint64_t count, uint32_t* out, uint64_t stride_words, cudaStream_t s);
bool concurrent_blocks_enabled();  // FPM_CONCURRENT_BLOCKS=0 disables the concurrent conversions
cudaStream_t side_stream(int dev);
// concurrent (2^33-bit inverse): the lower block's conversion runs on a second stream beside the
// upper block's (only its last step waits for the final upper block) -- device-resident products;
// host-buffer calls keep the upper block first and alone (its copy-out starts earlier).
void basis_cvt_device(uint32_t* w, size_t n_bits, size_t live_bits, bool inverse, cudaStream_t s,
                      const FinalFn* on_final = nullptr, const uint32_t* src = nullptr,
                      const EncodeSink* enc = nullptr, const DecodeSource* dec = nullptr,
                      bool concurrent = false);

// The halves of a 2^33-bit inverse conversion as separate calls (sharded products: the two 2^32-bit
// blocks converted on different GPUs).  Upper block: basis_cvt_device(w_hi, 2^32, 2^32, true, s); then
// the lower block with the fused top pass reading the final upper block (may be peer memory); then
// top_bit_fix_device on the upper block.
void basis_cvt_block32_inverse(uint32_t* w_lo, const uint32_t* top, cudaStream_t s);
void top_bit_fix_device(uint32_t* hi_block, cudaStream_t s);
// The sharded 2^32-bit conversion (k_basis.cu; fpm_multi.cu at P >= 4): phase steps on one rank's
// full-size replica of a block, Q = 2 or 4 ranks per block.
enum { kDistWindow = 0, kDistChunk = 1, kDistColumn = 2 };
struct RankPtrs {
  uint32_t* p[4];
};
void b32_regather(uint32_t* dst, const RankPtrs& src, int from, int to, int q, int Q, cudaStream_t s);
void b32_l1_outer(const uint32_t* src, uint32_t* w, uint32_t* side, bool inv, int q, int Q, cudaStream_t s);
void b32_l1_outer_fix(uint32_t* w, const uint32_t* side, bool inv, uint32_t e_lo, uint32_t e_hi, cudaStream_t s);
void b32_rows(uint32_t* w_rows, uint64_t rows, bool inv, cudaStream_t s);
void b32_cols(uint32_t* w, bool inv, int q, int Q, cudaStream_t s);
void b32_top_pass(uint32_t* lo, const RankPtrs& hi, int q, int Q, cudaStream_t s);
void b32_top_bit_fix(uint32_t* hi0, const uint32_t* hi_last_owner, cudaStream_t s);
std::vector<std::pair<uint64_t, uint64_t>> b32_window_ranges(int q, int Q);
void encode_cols_owners(const RankPtrs& polys, int Q, unsigned l, uint64_t col0, uint64_t ncols, uint4* ev,
                        int rows_live, cudaStream_t s, bool tower);
void decode_cols_owners(const uint4* ev, uint64_t ncols, uint64_t col0, uint64_t row_bits, const RankPtrs& los,
                        const RankPtrs& his, int Q, cudaStream_t s, bool tower);


// Encode / decode (k_codec.cu).  poly has 128 * 2^l bits; ev has 2^l uint4.
void encode_device(const uint32_t* poly, unsigned l, uint4* ev, cudaStream_t s);
// rows_live = 64: rows >= 64 of poly are known zero (pipeline operands) and not read.
// tower: write the elements in the tower representation R (product pipeline; n_p >= 1024).
void encode_device_rows(const uint32_t* poly, unsigned l, uint4* ev, int rows_live, cudaStream_t s, bool tower = false);
// Column (element) range of the partition matrix; used by the sharded multi-GPU product.
void encode_cols_device(const uint32_t* poly, unsigned l, uint64_t col0, uint64_t ncols, uint4* ev, int rows_live,
                        cudaStream_t s, bool tower = false);
void decode_cols_device(const uint4* ev, uint64_t ncols, uint32_t* slice, cudaStream_t s, bool tower = false);
// ncols elements -> columns [col0, col0 + ncols) of a 128-row partition matrix of row pitch row_bits,
// rows 0..63 written to lo, rows 64..127 to hi (each 64 rows of row_bits; either may be peer memory).
void decode_cols_split_device(const uint4* ev, uint64_t ncols, uint64_t col0, uint64_t row_bits, uint32_t* lo,
                              uint32_t* hi, cudaStream_t s, bool tower);
// One exchanged butterfly layer (sharded FFT): this rank holds `mine` (side 0 = p0 half, 1 = p1 half),
// the partner's half arrived in `theirs`; uniform twiddle w.  Result replaces `mine`.
// out (optional): write the result there instead of over `mine` (then `theirs` may be a peer GPU's
// memory that the partner reads concurrently: nothing of `mine` or `theirs` is overwritten).
void bfly_pair_device(uint4* mine, const uint4* theirs, uint64_t n, U128 w, int side, bool inverse, cudaStream_t s,
                      bool tower = false, uint4* out = nullptr);
void decode_device(const uint4* ev, unsigned l, uint32_t* poly, cudaStream_t s, bool tower = false);

// Butterflies (k_fft.cu).
void butterfly_device(uint4* ev, unsigned l, U128 base, bool inverse, cudaStream_t s);
void pointwise_device(const uint4* u, const uint4* v, uint4* out, size_t n, cudaStream_t s);
// Pipeline helpers exposing the split between top (radix-4 table passes) and bottom (tile) layers.
unsigned fft_tile_log2(unsigned l);
// tower: the elements are in the tower representation R (tables built in R).
void butterfly_top_device(uint4* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc& tw, cudaStream_t s,
                          bool tower = false, uint4* ev2 = nullptr);
void butterfly_tile_device(uint4* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc& tw, cudaStream_t s);
// Fused: forward layers [0, T) of b's tiles, pointwise * a, inverse layers [0, T).
bool tile_fused2_enabled(unsigned T);
bool tile64_fused2_enabled(unsigned T);
unsigned pipeline64_tile_log2(unsigned l);
void butterfly64_tile_fused2_device(const uint2* ea, uint2* eb, unsigned l, unsigned T, const TwiddleSrc64& tw,
                                    cudaStream_t s);
unsigned pipeline_tile_log2(unsigned l);
void butterfly_tile_fused2_device(const uint4* ea, uint4* eb, unsigned l, unsigned T, const TwiddleSrc& tw,
                                  cudaStream_t s);
// The same pass on tower-representation tiles (fft_tile_tower_kernel): every tile layer as one M8
// table of the tile's twiddle plus a GF(2^8)-scalar product for the per-block part; T in [10, 11].
bool tile_tower_enabled(unsigned T);
bool pipeline_fuses_operands(unsigned T);  // both operands' tile layers in one pass at depth T
bool pipeline_tower(unsigned T);           // ... on tower-representation tiles
void butterfly_tile_tower_device(const uint4* ea, uint4* eb, unsigned l, unsigned T, const TwiddleSrc& tw,
                                 cudaStream_t s,
                                 uint64_t batch = 0, uint64_t pre_tiles = 0);
// Host-buffer products: the forward R layers of operand a's first tower_pre_tiles(l, T) tiles run
// ahead of the fused pass, while operand b is still being uploaded.
uint64_t tower_pre_tiles(unsigned l, unsigned T);
void butterfly_tile_tower_pre_device(uint4* ev, unsigned l, unsigned T, const TwiddleSrc& tw, uint64_t pre_tiles,
                                     cudaStream_t s);
void butterfly_tile_fused_device(const uint4* ea, uint4* eb, unsigned l, unsigned T, const TwiddleSrc& tw,
                                 cudaStream_t s);

// GF(2^64) stages (k_fft64.cu, k_codec.cu): 64-row partition matrix, 8-byte elements.
unsigned fft64_tile_log2(unsigned l);
void butterfly64_device(uint2* ev, unsigned l, uint64_t base, bool inverse, cudaStream_t s);
void butterfly64_top_device(uint2* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc64& tw, cudaStream_t s,
                            bool tower = false, uint2* ev2 = nullptr);
bool tile64_tower_enabled(unsigned T);
void butterfly64_tile_tower_device(const uint2* ea, uint2* eb, unsigned l, unsigned T, const TwiddleSrc64& tw,
                                   cudaStream_t s, uint64_t pre_tiles = 0);
uint64_t tower64_pre_tiles(unsigned l, unsigned T);
void butterfly64_tile_tower_pre_device(uint2* ev, unsigned l, unsigned T, const TwiddleSrc64& tw, uint64_t pre_tiles,
                                       cudaStream_t s);
void butterfly64_tile_device(uint2* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc64& tw, cudaStream_t s);
void butterfly64_tile_fused_device(const uint2* ea, uint2* eb, unsigned l, unsigned T, const TwiddleSrc64& tw,
                                   cudaStream_t s);
void pointwise64_device(const uint2* u, const uint2* v, uint2* out, size_t n, cudaStream_t s);
// rows_live = 32: rows >= 32 known zero (pipeline operands); 64: general.
// tower: elements in the GF(2^64) tower representation (product pipeline; n_p >= 1024).
void encode64_device(const uint32_t* poly, unsigned l, uint2* ev, int rows_live, cudaStream_t s, bool tower = false);
void decode64_device(const uint2* ev, unsigned l, uint32_t* poly, cudaStream_t s, bool tower = false);

// Whole small products in one CTA each (k_batch.cu); n_bits = padded product length <= 2^17.
// Carry-less word product out[0 .. wa + wb) = a * b (k_clmul.cu; polymul.cpp:156-183, 268-282).
void clmul_words_device(const uint64_t* a, uint64_t wa, const uint64_t* b, uint64_t wb, uint64_t* out,
                        cudaStream_t s);
// fp_polymul's auto-mode threshold (MulOptions::fft_threshold_bits default, polymul.hpp:65).
constexpr size_t kFftThresholdBits = size_t{1} << 12;
void polymul_batch_device(const uint64_t* a, size_t a_bits, size_t a_stride_words,
                          const uint64_t* b, size_t b_bits, size_t b_stride_words, uint64_t* c,
                          size_t c_stride_words, size_t count, cudaStream_t s);

}  // namespace fpm
