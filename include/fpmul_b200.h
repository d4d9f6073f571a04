/*
 * fpmul_b200.h -- C-ABI of the B200-native Frobenius-partition additive-FFT multiplier of
 * GF(2)[x] polynomials (arXiv 1803.11301), implemented in libfpmul_b200.so.
 *
 * This is the drop-in boundary for the reference's hot path (/root/reference/proj).  The
 * reference has no FFI of its own; its boundary is the C++ API in proj/include/fpmul/, and each
 * entry point below is what a binding of that API needs.  The C++ mirror
 * of the reference API (namespace fpmul, paper_1803_11301_b200/cpp/include/fpmul/) is implemented
 * on top of these functions; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Polynomials are packed little-endian uint64 words: coefficient k is bit k%64 of word k/64
 *    (proj/include/fpmul/bitpoly.hpp:28-31).  An EvalVec of 2^l GF(2^128) elements is 2*2^l
 *    uint64 words {lo, hi} per element (gf.hpp:24-52, butterfly.hpp:30-31).
 *  - The field is GF(2^128) = GF(2)[x]/(x^128+x^7+x^2+x+1) (gf.hpp:115-123), the north-star field.
 *  - *_dev functions take device pointers and a cudaStream_t (NULL = legacy default stream) and
 *    are asynchronous; the others take host pointers and are synchronous.
 *  - Every function returns an fpm_status; on error fpm_last_error() (thread-local) says why.
 *    FPM_EINVAL is what the reference reports as std::invalid_argument, FPM_ECUDA / FPM_ENOMEM
 *    replace its std::runtime_error failures (SURVEY.md section 8(b) "Errors").
 *  - Thread safety: reentrant; per-device state (tables, stream, scratch) is created lazily under
 *    a mutex, mirroring the reference's thread-safe singletons (cantor.cpp:136-140,
 *    polymul.cpp:63-74).  Results are deterministic and bit-identical to the reference.
 */
#ifndef FPMUL_B200_H_
#define FPMUL_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FPM_OK = 0,
  FPM_EINVAL = 1, /* invalid argument (reference: std::invalid_argument) */
  FPM_ECUDA = 2,  /* CUDA/NCCL failure, no device, or missing kernels */
  FPM_ENOMEM = 3  /* device or host allocation failed */
} fpm_status;

/* Field selection, mirroring FieldChoice (proj/include/fpmul/polymul.hpp:28-32). */
enum { FPM_FIELD_AUTO = 0, FPM_FIELD_GF64 = 64, FPM_FIELD_GF128 = 128 };

/* MulPlan (polymul.hpp:36-43). */
typedef struct {
  uint64_t n_bits;
  uint32_t log2_n;
  uint32_t field_degree;
  uint32_t log2_field_degree;
  uint32_t l;
  uint64_t n_p;
} fpm_plan;

/* Per-stage seconds in the order of StageSeconds (polymul.hpp:51-59):
 * basiscvt, encode, butterfly, pointwise, ibutterfly, decode, ibasiscvt. */
#define FPM_NUM_STAGES 7

const char* fpm_last_error(void);
/* Library version string. */
const char* fpm_version(void);
/* Number of CUDA devices visible (0 when none); never fails. */
int fpm_device_count(void);

/* Schedule introspection (no reference counterpart): in the product pipeline the butterfly layers
 * [0, T) of a 2^l-element transform run in shared-memory tiles, layers [T, l) in radix-4 passes;
 * fpm_pipeline_fuses_operands(l) = 1 when both operands' tile layers run inside the fused
 * pointwise pass (else operand a has its own tile pass).  Used by bench.py to attribute work to
 * kernels; never fail. */
unsigned fpm_fft_tile_log2(unsigned l);
int fpm_pipeline_fuses_operands(unsigned l);

/* plan_mul (proj/src/polymul.cpp:187-219).  field: FPM_FIELD_*; the pipeline runs the field the
 * plan reports (GF(2^64) for FPM_FIELD_AUTO whenever it supports the size). */
fpm_status fpm_plan_mul(size_t a_bits, size_t b_bits, int field, fpm_plan* out);

/* random_bitpoly(n_bits, std::mt19937_64(seed)) (proj/src/bitpoly.cpp:19-24, bitpoly.hpp:101):
 * ceil(n_bits/64) words, one generator draw per word, bits >= n_bits cleared.  Host only; the
 * seeded inputs of the BASELINE configs and the golden fixtures. */
fpm_status fpm_random_bitpoly(size_t n_bits, uint64_t seed, uint64_t* out);

/* fp_polymul (polymul.hpp:74-75, polymul.cpp:223-239) on host buffers.
 * c receives ceil((a_bits+b_bits-1)/64) words (bits >= a_bits+b_bits-1 cleared); nothing is
 * written when either length is 0.  field: FPM_FIELD_AUTO (short inputs: karatsuba_mul, else
 * plan_mul's field), FPM_FIELD_GF64 or FPM_FIELD_GF128.  stage_seconds: NULL or
 * double[FPM_NUM_STAGES] (accumulated).  device: CUDA ordinal.
 * Any host memory works; page-locked buffers (cudaHostAlloc / cudaHostRegister) let the uploads and
 * the download run at the PCIe rate and overlap the kernels (pageable memory is staged by the
 * driver).  Reentrant: concurrent callers overlap one another's copies and kernels. */
fpm_status fpm_polymul(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c,
                       int field, int device, double* stage_seconds);

/* fp_polymul over several GPUs from one process (the n_gpus argument;
 * reference entry point fp_polymul, proj/include/fpmul/polymul.hpp:74-75): host buffers as
 * fpm_polymul; the product is sharded over the listed devices as logical ranks (a power of two in
 * [2, 64]; a device may repeat, e.g. {0, 0, 0, 0} runs 4 logical ranks on GPU 0): rank g owns
 * evaluation elements [g m, (g+1) m), the top log2 P butterfly layers read the partner rank's half
 * from its memory over NVLink (peer access is enabled on the listed devices), the operands'
 * conversions run on ranks 0 and 1, and a 2^33-bit product's two inverse-conversion blocks run on
 * ranks 0 and 1.  Needs >= 1024 evaluation elements per rank.  n_devices == 1 is fpm_polymul.
 * The transform is GF(2^128) for every field choice (products are field-independent); `field` is
 * validated as in fpm_plan_mul. */
fpm_status fpm_polymul_multi(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c,
                             int field, const int* devices, int n_devices);
/* fpm_polymul_multi on devices 0 .. n_gpus-1. */
fpm_status fpm_polymul_n(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c, int field,
                         int n_gpus);

/* The same on device-resident buffers (d_c sized as above).  Uses the calling thread's current
 * device.  Synchronizes `stream` only when stage_seconds != NULL. */
fpm_status fpm_polymul_dev(const uint64_t* d_a, size_t a_bits, const uint64_t* d_b, size_t b_bits, uint64_t* d_c,
                           int field, void* stream, double* stage_seconds);

/* `count` independent products of equal shapes (BASELINE config 2): operand k is at
 * d_a + k*a_stride_words etc.; product k at d_c + k*c_stride_words.  Requires
 * next_pow2(2*max(a_bits,b_bits)) <= 2^17 bits (batches of >= 64 2^17-bit products: batch-wide
 * kernels in the tower representation; otherwise one CTA per product, all in shared memory). */
fpm_status fpm_polymul_batch_dev(const uint64_t* d_a, size_t a_bits, size_t a_stride_words, const uint64_t* d_b,
                                 size_t b_bits, size_t b_stride_words, uint64_t* d_c, size_t c_stride_words,
                                 size_t count, void* stream);
/* The same on HOST buffers (synchronous): the batch is cut into chunks whose uploads, products and
 * downloads overlap on three streams (copy in / compute / copy out, triple-buffered device slots). */
fpm_status fpm_polymul_batch(const uint64_t* a, size_t a_bits, size_t a_stride_words, const uint64_t* b, size_t b_bits,
                             size_t b_stride_words, uint64_t* c, size_t c_stride_words, size_t count, int device);

/* karatsuba_mul (proj/include/fpmul/polymul.hpp:85-87, polymul.cpp:268-282) on host buffers: the
 * exact product by word-level carry-less multiplication (no FFT), c as for fpm_polymul.  Also what
 * fpm_polymul / fpm_polymul_dev run in FPM_FIELD_AUTO when max(a_bits, b_bits) < 4096, the
 * reference's fft_threshold_bits default (polymul.cpp:226-231, polymul.hpp:65).  It is the
 * independent cross-check of the FFT path, as in the reference. */
fpm_status fpm_karatsuba_mul(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c,
                             int device);
/* naive_mul_words_kernel (proj/include/fpmul/detail/kernels.hpp:115-118) on device buffers, except
 * that d_out[0 .. wa+wb) is overwritten (not accumulated): d_out = d_a * d_b carry-less. */
fpm_status fpm_clmul_words_dev(const uint64_t* d_a, size_t wa, const uint64_t* d_b, size_t wb, uint64_t* d_out,
                               void* stream);

/* ---- stage entry points on device buffers, field GF(2^128) ---- */

/* basis_cvt (proj/include/fpmul/basis_convert.hpp:34-35): in place on n_bits (power of two)
 * bits; bits >= content_bits must be zero (content_bits = (size_t)-1 for "all"). */
fpm_status fpm_basis_cvt_dev(uint64_t* d_w, size_t n_bits, size_t content_bits, void* stream);
/* i_basis_cvt (basis_convert.hpp:37). */
fpm_status fpm_i_basis_cvt_dev(uint64_t* d_w, size_t n_bits, void* stream);
/* encode<gf128> with make_partition_spec<gf128>(l) (encode.hpp:84-86, 40-41): d_poly holds
 * 128*2^l bits, d_ev receives 2^l elements.  l < 64. */
fpm_status fpm_encode_dev(const uint64_t* d_poly, unsigned l, uint64_t* d_ev, void* stream);
/* decode<gf128> (encode.hpp:88-91): inverse of fpm_encode_dev. */
fpm_status fpm_decode_dev(const uint64_t* d_ev, unsigned l, uint64_t* d_poly, void* stream);
/* lch_butterfly / i_lch_butterfly<gf128> with plan_butterflies(l, e_{l+64}) (butterfly.hpp:58-68). */
fpm_status fpm_butterfly_dev(uint64_t* d_ev, unsigned l, int inverse, void* stream);
/* The same for any plan_butterflies(l, base) (butterfly.cpp:32-53): base = Cantor coordinates
 * {lo, hi}; twiddle of layer i, block b = C2P((base >> i) ^ 2b).  l <= 64. */
fpm_status fpm_lch_butterfly_dev(uint64_t* d_ev, unsigned l, const uint64_t* base, int inverse, void* stream);
/* pointwise_mul<gf128> (polymul.hpp:78-80): d_out[i] = d_u[i]*d_v[i] over n elements (may alias). */
fpm_status fpm_pointwise_dev(const uint64_t* d_u, const uint64_t* d_v, uint64_t* d_out, size_t n, void* stream);

/* ---- sharded multi-GPU building blocks (one process per GPU) ----
 * Rank g of P owns elements [g*n_p/P, (g+1)*n_p/P) of every EvalVec.  Encode/decode are
 * element-local, the lower l - log2(P) butterfly layers are a sub-FFT with base ^ (g*n_p/P)
 * (fpm_lch_butterfly_dev), and only the top log2(P) layers exchange halves with a partner. */
/* encode of element columns [col0, col0+ncols) of the 128 x 2^l partition matrix in d_poly
 * (rows_live 64: rows >= 64 known zero, as for pipeline operands; else 128).  1024-aligned. */
fpm_status fpm_encode_cols_dev(const uint64_t* d_poly, unsigned l, size_t col0, size_t ncols, int rows_live,
                               uint64_t* d_ev, void* stream);
/* decode of ncols elements into a 128-row x ncols-bit slice (row pitch ncols bits). */
fpm_status fpm_decode_cols_dev(const uint64_t* d_ev, size_t ncols, uint64_t* d_slice, void* stream);
/* One exchanged butterfly layer: d_mine holds this rank's half (side 0 = the p0 block half,
 * side 1 = the p1 half), d_theirs the partner's; w (2 words, polynomial rep) is the layer's
 * twiddle for this block.  Forward: p0' = p0 + w p1, p1' = p1 + p0'; inverse undoes it. */
fpm_status fpm_bfly_pair_dev(uint64_t* d_mine, const uint64_t* d_theirs, size_t n, const uint64_t* w, int side,
                             int inverse, void* stream);
/* The same building blocks in the product pipeline's internal tower representation (tower.cuh),
 * so that each rank's coset runs the single-GPU fast path: fpm_shard_tower(l) says whether a coset
 * of 2^l elements takes it (l >= 18); encode/decode/pair as above but with tower-representation
 * elements; fpm_shard_local_product_dev multiplies two encoded, exchanged cosets (base in Cantor
 * coordinates: the partition base ^ the coset's first element): the local forward layers of both,
 * the pointwise product and the local inverse layers, result in d_eb. */
int fpm_shard_tower(unsigned l);
fpm_status fpm_encode_cols_r_dev(const uint64_t* d_poly, unsigned l, size_t col0, size_t ncols, int rows_live,
                                 uint64_t* d_ev, void* stream);
fpm_status fpm_decode_cols_r_dev(const uint64_t* d_ev, size_t ncols, uint64_t* d_slice, void* stream);
fpm_status fpm_bfly_pair_r_dev(uint64_t* d_mine, const uint64_t* d_theirs, size_t n, const uint64_t* w, int side,
                               int inverse, void* stream);
fpm_status fpm_shard_local_product_dev(uint64_t* d_ea, uint64_t* d_eb, unsigned l, const uint64_t* base,
                                       void* stream);
/* The exchanged layer with the exchange fused in (peer memory over NVLink instead of an NCCL copy):
 * d_theirs is the partner's half in the PARTNER GPU's memory (a pointer from fpm_ipc_open), read
 * directly by the kernel; the result goes to d_out, a third local buffer, so neither input is
 * overwritten while the partner may still be reading this rank's half (ping-pong buffers; one
 * barrier per layer).  tower: elements in the tower representation. */
fpm_status fpm_bfly_pair_peer_dev(const uint64_t* d_mine, const uint64_t* d_theirs, uint64_t* d_out, size_t n,
                                  const uint64_t* w, int side, int inverse, int tower, void* stream);
/* Peer-shareable device buffers: cudaMalloc + cudaIpcGetMemHandle (64-byte handle) / open a peer's
 * handle in this process (cudaIpcMemLazyEnablePeerAccess) / close / free. */
#define FPM_IPC_HANDLE_BYTES 64
/* The sharded product's conversions split over ranks instead of replicated (the
 * blocks of basis_convert.cpp's schedule, :60-67, that are independent):
 *  - fpm_load_operand_dev: dst[0 .. dst_words) <- the src_bits-bit operand, zero-padded (the padded
 *    copy run_pipeline converts, polymul.cpp:86-104);
 *  - fpm_decode_cols_split_dev: ncols elements (a rank's columns [col0, col0 + ncols)) decoded
 *    straight into the product matrix of row pitch row_bits -- rows 0..63 to d_lo, 64..127 to d_hi
 *    (either may be a peer GPU's memory): the all-gather of the columns disappears;
 *  - a 2^33-bit product's inverse conversion as its two independent 2^32-bit blocks: the upper block
 *    by fpm_i_basis_cvt_dev(d_hi, 2^32), then fpm_i_basis_cvt_block32_dev(d_lo, d_hi) (the array's
 *    top pass fused in, reading the final upper block), then fpm_top_bit_fix_dev(d_hi);
 *  - fpm_copy_dev: cudaMemcpyAsync(cudaMemcpyDefault) (peer / device copies for non-torch callers). */
fpm_status fpm_load_operand_dev(uint64_t* d_dst, size_t dst_words, const uint64_t* d_src, size_t src_bits, void* stream);
fpm_status fpm_decode_cols_split_dev(const uint64_t* d_ev, size_t ncols, size_t col0, size_t row_bits, uint64_t* d_lo,
                                     uint64_t* d_hi, int tower, void* stream);
fpm_status fpm_i_basis_cvt_block32_dev(uint64_t* d_lo, const uint64_t* d_top, void* stream);
fpm_status fpm_top_bit_fix_dev(uint64_t* d_hi, void* stream);
fpm_status fpm_copy_dev(void* d_dst, const void* d_src, size_t bytes, void* stream);
/* The sharded 2^32-bit conversion (P >= 4 ranks, build_schedule's phases
 * basis_convert.cpp:60-67, their tiling :278-327): a 2^32-bit block (an operand, or a block of the
 * 2^33-bit product) on Q = 2 or 4 ranks, each holding a full-size replica (d_w, 2^27 32-bit words) in
 * which it owns, phase by phase:
 *    FPM_DIST_WINDOW  the L1_outer windows [q wpr, (q+1) wpr) (wpr = ceil(16448 / Q); window w covers
 *                     words [32 w - 8 c, 32 w - 8 c + 32) of chunk c, a chunk = 2^19 words)
 *    FPM_DIST_CHUNK   the chunks [q 256/Q, (q+1) 256/Q)
 *    FPM_DIST_COLUMN  the words with (index mod 2048) in [q 2048/Q, (q+1) 2048/Q)
 *  - fpm_b32_regather_dev: d_w receives every 16-byte group it owns under `to` from its owner under
 *    `from` (d_srcs[0..Q): the group's replicas, peer pointers; d_srcs[q] = d_w);
 *  - fpm_b32_l1_outer_dev: L1_outer (z = x^(2^24) + x^256 over the 256 chunks) on rank q's windows,
 *    in place; beyond-window parts to d_side (2 MiB; rank Q-1's holds them all);
 *  - fpm_b32_l1_outer_fix_dev: its fix-up for chunks [e_lo, e_hi) reading d_side (rank Q-1's):
 *    forward on the chunk owners after the WINDOW -> CHUNK regather, inverse on rank 0 (all chunks);
 *  - fpm_b32_rows_dev: L1_inner + T_r (forward) / T_r^-1 + L1_inner^-1 of `rows` rows (whole chunks);
 *  - fpm_b32_cols_dev: T_d (conv over the row index) on rank q's columns;
 *  - fpm_b32_top_pass_dev / fpm_b32_top_bit_fix_dev: the 2^33-bit array's top pass on rank q's
 *    windows of the lower block, reading the upper block's window owners d_his[0..Q); then the upper
 *    block's bit 0 (d_hi0 = its rank 0) ^= its last bit (d_hi_last = its rank Q-1);
 *  - fpm_encode_cols_owners_dev / fpm_decode_cols_owners_dev: fpm_encode_cols(_r)_dev /
 *    fpm_decode_cols_split_dev with the operand / product columns at their owners (Q replicas).
 * Forward: [WINDOW] l1_outer, regather WINDOW->CHUNK, fix, rows, regather CHUNK->COLUMN, cols, encode.
 * Inverse: decode, cols, regather COLUMN->CHUNK, rows, regather CHUNK->WINDOW, l1_outer, fix (rank 0),
 * top pass, top bit fix.  Every step on one rank may only start after the group's previous step. */
#define FPM_DIST_WINDOW 0
#define FPM_DIST_CHUNK 1
#define FPM_DIST_COLUMN 2
fpm_status fpm_b32_regather_dev(uint64_t* d_w, const uint64_t* const* d_srcs, int from, int to, int q, int Q, void* stream);
fpm_status fpm_b32_l1_outer_dev(uint64_t* d_w, uint64_t* d_side, int inverse, int q, int Q, void* stream);
fpm_status fpm_b32_l1_outer_fix_dev(uint64_t* d_w, const uint64_t* d_side, int inverse, unsigned e_lo, unsigned e_hi,
                                    void* stream);
fpm_status fpm_b32_rows_dev(uint64_t* d_rows, size_t rows, int inverse, void* stream);
fpm_status fpm_b32_cols_dev(uint64_t* d_w, int inverse, int q, int Q, void* stream);
fpm_status fpm_b32_top_pass_dev(uint64_t* d_lo, const uint64_t* const* d_his, int q, int Q, void* stream);
fpm_status fpm_b32_top_bit_fix_dev(uint64_t* d_hi0, const uint64_t* d_hi_last, void* stream);
fpm_status fpm_encode_cols_owners_dev(const uint64_t* const* d_polys, int Q, unsigned l, size_t col0, size_t ncols,
                                      int rows_live, uint64_t* d_ev, int tower, void* stream);
fpm_status fpm_decode_cols_owners_dev(const uint64_t* d_ev, size_t ncols, size_t col0, size_t row_bits,
                                      const uint64_t* const* d_los, const uint64_t* const* d_his, int Q, int tower,
                                      void* stream);

fpm_status fpm_ipc_alloc(size_t bytes, void** d_ptr, uint8_t* handle);
fpm_status fpm_ipc_open(const uint8_t* handle, void** d_peer);
fpm_status fpm_ipc_close(void* d_peer);
fpm_status fpm_ipc_free(void* d_ptr);
/* Host: the twiddle C2P((base >> i) ^ 2b) of layer i, block b (butterfly.cpp:45-49); base in
 * Cantor coordinates {lo, hi}; out = {lo, hi} polynomial representation. */
fpm_status fpm_twiddle128(unsigned i, uint64_t b, const uint64_t* base, uint64_t* out);

/* ---- host-buffer stage wrappers (synchronous; same semantics as the *_dev calls) ---- */
fpm_status fpm_basis_cvt(uint64_t* w, size_t n_bits, size_t content_bits, int device);
fpm_status fpm_i_basis_cvt(uint64_t* w, size_t n_bits, int device);
fpm_status fpm_encode(const uint64_t* poly, unsigned l, uint64_t* ev, int device);
fpm_status fpm_decode(const uint64_t* ev, unsigned l, uint64_t* poly, int device);
fpm_status fpm_butterfly(uint64_t* ev, unsigned l, int inverse, int device);
fpm_status fpm_lch_butterfly(uint64_t* ev, unsigned l, const uint64_t* base, int inverse, int device);
fpm_status fpm_pointwise(const uint64_t* u, const uint64_t* v, uint64_t* out, size_t n, int device);
fpm_status fpm_gf128_mul(const uint64_t* a, const uint64_t* b, uint64_t* out, size_t n, int device);

/* Field tables as built by the library (CantorField<gf128>::basis, EncodeMatrix<gf128>::row /
 * inv_row): each 128 elements x {lo, hi}.  Host-only, no GPU needed. */
fpm_status fpm_tables128(uint64_t* cantor, uint64_t* rows, uint64_t* inv_rows);

/* ---- GF(2^64) stages (the reference's auto field; encode.hpp:84-91, butterfly.hpp:58-68,
 * polymul.hpp:78-80 instantiated for gf64, FPMUL_INSTANTIATE_*(gf64)).  Elements are one uint64
 * word (FieldElem<gf64>); the partition matrix has 64 rows of 2^l bits; l < 32 (PartitionSpec). */
fpm_status fpm_encode64_dev(const uint64_t* d_poly, unsigned l, uint64_t* d_ev, void* stream);
fpm_status fpm_decode64_dev(const uint64_t* d_ev, unsigned l, uint64_t* d_poly, void* stream);
/* base: Cantor coordinates of plan_butterflies<gf64>(l, base). */
fpm_status fpm_lch_butterfly64_dev(uint64_t* d_ev, unsigned l, uint64_t base, int inverse, void* stream);
fpm_status fpm_pointwise64_dev(const uint64_t* d_u, const uint64_t* d_v, uint64_t* d_out, size_t n, void* stream);
fpm_status fpm_encode64(const uint64_t* poly, unsigned l, uint64_t* ev, int device);
fpm_status fpm_decode64(const uint64_t* ev, unsigned l, uint64_t* poly, int device);
fpm_status fpm_lch_butterfly64(uint64_t* ev, unsigned l, uint64_t base, int inverse, int device);
fpm_status fpm_pointwise64(const uint64_t* u, const uint64_t* v, uint64_t* out, size_t n, int device);
/* CantorField<gf64>::basis, EncodeMatrix<gf64> rows / inverse rows: 64 words each (host only). */
fpm_status fpm_tables64(uint64_t* cantor, uint64_t* rows, uint64_t* inv_rows);

/* Diagnostic, not a reference interface: the tower representation the product pipeline's FFT uses
 * internally (paper_1803_11301_b200/csrc/tower.cuh) for field_degree 128 or 64 -- GF(2^m) as a
 * vector space over its subfield GF(2^8) with basis x^j t^s.  t: 2 words; to_poly / to_r: m
 * entries x 2 words (basis vector k in polynomial form / x^k in tower coordinates); tau: 8 bytes
 * (tower byte 0 of Cantor basis vectors v_1..v_7).  Host only; lets the CPU tests check the
 * construction against the oracle's field arithmetic. */
fpm_status fpm_tower_tables(int field_degree, uint64_t* t, uint64_t* to_poly, uint64_t* to_r, uint8_t* tau);

/* Fault-injection test hook, the device twin of EncodeMatrix::corrupt_for_test
 * (proj/include/fpmul/encode.hpp:70-71; used by the self-test, selftest.cpp:315-331): flips one bit
 * of the forward encode tables the kernels read on `device` (entry "row 0" of chunk 0, both fields,
 * polynomial and tower representation).  Calling it again restores them.  Not for production use:
 * every encode on the device sees the flipped table while it is active. */
fpm_status fpm_test_flip_encode_table(int device);

/* Returns the library's cached device scratch (its private stream-ordered memory pool; the
 * device's default pool is never modified) on `device` to the driver. */
fpm_status fpm_trim_pool(int device);

/* Grows the library's pool on `device` to at least `bytes` of cached scratch ahead of time.  The
 * first product (and the first product of every additional concurrent caller) otherwise pays for
 * fresh device memory inside the call -- hundreds of milliseconds for the ~5 GiB a 2^33-bit product
 * takes.  A serving process calls this once at start-up (about 5 GiB per concurrent 2^33-bit
 * caller).  No counterpart in the reference (its scratch is std::vector, polymul.cpp:78-135). */
fpm_status fpm_reserve_pool(int device, size_t bytes);

/* Number of kernel launches issued by this library on the calling thread since the last reset
 * (for the bench's gpu_launches accounting). */
uint64_t fpm_launch_count(int reset);

#ifdef __cplusplus
}
#endif

#endif /* FPMUL_B200_H_ */
