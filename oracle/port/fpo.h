/*
 * oracle/port/fpo.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference fpmul hot path (/root/reference/proj), used by
 * tests/ and bench.py's cpu_baseline leg as the CHECKER.  It is never linked into, loaded by,
 * or called from the product (paper_1803_11301_b200/); the product fails loudly without its
 * CUDA library instead of falling back here.
 *
 * Every function cites the reference file:line it restates.  Fields: m in {16, 64, 128} with
 * the reference moduli (proj/include/fpmul/gf.hpp:95-123).  Elements are fpo_u128 {lo, hi}
 * (bit k < 64 in lo), exactly the reference u128 layout (gf.hpp:24-52).
 *
 * Pinning: tests/test_oracle.py checks this port against the reference's own known answers
 * (proj/tests/test_*.cpp) and against outputs of the real reference library compiled by
 * oracle/Makefile into oracle/_ref/ (tests/golden/ holds committed vectors from it).
 */
#ifndef FPO_H_
#define FPO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t lo, hi;
} fpo_u128;

/* --- mt19937_64 (the reference's generator, proj/src/bitpoly.cpp:19-24) --- */
typedef struct {
  uint64_t mt[312];
  int idx;
} fpo_mt64;
void fpo_mt64_seed(fpo_mt64* s, uint64_t seed);
uint64_t fpo_mt64_next(fpo_mt64* s);
/* random_bitpoly(n_bits, mt19937_64(seed)): one draw per word, tail masked. */
void fpo_random_bitpoly(size_t n_bits, uint64_t seed, uint64_t* out);

/* --- field arithmetic (gf.hpp:95-123, kernels.hpp:51-94; restated bit-serially) --- */
fpo_u128 fpo_gf_mul(unsigned m, fpo_u128 a, fpo_u128 b);
fpo_u128 fpo_gf_sqr(unsigned m, fpo_u128 a);

/* --- Cantor basis and encode matrix (cantor.cpp:103-134, encode.cpp:52-84) --- */
/* Fills v[0..m) (C2P rows).  Returns 0 on success. */
int fpo_cantor_basis(unsigned m, fpo_u128* v);
/* rows[0..m) = r_j, inv_rows[0..m) = rows of E^{-1}.  Returns 0 on success. */
int fpo_encode_matrix(unsigned m, fpo_u128* rows, fpo_u128* inv_rows);
/* C2P of Cantor coordinates c (bitmat.hpp:29-35). */
fpo_u128 fpo_cantor_to_poly(unsigned m, fpo_u128 c);

/* --- stages; m in {64, 128}; n_p = 2^l --- */
/* basis_cvt / i_basis_cvt in place on n_bits (power of two) bits (basis_convert.cpp:26-67, 337-347).
 * The digit size is computed overflow-safely; identical to the reference below 2^33. */
int fpo_basis_cvt(uint64_t* w, size_t n_bits);
int fpo_i_basis_cvt(uint64_t* w, size_t n_bits);
/* encode: a has m*n_p bits; ev gets n_p elements (encode.cpp:244-255 reference::encode). */
int fpo_encode(unsigned m, const uint64_t* a, unsigned l, fpo_u128* ev);
/* decode: inverse of encode (encode.cpp:195-220). a gets m*n_p bits. */
int fpo_decode(unsigned m, const fpo_u128* ev, unsigned l, uint64_t* a);
/* twiddle of layer i, block b for the pipeline plan base = e_{l+m/2} (butterfly.cpp:32-53). */
fpo_u128 fpo_twiddle(unsigned m, unsigned l, unsigned i, size_t b);
/* LCH butterflies on 2^l elements, forward / inverse (butterfly.cpp:108-146). */
int fpo_butterfly(unsigned m, fpo_u128* ev, unsigned l, int inverse);
void fpo_pointwise(unsigned m, const fpo_u128* u, const fpo_u128* v, fpo_u128* out, size_t n);

/* --- products --- */
/* plan_mul (polymul.cpp:187-219): out6 = {n_bits, log2_n, m, log2_m, l, n_p}; field 0=auto. */
int fpo_plan_mul(size_t a_bits, size_t b_bits, int field, uint64_t* out6);
/* Full FFT pipeline (polymul.cpp:78-135, 223-239) for field m (64 or 128), no Karatsuba bypass.
 * c must hold ceil((a_bits+b_bits-1)/64) words. */
int fpo_fft_polymul(unsigned m, const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits,
                    uint64_t* c);
/* Schoolbook carry-less product (polymul.cpp:259-266 naive_mul). */
void fpo_naive_mul(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c);

const char* fpo_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* FPO_H_ */
