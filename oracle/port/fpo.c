/*
 * oracle/port/fpo.c -- TEST INFRASTRUCTURE ONLY (see fpo.h).  Plain-C restatement of the
 * reference fpmul hot path; every block cites the reference file:line it follows.
 */
#include "fpo.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* fpo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ mt19937_64 */
/* std::mt19937_64 as used by random_bitpoly (proj/src/bitpoly.cpp:19-24). */
void fpo_mt64_seed(fpo_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

uint64_t fpo_mt64_next(fpo_mt64* s) {
  static const uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & kUpper) | (s->mt[(i + 1) % 312] & kLower);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void fpo_random_bitpoly(size_t n_bits, uint64_t seed, uint64_t* out) {
  fpo_mt64 s;
  fpo_mt64_seed(&s, seed);
  const size_t words = (n_bits + 63) / 64;
  for (size_t w = 0; w < words; ++w) out[w] = fpo_mt64_next(&s);
  if (n_bits % 64) out[words - 1] &= (UINT64_C(1) << (n_bits % 64)) - 1;
}

/* ------------------------------------------------------------------ field */
static uint64_t modulus_tail(unsigned m) {
  /* gf.hpp:95-123: x^16+x^5+x^3+x^2+1, x^64+x^4+x^3+x+1, x^128+x^7+x^2+x+1 */
  return m == 16 ? 0x2D : m == 64 ? 0x1B : 0x87;
}
static int test_bit(fpo_u128 v, unsigned i) { return i < 64 ? (int)((v.lo >> i) & 1) : (int)((v.hi >> (i - 64)) & 1); }
static fpo_u128 unit_bit(unsigned i) {
  fpo_u128 r = {0, 0};
  if (i < 64) r.lo = UINT64_C(1) << i; else r.hi = UINT64_C(1) << (i - 64);
  return r;
}
static fpo_u128 x128(fpo_u128 a, fpo_u128 b) { fpo_u128 r = {a.lo ^ b.lo, a.hi ^ b.hi}; return r; }
static int nz(fpo_u128 a) { return (a.lo | a.hi) != 0; }
static int eq(fpo_u128 a, fpo_u128 b) { return a.lo == b.lo && a.hi == b.hi; }

/* Modular product, high bit first: the bit-serial form of the reference's field multiply
 * (gf.hpp FieldOps; tests/test_support.hpp:43-56 pins the same definition). */
fpo_u128 fpo_gf_mul(unsigned m, fpo_u128 a, fpo_u128 b) {
  const uint64_t tail = modulus_tail(m);
  fpo_u128 acc = {0, 0};
  for (int i = (int)m - 1; i >= 0; --i) {
    const int carry = test_bit(acc, m - 1);
    acc.hi = (acc.hi << 1) | (acc.lo >> 63);
    acc.lo <<= 1;
    if (m < 128) { /* clear bit m */
      if (m < 64) acc.lo &= (UINT64_C(1) << m) - 1;
      else if (m == 64) acc.hi = 0;
    }
    if (carry) acc.lo ^= tail;
    if (test_bit(b, (unsigned)i)) acc = x128(acc, a);
  }
  return acc;
}
fpo_u128 fpo_gf_sqr(unsigned m, fpo_u128 a) { return fpo_gf_mul(m, a, a); }

/* ------------------------------------------------------------------ GF(2) matrices */
/* Row-echelon solve of x*rows = target (bitmat.hpp:79-111): returns 0 if solvable. */
static int solve_rows(const fpo_u128* rows, unsigned m, fpo_u128 target, fpo_u128* x_out) {
  fpo_u128 ech[128], tag[128];
  unsigned lead[128], ne = 0;
  for (unsigned i = 0; i < m; ++i) {
    fpo_u128 r = rows[i], t = unit_bit(i);
    for (unsigned j = 0; j < ne; ++j)
      if (test_bit(r, lead[j])) { r = x128(r, ech[j]); t = x128(t, tag[j]); }
    if (nz(r)) {
      unsigned ld = 0;
      while (!test_bit(r, ld)) ++ld;
      /* keep echelon rows reduced on the new lead so later reductions stay valid */
      ech[ne] = r; tag[ne] = t; lead[ne] = ld; ++ne;
    }
  }
  fpo_u128 acc = target, x = {0, 0};
  for (unsigned j = 0; j < ne; ++j)
    if (test_bit(acc, lead[j])) { acc = x128(acc, ech[j]); x = x128(x, tag[j]); }
  if (nz(acc)) return 1;
  *x_out = x;
  return 0;
}

/* Gauss-Jordan inverse in the row convention (bitmat.hpp:55-74). */
static int invert_rows(const fpo_u128* rows, unsigned m, fpo_u128* inv_out) {
  fpo_u128 a[128], inv[128];
  for (unsigned i = 0; i < m; ++i) { a[i] = rows[i]; inv[i] = unit_bit(i); }
  for (unsigned col = 0; col < m; ++col) {
    unsigned piv = col;
    while (piv < m && !test_bit(a[piv], col)) ++piv;
    if (piv == m) return 1;
    fpo_u128 t = a[col]; a[col] = a[piv]; a[piv] = t;
    t = inv[col]; inv[col] = inv[piv]; inv[piv] = t;
    for (unsigned r = 0; r < m; ++r)
      if (r != col && test_bit(a[r], col)) { a[r] = x128(a[r], a[col]); inv[r] = x128(inv[r], inv[col]); }
  }
  memcpy(inv_out, inv, m * sizeof(fpo_u128));
  return 0;
}

static fpo_u128 row_mul(fpo_u128 x, const fpo_u128* rows, unsigned m) {
  fpo_u128 acc = {0, 0};
  for (unsigned j = 0; j < m; ++j)
    if (test_bit(x, j)) acc = x128(acc, rows[j]);
  return acc;
}

/* ------------------------------------------------------------------ Cantor basis */
/* CantorField ctor (cantor.cpp:103-134): v_0 = 1; v_i solves y^2 + y = v_{i-1}; of the two
 * roots {y, y+1} keep the one with bit 0 clear. */
int fpo_cantor_basis(unsigned m, fpo_u128* v) {
  fpo_u128 artin[128];
  for (unsigned k = 0; k < m; ++k) {
    const fpo_u128 e = unit_bit(k);
    artin[k] = x128(fpo_gf_sqr(m, e), e);
  }
  v[0] = unit_bit(0);
  for (unsigned i = 1; i < m; ++i) {
    fpo_u128 y;
    if (solve_rows(artin, m, v[i - 1], &y)) return fail(2, "cantor: Artin-Schreier equation unsolvable");
    y.lo &= ~UINT64_C(1);
    if (!eq(x128(fpo_gf_sqr(m, y), y), v[i - 1])) return fail(2, "cantor: recurrence check failed");
    v[i] = y;
  }
  return 0;
}

static const fpo_u128* cantor_cached(unsigned m) {
  static fpo_u128 v16[128], v64[128], v128[128];
  static int have16, have64, have128;
  if (m == 16) { if (!have16) { fpo_cantor_basis(16, v16); have16 = 1; } return v16; }
  if (m == 64) { if (!have64) { fpo_cantor_basis(64, v64); have64 = 1; } return v64; }
  if (!have128) { fpo_cantor_basis(128, v128); have128 = 1; }
  return v128;
}

fpo_u128 fpo_cantor_to_poly(unsigned m, fpo_u128 c) { return row_mul(c, cantor_cached(m), m); }

/* EncodeMatrix ctor (encode.cpp:52-70): r_j = prod over bits k of j of v_{m/2-k}. */
int fpo_encode_matrix(unsigned m, fpo_u128* rows, fpo_u128* inv_rows) {
  const fpo_u128* v = cantor_cached(m);
  unsigned logm = m == 16 ? 4 : m == 64 ? 6 : 7;
  for (unsigned j = 0; j < m; ++j) {
    fpo_u128 r = unit_bit(0);
    for (unsigned k = 0; k < logm; ++k)
      if ((j >> k) & 1) r = fpo_gf_mul(m, r, v[m / 2 - k]);
    rows[j] = r;
  }
  if (invert_rows(rows, m, inv_rows)) return fail(2, "encode matrix singular");
  return 0;
}

/* ------------------------------------------------------------------ bit helpers */
static uint64_t get_bits(const uint64_t* w, size_t nbits_total, size_t pos, unsigned len) {
  if (!len || pos >= nbits_total) return 0;
  const size_t iw = pos / 64;
  const unsigned ib = (unsigned)(pos % 64);
  uint64_t v = w[iw] >> ib;
  if (ib && (iw + 1) * 64 < nbits_total) v |= w[iw + 1] << (64 - ib);
  if (len < 64) v &= (UINT64_C(1) << len) - 1;
  return v;
}
static void xor_bits(uint64_t* w, size_t pos, uint64_t val, unsigned len) {
  if (!len) return;
  if (len < 64) val &= (UINT64_C(1) << len) - 1;
  const size_t iw = pos / 64;
  const unsigned ib = (unsigned)(pos % 64);
  w[iw] ^= val << ib;
  if (ib && ib + len > 64) w[iw + 1] ^= val >> (64 - ib);
}
static int bit_at(const uint64_t* w, size_t k) { return (int)((w[k / 64] >> (k % 64)) & 1); }

/* ------------------------------------------------------------------ basis conversion */
/* Schedule: basis_convert.cpp:53-67.  digit_size made overflow-safe. */
typedef struct { size_t S, D; } pass_t;
static size_t digit_size(size_t count) {
  size_t t = 2;
  while (t <= (count / 2) / t) t *= t;
  return t;
}
static void build_schedule(pass_t* out, size_t* n, size_t count, size_t unit) {
  if (count <= 2) return;
  const size_t t = digit_size(count);
  for (size_t s = count; s >= 2 * t; s /= 2) {
    out[*n].S = s * unit;
    out[*n].D = (s / 2 - s / (2 * t)) * unit;
    ++*n;
  }
  build_schedule(out, n, count / t, unit * t);
  build_schedule(out, n, t, unit);
}

/* One fold pass on every aligned S-span, from a pre-pass copy (basis_convert.cpp:34-46):
 *   forward  y[q] = x[q] ^ x[q+D] ^ (q+2D < S ? x[q+2D] : 0)
 *   inverse  x[q] = y[q] ^ y[q+D]        for q in [S/2-D, S-D). */
static void apply_pass(uint64_t* w, const uint64_t* src, size_t nbits, pass_t p, int inverse) {
  const size_t S = p.S, D = p.D, half = S / 2;
  for (size_t base = 0; base < nbits; base += S) {
    for (size_t q = half - D; q < S - D;) {
      const unsigned k = (unsigned)((S - D - q) < 64 ? (S - D - q) : 64);
      uint64_t v = get_bits(src, nbits, base + q + D, k);
      if (!inverse && q + 2 * D < S) {
        const size_t lim = S - 2 * D - q;
        const unsigned k2 = (unsigned)(lim < k ? lim : k);
        v ^= get_bits(src, nbits, base + q + 2 * D, k2);
      }
      xor_bits(w, base + q, v, k);
      q += k;
    }
  }
}

static int convert(uint64_t* w, size_t n_bits, int inverse) {
  if (n_bits == 0 || (n_bits & (n_bits - 1))) return fail(1, "basis_cvt: length must be a power of two");
  pass_t sched[512];
  size_t np = 0;
  build_schedule(sched, &np, n_bits, 1);
  const size_t words = (n_bits + 63) / 64;
  uint64_t* copy = (uint64_t*)malloc(words * 8);
  if (!copy) return fail(3, "oom");
  for (size_t k = 0; k < np; ++k) {
    const pass_t p = sched[inverse ? np - 1 - k : k];
    memcpy(copy, w, words * 8);
    apply_pass(w, copy, n_bits, p, inverse);
  }
  free(copy);
  return 0;
}
int fpo_basis_cvt(uint64_t* w, size_t n_bits) { return convert(w, n_bits, 0); }
int fpo_i_basis_cvt(uint64_t* w, size_t n_bits) { return convert(w, n_bits, 1); }

/* ------------------------------------------------------------------ encode / decode */
int fpo_encode(unsigned m, const uint64_t* a, unsigned l, fpo_u128* ev) {
  if (l >= m / 2) return fail(1, "PartitionSpec: l must satisfy l < m/2");
  fpo_u128 rows[128], inv[128];
  if (fpo_encode_matrix(m, rows, inv)) return 2;
  const size_t n_p = (size_t)1 << l;
  for (size_t i = 0; i < n_p; ++i) { /* reference::encode, encode.cpp:244-255 */
    fpo_u128 acc = {0, 0};
    for (unsigned j = 0; j < m; ++j)
      if (bit_at(a, j * n_p + i)) acc = x128(acc, rows[j]);
    ev[i] = acc;
  }
  return 0;
}

int fpo_decode(unsigned m, const fpo_u128* ev, unsigned l, uint64_t* a) {
  if (l >= m / 2) return fail(1, "PartitionSpec: l must satisfy l < m/2");
  fpo_u128 rows[128], inv[128];
  if (fpo_encode_matrix(m, rows, inv)) return 2;
  const size_t n_p = (size_t)1 << l;
  memset(a, 0, ((size_t)m * n_p + 63) / 64 * 8);
  for (size_t i = 0; i < n_p; ++i) { /* decode, encode.cpp:195-220 */
    const fpo_u128 y = row_mul(ev[i], inv, m);
    for (unsigned j = 0; j < m; ++j)
      if (test_bit(y, j)) a[(j * n_p + i) / 64] |= UINT64_C(1) << ((j * n_p + i) % 64);
  }
  return 0;
}

/* ------------------------------------------------------------------ butterflies */
/* w(i, b) = C2P((base >> i) ^ 2b) with base = e_{l+m/2} (butterfly.cpp:45-49, encode.cpp:47). */
fpo_u128 fpo_twiddle(unsigned m, unsigned l, unsigned i, size_t b) {
  const unsigned top = l + m / 2 - i; /* (e_{l+m/2} >> i) = e_{l+m/2-i} */
  fpo_u128 c = unit_bit(top);
  c.lo ^= (uint64_t)b << 1;
  return fpo_cantor_to_poly(m, c);
}

int fpo_butterfly(unsigned m, fpo_u128* v, unsigned l, int inverse) {
  if (l >= m / 2) return fail(1, "PartitionSpec: l must satisfy l < m/2");
  const size_t n = (size_t)1 << l;
  if (!inverse) { /* reference::run_layers, butterfly.cpp:108-123 */
    for (int i = (int)l - 1; i >= 0; --i) {
      const size_t half = (size_t)1 << i;
      for (size_t b = 0; b < (n >> (i + 1)); ++b) {
        const fpo_u128 w = fpo_twiddle(m, l, (unsigned)i, b);
        fpo_u128* p = v + (b << (i + 1));
        for (size_t j = 0; j < half; ++j) {
          p[j] = x128(p[j], fpo_gf_mul(m, w, p[j + half]));
          p[j + half] = x128(p[j + half], p[j]);
        }
      }
    }
  } else { /* reference::i_lch_butterfly, butterfly.cpp:131-146 */
    for (unsigned i = 0; i < l; ++i) {
      const size_t half = (size_t)1 << i;
      for (size_t b = 0; b < (n >> (i + 1)); ++b) {
        const fpo_u128 w = fpo_twiddle(m, l, i, b);
        fpo_u128* p = v + (b << (i + 1));
        for (size_t j = 0; j < half; ++j) {
          p[j + half] = x128(p[j + half], p[j]);
          p[j] = x128(p[j], fpo_gf_mul(m, w, p[j + half]));
        }
      }
    }
  }
  return 0;
}

void fpo_pointwise(unsigned m, const fpo_u128* u, const fpo_u128* v, fpo_u128* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = fpo_gf_mul(m, u[i], v[i]); /* kernels_impl.hpp:116-123 */
}

/* ------------------------------------------------------------------ products */
static unsigned log2_ceil(size_t n) { unsigned l = 0; while (((size_t)1 << l) < n) ++l; return l; }
static size_t next_pow2(size_t n) { size_t p = 1; while (p < n) p <<= 1; return p; }
static int field_supports(unsigned m, size_t n_bits) { /* polymul.cpp:45-49 */
  if (n_bits < m) return 0;
  const unsigned l = log2_ceil(n_bits) - log2_ceil(m);
  return l < m / 2 && l + 1 < m / 2;
}

int fpo_plan_mul(size_t a_bits, size_t b_bits, int field, uint64_t* out6) { /* polymul.cpp:187-219 */
  if (!a_bits || !b_bits) return fail(1, "plan_mul: input lengths must be positive");
  const size_t mx = a_bits > b_bits ? a_bits : b_bits;
  if (mx > ((size_t)1 << 62)) return fail(1, "plan_mul: input length out of range");
  size_t n = next_pow2(2 * mx);
  unsigned m = field == 64 ? 64 : field == 128 ? 128 : (field_supports(64, n < 64 ? 64 : n) ? 64 : 128);
  if (n < m) n = m;
  if (!field_supports(m, n)) return fail(1, "plan_mul: length exceeds the field's supported bound");
  out6[0] = n; out6[1] = log2_ceil(n); out6[2] = m; out6[3] = m == 64 ? 6 : 7;
  out6[4] = out6[1] - out6[3]; out6[5] = (uint64_t)1 << out6[4];
  return 0;
}

static int transform_input(unsigned m, const uint64_t* p, size_t bits, size_t n, unsigned l, fpo_u128* ev) {
  const size_t words = n / 64;
  uint64_t* pad = (uint64_t*)calloc(words, 8);
  if (!pad) return fail(3, "oom");
  memcpy(pad, p, (bits + 63) / 64 * 8);
  if (bits % 64) pad[bits / 64] &= (UINT64_C(1) << (bits % 64)) - 1;
  int rc = fpo_basis_cvt(pad, n);
  if (!rc) rc = fpo_encode(m, pad, l, ev);
  if (!rc) rc = fpo_butterfly(m, ev, l, 0);
  free(pad);
  return rc;
}

int fpo_fft_polymul(unsigned m, const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits,
                    uint64_t* c) { /* run_pipeline, polymul.cpp:78-135; trim :237 */
  if (!a_bits || !b_bits) return 0;
  uint64_t plan[6];
  int rc = fpo_plan_mul(a_bits, b_bits, (int)m, plan);
  if (rc) return rc;
  const size_t n = plan[0], n_p = plan[5];
  const unsigned l = (unsigned)plan[4];
  fpo_u128* ea = (fpo_u128*)malloc(n_p * sizeof(fpo_u128));
  fpo_u128* eb = (fpo_u128*)malloc(n_p * sizeof(fpo_u128));
  uint64_t* out = (uint64_t*)calloc(n / 64, 8);
  if (!ea || !eb || !out) { free(ea); free(eb); free(out); return fail(3, "oom"); }
  rc = transform_input(m, a, a_bits, n, l, ea);
  if (!rc) rc = transform_input(m, b, b_bits, n, l, eb);
  if (!rc) {
    fpo_pointwise(m, ea, eb, ea, n_p);
    rc = fpo_butterfly(m, ea, l, 1);
  }
  if (!rc) rc = fpo_decode(m, ea, l, out);
  if (!rc) rc = fpo_i_basis_cvt(out, n);
  if (!rc) {
    const size_t ob = a_bits + b_bits - 1, ow = (ob + 63) / 64;
    memcpy(c, out, ow * 8);
    if (ob % 64) c[ow - 1] &= (UINT64_C(1) << (ob % 64)) - 1;
  }
  free(ea); free(eb); free(out);
  return rc;
}

static void clmul64(uint64_t a, uint64_t b, uint64_t* lo, uint64_t* hi) { /* gf.cpp:33-41 */
  uint64_t l = 0, h = 0;
  for (unsigned i = 0; i < 64; ++i) {
    const uint64_t mask = ~(((b >> i) & 1) - 1);
    l ^= (a << i) & mask;
    if (i) h ^= (a >> (64 - i)) & mask;
  }
  *lo = l; *hi = h;
}

void fpo_naive_mul(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c) {
  if (!a_bits || !b_bits) return;
  const size_t wa = (a_bits + 63) / 64, wb = (b_bits + 63) / 64, ob = a_bits + b_bits - 1;
  uint64_t* out = (uint64_t*)calloc(wa + wb + 1, 8);
  for (size_t i = 0; i < wa; ++i) { /* naive_mul_words_kernel, kernels_impl.hpp:125-137 */
    uint64_t x = a[i];
    if (i == wa - 1 && a_bits % 64) x &= (UINT64_C(1) << (a_bits % 64)) - 1;
    if (!x) continue;
    for (size_t j = 0; j < wb; ++j) {
      uint64_t y = b[j];
      if (j == wb - 1 && b_bits % 64) y &= (UINT64_C(1) << (b_bits % 64)) - 1;
      uint64_t lo, hi;
      clmul64(x, y, &lo, &hi);
      out[i + j] ^= lo;
      out[i + j + 1] ^= hi;
    }
  }
  const size_t ow = (ob + 63) / 64;
  memcpy(c, out, ow * 8);
  if (ob % 64) c[ow - 1] &= (UINT64_C(1) << (ob % 64)) - 1;
  free(out);
}
