// fpm_tables.cpp -- host construction of the GF(2^128) / GF(2^64) Cantor bases and encode matrices.
// Restates proj/src/cantor.cpp:103-134 and proj/src/encode.cpp:52-70 (init-time only).
#include "fpm_tables.h"

#include <mutex>
#include <stdexcept>

namespace fpm {
namespace {

inline bool bit(U128 v, unsigned i) { return i < 64 ? (v.lo >> i) & 1 : (v.hi >> (i - 64)) & 1; }
inline U128 unit(unsigned i) {
  U128 r;
  if (i < 64) r.lo = uint64_t{1} << i; else r.hi = uint64_t{1} << (i - 64);
  return r;
}
inline U128 x(U128 a, U128 b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }
inline bool nz(U128 a) { return a.lo | a.hi; }
inline bool eq(U128 a, U128 b) { return a.lo == b.lo && a.hi == b.hi; }

U128 row_mul(U128 v, const U128* rows, unsigned m = 128) {
  U128 acc;
  for (unsigned j = 0; j < m; ++j)
    if (bit(v, j)) acc = x(acc, rows[j]);
  return acc;
}

// x * rows = target over GF(2) (row-echelon; bitmat.hpp:79-111).
bool solve(const U128* rows, U128 target, U128* out, unsigned m) {
  U128 ech[128], tag[128];
  unsigned lead[128], ne = 0;
  for (unsigned i = 0; i < m; ++i) {
    U128 r = rows[i], t = unit(i);
    for (unsigned j = 0; j < ne; ++j)
      if (bit(r, lead[j])) { r = x(r, ech[j]); t = x(t, tag[j]); }
    if (nz(r)) {
      unsigned ld = 0;
      while (!bit(r, ld)) ++ld;
      ech[ne] = r; tag[ne] = t; lead[ne] = ld; ++ne;
    }
  }
  U128 acc = target, sol;
  for (unsigned j = 0; j < ne; ++j)
    if (bit(acc, lead[j])) { acc = x(acc, ech[j]); sol = x(sol, tag[j]); }
  if (nz(acc)) return false;
  *out = sol;
  return true;
}

bool invert(const U128* rows, U128* inv_out, unsigned m) {  // bitmat.hpp:55-74
  U128 a[128], inv[128];
  for (unsigned i = 0; i < m; ++i) { a[i] = rows[i]; inv[i] = unit(i); }
  for (unsigned col = 0; col < m; ++col) {
    unsigned piv = col;
    while (piv < m && !bit(a[piv], col)) ++piv;
    if (piv == m) return false;
    std::swap(a[col], a[piv]);
    std::swap(inv[col], inv[piv]);
    for (unsigned r = 0; r < m; ++r)
      if (r != col && bit(a[r], col)) { a[r] = x(a[r], a[col]); inv[r] = x(inv[r], inv[col]); }
  }
  for (unsigned i = 0; i < m; ++i) inv_out[i] = inv[i];
  return true;
}

// Generic over the field degree m (128: gf128, 64: gf64; cantor.cpp and encode.cpp are templates).
void build(FieldTables& t, unsigned m) {
  auto mul = [m](U128 a, U128 b) { return m == 128 ? host_gf128_mul(a, b) : host_gf64_mul(a, b); };
  // Artin-Schreier map y -> y^2 + y, rows in polynomial representation.
  U128 artin[128];
  for (unsigned k = 0; k < m; ++k) artin[k] = x(mul(unit(k), unit(k)), unit(k));
  t.cantor[0] = unit(0);
  for (unsigned i = 1; i < m; ++i) {
    U128 y;
    if (!solve(artin, t.cantor[i - 1], &y, m))
      throw std::runtime_error("CantorField: Artin-Schreier equation has no solution (wrong modulus?)");
    y.lo &= ~uint64_t{1};  // of the roots {y, y+1} keep the one with bit 0 clear
    if (!eq(x(mul(y, y), y), t.cantor[i - 1]))
      throw std::runtime_error("CantorField: basis recurrence check failed");
    t.cantor[i] = y;
  }
  U128 probe[128];
  if (!invert(t.cantor, probe, m)) throw std::runtime_error("CantorField: basis-change matrix not invertible");
  const unsigned logm = m == 128 ? 7 : 6;
  for (unsigned j = 0; j < m; ++j) {  // r_j = prod over bits k of j of v_{m/2-k} (encode.cpp:60-66)
    U128 r = unit(0);
    for (unsigned k = 0; k < logm; ++k)
      if ((j >> k) & 1) r = mul(r, t.cantor[m / 2 - k]);
    t.enc_rows[j] = r;
  }
  if (!invert(t.enc_rows, t.inv_rows, m))
    throw std::runtime_error("EncodeMatrix: matrix is singular (field construction bug)");
}

}  // namespace

U128 host_gf128_mul(U128 a, U128 b) {
  // bit-serial, high bit first, modulo x^128 + x^7 + x^2 + x + 1 (gf.hpp:115-123)
  U128 acc;
  for (int i = 127; i >= 0; --i) {
    const uint64_t carry = acc.hi >> 63;
    acc.hi = (acc.hi << 1) | (acc.lo >> 63);
    acc.lo = (acc.lo << 1) ^ (carry ? 0x87u : 0u);
    if (bit(b, (unsigned)i)) acc = x(acc, a);
  }
  return acc;
}

U128 host_gf64_mul(U128 a, U128 b) {
  // bit-serial modulo x^64 + x^4 + x^3 + x + 1 (gf.hpp:105-113); only the lo words are used
  uint64_t acc = 0;
  for (int i = 63; i >= 0; --i) {
    const uint64_t carry = acc >> 63;
    acc = (acc << 1) ^ (carry ? 0x1Bu : 0u);
    if ((b.lo >> i) & 1) acc ^= a.lo;
  }
  U128 r;
  r.lo = acc;
  return r;
}

U128 host_cantor_to_poly(const FieldTables& t, U128 c) { return row_mul(c, t.cantor); }
U128 host_cantor_to_poly64(const FieldTables& t, uint64_t c) {
  U128 v;
  v.lo = c;
  return row_mul(v, t.cantor, 64);
}

const FieldTables& field_tables() {
  static FieldTables tables;
  static std::once_flag once;
  std::call_once(once, [] { build(tables, 128); });
  return tables;
}

const FieldTables& field_tables64() {
  static FieldTables tables;
  static std::once_flag once;
  std::call_once(once, [] { build(tables, 64); });
  return tables;
}

namespace {
void build_tower(TowerTables& tt, unsigned m) {
  const FieldTables& f = m == 128 ? field_tables() : field_tables64();
  auto mul = [m](U128 a, U128 b) { return m == 128 ? host_gf128_mul(a, b) : host_gf64_mul(a, b); };
  auto pw = [&](U128 a, int e) {
    U128 r = unit(0);
    for (int k = 0; k < e; ++k) r = mul(r, a);
    return r;
  };
  bool found = false;
  for (unsigned v = 2; v < 256 && !found; ++v) {  // GF(2^8) = span(v_0..v_7) (Cantor subfield property)
    U128 e;
    for (unsigned b = 0; b < 8; ++b)
      if (v >> b & 1) e = x(e, f.cantor[b]);
    const U128 r = x(x(x(pw(e, 8), pw(e, 4)), x(pw(e, 3), e)), unit(0));  // e^8 + e^4 + e^3 + e + 1
    if (!nz(r)) { tt.t = e; found = true; }
  }
  if (!found) throw std::runtime_error("tower: no root of y^8+y^4+y^3+y+1 in span(v_0..v_7)");
  U128 ts[8];
  ts[0] = unit(0);
  for (int s = 1; s < 8; ++s) ts[s] = mul(ts[s - 1], tt.t);
  U128 xj = unit(0);
  for (unsigned j = 0; j < m / 8; ++j) {
    for (int s = 0; s < 8; ++s) tt.to_poly[8 * j + s] = mul(xj, ts[s]);
    xj = mul(xj, unit(1));
  }
  if (!invert(tt.to_poly, tt.to_r, m)) throw std::runtime_error("tower: x^j t^s is not a basis");
  for (int b = 0; b < 8; ++b) {
    const U128 r = row_mul(f.cantor[b < 7 ? b + 1 : 0], tt.to_r, m);
    if (r.hi || (r.lo >> 8)) throw std::runtime_error("tower: Cantor subfield element outside GF(2^8)");
    tt.tau[b] = b < 7 ? (uint8_t)r.lo : 0;
  }
}
}  // namespace

const TowerTables& tower_tables() {
  static TowerTables tables;
  static std::once_flag once;
  std::call_once(once, [] { build_tower(tables, 128); });
  return tables;
}
const TowerTables& tower_tables64() {
  static TowerTables tables;
  static std::once_flag once;
  std::call_once(once, [] { build_tower(tables, 64); });
  return tables;
}
U128 host_to_r(U128 poly) { return row_mul(poly, tower_tables().to_r); }
U128 host_from_r(U128 r) { return row_mul(r, tower_tables().to_poly); }

size_t digit_size(size_t count) {
  size_t t = 2;
  while (t <= (count / 2) / t) t *= t;
  return t;
}

void build_schedule(Pass* out, size_t* n, size_t count, size_t unit) {
  if (count <= 2) return;
  const size_t t = digit_size(count);
  for (size_t s = count; s >= 2 * t; s /= 2) out[(*n)++] = Pass{s * unit, (s / 2 - s / (2 * t)) * unit};
  build_schedule(out, n, count / t, unit * t);
  build_schedule(out, n, t, unit);
}

}  // namespace fpm
