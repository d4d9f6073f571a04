// fpm_tables.h -- host-side field tables for the GF(2^128) / GF(2^64) Frobenius-partition pipelines.
//
// Product code (not the oracle): the CUDA library builds its own tables at first use, mirroring
// the reference singletons CantorField<gf128> (proj/src/cantor.cpp:103-140) and
// EncodeMatrix<gf128> (proj/src/encode.cpp:52-102).  They are uploaded once per device.
#pragma once
#include <cstddef>
#include <cstdint>

namespace fpm {

struct U128 {
  uint64_t lo = 0, hi = 0;
};

struct FieldTables {
  U128 cantor[128];    // v_i in polynomial representation (C2P rows), cantor.cpp:111-128
  U128 enc_rows[128];  // r_j = prod_{bits k of j} v_{64-k}, encode.cpp:60-66
  U128 inv_rows[128];  // rows of E^{-1}, encode.cpp:68-70
};

// Builds (once, thread-safe) and returns the tables; throws std::runtime_error on the same
// construction failures the reference reports (cantor.cpp:108-133, encode.cpp:69-70).
const FieldTables& field_tables();
// GF(2^64) (CantorField<gf64>, EncodeMatrix<gf64>): entries 0..63 used, hi words zero.
const FieldTables& field_tables64();

// Internal "tower" representation R of GF(2^128) for the product pipeline's FFT (not visible at any
// API boundary): GF(2^128) as a 16-dimensional vector space over its subfield GF(2^8) =
// span(v_0..v_7) (Cantor basis), basis e_{8j+s} = x^j t^s where t is a root of
// y^8 + y^4 + y^3 + y + 1 in GF(2^128).  Byte j of an R element holds the GF(2^8) coordinate of x^j in
// the basis 1, t, ..., t^7, so multiplying by a subfield element is 16 independent byte products
// (xtime mod 0x11B), while M8 tables work unchanged (any GF(2)-basis).
struct TowerTables {
  U128 t;             // the root t (polynomial representation)
  U128 to_poly[128];  // e_k in polynomial representation (R -> poly rows)
  U128 to_r[128];     // x^k in R coordinates (poly -> R rows)
  uint8_t tau[8];     // tau[b] = R byte 0 of v_{b+1} (b < 7): C2P(2d) for d < 128 is byte sum_b d_b tau[b]
};
const TowerTables& tower_tables();
// The same for GF(2^64) (8 coordinates, basis x^j t^s, j < 8): entries 0..63 used, hi words zero.
const TowerTables& tower_tables64();
U128 host_to_r(U128 poly);
U128 host_from_r(U128 r);

U128 host_gf128_mul(U128 a, U128 b);
U128 host_gf64_mul(U128 a, U128 b);                      // lo words only
U128 host_cantor_to_poly(const FieldTables& t, U128 c);  // bitmat.hpp:29-35
U128 host_cantor_to_poly64(const FieldTables& t, uint64_t c);

// Basis-conversion schedule (basis_convert.cpp:53-67) with the overflow-safe digit size
// (the reference loops forever for arrays of >= 2^33 bits).
struct Pass {
  size_t span;   // S (bits)
  size_t shift;  // D (bits)
};
size_t digit_size(size_t count);
void build_schedule(Pass* out, size_t* n, size_t count, size_t unit);

}  // namespace fpm
