// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (checker / CPU baseline, never the product).
//
// A C-ABI shim over the UNMODIFIED reference library (/root/reference/proj, compiled from its own
// sources by oracle/Makefile into oracle/_ref/).  It lets the Python tests and bench.py's
// cpu_baseline / --impl reference arm call the reference's own code path:
//   fp_polymul            proj/src/polymul.cpp:223-239
//   basis_cvt / i_basis_cvt proj/src/basis_convert.cpp:337-347
//   encode / decode        proj/src/encode.cpp:165-220
//   lch_butterfly / i_lch_butterfly proj/src/butterfly.cpp:55-85
//   pointwise_mul          proj/src/polymul.cpp:241-257
//   random_bitpoly         proj/src/bitpoly.cpp:19-24
// Only tests/, __graft_entry__.smoke() and bench.py may load the resulting library.
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "fpmul/basis_convert.hpp"
#include "fpmul/bitpoly.hpp"
#include "fpmul/butterfly.hpp"
#include "fpmul/cantor.hpp"
#include "fpmul/encode.hpp"
#include "fpmul/gf.hpp"
#include "fpmul/polymul.hpp"

using namespace fpmul;

namespace {
thread_local std::string g_err;

BitPoly make_poly(const uint64_t* w, size_t bits) {
  BitPoly p(bits);
  if (bits) std::memcpy(p.word_data(), w, p.word_count() * 8);
  p.resize_bits(bits);
  return p;
}
void store_poly(const BitPoly& p, uint64_t* out, size_t words) {
  std::memset(out, 0, words * 8);
  std::memcpy(out, p.word_data(), std::min(words, p.word_count()) * 8);
}
ExecPolicy pol(int parallel) { return parallel ? ExecPolicy::kParallel : ExecPolicy::kSerial; }

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
EvalVec<gf128> load_ev(const uint64_t* w, size_t n) {
  EvalVec<gf128> v(n);
  for (size_t i = 0; i < n; ++i) v[i].v = u128{w[2 * i + 1], w[2 * i]};
  return v;
}
void store_ev(const EvalVec<gf128>& v, uint64_t* w) {
  for (size_t i = 0; i < v.size(); ++i) {
    w[2 * i] = v[i].v.lo;
    w[2 * i + 1] = v[i].v.hi;
  }
}
EvalVec<gf64> load_ev64(const uint64_t* w, size_t n) {
  EvalVec<gf64> v(n);
  for (size_t i = 0; i < n; ++i) v[i].v = w[i];
  return v;
}
void store_ev64(const EvalVec<gf64>& v, uint64_t* w) {
  for (size_t i = 0; i < v.size(); ++i) w[i] = v[i].v;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void ref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

// field: 0 auto, 64, 128.  stage_seconds: optional double[7].
int ref_polymul(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c,
                int field, int parallel, double* stage_seconds) {
  return guard([&] {
    MulOptions o;
    o.field = field == 64 ? FieldChoice::kGF64 : field == 128 ? FieldChoice::kGF128 : FieldChoice::kAuto;
    o.policy = pol(parallel);
    StageSeconds st;
    if (stage_seconds) o.stage_seconds = &st;
    BitPoly r = fp_polymul(make_poly(a, a_bits), make_poly(b, b_bits), o);
    const size_t out_bits = a_bits && b_bits ? a_bits + b_bits - 1 : 0;
    store_poly(r, c, (out_bits + 63) / 64);
    if (stage_seconds) {
      double v[7] = {st.basiscvt, st.encode, st.butterfly, st.pointwise, st.ibutterfly, st.decode, st.ibasiscvt};
      std::memcpy(stage_seconds, v, sizeof v);
    }
  });
}

int ref_karatsuba(const uint64_t* a, size_t a_bits, const uint64_t* b, size_t b_bits, uint64_t* c) {
  return guard([&] {
    BitPoly r = karatsuba_mul(make_poly(a, a_bits), make_poly(b, b_bits));
    const size_t out_bits = a_bits && b_bits ? a_bits + b_bits - 1 : 0;
    store_poly(r, c, (out_bits + 63) / 64);
  });
}

int ref_plan_mul(size_t a_bits, size_t b_bits, int field, uint64_t* out6) {
  return guard([&] {
    MulPlan p = plan_mul(a_bits, b_bits,
                         field == 64 ? FieldChoice::kGF64 : field == 128 ? FieldChoice::kGF128 : FieldChoice::kAuto);
    out6[0] = p.n_bits; out6[1] = p.log2_n; out6[2] = p.field_degree;
    out6[3] = p.log2_field_degree; out6[4] = p.l; out6[5] = p.n_p;
  });
}

void ref_random_bitpoly(size_t n_bits, uint64_t seed, uint64_t* out) {
  std::mt19937_64 rng(seed);
  BitPoly p = random_bitpoly(n_bits, rng);
  std::memcpy(out, p.word_data(), p.word_count() * 8);
}

int ref_basis_cvt(uint64_t* w, size_t n_bits, size_t content_bits, int parallel) {
  return guard([&] {
    BitPoly p = make_poly(w, n_bits);
    basis_cvt(p, pol(parallel), content_bits);
    store_poly(p, w, (n_bits + 63) / 64);
  });
}
int ref_i_basis_cvt(uint64_t* w, size_t n_bits, int parallel) {
  return guard([&] {
    BitPoly p = make_poly(w, n_bits);
    i_basis_cvt(p, pol(parallel));
    store_poly(p, w, (n_bits + 63) / 64);
  });
}
int ref_basis_cvt_bits(uint64_t* w, size_t n_bits, int inverse) {
  return guard([&] {
    BitPoly p = make_poly(w, n_bits);
    if (inverse) reference::i_basis_cvt(p); else reference::basis_cvt(p);
    store_poly(p, w, (n_bits + 63) / 64);
  });
}

// gf128 stage APIs; an EvalVec is n_p x {lo, hi}.
int ref_encode128(const uint64_t* w, unsigned l, uint64_t* ev, int parallel) {
  return guard([&] {
    const auto spec = make_partition_spec<gf128>(l);
    BitPoly p = make_poly(w, size_t{128} << l);
    store_ev(encode<gf128>(p, spec, EncodeMatrix<gf128>::get(), pol(parallel)), ev);
  });
}
int ref_decode128(const uint64_t* ev, unsigned l, uint64_t* w, int parallel) {
  return guard([&] {
    const auto spec = make_partition_spec<gf128>(l);
    auto v = load_ev(ev, size_t{1} << l);
    BitPoly p = decode<gf128>(std::span<const FieldElem<gf128>>(v), spec, EncodeMatrix<gf128>::get(), pol(parallel));
    store_poly(p, w, (size_t{128} << l) / 64);
  });
}
int ref_butterfly128(uint64_t* ev, unsigned l, int inverse, int parallel) {
  return guard([&] {
    const auto spec = make_partition_spec<gf128>(l);
    const auto plan = plan_butterflies<gf128>(l, spec.base);
    auto v = load_ev(ev, size_t{1} << l);
    if (inverse) i_lch_butterfly<gf128>(std::span<FieldElem<gf128>>(v), plan, pol(parallel));
    else lch_butterfly<gf128>(std::span<FieldElem<gf128>>(v), plan, pol(parallel));
    store_ev(v, ev);
  });
}
// lch_butterfly / i_lch_butterfly<gf128> with plan_butterflies(l, base) for an arbitrary base
// (Cantor coordinates {lo, hi}) -- butterfly.cpp:32-85.
int ref_butterfly128_base(uint64_t* ev, unsigned l, uint64_t base_lo, uint64_t base_hi, int inverse) {
  return guard([&] {
    const auto plan = plan_butterflies<gf128>(l, CantorVec<gf128>{u128{base_hi, base_lo}});
    auto v = load_ev(ev, size_t{1} << l);
    if (inverse) i_lch_butterfly<gf128>(std::span<FieldElem<gf128>>(v), plan, ExecPolicy::kSerial);
    else lch_butterfly<gf128>(std::span<FieldElem<gf128>>(v), plan, ExecPolicy::kSerial);
    store_ev(v, ev);
  });
}
int ref_pointwise128(const uint64_t* u, const uint64_t* v, uint64_t* out, size_t n) {
  return guard([&] {
    auto a = load_ev(u, n), b = load_ev(v, n);
    store_ev(pointwise_mul<gf128>(a, b, ExecPolicy::kSerial), out);
  });
}
void ref_gf128_mul(const uint64_t* a, const uint64_t* b, uint64_t* out) {
  u128 r = gf128::mul(u128{a[1], a[0]}, u128{b[1], b[0]});
  out[0] = r.lo; out[1] = r.hi;
}
// Table dumps for pinning: cantor basis v_0..v_127, encode rows, inverse rows, twiddles of a plan.
void ref_tables128(uint64_t* cantor, uint64_t* rows, uint64_t* inv_rows) {
  const auto& f = CantorField<gf128>::get();
  const auto& m = EncodeMatrix<gf128>::get();
  for (unsigned i = 0; i < 128; ++i) {
    cantor[2 * i] = f.basis(i).v.lo; cantor[2 * i + 1] = f.basis(i).v.hi;
    rows[2 * i] = m.row(i).v.lo; rows[2 * i + 1] = m.row(i).v.hi;
    inv_rows[2 * i] = m.inv_row(i).v.lo; inv_rows[2 * i + 1] = m.inv_row(i).v.hi;
  }
}
// gf64 stage APIs (the reference's auto field); an EvalVec<gf64> is n_p x uint64.
int ref_encode64(const uint64_t* w, unsigned l, uint64_t* ev) {
  return guard([&] {
    const auto spec = make_partition_spec<gf64>(l);
    BitPoly p = make_poly(w, size_t{64} << l);
    store_ev64(encode<gf64>(p, spec, EncodeMatrix<gf64>::get(), ExecPolicy::kParallel), ev);
  });
}
int ref_decode64(const uint64_t* ev, unsigned l, uint64_t* w) {
  return guard([&] {
    const auto spec = make_partition_spec<gf64>(l);
    auto v = load_ev64(ev, (size_t)1 << l);
    BitPoly p = decode<gf64>(std::span<const FieldElem<gf64>>(v), spec, EncodeMatrix<gf64>::get(), ExecPolicy::kParallel);
    store_poly(p, w, ((size_t{64} << l) + 63) / 64);
  });
}
int ref_butterfly64(uint64_t* ev, unsigned l, uint64_t base, int inverse) {
  return guard([&] {
    const auto plan = plan_butterflies<gf64>(l, CantorVec<gf64>{base});
    auto v = load_ev64(ev, (size_t)1 << l);
    if (inverse) i_lch_butterfly<gf64>(std::span<FieldElem<gf64>>(v), plan, ExecPolicy::kParallel);
    else lch_butterfly<gf64>(std::span<FieldElem<gf64>>(v), plan, ExecPolicy::kParallel);
    store_ev64(v, ev);
  });
}
int ref_pointwise64(const uint64_t* u, const uint64_t* v, uint64_t* out, size_t n) {
  return guard([&] {
    auto a = load_ev64(u, n), b = load_ev64(v, n);
    store_ev64(pointwise_mul<gf64>(a, b, ExecPolicy::kSerial), out);
  });
}
void ref_tables64(uint64_t* cantor, uint64_t* rows, uint64_t* inv_rows) {
  const auto& f = CantorField<gf64>::get();
  const auto& m = EncodeMatrix<gf64>::get();
  for (unsigned i = 0; i < 64; ++i) {
    cantor[i] = f.basis(i).v;
    rows[i] = m.row(i).v;
    inv_rows[i] = m.inv_row(i).v;
  }
}
int ref_twiddles128(unsigned l, uint64_t* out) {
  return guard([&] {
    const auto spec = make_partition_spec<gf128>(l);
    const auto plan = plan_butterflies<gf128>(l, spec.base);
    for (size_t i = 0; i < plan.mults.size(); ++i) { out[2 * i] = plan.mults[i].lo; out[2 * i + 1] = plan.mults[i].hi; }
  });
}
}  // extern "C"
