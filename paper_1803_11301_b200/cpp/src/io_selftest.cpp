// io_selftest.cpp -- file I/O and the self-test suites of the fpmul API on the B200 backend.
//
// load_polynomial / store_polynomial follow the file format of proj/include/fpmul/io.hpp
// (io.cpp:23-56).  run_selftest follows proj/include/fpmul/selftest.hpp: named invariant suites,
// one log line each, failures collected in the report; the suites here exercise the GPU stages
// through the public API (GF(2^64) and GF(2^128) pipelines, basis conversion, encode/decode,
// butterflies, products), each checked against host arithmetic or an independent path.
#include <algorithm>
#include <cstdio>
#include <ostream>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/fpmul_b200.h"
#include "fpmul/basis_convert.hpp"
#include "fpmul/butterfly.hpp"
#include "fpmul/encode.hpp"
#include "fpmul/exec.hpp"
#include "fpmul/io.hpp"
#include "fpmul/polymul.hpp"
#include "fpmul/selftest.hpp"

namespace fpmul {

// ------------------------------------------------------------------ files
BitPoly load_polynomial(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("cannot open '" + path + "' for reading");
  std::vector<unsigned char> bytes;
  std::vector<unsigned char> chunk(size_t{1} << 20);
  size_t got;
  while ((got = std::fread(chunk.data(), 1, chunk.size(), f)) > 0) bytes.insert(bytes.end(), chunk.begin(), chunk.begin() + got);
  const bool failed = std::ferror(f) != 0;
  std::fclose(f);
  if (failed) throw std::runtime_error("read error on '" + path + "'");
  BitPoly p(bytes.size() * 8);
  uint64_t* w = p.word_data();
  for (size_t i = 0; i < bytes.size(); ++i) w[i >> 3] |= uint64_t{bytes[i]} << (8 * (i & 7));
  return p;
}

void store_polynomial(const std::string& path, const BitPoly& poly) {
  const size_t nbytes = (poly.max_degree_plus_one() + 7) / 8;
  std::vector<unsigned char> bytes(nbytes);
  const uint64_t* w = poly.word_data();
  for (size_t i = 0; i < nbytes; ++i) bytes[i] = static_cast<unsigned char>(w[i >> 3] >> (8 * (i & 7)));
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open '" + path + "' for writing");
  bool failed = nbytes && std::fwrite(bytes.data(), 1, nbytes, f) != nbytes;
  if (std::fclose(f) != 0) failed = true;
  if (failed) throw std::runtime_error("write error on '" + path + "'");
}

// ------------------------------------------------------------------ self test
namespace {

struct Checker {
  std::ostream& log;
  SelftestReport& report;
  void check(const std::string& name, bool ok) {
    log << (ok ? "  ok    " : "  FAIL  ") << name << "\n";
    if (!ok) {
      report.ok = false;
      report.failed_invariants.push_back(name);
    }
  }
  template <class Fn>
  void guarded(const std::string& name, Fn&& fn) {  // a thrown exception fails the invariant
    bool ok = false;
    try {
      ok = fn();
    } catch (const std::exception& e) {
      log << "  (" << name << ": " << e.what() << ")\n";
    }
    check(name, ok);
  }
};

template <class V>
V shl(V v, unsigned s) {
  return static_cast<V>(v << s);
}

template <class F>
typename F::value_type bitserial(typename F::value_type a, typename F::value_type b) {
  using V = typename F::value_type;
  V acc{};
  for (int i = static_cast<int>(F::kDegree) - 1; i >= 0; --i) {
    const bool carry = detail::test_bit(acc, F::kDegree - 1);
    acc = shl(acc, 1);
    if (carry) acc = static_cast<V>(acc ^ detail::from_low_word<V>(F::kModulusTail));
    if (detail::test_bit(b, static_cast<unsigned>(i))) acc = static_cast<V>(acc ^ a);
  }
  return acc;
}

template <class F>
typename F::value_type rand_value(std::mt19937_64& rng) {
  if constexpr (F::kDegree == 128) return u128{rng(), rng()};
  else return static_cast<typename F::value_type>(rng());
}

// Product over GF(2)[x] of small operands, bit-serial (the schoolbook oracle of test_polymul).
BitPoly schoolbook(const BitPoly& a, const BitPoly& b) {
  if (!a.bit_length() || !b.bit_length()) return BitPoly{};
  BitPoly c(a.bit_length() + b.bit_length() - 1);
  for (size_t i = 0; i < a.bit_length(); ++i)
    if (a.bit(i))
      for (size_t j = 0; j < b.bit_length(); ++j)
        if (b.bit(j)) c.flip_bit(i + j);
  return c;
}

BitPoly square(const BitPoly& a) {  // a(x)^2 = a(x^2) over GF(2)
  BitPoly s(a.bit_length() ? 2 * a.bit_length() - 1 : 0);
  for (size_t i = 0; i < a.bit_length(); ++i)
    if (a.bit(i)) s.set_bit(2 * i);
  return s;
}

template <class F>
void field_suite(Checker& c, std::mt19937_64& rng, const std::string& t, size_t samples) {
  // device pointwise products vs host bit-serial multiplication
  EvalVec<F> u(samples), v(samples);
  for (size_t i = 0; i < samples; ++i) { u[i].v = rand_value<F>(rng); v[i].v = rand_value<F>(rng); }
  c.guarded("gf." + t + ".device mul vs bit-serial", [&] {
    const auto p = pointwise_mul<F>(u, v);
    for (size_t i = 0; i < samples; ++i)
      if (p[i].v != bitserial<F>(u[i].v, v[i].v)) return false;
    return true;
  });
  c.guarded("cantor." + t + ".basis recurrence v_i^2+v_i=v_{i-1}", [&] {
    const auto& fld = CantorField<F>::get();
    for (unsigned i = 1; i < F::kDegree; ++i) {
      const auto vi = fld.basis(i);
      if (gf_add(gf_sqr(vi), vi) != fld.basis(i - 1)) return false;
    }
    return true;
  });
}

template <class F>
void butterfly_suite(Checker& c, std::mt19937_64& rng, const std::string& t, unsigned max_l) {
  using V = typename F::value_type;
  c.guarded("butterfly." + t + ".matches direct evaluation; inverse round trip", [&] {
    for (unsigned l = 1; l <= max_l; l += 3) {
      CantorVec<F> base{rand_value<F>(rng)};
      base.bits = static_cast<V>(detail::value_shr(base.bits, l));
      base.bits = shl(base.bits, l);  // low l bits clear: a coset of the subspace
      const auto plan = plan_butterflies<F>(l, base);
      EvalVec<F> coeffs(size_t{1} << l);
      for (auto& e : coeffs) e.v = rand_value<F>(rng);
      EvalVec<F> w = coeffs;
      lch_butterfly<F>(std::span<FieldElem<F>>(w), plan);
      for (size_t idx = 0; idx < w.size(); idx += 1 + w.size() / 16) {
        const CantorVec<F> pt{static_cast<V>(base.bits ^ detail::from_low_word<V>(idx))};
        if (direct_eval<F>(std::span<const FieldElem<F>>(coeffs), pt) != w[idx]) return false;
      }
      i_lch_butterfly<F>(std::span<FieldElem<F>>(w), plan);
      if (w != coeffs) return false;
    }
    return true;
  });
}

template <class F>
void encode_suite(Checker& c, std::mt19937_64& rng, const std::string& t, bool corrupt, unsigned max_l) {
  const auto& mat = EncodeMatrix<F>::get();
  c.guarded("encode." + t + ".rows r_0=1, r_1=v_{m/2}", [&] {
    const auto& fld = CantorField<F>::get();
    return mat.row(0) == FieldElem<F>{detail::from_low_word<typename F::value_type>(1)} &&
           mat.row(1) == fld.basis(F::kDegree / 2);
  });
  // The named round-trip invariant (selftest.cpp:315-331); with fault injection it runs while the
  // DEVICE encode tables have one bit flipped (fpm_test_flip_encode_table, the twin of
  // EncodeMatrix::corrupt_for_test), restored afterwards.
  struct DeviceFault {
    bool on;
    explicit DeviceFault(bool o) : on(o) {
      if (on && fpm_test_flip_encode_table(current_device()) != FPM_OK) throw std::runtime_error(fpm_last_error());
    }
    ~DeviceFault() { if (on) fpm_test_flip_encode_table(current_device()); }
  };
  c.guarded("encode." + t + ".encode/decode round-trip", [&] {
    const DeviceFault fault(corrupt);
    for (unsigned l : {0u, 1u, 4u, 6u, max_l}) {
      const auto spec = make_partition_spec<F>(l);
      const BitPoly a = random_bitpoly(size_t{F::kDegree} * spec.n_p, rng);
      const EvalVec<F> ev = encode<F>(a, spec, mat);
      if (decode<F>(std::span<const FieldElem<F>>(ev), spec, mat) != a) return false;
    }
    return true;
  });
}

}  // namespace

SelftestReport run_selftest(const SelftestOptions& opts, std::ostream& log) {
  SelftestReport report;
  Checker c{log, report};
  std::mt19937_64 rng(opts.seed);
  const bool full = opts.level == SelftestLevel::kFull;
  log << "fpmul selftest (B200 backend, " << (full ? "full" : "quick") << ", seed " << opts.seed << ")\n";

  field_suite<gf64>(c, rng, "gf64", full ? 4096 : 512);
  field_suite<gf128>(c, rng, "gf128", full ? 4096 : 512);

  c.guarded("basis.n4 example (0,1,0,1)->(0,0,1,1)", [&] {
    BitPoly p(4);
    p.set_bit(1);
    p.set_bit(3);
    basis_cvt(p);
    return !p.bit(0) && !p.bit(1) && p.bit(2) && p.bit(3);
  });
  c.guarded("basis.round trip and linearity", [&] {
    for (size_t lg : {size_t{8}, size_t{17}, full ? size_t{26} : size_t{21}}) {
      const size_t n = size_t{1} << lg;
      const BitPoly a = random_bitpoly(n, rng), b = random_bitpoly(n, rng);
      BitPoly x = a, y = b, s = a;
      s ^= b;
      basis_cvt(x);
      basis_cvt(y);
      basis_cvt(s);
      BitPoly xy = x;
      xy ^= y;
      if (xy != s) return false;
      i_basis_cvt(x);
      if (x != a) return false;
    }
    return true;
  });

  butterfly_suite<gf64>(c, rng, "gf64", full ? 16 : 10);
  butterfly_suite<gf128>(c, rng, "gf128", full ? 16 : 10);
  encode_suite<gf64>(c, rng, "gf64", opts.corrupt_encode_matrix, full ? 15 : 10);
  encode_suite<gf128>(c, rng, "gf128", opts.corrupt_encode_matrix, full ? 15 : 10);

  c.guarded("polymul.plan examples and size-bound rejection", [&] {
    const MulPlan p = plan_mul(size_t{1} << 20, size_t{1} << 20);
    bool rejected = false;
    try {
      (void)plan_mul(size_t{1} << 40, 8, FieldChoice::kGF64);
    } catch (const std::invalid_argument&) {
      rejected = true;
    }
    return p.n_bits == (size_t{1} << 21) && p.field_degree == 64 && p.l == 15 && rejected;
  });
  c.guarded("polymul.identity and monomial shift", [&] {
    BitPoly one(1);
    one.set_bit(0);
    const BitPoly b = random_bitpoly(50000, rng);
    BitPoly xa(1001), xb(4097);
    xa.set_bit(1000);
    xb.set_bit(4096);
    const BitPoly p = fp_polymul(xa, xb);
    return fp_polymul(one, b) == b && p.max_degree_plus_one() == 1000 + 4096 + 1;
  });
  c.guarded("polymul.fp_polymul vs schoolbook", [&] {
    MulOptions fft;  // short inputs: auto mode takes karatsuba_mul, kGF128 forces the FFT pipeline
    fft.field = FieldChoice::kGF128;
    for (int k = 0; k < (full ? 12 : 4); ++k) {
      const BitPoly a = random_bitpoly(1 + rng() % 3000, rng), b = random_bitpoly(1 + rng() % 3000, rng);
      const BitPoly want = schoolbook(a, b);
      if (fp_polymul(a, b) != want || fp_polymul(a, b, fft) != want) return false;
    }
    return true;
  });
  c.guarded("polymul.FFT pipeline vs karatsuba_mul (independent GPU paths)", [&] {
    for (size_t lg : {size_t{14}, full ? size_t{20} : size_t{17}}) {
      const BitPoly a = random_bitpoly((size_t{1} << lg) + 5, rng), b = random_bitpoly(size_t{1} << lg, rng);
      if (fp_polymul(a, b) != karatsuba_mul(a, b)) return false;
    }
    return true;
  });
  c.guarded("polymul.GF(2^64) and GF(2^128) pipelines agree", [&] {
    for (size_t lg : {size_t{18}, full ? size_t{26} : size_t{22}}) {
      const BitPoly a = random_bitpoly((size_t{1} << lg) - 7, rng), b = random_bitpoly(size_t{1} << lg, rng);
      MulOptions o64, o128;
      o64.field = FieldChoice::kGF64;
      o128.field = FieldChoice::kGF128;
      if (fp_polymul(a, b, o64) != fp_polymul(a, b, o128)) return false;
    }
    return true;
  });
  c.guarded("polymul.Frobenius identity C(a^2)=C(a)^2", [&] {
    const BitPoly a = random_bitpoly(size_t{1} << (full ? 20 : 16), rng);
    const BitPoly b = random_bitpoly((size_t{1} << (full ? 20 : 16)) + 3, rng);
    return fp_polymul(square(a), square(b)) == square(fp_polymul(a, b));
  });
  log << (report.ok ? "all invariants hold\n" : "invariant failures\n");
  return report;
}

}  // namespace fpmul
