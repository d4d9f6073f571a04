// tests/cpp/test_api.cpp -- the reference's C++ API (namespace fpmul) exercised through the B200
// backend's mirror headers (paper_1803_11301_b200/cpp/include) and libfpmul_b200.so, with checks
// restated from the reference's own tests (proj/tests/test_*.cpp) so callers of the reference
// compile and behave unchanged.  `test_api cpu` runs only the host-side parts (no GPU needed).
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "fpmul/basis_convert.hpp"
#include "fpmul/bitpoly.hpp"
#include "fpmul/butterfly.hpp"
#include "fpmul/cantor.hpp"
#include "fpmul/encode.hpp"
#include "fpmul/gf.hpp"
#include "fpmul/polymul.hpp"

using namespace fpmul;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                            \
  } while (0)
template <class E, class Fn>
static void check_throws(Fn&& fn, const char* what) {
  ++g_checks;
  try {
    fn();
    ++g_fail;
    std::printf("FAIL: no exception from %s\n", what);
  } catch (const E&) {
  } catch (...) {
    ++g_fail;
    std::printf("FAIL: wrong exception type from %s\n", what);
  }
}

template <class F>
static typename F::value_type bitserial_mul(typename F::value_type a, typename F::value_type b) {
  using V = typename F::value_type;
  V acc{};
  for (unsigned i = F::kDegree; i-- > 0;) {
    const bool carry = detail::test_bit(acc, F::kDegree - 1);
    acc = static_cast<V>(acc << 1);
    if (carry) acc ^= detail::from_low_word<V>(F::kModulusTail);
    if (detail::test_bit(b, i)) acc ^= a;
  }
  return acc;
}

static BitPoly schoolbook(const BitPoly& a, const BitPoly& b) {
  if (!a.bit_length() || !b.bit_length()) return BitPoly{};
  BitPoly c(a.bit_length() + b.bit_length() - 1);
  for (size_t i = 0; i < a.bit_length(); ++i)
    if (a.bit(i))
      for (size_t w = 0; w < b.word_count(); ++w) {
        const uint64_t x = b.word_data()[w];
        if (!x) continue;
        const size_t pos = i + 64 * w;
        uint64_t* cw = c.word_data();
        cw[pos / 64] ^= x << (pos % 64);
        if (pos % 64 && pos / 64 + 1 < c.word_count()) cw[pos / 64 + 1] ^= x >> (64 - pos % 64);
      }
  c.resize_bits(c.bit_length());
  return c;
}

static void host_tests() {
  // test_gf.cpp:67-69
  CHECK(gf64::mul(uint64_t{2}, uint64_t{1} << 63) == 0x1B);
  std::mt19937_64 rng(13);
  for (int i = 0; i < 2000; ++i) {
    const u128 a{rng(), rng()}, b{rng(), rng()};
    CHECK(gf128::mul(a, b) == bitserial_mul<gf128>(a, b));
    const uint64_t x = rng(), y = rng();
    CHECK(gf64::mul(x, y) == bitserial_mul<gf64>(x, y));
    const uint16_t p = (uint16_t)rng(), q = (uint16_t)rng();
    CHECK(gf16::mul(p, q) == bitserial_mul<gf16>(p, q));
  }
  // test_cantor.cpp:78-85 (leopard table for m = 16)
  const uint16_t leopard[16] = {0x0001, 0xACCA, 0x3C0E, 0x163E, 0xC582, 0xED2E, 0x914C, 0x4012,
                                0x6C98, 0x10D8, 0x6A72, 0xB900, 0xFDB8, 0xFB34, 0xFF38, 0x991E};
  for (unsigned i = 0; i < 16; ++i) CHECK(CantorField<gf16>::get().basis(i).v == leopard[i]);
  const auto& f128 = CantorField<gf128>::get();
  for (unsigned i = 1; i < 128; ++i) CHECK((gf128::sqr(f128.basis(i).v) ^ f128.basis(i).v) == f128.basis(i - 1).v);
  // test_encode.cpp:28-42
  const auto& mat = EncodeMatrix<gf128>::get();
  CHECK(mat.row(0).v == u128{1});
  CHECK(mat.row(1) == f128.basis(64));
  CHECK(mat.row(3) == gf_mul(f128.basis(64), f128.basis(63)));
  for (int t = 0; t < 100; ++t) {
    const u128 x{rng(), rng()};
    FieldElem<gf128> naive{};
    for (unsigned j = 0; j < 128; ++j)
      if (detail::test_bit(x, j)) naive = gf_add(naive, mat.row(j));
    CHECK(mat.m4r_mul(x) == naive);
    CHECK(mat.m4r_mul_inv(mat.m4r_mul(x).v).v == x);
  }
  // transpose64x64 involution and single-bit definition (test_encode.cpp:70-96)
  uint64_t m[64], o[64];
  for (int t = 0; t < 100; ++t) {
    for (auto& w : m) w = 0;
    const unsigned r = rng() % 64, c = rng() % 64;
    m[r] = uint64_t{1} << c;
    transpose64x64(m);
    for (unsigned j = 0; j < 64; ++j) CHECK(m[j] == (j == c ? uint64_t{1} << r : 0));
    for (unsigned j = 0; j < 64; ++j) o[j] = m[j] = rng();
    transpose64x64(m);
    transpose64x64(m);
    CHECK(std::memcmp(m, o, sizeof m) == 0);
  }
  // argument errors match the reference's exception types
  check_throws<std::invalid_argument>([] { make_partition_spec<gf128>(64); }, "make_partition_spec(64)");
  check_throws<std::invalid_argument>([] { plan_mul(0, 8); }, "plan_mul(0, 8)");
  check_throws<std::invalid_argument>([] { frobenius_order_of_basis(0); }, "frobenius_order_of_basis(0)");
  // plan_mul (test_polymul.cpp:30-48)
  const MulPlan p = plan_mul(size_t{1} << 20, size_t{1} << 20);
  CHECK(p.n_bits == size_t{1} << 21 && p.field_degree == 64 && p.l == 15 && p.n_p == size_t{1} << 15);
  CHECK(plan_mul(size_t{1} << 39, size_t{1} << 39).field_degree == 128);
  // Frobenius identity along Horner evaluation
  for (int t = 0; t < 50; ++t) {
    const BitPoly a = random_bitpoly(1 + rng() % 300, rng);
    CHECK(frobenius_value_check<gf128>(a, FieldElem<gf128>{u128{rng(), rng()}}));
  }
}

static void gpu_tests() {
  std::mt19937_64 rng(7);
  // basis_cvt n=4 truth table (test_basis_convert.cpp:29-63)
  for (unsigned bits = 0; bits < 16; ++bits) {
    BitPoly f(4);
    for (unsigned k = 0; k < 4; ++k) f.set_bit(k, (bits >> k) & 1);
    const bool f0 = f.bit(0), f1 = f.bit(1), f2 = f.bit(2), f3 = f.bit(3);
    basis_cvt(f);
    CHECK(f.bit(0) == f0 && f.bit(1) == (f1 ^ f2 ^ f3) && f.bit(2) == (f2 ^ f3) && f.bit(3) == f3);
  }
  for (unsigned lg = 1; lg <= 20; ++lg) {
    const BitPoly f = random_bitpoly(size_t{1} << lg, rng);
    BitPoly g = f;
    basis_cvt(g);
    i_basis_cvt(g);
    CHECK(g == f);
  }
  check_throws<std::invalid_argument>([] { BitPoly bad(96); basis_cvt(bad); }, "basis_cvt(96 bits)");
  // encode == the scalar definition, decode inverts it (test_encode.cpp:98-122)
  const auto& mat = EncodeMatrix<gf128>::get();
  for (unsigned l : {0u, 5u, 7u, 11u}) {
    const auto spec = make_partition_spec<gf128>(l);
    const BitPoly a = random_bitpoly(128 * spec.n_p, rng);
    const auto ev = encode<gf128>(a, spec, mat);
    bool ok = true;
    for (size_t i = 0; i < spec.n_p; ++i) {
      FieldElem<gf128> acc{};
      for (unsigned j = 0; j < 128; ++j)
        if (a.bit(j * spec.n_p + i)) acc = gf_add(acc, mat.row(j));
      ok &= ev[i] == acc;
    }
    CHECK(ok);
    CHECK(decode<gf128>(std::span<const FieldElem<gf128>>(ev), spec, mat) == a);
  }
  check_throws<std::invalid_argument>([&] { encode<gf128>(BitPoly(100), make_partition_spec<gf128>(3), mat); },
                                      "encode(bad length)");
  // gf64 (the auto field): encode == row combination, decode inverts (encode_suite<gf64>, selftest.cpp:485)
  for (unsigned l : {0u, 5u, 11u}) {
    const auto& m64 = EncodeMatrix<gf64>::get();
    const auto spec = make_partition_spec<gf64>(l);
    const BitPoly a = random_bitpoly(64 * spec.n_p, rng);
    const auto ev = encode<gf64>(a, spec, m64);
    bool ok64 = true;
    for (size_t i = 0; i < spec.n_p; ++i) {
      FieldElem<gf64> acc{};
      for (unsigned j = 0; j < 64; ++j)
        if (a.bit(j * spec.n_p + i)) acc = gf_add(acc, m64.row(j));
      ok64 &= ev[i] == acc;
    }
    CHECK(ok64);
    CHECK(decode<gf64>(std::span<const FieldElem<gf64>>(ev), spec, m64) == a);
  }
  check_throws<std::invalid_argument>([&] {
    encode<gf16>(BitPoly(16 * 8), make_partition_spec<gf16>(3), EncodeMatrix<gf16>::get());
  }, "encode<gf16>");
  // butterflies == direct evaluation for random bases (test_butterfly.cpp:28-47, 104-108)
  for (unsigned l = 0; l <= 8; ++l) {
    const CantorVec<gf128> base{u128{rng(), rng()}};
    const auto plan = plan_butterflies<gf128>(l, base);
    EvalVec<gf128> coeffs(size_t{1} << l);
    for (auto& e : coeffs) e.v = u128{rng(), rng()};
    EvalVec<gf128> v = coeffs;
    lch_butterfly<gf128>(std::span<FieldElem<gf128>>(v), plan);
    bool ok = true;
    for (size_t idx = 0; idx < v.size(); ++idx) {
      const CantorVec<gf128> pt{static_cast<u128>(base.bits ^ u128{idx})};
      ok &= direct_eval<gf128>(std::span<const FieldElem<gf128>>(coeffs), pt) == v[idx];
    }
    CHECK(ok);
    i_lch_butterfly<gf128>(std::span<FieldElem<gf128>>(v), plan);
    CHECK(v == coeffs);
  }
  {  // l = 14 (exercises the shared-memory tile + M4R layer kernels) against plan.mults
    const unsigned l = 14;
    const CantorVec<gf128> base{u128{rng(), rng()}};
    const auto plan = plan_butterflies<gf128>(l, base);
    EvalVec<gf128> v(size_t{1} << l), ref;
    for (auto& e : v) e.v = u128{rng(), rng()};
    ref = v;
    for (unsigned i = l; i-- > 0;) {  // reference::run_layers (butterfly.cpp:108-123)
      const size_t half = size_t{1} << i;
      for (size_t b = 0; b < ref.size() >> (i + 1); ++b) {
        const auto w = plan.multiplier(i, b);
        FieldElem<gf128>* q = ref.data() + (b << (i + 1));
        for (size_t j = 0; j < half; ++j) {
          q[j] = gf_add(q[j], gf_mul(w, q[j + half]));
          q[j + half] = gf_add(q[j + half], q[j]);
        }
      }
    }
    lch_butterfly<gf128>(std::span<FieldElem<gf128>>(v), plan);
    CHECK(v == ref);
  }
  // gf64 butterflies == direct evaluation, inverse restores (butterfly_suite<gf64>)
  for (unsigned l : {3u, 9u, 12u}) {
    const CantorVec<gf64> base{rng() & ~((uint64_t{1} << l) - 1)};
    const auto plan = plan_butterflies<gf64>(l, base);
    EvalVec<gf64> coeffs(size_t{1} << l);
    for (auto& e : coeffs) e.v = rng();
    EvalVec<gf64> v = coeffs;
    lch_butterfly<gf64>(std::span<FieldElem<gf64>>(v), plan);
    bool ok64 = true;
    for (size_t idx = 0; idx < v.size(); idx += 1 + v.size() / 64) {
      const CantorVec<gf64> pt{base.bits ^ idx};
      ok64 &= direct_eval<gf64>(std::span<const FieldElem<gf64>>(coeffs), pt) == v[idx];
    }
    CHECK(ok64);
    i_lch_butterfly<gf64>(std::span<FieldElem<gf64>>(v), plan);
    CHECK(v == coeffs);
  }
  {
    EvalVec<gf64> u64(257), w64(257);
    for (size_t i = 0; i < u64.size(); ++i) { u64[i].v = rng(); w64[i].v = rng(); }
    const auto p64 = pointwise_mul<gf64>(u64, w64);
    bool ok64 = true;
    for (size_t i = 0; i < u64.size(); ++i) ok64 &= p64[i].v == gf64::mul(u64[i].v, w64[i].v);
    CHECK(ok64);
  }
  // pointwise (test_polymul.cpp:136-152)
  EvalVec<gf128> u(300), w(300);
  for (size_t i = 0; i < u.size(); ++i) { u[i].v = u128{rng(), rng()}; w[i].v = u128{rng(), rng()}; }
  const auto pw = pointwise_mul<gf128>(u, w);
  bool ok = true;
  for (size_t i = 0; i < u.size(); ++i) ok &= pw[i].v == gf128::mul(u[i].v, w[i].v);
  CHECK(ok);
  check_throws<std::invalid_argument>([&] { pointwise_mul<gf128>(u, EvalVec<gf128>(5)); }, "pointwise_mul mismatch");
  // fp_polymul (test_polymul.cpp:50-126)
  BitPoly one(1);
  one.set_bit(0);
  const BitPoly b = random_bitpoly(50000, rng);
  CHECK(fp_polymul(one, b) == b);
  BitPoly xa(1001), xb(4097);
  xa.set_bit(1000);
  xb.set_bit(4096);
  const BitPoly prod = fp_polymul(xa, xb);
  CHECK(prod.bit_length() == 1001 + 4097 - 1 && prod.max_degree_plus_one() == 1000 + 4096 + 1);
  CHECK(fp_polymul(BitPoly{}, b).bit_length() == 0);
  for (int t = 0; t < 30; ++t) {
    const size_t la = 1 + rng() % 70000, lb = 1 + rng() % 70000;
    const BitPoly a = random_bitpoly(la, rng), c = random_bitpoly(lb, rng);
    MulOptions o;
    o.field = t % 3 == 0 ? FieldChoice::kGF128 : t % 3 == 1 ? FieldChoice::kGF64 : FieldChoice::kAuto;
    StageSeconds st;
    o.stage_seconds = &st;
    CHECK(fp_polymul(a, c, o) == schoolbook(a, c));
  }
  check_throws<std::invalid_argument>([&] {  // beyond GF(2^64)'s bound (field_supports, polymul.cpp:45-49)
    MulOptions o;
    o.field = FieldChoice::kGF64;
    (void)plan_mul(size_t{1} << 40, 8, o.field);
  }, "plan_mul(kGF64, 2^40)");
}

// fp_polymul sharded over P logical ranks on GPU 0 (MulOptions::devices = {0, ..., 0}: the
// multi-GPU path, fpm_polymul_multi, with peer pointers that happen to be local): bit-exact against
// karatsuba_mul (an independent algorithm) on both coset regimes of the sharded FFT, and against the
// single-GPU pipeline at a size whose cosets take the tower fast path.
void multi_gpu_tests() {
  std::mt19937_64 rng(77);
  for (int P : {2, 4, 8}) {
    MulOptions o;
    o.devices.assign(P, 0);
    const BitPoly a = random_bitpoly((size_t{1} << 19) + 321, rng), b = random_bitpoly(size_t{1} << 19, rng);
    CHECK(fp_polymul(a, b, o) == karatsuba_mul(a, b));
    const BitPoly x = random_bitpoly(size_t{1} << 25, rng), y = random_bitpoly((size_t{1} << 25) - 4099, rng);
    MulOptions single;
    single.field = FieldChoice::kGF128;
    CHECK(fp_polymul(x, y, o) == fp_polymul(x, y, single));
  }
  check_throws<std::invalid_argument>([&] {
    MulOptions o;
    o.devices = {0, 0, 0};  // not a power of two
    (void)fp_polymul(random_bitpoly(size_t{1} << 20, rng), random_bitpoly(size_t{1} << 20, rng), o);
  }, "fpm_polymul_multi: 3 ranks");
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::string(argv[1]) == "cpu";
  const bool multi_only = argc > 1 && std::string(argv[1]) == "multi";
  if (multi_only) {
    multi_gpu_tests();
    std::printf("%s: %d checks, %d failures\n", g_fail ? "FAIL" : "PASS", g_checks, g_fail);
    return g_fail ? 1 : 0;
  }
  host_tests();
  if (!cpu_only) {
    gpu_tests();
    multi_gpu_tests();
  }
  std::printf("%s: %d checks, %d failures\n", g_fail ? "FAIL" : "PASS", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
