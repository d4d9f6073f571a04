// fpmul_api.cpp -- the reference's C++ API (namespace fpmul, /root/reference/proj/include/fpmul)
// implemented over the B200 C-ABI (include/fpmul_b200.h).  Bulk work -- basis conversion,
// encode/decode, butterflies, pointwise products, whole products -- runs on the GPU for the
// north-star field GF(2^128); scalar field arithmetic and init-time tables stay on the host, as
// in the reference.  GF(2^128) and GF(2^64) stages run on the GPU; the GF(2^16) test field's stage
// calls are not built on this backend and throw std::invalid_argument.  Errors follow the reference:
// std::invalid_argument for shape/length problems, std::runtime_error otherwise.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/fpmul_b200.h"
#include "fpmul/basis_convert.hpp"
#include "fpmul/bitpoly.hpp"
#include "fpmul/butterfly.hpp"
#include "fpmul/cantor.hpp"
#include "fpmul/encode.hpp"
#include "fpmul/gf.hpp"
#include "fpmul/polymul.hpp"

namespace fpmul {
namespace {

std::atomic<int> g_device{0};

void check(fpm_status st) {
  if (st == FPM_OK) return;
  const std::string msg = fpm_last_error();
  if (st == FPM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

[[noreturn]] void not_built(const char* what) {
  throw std::invalid_argument(std::string(what) + ": the GF(2^16) test field is not built on the B200 backend");
}

template <class F>
constexpr bool is128() {
  return F::kDegree == 128;
}
template <class F>
constexpr bool is64() {
  return F::kDegree == 64;
}

using detail::test_bit;
using detail::unit_bit;

u128 clmul(uint64_t a, uint64_t b) { return detail::clmul64_portable(a, b); }

}  // namespace

void set_device(int device) { g_device.store(device); }
int current_device() { return g_device.load(); }

// ------------------------------------------------------------------ BitPoly
size_t BitPoly::max_degree_plus_one() const {
  for (size_t w = w_.size(); w > 0; --w)
    if (w_[w - 1]) return (w - 1) * 64 + (64 - __builtin_clzll(w_[w - 1]));
  return 0;
}

BitPoly& BitPoly::operator^=(const BitPoly& other) {
  if (other.bits_ > bits_) resize_bits(other.bits_);
  for (size_t w = 0; w < other.w_.size(); ++w) w_[w] ^= other.w_[w];
  return *this;
}

bool operator==(const BitPoly& a, const BitPoly& b) {
  const BitPoly& longer = a.w_.size() >= b.w_.size() ? a : b;
  const BitPoly& shorter = a.w_.size() >= b.w_.size() ? b : a;
  for (size_t w = 0; w < shorter.w_.size(); ++w)
    if (a.w_[w] != b.w_[w]) return false;
  for (size_t w = shorter.w_.size(); w < longer.w_.size(); ++w)
    if (longer.w_[w]) return false;
  return true;
}

BitPoly random_bitpoly(size_t n_bits, std::mt19937_64& rng) {
  BitPoly p(n_bits);
  uint64_t* w = p.word_data();
  for (size_t i = 0; i < p.word_count(); ++i) w[i] = rng();
  p.resize_bits(n_bits);
  return p;
}

// ------------------------------------------------------------------ fields
u128 detail::clmul64_portable(uint64_t a, uint64_t b) noexcept {
  uint64_t lo = 0, hi = 0;
  for (unsigned i = 0; i < 64; ++i)
    if ((b >> i) & 1) {
      lo ^= a << i;
      hi ^= i ? a >> (64 - i) : 0;
    }
  return u128{hi, lo};
}

gf16::value_type gf16::mul(value_type a, value_type b) noexcept {
  uint64_t p = clmul(a, b).lo;  // < 2^31
  for (int k = 30; k >= 16; --k)
    if ((p >> k) & 1) p ^= (uint64_t{1} << k) | (kModulusTail << (k - 16));
  return static_cast<value_type>(p);
}
gf16::value_type gf16::sqr(value_type a) noexcept { return mul(a, a); }

gf64::value_type gf64::mul(value_type a, value_type b) noexcept {
  const u128 p = clmul(a, b);
  // x^64 = x^4 + x^3 + x + 1: fold hi twice
  const u128 t = clmul(p.hi, kModulusTail);
  const u128 t2 = clmul(t.hi, kModulusTail);
  return p.lo ^ t.lo ^ t2.lo;
}
gf64::value_type gf64::sqr(value_type a) noexcept { return mul(a, a); }

gf128::value_type gf128::mul(value_type a, value_type b) noexcept {
  // schoolbook 128x128 -> 256 from four 64x64 products, then fold x^128 = x^7 + x^2 + x + 1
  const u128 ll = clmul(a.lo, b.lo), hh = clmul(a.hi, b.hi), lh = clmul(a.lo, b.hi), hl = clmul(a.hi, b.lo);
  uint64_t w0 = ll.lo, w1 = ll.hi ^ lh.lo ^ hl.lo, w2 = hh.lo ^ lh.hi ^ hl.hi, w3 = hh.hi;
  const u128 f3 = clmul(w3, kModulusTail), f2 = clmul(w2, kModulusTail);
  w1 ^= f3.lo;
  w2 = f3.hi;  // bits 128.. of the first fold (< 2^7)
  w0 ^= f2.lo;
  w1 ^= f2.hi;
  const u128 f = clmul(w2, kModulusTail);
  w0 ^= f.lo;
  return u128{w1, w0};
}
gf128::value_type gf128::sqr(value_type a) noexcept { return mul(a, a); }

unsigned frobenius_order_of_basis(unsigned i) {
  if (i == 0) throw std::invalid_argument("frobenius_order_of_basis: i must be positive (v_0 has order 1)");
  unsigned p = 1;
  while (p * 2 <= i) p *= 2;
  return 2 * p;
}

// ------------------------------------------------------------------ GF(2) row matrices
namespace {
template <class W>
W row_combo(W x, const W* rows, unsigned m) {
  W acc{};
  for (unsigned j = 0; j < m; ++j)
    if (test_bit(x, j)) acc ^= rows[j];
  return acc;
}

template <class W>
unsigned lead_bit(W v) {
  unsigned k = 0;
  while (!test_bit(v, k)) ++k;
  return k;
}

// x * rows = target (row-echelon with tags); false if unsolvable.
template <class W>
bool solve_combo(const W* rows, unsigned m, W target, W* out) {
  std::vector<W> ech, tag;
  std::vector<unsigned> lead;
  for (unsigned i = 0; i < m; ++i) {
    W r = rows[i], t = unit_bit<W>(i);
    for (size_t j = 0; j < ech.size(); ++j)
      if (test_bit(r, lead[j])) { r ^= ech[j]; t ^= tag[j]; }
    if (static_cast<bool>(r)) { ech.push_back(r); tag.push_back(t); lead.push_back(lead_bit(r)); }
  }
  W acc = target, x{};
  for (size_t j = 0; j < ech.size(); ++j)
    if (test_bit(acc, lead[j])) { acc ^= ech[j]; x ^= tag[j]; }
  if (static_cast<bool>(acc)) return false;
  *out = x;
  return true;
}

template <class W>
bool invert_rows(const std::vector<W>& rows, unsigned m, std::vector<W>& inv_out) {
  std::vector<W> a(rows), inv(m);
  for (unsigned i = 0; i < m; ++i) inv[i] = unit_bit<W>(i);
  for (unsigned col = 0; col < m; ++col) {
    unsigned piv = col;
    while (piv < m && !test_bit(a[piv], col)) ++piv;
    if (piv == m) return false;
    std::swap(a[col], a[piv]);
    std::swap(inv[col], inv[piv]);
    for (unsigned r = 0; r < m; ++r)
      if (r != col && test_bit(a[r], col)) { a[r] ^= a[col]; inv[r] ^= inv[col]; }
  }
  inv_out = inv;
  return true;
}
}  // namespace

template <class F>
CantorField<F>::CantorField() : c2p_(F::kDegree), p2c_(F::kDegree) {
  using V = value_type;
  constexpr unsigned m = F::kDegree;
  std::vector<V> artin(m);  // y -> y^2 + y, rows in polynomial representation
  for (unsigned k = 0; k < m; ++k) artin[k] = static_cast<V>(F::sqr(unit_bit<V>(k)) ^ unit_bit<V>(k));
  c2p_[0] = unit_bit<V>(0);
  for (unsigned i = 1; i < m; ++i) {
    V y{};
    if (!solve_combo(artin.data(), m, c2p_[i - 1], &y))
      throw std::runtime_error("CantorField: Artin-Schreier equation has no solution (wrong modulus?)");
    if (test_bit(y, 0)) y ^= unit_bit<V>(0);  // the root with bit 0 clear
    if (!(static_cast<V>(F::sqr(y) ^ y) == c2p_[i - 1])) throw std::runtime_error("CantorField: recurrence check failed");
    c2p_[i] = y;
  }
  if (!invert_rows(c2p_, m, p2c_)) throw std::runtime_error("CantorField: basis-change matrix not invertible");
}

template <class F>
const CantorField<F>& CantorField<F>::get() {
  static const CantorField field;
  return field;
}

template <class F>
FieldElem<F> CantorField<F>::cantor_to_poly(CantorVec<F> c) const {
  return {row_combo(c.bits, c2p_.data(), F::kDegree)};
}
template <class F>
CantorVec<F> CantorField<F>::poly_to_cantor(FieldElem<F> a) const {
  return {row_combo(a.v, p2c_.data(), F::kDegree)};
}

template class CantorField<gf16>;
template class CantorField<gf64>;
template class CantorField<gf128>;

// ------------------------------------------------------------------ basis conversion (GPU)
void basis_cvt(BitPoly& f, ExecPolicy, size_t content_bits) {
  const size_t n = f.bit_length();
  if (n == 0 || (n & (n - 1))) throw std::invalid_argument("basis_cvt: length must be a power of two");
  if (n <= 2) return;
  check(fpm_basis_cvt(f.word_data(), n, content_bits ? content_bits : 1, current_device()));
}

void i_basis_cvt(BitPoly& g, ExecPolicy) {
  const size_t n = g.bit_length();
  if (n == 0 || (n & (n - 1))) throw std::invalid_argument("basis_cvt: length must be a power of two");
  if (n <= 2) return;
  check(fpm_i_basis_cvt(g.word_data(), n, current_device()));
}

// ------------------------------------------------------------------ encode / decode
template <class F>
PartitionSpec<F> make_partition_spec(unsigned l) {
  if (l >= F::kDegree / 2) throw std::invalid_argument("PartitionSpec: l must satisfy l < m/2");
  PartitionSpec<F> s;
  s.l = l;
  s.base = CantorVec<F>{unit_bit<typename F::value_type>(l + F::kDegree / 2)};
  s.n_p = size_t{1} << l;
  return s;
}

template <class F>
EncodeMatrix<F>::EncodeMatrix() {
  constexpr unsigned m = F::kDegree;
  const auto& fld = CantorField<F>::get();
  rows_.resize(m);
  for (unsigned j = 0; j < m; ++j) {  // r_j = prod over bits k of j of v_{m/2-k} (encode.cpp:60-66)
    value_type r = unit_bit<value_type>(0);
    for (unsigned k = 0; k < F::kLogDegree; ++k)
      if ((j >> k) & 1) r = F::mul(r, fld.basis(m / 2 - k).v);
    rows_[j] = r;
  }
  if (!invert_rows(rows_, m, inv_)) throw std::runtime_error("EncodeMatrix: matrix is singular (field construction bug)");
  auto tables = [&](const std::vector<value_type>& rows, std::vector<value_type>& tab) {
    tab.assign(size_t{m / kChunkBits} * 16, value_type{});
    for (unsigned c = 0; c < m / kChunkBits; ++c)
      for (unsigned v = 1; v < 16; ++v) {
        const unsigned low = v & (0u - v), bit = __builtin_ctz(low);
        tab[c * 16 + v] = tab[c * 16 + (v ^ low)] ^ rows[c * kChunkBits + bit];
      }
  };
  tables(rows_, fwd_tab_);
  tables(inv_, inv_tab_);
}

template <class F>
typename EncodeMatrix<F>::value_type EncodeMatrix<F>::lookup(const std::vector<value_type>& tab, value_type x) const {
  value_type acc{};
  for (unsigned c = 0; c < F::kDegree / kChunkBits; ++c)
    acc ^= tab[c * 16 + (detail::low_word(detail::value_shr(x, c * kChunkBits)) & 0xF)];
  return acc;
}

template <class F>
const EncodeMatrix<F>& EncodeMatrix<F>::get() {
  static const EncodeMatrix mat;
  return mat;
}

template <class F>
EvalVec<F> encode(const BitPoly& a, const PartitionSpec<F>& spec, const EncodeMatrix<F>&, ExecPolicy) {
  if (a.bit_length() != size_t{F::kDegree} * spec.n_p) throw std::invalid_argument("encode: input length must be m * n_p bits");
  if constexpr (is64<F>()) {
    EvalVec<F> out(spec.n_p);
    check(fpm_encode64(a.word_data(), spec.l, reinterpret_cast<uint64_t*>(out.data()), current_device()));
    return out;
  } else if constexpr (!is128<F>()) {
    not_built("encode");
  } else {
    EvalVec<F> out(spec.n_p);
    check(fpm_encode(a.word_data(), spec.l, reinterpret_cast<uint64_t*>(out.data()), current_device()));
    return out;
  }
}

template <class F>
BitPoly decode(std::span<const FieldElem<F>> v, const PartitionSpec<F>& spec, const EncodeMatrix<F>&, ExecPolicy) {
  if (v.size() != spec.n_p) throw std::invalid_argument("decode: length must equal n_p");
  if constexpr (is64<F>()) {
    BitPoly a(size_t{F::kDegree} * spec.n_p);
    check(fpm_decode64(reinterpret_cast<const uint64_t*>(v.data()), spec.l, a.word_data(), current_device()));
    return a;
  } else if constexpr (!is128<F>()) {
    not_built("decode");
  } else {
    BitPoly a(size_t{F::kDegree} * spec.n_p);
    check(fpm_decode(reinterpret_cast<const uint64_t*>(v.data()), spec.l, a.word_data(), current_device()));
    return a;
  }
}

void transpose64x64(uint64_t m[64]) {
  // bit (r, c) <-> (c, r) by three-XOR block swaps at widths 32, 16, ..., 1
  uint64_t mask = 0x00000000FFFFFFFFull;
  for (unsigned w = 32; w; w >>= 1, mask ^= mask << w) {
    for (unsigned r = 0; r < 64; ++r) {
      if (r & w) continue;
      const uint64_t t = ((m[r] >> w) ^ m[r + w]) & mask;
      m[r] ^= t << w;
      m[r + w] ^= t;
    }
  }
}

template <class F>
std::vector<std::vector<typename F::value_type>> enumerate_partition(const PartitionSpec<F>& spec) {
  if (F::kDegree > 16) throw std::invalid_argument("enumerate_partition: only the m=16 test field is enumerable");
  const auto& fld = CantorField<F>::get();
  std::vector<std::vector<typename F::value_type>> it(F::kDegree);
  std::vector<typename F::value_type> cur(spec.n_p);
  for (size_t u = 0; u < spec.n_p; ++u) cur[u] = spec.base.bits ^ detail::from_low_word<typename F::value_type>(u);
  for (unsigned j = 0; j < F::kDegree; ++j) {
    it[j] = cur;
    for (auto& e : cur) e = fld.poly_to_cantor(gf_sqr(fld.cantor_to_poly(CantorVec<F>{e}))).bits;
  }
  return it;
}

#define FPMUL_B200_ENCODE(F)                                                                                   \
  template PartitionSpec<F> make_partition_spec<F>(unsigned);                                                  \
  template class EncodeMatrix<F>;                                                                              \
  template EvalVec<F> encode<F>(const BitPoly&, const PartitionSpec<F>&, const EncodeMatrix<F>&, ExecPolicy);  \
  template BitPoly decode<F>(std::span<const FieldElem<F>>, const PartitionSpec<F>&, const EncodeMatrix<F>&,   \
                             ExecPolicy);                                                                      \
  template std::vector<std::vector<typename F::value_type>> enumerate_partition<F>(const PartitionSpec<F>&);
FPMUL_B200_ENCODE(gf16)
FPMUL_B200_ENCODE(gf64)
FPMUL_B200_ENCODE(gf128)

// ------------------------------------------------------------------ butterflies
template <class F>
ButterflyPlan<F> plan_butterflies(unsigned layers, CantorVec<F> base) {
  using V = typename F::value_type;
  const auto& fld = CantorField<F>::get();
  ButterflyPlan<F> plan;
  plan.layers = layers;
  plan.base = base;
  if (!layers) return plan;
  plan.mults.reserve((size_t{1} << layers) - 1);
  for (unsigned i = layers; i-- > 0;)  // layer-major, top layer first
    for (size_t b = 0; b < (size_t{1} << (layers - 1 - i)); ++b)
      plan.mults.push_back(
          fld.cantor_to_poly(CantorVec<F>{static_cast<V>(detail::value_shr(base.bits, i) ^ detail::from_low_word<V>(b << 1))}).v);
  return plan;
}

namespace {
template <class F>
void run_butterfly(std::span<FieldElem<F>> v, const ButterflyPlan<F>& plan, bool inverse) {
  if (v.size() != size_t{1} << plan.layers) throw std::invalid_argument("lch_butterfly: vector length does not match plan");
  if constexpr (is64<F>()) {
    if (!plan.layers) return;
    check(fpm_lch_butterfly64(reinterpret_cast<uint64_t*>(v.data()), plan.layers, plan.base.bits, inverse ? 1 : 0,
                              current_device()));
  } else if constexpr (!is128<F>()) {
    not_built("lch_butterfly");
  } else {
    if (!plan.layers) return;
    const uint64_t base[2] = {plan.base.bits.lo, plan.base.bits.hi};
    check(fpm_lch_butterfly(reinterpret_cast<uint64_t*>(v.data()), plan.layers, base, inverse ? 1 : 0, current_device()));
  }
}
}  // namespace

template <class F>
void lch_butterfly(std::span<FieldElem<F>> v, const ButterflyPlan<F>& plan, ExecPolicy, size_t) {
  run_butterfly<F>(v, plan, false);
}
template <class F>
void i_lch_butterfly(std::span<FieldElem<F>> v, const ButterflyPlan<F>& plan, ExecPolicy, size_t) {
  run_butterfly<F>(v, plan, true);
}

template <class F>
FieldElem<F> direct_eval(std::span<const FieldElem<F>> coeffs, CantorVec<F> pt) {
  const auto& fld = CantorField<F>::get();
  FieldElem<F> acc{};
  for (size_t k = 0; k < coeffs.size(); ++k) {
    if (coeffs[k] == FieldElem<F>{}) continue;
    FieldElem<F> term = coeffs[k];
    for (unsigned i = 0; (size_t{1} << i) <= k; ++i)
      if ((k >> i) & 1) term = gf_mul(term, fld.cantor_to_poly(subspace_eval(i, pt)));
    acc = gf_add(acc, term);
  }
  return acc;
}

#define FPMUL_B200_BUTTERFLY(F)                                                                            \
  template ButterflyPlan<F> plan_butterflies<F>(unsigned, CantorVec<F>);                                   \
  template void lch_butterfly<F>(std::span<FieldElem<F>>, const ButterflyPlan<F>&, ExecPolicy, size_t);    \
  template void i_lch_butterfly<F>(std::span<FieldElem<F>>, const ButterflyPlan<F>&, ExecPolicy, size_t);  \
  template FieldElem<F> direct_eval<F>(std::span<const FieldElem<F>>, CantorVec<F>);
FPMUL_B200_BUTTERFLY(gf16)
FPMUL_B200_BUTTERFLY(gf64)
FPMUL_B200_BUTTERFLY(gf128)

// ------------------------------------------------------------------ products
MulPlan plan_mul(size_t len_a_bits, size_t len_b_bits, FieldChoice field) {
  fpm_plan p{};
  const int f = field == FieldChoice::kGF64 ? FPM_FIELD_GF64 : field == FieldChoice::kGF128 ? FPM_FIELD_GF128 : FPM_FIELD_AUTO;
  check(fpm_plan_mul(len_a_bits, len_b_bits, f, &p));
  MulPlan m;
  m.n_bits = p.n_bits;
  m.log2_n = p.log2_n;
  m.field_degree = p.field_degree;
  m.log2_field_degree = p.log2_field_degree;
  m.l = p.l;
  m.n_p = p.n_p;
  return m;
}

namespace {
BitPoly gpu_product(const BitPoly& a, const BitPoly& b, int field, StageSeconds* st) {
  if (!a.bit_length() || !b.bit_length()) return BitPoly{};
  BitPoly c(a.bit_length() + b.bit_length() - 1);
  double sec[FPM_NUM_STAGES] = {};
  check(fpm_polymul(a.word_data(), a.bit_length(), b.word_data(), b.bit_length(), c.word_data(), field,
                    current_device(), st ? sec : nullptr));
  if (st) {
    st->basiscvt += sec[0]; st->encode += sec[1]; st->butterfly += sec[2]; st->pointwise += sec[3];
    st->ibutterfly += sec[4]; st->decode += sec[5]; st->ibasiscvt += sec[6];
  }
  return c;
}
}  // namespace

BitPoly fp_polymul(const BitPoly& a, const BitPoly& b) { return fp_polymul(a, b, MulOptions{}); }

BitPoly karatsuba_mul(const BitPoly& a, const BitPoly& b) {
  if (!a.bit_length() || !b.bit_length()) return BitPoly{};
  BitPoly c(a.bit_length() + b.bit_length() - 1);
  check(fpm_karatsuba_mul(a.word_data(), a.bit_length(), b.word_data(), b.bit_length(), c.word_data(),
                          current_device()));
  return c;
}

// polymul.hpp:83: schoolbook and Karatsuba give the same words; both run the GPU word product.
BitPoly naive_mul(const BitPoly& a, const BitPoly& b) { return karatsuba_mul(a, b); }

BitPoly fp_polymul(const BitPoly& a, const BitPoly& b, const MulOptions& opts) {
  if (!a.bit_length() || !b.bit_length()) return BitPoly{};
  const size_t max_len = std::max(a.bit_length(), b.bit_length());
  // polymul.cpp:226-231: in auto mode short inputs take karatsuba_mul
  if (opts.field == FieldChoice::kAuto && max_len < opts.fft_threshold_bits) return karatsuba_mul(a, b);
  // The reference's field choice (plan_mul, polymul.cpp:203-205): kAuto runs GF(2^64) when it
  // supports the size.  Resolved here so that a caller-chosen fft_threshold_bits below the C-ABI's
  // default is honoured (the C-ABI applies the default threshold only to FPM_FIELD_AUTO).
  fpm_plan p{};
  const int req = opts.field == FieldChoice::kGF64 ? FPM_FIELD_GF64
                : opts.field == FieldChoice::kGF128 ? FPM_FIELD_GF128 : FPM_FIELD_AUTO;
  check(fpm_plan_mul(a.bit_length(), b.bit_length(), req, &p));
  if (opts.devices.size() > 1) {  // sharded over several GPUs (logical ranks), GF(2^128) transform
    BitPoly c(a.bit_length() + b.bit_length() - 1);
    check(fpm_polymul_multi(a.word_data(), a.bit_length(), b.word_data(), b.bit_length(), c.word_data(), req,
                            opts.devices.data(), static_cast<int>(opts.devices.size())));
    return c;
  }
  if (opts.devices.size() == 1) {
    const int prev = current_device();
    set_device(opts.devices[0]);
    struct Restore { int d; ~Restore() { set_device(d); } } restore{prev};
    return gpu_product(a, b, p.field_degree == 64 ? FPM_FIELD_GF64 : FPM_FIELD_GF128, opts.stage_seconds);
  }
  return gpu_product(a, b, p.field_degree == 64 ? FPM_FIELD_GF64 : FPM_FIELD_GF128, opts.stage_seconds);
}

template <class F>
EvalVec<F> pointwise_mul(std::span<const FieldElem<F>> u, std::span<const FieldElem<F>> v, ExecPolicy) {
  if (u.size() != v.size()) throw std::invalid_argument("pointwise_mul: length mismatch");
  if constexpr (is64<F>()) {
    EvalVec<F> out(u.size());
    if (!u.empty())
      check(fpm_pointwise64(reinterpret_cast<const uint64_t*>(u.data()), reinterpret_cast<const uint64_t*>(v.data()),
                            reinterpret_cast<uint64_t*>(out.data()), u.size(), current_device()));
    return out;
  } else if constexpr (!is128<F>()) {
    not_built("pointwise_mul");
  } else {
    EvalVec<F> out(u.size());
    if (!u.empty())
      check(fpm_pointwise(reinterpret_cast<const uint64_t*>(u.data()), reinterpret_cast<const uint64_t*>(v.data()),
                          reinterpret_cast<uint64_t*>(out.data()), u.size(), current_device()));
    return out;
  }
}

template <class F>
bool frobenius_value_check(const BitPoly& a, FieldElem<F> pt) {
  auto horner = [&](FieldElem<F> x) {
    FieldElem<F> acc{};
    const FieldElem<F> one{unit_bit<typename F::value_type>(0)};
    for (size_t k = a.bit_length(); k-- > 0;) {
      acc = gf_mul(acc, x);
      if (a.bit(k)) acc = gf_add(acc, one);
    }
    return acc;
  };
  return horner(gf_sqr(pt)) == gf_sqr(horner(pt));
}

#define FPMUL_B200_POLYMUL(F)                                                                                  \
  template EvalVec<F> pointwise_mul<F>(std::span<const FieldElem<F>>, std::span<const FieldElem<F>>, ExecPolicy); \
  template bool frobenius_value_check<F>(const BitPoly&, FieldElem<F>);
FPMUL_B200_POLYMUL(gf16)
FPMUL_B200_POLYMUL(gf64)
FPMUL_B200_POLYMUL(gf128)

}  // namespace fpmul
