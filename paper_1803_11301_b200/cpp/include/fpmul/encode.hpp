// fpmul/encode.hpp -- B200 backend mirror of /root/reference/proj/include/fpmul/encode.hpp:32-135.
#ifndef FPMUL_B200_ENCODE_HPP_
#define FPMUL_B200_ENCODE_HPP_

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "fpmul/bitpoly.hpp"
#include "fpmul/butterfly.hpp"
#include "fpmul/cantor.hpp"
#include "fpmul/exec.hpp"
#include "fpmul/gf.hpp"

namespace fpmul {

/// Frobenius partition Sigma = base + V_l with base = e_{l+m/2} (Cantor coordinates), |Sigma| = n_p.
template <class F>
struct PartitionSpec {
  unsigned l = 0;
  CantorVec<F> base{};
  size_t n_p = 1;
};

template <class F>
PartitionSpec<F> make_partition_spec(unsigned l);

/// Encode matrix E (rows r_j = prod_{bits k of j} v_{m/2-k}), its inverse, and 4-bit M4R tables.
template <class F>
class EncodeMatrix {
 public:
  using value_type = typename F::value_type;
  static constexpr unsigned kChunkBits = 4;
  static const EncodeMatrix& get();
  EncodeMatrix();

  FieldElem<F> row(unsigned j) const { return {rows_[j]}; }
  FieldElem<F> inv_row(unsigned j) const { return {inv_[j]}; }
  std::span<const value_type> rows() const { return rows_; }
  std::span<const value_type> inv_rows() const { return inv_; }
  FieldElem<F> m4r_mul(value_type x) const { return {lookup(fwd_tab_, x)}; }
  FieldElem<F> m4r_mul_inv(value_type x) const { return {lookup(inv_tab_, x)}; }
  /// Test hook (selftest fault injection): flips one bit of one forward-table entry.
  void corrupt_for_test() { fwd_tab_[1] ^= detail::unit_bit<value_type>(0); }

 private:
  value_type lookup(const std::vector<value_type>& tab, value_type x) const;
  std::vector<value_type> rows_, inv_, fwd_tab_, inv_tab_;
};

template <class F>
EvalVec<F> encode(const BitPoly& a, const PartitionSpec<F>& spec, const EncodeMatrix<F>& mat,
                  ExecPolicy policy = ExecPolicy::kParallel);
template <class F>
BitPoly decode(std::span<const FieldElem<F>> v, const PartitionSpec<F>& spec, const EncodeMatrix<F>& mat,
               ExecPolicy policy = ExecPolicy::kParallel);

void transpose64x64(uint64_t m[64]);

template <class F>
std::vector<std::vector<typename F::value_type>> enumerate_partition(const PartitionSpec<F>& spec);

#define FPMUL_B200_DECLARE_ENCODE(F)                                                                     \
  extern template PartitionSpec<F> make_partition_spec<F>(unsigned);                                     \
  extern template class EncodeMatrix<F>;                                                                 \
  extern template EvalVec<F> encode<F>(const BitPoly&, const PartitionSpec<F>&, const EncodeMatrix<F>&,  \
                                       ExecPolicy);                                                      \
  extern template BitPoly decode<F>(std::span<const FieldElem<F>>, const PartitionSpec<F>&,              \
                                    const EncodeMatrix<F>&, ExecPolicy);                                 \
  extern template std::vector<std::vector<typename F::value_type>> enumerate_partition<F>(               \
      const PartitionSpec<F>&);
FPMUL_B200_DECLARE_ENCODE(gf16)
FPMUL_B200_DECLARE_ENCODE(gf64)
FPMUL_B200_DECLARE_ENCODE(gf128)
#undef FPMUL_B200_DECLARE_ENCODE

}  // namespace fpmul

#endif  // FPMUL_B200_ENCODE_HPP_
