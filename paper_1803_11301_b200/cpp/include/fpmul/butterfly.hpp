// fpmul/butterfly.hpp -- B200 backend mirror of /root/reference/proj/include/fpmul/butterfly.hpp:30-91.
// GF(2^128) butterflies run on the GPU with twiddles generated on the fly from (layers, base);
// ButterflyPlan::mults is still filled for API compatibility (plan_butterflies), but the GPU
// never reads it.  Other fields are not built on this backend (std::invalid_argument).
#ifndef FPMUL_B200_BUTTERFLY_HPP_
#define FPMUL_B200_BUTTERFLY_HPP_

#include <cstddef>
#include <span>
#include <vector>

#include "fpmul/cantor.hpp"
#include "fpmul/exec.hpp"
#include "fpmul/gf.hpp"

namespace fpmul {

template <class F>
using EvalVec = std::vector<FieldElem<F>>;

template <class F>
struct ButterflyPlan {
  unsigned layers = 0;
  CantorVec<F> base{};
  std::vector<typename F::value_type> mults;  // layer-major, top layer first (2^layers - 1 values)

  size_t layer_offset(unsigned i) const { return (size_t{1} << (layers - 1 - i)) - 1; }
  FieldElem<F> multiplier(unsigned i, size_t block) const { return {mults[layer_offset(i) + block]}; }
};

template <class F>
ButterflyPlan<F> plan_butterflies(unsigned layers, CantorVec<F> base);

template <class F>
void lch_butterfly(std::span<FieldElem<F>> v, const ButterflyPlan<F>& plan, ExecPolicy policy = ExecPolicy::kParallel,
                   size_t cache_elems = kDefaultButterflyCacheElems);
template <class F>
void i_lch_butterfly(std::span<FieldElem<F>> v, const ButterflyPlan<F>& plan,
                     ExecPolicy policy = ExecPolicy::kParallel, size_t cache_elems = kDefaultButterflyCacheElems);

/// sum_k coeffs[k] * X_k(pt), X_k = prod_{bits i of k} s_i (host evaluation, for checks).
template <class F>
FieldElem<F> direct_eval(std::span<const FieldElem<F>> coeffs, CantorVec<F> pt);

#define FPMUL_B200_DECLARE_BUTTERFLY(F)                                                                  \
  extern template ButterflyPlan<F> plan_butterflies<F>(unsigned, CantorVec<F>);                          \
  extern template void lch_butterfly<F>(std::span<FieldElem<F>>, const ButterflyPlan<F>&, ExecPolicy,    \
                                        size_t);                                                         \
  extern template void i_lch_butterfly<F>(std::span<FieldElem<F>>, const ButterflyPlan<F>&, ExecPolicy,  \
                                          size_t);                                                       \
  extern template FieldElem<F> direct_eval<F>(std::span<const FieldElem<F>>, CantorVec<F>);
FPMUL_B200_DECLARE_BUTTERFLY(gf16)
FPMUL_B200_DECLARE_BUTTERFLY(gf64)
FPMUL_B200_DECLARE_BUTTERFLY(gf128)
#undef FPMUL_B200_DECLARE_BUTTERFLY

}  // namespace fpmul

#endif  // FPMUL_B200_BUTTERFLY_HPP_
