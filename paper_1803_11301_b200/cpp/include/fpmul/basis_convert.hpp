// fpmul/basis_convert.hpp -- B200 backend mirror of
// /root/reference/proj/include/fpmul/basis_convert.hpp:34-45.  Both directions run on the GPU
// (fpm_basis_cvt / fpm_i_basis_cvt); `reference::` keeps the pass-by-pass formulation for checks.
#ifndef FPMUL_B200_BASIS_CONVERT_HPP_
#define FPMUL_B200_BASIS_CONVERT_HPP_

#include "fpmul/bitpoly.hpp"
#include "fpmul/exec.hpp"

namespace fpmul {

/// Monomial -> novel-polynomial basis, in place; length a power of two.  Bits >= content_bits
/// must be zero (they are then skipped).  Throws std::invalid_argument on a bad length.
void basis_cvt(BitPoly& f, ExecPolicy policy = ExecPolicy::kParallel, size_t content_bits = ~size_t{0});
/// Inverse conversion.
void i_basis_cvt(BitPoly& g, ExecPolicy policy = ExecPolicy::kParallel);

}  // namespace fpmul

#endif  // FPMUL_B200_BASIS_CONVERT_HPP_
