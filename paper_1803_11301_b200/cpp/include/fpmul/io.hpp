// io.hpp -- binary polynomial files, the reference interface proj/include/fpmul/io.hpp (declarations
// only; implementation in cpp/src/io_selftest.cpp).
//
// Format (reference io.hpp / io.cpp:23-56): a raw little-endian byte stream, coefficient k is bit
// (k mod 8) of byte k/8.  Trailing zero bytes are accepted on input; output is trimmed to the last
// nonzero byte (the zero polynomial is an empty file).
#pragma once
#include <string>

#include "fpmul/bitpoly.hpp"

namespace fpmul {

/// Throws std::runtime_error on I/O failure.
BitPoly load_polynomial(const std::string& path);

/// Writes the canonical trim.  Throws std::runtime_error on I/O failure.
void store_polynomial(const std::string& path, const BitPoly& poly);

}  // namespace fpmul
