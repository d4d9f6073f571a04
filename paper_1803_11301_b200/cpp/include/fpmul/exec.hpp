// fpmul/exec.hpp -- B200 backend mirror of /root/reference/proj/include/fpmul/exec.hpp:24-31.
// On the GPU every stage is parallel; ExecPolicy is accepted for source compatibility and does
// not change results (the reference guarantees kSerial == kParallel bit for bit, too).
#ifndef FPMUL_B200_EXEC_HPP_
#define FPMUL_B200_EXEC_HPP_

#include <cstddef>

namespace fpmul {

enum class ExecPolicy {
  kSerial,
  kParallel,
};

inline constexpr size_t kDefaultButterflyCacheElems = size_t{1} << 15;

/// CUDA device used by the host-buffer entry points of this backend (default 0).
void set_device(int device);
int current_device();

}  // namespace fpmul

#endif  // FPMUL_B200_EXEC_HPP_
