// Drop-in for parsim/numerics.hpp (/root/reference/proj/include/parsim).
//
// Put include/parsim_dropin (and include/) BEFORE the reference's
// proj/include on the include path and link libpsb.so + cudart: the
// reference header is included unchanged (#include_next), its hot-path
// function is renamed out of the way, and the same signature is served by the
// sm_100a kernels.  Everything else (DenseVector, DenseMatrix, SeededRng,
// matmul, ...) is the reference's own.
//
//   vec_axpy   numerics.hpp:70-78   a*x + y with a separate RN multiply and
//                                   add, check_finite -> std::invalid_argument
#pragma once

#define vec_axpy parsim_reference_vec_axpy
#include_next "parsim/numerics.hpp"
#undef vec_axpy

#include "parsim_dropin_device.hpp"

namespace parsim {

inline DenseVector vec_axpy(double a, const DenseVector& x, const DenseVector& y) {
  detail::require(x.size() == y.size(), "vec_axpy: dimension mismatch (" + std::to_string(x.size()) + " vs " +
                                            std::to_string(y.size()) + ")");
  if (x.empty()) return DenseVector{};
  std::lock_guard<std::mutex> g(parsim_dropin::lock());
  return parsim_dropin::device().vec_axpy(a, x, y);
}

}  // namespace parsim
