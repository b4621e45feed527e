// Reference-order fp64 kernel shapes (kernels.hpp:93-134) shared by the fp64
// column / dense / pivoted-Cholesky kernels.
#pragma once
#include <cuda_runtime.h>

#include "gpk_internal.h"

namespace gpk {

// kernels.hpp:235-243 (which < 0) and :252-267 (which >= 0), bit-faithful
// operation order: s = (sq_r + sq_p) - 2 <sx_r, sx_p>, clamped; no FMA contraction.
__device__ __forceinline__ double ref_shape(int f, double s) {
  switch (f) {
    case kRBF: return exp(-0.5 * s);
    case kMatern12: return exp(-sqrt(s));
    case kMatern32: {
      const double r = sqrt(__dmul_rn(3.0, s));
      return __dmul_rn(__dadd_rn(1.0, r), exp(-r));
    }
    default: {
      const double r = sqrt(__dmul_rn(5.0, s));
      return __dmul_rn(__dadd_rn(__dadd_rn(1.0, r), __ddiv_rn(__dmul_rn(r, r), 3.0)), exp(-r));
    }
  }
}
__device__ __forceinline__ double ref_shape_ds(int f, double s) {
  switch (f) {
    case kRBF: return __dmul_rn(-0.5, exp(-0.5 * s));
    case kMatern12: {
      if (s <= 0.0) return 0.0;
      const double r = sqrt(s);
      return __ddiv_rn(-exp(-r), __dmul_rn(2.0, r));
    }
    case kMatern32: return __dmul_rn(-1.5, exp(-sqrt(__dmul_rn(3.0, s))));
    default: {
      const double r = sqrt(__dmul_rn(5.0, s));
      return __dmul_rn(__dmul_rn(-(5.0 / 6.0), __dadd_rn(1.0, r)), exp(-r));
    }
  }
}

}  // namespace gpk
