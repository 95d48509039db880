// txb_common.cuh — shared device/host helpers for the txb CUDA library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>

#include "../../include/txb.h"
#include "txb_device.cuh"

namespace txb {

// ---------------------------------------------------------------------------
// Error plumbing: thread-local message behind txb_last_error().
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define TXB_CUDA_TRY(expr)                                             \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) return ::txb::cuda_fail(_e, #expr);         \
  } while (0)


// ---------------------------------------------------------------------------
// Affine map inverse of a simplex, float64, in the reference's expression
// order (txfem/mesh.py:150-190): J's column k = v_{k+1} - v_0; 2D closed form,
// 3D cofactors; numpy evaluates a*b - c*d as two rounded products and one
// rounded difference and sums the 3x3 determinant left to right.  Every
// operation is an _rn intrinsic, so the result is bit-identical to numpy.
// ---------------------------------------------------------------------------
// x / det, correctly rounded.  A zero numerator (frequent: axis-aligned edges
// give exact zero cofactors) skips __ddiv_rn, whose range check would send
// the whole warp down its slow path: for det > 0, +-0 / det = +-0 exactly.
// (det <= 0 is an OrientationError in the reference; its cells' values are
// not compared.)
__device__ __forceinline__ double div_det(double x, double det) {
  if (x == 0.0) return det < 0.0 ? -x : x;
  return __ddiv_rn(x, det);
}

template <int D>
__device__ __forceinline__ void affine_inverse(const double (&X)[D + 1][D], double (&inv)[D * D], double& det) {
  double m[D][D];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int i = 0; i < D; ++i) m[i][k] = __dsub_rn(X[k + 1][i], X[0][i]);
  if constexpr (D == 2) {
    const double a = m[0][0], b = m[0][1], c = m[1][0], e = m[1][1];
    det = __dsub_rn(__dmul_rn(a, e), __dmul_rn(b, c));
    inv[0] = div_det(e, det);
    inv[1] = div_det(-b, det);
    inv[2] = div_det(-c, det);
    inv[3] = div_det(a, det);
  } else {
    const double cof00 = __dsub_rn(__dmul_rn(m[1][1], m[2][2]), __dmul_rn(m[1][2], m[2][1]));
    const double cof01 = __dsub_rn(__dmul_rn(m[1][2], m[2][0]), __dmul_rn(m[1][0], m[2][2]));
    const double cof02 = __dsub_rn(__dmul_rn(m[1][0], m[2][1]), __dmul_rn(m[1][1], m[2][0]));
    det = __dadd_rn(__dadd_rn(__dmul_rn(m[0][0], cof00), __dmul_rn(m[0][1], cof01)), __dmul_rn(m[0][2], cof02));
    inv[0 * 3 + 0] = div_det(cof00, det);
    inv[1 * 3 + 0] = div_det(cof01, det);
    inv[2 * 3 + 0] = div_det(cof02, det);
    inv[0 * 3 + 1] = div_det(__dsub_rn(__dmul_rn(m[0][2], m[2][1]), __dmul_rn(m[0][1], m[2][2])), det);
    inv[1 * 3 + 1] = div_det(__dsub_rn(__dmul_rn(m[0][0], m[2][2]), __dmul_rn(m[0][2], m[2][0])), det);
    inv[2 * 3 + 1] = div_det(__dsub_rn(__dmul_rn(m[0][1], m[2][0]), __dmul_rn(m[0][0], m[2][1])), det);
    inv[0 * 3 + 2] = div_det(__dsub_rn(__dmul_rn(m[0][1], m[1][2]), __dmul_rn(m[0][2], m[1][1])), det);
    inv[1 * 3 + 2] = div_det(__dsub_rn(__dmul_rn(m[0][2], m[1][0]), __dmul_rn(m[0][0], m[1][2])), det);
    inv[2 * 3 + 2] = div_det(__dsub_rn(__dmul_rn(m[0][0], m[1][1]), __dmul_rn(m[0][1], m[1][0])), det);
  }
}

}  // namespace txb
