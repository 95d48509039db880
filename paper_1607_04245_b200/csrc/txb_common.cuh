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
// x / det, correctly rounded (= numpy's x / det), for all the cofactors of one
// cell.  One correctly rounded reciprocal y = RN(1/det) per cell (__drcp_rn);
// per quotient q0 = RN(x*y), then two residual corrections
//   r_i = RN(x - det*q_i)  (one FMA),  q_{i+1} = RN(q_i + r_i*y)  (one FMA).
// q0 is within a few ulps of x/det and the first correction brings q1 within
// one ulp; for such q1 the residual r1 is exact and, with y = RN(1/det),
// Markstein's theorem (radix 2, round to nearest, no underflow/overflow) makes
// q2 the correctly rounded quotient.  The nine quotients of a 3D cell are
// independent 5-instruction chains instead of nine serial __ddiv_rn
// sequences, each with its own slow-path branch (the fused mesh kernel was
// latency-bound on them).  Outside a safe exponent range (|x|, det in
// [2^-500, 2^500]: quotients and residuals stay normal) and for det <= 0 (an
// OrientationError in the reference; its values are not compared) the
// quotient falls back to __ddiv_rn.  A zero numerator gives +-0 exactly.
struct DetDivider {
  double det, y;
  bool fast;
  __device__ __forceinline__ explicit DetDivider(double d) : det(d), y(0.0) {
    fast = d >= 0x1p-500 && d <= 0x1p500;
    if (fast) y = __drcp_rn(d);
  }
  __device__ __forceinline__ double operator()(double x) const {
    if (x == 0.0) return det < 0.0 ? -x : x;
    const double ax = fabs(x);
    if (!fast || ax < 0x1p-500 || ax > 0x1p500) return __ddiv_rn(x, det);
    const double q0 = __dmul_rn(x, y);
    const double q1 = __fma_rn(__fma_rn(-q0, det, x), y, q0);
    return __fma_rn(__fma_rn(-q1, det, x), y, q1);
  }
};

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
    const DetDivider div(det);
    inv[0] = div(e);
    inv[1] = div(-b);
    inv[2] = div(-c);
    inv[3] = div(a);
  } else {
    const double cof00 = __dsub_rn(__dmul_rn(m[1][1], m[2][2]), __dmul_rn(m[1][2], m[2][1]));
    const double cof01 = __dsub_rn(__dmul_rn(m[1][2], m[2][0]), __dmul_rn(m[1][0], m[2][2]));
    const double cof02 = __dsub_rn(__dmul_rn(m[1][0], m[2][1]), __dmul_rn(m[1][1], m[2][0]));
    det = __dadd_rn(__dadd_rn(__dmul_rn(m[0][0], cof00), __dmul_rn(m[0][1], cof01)), __dmul_rn(m[0][2], cof02));
    const DetDivider div(det);
    inv[0 * 3 + 0] = div(cof00);
    inv[1 * 3 + 0] = div(cof01);
    inv[2 * 3 + 0] = div(cof02);
    inv[0 * 3 + 1] = div(__dsub_rn(__dmul_rn(m[0][2], m[2][1]), __dmul_rn(m[0][1], m[2][2])));
    inv[1 * 3 + 1] = div(__dsub_rn(__dmul_rn(m[0][0], m[2][2]), __dmul_rn(m[0][2], m[2][0])));
    inv[2 * 3 + 1] = div(__dsub_rn(__dmul_rn(m[0][1], m[2][0]), __dmul_rn(m[0][0], m[2][1])));
    inv[0 * 3 + 2] = div(__dsub_rn(__dmul_rn(m[0][1], m[1][2]), __dmul_rn(m[0][2], m[1][1])));
    inv[1 * 3 + 2] = div(__dsub_rn(__dmul_rn(m[0][2], m[1][0]), __dmul_rn(m[0][0], m[1][2])));
    inv[2 * 3 + 2] = div(__dsub_rn(__dmul_rn(m[0][0], m[1][1]), __dmul_rn(m[0][1], m[1][0])));
  }
}

}  // namespace txb
