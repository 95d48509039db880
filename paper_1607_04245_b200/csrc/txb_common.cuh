// txb_common.cuh — shared device/host helpers for the txb CUDA library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>

#include "../../include/txb.h"

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
// Exact-rounding arithmetic.  The reference lanes are compiled with
// -ffp-contract=off (pkg/setup.py:17-20): every product and sum rounds on its
// own.  The _rn intrinsics are never contracted into FMA by nvcc, so the
// device reproduces the reference bit for bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// ---------------------------------------------------------------------------
// Shared-memory / bulk-copy / mbarrier primitives (sm_90+ PTX, used on sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// L2 policy for streamed-once inputs: evict first, keep L2 for the outputs'
// write-back and for the other CTAs' in-flight lines.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// One bulk (non-tensor TMA) copy global -> shared, completion counted on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16 (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Bulk prefetch of [src, src + bytes) into L2 (no completion, no data returned).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ constexpr int make_odd(int x) { return (x & 1) ? x : x + 1; }

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
