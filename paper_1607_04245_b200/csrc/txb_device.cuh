// txb_device.cuh — device primitives shared by the ahead-of-time kernels
// (nvcc) and the run-time compiled user-physics kernels (NVRTC, csrc/txb_jit.cu).
// No host headers: NVRTC compiles this file from memory.
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned long long uintptr_t;
#else
#include <cstdint>
#endif

#ifndef TXB_MAX_DIM
#define TXB_MAX_DIM 3
#define TXB_MAX_BASIS 4
#define TXB_MAX_COMP 3
#define TXB_MAX_QUAD 8
#endif

namespace txb {

// ---------------------------------------------------------------------------
// Exact-rounding arithmetic.  The reference lanes are compiled with
// -ffp-contract=off (pkg/setup.py:17-20): every product and sum rounds on its
// own.  The _rn intrinsics are never contracted into FMA, so the device
// reproduces the reference bit for bit.
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// try_wait with a suspend-time hint: the waiting thread sleeps up to `ns`
// nanoseconds (or until the phase completes) per attempt instead of retrying
// -- for the producer / gatherer warps, whose waits are long and whose spins
// would take issue slots from the consumer warps on their scheduler.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
  } while (!ok);
}

// ---------------------------------------------------------------------------
// Cluster launch control (sm_100): a running CTA cancels a CTA of its own grid
// that has not been launched yet and takes over its work -- hardware dynamic
// scheduling with no global counter (nothing to reset, nothing shared between
// launches, safe under CUDA-graph replay and concurrent streams).  The 16-byte
// response lands in shared memory through the async proxy and completes a
// transaction count of 16 bytes on `bar`.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void clc_try_cancel(void* resp16, uint64_t* bar) {
  mbar_arrive_expect_tx(bar, 16);
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
          smem_u32(resp16)),
      "r"(smem_u32(bar))
      : "memory");
}

// The cancelled CTA's blockIdx.x, or -1 when no CTA was left to cancel (after
// which no further request may be issued).
__device__ __forceinline__ int64_t clc_cancelled_cta(const void* resp16) {
  uint32_t ok, x;
  asm volatile(
      "{\n\t.reg .b128 r;\n\t.reg .pred p;\n\t"
      "ld.shared.b128 r, [%2];\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t"
      "mov.u32 %1, 0;\n\t"
      "@p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r;\n\t}"
      : "=r"(ok), "=r"(x)
      : "r"(smem_u32(resp16))
      : "memory");
  return ok ? (int64_t)x : -1;
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

// Element copy global -> shared (LDGSTS), BYTES = 4, 8 or 16.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}

// The mbarrier receives one arrival when all of this thread's prior cp.async
// copies have landed (noinc: the arrival is one of the barrier's expected count).
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Bulk prefetch of [src, src + bytes) into L2 (no completion, no data returned).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

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

// Branch-free variant for the fused kernels, whose outputs do not depend on
// the sign of a zero geometry entry (exactness note, txb_kernels.cuh): every
// quotient takes the reciprocal + two-correction path unconditionally (a
// zero numerator gives +0), and ONE predicate per cell says whether all of
// them were in the range where that path is the correctly rounded quotient
// (det and every nonzero numerator in [2^-500, 2^500], as DetDivider).  The
// caller redoes an unsafe cell with affine_inverse (rare: cells whose edge
// vectors span more than ~2^200 in scale).  No per-quotient branches: the
// nine chains interleave freely (the per-quotient branches serialised them).
#ifndef TXB_DD_RECIPROCAL
#define TXB_DD_RECIPROCAL 1
#endif
__device__ __forceinline__ bool dd_range_bad(double x) {
#ifdef TXB_DIAG_NO_NUM_CHECK  // diagnostic builds only (unsafe): what the per-numerator test costs
  return false;
#endif
  const unsigned hi = (unsigned)__double2hiint(x) & 0x7fffffffu, lo = (unsigned)__double2loint(x);
  return (hi - 0x20B00000u > 0x3E800000u) & ((hi | lo) != 0u);
}

// The reference's cofactor numerators (numpy's expression order, as
// affine_inverse) and det.
template <int D>
__device__ __forceinline__ void affine_numerators(const double (&X)[D + 1][D], double (&num)[D * D], double& det) {
  double m[D][D];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int i = 0; i < D; ++i) m[i][k] = __dsub_rn(X[k + 1][i], X[0][i]);
  if constexpr (D == 2) {
    const double a = m[0][0], b = m[0][1], c = m[1][0], e = m[1][1];
    det = __dsub_rn(__dmul_rn(a, e), __dmul_rn(b, c));
    num[0] = e;
    num[1] = -b;
    num[2] = -c;
    num[3] = a;
  } else {
    num[0] = __dsub_rn(__dmul_rn(m[1][1], m[2][2]), __dmul_rn(m[1][2], m[2][1]));
    num[3] = __dsub_rn(__dmul_rn(m[1][2], m[2][0]), __dmul_rn(m[1][0], m[2][2]));
    num[6] = __dsub_rn(__dmul_rn(m[1][0], m[2][1]), __dmul_rn(m[1][1], m[2][0]));
    det = __dadd_rn(__dadd_rn(__dmul_rn(m[0][0], num[0]), __dmul_rn(m[0][1], num[3])), __dmul_rn(m[0][2], num[6]));
    num[1] = __dsub_rn(__dmul_rn(m[0][2], m[2][1]), __dmul_rn(m[0][1], m[2][2]));
    num[4] = __dsub_rn(__dmul_rn(m[0][0], m[2][2]), __dmul_rn(m[0][2], m[2][0]));
    num[7] = __dsub_rn(__dmul_rn(m[0][1], m[2][0]), __dmul_rn(m[0][0], m[2][1]));
    num[2] = __dsub_rn(__dmul_rn(m[0][1], m[1][2]), __dmul_rn(m[0][2], m[1][1]));
    num[5] = __dsub_rn(__dmul_rn(m[0][2], m[1][0]), __dmul_rn(m[0][0], m[1][2]));
    num[8] = __dsub_rn(__dmul_rn(m[0][0], m[1][1]), __dmul_rn(m[0][1], m[1][0]));
  }
}

// EXACT_ZERO: a zero numerator returns itself (+-0, = numpy's x / det for
// det > 0) instead of +0 -- for callers that can see the sign of a zero
// geometry entry (the run-time compiled user forms); then every accepted cell
// is bit-identical to affine_inverse.
template <int D, bool EXACT_ZERO = false>
__device__ __forceinline__ bool affine_inverse_fast(const double (&X)[D + 1][D], double (&inv)[D * D], double& det) {
  double num[D * D];
  affine_numerators<D>(X, num, det);
  // det > 0 in range: the signed high word within [2^-500, 2^500]
  bool bad = ((unsigned)__double2hiint(det) - 0x20B00000u) > 0x3E800000u;
#if TXB_DD_RECIPROCAL
  // 1/det as y + yl (|yl| <= ulp(y)/2, the pair ~2^-104 relative): q0 =
  // RN(x y + RN(x yl)) is within ~0.5 ulp of x/det, so ONE residual
  // correction with y = RN(1/det) is correctly rounded (Markstein: q within
  // one ulp, y within half an ulp of 1/det) -- 4 operations per quotient.
  const double y = __drcp_rn(det);
  const double yl = __dmul_rn(__fma_rn(-det, y, 1.0), y);
#pragma unroll
  for (int i = 0; i < D * D; ++i) {
    const double x = num[i];
    bad |= dd_range_bad(x);
    const double q0 = __fma_rn(x, y, __dmul_rn(x, yl));
    const double q = __fma_rn(__fma_rn(-q0, det, x), y, q0);
    inv[i] = (EXACT_ZERO && x == 0.0) ? x : q;
  }
#else
  const double y = __drcp_rn(det);
#pragma unroll
  for (int i = 0; i < D * D; ++i) {
    const double x = num[i];
    bad |= dd_range_bad(x);
    const double q0 = __dmul_rn(x, y);
    const double q1 = __fma_rn(__fma_rn(-q0, det, x), y, q0);
    const double q = __fma_rn(__fma_rn(-q1, det, x), y, q1);
    inv[i] = (EXACT_ZERO && x == 0.0) ? x : q;
  }
#endif
  return !bad;
}

// float32 runs (the reference computes float64 geometry and casts it,
// executor._device_arrays): only float32(RN64(x / det)) is needed.  With
// y = RN(1/det) and q = RN(x y), |q - x/det| <= 2 ulp and so |q - RN64(x/det)|
// <= 3 ulp (bit-pattern distance, det and x/det in range).  float32 rounding of
// a double only changes across a float32 rounding midpoint (low 29 mantissa
// bits 0x10000000); when no midpoint lies within 8 ulp of q, float32(q) =
// float32(RN64(x/det)).  One product per quotient instead of the four of the
// correctly rounded double path.  The cell is rejected (the caller redoes it
// exactly) if det leaves [2^-500, 2^500], a nonzero quotient leaves the
// float32-normal range [2^-125, 2^127) or lies near a midpoint (~3e-7 of
// cells).  A zero numerator gives x * y = x: the sign of a zero is kept.
template <int D>
__device__ __forceinline__ bool affine_inverse_fast32(const double (&X)[D + 1][D], float (&inv)[D * D], double& det) {
  double num[D * D];
  affine_numerators<D>(X, num, det);
  bool bad = ((unsigned)__double2hiint(det) - 0x20B00000u) > 0x3E800000u;
  const double y = __drcp_rn(det);
#pragma unroll
  for (int i = 0; i < D * D; ++i) {
    const double x = num[i];
    const double q = __dmul_rn(x, y);
    const unsigned hi = (unsigned)__double2hiint(q) & 0x7fffffffu, lo = (unsigned)__double2loint(q);
    const bool near_mid = ((lo & 0x1FFFFFFFu) - 0x0FFFFFF8u) < 17u;
    const bool out_of_range = (hi - 0x38200000u) >= (0x47E00000u - 0x38200000u);
    bad |= (x != 0.0) & (near_mid | out_of_range);
    inv[i] = __double2float_rn(q);
  }
  return !bad;
}

// One cell's geometry in the run precision: the float64 quotients cast once
// (executor._device_arrays, executor.py:77-90) -- the branch-free paths above,
// affine_inverse for a rejected cell.  detd (float64) is for the orientation
// check.
template <typename T, int D, bool EXACT_ZERO = false>
__device__ __forceinline__ void cell_geometry(const double (&X)[D + 1][D], T (&J)[D * D], T& det, double& detd) {
  bool ok;
  if constexpr (sizeof(T) == 4) {
    float inv[D * D];
    ok = affine_inverse_fast32<D>(X, inv, detd);
#pragma unroll
    for (int i = 0; i < D * D; ++i) J[i] = (T)inv[i];
  } else {
    double inv[D * D];
    ok = affine_inverse_fast<D, EXACT_ZERO>(X, inv, detd);
#pragma unroll
    for (int i = 0; i < D * D; ++i) J[i] = (T)inv[i];
  }
  if (!ok) {
    double inv[D * D];
    affine_inverse<D>(X, inv, detd);
#pragma unroll
    for (int i = 0; i < D * D; ++i) J[i] = (T)inv[i];
  }
  det = (T)detd;
}

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ constexpr int make_odd(int x) { return (x & 1) ? x : x + 1; }

}  // namespace txb
