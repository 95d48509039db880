// txb_jit_prelude.cuh — the types a user-physics source string is written
// against (the reference's string-injection interface, txfem/physics.py:110-112:
// "each f1 is a function of (u, gradU, a, gradA, comp) returning a d-vector").
//
// The generated translation unit defines `real` (float or double) and
// TXB_DIM before including this file.  `realv` is the d-vector of the
// reference's OpenCL text (double2/double3 there): components .x .y (.z),
// component-wise + - and scaling by a scalar, each operation rounded on its
// own (the unit is compiled with -fmad=false, like the reference's
// -ffp-contract=off), so a user f1 evaluates exactly as numpy's f1_many does.
#pragma once

struct realv {
#if TXB_DIM == 2
  real x, y;
#else
  real x, y, z;
#endif
  __device__ realv() {}
  __device__ explicit realv(real s) {
    x = s;
    y = s;
#if TXB_DIM == 3
    z = s;
#endif
  }
  __device__ real& operator[](int i) { return (&x)[i]; }
  __device__ const real& operator[](int i) const { return (&x)[i]; }
};

#define TXB_REALV_EACH(k) for (int k = 0; k < TXB_DIM; ++k)

__device__ inline realv operator+(const realv& a, const realv& b) {
  realv r;
  TXB_REALV_EACH(k) r[k] = a[k] + b[k];
  return r;
}
__device__ inline realv operator-(const realv& a, const realv& b) {
  realv r;
  TXB_REALV_EACH(k) r[k] = a[k] - b[k];
  return r;
}
__device__ inline realv operator-(const realv& a) {
  realv r;
  TXB_REALV_EACH(k) r[k] = -a[k];
  return r;
}
__device__ inline realv operator*(const realv& a, const realv& b) {
  realv r;
  TXB_REALV_EACH(k) r[k] = a[k] * b[k];
  return r;
}
__device__ inline realv operator*(real s, const realv& a) {
  realv r;
  TXB_REALV_EACH(k) r[k] = s * a[k];
  return r;
}
__device__ inline realv operator*(const realv& a, real s) {
  realv r;
  TXB_REALV_EACH(k) r[k] = a[k] * s;
  return r;
}
__device__ inline realv operator/(const realv& a, real s) {
  realv r;
  TXB_REALV_EACH(k) r[k] = a[k] / s;
  return r;
}
__device__ inline realv& operator+=(realv& a, const realv& b) { return a = a + b; }
__device__ inline realv& operator-=(realv& a, const realv& b) { return a = a - b; }
__device__ inline realv& operator*=(realv& a, real s) { return a = a * s; }

// OpenCL's dot(): left-to-right sum of the component products.
__device__ inline real dot(const realv& a, const realv& b) {
  real s = a[0] * b[0];
  for (int k = 1; k < TXB_DIM; ++k) s = s + a[k] * b[k];
  return s;
}
