// Deterministic FP32 arithmetic of the sweep-v1 spec (docs/SWEEP_V1.md §2).
//
// Every function here is built only from IEEE-754 correctly-rounded
// operations (add, mul, fmaf, div, sqrt, rint, floor) and exact integer bit
// manipulation, evaluated in a fixed order.  The TU is compiled with
// --fmad=false so that no multiply-add is contracted behind our back; every
// FMA is written out as fmaf().  The consequence is that the CPU oracle
// (oracle/sweep_oracle.c, gcc -ffp-contract=off) reproduces every score bit
// for bit, which is what makes argmax / diversity / ranking decisions
// bit-exact between GPU and oracle.
//
// Accuracy against the reference's FP64 glibc exp/log1p (dock.cpp:23, :79):
// exp < 1e-8 rel (Taylor-7 after Cody-Waite reduction), log1p ~1.3e-7 rel
// (degree-9 polynomial in FP32), sin/cos < 1e-9 abs on |x| <= pi/2.
#pragma once
#include <cuda_runtime.h>

namespace vs {

// e^x for x <= 0; 0 below -87 (e^-87 < 1.7e-38).
__device__ __forceinline__ float det_exp_neg(float x) {
  if (x < -87.0f) return 0.0f;
  // k = rint(x log2 e) by the 1.5*2^23 shifter (same value as rintf, no F2I)
  const float sh = __fadd_rn(x * 1.44269504f, 12582912.0f);
  const float k = sh - 12582912.0f;
  float r = fmaf(k, -0.693145752f, x);
  r = fmaf(k, -1.42860677e-06f, r);
  float p = 1.98412698e-04f;
  p = fmaf(p, r, 1.38888889e-03f);
  p = fmaf(p, r, 8.33333333e-03f);
  p = fmaf(p, r, 4.16666667e-02f);
  p = fmaf(p, r, 1.66666667e-01f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const float s = __int_as_float((__float_as_int(sh) - 0x4B400000 + 127) << 23);
  return p * s;
}

// log(1 + u) for u in [0, 1]: u * P9(u), P9 a degree-9 fit of log1p(u)/u
// (rel. error ~1.3e-7 in FP32 Horner; no division).
__device__ __forceinline__ float det_log1p01(float u) {
  float p = -0x1.b5963cp-9f;
  p = fmaf(p, u, 0x1.4c35fap-6f);
  p = fmaf(p, u, -0x1.d92392p-5f);
  p = fmaf(p, u, 0x1.b59fa2p-4f);
  p = fmaf(p, u, -0x1.3a6dfep-3f);
  p = fmaf(p, u, 0x1.934c92p-3f);
  p = fmaf(p, u, -0x1.ff203ap-3f);
  p = fmaf(p, u, 0x1.554d4ep-2f);
  p = fmaf(p, u, -0x1.ffffc6p-2f);
  p = fmaf(p, u, 1.0f);
  return u * p;
}

// softplus(z) = log1p(exp z) (dock.cpp:23); z > 30 -> z; z < -30 -> 0
// (contribution < 1e-13, the spec's skip rule).
// Branch-free: the core is evaluated on z clamped to [-30, 30] (where it
// equals the unclamped core and exp_neg's underflow guard cannot fire) and
// the two tails are selected afterwards, so warps whose lanes straddle the
// tails do not diverge.
__device__ __forceinline__ float det_softplus(float z) {
  const float zc = fminf(fmaxf(z, -30.0f), 30.0f);
  const float a = -fabsf(zc);
  const float sh = __fadd_rn(a * 1.44269504f, 12582912.0f);
  const float k = sh - 12582912.0f;
  float r = fmaf(k, -0.693145752f, a);
  r = fmaf(k, -1.42860677e-06f, r);
  float p = 1.98412698e-04f;
  p = fmaf(p, r, 1.38888889e-03f);
  p = fmaf(p, r, 8.33333333e-03f);
  p = fmaf(p, r, 4.16666667e-02f);
  p = fmaf(p, r, 1.66666667e-01f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const float u = p * __int_as_float((__float_as_int(sh) - 0x4B400000 + 127) << 23);
  const float core = fmaxf(zc, 0.0f) + det_log1p01(u);
  return z > 30.0f ? z : (z < -30.0f ? 0.0f : core);
}

// sin and cos for |x| <= ~1.6 (half torsion angles).
__device__ __forceinline__ void det_sincos(float x, float* s, float* c) {
  const float x2 = x * x;
  float p = 1.60590438e-10f;
  p = fmaf(p, x2, -2.50521084e-08f);
  p = fmaf(p, x2, 2.75573192e-06f);
  p = fmaf(p, x2, -1.98412698e-04f);
  p = fmaf(p, x2, 8.33333333e-03f);
  p = fmaf(p, x2, -1.66666667e-01f);
  *s = fmaf(x * x2, p, x);
  float q = -1.14707456e-11f;
  q = fmaf(q, x2, 2.08767570e-09f);
  q = fmaf(q, x2, -2.75573192e-07f);
  q = fmaf(q, x2, 2.48015873e-05f);
  q = fmaf(q, x2, -1.38888889e-03f);
  q = fmaf(q, x2, 4.16666667e-02f);
  q = fmaf(q, x2, -0.5f);
  *c = fmaf(q, x2, 1.0f);
}

__device__ __forceinline__ float det_norm2(float x, float y, float z) {
  return fmaf(z, z, fmaf(y, y, x * x));
}

struct Mat3 {
  float m00, m01, m02, m10, m11, m12, m20, m21, m22;
};

// Rotation matrix of a (unit) quaternion (w, x, y, z); same map as
// Quat::rotate (geom.hpp:171-176) for unit q.
__device__ __forceinline__ Mat3 det_quat_mat(float w, float x, float y, float z) {
  const float xx = x * x, yy = y * y, zz = z * z;
  const float xy = x * y, xz = x * z, yz = y * z;
  const float wx = w * x, wy = w * y, wz = w * z;
  Mat3 R;
  R.m00 = 1.0f - 2.0f * (yy + zz);
  R.m01 = 2.0f * (xy - wz);
  R.m02 = 2.0f * (xz + wy);
  R.m10 = 2.0f * (xy + wz);
  R.m11 = 1.0f - 2.0f * (xx + zz);
  R.m12 = 2.0f * (yz - wx);
  R.m20 = 2.0f * (xz - wy);
  R.m21 = 2.0f * (yz + wx);
  R.m22 = 1.0f - 2.0f * (xx + yy);
  return R;
}

// out = R v + t
__device__ __forceinline__ void det_apply(const Mat3& R, float vx, float vy, float vz,
                                          float tx, float ty, float tz, float* ox,
                                          float* oy, float* oz) {
  *ox = fmaf(R.m00, vx, fmaf(R.m01, vy, fmaf(R.m02, vz, tx)));
  *oy = fmaf(R.m10, vx, fmaf(R.m11, vy, fmaf(R.m12, vz, ty)));
  *oz = fmaf(R.m20, vx, fmaf(R.m21, vy, fmaf(R.m22, vz, tz)));
}

// q / |q| (Quat::normalized, geom.hpp:167-170) as q * (1 / |q|)
__device__ __forceinline__ void det_quat_normalize(float* w, float* x, float* y, float* z) {
  const float inv = 1.0f / sqrtf(fmaf(*z, *z, fmaf(*y, *y, fmaf(*x, *x, (*w) * (*w)))));
  *w = *w * inv;
  *x = *x * inv;
  *y = *y * inv;
  *z = *z * inv;
}

// Hamilton product r (x) q
__device__ __forceinline__ void det_quat_mul(float rw, float rx, float ry, float rz, float qw,
                                             float qx, float qy, float qz, float* ow,
                                             float* ox, float* oy, float* oz) {
  *ow = fmaf(rz, -qz, fmaf(ry, -qy, fmaf(rx, -qx, rw * qw)));
  *ox = fmaf(rz, -qy, fmaf(ry, qz, fmaf(rx, qw, rw * qx)));
  *oy = fmaf(rz, qx, fmaf(ry, qw, fmaf(rx, -qz, rw * qy)));
  *oz = fmaf(rz, qw, fmaf(ry, -qx, fmaf(rx, qy, rw * qz)));
}

// Rotation of one torsion step (dock.cpp:57-59): axis from o to b, angle th.
__device__ __forceinline__ Mat3 det_torsion_mat(float ox, float oy, float oz, float bx, float by,
                                                float bz, float th) {
  const float dx = bx - ox, dy = by - oy, dz = bz - oz;
  const float n = sqrtf(det_norm2(dx, dy, dz));
  float ux = 0.0f, uy = 0.0f, uz = 0.0f;
  if (n > 0.0f) {
    ux = dx / n;
    uy = dy / n;
    uz = dz / n;
  }
  float s, c;
  det_sincos(0.5f * th, &s, &c);
  return det_quat_mat(c, ux * s, uy * s, uz * s);
}


// ------------------------------------------------------- FP64 geometry --
// Pose geometry (torsion chain, rigid transform, pair differences) is FP64:
// an FP32 chain accumulates ~1e-5 A of error over 8 nested torsions, which
// the steep clash ramp (10/A) turns into >1e-5 score error on
// ill-conditioned poses.  Transcendentals stay FP32.

// sin and cos for |x| <= ~1.6, Taylor to x^21 / x^22 (< 2e-18 truncation).
__device__ __forceinline__ void det_sincos_d(double x, double* s, double* c) {
  const double x2 = x * x;
  double p = 0x1.71b8ef6dcf572p-66;
  p = fma(p, x2, -0x1.2f49b46814157p-57);
  p = fma(p, x2, 0x1.952c77030ad4ap-49);
  p = fma(p, x2, -0x1.ae7f3e733b81fp-41);
  p = fma(p, x2, 0x1.6124613a86d09p-33);
  p = fma(p, x2, -0x1.ae64567f544e4p-26);
  p = fma(p, x2, 0x1.71de3a556c734p-19);
  p = fma(p, x2, -0x1.a01a01a01a01ap-13);
  p = fma(p, x2, 0x1.1111111111111p-7);
  p = fma(p, x2, -0x1.5555555555555p-3);
  *s = fma(x * x2, p, x);
  double q = -0x1.0ce396db7f853p-70;
  q = fma(q, x2, 0x1.e542ba4020225p-62);
  q = fma(q, x2, -0x1.6827863b97d97p-53);
  q = fma(q, x2, 0x1.ae7f3e733b81fp-45);
  q = fma(q, x2, -0x1.93974a8c07c9dp-37);
  q = fma(q, x2, 0x1.1eed8eff8d898p-29);
  q = fma(q, x2, -0x1.27e4fb7789f5cp-22);
  q = fma(q, x2, 0x1.a01a01a01a01ap-16);
  q = fma(q, x2, -0x1.6c16c16c16c17p-10);
  q = fma(q, x2, 0x1.5555555555555p-5);
  q = fma(q, x2, -0.5);
  *c = fma(q, x2, 1.0);
}

__device__ __forceinline__ double det_norm2_d(double x, double y, double z) {
  return fma(z, z, fma(y, y, x * x));
}

struct Mat3d {
  double m00, m01, m02, m10, m11, m12, m20, m21, m22;
};

__device__ __forceinline__ Mat3d det_quat_mat_d(double w, double x, double y, double z) {
  const double xx = x * x, yy = y * y, zz = z * z;
  const double xy = x * y, xz = x * z, yz = y * z;
  const double wx = w * x, wy = w * y, wz = w * z;
  Mat3d R;
  R.m00 = 1.0 - 2.0 * (yy + zz);
  R.m01 = 2.0 * (xy - wz);
  R.m02 = 2.0 * (xz + wy);
  R.m10 = 2.0 * (xy + wz);
  R.m11 = 1.0 - 2.0 * (xx + zz);
  R.m12 = 2.0 * (yz - wx);
  R.m20 = 2.0 * (xz - wy);
  R.m21 = 2.0 * (yz + wx);
  R.m22 = 1.0 - 2.0 * (xx + yy);
  return R;
}

__device__ __forceinline__ void det_apply_d(const Mat3d& R, double vx, double vy, double vz,
                                            double tx, double ty, double tz, double* ox,
                                            double* oy, double* oz) {
  *ox = fma(R.m00, vx, fma(R.m01, vy, fma(R.m02, vz, tx)));
  *oy = fma(R.m10, vx, fma(R.m11, vy, fma(R.m12, vz, ty)));
  *oz = fma(R.m20, vx, fma(R.m21, vy, fma(R.m22, vz, tz)));
}

// Rigid rotation of an FP32 pose quaternion, normalized in FP64 as
// Quat::normalized (geom.hpp:167-170) does.
__device__ __forceinline__ Mat3d det_pose_mat_d(float qw, float qx, float qy, float qz) {
  double w = qw, x = qx, y = qy, z = qz;
  const double inv = 1.0 / sqrt(fma(z, z, fma(y, y, fma(x, x, w * w))));
  return det_quat_mat_d(w * inv, x * inv, y * inv, z * inv);
}

// One torsion step (dock.cpp:57-59) in FP64: axis o -> b with unit vector
// (b - o) * inv_len (inv_len = 1 / |axis| of the conformer), FP32 angle th.
__device__ __forceinline__ Mat3d det_torsion_mat_d(double ox, double oy, double oz, double bx,
                                                   double by, double bz, float th,
                                                   double inv_len) {
  const double ux = (bx - ox) * inv_len, uy = (by - oy) * inv_len, uz = (bz - oz) * inv_len;
  double s, c;
  det_sincos_d(0.5 * static_cast<double>(th), &s, &c);
  return det_quat_mat_d(c, ux * s, uy * s, uz * s);
}

__device__ __forceinline__ float det_lerp(float a, float b, float t) { return fmaf(t, b - a, a); }

// float -> u32 whose unsigned order is the float order
__device__ __forceinline__ unsigned int det_orderable(float f) {
  const unsigned int b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

}  // namespace vs
