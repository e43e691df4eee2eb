// FP64 small-matrix math for the per-Gaussian preprocess and chain-rule kernels.
//
// The binning preprocess (rasterizer.cpp:24-99 cull + tile rectangles,
// voxelizer.cpp:60-80 brick ranges) must reproduce the reference's integer
// tile lists bit for bit. Every function here therefore evaluates the same
// sequence of IEEE double operations as the CPU restatement in
// oracle/splatct_oracle.cpp (products as left-to-right sums over k, Eigen's
// cofactor determinant/inverse), and the translation unit that uses them for
// binning is compiled with -fmad=false so no multiply-add is fused.
#pragma once

#include <cuda_runtime.h>

namespace sct {

struct dM3 {
  double m[3][3];
};
struct dM2 {
  double m[2][2];
};
struct dV3 {
  double v[3];
};

// FP64 reciprocal and square roots for values that feed no binning decision
// (the K5 item chain, K1's record fields): the MUFU seed (rcp / rsqrt
// .approx.ftz.f64, ~2^-22 relative) and two Newton steps (quadratic: < 2^-52,
// within an ulp or two of the correctly rounded result). The IEEE-rounded
// division and square root are subroutine calls of ~30 instructions each with
// a slow path. Explicit fma() calls, so -fmad=false translation units keep
// them. SCT_FASTDIV=0 restores the IEEE operations.
#ifndef SCT_FASTDIV
#define SCT_FASTDIV 1
#endif
__device__ __forceinline__ double d_fast_rcp(double x) {
#if SCT_FASTDIV
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}
// 1 / sqrt(x) for x > 0
__device__ __forceinline__ double d_fast_rsqrt(double x) {
#if SCT_FASTDIV
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
#else
  return 1.0 / sqrt(x);
#endif
}
// sqrt(x) for x >= 0 (0 -> 0; negative or NaN -> NaN as sqrt)
__device__ __forceinline__ double d_fast_sqrt(double x) {
#if SCT_FASTDIV
  if (!(x > 0.0)) return x == 0.0 ? 0.0 : sqrt(x);
  const double y = d_fast_rsqrt(x);
  const double r = x * y;
  return fma(fma(-r, r, x), 0.5 * y, r);  // one Newton correction of the root
#else
  return sqrt(x);
#endif
}

__device__ __forceinline__ dM3 d_zero3() {
  dM3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = 0.0;
  return r;
}
__device__ __forceinline__ dM3 d_mul(const dM3& a, const dM3& b) {
  dM3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
  return r;
}
__device__ __forceinline__ dM3 d_mul_bt(const dM3& a, const dM3& b) {  // a * b^T
  dM3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][0] * b.m[j][0] + a.m[i][1] * b.m[j][1] + a.m[i][2] * b.m[j][2];
  return r;
}
__device__ __forceinline__ dM3 d_mul_at(const dM3& a, const dM3& b) {  // a^T * b
  dM3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[0][i] * b.m[0][j] + a.m[1][i] * b.m[1][j] + a.m[2][i] * b.m[2][j];
  return r;
}
__device__ __forceinline__ dM3 d_add_t(const dM3& a) {  // a + a^T
  dM3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] + a.m[j][i];
  return r;
}
__device__ __forceinline__ double d_det3(const dM3& a) {
  return a.m[0][0] * (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) -
         a.m[0][1] * (a.m[1][0] * a.m[2][2] - a.m[1][2] * a.m[2][0]) +
         a.m[0][2] * (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]);
}
__device__ __forceinline__ dM3 d_inv3(const dM3& a) {
  dM3 c;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      c.m[i][j] = a.m[i1][j1] * a.m[i2][j2] - a.m[i1][j2] * a.m[i2][j1];
    }
  const double det = c.m[0][0] * a.m[0][0] + c.m[1][0] * a.m[1][0] + c.m[2][0] * a.m[2][0];
  const double inv = 1.0 / det;
  dM3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = c.m[j][i] * inv;
  return r;
}
__device__ __forceinline__ double d_det2(const dM2& a) { return a.m[0][0] * a.m[1][1] - a.m[1][0] * a.m[0][1]; }
__device__ __forceinline__ dM2 d_inv2(const dM2& a) {
  const double inv = 1.0 / d_det2(a);
  dM2 r;
  r.m[0][0] = a.m[1][1] * inv;
  r.m[1][0] = -a.m[1][0] * inv;
  r.m[0][1] = -a.m[0][1] * inv;
  r.m[1][1] = a.m[0][0] * inv;
  return r;
}

// gaussian_cloud.cpp:9-36 activations
__device__ __forceinline__ double d_act_density(double raw) { return raw > 30.0 ? raw : log1p(exp(raw)); }
__device__ __forceinline__ double d_act_density_grad(double raw) { return 1.0 / (1.0 + exp(-raw)); }

// gaussian_cloud.cpp:38-46 (q / sqrt(squaredNorm))
__device__ __forceinline__ dM3 d_rotation_matrix(const double qr[4]) {
  const double n2 = qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3];
  const double n = sqrt(n2);
  const double w = qr[0] / n, x = qr[1] / n, y = qr[2] / n, z = qr[3] / n;
  dM3 r;
  r.m[0][0] = 1 - 2 * (y * y + z * z);
  r.m[0][1] = 2 * (x * y - w * z);
  r.m[0][2] = 2 * (x * z + w * y);
  r.m[1][0] = 2 * (x * y + w * z);
  r.m[1][1] = 1 - 2 * (x * x + z * z);
  r.m[1][2] = 2 * (y * z - w * x);
  r.m[2][0] = 2 * (x * z - w * y);
  r.m[2][1] = 2 * (y * z + w * x);
  r.m[2][2] = 1 - 2 * (x * x + y * y);
  return r;
}

// Raw parameters of kernel i, widened to double.
struct dKernel {
  double p[3];
  double s[3];      // activated scale
  double sraw[3];
  double q[4];      // raw quaternion
  double rho_raw;
};
__device__ __forceinline__ dKernel d_load_kernel(const float* __restrict__ pos, const float* __restrict__ scale_raw,
                                                 const float* __restrict__ rot, const float* __restrict__ rho_raw,
                                                 long long i, double s_min) {
  dKernel k;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    k.p[a] = (double)pos[3 * i + a];
    k.sraw[a] = (double)scale_raw[3 * i + a];
    k.s[a] = s_min + exp(k.sraw[a]);  // act_scale
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) k.q[a] = (double)rot[4 * i + a];
  k.rho_raw = (double)rho_raw[i];
  return k;
}

// gaussian_cloud.cpp:134-138: (R * diag(s^2)) * R^T
__device__ __forceinline__ dM3 d_covariance(const dKernel& k, dM3* r_out = nullptr) {
  const dM3 r = d_rotation_matrix(k.q);
  double s2[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) s2[a] = k.s[a] * k.s[a];
  dM3 rd;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) rd.m[a][b] = r.m[a][b] * s2[b];
  if (r_out) *r_out = r;
  return d_mul_bt(rd, r);
}

}  // namespace sct
