// FP64 projection of one kernel into one view: rasterizer.cpp:24-99
// (project_impl + tile_range), evaluated in the oracle's exact operation
// order (see fp64_math.cuh).
#pragma once

#include "fp64_math.cuh"
#include "sct_internal.cuh"

namespace sct {

struct dProj {
  double cx, cy;
  dM2 cov;    // low-pass dilated 2D covariance
  dM2 conic;  // cov^-1
  double amp, mu, depth;
  // chain intermediates (rasterizer.cpp:10-22)
  double ps[3];
  dM3 a;          // J W
  dM3 sigma;      // 3D covariance
  dM3 sigma_ray;  // A Sigma A^T
  dM2 s2r;        // top-left block before low-pass
  double comp, rho, amp_pre;
};

// p: kernel position; sigma: its 3D covariance (d_covariance, bit-identical
// whether recomputed or read from the per-Gaussian prep buffer); rho: act_density.
__device__ __forceinline__ bool d_project(const double p[3], const dM3& sigma, double rho, const ViewParams& v,
                                          const DetParams& det, const RasterParams& rp, dProj& o) {
  double ps[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ps[i] = v.rot[3 * i + 0] * p[0] + v.rot[3 * i + 1] * p[1] + v.rot[3 * i + 2] * p[2];
    ps[i] = ps[i] + v.t[i];
  }
  const bool par = det.parallel != 0;  // parallel beam: affine map, no source plane
  if (!par && ps[2] < det.near_clip) return false;
  const double x = ps[0], y = ps[1], z = ps[2];
  const double n = sqrt(x * x + y * y + z * z);
  dM3 jac;
  if (par) {
    jac.m[0][0] = det.fx;
    jac.m[0][1] = 0.0;
    jac.m[0][2] = 0.0;
    jac.m[1][0] = 0.0;
    jac.m[1][1] = det.fy;
    jac.m[1][2] = 0.0;
    jac.m[2][0] = 0.0;
    jac.m[2][1] = 0.0;
    jac.m[2][2] = 1.0;
  } else {
    jac.m[0][0] = det.fx / z;
    jac.m[0][1] = 0.0;
    jac.m[0][2] = -det.fx * x / (z * z);
    jac.m[1][0] = 0.0;
    jac.m[1][1] = det.fy / z;
    jac.m[1][2] = -det.fy * y / (z * z);
    jac.m[2][0] = x / n;
    jac.m[2][1] = y / n;
    jac.m[2][2] = z / n;
  }
  dM3 W;
#pragma unroll
  for (int i = 0; i < 9; ++i) W.m[i / 3][i % 3] = v.rot[i];
  const dM3 a = d_mul(jac, W);
  const dM3 sigma_ray = d_mul_bt(d_mul(a, sigma), a);
  dM2 s2r;
  s2r.m[0][0] = sigma_ray.m[0][0];
  s2r.m[0][1] = sigma_ray.m[0][1];
  s2r.m[1][0] = sigma_ray.m[1][0];
  s2r.m[1][1] = sigma_ray.m[1][1];
  const double d3 = d_det3(sigma_ray);
  const double d2r = d_det2(s2r);
  const double mu = sqrt(2.0 * kPi * d3 / d2r);
  double amp = (rp.mode == SCT_MODE_RECTIFIED) ? mu * rho : rho;
  const double amp_pre = amp;
  dM2 s2 = s2r;
  s2.m[0][0] = s2r.m[0][0] + rp.eps2;
  s2.m[1][1] = s2r.m[1][1] + rp.eps2;
  double comp = 1.0;
  if (rp.dilation_compensation) {
    comp = sqrt(d2r / d_det2(s2));
    amp *= comp;
  }
  const double cx = par ? det.fx * x + det.cx : det.fx * x / z + det.cx;
  const double cy = par ? det.fy * y + det.cy : det.fy * y / z + det.cy;
  const double rx = rp.cull * sqrt(s2.m[0][0]);
  const double ry = rp.cull * sqrt(s2.m[1][1]);
  if (cx + rx < 0.0 || cx - rx > (double)det.w || cy + ry < 0.0 || cy - ry > (double)det.h) return false;
  o.cx = cx;
  o.cy = cy;
  o.cov = s2;
  o.conic = d_inv2(s2);
  o.amp = amp;
  o.mu = mu;
  o.depth = par ? z : n;
  o.ps[0] = x;
  o.ps[1] = y;
  o.ps[2] = z;
  o.a = a;
  o.sigma = sigma;
  o.sigma_ray = sigma_ray;
  o.s2r = s2r;
  o.comp = comp;
  o.rho = rho;
  o.amp_pre = amp_pre;
  return true;
}

// floor(v) -> int with the value clamped far outside any detector first, so
// that the conversion is defined for degenerate inputs (identical to the
// oracle's tile_range for every representable in-range value).
__device__ __forceinline__ int d_floor_int(double v) {
  double f = floor(v);
  f = fmin(fmax(f, -1073741824.0), 1073741824.0);
  return (int)f;
}

// rasterizer.cpp:89-99
__device__ __forceinline__ void d_tile_range(const dProj& g, const RasterParams& rp, int tiles_x, int tiles_y,
                                             int& tx0, int& tx1, int& ty0, int& ty1) {
  const double rx = rp.cull * sqrt(g.cov.m[0][0]);
  const double ry = rp.cull * sqrt(g.cov.m[1][1]);
  tx0 = max(0, d_floor_int((g.cx - rx) / (double)kTilePx));
  tx1 = min(tiles_x - 1, d_floor_int((g.cx + rx) / (double)kTilePx));
  ty0 = max(0, d_floor_int((g.cy - ry) / (double)kTilePx));
  ty1 = min(tiles_y - 1, d_floor_int((g.cy + ry) / (double)kTilePx));
}

}  // namespace sct
