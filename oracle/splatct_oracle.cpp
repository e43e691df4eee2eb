// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, called by, or shipped
// with the product path (paper_2405_20693_b200/). Only tests/, the smoke()
// checker in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
// arm may load this library.
//
// A line-by-line CPU restatement, in double precision, of the reference's
// differentiable hot path (R²-Gaussian "splatct", /root/reference/proj):
//   geometry.cpp:76-138        view_transform, detector_model, ray_space_point,
//                              local_jacobian, pixel_ray
//   gaussian_cloud.cpp:9-202   activations, rotation_matrix, covariance_at,
//                              density_at, rotation_matrix_jacobian,
//                              accumulate_covariance_param_grads,
//                              normalize_rotations
//   rasterizer.cpp:24-342      project_impl, tile_range, render,
//                              jacobian_derivative, render_backward
//   voxelizer.cpp:8-239        grid_for_extent, bin_kernels, precompute,
//                              voxelize, voxelize_backward,
//                              random_subvolume_spec
//   objectives.cpp:11-202      valid/adjoint filter, l1_loss, dssim_loss,
//                              tv3d_loss
//   trainer.cpp:34-36,144-163  lr_at, Adam::step
//   tests/helpers.hpp:18-160   test_scanner, random_cloud, ray_march_density,
//                              random_image (std::mt19937_64, libstdc++
//                              distributions: the same streams as the
//                              reference's own tests)
//
// The reference cannot be compiled here (Eigen3, libpng and vendor/ are absent,
// SURVEY.md §8c), so Eigen's fixed-size closed forms are restated by hand:
// 3x3 determinant by first-row cofactor expansion, 3x3 inverse by the
// cofactor/adjugate formula, 2x2 inverse by the adjugate, products as
// left-to-right sums over k. Build with -ffp-contract=off so that the FP64
// binning arithmetic (cull + tile rectangles, rasterizer.cpp:55-60,89-98 and
// voxelizer.cpp:60-80) is a fixed sequence of IEEE operations: the device
// preprocess kernels evaluate the very same sequence and are checked bit-exact
// against the tile lists produced here.
//
// OpenMP placement follows the reference exactly: parallel for
// schedule(static) only over tiles/bricks (rasterizer.cpp:136,216;
// voxelizer.cpp:115,158); projection/binning, reductions and per-kernel chain
// rules stay serial as in the reference.

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

namespace orc {

// ---------------------------------------------------------------- small math
struct V2 {
  double x = 0, y = 0;
};
struct V3 {
  double v[3] = {0, 0, 0};
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
struct M2 {
  double m[2][2] = {{0, 0}, {0, 0}};
};
struct M3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double& operator()(int i, int j) { return m[i][j]; }
  double operator()(int i, int j) const { return m[i][j]; }
};

static inline M3 mul(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
  return r;
}
// a * b^T
static inline M3 mul_bt(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[i][j] = a.m[i][0] * b.m[j][0] + a.m[i][1] * b.m[j][1] + a.m[i][2] * b.m[j][2];
  return r;
}
// a^T * b
static inline M3 mul_at(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[i][j] = a.m[0][i] * b.m[0][j] + a.m[1][i] * b.m[1][j] + a.m[2][i] * b.m[2][j];
  return r;
}
static inline M3 transpose(const M3& a) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
  return r;
}
static inline M3 add(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] + b.m[i][j];
  return r;
}
static inline M3 scale(const M3& a, double s) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] * s;
  return r;
}
static inline V3 mulv(const M3& a, const V3& p) {
  V3 r;
  for (int i = 0; i < 3; ++i) r[i] = a.m[i][0] * p[0] + a.m[i][1] * p[1] + a.m[i][2] * p[2];
  return r;
}
static inline V3 mulv_t(const M3& a, const V3& p) {  // a^T p
  V3 r;
  for (int i = 0; i < 3; ++i) r[i] = a.m[0][i] * p[0] + a.m[1][i] * p[1] + a.m[2][i] * p[2];
  return r;
}
static inline double det3(const M3& a) {
  return a.m[0][0] * (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) -
         a.m[0][1] * (a.m[1][0] * a.m[2][2] - a.m[1][2] * a.m[2][0]) +
         a.m[0][2] * (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]);
}
static inline M3 inv3(const M3& a) {
  // adjugate / det (Eigen compute_inverse_size3_helper: cofactors of column 0
  // give the determinant)
  M3 c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      c.m[i][j] = a.m[i1][j1] * a.m[i2][j2] - a.m[i1][j2] * a.m[i2][j1];
    }
  const double det = c.m[0][0] * a.m[0][0] + c.m[1][0] * a.m[1][0] + c.m[2][0] * a.m[2][0];
  const double inv = 1.0 / det;
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = c.m[j][i] * inv;
  return r;
}
static inline double det2(const M2& a) { return a.m[0][0] * a.m[1][1] - a.m[1][0] * a.m[0][1]; }
static inline M2 inv2(const M2& a) {
  const double inv = 1.0 / det2(a);
  M2 r;
  r.m[0][0] = a.m[1][1] * inv;
  r.m[1][0] = -a.m[1][0] * inv;
  r.m[0][1] = -a.m[0][1] * inv;
  r.m[1][1] = a.m[0][0] * inv;
  return r;
}
static inline double norm3(const V3& p) { return std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]); }

// ---------------------------------------------------------------- geometry
// geometry.hpp:12-31 ScannerConfig (angles passed per call)
struct Scanner {
  double l_so_mm = 8.0, l_sd_mm = 12.0;
  double det_size_mm[2] = {5.6, 5.6};
  int det_res_px[2] = {128, 128};
  double extent_min_mm[3] = {-1, -1, -1}, extent_max_mm[3] = {1, 1, 1};
  double near_clip_mm = 0.0;
  int parallel = 0;  // parallel-beam extension (not in the reference)
  double near_clip() const { return near_clip_mm > 0.0 ? near_clip_mm : 0.01 * l_so_mm; }
};
struct View {
  M3 rot;
  V3 t;
};
struct Det {
  double fx = 0, fy = 0, cx = 0, cy = 0;
  int w = 0, h = 0;
  double near = 0;
  bool parallel = false;
};

// geometry.cpp:76-86
static View view_transform(const Scanner& c, double theta) {
  const double s = std::sin(theta), co = std::cos(theta);
  View v;
  v.rot.m[0][0] = -s; v.rot.m[0][1] = co; v.rot.m[0][2] = 0.0;
  v.rot.m[1][0] = 0.0; v.rot.m[1][1] = 0.0; v.rot.m[1][2] = -1.0;
  v.rot.m[2][0] = -co; v.rot.m[2][1] = -s; v.rot.m[2][2] = 0.0;
  v.t[0] = 0.0; v.t[1] = 0.0; v.t[2] = c.l_so_mm;
  return v;
}
// geometry.cpp:88-98
static Det detector_model(const Scanner& c) {
  Det d;
  d.w = c.det_res_px[0];
  d.h = c.det_res_px[1];
  // parallel beam: orthographic, detector mm == scanner mm (no magnification)
  d.parallel = c.parallel != 0;
  d.fx = d.parallel ? d.w / c.det_size_mm[0] : c.l_sd_mm * d.w / c.det_size_mm[0];
  d.fy = d.parallel ? d.h / c.det_size_mm[1] : c.l_sd_mm * d.h / c.det_size_mm[1];
  d.cx = 0.5 * d.w;
  d.cy = 0.5 * d.h;
  d.near = c.near_clip();
  return d;
}
// geometry.cpp:105-109
static V3 ray_space_point(const Det& d, const V3& p) {
  V3 r;
  if (d.parallel) {  // affine map: phi(p) = (fx x + cx, fy y + cy, z)
    r[0] = d.fx * p[0] + d.cx;
    r[1] = d.fy * p[1] + d.cy;
    r[2] = p[2];
    return r;
  }
  r[0] = d.fx * p[0] / p[2] + d.cx;
  r[1] = d.fy * p[1] / p[2] + d.cy;
  r[2] = norm3(p);
  return r;
}
// geometry.cpp:111-123 (caller culls z < near first; rasterizer.cpp:28)
static M3 local_jacobian(const Det& d, const V3& p) {
  const double z = p[2], x = p[0], y = p[1];
  const double n = norm3(p);
  M3 j;
  if (d.parallel) {  // constant: diag(fx, fy, 1)
    j.m[0][0] = d.fx; j.m[0][1] = 0.0; j.m[0][2] = 0.0;
    j.m[1][0] = 0.0; j.m[1][1] = d.fy; j.m[1][2] = 0.0;
    j.m[2][0] = 0.0; j.m[2][1] = 0.0; j.m[2][2] = 1.0;
    return j;
  }
  j.m[0][0] = d.fx / z; j.m[0][1] = 0.0; j.m[0][2] = -d.fx * x / (z * z);
  j.m[1][0] = 0.0; j.m[1][1] = d.fy / z; j.m[1][2] = -d.fy * y / (z * z);
  j.m[2][0] = x / n; j.m[2][1] = y / n; j.m[2][2] = z / n;
  return j;
}

// ---------------------------------------------------------------- cloud
// gaussian_cloud.cpp:9-36
static double act_density(double raw) { return raw > 30.0 ? raw : std::log1p(std::exp(raw)); }
static double act_density_inv(double rho) {
  if (rho > 30.0) return rho;
  return rho + std::log1p(-std::exp(-rho));
}
static double act_density_grad(double raw) { return 1.0 / (1.0 + std::exp(-raw)); }
static double act_scale(double raw, double s_min) { return s_min + std::exp(raw); }
static double act_scale_inv(double s, double s_min) { return std::log(s - s_min); }
static double act_scale_grad(double raw) { return std::exp(raw); }

struct Cloud {  // gaussian_cloud.hpp:31-81 (raw arrays; adaptive stats)
  int m = 0;
  double s_min = 1e-4;
  const double* rho_raw = nullptr;
  const double* pos = nullptr;
  const double* scale_raw = nullptr;
  const double* rot = nullptr;
  double rho(int i) const { return act_density(rho_raw[i]); }
  V3 position(int i) const {
    V3 p;
    p[0] = pos[3 * i]; p[1] = pos[3 * i + 1]; p[2] = pos[3 * i + 2];
    return p;
  }
  V3 scalev(int i) const {
    V3 s;
    for (int k = 0; k < 3; ++k) s[k] = act_scale(scale_raw[3 * i + k], s_min);
    return s;
  }
};
struct Grads {  // CloudGrads, accumulate (+=)
  double* rho_raw;
  double* pos;
  double* scale_raw;
  double* rot;
};
struct Stats {  // adaptive-control statistics gaussian_cloud.hpp:74-77
  double* grad2d_norm_accum;
  int32_t* grad_count;
  double* grad3d_accum;
};

// gaussian_cloud.cpp:38-46 (normalized(): q / sqrt(squaredNorm))
static void normalize4(const double* q_raw, double q[4]) {
  const double n2 = q_raw[0] * q_raw[0] + q_raw[1] * q_raw[1] + q_raw[2] * q_raw[2] + q_raw[3] * q_raw[3];
  const double n = std::sqrt(n2);
  for (int k = 0; k < 4; ++k) q[k] = q_raw[k] / n;
}
static M3 rotation_matrix(const double* q_raw) {
  double q[4];
  normalize4(q_raw, q);
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  M3 r;
  r.m[0][0] = 1 - 2 * (y * y + z * z); r.m[0][1] = 2 * (x * y - w * z); r.m[0][2] = 2 * (x * z + w * y);
  r.m[1][0] = 2 * (x * y + w * z); r.m[1][1] = 1 - 2 * (x * x + z * z); r.m[1][2] = 2 * (y * z - w * x);
  r.m[2][0] = 2 * (x * z - w * y); r.m[2][1] = 2 * (y * z + w * x); r.m[2][2] = 1 - 2 * (x * x + y * y);
  return r;
}
// gaussian_cloud.cpp:134-138: R * diag(s^2) * R^T, evaluated (R*D) then *R^T
static M3 covariance_at(const Cloud& c, int i) {
  const M3 r = rotation_matrix(c.rot + 4 * i);
  const V3 s = c.scalev(i);
  double s2[3];
  for (int k = 0; k < 3; ++k) s2[k] = s[k] * s[k];
  M3 rd;
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < 3; ++k) rd.m[a][k] = r.m[a][k] * s2[k];
  return mul_bt(rd, r);
}
// gaussian_cloud.cpp:140-149
static double density_at(const Cloud& c, const V3& x) {
  double sum = 0.0;
  for (int i = 0; i < c.m; ++i) {
    V3 d;
    const V3 p = c.position(i);
    for (int k = 0; k < 3; ++k) d[k] = x[k] - p[k];
    const M3 q = inv3(covariance_at(c, i));
    const V3 qd = mulv(q, d);
    const double e = d[0] * qd[0] + d[1] * qd[1] + d[2] * qd[2];
    sum += c.rho(i) * std::exp(-0.5 * e);
  }
  return sum;
}
// gaussian_cloud.cpp:151-182
static std::array<M3, 4> rotation_matrix_jacobian(const double* q_raw) {
  const double nrm = std::sqrt(q_raw[0] * q_raw[0] + q_raw[1] * q_raw[1] + q_raw[2] * q_raw[2] + q_raw[3] * q_raw[3]);
  double q[4];
  for (int k = 0; k < 4; ++k) q[k] = q_raw[k] / nrm;
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  std::array<M3, 4> dn;
  const double d0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
  const double d1[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
  const double d2[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
  const double d3[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
  const double* src[4] = {d0, d1, d2, d3};
  for (int l = 0; l < 4; ++l)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) dn[l].m[a][b] = src[l][3 * a + b] * 2.0;
  std::array<M3, 4> out;
  for (int k = 0; k < 4; ++k) {
    M3 m;
    for (int l = 0; l < 4; ++l) {
      const double coeff = ((l == k ? 1.0 : 0.0) - q[l] * q[k]) / nrm;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m.m[a][b] += coeff * dn[l].m[a][b];
    }
    out[k] = m;
  }
  return out;
}
// gaussian_cloud.cpp:184-202
static void accumulate_covariance_param_grads(const Cloud& c, int i, const M3& g_sigma, Grads& g) {
  const M3 r = rotation_matrix(c.rot + 4 * i);
  const V3 s = c.scalev(i);
  M3 d;
  for (int k = 0; k < 3; ++k) d.m[k][k] = s[k] * s[k];
  const M3 g_r = mul(mul(add(g_sigma, transpose(g_sigma)), r), d);
  const M3 g_d = mul(mul_at(r, g_sigma), r);
  for (int k = 0; k < 3; ++k) {
    const double dL_ds = g_d.m[k][k] * 2.0 * s[k];
    g.scale_raw[3 * i + k] += dL_ds * act_scale_grad(c.scale_raw[3 * i + k]);
  }
  const auto dr = rotation_matrix_jacobian(c.rot + 4 * i);
  for (int k = 0; k < 4; ++k) {
    double sum = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) sum += g_r.m[a][b] * dr[k].m[a][b];
    g.rot[4 * i + k] += sum;
  }
}

// ---------------------------------------------------------------- rasterizer
constexpr int kTilePx = 16;   // common.hpp:24
constexpr int kTileVox = 8;   // common.hpp:25

struct RasterOptions {  // rasterizer.hpp:15-21
  int mode = 0;  // 0 rectified, 1 biased
  double lowpass_eps_px = 0.3;
  int dilation_compensation = 1;
  int freeze_jacobian = 0;
  double cull_mahalanobis = 3.0348542587702925;
};
struct Projected {  // rasterizer.hpp:24-32
  V2 center;
  M2 cov;
  M2 conic;
  double amplitude = 0, mu = 0, depth = 0;
  int kernel_index = -1;
};
struct Chain {  // rasterizer.cpp:10-22
  V3 p_s;
  M3 jac, a, sigma_ray;
  M2 sigma2_raw, sigma2;
  double mu = 1, comp = 1, rho = 0, amp_pre = 0;
};

// rasterizer.cpp:24-83
static bool project_impl(const Cloud& c, int i, const View& view, const Det& det,
                         const RasterOptions& o, Projected& out, Chain* ch) {
  const V3 p = c.position(i);
  V3 p_s = mulv(view.rot, p);
  for (int k = 0; k < 3; ++k) p_s[k] = p_s[k] + view.t[k];
  if (!det.parallel && p_s[2] < det.near) return false;  // no source plane for parallel rays

  const M3 jac = local_jacobian(det, p_s);
  const M3 a = mul(jac, view.rot);
  const M3 sigma = covariance_at(c, i);
  const M3 sigma_ray = mul_bt(mul(a, sigma), a);
  M2 s2r;
  s2r.m[0][0] = sigma_ray.m[0][0]; s2r.m[0][1] = sigma_ray.m[0][1];
  s2r.m[1][0] = sigma_ray.m[1][0]; s2r.m[1][1] = sigma_ray.m[1][1];

  const double d3 = det3(sigma_ray);
  const double d2r = det2(s2r);
  const double rho = c.rho(i);
  const double mu = std::sqrt(2.0 * M_PI * d3 / d2r);
  double amp = (o.mode == 0) ? mu * rho : rho;
  const double amp_pre = amp;

  const double eps2 = o.lowpass_eps_px * o.lowpass_eps_px;
  M2 s2 = s2r;
  s2.m[0][0] = s2r.m[0][0] + eps2;
  s2.m[1][1] = s2r.m[1][1] + eps2;
  double comp = 1.0;
  if (o.dilation_compensation) {
    comp = std::sqrt(d2r / det2(s2));
    amp *= comp;
  }
  const V3 rp = ray_space_point(det, p_s);
  const double rx = o.cull_mahalanobis * std::sqrt(s2.m[0][0]);
  const double ry = o.cull_mahalanobis * std::sqrt(s2.m[1][1]);
  if (rp[0] + rx < 0.0 || rp[0] - rx > det.w || rp[1] + ry < 0.0 || rp[1] - ry > det.h) return false;

  out.center.x = rp[0];
  out.center.y = rp[1];
  out.cov = s2;
  out.conic = inv2(s2);
  out.amplitude = amp;
  out.mu = mu;
  out.depth = rp[2];
  out.kernel_index = i;
  if (ch) {
    ch->p_s = p_s;
    ch->jac = jac;
    ch->a = a;
    ch->sigma_ray = sigma_ray;
    ch->sigma2_raw = s2r;
    ch->sigma2 = s2;
    ch->mu = mu;
    ch->comp = comp;
    ch->rho = rho;
    ch->amp_pre = amp_pre;
  }
  return true;
}

struct TileRange {
  int tx0, tx1, ty0, ty1;
};
// static_cast<int>(std::floor(v)) for every in-range value; clamped first so
// that degenerate (huge) footprints convert deterministically (the reference's
// cast is undefined there). The device kernels use the identical clamp.
static inline int floor_int(double v) {
  double f = std::floor(v);
  f = std::fmin(std::fmax(f, -1073741824.0), 1073741824.0);
  return static_cast<int>(f);
}
// rasterizer.cpp:89-99
static TileRange tile_range(const Projected& g, const RasterOptions& o, int tiles_x, int tiles_y) {
  const double rx = o.cull_mahalanobis * std::sqrt(g.cov.m[0][0]);
  const double ry = o.cull_mahalanobis * std::sqrt(g.cov.m[1][1]);
  TileRange r;
  r.tx0 = std::max(0, floor_int((g.center.x - rx) / kTilePx));
  r.tx1 = std::min(tiles_x - 1, floor_int((g.center.x + rx) / kTilePx));
  r.ty0 = std::max(0, floor_int((g.center.y - ry) / kTilePx));
  r.ty1 = std::min(tiles_y - 1, floor_int((g.center.y + ry) / kTilePx));
  return r;
}

struct Rendered {  // rasterizer.hpp:41-51
  int w = 0, h = 0, tiles_x = 0, tiles_y = 0;
  std::vector<double> image;
  std::vector<Projected> visible;
  std::vector<std::vector<int>> tile_visible;
};

// rasterizer.cpp:112-157
static Rendered* render(const Cloud& c, const Scanner& cfg, double theta, const RasterOptions& o) {
  const View view = view_transform(cfg, theta);
  const Det det = detector_model(cfg);
  auto* out = new Rendered();
  out->w = det.w;
  out->h = det.h;
  out->image.assign(static_cast<size_t>(det.w) * det.h, 0.0);
  out->tiles_x = (det.w + kTilePx - 1) / kTilePx;
  out->tiles_y = (det.h + kTilePx - 1) / kTilePx;
  out->tile_visible.resize(static_cast<size_t>(out->tiles_x) * out->tiles_y);
  out->visible.reserve(c.m);
  for (int i = 0; i < c.m; ++i) {  // serial, as in the reference
    Projected g;
    if (!project_impl(c, i, view, det, o, g, nullptr)) continue;
    const int vi = static_cast<int>(out->visible.size());
    out->visible.push_back(g);
    const TileRange r = tile_range(g, o, out->tiles_x, out->tiles_y);
    for (int ty = r.ty0; ty <= r.ty1; ++ty)
      for (int tx = r.tx0; tx <= r.tx1; ++tx)
        out->tile_visible[static_cast<size_t>(ty) * out->tiles_x + tx].push_back(vi);
  }
  const int n_tiles = static_cast<int>(out->tile_visible.size());
  Rendered& R = *out;
#pragma omp parallel for schedule(static)
  for (int t = 0; t < n_tiles; ++t) {
    const auto& list = R.tile_visible[t];
    if (list.empty()) continue;
    const int tx = t % R.tiles_x, ty = t / R.tiles_x;
    const int u0 = tx * kTilePx, u1 = std::min(u0 + kTilePx, det.w);
    const int v0 = ty * kTilePx, v1 = std::min(v0 + kTilePx, det.h);
    for (int v = v0; v < v1; ++v)
      for (int u = u0; u < u1; ++u) {
        const double xx = u + 0.5, xy = v + 0.5;
        double sum = 0.0;
        for (int vi : list) {
          const Projected& g = R.visible[vi];
          const double dx = xx - g.center.x, dy = xy - g.center.y;
          const double qx = g.conic.m[0][0] * dx + g.conic.m[0][1] * dy;
          const double qy = g.conic.m[1][0] * dx + g.conic.m[1][1] * dy;
          sum += g.amplitude * std::exp(-0.5 * (dx * qx + dy * qy));
        }
        R.image[static_cast<size_t>(v) * det.w + u] = sum;
      }
  }
  return out;
}

// rasterizer.cpp:162-191
static M3 jacobian_derivative(const Det& det, const V3& p, int c) {
  const double x = p[0], y = p[1], z = p[2];
  const double n = norm3(p);
  const double n3 = n * n * n;
  M3 d;
  if (det.parallel) return d;  // J is constant
  switch (c) {
    case 0:
      d.m[0][2] = -det.fx / (z * z);
      d.m[2][0] = 1.0 / n - x * x / n3;
      d.m[2][1] = -x * y / n3;
      d.m[2][2] = -x * z / n3;
      break;
    case 1:
      d.m[1][2] = -det.fy / (z * z);
      d.m[2][0] = -x * y / n3;
      d.m[2][1] = 1.0 / n - y * y / n3;
      d.m[2][2] = -y * z / n3;
      break;
    default:
      d.m[0][0] = -det.fx / (z * z);
      d.m[0][2] = 2.0 * det.fx * x / (z * z * z);
      d.m[1][1] = -det.fy / (z * z);
      d.m[1][2] = 2.0 * det.fy * y / (z * z * z);
      d.m[2][0] = -x * z / n3;
      d.m[2][1] = -y * z / n3;
      d.m[2][2] = 1.0 / n - z * z / n3;
      break;
  }
  return d;
}

struct Stat2 {
  double s0 = 0, s1[2] = {0, 0}, s2[3] = {0, 0, 0};  // xx yy xy
};

// Per-visible-kernel chain rule, rasterizer.cpp:262-341. Shared by
// render_backward and by the "from statistics" entry that lets tests feed
// device-produced tile statistics through the reference chain rule.
static void raster_chain(const Cloud& c, const View& view, const Det& det, const RasterOptions& o,
                         int i, const Stat2& s, Grads& grads, Stats* stats) {
  Projected pg;
  Chain ch;
  if (!project_impl(c, i, view, det, o, pg, &ch)) return;
  const M2 q = pg.conic;
  const double s1x = s.s1[0], s1y = s.s1[1];
  M2 s2;
  s2.m[0][0] = s.s2[0]; s2.m[0][1] = s.s2[2];
  s2.m[1][0] = s.s2[2]; s2.m[1][1] = s.s2[1];

  const double g_amp = s.s0;
  V2 g_center;
  g_center.x = pg.amplitude * (q.m[0][0] * s1x + q.m[0][1] * s1y);
  g_center.y = pg.amplitude * (q.m[1][0] * s1x + q.m[1][1] * s1y);
  M2 g_q;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) g_q.m[a][b] = -0.5 * pg.amplitude * s2.m[a][b];
  // g_sigma2 = -q * g_q * q
  M2 g_sigma2;
  {
    M2 t;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) t.m[a][b] = -q.m[a][0] * g_q.m[0][b] + -q.m[a][1] * g_q.m[1][b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) g_sigma2.m[a][b] = t.m[a][0] * q.m[0][b] + t.m[a][1] * q.m[1][b];
  }
  double g_amp_pre = g_amp;
  M2 g_sigma2_raw;
  if (o.dilation_compensation) {
    g_amp_pre = g_amp * ch.comp;
    const double g_comp = g_amp * ch.amp_pre;
    const M2 inv_raw = inv2(ch.sigma2_raw);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        g_sigma2_raw.m[a][b] += g_comp * 0.5 * ch.comp * inv_raw.m[a][b];
        g_sigma2.m[a][b] += g_comp * (-0.5) * ch.comp * q.m[a][b];
      }
  }
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) g_sigma2_raw.m[a][b] += g_sigma2.m[a][b];

  M3 g_sigma_ray;
  double g_rho = 0.0;
  if (o.mode == 0) {
    g_rho = g_amp_pre * ch.mu;
    const double g_mu = g_amp_pre * ch.rho;
    const M3 inv_ray = inv3(ch.sigma_ray);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) g_sigma_ray.m[a][b] += g_mu * 0.5 * ch.mu * inv_ray.m[a][b];
    const M2 inv_raw = inv2(ch.sigma2_raw);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) g_sigma2_raw.m[a][b] += g_mu * (-0.5) * ch.mu * inv_raw.m[a][b];
  } else {
    g_rho = g_amp_pre;
  }
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) g_sigma_ray.m[a][b] += g_sigma2_raw.m[a][b];

  const M3 sigma = covariance_at(c, i);
  const M3 g_a = mul(mul(add(g_sigma_ray, transpose(g_sigma_ray)), ch.a), sigma);
  const M3 g_sigma = mul(mul_at(ch.a, g_sigma_ray), ch.a);

  V3 g_ps;
  {
    const double zc = ch.p_s[2];
    const double d00 = det.parallel ? det.fx : det.fx / zc;
    const double d02 = det.parallel ? 0.0 : -det.fx * ch.p_s[0] / (zc * zc);
    const double d11 = det.parallel ? det.fy : det.fy / zc;
    const double d12 = det.parallel ? 0.0 : -det.fy * ch.p_s[1] / (zc * zc);
    g_ps[0] += d00 * g_center.x;
    g_ps[1] += d11 * g_center.y;
    g_ps[2] += d02 * g_center.x + d12 * g_center.y;
  }
  if (!o.freeze_jacobian) {
    const M3 g_jac = mul_bt(g_a, view.rot);
    for (int cc = 0; cc < 3; ++cc) {
      const M3 dj = jacobian_derivative(det, ch.p_s, cc);
      double sum = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) sum += g_jac.m[a][b] * dj.m[a][b];
      g_ps[cc] += sum;
    }
  }
  const V3 g_pos = mulv_t(view.rot, g_ps);

  grads.rho_raw[i] += g_rho * act_density_grad(c.rho_raw[i]);
  for (int k = 0; k < 3; ++k) grads.pos[3 * i + k] += g_pos[k];
  accumulate_covariance_param_grads(c, i, g_sigma, grads);

  if (stats) {
    const double nx = g_center.x * 0.5 * det.w, ny = g_center.y * 0.5 * det.h;
    stats->grad2d_norm_accum[i] += std::sqrt(nx * nx + ny * ny);
    stats->grad_count[i] += 1;
    for (int k = 0; k < 3; ++k) stats->grad3d_accum[3 * i + k] += g_pos[k];
  }
}

// rasterizer.cpp:195-342
static void render_backward(const Cloud& c, const Scanner& cfg, double theta, const Rendered& fwd,
                            const double* dL, Grads& grads, const RasterOptions& o, Stats* stats) {
  const View view = view_transform(cfg, theta);
  const Det det = detector_model(cfg);
  const int n_tiles = static_cast<int>(fwd.tile_visible.size());
  const int n_vis = static_cast<int>(fwd.visible.size());
  std::vector<std::vector<Stat2>> scratch(n_tiles);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < n_tiles; ++t) {
    const auto& list = fwd.tile_visible[t];
    if (list.empty()) continue;
    scratch[t].resize(list.size());
    const int tx = t % fwd.tiles_x, ty = t / fwd.tiles_x;
    const int u0 = tx * kTilePx, u1 = std::min(u0 + kTilePx, det.w);
    const int v0 = ty * kTilePx, v1 = std::min(v0 + kTilePx, det.h);
    for (int v = v0; v < v1; ++v)
      for (int u = u0; u < u1; ++u) {
        const double g = dL[static_cast<size_t>(v) * det.w + u];
        if (g == 0.0) continue;
        const double xx = u + 0.5, xy = v + 0.5;
        for (size_t li = 0; li < list.size(); ++li) {
          const Projected& pg = fwd.visible[list[li]];
          const double dx = xx - pg.center.x, dy = xy - pg.center.y;
          const double qx = pg.conic.m[0][0] * dx + pg.conic.m[0][1] * dy;
          const double qy = pg.conic.m[1][0] * dx + pg.conic.m[1][1] * dy;
          const double ge = g * std::exp(-0.5 * (dx * qx + dy * qy));
          Stat2& s = scratch[t][li];
          s.s0 += ge;
          s.s1[0] += ge * dx;
          s.s1[1] += ge * dy;
          s.s2[0] += ge * dx * dx;
          s.s2[1] += ge * dy * dy;
          s.s2[2] += ge * dx * dy;
        }
      }
  }
  std::vector<Stat2> total(n_vis);
  for (int t = 0; t < n_tiles; ++t) {  // fixed-order reduction, serial
    const auto& list = fwd.tile_visible[t];
    for (size_t li = 0; li < list.size(); ++li) {
      const Stat2& s = scratch[t][li];
      Stat2& acc = total[list[li]];
      acc.s0 += s.s0;
      acc.s1[0] += s.s1[0];
      acc.s1[1] += s.s1[1];
      for (int k = 0; k < 3; ++k) acc.s2[k] += s.s2[k];
    }
  }
  for (int vi = 0; vi < n_vis; ++vi)  // serial chain rule
    raster_chain(c, view, det, o, fwd.visible[vi].kernel_index, total[vi], grads, stats);
}

// ---------------------------------------------------------------- voxelizer
struct Grid {  // voxelizer.hpp:13-24
  int dims[3] = {0, 0, 0};
  double origin[3] = {0, 0, 0};
  double spacing[3] = {1, 1, 1};
  V3 center(int x, int y, int z) const {
    V3 c;
    c[0] = origin[0] + (x + 0.5) * spacing[0];
    c[1] = origin[1] + (y + 0.5) * spacing[1];
    c[2] = origin[2] + (z + 0.5) * spacing[2];
    return c;
  }
};
struct Bins {
  int tiles[3] = {0, 0, 0};
  std::vector<std::vector<int>> kernels;
};
// voxelizer.cpp:52-88
static Bins bin_kernels(const Cloud& c, const Grid& g, double radius) {
  Bins b;
  for (int k = 0; k < 3; ++k) b.tiles[k] = (g.dims[k] + kTileVox - 1) / kTileVox;
  b.kernels.resize(static_cast<size_t>(b.tiles[0]) * b.tiles[1] * b.tiles[2]);
  for (int i = 0; i < c.m; ++i) {
    const M3 sigma = covariance_at(c, i);
    const V3 p = c.position(i);
    int lo[3], hi[3];
    bool empty = false;
    for (int k = 0; k < 3; ++k) {
      const double r = radius * std::sqrt(std::max(sigma.m[k][k], 0.0));
      const double a = (p[k] - r - g.origin[k]) / g.spacing[k];
      const double bb = (p[k] + r - g.origin[k]) / g.spacing[k];
      int v0 = floor_int(a);
      int v1 = floor_int(bb);
      v0 = std::max(v0, 0);
      v1 = std::min(v1, g.dims[k] - 1);
      if (v0 > v1) {
        empty = true;
        break;
      }
      lo[k] = v0 / kTileVox;
      hi[k] = v1 / kTileVox;
    }
    if (empty) continue;
    for (int tz = lo[2]; tz <= hi[2]; ++tz)
      for (int ty = lo[1]; ty <= hi[1]; ++ty)
        for (int tx = lo[0]; tx <= hi[0]; ++tx)
          b.kernels[(static_cast<size_t>(tz) * b.tiles[1] + ty) * b.tiles[0] + tx].push_back(i);
  }
  return b;
}
struct KEval {
  V3 p;
  M3 q;
  double rho;
};
// voxelizer.cpp:96-104
static std::vector<KEval> precompute(const Cloud& c) {
  std::vector<KEval> ev(c.m);
  for (int i = 0; i < c.m; ++i) {
    ev[i].p = c.position(i);
    ev[i].q = inv3(covariance_at(c, i));
    ev[i].rho = c.rho(i);
  }
  return ev;
}
static inline double quad3(const M3& q, const V3& d) {
  const V3 qd = mulv(q, d);
  return d[0] * qd[0] + d[1] * qd[1] + d[2] * qd[2];
}
// voxelizer.cpp:108-138
static void voxelize(const Cloud& c, const Grid& g, double cull, double* vol) {
  const size_t nvox = static_cast<size_t>(g.dims[0]) * g.dims[1] * g.dims[2];
  std::fill(vol, vol + nvox, 0.0);
  const Bins bins = bin_kernels(c, g, cull);
  const auto ev = precompute(c);
  const int n_tiles = static_cast<int>(bins.kernels.size());
#pragma omp parallel for schedule(static)
  for (int t = 0; t < n_tiles; ++t) {
    const auto& list = bins.kernels[t];
    if (list.empty()) continue;
    const int tx = t % bins.tiles[0];
    const int ty = (t / bins.tiles[0]) % bins.tiles[1];
    const int tz = t / (bins.tiles[0] * bins.tiles[1]);
    const int x0 = tx * kTileVox, x1 = std::min(x0 + kTileVox, g.dims[0]);
    const int y0 = ty * kTileVox, y1 = std::min(y0 + kTileVox, g.dims[1]);
    const int z0 = tz * kTileVox, z1 = std::min(z0 + kTileVox, g.dims[2]);
    for (int z = z0; z < z1; ++z)
      for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) {
          const V3 cc = g.center(x, y, z);
          double sum = 0.0;
          for (int i : list) {
            V3 d;
            for (int k = 0; k < 3; ++k) d[k] = cc[k] - ev[i].p[k];
            sum += ev[i].rho * std::exp(-0.5 * quad3(ev[i].q, d));
          }
          vol[(static_cast<size_t>(z) * g.dims[1] + y) * g.dims[0] + x] += sum;
        }
  }
}
struct Stat3 {
  double s0 = 0, s1[3] = {0, 0, 0}, s2[6] = {0, 0, 0, 0, 0, 0};  // xx yy zz xy xz yz
};
// voxel chain rule voxelizer.cpp:207-223
static void voxel_chain(const Cloud& c, const KEval& k, int i, const Stat3& s, Grads& grads) {
  M3 s2;
  s2.m[0][0] = s.s2[0]; s2.m[0][1] = s.s2[3]; s2.m[0][2] = s.s2[4];
  s2.m[1][0] = s.s2[3]; s2.m[1][1] = s.s2[1]; s2.m[1][2] = s.s2[5];
  s2.m[2][0] = s.s2[4]; s2.m[2][1] = s.s2[5]; s2.m[2][2] = s.s2[2];
  grads.rho_raw[i] += s.s0 * act_density_grad(c.rho_raw[i]);
  V3 s1;
  for (int a = 0; a < 3; ++a) s1[a] = s.s1[a];
  const V3 qs1 = mulv(k.q, s1);
  for (int a = 0; a < 3; ++a) grads.pos[3 * i + a] += k.rho * qs1[a];
  const M3 g_q = scale(s2, -0.5 * k.rho);
  const M3 g_sigma = mul(mul(scale(k.q, -1.0), g_q), k.q);
  accumulate_covariance_param_grads(c, i, g_sigma, grads);
}
// voxelizer.cpp:140-224
static void voxelize_backward(const Cloud& c, const Grid& g, const double* dL, Grads& grads, double cull) {
  const Bins bins = bin_kernels(c, g, cull);
  const auto ev = precompute(c);
  const int n_tiles = static_cast<int>(bins.kernels.size());
  std::vector<std::vector<Stat3>> scratch(n_tiles);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < n_tiles; ++t) {
    const auto& list = bins.kernels[t];
    if (list.empty()) continue;
    scratch[t].resize(list.size());
    const int tx = t % bins.tiles[0];
    const int ty = (t / bins.tiles[0]) % bins.tiles[1];
    const int tz = t / (bins.tiles[0] * bins.tiles[1]);
    const int x0 = tx * kTileVox, x1 = std::min(x0 + kTileVox, g.dims[0]);
    const int y0 = ty * kTileVox, y1 = std::min(y0 + kTileVox, g.dims[1]);
    const int z0 = tz * kTileVox, z1 = std::min(z0 + kTileVox, g.dims[2]);
    for (int z = z0; z < z1; ++z)
      for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) {
          const double gv = dL[(static_cast<size_t>(z) * g.dims[1] + y) * g.dims[0] + x];
          if (gv == 0.0) continue;
          const V3 cc = g.center(x, y, z);
          for (size_t li = 0; li < list.size(); ++li) {
            const KEval& k = ev[list[li]];
            V3 d;
            for (int a = 0; a < 3; ++a) d[a] = cc[a] - k.p[a];
            const double ge = gv * std::exp(-0.5 * quad3(k.q, d));
            Stat3& s = scratch[t][li];
            s.s0 += ge;
            for (int a = 0; a < 3; ++a) s.s1[a] += ge * d[a];
            s.s2[0] += ge * d[0] * d[0];
            s.s2[1] += ge * d[1] * d[1];
            s.s2[2] += ge * d[2] * d[2];
            s.s2[3] += ge * d[0] * d[1];
            s.s2[4] += ge * d[0] * d[2];
            s.s2[5] += ge * d[1] * d[2];
          }
        }
  }
  std::vector<Stat3> total(c.m);
  std::vector<char> touched(c.m, 0);
  for (int t = 0; t < n_tiles; ++t) {
    const auto& list = bins.kernels[t];
    for (size_t li = 0; li < list.size(); ++li) {
      const Stat3& s = scratch[t][li];
      Stat3& acc = total[list[li]];
      acc.s0 += s.s0;
      for (int a = 0; a < 3; ++a) acc.s1[a] += s.s1[a];
      for (int a = 0; a < 6; ++a) acc.s2[a] += s.s2[a];
      touched[list[li]] = 1;
    }
  }
  for (int i = 0; i < c.m; ++i) {
    if (!touched[i]) continue;
    voxel_chain(c, ev[i], i, total[i], grads);
  }
}

// ---------------------------------------------------------------- objectives
constexpr int kWin = 11;
constexpr double kSigma = 1.5, kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;
static const std::array<double, kWin>& gauss_taps() {  // objectives.cpp:16-29
  static const std::array<double, kWin> taps = [] {
    std::array<double, kWin> t{};
    double sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
      const double x = i - (kWin - 1) / 2.0;
      t[i] = std::exp(-x * x / (2.0 * kSigma * kSigma));
      sum += t[i];
    }
    for (auto& v : t) v /= sum;
    return t;
  }();
  return taps;
}
struct Img {
  int w = 0, h = 0;
  std::vector<double> d;
  Img() = default;
  Img(int w_, int h_) : w(w_), h(h_), d(static_cast<size_t>(w_) * h_, 0.0) {}
  double& at(int x, int y) { return d[static_cast<size_t>(y) * w + x]; }
  double at(int x, int y) const { return d[static_cast<size_t>(y) * w + x]; }
};
static Img valid_filter(const Img& img) {  // objectives.cpp:32-49
  const auto& w = gauss_taps();
  Img tmp(img.w - kWin + 1, img.h);
  for (int y = 0; y < tmp.h; ++y)
    for (int x = 0; x < tmp.w; ++x) {
      double s = 0.0;
      for (int i = 0; i < kWin; ++i) s += w[i] * img.at(x + i, y);
      tmp.at(x, y) = s;
    }
  Img out(img.w - kWin + 1, img.h - kWin + 1);
  for (int y = 0; y < out.h; ++y)
    for (int x = 0; x < out.w; ++x) {
      double s = 0.0;
      for (int j = 0; j < kWin; ++j) s += w[j] * tmp.at(x, y + j);
      out.at(x, y) = s;
    }
  return out;
}
static Img adjoint_filter(const Img& f, int width, int height) {  // objectives.cpp:52-69
  const auto& w = gauss_taps();
  Img tmp(f.w, height);
  for (int y = 0; y < f.h; ++y)
    for (int x = 0; x < f.w; ++x) {
      const double v = f.at(x, y);
      if (v == 0.0) continue;
      for (int j = 0; j < kWin; ++j) tmp.at(x, y + j) += w[j] * v;
    }
  Img out(width, height);
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < tmp.w; ++x) {
      const double v = tmp.at(x, y);
      if (v == 0.0) continue;
      for (int i = 0; i < kWin; ++i) out.at(x + i, y) += w[i] * v;
    }
  return out;
}
static Img prod(const Img& a, const Img& b) {
  Img o(a.w, a.h);
  for (size_t i = 0; i < a.d.size(); ++i) o.d[i] = a.d[i] * b.d[i];
  return o;
}
// objectives.cpp:131-167
static double dssim_loss(const Img& a, const Img& b, double* grad) {
  const Img mu1 = valid_filter(a), mu2 = valid_filter(b);
  const Img m11 = valid_filter(prod(a, a)), m22 = valid_filter(prod(b, b)), m12 = valid_filter(prod(a, b));
  const size_t n = mu1.d.size();
  Img s1(mu1.w, mu1.h), s2(mu1.w, mu1.h), s12(mu1.w, mu1.h);
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    s1.d[i] = m11.d[i] - mu1.d[i] * mu1.d[i];
    s2.d[i] = m22.d[i] - mu2.d[i] * mu2.d[i];
    s12.d[i] = m12.d[i] - mu1.d[i] * mu2.d[i];
    const double a1 = 2.0 * mu1.d[i] * mu2.d[i] + kC1;
    const double b1 = mu1.d[i] * mu1.d[i] + mu2.d[i] * mu2.d[i] + kC1;
    const double a2 = 2.0 * s12.d[i] + kC2;
    const double b2 = s1.d[i] + s2.d[i] + kC2;
    sum += (a1 * a2) / (b1 * b2);
  }
  const double mean_ssim = sum / static_cast<double>(n);
  const double inv_p = 1.0 / static_cast<double>(n);
  Img g1(mu1.w, mu1.h), g2(mu1.w, mu1.h), g3(mu1.w, mu1.h);
  for (size_t i = 0; i < n; ++i) {
    const double m1 = mu1.d[i], m2 = mu2.d[i];
    const double a1 = 2.0 * m1 * m2 + kC1;
    const double b1 = m1 * m1 + m2 * m2 + kC1;
    const double a2 = 2.0 * s12.d[i] + kC2;
    const double b2 = s1.d[i] + s2.d[i] + kC2;
    const double l = a1 / b1, cs = a2 / b2;
    g1.d[i] = cs * 2.0 * (m2 * b1 - m1 * a1) / (b1 * b1);
    g2.d[i] = -l * a2 / (b2 * b2);
    g3.d[i] = l * 2.0 / b2;
  }
  const Img t1 = adjoint_filter(g1, a.w, a.h);
  const Img t2 = adjoint_filter(g2, a.w, a.h);
  const Img t2m = adjoint_filter(prod(g2, mu1), a.w, a.h);
  const Img t3 = adjoint_filter(g3, a.w, a.h);
  const Img t3m = adjoint_filter(prod(g3, mu2), a.w, a.h);
  for (size_t i = 0; i < a.d.size(); ++i) {
    const double ds = t1.d[i] + 2.0 * a.d[i] * t2.d[i] - 2.0 * t2m.d[i] + b.d[i] * t3.d[i] - t3m.d[i];
    grad[i] = -0.5 * inv_p * ds;
  }
  return 0.5 * (1.0 - mean_ssim);
}

}  // namespace orc

// =====================================================================
// C ABI for ctypes (tests / bench cpu leg only)
// =====================================================================
using namespace orc;

namespace {
thread_local std::string g_err;
Scanner make_scanner(const double* geo, const int* res) {
  // geo: l_so, l_sd, det_w_mm, det_h_mm, ext_min[3], ext_max[3], near_clip
  Scanner s;
  s.l_so_mm = geo[0];
  s.l_sd_mm = geo[1];
  s.det_size_mm[0] = geo[2];
  s.det_size_mm[1] = geo[3];
  for (int k = 0; k < 3; ++k) {
    s.extent_min_mm[k] = geo[4 + k];
    s.extent_max_mm[k] = geo[7 + k];
  }
  s.near_clip_mm = geo[10];
  s.det_res_px[0] = res[0];
  s.det_res_px[1] = res[1];
  s.parallel = res[2];  // res = {W, H, parallel_beam}
  return s;
}
RasterOptions make_opts(const double* o) {
  // o: mode, lowpass_eps_px, dilation_compensation, freeze_jacobian, cull
  RasterOptions r;
  r.mode = static_cast<int>(o[0]);
  r.lowpass_eps_px = o[1];
  r.dilation_compensation = static_cast<int>(o[2]);
  r.freeze_jacobian = static_cast<int>(o[3]);
  r.cull_mahalanobis = o[4];
  return r;
}
Cloud make_cloud(int m, double s_min, const double* rho, const double* pos, const double* sc,
                 const double* rot) {
  Cloud c;
  c.m = m;
  c.s_min = s_min;
  c.rho_raw = rho;
  c.pos = pos;
  c.scale_raw = sc;
  c.rot = rot;
  return c;
}
Grid make_grid(const int* dims, const double* origin, const double* spacing) {
  Grid g;
  for (int k = 0; k < 3; ++k) {
    g.dims[k] = dims[k];
    g.origin[k] = origin[k];
    g.spacing[k] = spacing[k];
  }
  return g;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
int orc_max_threads() { return omp_get_max_threads(); }

// --- RNG (std::mt19937_64 + libstdc++ distributions, as tests/helpers.hpp)
void* orc_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void orc_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
double orc_rng_uniform(void* r, double lo, double hi) {
  std::uniform_real_distribution<double> u(lo, hi);
  return u(*static_cast<std::mt19937_64*>(r));
}
double orc_rng_normal(void* r) {
  std::normal_distribution<double> g(0.0, 1.0);
  return g(*static_cast<std::mt19937_64*>(r));
}
// tests/helpers.hpp:30-48 random_cloud + gaussian_cloud.cpp:48-55 add_kernel
void orc_random_cloud(void* rp, int count, double pos_radius, double scale_min, double scale_max,
                      double s_min, double* rho_raw, double* pos, double* scale_raw, double* rot) {
  auto& rng = *static_cast<std::mt19937_64*>(rp);
  std::uniform_real_distribution<double> upos(-pos_radius, pos_radius);
  std::uniform_real_distribution<double> uscale(scale_min, scale_max);
  std::uniform_real_distribution<double> urho(0.2, 1.5);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int i = 0; i < count; ++i) {
    const double rho = urho(rng);
    // Vec3(upos(rng), upos(rng), upos(rng)): argument evaluation order of the
    // Eigen constructor under GCC is right-to-left for the call; the reference
    // build is GCC as well, so replicate that order.
    double p[3], s[3], q[4];
    p[2] = upos(rng); p[1] = upos(rng); p[0] = upos(rng);
    s[2] = uscale(rng); s[1] = uscale(rng); s[0] = uscale(rng);
    q[3] = gauss(rng); q[2] = gauss(rng); q[1] = gauss(rng); q[0] = gauss(rng);
    double qn[4];
    normalize4(q, qn);   // random_cloud normalizes ...
    double qn2[4];
    normalize4(qn, qn2); // ... and add_kernel normalizes again
    rho_raw[i] = act_density_inv(rho);
    for (int k = 0; k < 3; ++k) {
      pos[3 * i + k] = p[k];
      scale_raw[3 * i + k] = act_scale_inv(s[k], s_min);
    }
    for (int k = 0; k < 4; ++k) rot[4 * i + k] = qn2[k];
  }
}
// activated kernel -> raw parameters (gaussian_cloud.cpp:48-55)
void orc_kernel_to_raw(int n, double s_min, const double* rho, const double* scale, const double* rot_in,
                       double* rho_raw, double* scale_raw, double* rot_out) {
  for (int i = 0; i < n; ++i) {
    rho_raw[i] = act_density_inv(rho[i]);
    for (int k = 0; k < 3; ++k) scale_raw[3 * i + k] = act_scale_inv(scale[3 * i + k], s_min);
    normalize4(rot_in + 4 * i, rot_out + 4 * i);
  }
}
void orc_activate(int n, double s_min, const double* rho_raw, const double* scale_raw,
                  double* rho, double* scale) {
  for (int i = 0; i < n; ++i) {
    rho[i] = act_density(rho_raw[i]);
    for (int k = 0; k < 3; ++k) scale[3 * i + k] = act_scale(scale_raw[3 * i + k], s_min);
  }
}
void orc_random_image(void* rp, int n, double lo, double hi, double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rp);
  std::uniform_real_distribution<double> uni(lo, hi);
  for (int i = 0; i < n; ++i) out[i] = uni(rng);
}

// --- geometry
void orc_view_transform(const double* geo, const int* res, double theta, double* rot9, double* t3) {
  const Scanner s = make_scanner(geo, res);
  const View v = view_transform(s, theta);
  for (int i = 0; i < 3; ++i) {
    t3[i] = v.t[i];
    for (int j = 0; j < 3; ++j) rot9[3 * i + j] = v.rot.m[i][j];
  }
}
void orc_detector(const double* geo, const int* res, double* out4) {
  const Det d = detector_model(make_scanner(geo, res));
  out4[0] = d.fx; out4[1] = d.fy; out4[2] = d.cx; out4[3] = d.cy;
}
int orc_local_jacobian(const double* geo, const int* res, const double* p, double* j9) {
  const Det d = detector_model(make_scanner(geo, res));
  V3 pp;
  for (int k = 0; k < 3; ++k) pp[k] = p[k];
  if (pp[2] < d.near) {
    g_err = "KernelBehindSource: kernel center behind the near clip plane";
    return 3;
  }
  const M3 j = local_jacobian(d, pp);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) j9[3 * a + b] = j.m[a][b];
  return 0;
}
void orc_ray_space_point(const double* geo, const int* res, const double* p, double* out) {
  const Det d = detector_model(make_scanner(geo, res));
  V3 pp;
  for (int k = 0; k < 3; ++k) pp[k] = p[k];
  const V3 r = ray_space_point(d, pp);
  for (int k = 0; k < 3; ++k) out[k] = r[k];
}
// geometry.cpp:125-138
void orc_pixel_ray(const double* geo, const int* res, double theta, int u, int v, double* origin, double* dir) {
  const Scanner c = make_scanner(geo, res);
  const Det det = detector_model(c);
  const double du = c.det_size_mm[0] / det.w, dv = c.det_size_mm[1] / det.h;
  const double xd = (u + 0.5) * du - 0.5 * c.det_size_mm[0];
  const double yd = (v + 0.5) * dv - 0.5 * c.det_size_mm[1];
  V3 ds;
  if (c.parallel) {  // parallel beam: ray through the detector point along the view axis
    const View view = view_transform(c, theta);
    V3 os;
    os[0] = xd; os[1] = yd; os[2] = -view.t[2];
    const V3 o = mulv_t(view.rot, os);
    V3 dz;
    dz[0] = 0.0; dz[1] = 0.0; dz[2] = 1.0;
    const V3 d = mulv_t(view.rot, dz);
    for (int k = 0; k < 3; ++k) {
      origin[k] = o[k];
      dir[k] = d[k];
    }
    return;
  }
  ds[0] = xd; ds[1] = yd; ds[2] = c.l_sd_mm;
  const double n = norm3(ds);
  for (int k = 0; k < 3; ++k) ds[k] = ds[k] / n;
  const View view = view_transform(c, theta);
  const V3 src = mulv_t(view.rot, view.t);
  for (int k = 0; k < 3; ++k) origin[k] = -src[k];
  const V3 d = mulv_t(view.rot, ds);
  for (int k = 0; k < 3; ++k) dir[k] = d[k];
}

// --- cloud helpers
void orc_covariance(int m, double s_min, const double* rho, const double* pos, const double* sc,
                    const double* rot, int i, double* out9) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  const M3 s = covariance_at(c, i);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) out9[3 * a + b] = s.m[a][b];
}
double orc_density_at(int m, double s_min, const double* rho, const double* pos, const double* sc,
                      const double* rot, const double* x) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  V3 xx;
  for (int k = 0; k < 3; ++k) xx[k] = x[k];
  return density_at(c, xx);
}
void orc_normalize_rotations(int m, double* rot) {  // gaussian_cloud.cpp:112-117
  for (int i = 0; i < m; ++i) {
    double q[4];
    normalize4(rot + 4 * i, q);
    for (int k = 0; k < 4; ++k) rot[4 * i + k] = q[k];
  }
}
void orc_cov_param_grads(int m, double s_min, const double* rho, const double* pos, const double* sc,
                         const double* rot, int i, const double* g_sigma9, double* g_scale_raw,
                         double* g_rot) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  M3 gs;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) gs.m[a][b] = g_sigma9[3 * a + b];
  Grads g{nullptr, nullptr, g_scale_raw, g_rot};
  accumulate_covariance_param_grads(c, i, gs, g);
}

// tests/helpers.hpp:52-69 ray_march_density (midpoint quadrature of density_at)
double orc_ray_march_density(int m, double s_min, const double* rho, const double* pos, const double* sc,
                             const double* rot, const double* origin, const double* dir, double step) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  double t_lo = std::numeric_limits<double>::infinity();
  double t_hi = -std::numeric_limits<double>::infinity();
  for (int i = 0; i < c.m; ++i) {
    const V3 p = c.position(i);
    const double tc = (p[0] - origin[0]) * dir[0] + (p[1] - origin[1]) * dir[1] + (p[2] - origin[2]) * dir[2];
    const V3 s = c.scalev(i);
    const double pad = 8.0 * std::max({s[0], s[1], s[2]});
    t_lo = std::min(t_lo, tc - pad);
    t_hi = std::max(t_hi, tc + pad);
  }
  if (!(t_hi > t_lo)) return 0.0;
  const int n = static_cast<int>(std::ceil((t_hi - t_lo) / step));
  const double h = (t_hi - t_lo) / n;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    V3 x;
    for (int k = 0; k < 3; ++k) x[k] = origin[k] + (t_lo + (i + 0.5) * h) * dir[k];
    sum += density_at(c, x);
  }
  return sum * h;
}

// --- rasterizer
// project_kernel (rasterizer.cpp:103-110). out: cx cy cov00 cov01 cov11
// conic00 conic01 conic11 amp mu depth. returns 1 visible / 0 culled.
int orc_project_kernel(int m, double s_min, const double* rho, const double* pos, const double* sc,
                       const double* rot, int i, const double* geo, const int* res, double theta,
                       const double* opts, double* out) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  const Scanner s = make_scanner(geo, res);
  Projected p;
  if (!project_impl(c, i, view_transform(s, theta), detector_model(s), make_opts(opts), p, nullptr)) return 0;
  const double v[11] = {p.center.x, p.center.y, p.cov.m[0][0], p.cov.m[0][1], p.cov.m[1][1],
                        p.conic.m[0][0], p.conic.m[0][1], p.conic.m[1][1], p.amplitude, p.mu, p.depth};
  std::memcpy(out, v, sizeof(v));
  return 1;
}

void* orc_render(int m, double s_min, const double* rho, const double* pos, const double* sc,
                 const double* rot, const double* geo, const int* res, double theta, const double* opts) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  return render(c, make_scanner(geo, res), theta, make_opts(opts));
}
void orc_render_free(void* h) { delete static_cast<Rendered*>(h); }
void orc_render_image(void* h, double* out) {
  const auto* r = static_cast<Rendered*>(h);
  std::memcpy(out, r->image.data(), r->image.size() * sizeof(double));
}
int orc_render_n_visible(void* h) { return static_cast<int>(static_cast<Rendered*>(h)->visible.size()); }
int64_t orc_render_n_pairs(void* h) {
  int64_t n = 0;
  for (const auto& l : static_cast<Rendered*>(h)->tile_visible) n += static_cast<int64_t>(l.size());
  return n;
}
// tile lists expressed in kernel indices (visible[vi].kernel_index): offsets[T+1], idx[pairs]
void orc_render_tile_lists(void* h, int64_t* offsets, int32_t* kernel_idx) {
  const auto* r = static_cast<Rendered*>(h);
  int64_t o = 0;
  for (size_t t = 0; t < r->tile_visible.size(); ++t) {
    offsets[t] = o;
    for (int vi : r->tile_visible[t]) kernel_idx[o++] = r->visible[vi].kernel_index;
  }
  offsets[r->tile_visible.size()] = o;
}
// visible records: kernel_index, and 11 doubles each as orc_project_kernel
void orc_render_visible(void* h, int32_t* kidx, double* rec) {
  const auto* r = static_cast<Rendered*>(h);
  for (size_t vi = 0; vi < r->visible.size(); ++vi) {
    const Projected& p = r->visible[vi];
    kidx[vi] = p.kernel_index;
    const double v[11] = {p.center.x, p.center.y, p.cov.m[0][0], p.cov.m[0][1], p.cov.m[1][1],
                          p.conic.m[0][0], p.conic.m[0][1], p.conic.m[1][1], p.amplitude, p.mu, p.depth};
    std::memcpy(rec + 11 * vi, v, sizeof(v));
  }
}
int orc_render_backward(void* h, int m, double s_min, const double* rho, const double* pos, const double* sc,
                        const double* rot, const double* geo, const int* res, double theta, const double* opts,
                        const double* dL, double* g_rho, double* g_pos, double* g_sc, double* g_rot,
                        double* st_norm, int32_t* st_count, double* st_3d) {
  const auto* r = static_cast<Rendered*>(h);
  const Scanner s = make_scanner(geo, res);
  if (r->w != s.det_res_px[0] || r->h != s.det_res_px[1]) {
    g_err = "DimMismatch: render_backward: upstream gradient dims mismatch";
    return 3;
  }
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  Grads g{g_rho, g_pos, g_sc, g_rot};
  Stats st{st_norm, st_count, st_3d};
  render_backward(c, s, theta, *r, dL, g, make_opts(opts), st_norm ? &st : nullptr);
  return 0;
}
// Feeds per-visible tile statistics (6 per visible: s0 s1x s1y s2xx s2yy s2xy)
// through the reference chain rule (rasterizer.cpp:262-341). Used by tests to
// separate pixel-statistics error from chain-rule error.
void orc_raster_chain_from_stats(int m, double s_min, const double* rho, const double* pos, const double* sc,
                                 const double* rot, const double* geo, const int* res, double theta,
                                 const double* opts, int n_vis, const int32_t* kidx, const double* stats6,
                                 double* g_rho, double* g_pos, double* g_sc, double* g_rot) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  const Scanner s = make_scanner(geo, res);
  const View view = view_transform(s, theta);
  const Det det = detector_model(s);
  const RasterOptions o = make_opts(opts);
  Grads g{g_rho, g_pos, g_sc, g_rot};
  for (int vi = 0; vi < n_vis; ++vi) {
    Stat2 st;
    st.s0 = stats6[6 * vi];
    st.s1[0] = stats6[6 * vi + 1];
    st.s1[1] = stats6[6 * vi + 2];
    st.s2[0] = stats6[6 * vi + 3];
    st.s2[1] = stats6[6 * vi + 4];
    st.s2[2] = stats6[6 * vi + 5];
    raster_chain(c, view, det, o, kidx[vi], st, g, nullptr);
  }
}

// --- voxelizer
void orc_grid_for_extent(const double* lo, const double* hi, const int* dims, double* origin, double* spacing) {
  for (int k = 0; k < 3; ++k) {  // voxelizer.cpp:8-14
    origin[k] = lo[k];
    spacing[k] = (hi[k] - lo[k]) / static_cast<double>(dims[k]);
  }
}
void orc_voxelize(int m, double s_min, const double* rho, const double* pos, const double* sc, const double* rot,
                  const int* dims, const double* origin, const double* spacing, double cull, double* vol) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  voxelize(c, make_grid(dims, origin, spacing), cull, vol);
}
int orc_voxelize_backward(int m, double s_min, const double* rho, const double* pos, const double* sc,
                          const double* rot, const int* dims, const double* origin, const double* spacing,
                          double cull, const double* dL, double* g_rho, double* g_pos, double* g_sc,
                          double* g_rot) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  Grads g{g_rho, g_pos, g_sc, g_rot};
  voxelize_backward(c, make_grid(dims, origin, spacing), dL, g, cull);
  return 0;
}
// brick lists (voxelizer.cpp:52-88): offsets[B+1], kernel idx[pairs]; returns pair count
// when offsets==nullptr.
int64_t orc_voxel_bins(int m, double s_min, const double* rho, const double* pos, const double* sc,
                       const double* rot, const int* dims, const double* origin, const double* spacing,
                       double cull, int64_t* offsets, int32_t* idx) {
  const Cloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  const Bins b = bin_kernels(c, make_grid(dims, origin, spacing), cull);
  int64_t o = 0;
  for (size_t t = 0; t < b.kernels.size(); ++t) {
    if (offsets) offsets[t] = o;
    for (int i : b.kernels[t]) {
      if (idx) idx[o] = i;
      ++o;
    }
  }
  if (offsets) offsets[b.kernels.size()] = o;
  return o;
}
// voxelizer.cpp:226-239
void orc_random_subvolume_spec(void* rp, const double* lo, const double* hi, const double* spacing, int d,
                               double* origin) {
  auto& rng = *static_cast<std::mt19937_64*>(rp);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  for (int k = 0; k < 3; ++k) {
    const double span = (hi[k] - lo[k]) - d * spacing[k];
    const double u = uni(rng);
    origin[k] = span > 0.0 ? lo[k] + u * span : 0.5 * (lo[k] + hi[k]) - 0.5 * d * spacing[k];
  }
}

// --- objectives
// objectives.cpp:169-202. returns 3 on dims < 2 (DimMismatch).
int orc_tv3d(const int* dims, const double* vol, double* value, double* grad) {
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  if (std::min({nx, ny, nz}) < 2) {
    g_err = "DimMismatch: tv3d_loss: need at least 2 voxels per axis";
    return 3;
  }
  const size_t n = static_cast<size_t>(nx) * ny * nz;
  std::fill(grad, grad + n, 0.0);
  const int strides[3] = {1, nx, nx * ny};
  const int counts[3] = {(nx - 1) * ny * nz, nx * (ny - 1) * nz, nx * ny * (nz - 1)};
  double val = 0.0;
  for (int axis = 0; axis < 3; ++axis) {
    if (counts[axis] == 0) continue;
    const double inv_n = 1.0 / static_cast<double>(counts[axis]);
    const int ex = axis == 0 ? nx - 1 : nx, ey = axis == 1 ? ny - 1 : ny, ez = axis == 2 ? nz - 1 : nz;
    double sum = 0.0;
    for (int z = 0; z < ez; ++z)
      for (int y = 0; y < ey; ++y)
        for (int x = 0; x < ex; ++x) {
          const size_t i = (static_cast<size_t>(z) * ny + y) * nx + x;
          const double d = vol[i + strides[axis]] - vol[i];
          sum += std::abs(d);
          if (d > 0.0) {
            grad[i + strides[axis]] += inv_n;
            grad[i] -= inv_n;
          } else if (d < 0.0) {
            grad[i + strides[axis]] -= inv_n;
            grad[i] += inv_n;
          }
        }
    val += sum * inv_n;
  }
  *value = val;
  return 0;
}
// objectives.cpp:113-127
int orc_l1(int n, const double* r, const double* m, double* value, double* grad) {
  const double inv_n = 1.0 / static_cast<double>(n);
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = r[i] - m[i];
    sum += std::abs(d);
    grad[i] = d > 0.0 ? inv_n : (d < 0.0 ? -inv_n : 0.0);
  }
  *value = sum * inv_n;
  return 0;
}
int orc_dssim(int w, int h, const double* a, const double* b, double* value, double* grad) {
  if (w < kWin || h < kWin) {
    g_err = "DimMismatch: ssim: image smaller than the 11x11 window";
    return 3;
  }
  Img A(w, h), B(w, h);
  std::memcpy(A.d.data(), a, sizeof(double) * w * h);
  std::memcpy(B.d.data(), b, sizeof(double) * w * h);
  *value = dssim_loss(A, B, grad);
  return 0;
}

// --- adaptive control: trainer.cpp:167-230 (prune / clone / split), with
// GaussianCloud::remove_kernels (gaussian_cloud.cpp:89-110, order-preserving
// compaction) and add_kernel (:48-72, fresh zero Adam state), reset_grad_stats.
// arrays: 0 rho_raw, 1 pos, 2 scale_raw, 3 rot, 4..11 Adam m/v (rho, pos, scale, rot).
struct ACResult {
  std::vector<double> a[12];
  int pruned = 0, cloned = 0, split = 0;
};
void* orc_adaptive_control(void* rp, int m, double s_min, const double* const* arrays, const double* norm_acc,
                           const int32_t* count, const double* g3d, double prune_thr, double densify_thr,
                           double split_frac, double split_factor, const double* extent_size) {
  auto& rng = *static_cast<std::mt19937_64*>(rp);
  const int stride[12] = {1, 3, 3, 4, 1, 1, 3, 3, 3, 3, 4, 4};
  Cloud c = make_cloud(m, s_min, arrays[0], arrays[1], arrays[2], arrays[3]);
  auto* res = new ACResult();
  std::vector<double> rho_raw(arrays[0], arrays[0] + m);
  std::vector<char> keep(m, 1);
  for (int i = 0; i < m; ++i)
    if (c.rho(i) < prune_thr) {
      keep[i] = 0;
      ++res->pruned;
    }
  struct NK {
    double rho, pos[3], scale[3], q[4];
  };
  std::vector<NK> added;
  const double size_thr = split_frac * std::max({extent_size[0], extent_size[1], extent_size[2]});
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int i = 0; i < m; ++i) {
    if (!keep[i]) continue;
    if (count[i] == 0) continue;
    const double mean_grad = norm_acc[i] / count[i];
    if (mean_grad <= densify_thr) continue;
    const V3 s = c.scalev(i);
    const double rho_half = 0.5 * c.rho(i);
    if (rho_half <= 0.0) continue;
    double qn[4];
    normalize4(c.rot + 4 * i, qn);  // kernel(i).rotation = quat_raw(i).normalized()
    if (std::max({s[0], s[1], s[2]}) <= size_thr) {
      NK ch{};
      ch.rho = rho_half;
      for (int k = 0; k < 3; ++k) {
        ch.pos[k] = c.pos[3 * i + k];
        ch.scale[k] = s[k];
      }
      for (int k = 0; k < 4; ++k) ch.q[k] = qn[k];
      const double gd[3] = {g3d[3 * i], g3d[3 * i + 1], g3d[3 * i + 2]};
      const double norm = std::sqrt(gd[0] * gd[0] + gd[1] * gd[1] + gd[2] * gd[2]);
      if (norm > 0.0) {
        const double smean = (s[0] + s[1] + s[2]) / 3.0;
        for (int k = 0; k < 3; ++k) ch.pos[k] -= (smean / norm) * gd[k];
      }
      rho_raw[i] = act_density_inv(rho_half);
      added.push_back(ch);
      ++res->cloned;
    } else {
      keep[i] = 0;
      const M3 rot = rotation_matrix(c.rot + 4 * i);
      for (int cc = 0; cc < 2; ++cc) {
        NK ch{};
        ch.rho = rho_half;
        for (int k = 0; k < 3; ++k) {
          ch.pos[k] = c.pos[3 * i + k];
          ch.scale[k] = std::max(s[k] / split_factor, s_min * (1.0 + 1e-6));
        }
        for (int k = 0; k < 4; ++k) ch.q[k] = qn[k];
        // Vec3 local(gauss*s.x, gauss*s.y, gauss*s.z): GCC evaluates the
        // constructor arguments right to left (z draw first)
        V3 local;
        local[2] = gauss(rng) * s[2];
        local[1] = gauss(rng) * s[1];
        local[0] = gauss(rng) * s[0];
        const V3 d = mulv(rot, local);
        for (int k = 0; k < 3; ++k) ch.pos[k] += d[k];
        added.push_back(ch);
      }
      ++res->split;
    }
  }
  // remove_kernels(keep): compaction in order; parent clones keep halved rho_raw
  for (int a = 0; a < 12; ++a) {
    const double* src = a == 0 ? rho_raw.data() : arrays[a];
    for (int i = 0; i < m; ++i)
      if (keep[i])
        for (int k = 0; k < stride[a]; ++k) res->a[a].push_back(src[stride[a] * i + k]);
  }
  // add_kernel for every new kernel (activated values -> raw, zero Adam state)
  for (const NK& n : added) {
    res->a[0].push_back(act_density_inv(n.rho));
    for (int k = 0; k < 3; ++k) res->a[1].push_back(n.pos[k]);
    for (int k = 0; k < 3; ++k) res->a[2].push_back(act_scale_inv(n.scale[k], s_min));
    double q2[4];
    normalize4(n.q, q2);
    for (int k = 0; k < 4; ++k) res->a[3].push_back(q2[k]);
    for (int a = 4; a < 12; ++a)
      for (int k = 0; k < stride[a]; ++k) res->a[a].push_back(0.0);
  }
  return res;
}
int orc_ac_size(void* h) { return static_cast<int>(static_cast<ACResult*>(h)->a[0].size()); }
void orc_ac_counts(void* h, int* out3) {
  auto* r = static_cast<ACResult*>(h);
  out3[0] = r->pruned;
  out3[1] = r->cloned;
  out3[2] = r->split;
}
void orc_ac_get(void* h, int a, double* out) {
  auto* r = static_cast<ACResult*>(h);
  std::memcpy(out, r->a[a].data(), r->a[a].size() * sizeof(double));
}
// Statistics the cloud carries after adaptive control: remove_kernels compacts
// them and add_kernel appends zeros (gaussian_cloud.cpp:48-110), then
// reset_grad_stats (gaussian_cloud.cpp:119-123, called at trainer.cpp:228)
// zeroes all three arrays.
void orc_ac_stats(void* h, double* norm_acc, int32_t* count, double* g3d) {
  const size_t n = static_cast<ACResult*>(h)->a[0].size();
  std::fill(norm_acc, norm_acc + n, 0.0);
  std::fill(count, count + n, 0);
  std::fill(g3d, g3d + 3 * n, 0.0);
}
void orc_ac_free(void* h) { delete static_cast<ACResult*>(h); }
// n consecutive draws of one std::normal_distribution(0,1) object
void orc_normal_draws(void* rp, int n, double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rp);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int i = 0; i < n; ++i) out[i] = gauss(rng);
}

// --- optimizer: trainer.cpp:34-36 lr_at, :144-163 Adam::step
double orc_lr_at(double lr_init, double ratio, int t, int iters) {
  return lr_init * std::pow(ratio, static_cast<double>(t) / iters);
}
void orc_adam_step(int64_t n, double* params, double* m, double* v, const double* g, double lr, int step,
                   double beta1, double beta2, double eps) {
  const double bc1 = 1.0 - std::pow(beta1, step);
  const double bc2 = 1.0 - std::pow(beta2, step);
  for (int64_t i = 0; i < n; ++i) {
    const double gi = g[i];
    m[i] = beta1 * m[i] + (1.0 - beta1) * gi;
    v[i] = beta2 * v[i] + (1.0 - beta2) * gi * gi;
    const double mhat = m[i] / bc1;
    const double vhat = v[i] / bc2;
    params[i] -= lr * mhat / (std::sqrt(vhat) + eps);
  }
}

}  // extern "C"
