// splatct_b200.hpp — header-only C++ mirror of the reference's host API for
// the hot path, implemented over the C ABI (splatct_gpu.h, host-buffer entry
// points). Same names, argument meaning, accumulate semantics and exception
// types as /root/reference/proj/core/include/splatct/{rasterizer,voxelizer,
// objectives,gaussian_cloud,geometry}.hpp; Eigen vectors are replaced by
// std::array so the header has no third-party dependency.
//
//   render            rasterizer.hpp:53-54      render_backward  rasterizer.hpp:61-64
//   voxelize          voxelizer.hpp:60-61       voxelize_backward voxelizer.hpp:65-67
//   tv3d_loss         objectives.hpp:31         grid_for_extent  voxelizer.hpp:26-27
//
// Link with -lsplatct_b200 (paper_2405_20693_b200/libsplatct_b200.so).
#pragma once

#include <array>
#include <chrono>
#include <functional>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "splatct_gpu.h"

namespace splatct_b200 {

// ---- exceptions (common.hpp:27-64) ------------------------------------------
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DimMismatch : DataError {
  using DataError::DataError;
};
struct DivergenceDetected : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == SCT_OK) return;
  const std::string msg = sct_last_error();
  switch (rc) {
    case SCT_ERR_CONFIG: throw ConfigError(msg);
    case SCT_ERR_DATA:
      if (msg.rfind("DimMismatch", 0) == 0) throw DimMismatch(msg);
      throw DataError(msg);
    case SCT_ERR_DIVERGENCE: throw DivergenceDetected(msg);
    case SCT_ERR_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// ---- types -------------------------------------------------------------------
using Vec2 = std::array<double, 2>;
using Vec3 = std::array<double, 3>;

struct ScannerConfig {  // geometry.hpp:12-31
  double l_so_mm = 8.0;
  double l_sd_mm = 12.0;
  Vec2 detector_size_mm{5.6, 5.6};
  std::array<int, 2> detector_res_px{128, 128};
  std::vector<double> angles_rad;
  Vec3 extent_min_mm{-1.0, -1.0, -1.0};
  Vec3 extent_max_mm{1.0, 1.0, 1.0};
  double near_clip_mm = 0.0;
  bool parallel_beam = false;  // extension; the reference is cone-beam only

  sct_scanner c() const {
    sct_scanner s{};
    s.l_so_mm = l_so_mm;
    s.l_sd_mm = l_sd_mm;
    for (int k = 0; k < 2; ++k) {
      s.det_size_mm[k] = detector_size_mm[k];
      s.det_res_px[k] = detector_res_px[k];
    }
    for (int k = 0; k < 3; ++k) {
      s.extent_min_mm[k] = extent_min_mm[k];
      s.extent_max_mm[k] = extent_max_mm[k];
    }
    s.near_clip_mm = near_clip_mm;
    s.parallel_beam = parallel_beam ? 1 : 0;
    return s;
  }
};

inline std::vector<double> full_circle_angles(int n) {  // geometry.cpp:63-67
  std::vector<double> a(n);
  for (int i = 0; i < n; ++i) a[i] = 2.0 * M_PI * i / n;
  return a;
}

enum class RenderMode { kRectified, kBiased };

struct RasterOptions {  // rasterizer.hpp:15-21
  RenderMode mode = RenderMode::kRectified;
  double lowpass_eps_px = 0.3;
  bool dilation_compensation = true;
  bool freeze_jacobian = false;
  double cull_mahalanobis = 3.0348542587702925;

  sct_raster_opts c() const {
    sct_raster_opts o{};
    o.mode = mode == RenderMode::kRectified ? SCT_MODE_RECTIFIED : SCT_MODE_BIASED;
    o.lowpass_eps_px = lowpass_eps_px;
    o.dilation_compensation = dilation_compensation;
    o.freeze_jacobian = freeze_jacobian;
    o.cull_mahalanobis = cull_mahalanobis;
    return o;
  }
};

// Raw parameters in the reference's SoA layout (gaussian_cloud.hpp:62-77).
struct GaussianCloud {
  double s_min_mm = 1e-4;
  std::vector<double> rho_raw, pos, scale_raw, rot;
  std::vector<double> grad2d_norm_accum;
  std::vector<int> grad_count;
  std::vector<double> grad3d_accum;
  int size() const { return static_cast<int>(rho_raw.size()); }
  double s_min() const { return s_min_mm; }
};

struct CloudGrads {  // gaussian_cloud.hpp:84-96
  std::vector<double> rho_raw, pos, scale_raw, rot;
  void resize(int m) {
    rho_raw.assign(m, 0.0);
    pos.assign(3 * static_cast<size_t>(m), 0.0);
    scale_raw.assign(3 * static_cast<size_t>(m), 0.0);
    rot.assign(4 * static_cast<size_t>(m), 0.0);
  }
};

struct Image {  // common.hpp:66-79
  int width = 0, height = 0;
  std::vector<double> data;
  Image() = default;
  Image(int w, int h, double fill = 0.0) : width(w), height(h), data(static_cast<size_t>(w) * h, fill) {}
  double at(int u, int v) const { return data[static_cast<size_t>(v) * width + u]; }
  double& at(int u, int v) { return data[static_cast<size_t>(v) * width + u]; }
};

struct GridSpec {  // voxelizer.hpp:13-24
  std::array<int, 3> dims{0, 0, 0};
  Vec3 origin_mm{0, 0, 0};
  Vec3 spacing_mm{1, 1, 1};
  size_t voxel_count() const { return static_cast<size_t>(dims[0]) * dims[1] * dims[2]; }
  sct_grid c() const {
    sct_grid g{};
    for (int k = 0; k < 3; ++k) {
      g.dims[k] = dims[k];
      g.origin_mm[k] = origin_mm[k];
      g.spacing_mm[k] = spacing_mm[k];
    }
    return g;
  }
};

inline GridSpec grid_for_extent(const Vec3& lo, const Vec3& hi, const std::array<int, 3>& dims) {
  GridSpec g;  // voxelizer.cpp:8-14
  g.dims = dims;
  g.origin_mm = lo;
  for (int k = 0; k < 3; ++k) g.spacing_mm[k] = (hi[k] - lo[k]) / static_cast<double>(dims[k]);
  return g;
}

struct DensityVolume {  // voxelizer.hpp:29-48
  std::array<int, 3> dims{0, 0, 0};
  Vec3 origin_mm{0, 0, 0}, spacing_mm{1, 1, 1};
  std::vector<double> data;
  GridSpec grid() const { return {dims, origin_mm, spacing_mm}; }
  size_t index(int x, int y, int z) const { return (static_cast<size_t>(z) * dims[1] + y) * dims[0] + x; }
  double at(int x, int y, int z) const { return data[index(x, y, z)]; }
};

struct VoxelizeOptions {  // voxelizer.hpp:53-57
  double cull_mahalanobis = 3.3681993876652464;
};

// ---- engine context (one per thread; the reference's calls are synchronous) --
class Context {
 public:
  static Context& get() {
    thread_local Context ctx;
    return ctx;
  }
  sct_ctx* handle() { return ctx_; }
  ~Context() {
    if (ctx_) sct_ctx_destroy(ctx_);
  }

 private:
  Context() { check(sct_ctx_create(0, nullptr, &ctx_)); }
  sct_ctx* ctx_ = nullptr;
};

// fp32 staging of a cloud in the reference's field order
struct CloudF32 {
  std::vector<float> rho_raw, pos, scale_raw, rot;
  sct_cloud c{};
  explicit CloudF32(const GaussianCloud& g) {
    auto cv = [](const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); };
    rho_raw = cv(g.rho_raw);
    pos = cv(g.pos);
    scale_raw = cv(g.scale_raw);
    rot = cv(g.rot);
    c.m = g.size();
    c.s_min_mm = g.s_min_mm;
    c.rho_raw = rho_raw.data();
    c.pos = pos.data();
    c.scale_raw = scale_raw.data();
    c.rot = rot.data();
  }
};

struct GradsF32 {
  std::vector<float> rho_raw, pos, scale_raw, rot;
  sct_grads c{};
  explicit GradsF32(const CloudGrads& g) {
    auto cv = [](const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); };
    rho_raw = cv(g.rho_raw);
    pos = cv(g.pos);
    scale_raw = cv(g.scale_raw);
    rot = cv(g.rot);
    c.rho_raw = rho_raw.data();
    c.pos = pos.data();
    c.scale_raw = scale_raw.data();
    c.rot = rot.data();
  }
  void store(CloudGrads& g) const {
    g.rho_raw.assign(rho_raw.begin(), rho_raw.end());
    g.pos.assign(pos.begin(), pos.end());
    g.scale_raw.assign(scale_raw.begin(), scale_raw.end());
    g.rot.assign(rot.begin(), rot.end());
  }
};

// ProjectedGaussian2D (rasterizer.hpp:24-32), row-major 2x2 matrices.
struct ProjectedGaussian2D {
  double center_px[2] = {0.0, 0.0};
  double cov_px[2][2] = {{1.0, 0.0}, {0.0, 1.0}};    // low-pass dilated
  double conic_px[2][2] = {{1.0, 0.0}, {0.0, 1.0}};  // cov_px inverse
  double amplitude = 0.0;
  double mu = 0.0;
  double depth_mm = 0.0;
  int kernel_index = -1;
};

// project_kernel (rasterizer.hpp:36-38, rasterizer.cpp:103-110) for every kernel
// of the cloud in one device call (FP64): the visible kernels in index order —
// exactly RenderedProjection::visible of the reference's render()
inline std::vector<ProjectedGaussian2D> project_kernels(const GaussianCloud& cloud, const ScannerConfig& config,
                                                        double theta_rad, const RasterOptions& opts = {});

// RenderedProjection (rasterizer.hpp:41-51): image + the device forward state.
struct RenderedProjection {
  Image image;
  int tiles_x = 0, tiles_y = 0;
  std::shared_ptr<sct_fwd> state;
  // what the device state was built with: render_backward rebuilds nothing, so
  // a backward call with another angle or other options is rejected
  double theta_rad = 0.0;
  RasterOptions opts;
  // tile_visible expressed in kernel indices (visible[vi].kernel_index)
  std::vector<std::vector<int>> tile_kernels() const {
    const int T = tiles_x * tiles_y;
    std::vector<int64_t> off(T + 1);
    check(sct_fwd_tile_lists(state.get(), 0, off.data(), nullptr));
    std::vector<int32_t> idx(off[T] > 0 ? off[T] : 1);
    check(sct_fwd_tile_lists(state.get(), 0, off.data(), idx.data()));
    std::vector<std::vector<int>> out(T);
    for (int t = 0; t < T; ++t) out[t].assign(idx.begin() + off[t], idx.begin() + off[t + 1]);
    return out;
  }
  int tile_of_pixel(int u, int v) const { return (v / 16) * tiles_x + (u / 16); }
  // the reference's `visible` and `tile_visible` (indices into visible), built on
  // request: the engine keeps its projection on the device, and an export costs
  // an FP64 re-projection of every kernel (project_kernels) plus the tile lists
  std::vector<ProjectedGaussian2D> visible(const GaussianCloud& cloud, const ScannerConfig& config) const {
    return project_kernels(cloud, config, theta_rad, opts);
  }
  std::vector<std::vector<int>> tile_visible(const std::vector<ProjectedGaussian2D>& vis) const {
    std::vector<int> pos_of;  // kernel index -> position in vis
    for (size_t i = 0; i < vis.size(); ++i) {
      const int k = vis[i].kernel_index;
      if (k >= static_cast<int>(pos_of.size())) pos_of.resize(k + 1, -1);
      pos_of[k] = static_cast<int>(i);
    }
    std::vector<std::vector<int>> out = tile_kernels();
    for (auto& list : out)
      for (int& k : list) k = pos_of[k];
    return out;
  }
};

inline std::vector<ProjectedGaussian2D> project_kernels(const GaussianCloud& cloud, const ScannerConfig& config,
                                                        double theta_rad, const RasterOptions& opts) {
  CloudF32 cf(cloud);
  const sct_scanner sc = config.c();
  const sct_raster_opts op = opts.c();
  const int64_t m = cloud.size();
  std::vector<int32_t> vis(m > 0 ? m : 1);
  std::vector<double> rec(11 * (m > 0 ? m : 1));
  check(sct_project_kernels_host(Context::get().handle(), &cf.c, &sc, theta_rad, &op, vis.data(), rec.data()));
  std::vector<ProjectedGaussian2D> out;
  for (int64_t i = 0; i < m; ++i) {
    if (!vis[i]) continue;
    const double* r = &rec[11 * i];  // cx cy cov00 cov01 cov11 conic00 conic01 conic11 amplitude mu depth
    ProjectedGaussian2D g;
    g.center_px[0] = r[0];
    g.center_px[1] = r[1];
    g.cov_px[0][0] = r[2];
    g.cov_px[0][1] = g.cov_px[1][0] = r[3];
    g.cov_px[1][1] = r[4];
    g.conic_px[0][0] = r[5];
    g.conic_px[0][1] = g.conic_px[1][0] = r[6];
    g.conic_px[1][1] = r[7];
    g.amplitude = r[8];
    g.mu = r[9];
    g.depth_mm = r[10];
    g.kernel_index = static_cast<int>(i);
    out.push_back(g);
  }
  return out;
}

// ---- the hot path --------------------------------------------------------------
inline RenderedProjection render(const GaussianCloud& cloud, const ScannerConfig& config, double theta_rad,
                                 const RasterOptions& opts = {}) {
  CloudF32 cf(cloud);
  const sct_scanner sc = config.c();
  const sct_raster_opts op = opts.c();
  const int w = config.detector_res_px[0], h = config.detector_res_px[1];
  std::vector<float> img(static_cast<size_t>(w) * h);
  sct_fwd* st = nullptr;
  check(sct_render_fwd_host(Context::get().handle(), &cf.c, &sc, &theta_rad, 1, &op, img.data(), &st));
  RenderedProjection r;
  r.state = std::shared_ptr<sct_fwd>(st, [](sct_fwd* p) { sct_fwd_free(p); });
  r.image = Image(w, h);
  r.image.data.assign(img.begin(), img.end());
  r.tiles_x = (w + 15) / 16;
  r.tiles_y = (h + 15) / 16;
  r.theta_rad = theta_rad;
  r.opts = opts;
  return r;
}

// rasterizer.cpp:195-198. The reference re-projects each visible kernel with the
// caller's theta_rad / opts (rasterizer.cpp:199,266); the engine keeps the forward
// pass's projection on the device, so both must equal the forward call's.
inline void render_backward(GaussianCloud& cloud, const ScannerConfig& config, double theta_rad,
                            const RenderedProjection& fwd, const Image& dL_dimage, CloudGrads& grads,
                            const RasterOptions& opts = {}, bool accumulate_stats = false) {
  if (!fwd.state) throw ConfigError("render_backward: no forward state");
  const RasterOptions& f = fwd.opts;
  if (theta_rad != fwd.theta_rad || opts.mode != f.mode || opts.lowpass_eps_px != f.lowpass_eps_px ||
      opts.dilation_compensation != f.dilation_compensation || opts.freeze_jacobian != f.freeze_jacobian ||
      opts.cull_mahalanobis != f.cull_mahalanobis)
    throw ConfigError("render_backward: theta_rad / opts differ from the forward call's");
  if (dL_dimage.width != config.detector_res_px[0] || dL_dimage.height != config.detector_res_px[1])
    throw DimMismatch("render_backward: upstream gradient dims mismatch");
  const int m = cloud.size();
  if (static_cast<int>(grads.rho_raw.size()) != m) throw DimMismatch("render_backward: grads not sized");
  CloudF32 cf(cloud);
  GradsF32 gf(grads);
  std::vector<float> dl(dL_dimage.data.begin(), dL_dimage.data.end());
  std::vector<float> s_norm, s_3d;
  std::vector<int32_t> s_cnt;
  sct_stats st{};
  if (accumulate_stats) {
    if (cloud.grad2d_norm_accum.size() != static_cast<size_t>(m)) {
      cloud.grad2d_norm_accum.assign(m, 0.0);
      cloud.grad_count.assign(m, 0);
      cloud.grad3d_accum.assign(3 * static_cast<size_t>(m), 0.0);
    }
    s_norm.assign(cloud.grad2d_norm_accum.begin(), cloud.grad2d_norm_accum.end());
    s_cnt.assign(cloud.grad_count.begin(), cloud.grad_count.end());
    s_3d.assign(cloud.grad3d_accum.begin(), cloud.grad3d_accum.end());
    st.grad2d_norm_accum = s_norm.data();
    st.grad_count = s_cnt.data();
    st.grad3d_accum = s_3d.data();
  }
  check(sct_render_bwd_host(Context::get().handle(), fwd.state.get(), &cf.c, dl.data(), &gf.c,
                            accumulate_stats ? &st : nullptr));
  gf.store(grads);
  if (accumulate_stats) {
    cloud.grad2d_norm_accum.assign(s_norm.begin(), s_norm.end());
    cloud.grad_count.assign(s_cnt.begin(), s_cnt.end());
    cloud.grad3d_accum.assign(s_3d.begin(), s_3d.end());
  }
}

inline DensityVolume voxelize(const GaussianCloud& cloud, const GridSpec& grid, const VoxelizeOptions& opts = {}) {
  CloudF32 cf(cloud);
  const sct_grid g = grid.c();
  std::vector<float> vol(grid.voxel_count());
  check(sct_voxelize_fwd_host(Context::get().handle(), &cf.c, &g, opts.cull_mahalanobis, vol.data()));
  DensityVolume v;
  v.dims = grid.dims;
  v.origin_mm = grid.origin_mm;
  v.spacing_mm = grid.spacing_mm;
  v.data.assign(vol.begin(), vol.end());
  return v;
}

inline void voxelize_backward(const GaussianCloud& cloud, const GridSpec& grid, const DensityVolume& dL_dV,
                              CloudGrads& grads, const VoxelizeOptions& opts = {}) {
  if (dL_dV.dims != grid.dims) throw DimMismatch("voxelize_backward: gradient volume dims mismatch");
  CloudF32 cf(cloud);
  GradsF32 gf(grads);
  const sct_grid g = grid.c();
  std::vector<float> dl(dL_dV.data.begin(), dL_dV.data.end());
  check(sct_voxelize_bwd_host(Context::get().handle(), &cf.c, &g, opts.cull_mahalanobis, dl.data(), &gf.c));
  gf.store(grads);
}

// ---- training (trainer.hpp / trainer.cpp:232-345) ------------------------------
struct ProjectionSet {  // simulator.hpp:57-66 (the fields train() reads)
  std::vector<Image> images;
  std::vector<double> angles_rad;
  ScannerConfig scanner;
  int n_views() const { return static_cast<int>(images.size()); }
};

struct TrainConfig {  // trainer.hpp:13-44 (the fields the loop uses)
  int iters = 30000;
  double lr_position = 0.0002, lr_density = 0.01, lr_scale = 0.005, lr_rotation = 0.001;
  double lr_final_ratio = 0.1;
  double lambda_ssim = 0.25, lambda_tv = 0.05;
  int tv_grid_dim = 32;
  int adaptive_start = 500, adaptive_end = 15000, densify_interval = 100;
  double densify_grad_threshold = 0.00005, prune_density_threshold = 0.005;
  double split_scale_threshold_frac = 0.01, split_factor = 1.6;
  uint64_t seed = 0;
  RenderMode mode = RenderMode::kRectified;
  std::array<int, 3> output_dims{64, 64, 64};
  int history_interval = 10;
  bool deterministic = false;  // zeroes wall-clock fields in history records
  // engine extensions: sync-free binning after a calibration iteration (capacity
  // = margin x measured pairs), and the non-finite check interval (1 = the reference)
  bool sync_free = true;
  double capacity_margin = 3.0;
  int check_every = 1;
};

struct HistoryRecord {  // trainer.hpp:51-59
  int iter = 0;
  double l1 = 0.0, dssim = 0.0, tv = 0.0, total = 0.0;
  int kernels = 0;
  double wall_ms = 0.0;
};

struct TrainResult {  // trainer.hpp:80-84
  GaussianCloud cloud;
  std::vector<HistoryRecord> history;
  double projection_norm = 1.0;
};

using TrainCallback = std::function<void(const HistoryRecord&)>;

// train() (trainer.hpp:88-89): the whole loop on the device (sct_trainer_*), the
// same random stream, adaptive control and history as the reference's.
inline TrainResult train(GaussianCloud cloud, const ProjectionSet& projections, const TrainConfig& cfg,
                         TrainCallback callback = nullptr) {
  if (projections.n_views() < 1) throw DataError("InsufficientViews: train: need >= 1 projection");
  if (cloud.size() < 1) throw ConfigError("train: empty initial cloud");
  const ScannerConfig& config = projections.scanner;
  const int w = config.detector_res_px[0], h = config.detector_res_px[1];
  const size_t px = static_cast<size_t>(w) * h;
  std::vector<float> proj(px * projections.n_views());
  double norm = 0.0;
  for (int v = 0; v < projections.n_views(); ++v) {
    const Image& im = projections.images[v];
    if (im.width != w || im.height != h) throw DimMismatch("train: projection dims differ from the detector");
    for (size_t i = 0; i < px; ++i) {
      proj[v * px + i] = static_cast<float>(im.data[i]);
      norm = std::max(norm, static_cast<double>(proj[v * px + i]));
    }
  }
  sct_train_cfg c{};
  c.iters = cfg.iters;
  c.lr_position = cfg.lr_position;
  c.lr_density = cfg.lr_density;
  c.lr_scale = cfg.lr_scale;
  c.lr_rotation = cfg.lr_rotation;
  c.lr_final_ratio = cfg.lr_final_ratio;
  c.lambda_ssim = cfg.lambda_ssim;
  c.lambda_tv = cfg.lambda_tv;
  c.tv_grid_dim = cfg.tv_grid_dim;
  c.adaptive_start = cfg.adaptive_start;
  c.adaptive_end = cfg.adaptive_end;
  c.densify_interval = cfg.densify_interval;
  c.densify_grad_threshold = cfg.densify_grad_threshold;
  c.prune_density_threshold = cfg.prune_density_threshold;
  c.split_scale_threshold_frac = cfg.split_scale_threshold_frac;
  c.split_factor = cfg.split_factor;
  c.seed = cfg.seed;
  c.mode = cfg.mode == RenderMode::kRectified ? SCT_MODE_RECTIFIED : SCT_MODE_BIASED;
  for (int k = 0; k < 3; ++k) c.output_dims[k] = cfg.output_dims[k];
  c.check_every = cfg.check_every;
  c.sync_free = cfg.sync_free ? 1 : 0;
  c.capacity_margin = cfg.capacity_margin;
  CloudF32 cf(cloud);
  const sct_scanner sc = config.c();
  sct_trainer* tr = nullptr;
  check(sct_trainer_create(Context::get().handle(), &cf.c, proj.data(), projections.angles_rad.data(),
                           projections.n_views(), &sc, &c, &tr));
  std::unique_ptr<sct_trainer, int (*)(sct_trainer*)> guard(tr, sct_trainer_destroy);
  TrainResult result;
  result.projection_norm = norm > 0.0 ? norm : 1.0;
  const auto t0 = std::chrono::steady_clock::now();
  sct_train_record rec{};
  for (int t = 1; t <= cfg.iters; ++t) {
    check(sct_trainer_step(tr, nullptr));
    if (t % cfg.history_interval == 0 || t == cfg.iters) {
      check(sct_trainer_record(tr, &rec));
      HistoryRecord hr;
      hr.iter = t;
      hr.l1 = rec.l1;
      hr.dssim = rec.dssim;
      hr.tv = rec.tv;
      hr.total = rec.total;
      hr.kernels = static_cast<int>(rec.kernels);
      hr.wall_ms = cfg.deterministic ? 0.0
                                     : std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                                           .count();
      result.history.push_back(hr);
      if (callback) callback(hr);
    }
  }
  check(sct_trainer_record(tr, &rec));
  const int64_t m = rec.kernels;
  std::vector<float> p[4] = {std::vector<float>(m), std::vector<float>(3 * m), std::vector<float>(3 * m),
                             std::vector<float>(4 * m)};
  sct_cloud out{};
  out.m = m;
  out.rho_raw = p[0].data();
  out.pos = p[1].data();
  out.scale_raw = p[2].data();
  out.rot = p[3].data();
  std::vector<float> s_norm(m), s_3d(3 * m);
  std::vector<int32_t> s_cnt(m);
  sct_stats st{};
  st.grad2d_norm_accum = s_norm.data();
  st.grad_count = s_cnt.data();
  st.grad3d_accum = s_3d.data();
  check(sct_trainer_download(tr, &out, nullptr, &st));
  result.cloud.s_min_mm = out.s_min_mm;
  result.cloud.rho_raw.assign(p[0].begin(), p[0].end());
  result.cloud.pos.assign(p[1].begin(), p[1].end());
  result.cloud.scale_raw.assign(p[2].begin(), p[2].end());
  result.cloud.rot.assign(p[3].begin(), p[3].end());
  result.cloud.grad2d_norm_accum.assign(s_norm.begin(), s_norm.end());
  result.cloud.grad_count.assign(s_cnt.begin(), s_cnt.end());
  result.cloud.grad3d_accum.assign(s_3d.begin(), s_3d.end());
  return result;
}

}  // namespace splatct_b200
