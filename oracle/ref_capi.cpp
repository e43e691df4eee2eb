// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, called by, or shipped
// with the product path (paper_2405_20693_b200/).
//
// C-ABI over the REFERENCE ITSELF: the unmodified reference sources under
// /root/reference/proj/core/src, compiled by oracle/Makefile (target `ref`)
// into oracle/_ref/libsplatct_ref.so against the build shims in
// oracle/ref_shim/ (Eigen subset, nlohmann::json, libpng stubs — the three
// dependencies absent from this image). The exported symbols carry the same
// names and signatures as the restated oracle's (`orc_*`,
// splatct_oracle.cpp / fixtures_oracle.cpp), so oracle/oracle.py can run
// every oracle call against either library and the tests can diff them.
//
// rasterizer.cpp, voxelizer.cpp and trainer.cpp are #included below (not
// edited) so that their internal-linkage helpers — project_impl
// (rasterizer.cpp:24-83), bin_kernels (voxelizer.cpp:52-88) and Adam
// (trainer.cpp:144-163) — can be called directly; the remaining reference
// translation units are compiled separately and linked.
// tests/helpers.hpp supplies the reference tests' own scene builders.

#include <rasterizer.cpp>
#include <trainer.cpp>
#include <voxelizer.cpp>

#include <cstring>
#include <limits>
#include <optional>
#include <string>

#include <omp.h>

#include "helpers.hpp"
#include "splatct/io.hpp"

namespace {

using namespace splatct;

thread_local std::string g_err;

int fail(int rc, const std::string& msg) {
  g_err = msg;
  return rc;
}

// geo = {l_so, l_sd, det_w_mm, det_h_mm, min xyz, max xyz, near_clip}, res = {W, H, parallel}
bool make_scanner(const double* geo, const int* res, ScannerConfig& c) {
  if (res[2] != 0) {
    g_err = "ConfigError: the reference has no parallel-beam geometry";
    return false;
  }
  c.l_so_mm = geo[0];
  c.l_sd_mm = geo[1];
  c.detector_size_mm = Vec2(geo[2], geo[3]);
  c.detector_res_px = Vec2i(res[0], res[1]);
  c.extent_min_mm = Vec3(geo[4], geo[5], geo[6]);
  c.extent_max_mm = Vec3(geo[7], geo[8], geo[9]);
  c.near_clip_mm = geo[10];
  return true;
}

RasterOptions make_opts(const double* o) {
  RasterOptions r;
  r.mode = static_cast<int>(o[0]) == 0 ? RenderMode::kRectified : RenderMode::kBiased;
  r.lowpass_eps_px = o[1];
  r.dilation_compensation = static_cast<int>(o[2]) != 0;
  r.freeze_jacobian = static_cast<int>(o[3]) != 0;
  r.cull_mahalanobis = o[4];
  return r;
}

GaussianCloud make_cloud(int m, double s_min, const double* rho, const double* pos, const double* sc,
                         const double* rot) {
  GaussianCloud c(s_min);
  c.rho_raw.assign(rho, rho + m);
  c.pos.assign(pos, pos + 3 * static_cast<size_t>(m));
  c.scale_raw.assign(sc, sc + 3 * static_cast<size_t>(m));
  c.rot.assign(rot, rot + 4 * static_cast<size_t>(m));
  const size_t mm = static_cast<size_t>(m);
  c.adam_m_rho.assign(mm, 0.0);
  c.adam_v_rho.assign(mm, 0.0);
  c.adam_m_pos.assign(3 * mm, 0.0);
  c.adam_v_pos.assign(3 * mm, 0.0);
  c.adam_m_scale.assign(3 * mm, 0.0);
  c.adam_v_scale.assign(3 * mm, 0.0);
  c.adam_m_rot.assign(4 * mm, 0.0);
  c.adam_v_rot.assign(4 * mm, 0.0);
  c.grad2d_norm_accum.assign(mm, 0.0);
  c.grad_count.assign(mm, 0);
  c.grad3d_accum.assign(3 * mm, 0.0);
  return c;
}

GridSpec make_grid(const int* dims, const double* origin, const double* spacing) {
  GridSpec g;
  g.dims = Vec3i(dims[0], dims[1], dims[2]);
  g.origin_mm = Vec3(origin[0], origin[1], origin[2]);
  g.spacing_mm = Vec3(spacing[0], spacing[1], spacing[2]);
  return g;
}

void add_into(double* dst, const std::vector<double>& src) {
  for (size_t i = 0; i < src.size(); ++i) dst[i] += src[i];
}

void export_projected(const ProjectedGaussian2D& p, double* out) {
  const double v[11] = {p.center_px.x(), p.center_px.y(), p.cov_px(0, 0), p.cov_px(0, 1), p.cov_px(1, 1),
                        p.conic_px(0, 0), p.conic_px(0, 1), p.conic_px(1, 1), p.amplitude, p.mu, p.depth_mm};
  std::memcpy(out, v, sizeof(v));
}

struct RefRendered {
  RenderedProjection r;
};

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const DimMismatch& e) {
    return fail(3, std::string("DimMismatch: ") + e.what());
  } catch (const DataError& e) {
    return fail(3, std::string("DataError: ") + e.what());
  } catch (const ConfigError& e) {
    return fail(2, std::string("ConfigError: ") + e.what());
  } catch (const KernelBehindSource& e) {
    return fail(3, std::string("KernelBehindSource: ") + e.what());
  } catch (const DivergenceDetected& e) {
    return fail(4, std::string("DivergenceDetected: ") + e.what());
  } catch (const std::exception& e) {
    return fail(1, e.what());
  }
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
const char* orc_flavour() { return "reference"; }
void orc_set_threads(int n) { splatct::set_num_threads(n > 0 ? n : 0); }
int orc_max_threads() { return omp_get_max_threads(); }

// --- RNG: std::mt19937_64 + libstdc++ distributions (the reference's own)
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
// tests/helpers.hpp:30-48
void orc_random_cloud(void* rp, int count, double pos_radius, double scale_min, double scale_max,
                      double s_min, double* rho_raw, double* pos, double* scale_raw, double* rot) {
  const GaussianCloud c = splatct::testing::random_cloud(*static_cast<std::mt19937_64*>(rp), count, pos_radius,
                                                         scale_min, scale_max, s_min);
  std::memcpy(rho_raw, c.rho_raw.data(), c.rho_raw.size() * sizeof(double));
  std::memcpy(pos, c.pos.data(), c.pos.size() * sizeof(double));
  std::memcpy(scale_raw, c.scale_raw.data(), c.scale_raw.size() * sizeof(double));
  std::memcpy(rot, c.rot.data(), c.rot.size() * sizeof(double));
}
// gaussian_cloud.cpp:48-72 add_kernel
void orc_kernel_to_raw(int n, double s_min, const double* rho, const double* scale, const double* rot_in,
                       double* rho_raw, double* scale_raw, double* rot_out) {
  GaussianCloud c(s_min);
  for (int i = 0; i < n; ++i) {
    RadiativeGaussian g;
    g.rho = rho[i];
    g.scale_mm = Vec3(scale[3 * i], scale[3 * i + 1], scale[3 * i + 2]);
    g.rotation = Vec4(rot_in[4 * i], rot_in[4 * i + 1], rot_in[4 * i + 2], rot_in[4 * i + 3]);
    c.add_kernel(g);
  }
  std::memcpy(rho_raw, c.rho_raw.data(), c.rho_raw.size() * sizeof(double));
  std::memcpy(scale_raw, c.scale_raw.data(), c.scale_raw.size() * sizeof(double));
  std::memcpy(rot_out, c.rot.data(), c.rot.size() * sizeof(double));
}
void orc_activate(int n, double s_min, const double* rho_raw, const double* scale_raw, double* rho,
                  double* scale) {
  for (int i = 0; i < n; ++i) {
    rho[i] = act_density(rho_raw[i]);
    for (int k = 0; k < 3; ++k) scale[3 * i + k] = act_scale(scale_raw[3 * i + k], s_min);
  }
}
// tests/helpers.hpp:115-121
void orc_random_image(void* rp, int n, double lo, double hi, double* out) {
  const Image img = splatct::testing::random_image(*static_cast<std::mt19937_64*>(rp), n, 1, lo, hi);
  std::memcpy(out, img.data.data(), img.data.size() * sizeof(double));
}

// --- geometry (geometry.cpp:76-138)
void orc_view_transform(const double* geo, const int* res, double theta, double* rot9, double* t3) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return;
  const ViewTransform v = view_transform(s, theta);
  for (int i = 0; i < 3; ++i) {
    t3[i] = v.t[i];
    for (int j = 0; j < 3; ++j) rot9[3 * i + j] = v.rot(i, j);
  }
}
void orc_detector(const double* geo, const int* res, double* out4) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return;
  const DetectorModel d = detector_model(s);
  out4[0] = d.fx_px;
  out4[1] = d.fy_px;
  out4[2] = d.cx_px;
  out4[3] = d.cy_px;
}
int orc_local_jacobian(const double* geo, const int* res, const double* p, double* j9) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return 2;
  return guarded([&] {
    const Mat3 j = local_jacobian(detector_model(s), Vec3(p[0], p[1], p[2]));
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) j9[3 * a + b] = j(a, b);
    return 0;
  });
}
void orc_ray_space_point(const double* geo, const int* res, const double* p, double* out) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return;
  const Vec3 r = ray_space_point(detector_model(s), Vec3(p[0], p[1], p[2]));
  for (int k = 0; k < 3; ++k) out[k] = r[k];
}
void orc_pixel_ray(const double* geo, const int* res, double theta, int u, int v, double* origin, double* dir) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return;
  const Ray r = pixel_ray(s, theta, u, v);
  for (int k = 0; k < 3; ++k) {
    origin[k] = r.origin_mm[k];
    dir[k] = r.dir[k];
  }
}

// --- cloud helpers (gaussian_cloud.cpp)
void orc_covariance(int m, double s_min, const double* rho, const double* pos, const double* sc,
                    const double* rot, int i, double* out9) {
  const GaussianCloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  const Mat3 s = c.covariance_at(i);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) out9[3 * a + b] = s(a, b);
}
double orc_density_at(int m, double s_min, const double* rho, const double* pos, const double* sc,
                      const double* rot, const double* x) {
  return density_at(make_cloud(m, s_min, rho, pos, sc, rot), Vec3(x[0], x[1], x[2]));
}
void orc_normalize_rotations(int m, double* rot) {
  GaussianCloud c;
  c.rot.assign(rot, rot + 4 * static_cast<size_t>(m));
  c.rho_raw.assign(m, 0.0);
  c.normalize_rotations();
  std::memcpy(rot, c.rot.data(), c.rot.size() * sizeof(double));
}
void orc_cov_param_grads(int m, double s_min, const double* rho, const double* pos, const double* sc,
                         const double* rot, int i, const double* g_sigma9, double* g_scale_raw, double* g_rot) {
  const GaussianCloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  Mat3 gs;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) gs(a, b) = g_sigma9[3 * a + b];
  CloudGrads g;
  g.resize(m);
  accumulate_covariance_param_grads(c, i, gs, g);
  add_into(g_scale_raw, g.scale_raw);
  add_into(g_rot, g.rot);
}
// tests/helpers.hpp:52-69
double orc_ray_march_density(int m, double s_min, const double* rho, const double* pos, const double* sc,
                             const double* rot, const double* origin, const double* dir, double step) {
  return splatct::testing::ray_march_density(make_cloud(m, s_min, rho, pos, sc, rot),
                                             Vec3(origin[0], origin[1], origin[2]), Vec3(dir[0], dir[1], dir[2]),
                                             step);
}

// --- rasterizer (rasterizer.cpp)
int orc_project_kernel(int m, double s_min, const double* rho, const double* pos, const double* sc,
                       const double* rot, int i, const double* geo, const int* res, double theta,
                       const double* opts, double* out) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return 0;
  const GaussianCloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  const auto p = project_kernel(c, i, view_transform(s, theta), detector_model(s), make_opts(opts));
  if (!p) return 0;
  export_projected(*p, out);
  return 1;
}
void* orc_render(int m, double s_min, const double* rho, const double* pos, const double* sc, const double* rot,
                 const double* geo, const int* res, double theta, const double* opts) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return nullptr;
  const GaussianCloud c = make_cloud(m, s_min, rho, pos, sc, rot);
  auto* h = new RefRendered();
  h->r = render(c, s, theta, make_opts(opts));
  return h;
}
void orc_render_free(void* h) { delete static_cast<RefRendered*>(h); }
void orc_render_image(void* h, double* out) {
  const auto& img = static_cast<RefRendered*>(h)->r.image;
  std::memcpy(out, img.data.data(), img.data.size() * sizeof(double));
}
int orc_render_n_visible(void* h) { return static_cast<int>(static_cast<RefRendered*>(h)->r.visible.size()); }
int64_t orc_render_n_pairs(void* h) {
  int64_t n = 0;
  for (const auto& l : static_cast<RefRendered*>(h)->r.tile_visible) n += static_cast<int64_t>(l.size());
  return n;
}
void orc_render_tile_lists(void* h, int64_t* offsets, int32_t* kernel_idx) {
  const auto& r = static_cast<RefRendered*>(h)->r;
  int64_t o = 0;
  for (size_t t = 0; t < r.tile_visible.size(); ++t) {
    offsets[t] = o;
    for (int vi : r.tile_visible[t]) kernel_idx[o++] = r.visible[vi].kernel_index;
  }
  offsets[r.tile_visible.size()] = o;
}
void orc_render_visible(void* h, int32_t* kidx, double* rec) {
  const auto& r = static_cast<RefRendered*>(h)->r;
  for (size_t vi = 0; vi < r.visible.size(); ++vi) {
    kidx[vi] = r.visible[vi].kernel_index;
    export_projected(r.visible[vi], rec + 11 * vi);
  }
}
int orc_render_backward(void* h, int m, double s_min, const double* rho, const double* pos, const double* sc,
                        const double* rot, const double* geo, const int* res, double theta, const double* opts,
                        const double* dL, double* g_rho, double* g_pos, double* g_sc, double* g_rot,
                        double* st_norm, int32_t* st_count, double* st_3d) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return 2;
  const auto& fwd = static_cast<RefRendered*>(h)->r;
  return guarded([&] {
    GaussianCloud c = make_cloud(m, s_min, rho, pos, sc, rot);
    Image up(fwd.image.width, fwd.image.height);
    std::memcpy(up.data.data(), dL, up.data.size() * sizeof(double));
    if (fwd.image.width != s.detector_res_px.x() || fwd.image.height != s.detector_res_px.y())
      up = Image(1, 1);  // make the reference raise its own DimMismatch
    CloudGrads g;
    g.resize(m);
    const bool stats = st_norm != nullptr;
    render_backward(c, s, theta, fwd, up, g, make_opts(opts), stats);
    add_into(g_rho, g.rho_raw);
    add_into(g_pos, g.pos);
    add_into(g_sc, g.scale_raw);
    add_into(g_rot, g.rot);
    if (stats) {
      add_into(st_norm, c.grad2d_norm_accum);
      for (int i = 0; i < m; ++i) st_count[i] += c.grad_count[i];
      add_into(st_3d, c.grad3d_accum);
    }
    return 0;
  });
}

// --- voxelizer (voxelizer.cpp)
void orc_grid_for_extent(const double* lo, const double* hi, const int* dims, double* origin, double* spacing) {
  const GridSpec g = grid_for_extent(Vec3(lo[0], lo[1], lo[2]), Vec3(hi[0], hi[1], hi[2]),
                                     Vec3i(dims[0], dims[1], dims[2]));
  for (int k = 0; k < 3; ++k) {
    origin[k] = g.origin_mm[k];
    spacing[k] = g.spacing_mm[k];
  }
}
void orc_voxelize(int m, double s_min, const double* rho, const double* pos, const double* sc, const double* rot,
                  const int* dims, const double* origin, const double* spacing, double cull, double* vol) {
  VoxelizeOptions o;
  o.cull_mahalanobis = cull;
  const DensityVolume v = voxelize(make_cloud(m, s_min, rho, pos, sc, rot), make_grid(dims, origin, spacing), o);
  std::memcpy(vol, v.data.data(), v.data.size() * sizeof(double));
}
int orc_voxelize_backward(int m, double s_min, const double* rho, const double* pos, const double* sc,
                          const double* rot, const int* dims, const double* origin, const double* spacing,
                          double cull, const double* dL, double* g_rho, double* g_pos, double* g_sc,
                          double* g_rot) {
  return guarded([&] {
    const GridSpec grid = make_grid(dims, origin, spacing);
    DensityVolume up(grid);
    std::memcpy(up.data.data(), dL, up.data.size() * sizeof(double));
    VoxelizeOptions o;
    o.cull_mahalanobis = cull;
    CloudGrads g;
    g.resize(m);
    voxelize_backward(make_cloud(m, s_min, rho, pos, sc, rot), grid, up, g, o);
    add_into(g_rho, g.rho_raw);
    add_into(g_pos, g.pos);
    add_into(g_sc, g.scale_raw);
    add_into(g_rot, g.rot);
    return 0;
  });
}
// bin_kernels (voxelizer.cpp:52-88): offsets[B+1], idx[pairs]; pair count when offsets == nullptr
int64_t orc_voxel_bins(int m, double s_min, const double* rho, const double* pos, const double* sc,
                       const double* rot, const int* dims, const double* origin, const double* spacing,
                       double cull, int64_t* offsets, int32_t* idx) {
  const TileBins b = bin_kernels(make_cloud(m, s_min, rho, pos, sc, rot), make_grid(dims, origin, spacing), cull);
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
void orc_random_subvolume_spec(void* rp, const double* lo, const double* hi, const double* spacing, int d,
                               double* origin) {
  const GridSpec g = random_subvolume_spec(Vec3(lo[0], lo[1], lo[2]), Vec3(hi[0], hi[1], hi[2]),
                                           Vec3(spacing[0], spacing[1], spacing[2]), d,
                                           *static_cast<std::mt19937_64*>(rp));
  for (int k = 0; k < 3; ++k) origin[k] = g.origin_mm[k];
}

// --- objectives (objectives.cpp)
int orc_tv3d(const int* dims, const double* vol, double* value, double* grad) {
  return guarded([&] {
    GridSpec g;
    g.dims = Vec3i(dims[0], dims[1], dims[2]);
    DensityVolume v(g);
    std::memcpy(v.data.data(), vol, v.data.size() * sizeof(double));
    const VolumeLossResult r = tv3d_loss(v);
    *value = r.value;
    std::memcpy(grad, r.grad.data.data(), r.grad.data.size() * sizeof(double));
    return 0;
  });
}
int orc_l1(int n, const double* r, const double* m, double* value, double* grad) {
  return guarded([&] {
    Image a(n, 1), b(n, 1);
    std::memcpy(a.data.data(), r, n * sizeof(double));
    std::memcpy(b.data.data(), m, n * sizeof(double));
    const LossResult l = l1_loss(a, b);
    *value = l.value;
    std::memcpy(grad, l.grad.data.data(), n * sizeof(double));
    return 0;
  });
}
int orc_dssim(int w, int h, const double* a, const double* b, double* value, double* grad) {
  return guarded([&] {
    Image A(w, h), B(w, h);
    std::memcpy(A.data.data(), a, sizeof(double) * w * h);
    std::memcpy(B.data.data(), b, sizeof(double) * w * h);
    const LossResult l = dssim_loss(A, B);
    *value = l.value;
    std::memcpy(grad, l.grad.data.data(), sizeof(double) * w * h);
    return 0;
  });
}

// --- adaptive control (trainer.cpp:167-230 adaptive_control, unmodified)
// arrays: 0 rho_raw, 1 pos, 2 scale_raw, 3 rot, 4..11 Adam m/v (rho, pos, scale, rot).
struct ACResult {
  std::vector<double> a[12];
  std::vector<double> st_norm, st_3d;
  std::vector<int> st_count;
  int pruned = 0, cloned = 0, split = 0;
};
void* orc_adaptive_control(void* rp, int m, double s_min, const double* const* arrays, const double* norm_acc,
                           const int32_t* count, const double* g3d, double prune_thr, double densify_thr,
                           double split_frac, double split_factor, const double* extent_size) {
  GaussianCloud c = make_cloud(m, s_min, arrays[0], arrays[1], arrays[2], arrays[3]);
  std::vector<double>* adam[8] = {&c.adam_m_rho, &c.adam_v_rho, &c.adam_m_pos,   &c.adam_v_pos,
                                  &c.adam_m_scale, &c.adam_v_scale, &c.adam_m_rot, &c.adam_v_rot};
  const int stride[12] = {1, 3, 3, 4, 1, 1, 3, 3, 3, 3, 4, 4};
  for (int a = 0; a < 8; ++a) adam[a]->assign(arrays[4 + a], arrays[4 + a] + stride[4 + a] * m);
  c.grad2d_norm_accum.assign(norm_acc, norm_acc + m);
  c.grad_count.assign(count, count + m);
  c.grad3d_accum.assign(g3d, g3d + 3 * m);
  TrainConfig cfg;
  cfg.prune_density_threshold = prune_thr;
  cfg.densify_grad_threshold = densify_thr;
  cfg.split_scale_threshold_frac = split_frac;
  cfg.split_factor = split_factor;
  const AdaptiveControlStats st = adaptive_control(c, cfg, Vec3(extent_size[0], extent_size[1], extent_size[2]),
                                                   *static_cast<std::mt19937_64*>(rp));
  auto* res = new ACResult();
  res->a[0] = c.rho_raw;
  res->a[1] = c.pos;
  res->a[2] = c.scale_raw;
  res->a[3] = c.rot;
  for (int a = 0; a < 8; ++a) res->a[4 + a] = *adam[a];
  res->st_norm = c.grad2d_norm_accum;
  res->st_count = c.grad_count;
  res->st_3d = c.grad3d_accum;
  res->pruned = st.pruned;
  res->cloned = st.cloned;
  res->split = st.split;
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
// the adaptive statistics the cloud carries after adaptive_control
void orc_ac_stats(void* h, double* norm_acc, int32_t* count, double* g3d) {
  auto* r = static_cast<ACResult*>(h);
  std::memcpy(norm_acc, r->st_norm.data(), r->st_norm.size() * sizeof(double));
  for (size_t i = 0; i < r->st_count.size(); ++i) count[i] = r->st_count[i];
  std::memcpy(g3d, r->st_3d.data(), r->st_3d.size() * sizeof(double));
}
void orc_ac_free(void* h) { delete static_cast<ACResult*>(h); }
// trainer.cpp:270: std::shuffle(order.begin(), order.end(), rng) on a std::vector<int>
void orc_shuffle(void* rp, int n, int32_t* values) {
  std::vector<int> order(values, values + n);
  std::shuffle(order.begin(), order.end(), *static_cast<std::mt19937_64*>(rp));
  for (int i = 0; i < n; ++i) values[i] = order[i];
}
void orc_normal_draws(void* rp, int n, double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rp);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int i = 0; i < n; ++i) out[i] = gauss(rng);
}

// --- optimizer (trainer.cpp:34-36 lr_at, :144-163 Adam::step)
double orc_lr_at(double lr_init, double ratio, int t, int iters) { return lr_at(lr_init, ratio, t, iters); }
void orc_adam_step(int64_t n, double* params, double* m, double* v, const double* g, double lr, int step,
                   double beta1, double beta2, double eps) {
  Adam adam;
  adam.beta1 = beta1;
  adam.beta2 = beta2;
  adam.eps = eps;
  adam.step_count = step;
  std::vector<double> P(params, params + n), M(m, m + n), V(v, v + n), G(g, g + n);
  adam.step(P, M, V, G, lr);
  std::memcpy(params, P.data(), n * sizeof(double));
  std::memcpy(m, M.data(), n * sizeof(double));
  std::memcpy(v, V.data(), n * sizeof(double));
}

// --- the reference training loop (trainer.cpp:232-345 train, unmodified).
// images [V][H][W], angles [V]; cfg_d = {lr_pos, lr_rho, lr_scale, lr_rot, lr_final_ratio, lambda_ssim,
// lambda_tv, densify_grad_threshold, prune_density_threshold, split_scale_threshold_frac, split_factor};
// cfg_i = {iters, tv_grid_dim, adaptive_start, adaptive_end, densify_interval, mode, out_x, out_y, out_z,
// history_interval}. Returns a handle to the trained cloud (read with orc_ac_*) and fills
// history [iters/history_interval][6] = {iter, l1, dssim, tv, total, kernels} up to max_hist rows.
void* orc_train(int m, double s_min, const double* rho, const double* pos, const double* sc, const double* rot,
                const double* geo, const int* res, int n_views, const double* angles, const double* images,
                const double* cfg_d, const int* cfg_i, uint64_t seed, double* history, int max_hist,
                int* n_hist) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return nullptr;
  try {
    ProjectionSet ps;
    ps.scanner = s;
    ps.angles_rad.assign(angles, angles + n_views);
    ps.scanner.angles_rad = ps.angles_rad;
    const size_t npx = static_cast<size_t>(res[0]) * res[1];
    for (int v = 0; v < n_views; ++v) {
      Image img(res[0], res[1]);
      std::memcpy(img.data.data(), images + v * npx, npx * sizeof(double));
      ps.images.push_back(img);
    }
    TrainConfig cfg;
    cfg.lr_position = cfg_d[0];
    cfg.lr_density = cfg_d[1];
    cfg.lr_scale = cfg_d[2];
    cfg.lr_rotation = cfg_d[3];
    cfg.lr_final_ratio = cfg_d[4];
    cfg.lambda_ssim = cfg_d[5];
    cfg.lambda_tv = cfg_d[6];
    cfg.densify_grad_threshold = cfg_d[7];
    cfg.prune_density_threshold = cfg_d[8];
    cfg.split_scale_threshold_frac = cfg_d[9];
    cfg.split_factor = cfg_d[10];
    cfg.iters = cfg_i[0];
    cfg.tv_grid_dim = cfg_i[1];
    cfg.adaptive_start = cfg_i[2];
    cfg.adaptive_end = cfg_i[3];
    cfg.densify_interval = cfg_i[4];
    cfg.mode = cfg_i[5] == 0 ? RenderMode::kRectified : RenderMode::kBiased;
    cfg.output_dims = Vec3i(cfg_i[6], cfg_i[7], cfg_i[8]);
    cfg.history_interval = cfg_i[9];
    cfg.seed = seed;
    cfg.deterministic = true;
    const TrainResult tr = train(make_cloud(m, s_min, rho, pos, sc, rot), ps, cfg);
    int nh = 0;
    for (const auto& h : tr.history) {
      if (nh >= max_hist) break;
      const double row[6] = {static_cast<double>(h.iter), h.l1, h.dssim, h.tv, h.total,
                             static_cast<double>(h.kernels)};
      std::memcpy(history + 6 * nh, row, sizeof(row));
      ++nh;
    }
    *n_hist = nh;
    auto* out = new ACResult();
    const GaussianCloud& c = tr.cloud;
    out->a[0] = c.rho_raw;
    out->a[1] = c.pos;
    out->a[2] = c.scale_raw;
    out->a[3] = c.rot;
    const std::vector<double>* adam[8] = {&c.adam_m_rho, &c.adam_v_rho, &c.adam_m_pos,   &c.adam_v_pos,
                                          &c.adam_m_scale, &c.adam_v_scale, &c.adam_m_rot, &c.adam_v_rot};
    for (int a = 0; a < 8; ++a) out->a[4 + a] = *adam[a];
    out->st_norm = c.grad2d_norm_accum;
    out->st_count = c.grad_count;
    out->st_3d = c.grad3d_accum;
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// --- fixtures (simulator.cpp, fdk.cpp)
// ell = [n][8] {intensity, a, b, c, x0, y0, z0, phi}
void orc_phantom(int n_ell, const double* ell, const int* dims, const double* lo, const double* hi, float* out) {
  std::vector<PhantomEllipsoid> e(n_ell);
  for (int i = 0; i < n_ell; ++i) {
    const double* E = ell + 8 * i;
    e[i] = PhantomEllipsoid{E[0], E[1], E[2], E[3], E[4], E[5], E[6], E[7]};
  }
  const DensityVolume v = phantom_from_ellipsoids(e, Vec3i(dims[0], dims[1], dims[2]), Vec3(lo[0], lo[1], lo[2]),
                                                  Vec3(hi[0], hi[1], hi[2]));
  for (size_t i = 0; i < v.data.size(); ++i) out[i] = static_cast<float>(v.data[i]);
}
// the reference's own Shepp-Logan table (simulator.cpp:14-27)
int orc_shepp_logan(double* ell, int max_n) {
  const auto& t = shepp_logan_ellipsoids_3d();
  const int n = static_cast<int>(t.size());
  for (int i = 0; i < n && i < max_n; ++i) {
    const double row[8] = {t[i].intensity, t[i].a, t[i].b, t[i].c, t[i].x0, t[i].y0, t[i].z0, t[i].phi_rad};
    std::memcpy(ell + 8 * i, row, sizeof(row));
  }
  return n;
}
DensityVolume volume_from(const float* vol, const int* dims, const double* origin, const double* spacing) {
  DensityVolume v(make_grid(dims, origin, spacing));
  for (size_t i = 0; i < v.data.size(); ++i) v.data[i] = vol[i];
  return v;
}
double orc_sample_trilinear(const float* vol, const int* dims, const double* origin, const double* spacing,
                            const double* x) {
  return sample_trilinear(volume_from(vol, dims, origin, spacing), Vec3(x[0], x[1], x[2]));
}
int orc_project_volume(const float* vol, const int* dims, const double* origin, const double* spacing,
                       const double* geo, const int* res, double theta, double step_mm, double* out) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return 2;
  return guarded([&] {
    const Image img = project_volume(volume_from(vol, dims, origin, spacing), s, theta, step_mm);
    std::memcpy(out, img.data.data(), img.data.size() * sizeof(double));
    return 0;
  });
}
int orc_add_noise(const float* clean, int n, double i0, double gauss_sigma, uint64_t seed, int view, double* out) {
  return guarded([&] {
    Image img(n, 1);
    for (int i = 0; i < n; ++i) img.data[i] = clean[i];
    NoiseParams p;
    p.i0 = i0;
    p.gauss_sigma = gauss_sigma;
    p.seed = seed;
    std::mt19937_64 rng = view_rng(seed, view);
    const Image r = add_noise(img, p, rng);
    std::memcpy(out, r.data.data(), n * sizeof(double));
    return 0;
  });
}
int orc_fdk(const float* images, int n_views, const double* geo, const int* res, const double* angles,
            const int* dims, const double* origin, const double* spacing, int window, double* out) {
  ScannerConfig s;
  if (!make_scanner(geo, res, s)) return 2;
  return guarded([&] {
    ProjectionSet ps;
    ps.scanner = s;
    ps.angles_rad.assign(angles, angles + n_views);
    ps.scanner.angles_rad = ps.angles_rad;
    const size_t npx = static_cast<size_t>(res[0]) * res[1];
    for (int v = 0; v < n_views; ++v) {
      Image img(res[0], res[1]);
      for (size_t i = 0; i < npx; ++i) img.data[i] = images[v * npx + i];
      ps.images.push_back(img);
    }
    const RampWindow w = window == 0 ? RampWindow::kRamLak : (window == 1 ? RampWindow::kHann : RampWindow::kAuto);
    const DensityVolume vol = fdk_reconstruct(ps, make_grid(dims, origin, spacing), w);
    std::memcpy(out, vol.data.data(), vol.data.size() * sizeof(double));
    return 0;
  });
}
void orc_nn_distances(int n, const double* pts, double* out) {
  std::vector<Vec3> p(n);
  for (int i = 0; i < n; ++i) p[i] = Vec3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  const std::vector<double> d = nearest_neighbor_distances(p);
  std::memcpy(out, d.data(), d.size() * sizeof(double));
}
int orc_sample_init_cloud(void* rp, const float* vol, const int* dims, const double* origin, const double* spacing,
                          int count, double threshold, double density_scale, double s_min, double* rho_raw,
                          double* pos, double* scale_raw, double* rot) {
  return guarded([&] {
    InitParams ip;
    ip.count = count;
    ip.density_threshold = threshold;
    ip.density_scale = density_scale;
    const GaussianCloud c = sample_init_cloud(volume_from(vol, dims, origin, spacing), ip, s_min,
                                              *static_cast<std::mt19937_64*>(rp));
    std::memcpy(rho_raw, c.rho_raw.data(), c.rho_raw.size() * sizeof(double));
    std::memcpy(pos, c.pos.data(), c.pos.size() * sizeof(double));
    std::memcpy(scale_raw, c.scale_raw.data(), c.scale_raw.size() * sizeof(double));
    std::memcpy(rot, c.rot.data(), c.rot.size() * sizeof(double));
    return 0;
  });
}

// --- I/O containers (io.cpp): round trips for the f4 parity tests
int orc_save_cloud(const char* path, int m, double s_min, const double* rho, const double* pos, const double* sc,
                   const double* rot) {
  return guarded([&] {
    save_cloud(make_cloud(m, s_min, rho, pos, sc, rot), path);
    return 0;
  });
}
int orc_load_cloud(const char* path, int max_m, int* m, double* s_min, double* rho, double* pos, double* sc,
                   double* rot) {
  return guarded([&] {
    const GaussianCloud c = load_cloud(path);
    *m = c.size();
    *s_min = c.s_min();
    if (c.size() > max_m) return 0;
    std::memcpy(rho, c.rho_raw.data(), c.rho_raw.size() * sizeof(double));
    std::memcpy(pos, c.pos.data(), c.pos.size() * sizeof(double));
    std::memcpy(sc, c.scale_raw.data(), c.scale_raw.size() * sizeof(double));
    std::memcpy(rot, c.rot.data(), c.rot.size() * sizeof(double));
    return 0;
  });
}
int orc_write_volume(const char* path, const int* dims, const double* origin, const double* spacing,
                     const double* data) {
  return guarded([&] {
    DensityVolume v(make_grid(dims, origin, spacing));
    std::memcpy(v.data.data(), data, v.data.size() * sizeof(double));
    write_volume(v, path);
    return 0;
  });
}
int orc_read_volume(const char* path, int64_t max_n, int* dims, double* origin, double* spacing, double* data) {
  return guarded([&] {
    const DensityVolume v = read_volume(path);
    for (int k = 0; k < 3; ++k) {
      dims[k] = v.dims[k];
      origin[k] = v.origin_mm[k];
      spacing[k] = v.spacing_mm[k];
    }
    if (static_cast<int64_t>(v.data.size()) <= max_n)
      std::memcpy(data, v.data.data(), v.data.size() * sizeof(double));
    return 0;
  });
}
int orc_write_image(const char* path, int w, int h, const double* data) {
  return guarded([&] {
    Image img(w, h);
    std::memcpy(img.data.data(), data, img.data.size() * sizeof(double));
    write_image(img, path);
    return 0;
  });
}
int orc_read_image(const char* path, int64_t max_n, int* wh, double* data) {
  return guarded([&] {
    const Image img = read_image(path);
    wh[0] = img.width;
    wh[1] = img.height;
    if (static_cast<int64_t>(img.data.size()) <= max_n)
      std::memcpy(data, img.data.data(), img.data.size() * sizeof(double));
    return 0;
  });
}

}  // extern "C"
