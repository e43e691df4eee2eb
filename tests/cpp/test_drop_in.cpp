// C++ drop-in check: the reference-shaped API of include/splatct_b200.hpp
// (render / render_backward / voxelize / voxelize_backward with the
// reference's types and accumulate semantics) against the FP64 oracle
// (oracle/liborc.so, test infrastructure) on the reference test scanner.
// Prints one "PASS"/"FAIL" line per check; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <vector>

#include "splatct_b200.hpp"

extern "C" {  // oracle C ABI (oracle/splatct_oracle.cpp)
void* orc_rng_new(uint64_t seed);
void orc_rng_free(void*);
void orc_random_cloud(void*, int, double, double, double, double, double*, double*, double*, double*);
void orc_random_image(void*, int, double, double, double*);
void* orc_render(int, double, const double*, const double*, const double*, const double*, const double*,
                 const int*, double, const double*);
void orc_render_free(void*);
void orc_render_image(void*, double*);
int orc_render_n_visible(void*);
void orc_render_visible(void*, int32_t*, double*);
void orc_render_tile_lists(void*, int64_t*, int32_t*);
int orc_render_backward(void*, int, double, const double*, const double*, const double*, const double*,
                        const double*, const int*, double, const double*, const double*, double*, double*, double*,
                        double*, double*, int32_t*, double*);
void orc_voxelize(int, double, const double*, const double*, const double*, const double*, const int*,
                  const double*, const double*, double, double*);
int orc_voxelize_backward(int, double, const double*, const double*, const double*, const double*, const int*,
                          const double*, const double*, double, const double*, double*, double*, double*, double*);
}

namespace S = splatct_b200;

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

static int report(const char* what, double err, double tol) {
  const bool ok = err <= tol;
  std::printf("%s %-40s rel L2 %.3e (tol %.0e)\n", ok ? "PASS" : "FAIL", what, err, tol);
  return ok ? 0 : 1;
}

int main() {
  int fails = 0;
  const int m = 1500;
  S::GaussianCloud cloud;
  cloud.s_min_mm = 2e-4;
  cloud.rho_raw.resize(m);
  cloud.pos.resize(3 * m);
  cloud.scale_raw.resize(3 * m);
  cloud.rot.resize(4 * m);
  void* rng = orc_rng_new(21);
  orc_random_cloud(rng, m, 0.85, 0.02, 0.08, 2e-4, cloud.rho_raw.data(), cloud.pos.data(), cloud.scale_raw.data(),
                   cloud.rot.data());
  // the engine computes on fp32 parameters: give the oracle the same values
  for (auto* v : {&cloud.rho_raw, &cloud.pos, &cloud.scale_raw, &cloud.rot})
    for (double& x : *v) x = static_cast<float>(x);

  S::ScannerConfig cfg;  // tests/helpers.hpp:18-28 desk scanner
  cfg.detector_res_px = {129, 129};
  const double geo[11] = {8.0, 12.0, 5.6, 5.6, -1, -1, -1, 1, 1, 1, 0.0};
  const int res[2] = {129, 129};
  const double opts[5] = {0, 0.3, 1, 0, 3.0348542587702925};
  const double theta = 0.37;

  // render
  S::RenderedProjection fwd = S::render(cloud, cfg, theta);
  void* ref = orc_render(m, cloud.s_min_mm, cloud.rho_raw.data(), cloud.pos.data(), cloud.scale_raw.data(),
                         cloud.rot.data(), geo, res, theta, opts);
  std::vector<double> ref_img(129 * 129);
  orc_render_image(ref, ref_img.data());
  fails += report("render image", rel_l2(fwd.image.data, ref_img), 1e-4);
  // RenderedProjection::visible / tile_visible (rasterizer.hpp:41-51) on request
  {
    const std::vector<S::ProjectedGaussian2D> vis = fwd.visible(cloud, cfg);
    const int nv = orc_render_n_visible(ref);
    std::vector<int32_t> rk(nv > 0 ? nv : 1);
    std::vector<double> rr(11 * (nv > 0 ? nv : 1));
    orc_render_visible(ref, rk.data(), rr.data());
    int idx_bad = static_cast<int>(vis.size()) != nv;
    std::vector<double> mine, theirs;
    for (int i = 0; !idx_bad && i < nv; ++i) {
      idx_bad += vis[i].kernel_index != rk[i];
      const S::ProjectedGaussian2D& g = vis[i];
      const double v[11] = {g.center_px[0], g.center_px[1], g.cov_px[0][0], g.cov_px[0][1], g.cov_px[1][1],
                            g.conic_px[0][0], g.conic_px[0][1], g.conic_px[1][1], g.amplitude, g.mu, g.depth_mm};
      for (int k = 0; k < 11; ++k) {
        mine.push_back(v[k]);
        theirs.push_back(rr[11 * i + k]);
      }
    }
    fails += report("visible kernel indices (exact)", idx_bad, 0);
    fails += report("visible records (FP64)", idx_bad ? 1.0 : rel_l2(mine, theirs), 1e-10);
    const std::vector<std::vector<int>> tv = fwd.tile_visible(vis);
    const int T = fwd.tiles_x * fwd.tiles_y;
    std::vector<int64_t> off(T + 1);
    std::vector<int32_t> tk(static_cast<size_t>(nv > 0 ? nv : 1) * T);  // bound: every visible kernel on every tile
    orc_render_tile_lists(ref, off.data(), tk.data());
    int tv_bad = static_cast<int>(tv.size()) != T;
    for (int t = 0; !tv_bad && t < T; ++t) {
      tv_bad += static_cast<int64_t>(tv[t].size()) != off[t + 1] - off[t];
      for (size_t j = 0; !tv_bad && j < tv[t].size(); ++j) tv_bad += vis[tv[t][j]].kernel_index != tk[off[t] + j];
    }
    fails += report("tile_visible (exact)", tv_bad, 0);
  }

  // render_backward (accumulate into zeroed grads, with adaptive stats)
  S::Image up(129, 129);
  orc_random_image(rng, 129 * 129, -1.0, 1.0, up.data.data());
  for (double& x : up.data) x = static_cast<float>(x);
  S::CloudGrads g;
  g.resize(m);
  S::render_backward(cloud, cfg, theta, fwd, up, g, {}, true);
  std::vector<double> gr(m), gp(3 * m), gs(3 * m), gq(4 * m), sn(m), s3(3 * m);
  std::vector<int32_t> sc(m);
  orc_render_backward(ref, m, cloud.s_min_mm, cloud.rho_raw.data(), cloud.pos.data(), cloud.scale_raw.data(),
                      cloud.rot.data(), geo, res, theta, opts, up.data.data(), gr.data(), gp.data(), gs.data(),
                      gq.data(), sn.data(), sc.data(), s3.data());
  fails += report("render_backward d/drho_raw", rel_l2(g.rho_raw, gr), 1e-3);
  fails += report("render_backward d/dpos", rel_l2(g.pos, gp), 1e-3);
  fails += report("render_backward d/dscale_raw", rel_l2(g.scale_raw, gs), 1e-3);
  fails += report("render_backward d/drot", rel_l2(g.rot, gq), 1e-3);
  fails += report("adaptive stats grad2d_norm_accum", rel_l2(cloud.grad2d_norm_accum, sn), 1e-3);
  int cnt_bad = 0;
  for (int i = 0; i < m; ++i) cnt_bad += cloud.grad_count[i] != sc[i];
  fails += report("adaptive stats grad_count (exact)", cnt_bad, 0);
  // accumulate semantics: a second call doubles the gradients
  std::vector<double> first = g.pos;
  S::render_backward(cloud, cfg, theta, fwd, up, g);
  std::vector<double> twice(first.size());
  for (size_t i = 0; i < first.size(); ++i) twice[i] = 2 * first[i];
  fails += report("render_backward accumulates (+=)", rel_l2(g.pos, twice), 1e-6);
  orc_render_free(ref);

  // voxelize / voxelize_backward on a non-multiple-of-8 grid
  const S::GridSpec grid = S::grid_for_extent({-1, -1, -1}, {1, 1, 1}, {36, 30, 28});
  const S::DensityVolume vol = S::voxelize(cloud, grid);
  std::vector<double> rvol(grid.voxel_count());
  orc_voxelize(m, cloud.s_min_mm, cloud.rho_raw.data(), cloud.pos.data(), cloud.scale_raw.data(), cloud.rot.data(),
               grid.dims.data(), grid.origin_mm.data(), grid.spacing_mm.data(), 3.3681993876652464, rvol.data());
  fails += report("voxelize volume", rel_l2(vol.data, rvol), 1e-4);
  S::DensityVolume dV = vol;
  orc_random_image(rng, static_cast<int>(grid.voxel_count()), -1.0, 1.0, dV.data.data());
  for (double& x : dV.data) x = static_cast<float>(x);
  S::CloudGrads gv;
  gv.resize(m);
  S::voxelize_backward(cloud, grid, dV, gv);
  std::vector<double> vr(m, 0), vp(3 * m, 0), vs(3 * m, 0), vq(4 * m, 0);
  orc_voxelize_backward(m, cloud.s_min_mm, cloud.rho_raw.data(), cloud.pos.data(), cloud.scale_raw.data(),
                        cloud.rot.data(), grid.dims.data(), grid.origin_mm.data(), grid.spacing_mm.data(),
                        3.3681993876652464, dV.data.data(), vr.data(), vp.data(), vs.data(), vq.data());
  fails += report("voxelize_backward d/drho_raw", rel_l2(gv.rho_raw, vr), 1e-3);
  fails += report("voxelize_backward d/dpos", rel_l2(gv.pos, vp), 1e-3);
  fails += report("voxelize_backward d/dscale_raw", rel_l2(gv.scale_raw, vs), 1e-3);
  fails += report("voxelize_backward d/drot", rel_l2(gv.rot, vq), 1e-3);

  // errors map to the reference's exception types
  try {
    S::render_backward(cloud, cfg, theta, fwd, S::Image(8, 8), g);
    fails += report("DimMismatch thrown", 1, 0);
  } catch (const S::DimMismatch&) {
    fails += report("DimMismatch thrown", 0, 0);
  }
  // backward with another angle / other options than the forward call: rejected
  try {
    S::render_backward(cloud, cfg, theta + 0.1, fwd, up, g);
    fails += report("ConfigError on theta mismatch", 1, 0);
  } catch (const S::ConfigError&) {
    fails += report("ConfigError on theta mismatch", 0, 0);
  }
  try {
    S::RasterOptions frozen;
    frozen.freeze_jacobian = true;
    S::render_backward(cloud, cfg, theta, fwd, up, g, frozen);
    fails += report("ConfigError on opts mismatch", 1, 0);
  } catch (const S::ConfigError&) {
    fails += report("ConfigError on opts mismatch", 0, 0);
  }
  // train() (trainer.hpp:88-89) on the device: a short seeded run with TV and
  // adaptive control; history bookkeeping and bit-reproducibility (test_trainer.cpp:87-105)
  {
    S::ProjectionSet ps;
    ps.scanner = cfg;
    for (int v = 0; v < 4; ++v) {
      ps.angles_rad.push_back(2.0 * M_PI * v / 4);
      ps.images.push_back(S::render(cloud, cfg, ps.angles_rad.back()).image);
    }
    S::GaussianCloud init = cloud;
    for (double& x : init.rho_raw) x -= 0.3;  // start away from the target
    S::TrainConfig tc;
    tc.iters = 9;
    tc.output_dims = {32, 32, 32};
    tc.tv_grid_dim = 8;
    tc.adaptive_start = 3;
    tc.densify_interval = 3;
    tc.densify_grad_threshold = 1e-7;
    tc.history_interval = 1;
    tc.deterministic = true;
    tc.seed = 5;
    int calls = 0;
    const S::TrainResult r1 = S::train(init, ps, tc, [&](const S::HistoryRecord&) { ++calls; });
    const S::TrainResult r2 = S::train(init, ps, tc);
    int bad = static_cast<int>(r1.history.size()) != 9 || calls != 9;
    for (size_t i = 0; !bad && i < r1.history.size(); ++i) {
      const S::HistoryRecord &a = r1.history[i], &b = r2.history[i];
      bad += a.iter != static_cast<int>(i) + 1 || !std::isfinite(a.total) || a.total != b.total || a.l1 != b.l1 ||
             a.kernels != b.kernels || a.wall_ms != 0.0;
    }
    bad += r1.cloud.size() != r1.history.back().kernels || r1.cloud.pos != r2.cloud.pos ||
           r1.cloud.rho_raw != r2.cloud.rho_raw;
    fails += report("train(): history, determinism (exact)", bad, 0);
  }
  orc_rng_free(rng);
  std::printf("%s (%d failures)\n", fails ? "FAIL" : "ALL PASS", fails);
  return fails;
}
