// The reference's train() loop (trainer.cpp:232-345) as a native object over
// the engine: the view shuffle, sub-grid origin and split draws from one
// std::mt19937_64 (sct_rng, trainer.cpp:254-258), one sct_train_step per
// iteration, adaptive density control (trainer.cpp:167-230, sct_adaptive_*)
// at the reference's iterations, and the loss values read back only where the
// caller asks for them (history points) or the non-finite check runs. With
// sync_free the binning runs in capacity mode, calibrated on the first
// iteration and after each adaptive-control pass, as train.py's Trainer.
//
// The cloud, its Adam moments, the adaptive statistics and the gradients live
// on the device for the whole run: cloud and grads as one 11*M float buffer
// each ({rho, pos, scale, rot}), the Adam moments as one 22*M buffer.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "sct_internal.cuh"

using namespace sct;

struct sct_trainer {
  sct_ctx* c = nullptr;
  sct_train_cfg cfg{};
  sct_scanner scanner{};
  sct_raster_opts opts{};
  int32_t n_views = 0, W = 0, H = 0;
  std::vector<double> angles;
  float* meas = nullptr;  // [V][H][W], normalised by the dataset maximum
  double inv_norm = 1.0;
  double extent[3] = {0, 0, 0}, spacing[3] = {0, 0, 0};
  // device state
  int64_t m = 0;
  double s_min = 0.0;
  float* params = nullptr;  // 11 m
  float* moments = nullptr; // 22 m
  float* grads = nullptr;   // 11 m
  float* stats = nullptr;   // m (norm) + m (count, int32) + 3 m (3d)
  double* values = nullptr; // [4]
  sct_rng* rng = nullptr;
  std::vector<int32_t> order;
  int32_t epoch_pos = 0;
  int32_t t = 0;
  bool calibrate = false;
  int32_t last_counts[3] = {0, 0, 0};
  int32_t last_view = -1;
};

namespace {

sct_cloud cloud_of(const sct_trainer* r, float* p, int64_t m) {
  sct_cloud cl{};
  cl.m = m;
  cl.s_min_mm = r->s_min;
  cl.rho_raw = p;
  cl.pos = p + m;
  cl.scale_raw = p + 4 * m;
  cl.rot = p + 7 * m;
  return cl;
}
sct_grads grads_of(float* g, int64_t m) {
  sct_grads gr{};
  gr.rho_raw = g;
  gr.pos = g + m;
  gr.scale_raw = g + 4 * m;
  gr.rot = g + 7 * m;
  return gr;
}
sct_adam_state adam_of(float* a, int64_t m) {  // m_rho v_rho m_pos v_pos m_scale v_scale m_rot v_rot
  sct_adam_state s{};
  s.m_rho = a;
  s.v_rho = a + m;
  s.m_pos = a + 2 * m;
  s.v_pos = a + 5 * m;
  s.m_scale = a + 8 * m;
  s.v_scale = a + 11 * m;
  s.m_rot = a + 14 * m;
  s.v_rot = a + 18 * m;
  return s;
}
sct_stats stats_of(float* s, int64_t m) {
  sct_stats st{};
  st.grad2d_norm_accum = s;
  st.grad_count = reinterpret_cast<int32_t*>(s + m);
  st.grad3d_accum = s + 2 * m;
  return st;
}

int alloc_state(sct_trainer* r, int64_t m, float** params, float** moments, float** grads, float** stats) {
  const size_t f = sizeof(float), n = (size_t)std::max<int64_t>(m, 1);
  if (cudaMalloc((void**)params, 11 * n * f) != cudaSuccess || cudaMalloc((void**)moments, 22 * n * f) != cudaSuccess ||
      cudaMalloc((void**)grads, 11 * n * f) != cudaSuccess || cudaMalloc((void**)stats, 5 * n * f) != cudaSuccess) {
    set_error("CUDA error: trainer allocation failed");
    return SCT_ERR_CUDA;
  }
  SCT_CUDA_TRY(cudaMemsetAsync(*moments, 0, 22 * n * f, r->c->stream));
  SCT_CUDA_TRY(cudaMemsetAsync(*grads, 0, 11 * n * f, r->c->stream));
  SCT_CUDA_TRY(cudaMemsetAsync(*stats, 0, 5 * n * f, r->c->stream));
  return SCT_OK;
}

void free_state(float* a, float* b, float* g, float* s) {
  cudaFree(a);
  cudaFree(b);
  cudaFree(g);
  cudaFree(s);
}

// trainer.cpp:269-273: shuffled epochs, the order reshuffled in place
int next_view(sct_trainer* r) {
  if (r->epoch_pos >= r->n_views) {
    sct_rng_shuffle(r->rng, r->order.data(), r->n_views);
    r->epoch_pos = 0;
  }
  return r->order[r->epoch_pos++];
}

// capacity-mode calibration (train.py Trainer.step): the view's exact pair count
// and the full-extent voxel grid's pair count bound the buffers of later steps.
// The calibration iteration itself runs in exact mode (as Trainer's), and the
// capacities apply from the next one: *raster / *voxel receive them.
int calibrate(sct_trainer* r, const sct_cloud& cl, double theta, int64_t* raster, int64_t* voxel) {
  sct_fwd* f = nullptr;
  SCT_TRY(sct_ctx_set_capacity(r->c, 0, 0));
  SCT_TRY(sct_render_fwd(r->c, &cl, &r->scanner, &theta, 1, &r->opts, nullptr, &f));
  int64_t gpe = 0, pairs = 0;
  int rc = sct_fwd_work(f, &gpe, &pairs);
  sct_fwd_free(f);
  SCT_TRY(rc);
  int64_t vpairs = 0;
  if (r->cfg.lambda_tv > 0.0) {
    sct_grid full{};
    for (int k = 0; k < 3; ++k) {
      full.dims[k] = (int32_t)std::llround(r->extent[k] / r->spacing[k]);
      full.origin_mm[k] = r->scanner.extent_min_mm[k];
      full.spacing_mm[k] = r->spacing[k];
    }
    int64_t vge = 0;
    SCT_TRY(sct_voxel_work(r->c, &cl, &full, 3.3681993876652464, &vge, &vpairs));
    vpairs = std::max<int64_t>(1, vpairs);
  }
  const double mg = r->cfg.capacity_margin;
  *raster = (int64_t)(mg * (double)pairs) + 65536;
  *voxel = r->cfg.lambda_tv > 0.0 ? (int64_t)std::min(8.0 * (double)vpairs, mg * (double)vpairs) + 65536 : 0;
  return SCT_OK;
}

// trainer.cpp:167-230 on the device; the new state replaces the old one
int adaptive(sct_trainer* r) {
  const int64_t m = r->m;
  sct_cloud cl = cloud_of(r, r->params, m);
  sct_stats st = stats_of(r->stats, m);
  sct_ac_plan* plan = nullptr;
  int64_t new_m = 0, n_split = 0;
  int32_t counts[3] = {0, 0, 0};
  SCT_TRY(sct_adaptive_plan(r->c, &cl, &st, r->cfg.prune_density_threshold, r->cfg.densify_grad_threshold,
                            r->cfg.split_scale_threshold_frac, r->cfg.split_factor, r->extent, &plan, &new_m, &n_split,
                            counts));
  float *p2 = nullptr, *a2 = nullptr, *g2 = nullptr, *s2 = nullptr;
  double* gauss = nullptr;
  int rc = alloc_state(r, new_m, &p2, &a2, &g2, &s2);
  if (rc == SCT_OK && n_split > 0) {  // the reference's normal draws, in its order (trainer.cpp:213-216)
    std::vector<double> h(6 * n_split);
    rc = sct_rng_normal(r->rng, 6 * n_split, h.data());
    if (rc == SCT_OK && cudaMalloc((void**)&gauss, h.size() * sizeof(double)) != cudaSuccess) rc = SCT_ERR_CUDA;
    if (rc == SCT_OK &&
        cudaMemcpyAsync(gauss, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, r->c->stream) !=
            cudaSuccess)
      rc = SCT_ERR_CUDA;
    if (rc == SCT_OK) rc = cudaStreamSynchronize(r->c->stream) == cudaSuccess ? SCT_OK : SCT_ERR_CUDA;
  }
  if (rc == SCT_OK) {
    sct_adam_state ad = adam_of(r->moments, m);
    sct_cloud out = cloud_of(r, p2, new_m);
    sct_adam_state out_ad = adam_of(a2, new_m);
    rc = sct_adaptive_apply(r->c, plan, &cl, &ad, st.grad3d_accum, gauss, &out, &out_ad);
  }
  sct_adaptive_free(plan);
  if (gauss) {
    cudaStreamSynchronize(r->c->stream);
    cudaFree(gauss);
  }
  if (rc != SCT_OK) {
    free_state(p2, a2, g2, s2);
    return rc;
  }
  SCT_CUDA_TRY(cudaStreamSynchronize(r->c->stream));
  free_state(r->params, r->moments, r->grads, r->stats);
  r->params = p2;
  r->moments = a2;
  r->grads = g2;
  r->stats = s2;  // zeroed: reset_grad_stats (gaussian_cloud.cpp:119-123)
  r->m = new_m;
  std::memcpy(r->last_counts, counts, sizeof(counts));
  r->calibrate = r->cfg.sync_free != 0;  // new kernel count: re-measure the pair counts
  return SCT_OK;
}

}  // namespace

extern "C" {

int sct_trainer_create(sct_ctx* c, const sct_cloud* cloud_host, const float* projections_host, const double* angles,
                       int32_t n_views, const sct_scanner* scanner, const sct_train_cfg* cfg, sct_trainer** out) {
  if (!c || !cloud_host || !projections_host || !angles || !scanner || !cfg || !out) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  *out = nullptr;
  if (n_views < 1) {
    set_error("InsufficientViews: train: need >= 1 projection");
    return SCT_ERR_CONFIG;
  }
  if (cloud_host->m < 1) {
    set_error("ConfigError: train: empty initial cloud");
    return SCT_ERR_CONFIG;
  }
  if (cfg->iters < 1 || cfg->tv_grid_dim < 2 || cfg->densify_interval < 1 || !(cfg->split_factor > 1.0) ||
      cfg->output_dims[0] < 1 || cfg->output_dims[1] < 1 || cfg->output_dims[2] < 1) {
    set_error("ConfigError: train: invalid configuration");
    return SCT_ERR_CONFIG;
  }
  auto* r = new sct_trainer();
  r->c = c;
  r->cfg = *cfg;
  r->scanner = *scanner;
  r->opts.mode = cfg->mode;
  r->opts.lowpass_eps_px = 0.3;
  r->opts.dilation_compensation = 1;
  r->opts.freeze_jacobian = 0;
  r->opts.cull_mahalanobis = 3.0348542587702925;
  r->n_views = n_views;
  r->W = scanner->det_res_px[0];
  r->H = scanner->det_res_px[1];
  r->angles.assign(angles, angles + n_views);
  r->m = cloud_host->m;
  r->s_min = cloud_host->s_min_mm;
  for (int k = 0; k < 3; ++k) {
    r->extent[k] = scanner->extent_max_mm[k] - scanner->extent_min_mm[k];
    r->spacing[k] = r->extent[k] / cfg->output_dims[k];
  }
  // trainer.cpp:243-252: projections normalised by the dataset maximum
  const size_t px = (size_t)r->W * r->H, tot = px * n_views;
  float mx = 0.f;
  bool any = false;
  for (size_t i = 0; i < tot; ++i)
    if (!any || projections_host[i] > mx) {
      mx = projections_host[i];
      any = true;
    }
  double norm = mx;
  if (!(norm > 0.0)) norm = 1.0;
  r->inv_norm = 1.0 / norm;
  std::vector<float> h(tot);
  const float s = (float)r->inv_norm;
  for (size_t i = 0; i < tot; ++i) h[i] = projections_host[i] * s;
  int rc = SCT_OK;
  auto fail = [&](int code) {
    sct_trainer_destroy(r);
    return code;
  };
  if (cudaMalloc((void**)&r->meas, tot * sizeof(float)) != cudaSuccess ||
      cudaMalloc((void**)&r->values, 4 * sizeof(double)) != cudaSuccess) {
    set_error("CUDA error: trainer allocation failed");
    return fail(SCT_ERR_CUDA);
  }
  if (cudaMemcpy(r->meas, h.data(), tot * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) return fail(SCT_ERR_CUDA);
  if ((rc = alloc_state(r, r->m, &r->params, &r->moments, &r->grads, &r->stats))) return fail(rc);
  const int64_t m = r->m;
  const float* src[4] = {cloud_host->rho_raw, cloud_host->pos, cloud_host->scale_raw, cloud_host->rot};
  const int64_t off[4] = {0, m, 4 * m, 7 * m}, cnt[4] = {m, 3 * m, 3 * m, 4 * m};
  for (int a = 0; a < 4; ++a)
    if (cudaMemcpy(r->params + off[a], src[a], cnt[a] * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(SCT_ERR_CUDA);
  if ((rc = sct_rng_create(cfg->seed, &r->rng))) return fail(rc);
  r->order.resize(n_views);
  std::iota(r->order.begin(), r->order.end(), 0);
  r->epoch_pos = n_views;  // forces a shuffle on first use
  r->calibrate = cfg->sync_free != 0;
  *out = r;
  return SCT_OK;
}

int sct_trainer_step(sct_trainer* r, int32_t* adapted) {
  if (!r) {
    set_error("ConfigError: null trainer");
    return SCT_ERR_CONFIG;
  }
  const sct_train_cfg& cfg = r->cfg;
  const int32_t t = ++r->t;
  const int view = next_view(r);
  r->last_view = view;
  sct_cloud cl = cloud_of(r, r->params, r->m);
  const bool calib = r->calibrate;
  int64_t cap_raster = 0, cap_voxel = 0;
  if (calib) SCT_TRY(calibrate(r, cl, r->angles[view], &cap_raster, &cap_voxel));
  sct_train_args a{};
  a.theta_rad = r->angles[view];
  a.measured = r->meas + (size_t)view * r->W * r->H;
  a.render_scale = a.grad_scale = (float)r->inv_norm;
  a.lambda_ssim = cfg.lambda_ssim;
  a.lambda_tv = cfg.lambda_tv;
  if (cfg.lambda_tv > 0.0) {  // voxelizer.cpp:226-239 on the trainer's stream
    double origin[3];
    SCT_TRY(sct_rng_subvolume_origin(r->rng, r->scanner.extent_min_mm, r->scanner.extent_max_mm, r->spacing,
                                     cfg.tv_grid_dim, origin));
    for (int k = 0; k < 3; ++k) {
      a.tv_grid.dims[k] = cfg.tv_grid_dim;
      a.tv_grid.origin_mm[k] = origin[k];
      a.tv_grid.spacing_mm[k] = r->spacing[k];
    }
  }
  a.cull_mahalanobis = 3.3681993876652464;
  a.t = t;
  a.lr[0] = sct_lr_at(cfg.lr_position, cfg.lr_final_ratio, t, cfg.iters);
  a.lr[1] = sct_lr_at(cfg.lr_density, cfg.lr_final_ratio, t, cfg.iters);
  a.lr[2] = sct_lr_at(cfg.lr_scale, cfg.lr_final_ratio, t, cfg.iters);
  a.lr[3] = sct_lr_at(cfg.lr_rotation, cfg.lr_final_ratio, t, cfg.iters);
  a.beta1 = 0.9;
  a.beta2 = 0.999;
  a.eps = 1e-15;
  a.values_dev = r->values;
  sct_adam_state ad = adam_of(r->moments, r->m);
  sct_stats st = stats_of(r->stats, r->m);
  sct_grads gr = grads_of(r->grads, r->m);
  SCT_TRY(sct_train_step(r->c, &cl, &ad, &st, &gr, &r->scanner, &r->opts, &a));
  if (calib) {
    SCT_TRY(sct_ctx_set_capacity(r->c, cap_raster, cap_voxel));
    r->calibrate = false;
  }
  if (cfg.check_every > 0 && t % cfg.check_every == 0) {  // trainer.cpp:302-308
    double v[4];
    SCT_CUDA_TRY(cudaMemcpyAsync(v, r->values, sizeof(v), cudaMemcpyDeviceToHost, r->c->stream));
    SCT_CUDA_TRY(cudaStreamSynchronize(r->c->stream));
    if (!std::isfinite(v[3])) {
      set_error("DivergenceDetected: non-finite loss at iteration " + std::to_string(t));
      return SCT_ERR_DIVERGENCE;
    }
    if (cfg.sync_free && !calib) {
      int32_t of = 0;
      SCT_TRY(sct_ctx_take_overflow(r->c, &of));
      if (of) {
        set_error("DataError: sync-free binning exceeded its pair capacity by iteration " + std::to_string(t));
        return SCT_ERR_DATA;
      }
    }
  }
  int32_t did = 0;
  if (t >= cfg.adaptive_start && t <= cfg.adaptive_end && t > cfg.adaptive_start &&
      (t - cfg.adaptive_start) % cfg.densify_interval == 0) {  // trainer.cpp:321-323
    SCT_TRY(adaptive(r));
    did = 1;
  }
  if (adapted) *adapted = did;
  return SCT_OK;
}

int sct_trainer_record(sct_trainer* r, sct_train_record* rec) {
  if (!r || !rec) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  double v[4] = {0, 0, 0, 0};
  if (r->t > 0) {
    SCT_CUDA_TRY(cudaMemcpyAsync(v, r->values, sizeof(v), cudaMemcpyDeviceToHost, r->c->stream));
    SCT_CUDA_TRY(cudaStreamSynchronize(r->c->stream));
  }
  rec->iter = r->t;
  rec->view = r->last_view;
  rec->l1 = v[0];
  rec->dssim = v[1];
  rec->tv = v[2];
  rec->total = v[3];
  rec->kernels = r->m;
  for (int k = 0; k < 3; ++k) rec->counts[k] = r->last_counts[k];
  return SCT_OK;
}

int sct_trainer_download(sct_trainer* r, sct_cloud* cloud_host, sct_adam_state* adam_host, sct_stats* stats_host) {
  if (!r || !cloud_host) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  if (cloud_host->m != r->m) {
    set_error("DimMismatch: trainer download: host cloud holds " + std::to_string(cloud_host->m) + " kernels, the " +
              "trainer " + std::to_string(r->m));
    return SCT_ERR_DATA;
  }
  const int64_t m = r->m;
  cudaStream_t s = r->c->stream;
  const sct_cloud d = cloud_of(r, r->params, m);
  SCT_CUDA_TRY(cudaMemcpyAsync(cloud_host->rho_raw, d.rho_raw, m * sizeof(float), cudaMemcpyDeviceToHost, s));
  SCT_CUDA_TRY(cudaMemcpyAsync(cloud_host->pos, d.pos, 3 * m * sizeof(float), cudaMemcpyDeviceToHost, s));
  SCT_CUDA_TRY(cudaMemcpyAsync(cloud_host->scale_raw, d.scale_raw, 3 * m * sizeof(float), cudaMemcpyDeviceToHost, s));
  SCT_CUDA_TRY(cudaMemcpyAsync(cloud_host->rot, d.rot, 4 * m * sizeof(float), cudaMemcpyDeviceToHost, s));
  cloud_host->s_min_mm = r->s_min;
  if (adam_host) {
    const sct_adam_state a = adam_of(r->moments, m);
    float* hs[8] = {adam_host->m_rho, adam_host->v_rho, adam_host->m_pos, adam_host->v_pos,
                    adam_host->m_scale, adam_host->v_scale, adam_host->m_rot, adam_host->v_rot};
    const float* ds[8] = {a.m_rho, a.v_rho, a.m_pos, a.v_pos, a.m_scale, a.v_scale, a.m_rot, a.v_rot};
    const int64_t n[8] = {m, m, 3 * m, 3 * m, 3 * m, 3 * m, 4 * m, 4 * m};
    for (int k = 0; k < 8; ++k)
      if (hs[k]) SCT_CUDA_TRY(cudaMemcpyAsync(hs[k], ds[k], n[k] * sizeof(float), cudaMemcpyDeviceToHost, s));
  }
  if (stats_host) {
    const sct_stats t = stats_of(r->stats, m);
    if (stats_host->grad2d_norm_accum)
      SCT_CUDA_TRY(cudaMemcpyAsync(stats_host->grad2d_norm_accum, t.grad2d_norm_accum, m * sizeof(float),
                                   cudaMemcpyDeviceToHost, s));
    if (stats_host->grad_count)
      SCT_CUDA_TRY(cudaMemcpyAsync(stats_host->grad_count, t.grad_count, m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (stats_host->grad3d_accum)
      SCT_CUDA_TRY(cudaMemcpyAsync(stats_host->grad3d_accum, t.grad3d_accum, 3 * m * sizeof(float),
                                   cudaMemcpyDeviceToHost, s));
  }
  SCT_CUDA_TRY(cudaStreamSynchronize(s));
  return SCT_OK;
}

int sct_trainer_destroy(sct_trainer* r) {
  if (!r) return SCT_OK;
  if (r->c) cudaStreamSynchronize(r->c->stream);
  free_state(r->params, r->moments, r->grads, r->stats);
  cudaFree(r->meas);
  cudaFree(r->values);
  if (r->rng) sct_rng_destroy(r->rng);
  if (r->c) sct_ctx_set_capacity(r->c, 0, 0);
  delete r;
  return SCT_OK;
}

}  // extern "C"
