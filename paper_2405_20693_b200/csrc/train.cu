// One training iteration of the reference trainer in native code
// (trainer.cpp:268-319): the host-side sequence of engine launches that
// train.py's Trainer.step issues call by call, as a single C-ABI entry point.
//
//   render the view (rasterizer.cpp:112-157) into a context-owned image
//   L1 + lambda_ssim D-SSIM and dL/dI (objectives.cpp:113-167, trainer.cpp:277-287)
//   zero the gradients, render_backward with adaptive statistics (trainer.cpp:283-288)
//   TV on the D^3 sub-grid: voxelize -> tv3d -> voxelize_backward sharing one
//     binning (trainer.cpp:290-300, voxelizer.cpp:226-239 placement by the caller)
//   total = l1 + lambda_ssim dssim + lambda_tv tv (trainer.cpp:302-303), on the device
//   Adam over the four groups + quaternion renormalisation (trainer.cpp:310-319)
//
// Nothing is read back: with capacity-mode binning (sct_ctx_set_capacity) the
// iteration is free of host synchronisation, so consecutive calls queue ahead
// of the GPU. Scratch images and volumes are grow-only context buffers.
#include <cuda_runtime.h>

#include <cmath>

#include "sct_internal.cuh"

namespace sct {
namespace {

// (l1 + lambda_ssim dssim) + lambda_tv tv with separately rounded products, as the
// host-side composition does (no FMA contraction)
__global__ void train_total_kernel(double* v, double lambda_ssim, double lambda_tv) {
  pdl_prologue();
  v[3] = __dadd_rn(__dadd_rn(v[0], __dmul_rn(lambda_ssim, v[1])), __dmul_rn(lambda_tv, v[2]));
}

int zero_grads(Ctx* c, const sct_grads* g, int64_t m) {
  const size_t f = sizeof(float);
  if (g->pos == g->rho_raw + m && g->scale_raw == g->pos + 3 * m && g->rot == g->scale_raw + 3 * m) {
    return launch_zero(c, g->rho_raw, 11 * m * f);  // one contiguous 11*M buffer (PDL chain kept)
  }
  SCT_CUDA_TRY(cudaMemsetAsync(g->rho_raw, 0, m * f, c->stream));
  SCT_CUDA_TRY(cudaMemsetAsync(g->pos, 0, 3 * m * f, c->stream));
  SCT_CUDA_TRY(cudaMemsetAsync(g->scale_raw, 0, 3 * m * f, c->stream));
  SCT_CUDA_TRY(cudaMemsetAsync(g->rot, 0, 4 * m * f, c->stream));
  return SCT_OK;
}

}  // namespace
}  // namespace sct

using namespace sct;

extern "C" int sct_train_step(sct_ctx* c, sct_cloud* cloud, sct_adam_state* adam, sct_stats* stats,
                              sct_grads* grads, const sct_scanner* scanner, const sct_raster_opts* opts,
                              const sct_train_args* a) {
  if (!c || !cloud || !adam || !grads || !scanner || !opts || !a || !a->measured || !a->values_dev) {
    set_error("ConfigError: train_step: null argument");
    return SCT_ERR_CONFIG;
  }
  if (a->t < 1) {
    set_error("ConfigError: train_step: iteration t must be >= 1");
    return SCT_ERR_CONFIG;
  }
  const int w = scanner->det_res_px[0], h = scanner->det_res_px[1];
  float *img = nullptr, *dl = nullptr;
  SCT_TRY(stage_buf(c, 28, (size_t)w * h * sizeof(float), (void**)&img));
  SCT_TRY(stage_buf(c, 29, (size_t)w * h * sizeof(float), (void**)&dl));
  sct_fwd* fwd = nullptr;
  SCT_TRY(sct_render_fwd(c, cloud, scanner, &a->theta_rad, 1, opts, img, &fwd));
  int rc = sct_photometric_loss(c, img, a->measured, 1, w, h, a->render_scale, (float)a->lambda_ssim,
                                a->grad_scale, a->values_dev, dl);
  if (rc == SCT_OK) rc = zero_grads(c, grads, cloud->m);
  // the backward up to the chain's view-range partials; their finalize runs
  // inside the Adam kernel below, after the TV term added its gradients
  double* vsum = nullptr;
  int groups = 0;
  if (rc == SCT_OK) rc = sct_render_bwd_chunked(c, fwd, cloud, dl, grads, stats, 0, &vsum, &groups);
  sct_fwd_free(fwd);
  SCT_TRY(rc);
  if (a->lambda_tv > 0.0) {
    const sct_grid& g = a->tv_grid;
    const size_t nvox = (size_t)g.dims[0] * g.dims[1] * g.dims[2];
    float *vol = nullptr, *gtv = nullptr;
    SCT_TRY(stage_buf(c, 30, nvox * sizeof(float), (void**)&vol));
    SCT_TRY(stage_buf(c, 31, nvox * sizeof(float), (void**)&gtv));
    sct_vox_state* vs = nullptr;
    SCT_TRY(sct_voxelize_fwd_state(c, cloud, &g, a->cull_mahalanobis, 0, INT32_MAX, vol, &vs));
    rc = sct_tv3d(c, vol, g.dims, (float)a->lambda_tv, a->values_dev + 2, gtv);
    if (rc == SCT_OK) rc = sct_voxelize_bwd_state(c, vs, cloud, gtv, grads);
    sct_vox_free(vs);
    SCT_TRY(rc);
  } else {
    SCT_CUDA_TRY(cudaMemsetAsync(a->values_dev + 2, 0, sizeof(double), c->stream));
  }
  if (cloud->m == 0) {
    pdl_launch(train_total_kernel, dim3(1), dim3(1), 0, c->stream, a->values_dev, a->lambda_ssim, a->lambda_tv);
    ++c->launches;
    SCT_CUDA_TRY(cudaGetLastError());
    return SCT_OK;
  }
  // raster finalize + Adam (sct_adam_step's bias corrections, trainer.cpp:152-153)
  // + the total loss, in one kernel
  const double bc1 = 1.0 - std::pow(a->beta1, a->t), bc2 = 1.0 - std::pow(a->beta2, a->t);
  const float lrf[4] = {(float)a->lr[0], (float)a->lr[1], (float)a->lr[2], (float)a->lr[3]};
  launch_raster_finalize_adam(c, cloud->m, nullptr, cloud, vsum, groups, grads, stats, adam, lrf, (float)bc1,
                              (float)bc2, (float)a->beta1, (float)a->beta2, (float)a->eps, a->values_dev,
                              a->lambda_ssim, a->lambda_tv);
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}
