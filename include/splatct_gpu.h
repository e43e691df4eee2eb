/*
 * splatct_gpu.h — C ABI of the B200-native R²-Gaussian hot-path engine.
 *
 * Drop-in boundary for the reference's C++ host API (splatct, CPU/fp64):
 *   render            rasterizer.hpp:53-54   (rasterizer.cpp:112-157)
 *   render_backward   rasterizer.hpp:61-64   (rasterizer.cpp:195-342)
 *   project_kernel    rasterizer.hpp:36-38   (rasterizer.cpp:103-110)
 *   voxelize          voxelizer.hpp:60-61    (voxelizer.cpp:108-138)
 *   voxelize_backward voxelizer.hpp:65-67    (voxelizer.cpp:140-224)
 *   tv3d_loss         objectives.hpp:31      (objectives.cpp:169-202)
 *   l1_loss/dssim_loss objectives.hpp        (objectives.cpp:113-167)
 *   Adam::step + normalize_rotations         (trainer.cpp:144-163,310-319;
 *                                             gaussian_cloud.cpp:112-117)
 *   lr_at             trainer.hpp            (trainer.cpp:34-36)
 * Types:
 *   sct_scanner  = ScannerConfig minus angles (geometry.hpp:12-31); thetas are per call
 *   sct_raster_opts = RasterOptions (rasterizer.hpp:15-21)
 *   sct_grid     = GridSpec (voxelizer.hpp:13-24)
 *   sct_cloud    = GaussianCloud raw arrays (gaussian_cloud.hpp:62-66), fp32,
 *                  same field order/layout: rho_raw[M], pos[3M] (xyz per kernel),
 *                  scale_raw[3M], rot[4M] (w,x,y,z)
 *   sct_grads    = CloudGrads (gaussian_cloud.hpp:84-96): ACCUMULATE (+=) semantics
 *   sct_stats    = adaptive-control statistics (gaussian_cloud.hpp:74-77)
 *
 * Conventions
 *   - Every function returns an int status: 0 ok, 2 config error (ConfigError),
 *     3 data/dims error (DataError / DimMismatch), 4 divergence (non-finite
 *     loss), 5 CUDA error, 1 other. sct_last_error() returns a thread-local
 *     message for the last failure (common.hpp:27-64 exception taxonomy,
 *     splatct_main.cpp:327-339 exit codes).
 *   - Pointers in sct_cloud / sct_grads / sct_stats and image/volume buffers are
 *     DEVICE pointers unless the function name ends in _host.
 *   - Images are [n_views][H][W] row-major (pixel (u,v) at v*W+u, common.hpp:66-79);
 *     volumes are x-fastest [(z*Y+y)*X+x] (voxelizer.hpp:29-31).
 *   - One context serialises its calls on its stream (the reference's
 *     exclusive-mutation contract); distinct contexts may run
 *     concurrently. All work is enqueued on the context's stream.
 *   - The cloud must not change between sct_render_fwd and sct_render_bwd
 *     (the backward re-derives the projection chain from it, rasterizer.cpp:266-268).
 */
#ifndef SPLATCT_GPU_H
#define SPLATCT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCT_OK 0
#define SCT_ERR_OTHER 1
#define SCT_ERR_CONFIG 2
#define SCT_ERR_DATA 3
#define SCT_ERR_DIVERGENCE 4
#define SCT_ERR_CUDA 5

#define SCT_MODE_RECTIFIED 0
#define SCT_MODE_BIASED 1

typedef struct sct_ctx sct_ctx;
typedef struct sct_fwd sct_fwd;

typedef struct {
  double l_so_mm;          /* source to rotation axis */
  double l_sd_mm;          /* source to detector plane */
  double det_size_mm[2];   /* detector_size_mm */
  int32_t det_res_px[2];   /* detector_res_px (W, H) */
  double extent_min_mm[3];
  double extent_max_mm[3];
  double near_clip_mm;     /* <= 0 selects 1% of l_so_mm (geometry.hpp:24-28) */
  int32_t parallel_beam;   /* 0: cone beam (the reference); 1: parallel beam, an extension
                              (orthographic: detector mm = scanner mm, J = diag(fx, fy, 1),
                              no near-clip cull); zero-initialise for the reference behaviour */
} sct_scanner;

typedef struct {
  int32_t mode;                  /* SCT_MODE_RECTIFIED | SCT_MODE_BIASED */
  double lowpass_eps_px;         /* 0.3 */
  int32_t dilation_compensation; /* 1 */
  int32_t freeze_jacobian;       /* 0 */
  double cull_mahalanobis;       /* 3.0348542587702925 */
} sct_raster_opts;

typedef struct {
  int32_t dims[3];
  double origin_mm[3];
  double spacing_mm[3];
} sct_grid;

typedef struct {
  int64_t m;
  double s_min_mm;
  float* rho_raw;   /* [m] */
  float* pos;       /* [3m] */
  float* scale_raw; /* [3m] */
  float* rot;       /* [4m] (w,x,y,z) */
} sct_cloud;

typedef struct {
  float* rho_raw;
  float* pos;
  float* scale_raw;
  float* rot;
} sct_grads;

typedef struct {
  float* grad2d_norm_accum; /* [m] */
  int32_t* grad_count;      /* [m] */
  float* grad3d_accum;      /* [3m] */
} sct_stats;

typedef struct {
  float *m_rho, *v_rho;     /* [m]  */
  float *m_pos, *v_pos;     /* [3m] */
  float *m_scale, *v_scale; /* [3m] */
  float *m_rot, *v_rot;     /* [4m] */
} sct_adam_state;

/* ---- context ------------------------------------------------------------ */
/* stream: a cudaStream_t (NULL = legacy default stream). */
int sct_ctx_create(int device, void* stream, sct_ctx** out);
int sct_ctx_destroy(sct_ctx* ctx);
int sct_ctx_set_stream(sct_ctx* ctx, void* stream);
int sct_ctx_sync(sct_ctx* ctx);
/* deterministic != 0: fixed-order reductions everywhere (default 1). */
/* Sync-free binning (capacity mode). With a capacity > 0 the render forward
 * (when its tile table fits the counting scatter) and the voxel binning do not
 * read the pair count back to the host: their pair buffers hold `capacity`
 * pairs and a device word records any call whose pairs exceeded it (those
 * pairs are dropped). sct_ctx_take_overflow synchronises, returns and clears
 * that word; a caller checks it before trusting results. 0 = exact mode
 * (default: one host readback per binning). Lets a training loop run without
 * host synchronisation. */
int sct_ctx_set_capacity(sct_ctx* ctx, int64_t raster_pairs, int64_t voxel_pairs);
int sct_ctx_take_overflow(sct_ctx* ctx, int32_t* overflowed);
int sct_ctx_set_deterministic(sct_ctx* ctx, int deterministic);
const char* sct_last_error(void);
const char* sct_version(void);
/* number of engine kernels launched by this context so far (instrumentation). */
int64_t sct_ctx_kernel_launches(const sct_ctx* ctx);

/* per-kernel CUDA-event timing of engine launches on the context stream.
 * report: JSON object {"kernel": [total_ms, launches], ...}; synchronises and resets. */
int sct_ctx_set_timing(sct_ctx* ctx, int enable);
int sct_ctx_timing_report(sct_ctx* ctx, char* buf, int32_t buflen);

/* ---- rasterizer --------------------------------------------------------- */
/* Projects + bins + composites n_views views (one batched launch sequence).
 * images: device [n_views][H][W] float. *state receives the forward state
 * (tile lists, projected records) that sct_render_bwd consumes. */
int sct_render_fwd(sct_ctx* ctx, const sct_cloud* cloud, const sct_scanner* scanner,
                   const double* thetas, int32_t n_views, const sct_raster_opts* opts,
                   float* images, sct_fwd** state);
/* Accumulates dL/d(raw params) of all views of `state` into grads (+=);
 * stats (nullable) receives the adaptive statistics as render_backward with
 * accumulate_stats=true. dL_dimages: device [n_views][H][W]. */
int sct_render_bwd(sct_ctx* ctx, sct_fwd* state, const sct_cloud* cloud, const float* dL_dimages,
                   sct_grads* grads, sct_stats* stats);
int sct_fwd_free(sct_fwd* state);
/* algorithmic work of a forward state: Gaussian-pixel evaluations (GPE) and pairs */
int sct_fwd_work(sct_fwd* state, int64_t* gpe, int64_t* n_pairs);
/* forward-state introspection (host outputs; synchronises the context) */
int sct_fwd_info(sct_fwd* state, int64_t* n_pairs, int32_t* tiles_x, int32_t* tiles_y,
                 int64_t* n_visible);
/* per-view tile lists in kernel indices: offsets[T+1], kernel_idx[pairs of this view]
 * (host arrays; kernel_idx may be NULL to query offsets only). */
int sct_fwd_tile_lists(sct_fwd* state, int32_t view, int64_t* offsets, int32_t* kernel_idx);
/* per-view projected kernels (project_kernel for every kernel): host outputs
 * visible[m] (0/1) and rec[m][11] = cx cy cov00 cov01 cov11 conic00 conic01
 * conic11 amplitude mu depth, computed in FP64. */
int sct_project_kernels(sct_ctx* ctx, const sct_cloud* cloud, const sct_scanner* scanner, double theta,
                        const sct_raster_opts* opts, int32_t* visible, double* rec);
/* the same with the cloud arrays in host memory */
int sct_project_kernels_host(sct_ctx* ctx, const sct_cloud* cloud_host, const sct_scanner* scanner, double theta,
                             const sct_raster_opts* opts, int32_t* visible, double* rec);

/* Host-buffer entry points (reference-facing: host arrays in, host arrays out;
 * the H2D/D2H copies run on the context stream). cloud arrays are host fp32.
 * images_host [n_views][H][W]. */
int sct_render_fwd_host(sct_ctx* ctx, const sct_cloud* cloud_host, const sct_scanner* scanner,
                        const double* thetas, int32_t n_views, const sct_raster_opts* opts,
                        float* images_host, sct_fwd** state);
int sct_render_bwd_host(sct_ctx* ctx, sct_fwd* state, const sct_cloud* cloud_host,
                        const float* dL_dimages_host, sct_grads* grads_host, sct_stats* stats_host);

/* ---- voxelizer ---------------------------------------------------------- */
/* Evaluates the brick-binned kernel sum on the grid. Only bricks with z index
 * in [z_brick_begin, z_brick_end) are evaluated/written (z-slab sharding;
 * pass 0, INT32_MAX for the whole grid). vol: device x-fastest [Z][Y][X];
 * the slab's voxels are overwritten, others untouched. */
int sct_voxelize_fwd(sct_ctx* ctx, const sct_cloud* cloud, const sct_grid* grid, double cull_mahalanobis,
                     int32_t z_brick_begin, int32_t z_brick_end, float* vol);
int sct_voxelize_bwd(sct_ctx* ctx, const sct_cloud* cloud, const sct_grid* grid, double cull_mahalanobis,
                     int32_t z_brick_begin, int32_t z_brick_end, const float* dL_dvol, sct_grads* grads);
/* brick lists for parity checks (host outputs, synchronises) */
int sct_voxel_bins(sct_ctx* ctx, const sct_cloud* cloud, const sct_grid* grid, double cull_mahalanobis,
                   int64_t* n_pairs, int64_t* offsets, int32_t* kernel_idx);
/* voxel-Gaussian evaluations (VGE) and (brick, kernel) pairs of a full-grid voxelize */
int sct_voxel_work(sct_ctx* ctx, const sct_cloud* cloud, const sct_grid* grid, double cull_mahalanobis,
                   int64_t* vge, int64_t* n_pairs);
int sct_voxelize_fwd_host(sct_ctx* ctx, const sct_cloud* cloud_host, const sct_grid* grid,
                          double cull_mahalanobis, float* vol_host);
/* grads_host accumulate (+=), like voxelize_backward (voxelizer.cpp:140-224) */
int sct_voxelize_bwd_host(sct_ctx* ctx, const sct_cloud* cloud_host, const sct_grid* grid,
                          double cull_mahalanobis, const float* dL_dvol_host, sct_grads* grads_host);

/* Forward + backward sharing one binning: sct_voxelize_fwd_state bins the
 * kernels (as sct_voxelize_fwd; vol may be NULL to bin only) and keeps the brick
 * lists in *state; sct_voxelize_bwd_state reuses them (the cloud must not change
 * in between, as for sct_render_bwd); sct_vox_free releases the state. Results
 * equal sct_voxelize_fwd / sct_voxelize_bwd, which re-bin like the reference. */
typedef struct sct_vox_state sct_vox_state;
int sct_voxelize_fwd_state(sct_ctx* ctx, const sct_cloud* cloud, const sct_grid* grid, double cull_mahalanobis,
                           int32_t z_brick_begin, int32_t z_brick_end, float* vol, sct_vox_state** state);
int sct_voxelize_bwd_state(sct_ctx* ctx, sct_vox_state* state, const sct_cloud* cloud, const float* dL_dvol,
                           sct_grads* grads);
int sct_vox_free(sct_vox_state* state);

/* ---- objectives / optimizer -------------------------------------------- */
/* TV value (device double [1], written) and lambda-scaled gradient (device, overwritten). */
int sct_tv3d(sct_ctx* ctx, const float* vol, const int32_t dims[3], float lambda, double* value_dev,
             float* grad);
/* L1 + lambda_ssim * D-SSIM of n images (device [n][H][W]) against measured;
 * writes per-image values (device double [n][2]: l1, dssim) and
 * dL/dI = (g_l1 + lambda_ssim*g_dssim) * grad_scale (device [n][H][W]). */
int sct_photometric_loss(sct_ctx* ctx, const float* rendered, const float* measured, int32_t n, int32_t w,
                         int32_t h, float render_scale, float lambda_ssim, float grad_scale,
                         double* values_dev, float* dL_dI);
/* Fused Adam over all four parameter groups + quaternion renormalisation.
 * lr[4] = {pos, rho, scale, rot} (trainer.cpp:310-318 order), step t >= 1. */
int sct_adam_step(sct_ctx* ctx, sct_cloud* params, sct_adam_state* state, const sct_grads* grads, int32_t t,
                  const double lr[4], double beta1, double beta2, double eps);
double sct_lr_at(double lr_init, double final_ratio, int32_t t, int32_t iters);

/* ---- one training iteration in native code (trainer.cpp:268-319) ---------- */
/* Render theta_rad, L1 + lambda_ssim D-SSIM against `measured` (device [H][W],
 * normalised by the dataset maximum; render_scale / grad_scale as
 * sct_photometric_loss), zero `grads` and accumulate render_backward (with the
 * adaptive statistics when stats != NULL), the TV term on tv_grid when
 * lambda_tv > 0 (voxelize / tv3d / voxelize_backward sharing one binning), then
 * Adam step t with lr = {pos, rho, scale, rot} and the quaternion
 * renormalisation. values_dev (device double [4]) receives l1, dssim, tv and
 * total = l1 + lambda_ssim dssim + lambda_tv tv. Reads nothing back: with
 * capacity-mode binning (sct_ctx_set_capacity) the call is sync-free. Replaces
 * the body of the reference's train() loop, trainer.cpp:268-319; the caller
 * draws the view and the sub-grid origin (sct_rng_*) and runs adaptive control. */
typedef struct {
  double theta_rad;
  const float* measured;
  float render_scale, grad_scale;
  double lambda_ssim, lambda_tv;
  sct_grid tv_grid;
  double cull_mahalanobis; /* voxelizer cull (voxelizer.hpp: sqrt(chi2 99% dof 3)) */
  int32_t t;
  double lr[4];
  double beta1, beta2, eps;
  double* values_dev;
} sct_train_args;
int sct_train_step(sct_ctx* ctx, sct_cloud* cloud, sct_adam_state* adam, sct_stats* stats, sct_grads* grads,
                   const sct_scanner* scanner, const sct_raster_opts* opts, const sct_train_args* args);

/* ---- the reference's train() loop as a native object (trainer.cpp:232-345) --- */
/* The whole run on the device: sct_trainer_create uploads the cloud and the
 * projections (normalised by their maximum, trainer.cpp:243-252); each
 * sct_trainer_step draws the view (std::shuffle epochs) and the TV sub-grid
 * origin from std::mt19937_64(seed), runs sct_train_step, the non-finite check
 * every check_every iterations (the reference: 1) and adaptive control at the
 * reference's iterations (split draws from the same stream). sync_free: binning
 * in capacity mode (capacity_margin x the pairs measured on a calibration step,
 * the first and after each adaptive control). sct_trainer_record syncs and
 * returns the last iteration's losses (the reference's HistoryRecord without
 * wall time); sct_trainer_download copies the cloud (and, when non-NULL, the
 * Adam moments and statistics) into host arrays of the trainer's current size. */
typedef struct {
  int32_t iters;
  double lr_position, lr_density, lr_scale, lr_rotation, lr_final_ratio;
  double lambda_ssim, lambda_tv;
  int32_t tv_grid_dim;
  int32_t adaptive_start, adaptive_end, densify_interval;
  double densify_grad_threshold, prune_density_threshold, split_scale_threshold_frac, split_factor;
  uint64_t seed;
  int32_t mode; /* SCT_MODE_RECTIFIED | SCT_MODE_BIASED */
  int32_t output_dims[3];
  int32_t check_every;
  int32_t sync_free;
  double capacity_margin;
} sct_train_cfg;
typedef struct {
  int32_t iter, view;
  double l1, dssim, tv, total;
  int64_t kernels;
  int32_t counts[3]; /* the last adaptive control's pruned, cloned, split */
} sct_train_record;
typedef struct sct_trainer sct_trainer;
int sct_trainer_create(sct_ctx* ctx, const sct_cloud* cloud_host, const float* projections_host,
                       const double* angles_rad, int32_t n_views, const sct_scanner* scanner,
                       const sct_train_cfg* cfg, sct_trainer** out);
int sct_trainer_step(sct_trainer* trainer, int32_t* adapted);
int sct_trainer_record(sct_trainer* trainer, sct_train_record* rec);
int sct_trainer_download(sct_trainer* trainer, sct_cloud* cloud_host, sct_adam_state* adam_host,
                         sct_stats* stats_host);
int sct_trainer_destroy(sct_trainer* trainer);

/* ---- adaptive density control (trainer.cpp:167-230) ---------------------- */
/* Two phases so the caller can size the new cloud: sct_adaptive_plan classifies
 * every kernel (prune rho < prune_density_threshold; clone or split kernels whose
 * mean accumulated screen-space gradient exceeds densify_grad_threshold, split
 * when max scale > split_scale_threshold_frac * max(extent_size_mm)) and reports
 * the new size, the number of split kernels and counts = {pruned, cloned, split}
 * (synchronises the context stream). sct_adaptive_apply writes the compacted
 * survivors (Adam state carried) followed by the new kernels in parent order
 * (zero Adam state) into out / out_adam (device buffers of new_m kernels).
 * gauss: device double [6 * n_split] standard-normal draws, per split kernel and
 * child in the order (z, y, x) — the reference's consumption order, e.g. from
 * sct_rng_normal — may be NULL when n_split == 0. The caller resets the
 * gradient statistics (gaussian_cloud.cpp:119-123 zeroes all three). */
typedef struct sct_ac_plan sct_ac_plan;
int sct_adaptive_plan(sct_ctx* ctx, const sct_cloud* cloud, const sct_stats* stats, double prune_density_threshold,
                      double densify_grad_threshold, double split_scale_threshold_frac, double split_factor,
                      const double extent_size_mm[3], sct_ac_plan** plan, int64_t* new_m, int64_t* n_split,
                      int32_t counts[3]);
int sct_adaptive_apply(sct_ctx* ctx, sct_ac_plan* plan, const sct_cloud* cloud, const sct_adam_state* adam,
                       const float* grad3d_accum, const double* gauss, sct_cloud* out, sct_adam_state* out_adam);
int sct_adaptive_free(sct_ac_plan* plan);

/* ---- the trainer's host random stream (trainer.cpp:254-258) -------------- */
/* One std::mt19937_64(seed) with libstdc++'s distributions, drawn in the
 * reference trainer's order: sct_rng_shuffle = std::shuffle of the view order
 * at each epoch start (trainer.cpp:269-273, reshuffled in place);
 * sct_rng_subvolume_origin = random_subvolume_spec's origin (voxelizer.cpp:226-239,
 * three uniform(0,1) draws); sct_rng_normal = n draws of ONE
 * std::normal_distribution(0,1) object (one adaptive_control call, trainer.cpp:184). */
typedef struct sct_rng sct_rng;
int sct_rng_create(uint64_t seed, sct_rng** out);
int sct_rng_destroy(sct_rng* rng);
int sct_rng_shuffle(sct_rng* rng, int32_t* values, int32_t n);
int sct_rng_subvolume_origin(sct_rng* rng, const double lo[3], const double hi[3], const double spacing[3], int32_t d,
                             double origin[3]);
int sct_rng_normal(sct_rng* rng, int64_t n, double* out);
int sct_rng_uniform(sct_rng* rng, int64_t n, double lo, double hi, double* out);

/* ---- fixture generation (simulator.cpp, fdk.cpp) ------- */
/* Analytic ellipsoid phantom (simulator.cpp:31-65): ellipsoids [n][8] host
 * {intensity, a, b, c, x0, y0, z0, phi_rad} in coordinates normalised to the
 * box [lo, hi]; vol device [Z][Y][X] on grid_for_extent(lo, hi, dims); dims >= 16. */
int sct_phantom(sct_ctx* ctx, int32_t n_ellipsoids, const double* ellipsoids, const double lo_mm[3],
                const double hi_mm[3], const int32_t dims[3], float* vol);
/* Quadrature projector project_volume (simulator.cpp:109-132), FP64 per ray:
 * images device [n_views][H][W] (clean log-domain line integrals). */
int sct_project_volume(sct_ctx* ctx, const float* vol, const sct_grid* grid, const sct_scanner* scanner,
                       const double* thetas, int32_t n_views, double step_mm, float* images);
/* add_noise (simulator.cpp:143-157) in place on HOST images [n_views][H][W]; view v uses
 * the reference stream view_rng(seed, view0 + v) (simulator.cpp:134-141), so results equal
 * simulate_projections bit-for-bit up to the fp32 storage. Views run in parallel threads. */
int sct_add_noise_host(float* images, int32_t n_views, int32_t w, int32_t h, double i0, double gauss_sigma,
                       uint64_t seed, int32_t view0);
/* fdk_reconstruct (fdk.cpp:53-134): images device [n_views][H][W]; window 0 ramp, 1 Hann,
 * 2 auto (Hann when n_views < 100); vol device [Z][Y][X]. n_views < 2 -> SCT_ERR_DATA. */
int sct_fdk(sct_ctx* ctx, const float* images, int32_t n_views, const sct_scanner* scanner, const double* thetas,
            const sct_grid* grid, int32_t window, float* vol);
/* exact nearest-neighbour distances (fdk.cpp:136-201): points/out device double [n][3] / [n]. */
int sct_nn_distances(sct_ctx* ctx, int64_t n, const double* points, double* out);
/* sample_init_cloud (fdk.cpp:203-247) with std::mt19937_64(seed): out = device cloud with
 * out->m == count (raw parameters as add_kernel stores them). Too few voxels above the
 * threshold -> SCT_ERR_DATA (TooFewOccupiedVoxels). Synchronises the context stream. */
int sct_sample_init_cloud(sct_ctx* ctx, const float* vol, const sct_grid* grid, int32_t count,
                          double density_threshold, double density_scale, double s_min_mm, uint64_t seed,
                          sct_cloud* out);

/* ---- multi-GPU exchange (NCCL) ------------------------ */
/* Views are sharded across ranks, each rank holding the whole cloud; the only
 * exchange is a sum over ranks of the per-kernel gradients (and adaptive
 * statistics). NCCL is resolved at run time (libnccl.so.2); these return
 * SCT_ERR_CUDA if it is absent and SCT_ERR_CONFIG without a communicator.
 * sct_nccl_unique_id: rank 0 makes the id, the caller broadcasts it.
 * sct_ctx_comm_init: context-owned communicator (destroyed with the context).
 * sct_ctx_set_comm: caller-owned ncclComm_t (NULL detaches).
 * sct_allreduce_grads: in-place sum of grads (and stats when non-NULL).
 * sct_render_bwd_allreduce / sct_voxelize_bwd_allreduce: as sct_render_bwd /
 * sct_voxelize_bwd, but every rank gets grads += sum over ranks of the ranks'
 * contributions (one contiguous 11*M-float collective on the context stream). */
int sct_nccl_unique_id(uint8_t id[128]);
int sct_ctx_comm_init(sct_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[128]);
int sct_ctx_set_comm(sct_ctx* ctx, void* nccl_comm);
int sct_ctx_comm_info(sct_ctx* ctx, int32_t* nranks, int32_t* rank);
int sct_allreduce_grads(sct_ctx* ctx, int64_t m, sct_grads* grads, sct_stats* stats);
int sct_render_bwd_allreduce(sct_ctx* ctx, sct_fwd* state, const sct_cloud* cloud, const float* dL_dimages,
                             sct_grads* grads, sct_stats* stats);
int sct_voxelize_bwd_allreduce(sct_ctx* ctx, const sct_cloud* cloud, const sct_grid* grid, double cull_mahalanobis,
                               int32_t z_brick_begin, int32_t z_brick_end, const float* dL_dvol, sct_grads* grads);

/* ---- host memory --------------------------------------------------------- */
/* page-locked host buffers for the _host entry points (full-bandwidth,
 * asynchronous copies); sct_debug_pointer_type reports how the engine's CUDA
 * runtime classifies a pointer (0 unregistered, 1 host, 2 device, 3 managed). */
int sct_host_alloc(void** p, size_t bytes);
int sct_host_free(void* p);
int sct_debug_pointer_type(const void* p);

#ifdef __cplusplus
}
#endif
#endif /* SPLATCT_GPU_H */
