// Regulariser, photometric losses and optimizer (HBM-bound kernels).
//
//   K9  tv3d           — objectives.cpp:169-202 (value: deterministic two-pass
//                        block reduction; gradient in gather form, no atomics)
//   K10 adam           — trainer.cpp:144-163 for all four groups in one pass,
//                        then gaussian_cloud.cpp:112-117 quaternion renorm
//   K11 photometric    — objectives.cpp:11-167 L1 + D-SSIM (valid 11x11
//                        separable window) and the dL/dI assembly of
//                        trainer.cpp:277-287
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "adam.cuh"
#include "sct_internal.cuh"

namespace sct {

namespace {

// ---------------------------------------------------------------- TV
__device__ __forceinline__ float sgnf(float d) { return d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f); }

__device__ void tv3d_finish_warp(const double* partials, int n_blocks, double inv_x, double inv_y, double inv_z,
                                 double* value);
__device__ __forceinline__ bool last_block(int* counter, int n_blocks);
__global__ void __launch_bounds__(256) tv3d_kernel(const float* __restrict__ vol, int nx, int ny, int nz,
                                                   float inv_x, float inv_y, float inv_z, float lambda,
                                                   float* __restrict__ grad, double* __restrict__ partials,
                                                   double dinv_x, double dinv_y, double dinv_z,
                                                   double* __restrict__ value, int* __restrict__ counter) {
  pdl_prologue();
  const long long n = (long long)nx * ny * nz;
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx);
    const int y = (int)((i / nx) % ny);
    const int z = (int)(i / ((long long)nx * ny));
    const float c = vol[i];
    float g = 0.f;
    // reference accumulation order per voxel: x-, x+, y-, y+, z-, z+
    if (x > 0) g += sgnf(c - vol[i - 1]) * inv_x;
    if (x < nx - 1) {
      const float d = vol[i + 1] - c;
      g -= sgnf(d) * inv_x;
      sx += fabs((double)d);
    }
    if (y > 0) g += sgnf(c - vol[i - nx]) * inv_y;
    if (y < ny - 1) {
      const float d = vol[i + nx] - c;
      g -= sgnf(d) * inv_y;
      sy += fabs((double)d);
    }
    if (z > 0) g += sgnf(c - vol[i - (long long)nx * ny]) * inv_z;
    if (z < nz - 1) {
      const float d = vol[i + (long long)nx * ny] - c;
      g -= sgnf(d) * inv_z;
      sz += fabs((double)d);
    }
    grad[i] = g * lambda;
  }
  // block reduction (fixed order) of the three axis sums
  __shared__ double red[3][256];
  red[0][threadIdx.x] = sx;
  red[1][threadIdx.x] = sy;
  red[2][threadIdx.x] = sz;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int a = 0; a < 3; ++a) red[a][threadIdx.x] += red[a][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int a = 0; a < 3; ++a) partials[3 * blockIdx.x + a] = red[a][0];
  // the last block sums the partials (the former tv3d_finish_kernel)
  if (last_block(counter, (int)gridDim.x) && threadIdx.x < 32)
    tv3d_finish_warp(partials, gridDim.x, dinv_x, dinv_y, dinv_z, value);
}

// fixed-order sum of the block partials: lane j sums partials j, j + 32, ... in
// order, then a fixed xor tree (one warp)
__device__ void tv3d_finish_warp(const double* partials, int n_blocks, double inv_x, double inv_y, double inv_z,
                                 double* value) {
  const int lane = threadIdx.x & 31;
  double s[3] = {0, 0, 0};
  for (int b = lane; b < n_blocks; b += 32)
    for (int a = 0; a < 3; ++a) s[a] += __ldcg(partials + 3 * b + a);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    for (int a = 0; a < 3; ++a) s[a] += __shfl_xor_sync(0xffffffffu, s[a], off);
  if (lane == 0) *value = s[0] * inv_x + s[1] * inv_y + s[2] * inv_z;
}

// ---------------------------------------------------------------- Adam
// One thread per kernel: rho (1), pos (3), scale (3), rot (4) + renormalisation (adam.cuh).
__global__ void __launch_bounds__(256) adam_kernel(long long m, float* __restrict__ rho, float* __restrict__ pos,
                                                   float* __restrict__ sc, float* __restrict__ rot,
                                                   sct_adam_state st, const float* __restrict__ g_rho,
                                                   const float* __restrict__ g_pos, const float* __restrict__ g_sc,
                                                   const float* __restrict__ g_rot, AdamParams ap,
                                                   double* __restrict__ total, double lambda_ssim, double lambda_tv) {
  pdl_prologue();
  // native train step: the total loss of this iteration
  if (total && blockIdx.x == 0 && threadIdx.x == 0) train_total(total, lambda_ssim, lambda_tv);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    float g[11];
    g[0] = g_rho[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) g[1 + k] = g_pos[3 * i + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) g[4 + k] = g_sc[3 * i + k];
#pragma unroll
    for (int k = 0; k < 4; ++k) g[7 + k] = g_rot[4 * i + k];
    adam_kernel_update(i, rho, pos, sc, rot, st, g, ap);
  }
}

// ---------------------------------------------------------------- photometric
constexpr int kWin = 11;
struct Taps {
  float w[kWin];
};

// horizontal valid pass of the five SSIM moments: tmp[img][5][H][Wv]
__global__ void ssim_h_kernel(const float* __restrict__ r, const float* __restrict__ mm, int n, int W, int H,
                              float rscale, Taps taps, float* __restrict__ tmp) {
  pdl_prologue();
  const int Wv = W - kWin + 1;
  const long long total = (long long)n * H * Wv;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(t % Wv);
    const int y = (int)((t / Wv) % H);
    const long long img = t / ((long long)Wv * H);
    const float* ra = r + (img * H + y) * W + x;
    const float* rb = mm + (img * H + y) * W + x;
    float s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
    for (int i = 0; i < kWin; ++i) {
      const float a = ra[i] * rscale, b = rb[i];
      const float w = taps.w[i];
      s0 = fmaf(w, a, s0);
      s1 = fmaf(w, b, s1);
      s2 = fmaf(w, a * a, s2);
      s3 = fmaf(w, b * b, s3);
      s4 = fmaf(w, a * b, s4);
    }
    const long long plane = (long long)H * Wv;
    float* o = tmp + img * 5 * plane + (long long)y * Wv + x;
    o[0] = s0; o[plane] = s1; o[2 * plane] = s2; o[3 * plane] = s3; o[4 * plane] = s4;
  }
}

// Deterministic per-block sum: block b of image img writes partial[img][b];
// photometric_finish_kernel adds the partials in block order.
__device__ __forceinline__ void block_sum_to(double v, double* __restrict__ dst) {
  __shared__ double s_red[8];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += s_red[w];
    *dst = s;
  }
}

// After every block has written its partial(s): true in exactly one block, the
// last to arrive (which then finishes the reduction; counter self-resets).
__device__ __forceinline__ bool last_block(int* counter, int n_blocks) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    s_last = atomicAdd(counter, 1) == n_blocks - 1;
    if (s_last) *counter = 0;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// values[i] = {L1 mean, D-SSIM}: the per-block partials added in block order
// (one warp per image: lane-strided partial sums, then a fixed shuffle tree)
__device__ __forceinline__ void photometric_finish_warp(const double* l1_part, int nb_l1, const double* ssim_part,
                                                        int nb_ssim, double* values, int i, int W, int H) {
  const int Wv = W - kWin + 1, Hv = H - kWin + 1;
  const int lane = threadIdx.x & 31;
  double a = 0.0, b = 0.0;
  for (int k = lane; k < nb_l1; k += 32) a += __ldcg(l1_part + (long long)i * nb_l1 + k);
  for (int k = lane; k < nb_ssim; k += 32) b += __ldcg(ssim_part + (long long)i * nb_ssim + k);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    values[2 * i] = a / ((double)W * H);
    values[2 * i + 1] = 0.5 * (1.0 - b / ((double)Wv * Hv));
  }
}

// vertical valid pass + per-window SSIM partials (objectives.cpp:93-149):
// fields[img][5][Hv][Wv] = g1, g2, g2*mu1, g3, g3*mu2; SSIM-map sum per image
// as per-block partials (grid: blocks per image x images).
__global__ void __launch_bounds__(256) ssim_v_kernel(const float* __restrict__ tmp, int n, int W, int H, Taps taps,
                                                     float* __restrict__ fields, double* __restrict__ partial) {
  pdl_prologue();
  const float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;
  const int Wv = W - kWin + 1, Hv = H - kWin + 1;
  const long long img = blockIdx.y;
  const long long total = (long long)Hv * Wv;
  double acc = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(t % Wv);
    const int y = (int)(t / Wv);
    const long long plane = (long long)H * Wv;
    const float* src = tmp + img * 5 * plane + (long long)y * Wv + x;
    float f[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < kWin; ++j)
#pragma unroll
      for (int k = 0; k < 5; ++k) f[k] = fmaf(taps.w[j], src[k * plane + (long long)j * Wv], f[k]);
    const float mu1 = f[0], mu2 = f[1];
    const float s1 = f[2] - mu1 * mu1, s2 = f[3] - mu2 * mu2, s12 = f[4] - mu1 * mu2;
    const float a1 = 2.f * mu1 * mu2 + kC1, b1 = mu1 * mu1 + mu2 * mu2 + kC1;
    const float a2 = 2.f * s12 + kC2, b2 = s1 + s2 + kC2;
    const float l = a1 / b1, cs = a2 / b2;
    const float g1 = cs * 2.f * (mu2 * b1 - mu1 * a1) / (b1 * b1);
    const float g2 = -l * a2 / (b2 * b2);
    const float g3 = l * 2.f / b2;
    const long long vplane = (long long)Hv * Wv;
    float* o = fields + img * 5 * vplane + (long long)y * Wv + x;
    o[0] = g1; o[vplane] = g2; o[2 * vplane] = g2 * mu1; o[3 * vplane] = g3; o[4 * vplane] = g3 * mu2;
    acc += (double)(l * cs);
  }
  block_sum_to(acc, partial + img * gridDim.x + blockIdx.x);
}

// adjoint vertical pass: atmp[img][5][H][Wv]
__global__ void ssim_adj_v_kernel(const float* __restrict__ fields, int n, int W, int H, Taps taps,
                                  float* __restrict__ atmp) {
  pdl_prologue();
  const int Wv = W - kWin + 1, Hv = H - kWin + 1;
  const long long total = (long long)n * H * Wv;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(t % Wv);
    const int y = (int)((t / Wv) % H);
    const long long img = t / ((long long)Wv * H);
    const long long vplane = (long long)Hv * Wv, plane = (long long)H * Wv;
    float f[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < kWin; ++j) {
      const int yy = y - j;
      if (yy < 0 || yy >= Hv) continue;
      const float* src = fields + img * 5 * vplane + (long long)yy * Wv + x;
#pragma unroll
      for (int k = 0; k < 5; ++k) f[k] = fmaf(taps.w[j], src[k * vplane], f[k]);
    }
    float* o = atmp + img * 5 * plane + (long long)y * Wv + x;
#pragma unroll
    for (int k = 0; k < 5; ++k) o[k * plane] = f[k];
  }
}

// adjoint horizontal pass + dL/dI assembly (objectives.cpp:151-166, trainer.cpp:284-287)
__global__ void __launch_bounds__(256) ssim_adj_h_kernel(const float* __restrict__ atmp, const float* __restrict__ r,
                                                         const float* __restrict__ mm, int n, int W, int H,
                                                         float rscale, Taps taps, float lambda_ssim, float grad_scale,
                                                         float* __restrict__ dL, double* __restrict__ partial,
                                                         const double* __restrict__ ssim_part, int nb_ssim,
                                                         double* __restrict__ values, int* __restrict__ counter) {
  pdl_prologue();
  const int Wv = W - kWin + 1, Hv = H - kWin + 1;
  const float inv_p = 1.f / ((float)Wv * (float)Hv);
  const float inv_n = 1.f / ((float)W * (float)H);
  const long long img = blockIdx.y;
  const long long total = (long long)H * W;
  double acc = 0.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(p % W);
    const int y = (int)(p / W);
    const long long t = img * total + p;
    const long long plane = (long long)H * Wv;
    float f[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < kWin; ++i) {
      const int xx = x - i;
      if (xx < 0 || xx >= Wv) continue;
      const float* src = atmp + img * 5 * plane + (long long)y * Wv + xx;
#pragma unroll
      for (int k = 0; k < 5; ++k) f[k] = fmaf(taps.w[i], src[k * plane], f[k]);
    }
    const float a = r[t] * rscale, b = mm[t];
    const float ds = f[0] + 2.f * a * f[1] - 2.f * f[2] + b * f[3] - f[4];
    const float g_dssim = -0.5f * inv_p * ds;
    const float d = a - b;
    const float g_l1 = d > 0.f ? inv_n : (d < 0.f ? -inv_n : 0.f);
    dL[t] = (g_l1 + lambda_ssim * g_dssim) * grad_scale;
    acc += (double)fabsf(d);
  }
  block_sum_to(acc, partial + img * gridDim.x + blockIdx.x);
  // the last block finishes both losses (the former photometric_finish_kernel)
  if (last_block(counter, (int)(gridDim.x * gridDim.y)))
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
      photometric_finish_warp(partial, gridDim.x, ssim_part, nb_ssim, values, i, W, H);
}

int grid_cap(Ctx* c, long long n, int block) {
  long long b = (n + block - 1) / block;
  const long long cap = (long long)c->sm_count * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

void launch_tv3d(Ctx* c, const float* vol, const int32_t dims[3], float lambda, double* value, float* grad,
                 double* partials, int n_partials) {
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const double cx = (double)(nx - 1) * ny * nz, cy = (double)nx * (ny - 1) * nz, cz = (double)nx * ny * (nz - 1);
  const double ix = cx > 0 ? 1.0 / cx : 0.0, iy = cy > 0 ? 1.0 / cy : 0.0, iz = cz > 0 ? 1.0 / cz : 0.0;
  {
    KScope _ks(c, "K9_tv3d");
    pdl_launch(tv3d_kernel, dim3(n_partials), dim3(256), 0, c->stream, vol, nx, ny, nz, (float)ix, (float)iy, (float)iz, lambda, grad,
                                                   partials, ix, iy, iz, value, c->fin_counter + 1);
  }
}

void launch_adam(Ctx* c, sct_cloud* p, sct_adam_state* st, const sct_grads* g, const float lr[4], float bc1,
                 float bc2, float beta1, float beta2, float eps, double* total, double lambda_ssim,
                 double lambda_tv) {
  if (p->m == 0) return;
  {
    KScope _ks(c, "K10_adam");
    const AdamParams ap{lr[0], lr[1], lr[2], lr[3], bc1, bc2, beta1, beta2, eps};
    pdl_launch(adam_kernel, dim3(grid_cap(c, p->m, 256)), dim3(256), 0, c->stream, p->m, p->rho_raw, p->pos, p->scale_raw, p->rot, *st,
                                                               g->rho_raw, g->pos, g->scale_raw, g->rot, ap, total,
                                                               lambda_ssim, lambda_tv);
  }
}

int photometric_loss(Ctx* c, const float* rendered, const float* measured, int n, int w, int h,
                     float render_scale, float lambda_ssim, float grad_scale, double* values, float* dL) {
  if (w < kWin || h < kWin) {
    set_error("DimMismatch: ssim: image smaller than the 11x11 window");
    return SCT_ERR_DATA;
  }
  Taps taps;
  {
    double t[kWin], sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
      const double x = i - (kWin - 1) / 2.0;
      t[i] = std::exp(-x * x / (2.0 * 1.5 * 1.5));
      sum += t[i];
    }
    for (int i = 0; i < kWin; ++i) taps.w[i] = (float)(t[i] / sum);
  }
  const int Wv = w - kWin + 1, Hv = h - kWin + 1;
  const size_t tmp_elems = (size_t)n * 5 * h * Wv;
  const size_t field_elems = (size_t)n * 5 * Hv * Wv;
  float* tmp = nullptr;
  float* fields = nullptr;
  SCT_TRY(dev_alloc(c, (void**)&tmp, tmp_elems * sizeof(float)));
  SCT_TRY(dev_alloc(c, (void**)&fields, field_elems * sizeof(float)));
  // blocks per image for the two reducing passes (deterministic partials)
  auto per_img = [&](long long px) {
    long long b = (px + 255) / 256;
    const long long cap = std::max<long long>(1, (long long)c->sm_count * 8 / n);
    return (int)std::max<long long>(1, std::min(b, cap));
  };
  const int nb_ssim = per_img((long long)Hv * Wv), nb_l1 = per_img((long long)h * w);
  double* part = nullptr;
  SCT_TRY(stage_buf(c, 23, sizeof(double) * (size_t)n * (nb_ssim + nb_l1), (void**)&part));
  double* ssim_part = part;
  double* l1_part = part + (size_t)n * nb_ssim;
  {
    KScope _ks(c, "K11_ssim_h");
    pdl_launch(ssim_h_kernel, dim3(grid_cap(c, (long long)n * h * Wv, 256)), dim3(256), 0, c->stream, rendered, measured, n, w, h,
                                                                                   render_scale, taps, tmp);
  }
  {
    KScope _ks(c, "K11_ssim_v");
    pdl_launch(ssim_v_kernel, dim3(dim3(nb_ssim, n)), dim3(256), 0, c->stream, tmp, n, w, h, taps, fields, ssim_part);
  }
  {
    KScope _ks(c, "K11_ssim_adj_v");
    pdl_launch(ssim_adj_v_kernel, dim3(grid_cap(c, (long long)n * h * Wv, 256)), dim3(256), 0, c->stream, fields, n, w, h, taps, tmp);
  }
  {
    KScope _ks(c, "K11_ssim_adj_h");
    pdl_launch(ssim_adj_h_kernel, dim3(dim3(nb_l1, n)), dim3(256), 0, c->stream, tmp, rendered, measured, n, w, h, render_scale, taps,
                                                             lambda_ssim, grad_scale, dL, l1_part, ssim_part, nb_ssim,
                                                             values, c->fin_counter);
  }
  dev_free(c, tmp);
  dev_free(c, fields);
  return SCT_OK;
}

}  // namespace sct
