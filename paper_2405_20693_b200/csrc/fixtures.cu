// Fixture generation on the device: the input side of
// the hot path, which the reference runs on the CPU before training.
//   K12 phantom        simulator.cpp:31-65   analytic ellipsoid phantom, FP64
//   K13 projector      simulator.cpp:87-132  composite-midpoint quadrature of the
//                                            trilinear volume along each pixel ray, FP64
//   noise (host)       simulator.cpp:134-158 Poisson + Gaussian with the reference's
//                                            std::mt19937_64 per-view streams (views in parallel)
//   K14 FDK filter     fdk.cpp:53-98         cosine weight + ramp / Hann filter as a direct
//                                            FP64 convolution with the filter's spatial kernel
//   K15 FDK backproj.  fdk.cpp:100-134       distance-weighted bilinear backprojection, FP64
//   K16 NN distances   fdk.cpp:136-201       exact nearest-neighbour distances, FP64 tiles
//   init               fdk.cpp:203-247       occupancy + partial Fisher-Yates + jitter on the
//                                            host (sequential std::mt19937_64), NN + trilinear
//                                            density + raw parameters on the device
// This TU is compiled with -fmad=false: the FP64 comparisons that decide
// phantom membership, ray/box clipping, detector bounds and nearest
// neighbours follow the oracle's IEEE sequence.
//
// Ramp filter: ramp_response() is the DFT of the band-limited Ram-Lak kernel
// h[n] (fdk.cpp:22-43), optionally times the Hann window 0.5(1+cos 2πk/P);
// the row is zero-padded to P >= 2W, so the FFT product is exactly the linear
// convolution with IDFT(response): h itself, or for Hann the three-tap
// smoothing 0.25 h[n-1] + 0.5 h[n] + 0.25 h[n+1]. K14 applies that kernel
// directly (W^2 FMAs per row; B200 FP64 makes this ~0.5 ms at 75 x 512^2).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <random>
#include <thread>
#include <vector>

#include "sct_internal.cuh"

namespace sct {
namespace {

constexpr int kMaxEllipsoids = 32;

struct Ellipsoids {
  int n;
  double v[kMaxEllipsoids][10];  // intensity a b c x0 y0 z0 cos(phi) sin(phi) -
};

__global__ void phantom_kernel(Ellipsoids E, int nx, int ny, int nz, double3 origin, double3 spacing,
                               double3 center, double3 half, float* __restrict__ out) {
  const int64_t n = (int64_t)nx * ny * nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((int64_t)nx * ny));
    const double px = (origin.x + (x + 0.5) * spacing.x - center.x) / half.x;
    const double py = (origin.y + (y + 0.5) * spacing.y - center.y) / half.y;
    const double pz = (origin.z + (z + 0.5) * spacing.z - center.z) / half.z;
    double v = 0.0;
    for (int e = 0; e < E.n; ++e) {
      const double* P = E.v[e];
      const double dx = px - P[4], dy = py - P[5], dz = pz - P[6];
      const double c = P[7], s = P[8];
      const double xr = c * dx + s * dy;
      const double yr = -s * dx + c * dy;
      const double q = (xr * xr) / (P[1] * P[1]) + (yr * yr) / (P[2] * P[2]) + (dz * dz) / (P[3] * P[3]);
      if (q <= 1.0) v += P[0];
    }
    out[i] = (float)v;
  }
}

struct VolGeo {
  int nx, ny, nz;
  double ox, oy, oz, sx, sy, sz;
};

// voxelizer.cpp:16-37
__device__ double trilinear(const float* __restrict__ vol, const VolGeo& g, double x, double y, double z) {
  const double p[3] = {x, y, z}, o[3] = {g.ox, g.oy, g.oz}, s[3] = {g.sx, g.sy, g.sz};
  const int dims[3] = {g.nx, g.ny, g.nz};
  int ix[3], f1[3];
  double w[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double gk = (p[k] - o[k]) / s[k] - 0.5;
    const double c = fmin(fmax(gk, 0.0), (double)(dims[k] - 1));
    ix[k] = min((int)floor(c), dims[k] - 1);
    f1[k] = min(ix[k] + 1, dims[k] - 1);
    w[k] = c - ix[k];
  }
  double out = 0.0;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const double weight = (dx ? w[0] : 1 - w[0]) * (dy ? w[1] : 1 - w[1]) * (dz ? w[2] : 1 - w[2]);
        const int64_t idx = ((int64_t)(dz ? f1[2] : ix[2]) * g.ny + (dy ? f1[1] : ix[1])) * g.nx + (dx ? f1[0] : ix[0]);
        out += weight * (double)__ldg(vol + idx);
      }
  return out;
}

struct ViewRot {
  double m[9];  // W(theta), row-major (geometry.cpp:76-86)
};

struct ScanGeo {
  double l_so, l_sd, dw, dh;
  int w, h, parallel;
};

__device__ __forceinline__ void view_rot(double s, double c, double m[9]) {
  m[0] = -s; m[1] = c; m[2] = 0.0;
  m[3] = 0.0; m[4] = 0.0; m[5] = -1.0;
  m[6] = -c; m[7] = -s; m[8] = 0.0;
}

// simulator.cpp:109-132, one thread per (view, pixel); sin/cos of the view angles
// come from the host (the reference's libm values)
__global__ void project_volume_kernel(const float* __restrict__ vol, VolGeo g, ScanGeo sc,
                                      const double2* __restrict__ sincos_v, int n_views, double step,
                                      float* __restrict__ out) {
  const int64_t npx = (int64_t)sc.w * sc.h;
  const int64_t n = npx * n_views;
  const double lo[3] = {g.ox, g.oy, g.oz};
  const double hi[3] = {g.ox + g.sx * (double)g.nx, g.oy + g.sy * (double)g.ny, g.oz + g.sz * (double)g.nz};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int view = (int)(i / npx);
    const int64_t px = i - (int64_t)view * npx;
    const int u = (int)(px % sc.w), v = (int)(px / sc.w);
    // geometry.cpp:125-138 pixel_ray
    const double du = sc.dw / sc.w, dv = sc.dh / sc.h;
    const double xd = (u + 0.5) * du - 0.5 * sc.dw;
    const double yd = (v + 0.5) * dv - 0.5 * sc.dh;
    double m[9];
    view_rot(sincos_v[view].x, sincos_v[view].y, m);
    double o[3], d[3];
    if (sc.parallel) {  // parallel-beam extension: ray through (xd, yd) along the view axis
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o[k] = m[0 * 3 + k] * xd + m[1 * 3 + k] * yd + m[2 * 3 + k] * -sc.l_so;
        d[k] = m[0 * 3 + k] * 0.0 + m[1 * 3 + k] * 0.0 + m[2 * 3 + k] * 1.0;
      }
    } else {
      const double nrm = sqrt(xd * xd + yd * yd + sc.l_sd * sc.l_sd);
      const double ds[3] = {xd / nrm, yd / nrm, sc.l_sd / nrm};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o[k] = -(m[0 * 3 + k] * 0.0 + m[1 * 3 + k] * 0.0 + m[2 * 3 + k] * sc.l_so);
        d[k] = m[0 * 3 + k] * ds[0] + m[1 * 3 + k] * ds[1] + m[2 * 3 + k] * ds[2];
      }
    }
    // simulator.cpp:90-107 box_clip
    double t0 = 0.0, t1 = INFINITY;
    bool hit = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (fabs(d[k]) < 1e-15) {
        if (o[k] < lo[k] || o[k] > hi[k]) hit = false;
        continue;
      }
      double a = (lo[k] - o[k]) / d[k];
      double b = (hi[k] - o[k]) / d[k];
      if (a > b) {
        const double t = a;
        a = b;
        b = t;
      }
      t0 = fmax(t0, a);
      t1 = fmin(t1, b);
    }
    double val = 0.0;
    if (hit && t1 > t0) {
      const int ns = max(1, (int)ceil((t1 - t0) / step));
      const double h = (t1 - t0) / ns;
      double sum = 0.0;
      for (int j = 0; j < ns; ++j) {
        const double t = t0 + (j + 0.5) * h;
        sum += trilinear(vol, g, o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]);
      }
      val = sum * h;
    }
    out[i] = (float)val;
  }
}

// K14: one CTA per (view, row). Row (cosine-weighted, FP64) and the spatial
// filter kernel g[-(W-1) .. W-1] in shared memory; output u = sum_j row[j] g[u-j].
__global__ void fdk_filter_kernel(const float* __restrict__ images, ScanGeo sc, const double* __restrict__ gker,
                                  double da, double* __restrict__ filt) {
  extern __shared__ double sm[];
  const int w = sc.w, h = sc.h;
  double* row = sm;           // [w]
  double* gk = sm + w;        // [2w-1], gk[n + w - 1] = g[n]
  const int view = blockIdx.x / h, v = blockIdx.x % h;
  const double du = sc.dw / w, dv = sc.dh / h;
  const double yd = (v + 0.5) * dv - 0.5 * sc.dh;
  const float* src = images + ((int64_t)view * h + v) * w;
  for (int u = threadIdx.x; u < w; u += blockDim.x) {
    const double xd = (u + 0.5) * du - 0.5 * sc.dw;
    const double cosw = sc.l_sd / sqrt(sc.l_sd * sc.l_sd + xd * xd + yd * yd);
    row[u] = (double)src[u] * cosw;
  }
  for (int k = threadIdx.x; k < 2 * w - 1; k += blockDim.x) gk[k] = gker[k];
  __syncthreads();
  double* dst = filt + ((int64_t)view * h + v) * w;
  for (int u = threadIdx.x; u < w; u += blockDim.x) {
    double acc = 0.0;
    const double* gu = gk + u + w - 1;  // gu[-j] = g[u - j]
    for (int j = 0; j < w; ++j) acc = __fma_rn(row[j], gu[-j], acc);
    dst[u] = acc * da;
  }
}

struct FdkGeo {
  double l_so, l_sd, dw, dh, du, dv;
  int w, h;
};

// K15: one thread per voxel, views looped in order (fdk.cpp:110-132)
__global__ void fdk_backproject_kernel(const double* __restrict__ filt, FdkGeo f, VolGeo g,
                                       const double2* __restrict__ sincos_v, int n_views, double scale,
                                       float* __restrict__ out) {
  const int64_t n = (int64_t)g.nx * g.ny * g.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.nx), y = (int)((i / g.nx) % g.ny), z = (int)(i / ((int64_t)g.nx * g.ny));
    const double p0 = g.ox + (x + 0.5) * g.sx, p1 = g.oy + (y + 0.5) * g.sy, p2 = g.oz + (z + 0.5) * g.sz;
    double acc = 0.0;
    for (int vi = 0; vi < n_views; ++vi) {
      double m[9];
      view_rot(sincos_v[vi].x, sincos_v[vi].y, m);
      const double pc0 = m[0] * p0 + m[1] * p1 + m[2] * p2;
      const double pc1 = m[3] * p0 + m[4] * p1 + m[5] * p2;
      const double pc2 = (m[6] * p0 + m[7] * p1 + m[8] * p2) + f.l_so;
      if (pc2 <= 0.0) continue;
      const double xd = pc0 * f.l_sd / pc2;
      const double yd = pc1 * f.l_sd / pc2;
      const double uc = (xd + 0.5 * f.dw) / f.du - 0.5;
      const double vc = (yd + 0.5 * f.dh) / f.dv - 0.5;
      if (uc < 0.0 || uc > f.w - 1 || vc < 0.0 || vc > f.h - 1) continue;
      const int u0 = min((int)uc, f.w - 2);
      const int v0 = min((int)vc, f.h - 2);
      const double fu = uc - u0, fv = vc - v0;
      const double* q = filt + (int64_t)vi * f.w * f.h;
      const double val = (1 - fu) * (1 - fv) * q[v0 * f.w + u0] + fu * (1 - fv) * q[v0 * f.w + u0 + 1] +
                         (1 - fu) * fv * q[(v0 + 1) * f.w + u0] + fu * fv * q[(v0 + 1) * f.w + u0 + 1];
      const double ratio = f.l_so / pc2;
      acc += ratio * ratio * val;
    }
    out[i] = (float)(scale * acc);
  }
}

// K16: exact nearest-neighbour distances. Each CTA takes 128 query points and
// streams all points through shared memory in tiles of 256.
constexpr int kNNThreads = 128, kNNTile = 256;
__global__ void __launch_bounds__(kNNThreads) nn_kernel(int n, const double* __restrict__ pts,
                                                        double* __restrict__ out) {
  __shared__ double tile[kNNTile * 3];
  const int i = blockIdx.x * kNNThreads + threadIdx.x;
  double qx = 0, qy = 0, qz = 0;
  if (i < n) {
    qx = pts[3 * i];
    qy = pts[3 * i + 1];
    qz = pts[3 * i + 2];
  }
  double best = INFINITY;
  for (int base = 0; base < n; base += kNNTile) {
    const int cnt = min(kNNTile, n - base);
    __syncthreads();
    for (int k = threadIdx.x; k < 3 * cnt; k += kNNThreads) tile[k] = pts[3 * (int64_t)base + k];
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      const double dx = qx - tile[3 * j], dy = qy - tile[3 * j + 1], dz = qz - tile[3 * j + 2];
      const double d2 = dx * dx + dy * dy + dz * dz;
      if (base + j != i) best = fmin(best, d2);
    }
  }
  if (i < n) out[i] = n < 2 ? 0.0 : sqrt(best);
}

__device__ __forceinline__ double d_density_inv(double rho) {  // gaussian_cloud.cpp:15-20
  return rho > 30.0 ? rho : rho + log1p(-exp(-rho));
}

// fdk.cpp:233-245 + add_kernel (gaussian_cloud.cpp:48-72): raw parameters
__global__ void init_params_kernel(int count, const double* __restrict__ pos, const double* __restrict__ nn,
                                   const float* __restrict__ vol, VolGeo g, double density_scale, double s_min,
                                   sct_cloud out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const double s = fmax(nn[i], s_min * (1.0 + 1e-6));
    const double rho = fmax(density_scale * trilinear(vol, g, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), 1e-6);
    out.rho_raw[i] = (float)d_density_inv(rho);
    const float sr = (float)log(s - s_min);
    for (int k = 0; k < 3; ++k) {
      out.pos[3 * i + k] = (float)pos[3 * i + k];
      out.scale_raw[3 * i + k] = sr;
    }
    out.rot[4 * i] = 1.f;
    out.rot[4 * i + 1] = out.rot[4 * i + 2] = out.rot[4 * i + 3] = 0.f;
  }
}

int grid_blocks(Ctx* c, int64_t n, int block) {
  int64_t b = (n + block - 1) / block;
  const int64_t cap = (int64_t)c->sm_count * 32;
  return (int)std::max<int64_t>(1, std::min(b, cap));
}

VolGeo vol_geo(const sct_grid* g) {
  return VolGeo{g->dims[0], g->dims[1], g->dims[2], g->origin_mm[0], g->origin_mm[1], g->origin_mm[2],
                g->spacing_mm[0], g->spacing_mm[1], g->spacing_mm[2]};
}

int check_scan(const sct_scanner* s) {
  if (!s || s->det_res_px[0] <= 0 || s->det_res_px[1] <= 0 || !(s->det_size_mm[0] > 0.0) ||
      !(s->det_size_mm[1] > 0.0) || !(s->l_so_mm > 0.0) || !(s->l_sd_mm > s->l_so_mm)) {
    set_error("ConfigError: scanner: invalid detector resolution/size or distances");
    return SCT_ERR_CONFIG;
  }
  return SCT_OK;
}

int check_vol_grid(const sct_grid* g) {
  if (!g || g->dims[0] <= 0 || g->dims[1] <= 0 || g->dims[2] <= 0 || !(g->spacing_mm[0] > 0.0) ||
      !(g->spacing_mm[1] > 0.0) || !(g->spacing_mm[2] > 0.0)) {
    set_error("ConfigError: grid dims and spacing must be positive");
    return SCT_ERR_CONFIG;
  }
  return SCT_OK;
}

int upload_sincos(Ctx* c, const double* thetas, int n, double2** d) {
  std::vector<double2> h(n);
  for (int i = 0; i < n; ++i) h[i] = make_double2(std::sin(thetas[i]), std::cos(thetas[i]));
  SCT_TRY(stage_buf(c, 18, n * sizeof(double2), (void**)d));
  SCT_CUDA_TRY(cudaMemcpyAsync(*d, h.data(), n * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));  // h is a stack buffer
  return SCT_OK;
}

// simulator.cpp:134-141
uint64_t view_seed(uint64_t master, int view) {
  uint64_t z = master + 0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(view) + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace
}  // namespace sct

using namespace sct;

extern "C" {

int sct_phantom(sct_ctx* c, int32_t n_ellipsoids, const double* ellipsoids, const double lo_mm[3],
                const double hi_mm[3], const int32_t dims[3], float* vol) {
  if (!c || !ellipsoids || !lo_mm || !hi_mm || !dims || !vol || n_ellipsoids < 0 ||
      n_ellipsoids > kMaxEllipsoids) {
    set_error("ConfigError: phantom: bad arguments (at most 32 ellipsoids)");
    return SCT_ERR_CONFIG;
  }
  if (std::min({dims[0], dims[1], dims[2]}) < 16) {  // simulator.cpp:47-48
    set_error("ConfigError: phantom: dims must be >= 16 per axis");
    return SCT_ERR_CONFIG;
  }
  Ellipsoids E{};
  E.n = n_ellipsoids;
  for (int e = 0; e < n_ellipsoids; ++e) {
    for (int k = 0; k < 7; ++k) E.v[e][k] = ellipsoids[8 * e + k];
    E.v[e][7] = std::cos(ellipsoids[8 * e + 7]);
    E.v[e][8] = std::sin(ellipsoids[8 * e + 7]);
  }
  double3 o, s, ce, ha;
  double* od = &o.x;
  double* sd = &s.x;
  double* cd = &ce.x;
  double* hd = &ha.x;
  for (int k = 0; k < 3; ++k) {
    od[k] = lo_mm[k];
    sd[k] = (hi_mm[k] - lo_mm[k]) / static_cast<double>(dims[k]);
    cd[k] = 0.5 * (lo_mm[k] + hi_mm[k]);
    hd[k] = 0.5 * (hi_mm[k] - lo_mm[k]);
  }
  const int64_t n = (int64_t)dims[0] * dims[1] * dims[2];
  {
    KScope _ks(c, "K12_phantom");
    phantom_kernel<<<grid_blocks(c, n, 256), 256, 0, c->stream>>>(E, dims[0], dims[1], dims[2], o, s, ce, ha, vol);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_project_volume(sct_ctx* c, const float* vol, const sct_grid* grid, const sct_scanner* scanner,
                       const double* thetas, int32_t n_views, double step_mm, float* images) {
  if (!c || !vol || !thetas || !images || n_views < 0) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(check_vol_grid(grid));
  SCT_TRY(check_scan(scanner));
  if (!(step_mm > 0.0)) {
    set_error("ConfigError: project_volume: step_mm must be > 0");
    return SCT_ERR_CONFIG;
  }
  if (n_views == 0) return SCT_OK;
  double2* sc = nullptr;
  SCT_TRY(upload_sincos(c, thetas, n_views, &sc));
  const ScanGeo g{scanner->l_so_mm, scanner->l_sd_mm, scanner->det_size_mm[0], scanner->det_size_mm[1],
                  scanner->det_res_px[0], scanner->det_res_px[1], scanner->parallel_beam != 0};
  const int64_t n = (int64_t)g.w * g.h * n_views;
  {
    KScope _ks(c, "K13_project_volume");
    project_volume_kernel<<<grid_blocks(c, n, 128), 128, 0, c->stream>>>(vol, vol_geo(grid), g, sc, n_views,
                                                                          step_mm, images);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_add_noise_host(float* images, int32_t n_views, int32_t w, int32_t h, double i0, double gauss_sigma,
                       uint64_t seed, int32_t view0) {
  if (!images || n_views < 0 || w <= 0 || h <= 0) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  if (!(i0 > 0.0)) {  // simulator.cpp:144
    set_error("ConfigError: add_noise: i0 must be > 0");
    return SCT_ERR_CONFIG;
  }
  const int64_t npx = (int64_t)w * h;
  auto one_view = [&](int v) {  // simulator.cpp:143-157 with view_rng(seed, view0 + v)
    std::mt19937_64 rng(view_seed(seed, view0 + v));
    std::normal_distribution<double> gauss(0.0, 1.0);
    const double log_i0 = std::log(i0);
    float* img = images + v * npx;
    for (int64_t i = 0; i < npx; ++i) {
      const double lambda = i0 * std::exp(-static_cast<double>(img[i]));
      std::poisson_distribution<long> poisson(lambda);
      double counts = static_cast<double>(poisson(rng));
      if (gauss_sigma > 0.0) counts += gauss_sigma * gauss(rng);
      counts = std::max(counts, 1.0);
      img[i] = static_cast<float>(log_i0 - std::log(counts));
    }
  };
  const int nt = std::max(1, std::min<int>(n_views, (int)std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (int v = t; v < n_views; v += nt) one_view(v);
    });
  for (auto& th : pool) th.join();
  return SCT_OK;
}

int sct_fdk(sct_ctx* c, const float* images, int32_t n_views, const sct_scanner* scanner, const double* thetas,
            const sct_grid* grid, int32_t window, float* vol) {
  if (!c || !images || !thetas || !vol) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(check_vol_grid(grid));
  SCT_TRY(check_scan(scanner));
  if (scanner->parallel_beam) {
    set_error("ConfigError: fdk: cone-beam geometry only (fdk.cpp is Feldkamp-Davis-Kress)");
    return SCT_ERR_CONFIG;
  }
  if (n_views < 2) {  // fdk.cpp:55
    set_error("DataError: fdk: need at least 2 views");
    return SCT_ERR_DATA;
  }
  const int w = scanner->det_res_px[0], h = scanner->det_res_px[1];
  const double du = scanner->det_size_mm[0] / w, dv = scanner->det_size_mm[1] / h;
  const double da = du * (scanner->l_so_mm / scanner->l_sd_mm);
  const bool hann = window == 1 || (window == 2 && n_views < 100);
  size_t padded = 1;
  while (padded < static_cast<size_t>(2 * w)) padded <<= 1;
  // spatial kernel g[n], |n| < w (fdk.cpp:22-43; see the header comment)
  auto ramp = [&](long n) -> double {
    n = n < 0 ? -n : n;
    n %= (long)padded;
    if (n > (long)padded / 2) n = (long)padded - n;
    if (n == 0) return 1.0 / (4.0 * da * da);
    if (n % 2 == 1) return -1.0 / (M_PI * M_PI * n * n * da * da);
    return 0.0;
  };
  std::vector<double> gk(2 * w - 1);
  for (int k = 0; k < 2 * w - 1; ++k) {
    const long n = k - (w - 1);
    gk[k] = hann ? 0.25 * ramp(n - 1) + 0.5 * ramp(n) + 0.25 * ramp(n + 1) : ramp(n);
  }
  double* d_gk = nullptr;
  double* filt = nullptr;
  SCT_TRY(stage_buf(c, 19, gk.size() * sizeof(double), (void**)&d_gk));
  SCT_CUDA_TRY(cudaMemcpyAsync(d_gk, gk.data(), gk.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  SCT_TRY(dev_alloc(c, (void**)&filt, (size_t)n_views * w * h * sizeof(double)));
  const ScanGeo sg{scanner->l_so_mm, scanner->l_sd_mm, scanner->det_size_mm[0], scanner->det_size_mm[1], w, h, 0};
  const size_t smem = (3 * (size_t)w - 1) * sizeof(double);
  if (smem > 48 * 1024) SCT_CUDA_TRY(cudaFuncSetAttribute(fdk_filter_kernel,
                                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  {
    KScope _ks(c, "K14_fdk_filter");
    fdk_filter_kernel<<<n_views * h, 256, smem, c->stream>>>(images, sg, d_gk, da, filt);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  // fdk.cpp:45-51 median angular gap, fdk.cpp:100 scaling
  std::vector<double> a(thetas, thetas + n_views);
  std::sort(a.begin(), a.end());
  std::vector<double> gaps;
  for (size_t i = 1; i < a.size(); ++i) gaps.push_back(a[i] - a[i - 1]);
  std::sort(gaps.begin(), gaps.end());
  const double dtheta = gaps[gaps.size() / 2];
  double2* sc = nullptr;
  SCT_TRY(upload_sincos(c, thetas, n_views, &sc));
  const FdkGeo fg{scanner->l_so_mm, scanner->l_sd_mm, scanner->det_size_mm[0], scanner->det_size_mm[1], du, dv, w, h};
  const int64_t n = (int64_t)grid->dims[0] * grid->dims[1] * grid->dims[2];
  {
    KScope _ks(c, "K15_fdk_backproject");
    fdk_backproject_kernel<<<grid_blocks(c, n, 128), 128, 0, c->stream>>>(filt, fg, vol_geo(grid), sc, n_views,
                                                                           0.5 * dtheta, vol);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  dev_free(c, filt);
  return SCT_OK;
}

int sct_nn_distances(sct_ctx* c, int64_t n, const double* points, double* out) {
  if (!c || n < 0 || (n > 0 && (!points || !out)) || n > INT32_MAX) {
    set_error("ConfigError: nn_distances: bad arguments");
    return SCT_ERR_CONFIG;
  }
  if (n == 0) return SCT_OK;
  {
    KScope _ks(c, "K16_nn_distances");
    nn_kernel<<<(int)((n + kNNThreads - 1) / kNNThreads), kNNThreads, 0, c->stream>>>((int)n, points, out);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_sample_init_cloud(sct_ctx* c, const float* vol, const sct_grid* grid, int32_t count,
                          double density_threshold, double density_scale, double s_min_mm, uint64_t seed,
                          sct_cloud* out) {
  if (!c || !vol || !out || count < 0 || out->m != count) {
    set_error("ConfigError: sample_init_cloud: bad arguments (out->m must equal count)");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(check_vol_grid(grid));
  const int nx = grid->dims[0], ny = grid->dims[1], nz = grid->dims[2];
  const int64_t nvox = (int64_t)nx * ny * nz;
  std::vector<float> hv(nvox);
  SCT_CUDA_TRY(cudaMemcpyAsync(hv.data(), vol, nvox * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  // fdk.cpp:205-230 on the host: the sampling consumes one sequential std::mt19937_64 stream
  std::vector<int64_t> occ;
  for (int64_t i = 0; i < nvox; ++i)
    if (static_cast<double>(hv[i]) > density_threshold) occ.push_back(i);
  if ((int64_t)occ.size() < count) {
    set_error("DataError: init: only " + std::to_string(occ.size()) +
              " voxels above the density threshold, need " + std::to_string(count));
    return SCT_ERR_DATA;
  }
  if (count == 0) return SCT_OK;
  std::mt19937_64 rng(seed);
  for (int i = 0; i < count; ++i) {
    std::uniform_int_distribution<size_t> pick(i, occ.size() - 1);
    std::swap(occ[i], occ[pick(rng)]);
  }
  std::uniform_real_distribution<double> jitter(-0.5, 0.5);
  std::vector<double> pos(3 * (size_t)count);
  for (int i = 0; i < count; ++i) {
    const int64_t idx = occ[i];
    const int xyz[3] = {(int)(idx % nx), (int)((idx / nx) % ny), (int)(idx / ((int64_t)nx * ny))};
    for (int k = 0; k < 3; ++k) {
      double p = grid->origin_mm[k] + (xyz[k] + 0.5) * grid->spacing_mm[k];
      p += jitter(rng) * grid->spacing_mm[k];
      pos[3 * i + k] = p;
    }
  }
  double *d_pos = nullptr, *d_nn = nullptr;
  SCT_TRY(dev_alloc(c, (void**)&d_pos, pos.size() * sizeof(double)));
  SCT_TRY(dev_alloc(c, (void**)&d_nn, (size_t)count * sizeof(double)));
  SCT_CUDA_TRY(cudaMemcpyAsync(d_pos, pos.data(), pos.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  SCT_TRY(sct_nn_distances(c, count, d_pos, d_nn));
  {
    KScope _ks(c, "init_params");
    init_params_kernel<<<grid_blocks(c, count, 256), 256, 0, c->stream>>>(count, d_pos, d_nn, vol, vol_geo(grid),
                                                                          density_scale, s_min_mm, *out);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  dev_free(c, d_pos);
  dev_free(c, d_nn);
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));  // pos is a host vector
  return SCT_OK;
}

}  // extern "C"
