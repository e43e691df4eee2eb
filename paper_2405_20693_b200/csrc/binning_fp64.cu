// Binning preprocess kernels, FP64. This translation unit is compiled with
// -fmad=false: together with the fixed operation order in fp64_math.cuh /
// project.cuh it makes the cull decisions, tile rectangles and brick ranges
// bit-identical to the reference restatement (oracle/splatct_oracle.cpp).
//
//   K1 raster_preprocess  — rasterizer.cpp:24-99 over every (view, kernel)
//   K6 voxel_preprocess   — voxelizer.cpp:52-104 over every kernel
//   project_export        — project_kernel (rasterizer.cpp:103-110)
#include "project.cuh"
#include "sct_internal.cuh"

namespace sct {

namespace {

// K0: view-independent per-Gaussian quantities, once per kernel: the 3D
// covariance Sigma (all 9 entries, d_covariance order — its rounding is not
// symmetric, so both halves are kept) and rho = act_density(rho_raw).
// prep[a][i] (SoA, a = 0..17) = {S00 S01 S02 S10 S11 S12 S20 S21 S22, rho, Sigma^-1 (6), det Sigma, 0}.
__global__ void __launch_bounds__(256) gauss_prep_kernel(long long m, double s_min, const float* __restrict__ rho_raw,
                                                         const float* __restrict__ pos,
                                                         const float* __restrict__ scale_raw,
                                                         const float* __restrict__ rot, double* __restrict__ prep) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const dKernel k = d_load_kernel(pos, scale_raw, rot, rho_raw, i, s_min);
    dM3 r;
    const dM3 s = d_covariance(k, &r);
    auto o = [&](int a) -> double& { return prep[(long long)a * m + i]; };  // SoA: coalesced across kernels
#pragma unroll
    for (int a = 0; a < 9; ++a) o(a) = s.m[a / 3][a % 3];
    o(9) = d_act_density(k.rho_raw);
    // Sigma^-1 = R diag(1/s^2) R^T (well conditioned: no inversion of Sigma)
    // and det Sigma = prod s_k^2, for the chain kernel's identities
    double is2[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) is2[a] = 1.0 / (k.s[a] * k.s[a]);
    const int ij[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const int a = ij[e][0], b = ij[e][1];
      o(10 + e) = __fma_rn(r.m[a][0] * is2[0], r.m[b][0],
                           __fma_rn(r.m[a][1] * is2[1], r.m[b][1], r.m[a][2] * is2[2] * r.m[b][2]));
    }
    o(16) = (k.s[0] * k.s[0]) * (k.s[1] * k.s[1]) * (k.s[2] * k.s[2]);
    o(17) = 0.0;
  }
}

// One thread per (view, kernel) item; item = view * m + kernel (view-major, so
// a stable sort on the (view, tile) key leaves each tile list ascending in
// kernel index exactly like the reference's serial push_back, rasterizer.cpp:124-133).
// (3 CTAs per SM: 80 registers with a small spill beat 95 registers at two
// CTAs — FP64 latency-bound; 0.293 -> 0.285 ms at cfg3)
// K1's projection of one (view, kernel) item. The binning quantities — the
// near-plane test, the centre, the low-pass-dilated 2D covariance and the cull
// — follow d_project (project.cuh) operation for operation: only rows 0-1 of
// A = J W and the top-left 2x2 block of A Sigma A^T reach them, so the tile
// lists stay bit-identical to the oracle's. The record-only quantities (mu,
// amplitude, conic) use det(A Sigma A^T) = det(J)^2 det(Sigma) (det W = 1;
// det J = fx fy n / z^3 for the cone beam, fx fy for the parallel beam) instead
// of the full 3x3 product and its determinant, and the Newton reciprocals /
// roots of fp64_math.cuh: they feed only the FP32 records of K3/K4.
struct BinProj {
  dProj g;  // cx, cy, cov (the tile range's inputs)
  double q00, q01, q11, amp;
};
__device__ __forceinline__ bool d_project_bin(const double p[3], const dM3& sigma, double rho, double det_sigma,
                                              const ViewParams& v, const DetParams& det, const RasterParams& rp,
                                              BinProj& o) {
  double ps[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ps[i] = v.rot[3 * i + 0] * p[0] + v.rot[3 * i + 1] * p[1] + v.rot[3 * i + 2] * p[2];
    ps[i] = ps[i] + v.t[i];
  }
  const bool par = det.parallel != 0;
  if (!par && ps[2] < det.near_clip) return false;
  const double x = ps[0], y = ps[1], z = ps[2];
  double jac[2][3];
  if (par) {
    jac[0][0] = det.fx;
    jac[0][1] = 0.0;
    jac[0][2] = 0.0;
    jac[1][0] = 0.0;
    jac[1][1] = det.fy;
    jac[1][2] = 0.0;
  } else {
    jac[0][0] = det.fx / z;
    jac[0][1] = 0.0;
    jac[0][2] = -det.fx * x / (z * z);
    jac[1][0] = 0.0;
    jac[1][1] = det.fy / z;
    jac[1][2] = -det.fy * y / (z * z);
  }
  // rows 0-1 of d_mul(jac, W), d_mul(a, sigma) and d_mul_bt(., a)
  double a[2][3], X[2][3], sr[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      a[i][j] = jac[i][0] * v.rot[j] + jac[i][1] * v.rot[3 + j] + jac[i][2] * v.rot[6 + j];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      X[i][j] = a[i][0] * sigma.m[0][j] + a[i][1] * sigma.m[1][j] + a[i][2] * sigma.m[2][j];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) sr[i][j] = X[i][0] * a[j][0] + X[i][1] * a[j][1] + X[i][2] * a[j][2];
  const double d2r = sr[0][0] * sr[1][1] - sr[1][0] * sr[0][1];
  dM2& s2 = o.g.cov;
  s2.m[0][0] = sr[0][0] + rp.eps2;
  s2.m[0][1] = sr[0][1];
  s2.m[1][0] = sr[1][0];
  s2.m[1][1] = sr[1][1] + rp.eps2;
  const double cx = par ? det.fx * x + det.cx : det.fx * x / z + det.cx;
  const double cy = par ? det.fy * y + det.cy : det.fy * y / z + det.cy;
  const double rx = rp.cull * sqrt(s2.m[0][0]);
  const double ry = rp.cull * sqrt(s2.m[1][1]);
  if (cx + rx < 0.0 || cx - rx > (double)det.w || cy + ry < 0.0 || cy - ry > (double)det.h) return false;
  o.g.cx = cx;
  o.g.cy = cy;
  // record-only part
  double det_j = det.fx * det.fy;
  if (!par) {
    const double n2 = fma(x, x, fma(y, y, z * z));
    const double iz = d_fast_rcp(z);
    det_j = det_j * (n2 * d_fast_rsqrt(n2)) * (iz * iz * iz);
  }
  const double d3 = det_j * det_j * det_sigma;
  const double mu = d_fast_sqrt(2.0 * kPi * d3 * d_fast_rcp(d2r));
  double amp = (rp.mode == SCT_MODE_RECTIFIED) ? mu * rho : rho;
  const double inv = d_fast_rcp(s2.m[0][0] * s2.m[1][1] - s2.m[1][0] * s2.m[0][1]);
  if (rp.dilation_compensation) amp *= d_fast_sqrt(d2r * inv);
  o.q00 = s2.m[1][1] * inv;
  o.q01 = -s2.m[0][1] * inv;
  o.q11 = s2.m[0][0] * inv;
  o.amp = amp;
  return true;
}

#ifndef SCT_K1_FAST
#define SCT_K1_FAST 1
#endif

__global__ void __launch_bounds__(256, 3) raster_preprocess_kernel(
    long long m, long long n_items, const float* __restrict__ pos, const double* __restrict__ prep,
    const ViewParams* __restrict__ views, DetParams det, RasterParams rp, float4* __restrict__ rec,
    short4* __restrict__ rect, int32_t* __restrict__ count, uint8_t* __restrict__ vis) {
  pdl_prologue();
  const double kA = -0.5 * kLog2e;
  for (long long item = blockIdx.x * (long long)blockDim.x + threadIdx.x; item < n_items;
       item += (long long)gridDim.x * blockDim.x) {
    const long long v = item / m;
    const long long i = item - v * m;
    const double p[3] = {(double)pos[3 * i], (double)pos[3 * i + 1], (double)pos[3 * i + 2]};
    dM3 sigma;
    auto pr = [&](int a) { return prep[(long long)a * m + i]; };
#pragma unroll
    for (int a = 0; a < 9; ++a) sigma.m[a / 3][a % 3] = pr(a);
    const ViewParams view = views[v];
#if SCT_K1_FAST
    BinProj bp;
    const bool ok = d_project_bin(p, sigma, pr(9), pr(16), view, det, rp, bp);
    const dProj& g = bp.g;
#else
    dProj g;
    const bool ok = d_project(p, sigma, pr(9), view, det, rp, g);
#endif
    if (!ok) {
      count[item] = 0;
      vis[item] = 0;
      rect[item] = make_short4(1, 0, 1, 0);
      continue;
    }
    int tx0, tx1, ty0, ty1;
    d_tile_range(g, rp, det.tiles_x, det.tiles_y, tx0, tx1, ty0, ty1);
    const int nx = tx1 - tx0 + 1, ny = ty1 - ty0 + 1;
    const int c = (nx > 0 && ny > 0) ? nx * ny : 0;
    count[item] = c;
    vis[item] = 1;
    rect[item] = make_short4((short)tx0, (short)tx1, (short)ty0, (short)ty1);
    // exp(-1/2 d^T Q d) = exp2(A dx^2 + B dx dy + C dy^2). The FP32 kernels
    // evaluate it as 2^(L + 64) along 4-pixel runs with the ratio recurrence
    // E(dx+1) = E(dx) * 2^(2A dx + A + B dy), ratio(dx+1) = ratio(dx) * 2^(2A);
    // the record carries amp * 2^-64 and K = 2^(2A) for that.
#if SCT_K1_FAST
    const double A = kA * bp.q00;
    rec[2 * item + 0] = make_float4((float)g.cx, (float)g.cy, (float)(bp.amp * 0x1p-64), exp2f((float)(2.0 * A)));
    rec[2 * item + 1] = make_float4((float)A, (float)(2.0 * kA * bp.q01), (float)(kA * bp.q11), (float)(2.0 * A));
#else
    const double A = kA * g.conic.m[0][0];
    rec[2 * item + 0] = make_float4((float)g.cx, (float)g.cy, (float)(g.amp * 0x1p-64), (float)exp2(2.0 * A));
    rec[2 * item + 1] = make_float4((float)A, (float)(2.0 * kA * g.conic.m[0][1]), (float)(kA * g.conic.m[1][1]),
                                    (float)(2.0 * A));
#endif
  }
}

// voxelizer.cpp:52-88 bin_kernels (+ :96-104 precompute). Brick ranges are
// restricted to the z-slab [zb0, zb1) for z-sharding; inside the slab the
// lists equal the full-grid lists.
__global__ void __launch_bounds__(256) voxel_preprocess_kernel(
    long long m, double s_min, const float* __restrict__ rho_raw, const float* __restrict__ pos,
    const float* __restrict__ scale_raw, const float* __restrict__ rot, int3 dims, double3 origin,
    double3 spacing, double cull, int32_t zb0, int32_t zb1, float4* __restrict__ rec,
    short4* __restrict__ lo_out, short4* __restrict__ hi_out, int32_t* __restrict__ count) {
  pdl_prologue();
  const double kA = -0.5 * kLog2e;
  const int dimv[3] = {dims.x, dims.y, dims.z};
  const double org[3] = {origin.x, origin.y, origin.z};
  const double sp[3] = {spacing.x, spacing.y, spacing.z};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const dKernel k = d_load_kernel(pos, scale_raw, rot, rho_raw, i, s_min);
    const dM3 sigma = d_covariance(k);
    int lo[3], hi[3];
    bool empty = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double r = cull * sqrt(fmax(sigma.m[a][a], 0.0));
      const double fa = (k.p[a] - r - org[a]) / sp[a];
      const double fb = (k.p[a] + r - org[a]) / sp[a];
      int v0 = d_floor_int(fa);
      int v1 = d_floor_int(fb);
      v0 = max(v0, 0);
      v1 = min(v1, dimv[a] - 1);
      if (v0 > v1) empty = true;
      lo[a] = v0 / kTileVox;
      hi[a] = v1 / kTileVox;
    }
    if (!empty) {
      lo[2] = max(lo[2], zb0);
      hi[2] = min(hi[2], zb1 - 1);
      if (lo[2] > hi[2]) empty = true;
    }
    count[i] = empty ? 0 : (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
    lo_out[i] = make_short4((short)lo[0], (short)lo[1], (short)lo[2], 0);
    // an empty kernel gets an empty box (hi < lo on every axis): the counting
    // scatter binning reads boxes, not counts
    hi_out[i] = empty ? make_short4((short)(lo[0] - 1), (short)(lo[1] - 1), (short)(lo[2] - 1), 0)
                      : make_short4((short)hi[0], (short)hi[1], (short)hi[2], 0);
    // precompute(): Q = Sigma^-1, rho (log2-scaled for exp2; cross terms doubled)
    const dM3 q = d_inv3(sigma);
    const double rho = d_act_density(k.rho_raw);
    rec[3 * i + 0] = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], (float)rho);
    // .w = K = 2^(2 Qxx sx^2): voxel-to-voxel ratio step of the x recurrence (voxel.cu)
    rec[3 * i + 1] = make_float4((float)(kA * q.m[0][0]), (float)(kA * q.m[1][1]), (float)(kA * q.m[2][2]),
                                 (float)exp2(2.0 * kA * q.m[0][0] * sp[0] * sp[0]));
    rec[3 * i + 2] = make_float4((float)(2.0 * kA * q.m[0][1]), (float)(2.0 * kA * q.m[0][2]),
                                 (float)(2.0 * kA * q.m[1][2]), 0.f);
  }
}

__global__ void project_export_kernel(long long m, double s_min, const float* __restrict__ rho_raw,
                                      const float* __restrict__ pos, const float* __restrict__ scale_raw,
                                      const float* __restrict__ rot, const ViewParams* __restrict__ view,
                                      DetParams det, RasterParams rp, int32_t* __restrict__ vis,
                                      double* __restrict__ out) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const dKernel k = d_load_kernel(pos, scale_raw, rot, rho_raw, i, s_min);
    dProj g;
    const bool ok = d_project(k.p, d_covariance(k), d_act_density(k.rho_raw), view[0], det, rp, g);
    vis[i] = ok ? 1 : 0;
    double* o = out + 11 * i;
    if (!ok) {
      for (int a = 0; a < 11; ++a) o[a] = 0.0;
      continue;
    }
    o[0] = g.cx;
    o[1] = g.cy;
    o[2] = g.cov.m[0][0];
    o[3] = g.cov.m[0][1];
    o[4] = g.cov.m[1][1];
    o[5] = g.conic.m[0][0];
    o[6] = g.conic.m[0][1];
    o[7] = g.conic.m[1][1];
    o[8] = g.amp;
    o[9] = g.mu;
    o[10] = g.depth;
  }
}

int grid_for(Ctx* c, long long n, int block) {
  long long b = (n + block - 1) / block;
  const long long cap = (long long)c->sm_count * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

void launch_gauss_prep(Ctx* c, const sct_cloud& cl, double* prep) {
  if (cl.m == 0) return;
  KScope _ks(c, "K0_gauss_prep");
  pdl_launch(gauss_prep_kernel, dim3(grid_for(c, cl.m, 256)), dim3(256), 0, c->stream, cl.m, cl.s_min_mm, cl.rho_raw, cl.pos,
                                                                   cl.scale_raw, cl.rot, prep);
}

void launch_raster_preprocess(Ctx* c, const sct_cloud& cl, const double* prep, const ViewParams* d_views,
                              int n_views, const DetParams& det, const RasterParams& rp, float4* rec, short4* rect,
                              int32_t* count, uint8_t* vis) {
  const long long n_items = (long long)cl.m * n_views;
  if (n_items == 0) return;
  KScope _ks(c, "K1_raster_preprocess");
  pdl_launch(raster_preprocess_kernel, dim3(grid_for(c, n_items, 256)), dim3(256), 0, c->stream, cl.m, n_items, cl.pos, prep, d_views,
                                                                             det, rp, rec, rect, count, vis);
}

void launch_voxel_preprocess(Ctx* c, const sct_cloud& cl, const sct_grid& g, double cull, int32_t zb0,
                             int32_t zb1, int32_t, int32_t, float4* rec, short4* rect_lo, short4* rect_hi,
                             int32_t* count) {
  if (cl.m == 0) return;
  {
    KScope _ks(c, "K6_voxel_preprocess");
    pdl_launch(voxel_preprocess_kernel, dim3(grid_for(c, cl.m, 256)), dim3(256), 0, c->stream, cl.m, cl.s_min_mm, cl.rho_raw, cl.pos, cl.scale_raw, cl.rot, make_int3(g.dims[0], g.dims[1], g.dims[2]),
        make_double3(g.origin_mm[0], g.origin_mm[1], g.origin_mm[2]),
        make_double3(g.spacing_mm[0], g.spacing_mm[1], g.spacing_mm[2]), cull, zb0, zb1, rec, rect_lo, rect_hi,
        count);
  }
}

void launch_project_export(Ctx* c, const sct_cloud& cl, const ViewParams* d_view, const DetParams& det,
                           const RasterParams& rp, int32_t* vis, double* rec) {
  if (cl.m == 0) return;
  {
    KScope _ks(c, "project_export");
    pdl_launch(project_export_kernel, dim3(grid_for(c, cl.m, 128)), dim3(128), 0, c->stream, cl.m, cl.s_min_mm, cl.rho_raw, cl.pos, cl.scale_raw, cl.rot, d_view, det, rp, vis, rec);
  }
}

}  // namespace sct
