// FP64 per-Gaussian chain rules (K5, K8-chain).
//
// raster_chain_kernel: one thread per visible (view, kernel) item. Sums the
//   item's per-tile statistics in the reference's fixed tile order
//   (rasterizer.cpp:245-257), rebuilds the projection chain in FP64
//   (rasterizer.cpp:266-268) and runs rasterizer.cpp:270-327 down to
//   dL/drho, dL/dpos and dL/dSigma. Writes 11 floats per item.
// raster_finalize_kernel: one thread per kernel. Sums its items over the
//   views in view order, then applies the parts of the chain that are linear
//   and view-independent once per kernel: rho through the softplus
//   (rasterizer.cpp:329) and Sigma -> (scale_raw, q_raw)
//   (gaussian_cloud.cpp:151-202). Also the adaptive statistics
//   (rasterizer.cpp:333-340). Accumulates (+=) like the reference.
// voxel_chain_kernel: voxelizer.cpp:192-223 per touched kernel.
#include <cuda_runtime.h>

#include "fp64_math.cuh"
#include "project.cuh"
#include "sct_internal.cuh"

namespace sct {

namespace {

constexpr int kItemOut = 11;  // g_rho, g_pos[3], g_sigma (xx yy zz xy xz yz), ndc_norm

// d(J)/d(p_c) contracted with g_jac: sum_ab g_jac(a,b) * dJ/dp_c(a,b)
// (rasterizer.cpp:162-191, :322-326)
__device__ __forceinline__ double jac_contract(const dM3& gj, const DetParams& det, const double p[3], int c) {
  const double x = p[0], y = p[1], z = p[2];
  const double n = sqrt(x * x + y * y + z * z);
  const double n3 = n * n * n;
  if (c == 0)
    return gj.m[0][2] * (-det.fx / (z * z)) + gj.m[2][0] * (1.0 / n - x * x / n3) + gj.m[2][1] * (-x * y / n3) +
           gj.m[2][2] * (-x * z / n3);
  if (c == 1)
    return gj.m[1][2] * (-det.fy / (z * z)) + gj.m[2][0] * (-x * y / n3) + gj.m[2][1] * (1.0 / n - y * y / n3) +
           gj.m[2][2] * (-y * z / n3);
  return gj.m[0][0] * (-det.fx / (z * z)) + gj.m[0][2] * (2.0 * det.fx * x / (z * z * z)) +
         gj.m[1][1] * (-det.fy / (z * z)) + gj.m[1][2] * (2.0 * det.fy * y / (z * z * z)) +
         gj.m[2][0] * (-x * z / n3) + gj.m[2][1] * (-y * z / n3) + gj.m[2][2] * (1.0 / n - z * z / n3);
}

__global__ void __launch_bounds__(128) raster_chain_kernel(
    long long m, long long n_items, double s_min, const float* __restrict__ rho_raw, const float* __restrict__ pos,
    const float* __restrict__ scale_raw, const float* __restrict__ rot, const ViewParams* __restrict__ views,
    DetParams det, RasterParams rp, const uint8_t* __restrict__ vis, const int32_t* __restrict__ offset,
    const float4* __restrict__ pair_stats, float* __restrict__ out) {
  for (long long item = blockIdx.x * (long long)blockDim.x + threadIdx.x; item < n_items;
       item += (long long)gridDim.x * blockDim.x) {
    if (!vis[item]) continue;
    const long long v = item / m;
    const long long i = item - v * m;
    // fixed-order reduction over the item's tiles
    double S0 = 0, S1x = 0, S1y = 0, Sxx = 0, Syy = 0, Sxy = 0;
    const int32_t p0 = offset[item], p1 = offset[item + 1];
    for (int32_t p = p0; p < p1; ++p) {
      const float4 a = pair_stats[2 * (long long)p];
      const float4 b = pair_stats[2 * (long long)p + 1];
      S0 += a.x;
      S1x += a.y;
      S1y += a.z;
      Sxx += a.w;
      Syy += b.x;
      Sxy += b.y;
    }
    const dKernel k = d_load_kernel(pos, scale_raw, rot, rho_raw, i, s_min);
    const ViewParams view = views[v];
    dProj g;
    d_project(k, view, det, rp, g);  // visible by construction (vis[item])
    const dM2& q = g.conic;
    // pixel value: amp * exp(-1/2 d^T Q d), d = x - p_hat   (rasterizer.cpp:277-281)
    const double g_amp = S0;
    const double gcx = g.amp * (q.m[0][0] * S1x + q.m[0][1] * S1y);
    const double gcy = g.amp * (q.m[1][0] * S1x + q.m[1][1] * S1y);
    dM2 gq;
    gq.m[0][0] = -0.5 * g.amp * Sxx;
    gq.m[0][1] = -0.5 * g.amp * Sxy;
    gq.m[1][0] = -0.5 * g.amp * Sxy;
    gq.m[1][1] = -0.5 * g.amp * Syy;
    dM2 t, gs2;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) t.m[a][b] = -q.m[a][0] * gq.m[0][b] + -q.m[a][1] * gq.m[1][b];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) gs2.m[a][b] = t.m[a][0] * q.m[0][b] + t.m[a][1] * q.m[1][b];
    // low-pass (rasterizer.cpp:283-293)
    double g_amp_pre = g_amp;
    dM2 gs2r;
    gs2r.m[0][0] = gs2r.m[0][1] = gs2r.m[1][0] = gs2r.m[1][1] = 0.0;
    const dM2 inv_raw = d_inv2(g.s2r);
    if (rp.dilation_compensation) {
      g_amp_pre = g_amp * g.comp;
      const double g_comp = g_amp * g.amp_pre;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          gs2r.m[a][b] += g_comp * 0.5 * g.comp * inv_raw.m[a][b];
          gs2.m[a][b] += g_comp * (-0.5) * g.comp * q.m[a][b];
        }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) gs2r.m[a][b] += gs2.m[a][b];
    // amplitude chain (rasterizer.cpp:295-306)
    dM3 G = d_zero3();
    double g_rho;
    if (rp.mode == SCT_MODE_RECTIFIED) {
      g_rho = g_amp_pre * g.mu;
      const double g_mu = g_amp_pre * g.rho;
      const dM3 inv_ray = d_inv3(g.sigma_ray);
      const double c3 = g_mu * 0.5 * g.mu, c2 = g_mu * (-0.5) * g.mu;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) G.m[a][b] += c3 * inv_ray.m[a][b];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) gs2r.m[a][b] += c2 * inv_raw.m[a][b];
    } else {
      g_rho = g_amp_pre;
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) G.m[a][b] += gs2r.m[a][b];
    // sigma_ray = A Sigma A^T (rasterizer.cpp:308-311)
    const dM3 gsig = d_mul(d_mul_at(g.a, G), g.a);
    // centre chain + dJ/dp chain (rasterizer.cpp:313-327)
    const double zc = g.ps[2];
    double gp[3];
    gp[0] = (det.fx / zc) * gcx;
    gp[1] = (det.fy / zc) * gcy;
    gp[2] = (-det.fx * g.ps[0] / (zc * zc)) * gcx + (-det.fy * g.ps[1] / (zc * zc)) * gcy;
    if (!rp.freeze_jacobian) {
      const dM3 g_a = d_mul(d_mul(d_add_t(G), g.a), g.sigma);
      dM3 W;
#pragma unroll
      for (int a = 0; a < 9; ++a) W.m[a / 3][a % 3] = view.rot[a];
      const dM3 g_jac = d_mul_bt(g_a, W);
#pragma unroll
      for (int c = 0; c < 3; ++c) gp[c] += jac_contract(g_jac, det, g.ps, c);
    }
    double gpos[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      gpos[a] = view.rot[0 * 3 + a] * gp[0] + view.rot[1 * 3 + a] * gp[1] + view.rot[2 * 3 + a] * gp[2];
    const double nx = gcx * 0.5 * det.w, ny = gcy * 0.5 * det.h;
    // item outputs, [kItemOut][n_items]
    out[0 * n_items + item] = (float)g_rho;
    out[1 * n_items + item] = (float)gpos[0];
    out[2 * n_items + item] = (float)gpos[1];
    out[3 * n_items + item] = (float)gpos[2];
    out[4 * n_items + item] = (float)gsig.m[0][0];
    out[5 * n_items + item] = (float)gsig.m[1][1];
    out[6 * n_items + item] = (float)gsig.m[2][2];
    out[7 * n_items + item] = (float)(0.5 * (gsig.m[0][1] + gsig.m[1][0]));
    out[8 * n_items + item] = (float)(0.5 * (gsig.m[0][2] + gsig.m[2][0]));
    out[9 * n_items + item] = (float)(0.5 * (gsig.m[1][2] + gsig.m[2][1]));
    out[10 * n_items + item] = (float)sqrt(nx * nx + ny * ny);
  }
}

// gaussian_cloud.cpp:151-202 accumulate_covariance_param_grads for a
// symmetric dL/dSigma (Gs), adding into g_scale[3], g_rot[4].
__device__ __forceinline__ void d_cov_param_grads(const dKernel& k, const dM3& Gs, double g_scale[3],
                                                  double g_rot[4]) {
  const dM3 r = d_rotation_matrix(k.q);
  dM3 d = d_zero3();
#pragma unroll
  for (int a = 0; a < 3; ++a) d.m[a][a] = k.s[a] * k.s[a];
  const dM3 g_r = d_mul(d_mul(d_add_t(Gs), r), d);
  const dM3 g_d = d_mul(d_mul_at(r, Gs), r);
#pragma unroll
  for (int a = 0; a < 3; ++a) g_scale[a] = g_d.m[a][a] * 2.0 * k.s[a] * exp(k.sraw[a]);
  // rotation_matrix_jacobian with the normalisation chain
  const double nrm = sqrt(k.q[0] * k.q[0] + k.q[1] * k.q[1] + k.q[2] * k.q[2] + k.q[3] * k.q[3]);
  double qn[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) qn[a] = k.q[a] / nrm;
  const double w = qn[0], x = qn[1], y = qn[2], z = qn[3];
  // dR/d(qn_l) contracted with g_r: c_l = 2 * sum(g_r .* dn_l)
  double c[4];
  c[0] = 2.0 * (g_r.m[0][1] * -z + g_r.m[0][2] * y + g_r.m[1][0] * z + g_r.m[1][2] * -x + g_r.m[2][0] * -y +
                g_r.m[2][1] * x);
  c[1] = 2.0 * (g_r.m[0][1] * y + g_r.m[0][2] * z + g_r.m[1][0] * y + g_r.m[1][1] * (-2 * x) + g_r.m[1][2] * -w +
                g_r.m[2][0] * z + g_r.m[2][1] * w + g_r.m[2][2] * (-2 * x));
  c[2] = 2.0 * (g_r.m[0][0] * (-2 * y) + g_r.m[0][1] * x + g_r.m[0][2] * w + g_r.m[1][0] * x + g_r.m[1][2] * z +
                g_r.m[2][0] * -w + g_r.m[2][1] * z + g_r.m[2][2] * (-2 * y));
  c[3] = 2.0 * (g_r.m[0][0] * (-2 * z) + g_r.m[0][1] * -w + g_r.m[0][2] * x + g_r.m[1][0] * w +
                g_r.m[1][1] * (-2 * z) + g_r.m[1][2] * y + g_r.m[2][0] * x + g_r.m[2][1] * y);
  const double qc = qn[0] * c[0] + qn[1] * c[1] + qn[2] * c[2] + qn[3] * c[3];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) g_rot[kk] = (c[kk] - qn[kk] * qc) / nrm;
}

__global__ void __launch_bounds__(128) raster_finalize_kernel(
    long long m, int n_views, double s_min, const float* __restrict__ rho_raw, const float* __restrict__ pos,
    const float* __restrict__ scale_raw, const float* __restrict__ rot, const uint8_t* __restrict__ vis,
    const float* __restrict__ item, float* __restrict__ g_rho, float* __restrict__ g_pos,
    float* __restrict__ g_scale, float* __restrict__ g_rotp, float* __restrict__ st_norm,
    int32_t* __restrict__ st_count, float* __restrict__ st_3d) {
  const long long n_items = m * n_views;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    double acc[kItemOut];
#pragma unroll
    for (int a = 0; a < kItemOut; ++a) acc[a] = 0.0;
    int nvis = 0;
    for (int v = 0; v < n_views; ++v) {
      const long long it = (long long)v * m + i;
      if (!vis[it]) continue;
      ++nvis;
#pragma unroll
      for (int a = 0; a < kItemOut; ++a) acc[a] += (double)item[a * n_items + it];
    }
    if (nvis == 0) continue;
    const dKernel k = d_load_kernel(pos, scale_raw, rot, rho_raw, i, s_min);
    g_rho[i] += (float)(acc[0] * d_act_density_grad(k.rho_raw));
#pragma unroll
    for (int a = 0; a < 3; ++a) g_pos[3 * i + a] += (float)acc[1 + a];
    dM3 Gs;
    Gs.m[0][0] = acc[4];
    Gs.m[1][1] = acc[5];
    Gs.m[2][2] = acc[6];
    Gs.m[0][1] = Gs.m[1][0] = acc[7];
    Gs.m[0][2] = Gs.m[2][0] = acc[8];
    Gs.m[1][2] = Gs.m[2][1] = acc[9];
    double gs[3], gr[4];
    d_cov_param_grads(k, Gs, gs, gr);
#pragma unroll
    for (int a = 0; a < 3; ++a) g_scale[3 * i + a] += (float)gs[a];
#pragma unroll
    for (int a = 0; a < 4; ++a) g_rotp[4 * i + a] += (float)gr[a];
    if (st_norm) {
      st_norm[i] += (float)acc[10];
      st_count[i] += nvis;
#pragma unroll
      for (int a = 0; a < 3; ++a) st_3d[3 * i + a] += (float)acc[1 + a];
    }
  }
}

// voxelizer.cpp:192-223
__global__ void __launch_bounds__(128) voxel_chain_kernel(
    long long m, double s_min, const float* __restrict__ rho_raw, const float* __restrict__ pos,
    const float* __restrict__ scale_raw, const float* __restrict__ rot, const int32_t* __restrict__ offset,
    const int32_t* __restrict__ count, const float4* __restrict__ ps, float* __restrict__ g_rho,
    float* __restrict__ g_pos, float* __restrict__ g_scale, float* __restrict__ g_rotp) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int32_t n = count[i];
    if (n == 0) continue;  // not touched
    double s[10];
#pragma unroll
    for (int a = 0; a < 10; ++a) s[a] = 0.0;
    const long long p0 = offset[i];
    for (long long p = p0; p < p0 + n; ++p) {
      const float4 a = ps[3 * p], b = ps[3 * p + 1], c = ps[3 * p + 2];
      s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
      s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
      s[8] += c.x; s[9] += c.y;
    }
    const dKernel k = d_load_kernel(pos, scale_raw, rot, rho_raw, i, s_min);
    const dM3 q = d_inv3(d_covariance(k));
    const double rho = d_act_density(k.rho_raw);
    g_rho[i] += (float)(s[0] * d_act_density_grad(k.rho_raw));
    const double s1[3] = {s[1], s[2], s[3]};
#pragma unroll
    for (int a = 0; a < 3; ++a)
      g_pos[3 * i + a] += (float)(rho * (q.m[a][0] * s1[0] + q.m[a][1] * s1[1] + q.m[a][2] * s1[2]));
    // s2 order xx yy zz xy xz yz; g_q = -1/2 rho s2; g_sigma = -Q g_q Q = 1/2 rho Q s2 Q
    dM3 s2;
    s2.m[0][0] = s[4]; s2.m[1][1] = s[5]; s2.m[2][2] = s[6];
    s2.m[0][1] = s2.m[1][0] = s[7];
    s2.m[0][2] = s2.m[2][0] = s[8];
    s2.m[1][2] = s2.m[2][1] = s[9];
    dM3 gq;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) gq.m[a][b] = -0.5 * rho * s2.m[a][b];
    dM3 nq;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) nq.m[a][b] = -q.m[a][b];
    const dM3 gsig = d_mul(d_mul(nq, gq), q);
    double gs[3], gr[4];
    d_cov_param_grads(k, gsig, gs, gr);
#pragma unroll
    for (int a = 0; a < 3; ++a) g_scale[3 * i + a] += (float)gs[a];
#pragma unroll
    for (int a = 0; a < 4; ++a) g_rotp[4 * i + a] += (float)gr[a];
  }
}

int grid_cap(Ctx* c, long long n, int block) {
  long long b = (n + block - 1) / block;
  const long long cap = (long long)c->sm_count * 32;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

void launch_raster_chain(Ctx* c, const sct_fwd* s, const sct_cloud& cl, const float4* pair_stats,
                         float* item_grads) {
  if (s->n_items == 0) return;
  {
    KScope _ks(c, "K5_raster_chain");
    raster_chain_kernel<<<grid_cap(c, s->n_items, 128), 128, 0, c->stream>>>(
        s->m, s->n_items, cl.s_min_mm, cl.rho_raw, cl.pos, cl.scale_raw, cl.rot, s->d_views, s->det, s->rp, s->d_vis,
        s->d_offset, pair_stats, item_grads);
  }
}

void launch_raster_finalize(Ctx* c, const sct_fwd* s, const sct_cloud& cl, const float* item_grads, sct_grads* g,
                            sct_stats* st) {
  if (s->m == 0) return;
  {
    KScope _ks(c, "K5_raster_finalize");
    raster_finalize_kernel<<<grid_cap(c, s->m, 128), 128, 0, c->stream>>>(
        s->m, s->n_views, cl.s_min_mm, cl.rho_raw, cl.pos, cl.scale_raw, cl.rot, s->d_vis, item_grads, g->rho_raw,
        g->pos, g->scale_raw, g->rot, st ? st->grad2d_norm_accum : nullptr, st ? st->grad_count : nullptr,
        st ? st->grad3d_accum : nullptr);
  }
}

void launch_voxel_chain(Ctx* c, const sct_cloud& cl, const int32_t* offset, const int32_t* count,
                        const float4* pair_stats, sct_grads* g) {
  if (cl.m == 0) return;
  {
    KScope _ks(c, "K8_voxel_chain");
    voxel_chain_kernel<<<grid_cap(c, cl.m, 128), 128, 0, c->stream>>>(cl.m, cl.s_min_mm, cl.rho_raw, cl.pos,
                                                                     cl.scale_raw, cl.rot, offset, count, pair_stats,
                                                                     g->rho_raw, g->pos, g->scale_raw, g->rot);
  }
}

}  // namespace sct
