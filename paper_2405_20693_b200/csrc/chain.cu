// FP64 per-Gaussian chain rules (K5, K8-chain).
//
// raster_chain_kernel: L lanes per kernel (L a power of two <= 32 chosen from
//   the view count), lane l taking the kernel's views l, l + L, ... of a view
//   range. Per visible (view, kernel) item: sums the item's per-tile
//   statistics in the reference's fixed tile order (rasterizer.cpp:245-257),
//   rebuilds the projection chain in FP64 (rasterizer.cpp:266-268) and runs
//   rasterizer.cpp:270-327 down to dL/drho, dL/dpos and dL/dSigma. The lanes
//   sum their items in view order, then a fixed xor tree sums the L lanes:
//   the view sums leave the kernel as 11 doubles + a visible count per kernel
//   and view range (no per-item outputs through HBM; deterministic).
// raster_finalize_kernel: one thread per kernel. Sums the view-range partials
//   in range order, then applies the parts of the chain that are linear and
//   view-independent once per kernel: rho through the softplus
//   (rasterizer.cpp:329) and Sigma -> (scale_raw, q_raw)
//   (gaussian_cloud.cpp:151-202). Also the adaptive statistics
//   (rasterizer.cpp:333-340). Accumulates (+=) like the reference.
// voxel_chain_kernel: voxelizer.cpp:192-223 per touched kernel.
#include <cuda_runtime.h>

#include <cstdlib>

#include "adam.cuh"
#include "fp64_math.cuh"
#include "project.cuh"
#include "sct_internal.cuh"

namespace sct {

namespace {

constexpr int kItemOut = 11;  // g_rho, g_pos[3], g_sigma (xx yy zz xy xz yz), ndc_norm

// Symmetric 3x3 as (xx, xy, xz, yy, yz, zz).
struct Sym3 {
  double xx, xy, xz, yy, yz, zz;
};

// K5 item chain. The projection chain is re-derived in FP64 as the reference
// does (rasterizer.cpp:266-268) but written for the GPU: reciprocals computed
// once (5 divisions instead of ~25), symmetric matrices kept as 6 values,
// Sigma and rho read from the per-Gaussian prep record, FMAs allowed. The
// math is the same chain as rasterizer.cpp:270-327; it does not feed binning,
// so it need not be bit-identical to the preprocess.
// the chain of one visible item (view v, kernel i) into out[kItemOut]
template <bool kParallel>
__device__ __forceinline__ void item_chain(long long m, long long v, long long i, const float* __restrict__ pos,
                                           const double* __restrict__ prep, const ViewParams* __restrict__ views,
                                           const DetParams& det, const RasterParams& rp,
                                           const int32_t* __restrict__ offset, const float4* __restrict__ pair_stats,
                                           double out[kItemOut]) {
  {
    const long long item = v * m + i;
    // fixed-order reduction over the item's tiles (rasterizer.cpp:245-257)
    double S0 = 0, S1x = 0, S1y = 0, Sxx = 0, Syy = 0, Sxy = 0;
    // offset == nullptr: parallel-atomic mode, one pre-summed record per item
    const int32_t p0 = offset ? offset[item] : (int32_t)item, p1 = offset ? offset[item + 1] : (int32_t)item + 1;
    for (int32_t p = p0; p < p1; ++p) {
      const float4 a = pair_stats[2 * (long long)p];
      const float2 b = *reinterpret_cast<const float2*>(pair_stats + 2 * (long long)p + 1);
      S0 += a.x;
      S1x += a.y;
      S1y += a.z;
      Sxx += a.w;
      Syy += b.x;
      Sxy += b.y;
    }
    const ViewParams& V = views[v];
    const double* W = V.rot;
    const double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
    auto pr = [&](int a) { return prep[(long long)a * m + i]; };  // SoA [kPrepStride][m]
    const Sym3 Sg{pr(0), pr(1), pr(2), pr(4), pr(5), pr(8)};
    const double rho = pr(9);
    const Sym3 Si{pr(10), pr(11), pr(12), pr(13), pr(14), pr(15)};  // Sigma^-1
    const double detS = pr(16);
    const double x = fma(W[0], px, fma(W[1], py, W[2] * pz)) + V.t[0];
    const double y = fma(W[3], px, fma(W[4], py, W[5] * pz)) + V.t[1];
    const double z = fma(W[6], px, fma(W[7], py, W[8] * pz)) + V.t[2];
    const double iz = d_fast_rcp(z);
    const double n2 = fma(x, x, fma(y, y, z * z));
    const double in = d_fast_rsqrt(n2);
    // J (geometry.cpp:111-123): rows (a 0 b), (0 c d), (e f g)
    // parallel beam: J = diag(fx, fy, 1), constant
    constexpr bool par = kParallel;
    const double ja = par ? det.fx : det.fx * iz, jc = par ? det.fy : det.fy * iz;
    const double jb = par ? 0.0 : -ja * x * iz, jd = par ? 0.0 : -jc * y * iz;
    const double je = par ? 0.0 : x * in, jf = par ? 0.0 : y * in, jg = par ? 1.0 : z * in;
    // A2 = first two rows of A = J W (only they reach the 2D covariance)
    double A[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      A[0][k] = fma(ja, W[k], jb * W[6 + k]);
      A[1][k] = fma(jc, W[3 + k], jd * W[6 + k]);
    }
    // T2 = A2 Sigma; sigma2_raw = T2 A2^T
    double T[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      T[r][0] = fma(A[r][0], Sg.xx, fma(A[r][1], Sg.xy, A[r][2] * Sg.xz));
      T[r][1] = fma(A[r][0], Sg.xy, fma(A[r][1], Sg.yy, A[r][2] * Sg.yz));
      T[r][2] = fma(A[r][0], Sg.xz, fma(A[r][1], Sg.yz, A[r][2] * Sg.zz));
    }
    auto dot3 = [](const double* a, const double* b) { return fma(a[0], b[0], fma(a[1], b[1], a[2] * b[2])); };
    const double Rxx = dot3(T[0], A[0]), Rxy = dot3(T[0], A[1]), Ryy = dot3(T[1], A[1]);
    const double d2r = fma(Rxx, Ryy, -Rxy * Rxy);
    // cofactors of J: J^-T = C / det J; det(sigma_ray) = det(J)^2 det(Sigma)
    // (det W = 1) — exact identities that avoid inverting the ill-conditioned
    // sigma_ray (cond ~1e5)
    const double C00 = fma(jc, jg, -jd * jf), C01 = jd * je, C02 = -jc * je;
    const double C10 = jb * jf, C11 = fma(ja, jg, -jb * je), C12 = -ja * jf;
    const double C20 = -jb * jc, C21 = -ja * jd, C22 = ja * jc;
    const double detJ = fma(ja, C00, jb * C02);
    const double d3 = detJ * detJ * detS;
    const double id2r = d_fast_rcp(d2r);
    const double mu = d_fast_sqrt(2.0 * kPi * d3 * id2r);
    const double amp_pre = (rp.mode == SCT_MODE_RECTIFIED) ? mu * rho : rho;
    const double s00 = Rxx + rp.eps2, s11 = Ryy + rp.eps2, s01 = Rxy;
    const double id2 = d_fast_rcp(fma(s00, s11, -s01 * s01));
    const double comp = rp.dilation_compensation ? d_fast_sqrt(d2r * id2) : 1.0;
    const double amp = amp_pre * comp;
    const double q00 = s11 * id2, q01 = -s01 * id2, q11 = s00 * id2;  // conic
    // rasterizer.cpp:277-281
    const double gcx = amp * fma(q00, S1x, q01 * S1y);
    const double gcy = amp * fma(q01, S1x, q11 * S1y);
    // g_sigma2 = -Q g_Q Q = 1/2 amp Q S2 Q
    const double h = 0.5 * amp;
    const double u00 = fma(q00, Sxx, q01 * Sxy), u01 = fma(q00, Sxy, q01 * Syy);
    const double u10 = fma(q01, Sxx, q11 * Sxy), u11 = fma(q01, Sxy, q11 * Syy);
    double g00 = h * fma(u00, q00, u01 * q01);
    double g01 = h * fma(u00, q01, u01 * q11);
    double g11 = h * fma(u10, q01, u11 * q11);
    // low-pass (rasterizer.cpp:283-293)
    const double ir00 = Ryy * id2r, ir01 = -Rxy * id2r, ir11 = Rxx * id2r;  // sigma2_raw^-1
    double r00 = 0.0, r01 = 0.0, r11 = 0.0;
    double g_amp_pre = S0;
    if (rp.dilation_compensation) {
      g_amp_pre = S0 * comp;
      const double gc = S0 * amp_pre * comp * 0.5;
      r00 = gc * ir00;
      r01 = gc * ir01;
      r11 = gc * ir11;
      g00 -= gc * q00;
      g01 -= gc * q01;
      g11 -= gc * q11;
    }
    r00 += g00;
    r01 += g01;
    r11 += g11;
    // amplitude chain (rasterizer.cpp:295-306): dL/dsigma_ray = hm sigma_ray^-1 + [r 0; 0 0]
    double g_rho, hm = 0.0;
    if (rp.mode == SCT_MODE_RECTIFIED) {
      g_rho = g_amp_pre * mu;
      hm = 0.5 * g_amp_pre * rho * mu;
      r00 -= hm * ir00;
      r01 -= hm * ir01;
      r11 -= hm * ir11;
    } else {
      g_rho = g_amp_pre;
    }
    // g_Sigma = A^T G A (rasterizer.cpp:311) = hm Sigma^-1 + A2^T r A2
    double Vr[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      Vr[0][k] = fma(r00, A[0][k], r01 * A[1][k]);
      Vr[1][k] = fma(r01, A[0][k], r11 * A[1][k]);
    }
    auto arA = [&](int a, int b) { return fma(A[0][a], Vr[0][b], A[1][a] * Vr[1][b]); };
    const Sym3 gS{fma(hm, Si.xx, arA(0, 0)), fma(hm, Si.xy, 0.5 * (arA(0, 1) + arA(1, 0))),
                  fma(hm, Si.xz, 0.5 * (arA(0, 2) + arA(2, 0))), fma(hm, Si.yy, arA(1, 1)),
                  fma(hm, Si.yz, 0.5 * (arA(1, 2) + arA(2, 1))), fma(hm, Si.zz, arA(2, 2))};
    // centre chain (rasterizer.cpp:313-321)
    double gp0 = ja * gcx, gp1 = jc * gcy, gp2 = fma(jb, gcx, jd * gcy);
    if (!rp.freeze_jacobian && !par) {  // dJ/dp = 0 for parallel beam
      // g_A = (G + G^T) A Sigma and g_J = g_A W^T (rasterizer.cpp:310,322-326);
      // with sigma_ray^-1 A Sigma = A^-T and A^-T W^T = J^-T:
      // g_J = 2 hm J^-T + 2 [r A2 Sigma W^T ; 0]
      double X[2][3];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        X[r][0] = fma(Vr[r][0], Sg.xx, fma(Vr[r][1], Sg.xy, Vr[r][2] * Sg.xz));
        X[r][1] = fma(Vr[r][0], Sg.xy, fma(Vr[r][1], Sg.yy, Vr[r][2] * Sg.yz));
        X[r][2] = fma(Vr[r][0], Sg.xz, fma(Vr[r][1], Sg.yz, Vr[r][2] * Sg.zz));
      }
      const double k2 = 2.0 * hm * d_fast_rcp(detJ);
      double gJ[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        gJ[0][c] = 2.0 * fma(X[0][0], W[3 * c], fma(X[0][1], W[3 * c + 1], X[0][2] * W[3 * c + 2]));
        gJ[1][c] = 2.0 * fma(X[1][0], W[3 * c], fma(X[1][1], W[3 * c + 1], X[1][2] * W[3 * c + 2]));
      }
      gJ[0][0] = fma(k2, C00, gJ[0][0]);
      gJ[0][1] = fma(k2, C01, gJ[0][1]);
      gJ[0][2] = fma(k2, C02, gJ[0][2]);
      gJ[1][0] = fma(k2, C10, gJ[1][0]);
      gJ[1][1] = fma(k2, C11, gJ[1][1]);
      gJ[1][2] = fma(k2, C12, gJ[1][2]);
      gJ[2][0] = k2 * C20;
      gJ[2][1] = k2 * C21;
      gJ[2][2] = k2 * C22;
      // dJ/dp contractions (jacobian_derivative, rasterizer.cpp:162-191)
      const double in3 = in * in * in;
      const double fz2 = det.fx * iz * iz, gz2 = det.fy * iz * iz;
      gp0 += -gJ[0][2] * fz2 + gJ[2][0] * (in - x * x * in3) - gJ[2][1] * x * y * in3 - gJ[2][2] * x * z * in3;
      gp1 += -gJ[1][2] * gz2 - gJ[2][0] * x * y * in3 + gJ[2][1] * (in - y * y * in3) - gJ[2][2] * y * z * in3;
      gp2 += -gJ[0][0] * fz2 + gJ[0][2] * 2.0 * fz2 * x * iz - gJ[1][1] * gz2 + gJ[1][2] * 2.0 * gz2 * y * iz -
             gJ[2][0] * x * z * in3 - gJ[2][1] * y * z * in3 + gJ[2][2] * (in - z * z * in3);
    }
    // g_pos = W^T g_ps (rasterizer.cpp:327)
    const double gx = fma(W[0], gp0, fma(W[3], gp1, W[6] * gp2));
    const double gy = fma(W[1], gp0, fma(W[4], gp1, W[7] * gp2));
    const double gz = fma(W[2], gp0, fma(W[5], gp1, W[8] * gp2));
    const double nx = gcx * 0.5 * det.w, ny = gcy * 0.5 * det.h;
    out[0] = g_rho;
    out[1] = gx;
    out[2] = gy;
    out[3] = gz;
    out[4] = gS.xx;
    out[5] = gS.yy;
    out[6] = gS.zz;
    out[7] = gS.xy;
    out[8] = gS.xz;
    out[9] = gS.yz;
    out[10] = d_fast_sqrt(fma(nx, nx, ny * ny));
  }
}

// K5: L lanes per kernel over views [v0, v1); writes vsum[a * m + i] (a < kItemOut:
// the view sums, a = kItemOut: the visible count). All lanes of a warp take the
// same number of kernel iterations (m rounded up to 32 / L) for the shuffles.
#ifndef SCT_CHAIN_MINB
#define SCT_CHAIN_MINB 4
#endif
template <bool kParallel, int L>
__global__ void __launch_bounds__(128, SCT_CHAIN_MINB) raster_chain_kernel(
    long long m, int v0, int v1, const float* __restrict__ pos, const double* __restrict__ prep,
    const ViewParams* __restrict__ views, DetParams det, RasterParams rp, const uint8_t* __restrict__ vis,
    const int32_t* __restrict__ offset, const float4* __restrict__ pair_stats, double* __restrict__ vsum) {
  pdl_prologue();
  // lane-private running sums in shared memory ([a][thread], FP64): keeps the
  // chain's register budget at 128 without spills
  __shared__ double s_acc[kItemOut + 1][128];
  const int tid = threadIdx.x, lane = tid & (L - 1);
  const long long seg_stride = (long long)gridDim.x * blockDim.x / L;
  const long long m_pad = (m + (32 / L) - 1) / (32 / L) * (32 / L);
  for (long long i = (blockIdx.x * (long long)blockDim.x + tid) / L; i < m_pad; i += seg_stride) {
#pragma unroll
    for (int a = 0; a <= kItemOut; ++a) s_acc[a][tid] = 0.0;
    if (i < m) {
      for (int v = v0 + lane; v < v1; v += L) {
        if (!vis[(long long)v * m + i]) continue;  // culled in this view: contributes nothing
        double o[kItemOut];
        item_chain<kParallel>(m, v, i, pos, prep, views, det, rp, offset, pair_stats, o);
#pragma unroll
        for (int a = 0; a < kItemOut; ++a) s_acc[a][tid] += o[a];
        s_acc[kItemOut][tid] += 1.0;
      }
    }
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) {  // fixed tree over the L lanes
      __syncwarp();
      if (lane < off) {
#pragma unroll
        for (int a = 0; a <= kItemOut; ++a) s_acc[a][tid] += s_acc[a][tid + off];
      }
    }
    __syncwarp();
    if (lane == 0 && i < m) {
#pragma unroll
      for (int a = 0; a <= kItemOut; ++a) vsum[a * m + i] = s_acc[a][tid];
    }
    __syncwarp();
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
  // (the Newton reciprocal / root of fp64_math.cuh: gradients only)
  const double inv_nrm = d_fast_rsqrt(k.q[0] * k.q[0] + k.q[1] * k.q[1] + k.q[2] * k.q[2] + k.q[3] * k.q[3]);
  double qn[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) qn[a] = k.q[a] * inv_nrm;
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
  for (int kk = 0; kk < 4; ++kk) g_rot[kk] = (c[kk] - qn[kk] * qc) * inv_nrm;
}

__global__ void __launch_bounds__(128) raster_finalize_kernel(
    long long m, double s_min, const float* __restrict__ rho_raw, const float* __restrict__ pos,
    const float* __restrict__ scale_raw, const float* __restrict__ rot, const double* __restrict__ vsum,
    float* __restrict__ g_rho, float* __restrict__ g_pos,
    float* __restrict__ g_scale, float* __restrict__ g_rotp, float* __restrict__ st_norm,
    int32_t* __restrict__ st_count, float* __restrict__ st_3d, int groups) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    // view-range partials from raster_chain_kernel: [groups][kItemOut + 1][m], summed in range order
    double acc[kItemOut];
#pragma unroll
    for (int a = 0; a < kItemOut; ++a) acc[a] = vsum[a * m + i];
    double nv = vsum[kItemOut * m + i];
    for (int g = 1; g < groups; ++g) {
      const double* p = vsum + (long long)g * (kItemOut + 1) * m;
#pragma unroll
      for (int a = 0; a < kItemOut; ++a) acc[a] += p[a * m + i];
      nv += p[kItemOut * m + i];
    }
    const int nvis = (int)nv;
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

// The native train step's tail (sct_train_step): raster_finalize_kernel's
// per-kernel chain added to gradients that already hold the TV contribution
// (the same two float additions as finalize-then-voxelize_backward: a + b ==
// b + a), the adaptive statistics, and Adam — one pass over the kernels instead
// of two, and the gradients never written back.
__global__ void __launch_bounds__(128) raster_finalize_adam_kernel(
    long long m, double s_min, float* __restrict__ rho_raw, float* __restrict__ pos, float* __restrict__ scale_raw,
    float* __restrict__ rot, const double* __restrict__ vsum, int groups, const float* __restrict__ g_rho,
    const float* __restrict__ g_pos, const float* __restrict__ g_scale, const float* __restrict__ g_rotp,
    float* __restrict__ st_norm, int32_t* __restrict__ st_count, float* __restrict__ st_3d, sct_adam_state adam,
    AdamParams ap, double* __restrict__ total, double lambda_ssim, double lambda_tv) {
  pdl_prologue();
  if (total && blockIdx.x == 0 && threadIdx.x == 0) train_total(total, lambda_ssim, lambda_tv);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    float g[11];
    g[0] = g_rho[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) g[1 + k] = g_pos[3 * i + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) g[4 + k] = g_scale[3 * i + k];
#pragma unroll
    for (int k = 0; k < 4; ++k) g[7 + k] = g_rotp[4 * i + k];
    if (vsum) {
      double acc[kItemOut];
#pragma unroll
      for (int a = 0; a < kItemOut; ++a) acc[a] = vsum[a * m + i];
      double nv = vsum[kItemOut * m + i];
      for (int gi = 1; gi < groups; ++gi) {
        const double* p = vsum + (long long)gi * (kItemOut + 1) * m;
#pragma unroll
        for (int a = 0; a < kItemOut; ++a) acc[a] += p[a * m + i];
        nv += p[kItemOut * m + i];
      }
      const int nvis = (int)nv;
      if (nvis > 0) {  // as raster_finalize_kernel
        const dKernel k = d_load_kernel(pos, scale_raw, rot, rho_raw, i, s_min);
        g[0] += (float)(acc[0] * d_act_density_grad(k.rho_raw));
#pragma unroll
        for (int a = 0; a < 3; ++a) g[1 + a] += (float)acc[1 + a];
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
        for (int a = 0; a < 3; ++a) g[4 + a] += (float)gs[a];
#pragma unroll
        for (int a = 0; a < 4; ++a) g[7 + a] += (float)gr[a];
        if (st_norm) {
          st_norm[i] += (float)acc[10];
          st_count[i] += nvis;
#pragma unroll
          for (int a = 0; a < 3; ++a) st_3d[3 * i + a] += (float)acc[1 + a];
        }
      }
    }
    adam_kernel_update(i, rho_raw, pos, scale_raw, rot, adam, g, ap);
  }
}

// The 10 pair-statistic sums of every kernel (FP64): eight lanes per kernel,
// lane j summing pairs j, j + 8, ... in order, then a fixed xor-shuffle tree
// — deterministic, and eight times the threads of the one-thread-per-kernel
// chain for the latency-bound 48-byte pair gathers.
__global__ void __launch_bounds__(256) voxel_pair_sum_kernel(long long m, const int32_t* __restrict__ offset,
                                                             const int32_t* __restrict__ count,
                                                             const float4* __restrict__ ps,
                                                             double* __restrict__ sums) {
  pdl_prologue();
  const int j = threadIdx.x & 7;
  for (long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 3; g < ((m + 3) & ~3LL);
       g += ((long long)gridDim.x * blockDim.x) >> 3) {  // all lanes of a warp iterate together
    const bool live = g < m;
    const int32_t n = live ? count[g] : 0;
    const long long p0 = live ? offset[g] : 0;
    // FP32 lane sums and tree (the per-pair float -> double conversions and
    // FP64 shuffles bound the kernel on the XU pipe: 0.117 ms at cfg4); the
    // kernel's total is widened once. Same fixed order, so still deterministic.
    float s[10];
#pragma unroll
    for (int a = 0; a < 10; ++a) s[a] = 0.f;
    for (int q = j; q < n; q += 8) {
      const float4 a = __ldg(ps + 3 * (p0 + q)), b = __ldg(ps + 3 * (p0 + q) + 1), c = __ldg(ps + 3 * (p0 + q) + 2);
      s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
      s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
      s[8] += c.x; s[9] += c.y;
    }
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
      for (int a = 0; a < 10; ++a) s[a] += __shfl_xor_sync(0xffffffffu, s[a], off);
    if (live) {  // lane j writes sums j and j + 8 (all lanes hold all ten)
#pragma unroll
      for (int a = 0; a < 10; ++a)
        if ((a & 7) == j) sums[a * m + g] = (double)s[a];
    }
  }
}

// voxelizer.cpp:192-223
__global__ void __launch_bounds__(128) voxel_chain_kernel(
    long long m, double s_min, const float* __restrict__ rho_raw, const float* __restrict__ pos,
    const float* __restrict__ scale_raw, const float* __restrict__ rot, const int32_t* __restrict__ offset,
    const int32_t* __restrict__ count, const float4* __restrict__ ps, const double* __restrict__ sums,
    float* __restrict__ g_rho, float* __restrict__ g_pos, float* __restrict__ g_scale,
    float* __restrict__ g_rotp) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int32_t n = count[i];
    if (n == 0) continue;  // not touched
    double s[10];
    if (sums) {  // pre-summed by voxel_pair_sum_kernel
#pragma unroll
      for (int a = 0; a < 10; ++a) s[a] = sums[a * m + i];
    } else {
#pragma unroll
      for (int a = 0; a < 10; ++a) s[a] = 0.0;
      const long long p0 = offset[i];
      for (long long p = p0; p < p0 + n; ++p) {
        const float4 a = ps[3 * p], b = ps[3 * p + 1], c = ps[3 * p + 2];
        s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
        s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
        s[8] += c.x; s[9] += c.y;
      }
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

int64_t chain_sums_bytes(const sct_fwd* s, int groups) {
  return (int64_t)groups * (kItemOut + 1) * s->m * (int64_t)sizeof(double);
}

template <bool P>
static void chain_launch(int lanes, int grid, cudaStream_t st, long long m, int v0, int v1, const float* pos,
                         const double* prep, const ViewParams* views, const DetParams& det, const RasterParams& rp,
                         const uint8_t* vis, const int32_t* offset, const float4* ps, double* vsum) {
#define SCT_CHAIN_L(L) \
  case L:              \
    pdl_launch(raster_chain_kernel<P, L>, dim3(grid), dim3(128), 0, st, m, v0, v1, pos, prep, views, det, rp, vis, offset, ps, vsum); \
    break;
  switch (lanes) {
    SCT_CHAIN_L(1)
    SCT_CHAIN_L(2)
    SCT_CHAIN_L(4)
    SCT_CHAIN_L(8)
    SCT_CHAIN_L(16)
    SCT_CHAIN_L(32)
  }
#undef SCT_CHAIN_L
}

void launch_raster_chain(Ctx* c, const sct_fwd* s, const sct_cloud& cl, const float4* pair_stats, double* vsum,
                         bool per_item, int v0, int v1, cudaStream_t stream) {
  if (v1 < 0) v1 = s->n_views;
  if (s->m == 0) return;
  cudaStream_t st = stream ? stream : c->stream;
  KScope _ks(c, "K5_raster_chain", true, st);
  // lanes per kernel: the widest power of two up to 4 that leaves at most ~10%
  // of the (view, lane) slots idle (measured at cfg3, 75 views: 1 / 2 / 4 / 16
  // lanes -> 0.42 / 0.35 / 0.34 / 0.45 ms; wider segments scatter the view
  // records and statistics over more lines per load)
  const int nv = std::max(0, v1 - v0);
  int lanes = 4;
  while (lanes > 1 && (long long)((nv + lanes - 1) / lanes) * lanes * 10 > 11LL * nv) lanes >>= 1;
  static const int forced = [] {
    const char* e = std::getenv("SCT_CHAIN_LANES");
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2 || forced == 4 || forced == 8 || forced == 16 || forced == 32) lanes = forced;
  const int grid = grid_cap(c, s->m * lanes, 128);
  const int32_t* off = per_item ? nullptr : s->d_offset;
  if (s->det.parallel)
    chain_launch<true>(lanes, grid, st, s->m, v0, v1, cl.pos, s->d_prep, s->d_views, s->det, s->rp, s->d_vis, off,
                       pair_stats, vsum);
  else
    chain_launch<false>(lanes, grid, st, s->m, v0, v1, cl.pos, s->d_prep, s->d_views, s->det, s->rp, s->d_vis, off,
                        pair_stats, vsum);
}

void launch_raster_finalize(Ctx* c, const sct_fwd* s, const sct_cloud& cl, const double* vsum, int groups,
                            sct_grads* g, sct_stats* st) {
  if (s->m == 0) return;
  KScope _ks(c, "K5_raster_finalize");
  pdl_launch(raster_finalize_kernel, dim3(grid_cap(c, s->m, 128)), dim3(128), 0, c->stream, s->m, cl.s_min_mm, cl.rho_raw, cl.pos, cl.scale_raw, cl.rot, vsum, g->rho_raw, g->pos, g->scale_raw, g->rot,
      st ? st->grad2d_norm_accum : nullptr, st ? st->grad_count : nullptr, st ? st->grad3d_accum : nullptr, groups);
}

void launch_raster_finalize_adam(Ctx* c, int64_t m, const sct_fwd* s, sct_cloud* cl, const double* vsum, int groups,
                                 const sct_grads* g, sct_stats* st, sct_adam_state* adam, const float lr[4],
                                 float bc1, float bc2, float b1, float b2, float eps, double* total,
                                 double lambda_ssim, double lambda_tv) {
  if (m == 0) return;
  (void)s;
  KScope _ks(c, "K10_finalize_adam");
  const AdamParams ap{lr[0], lr[1], lr[2], lr[3], bc1, bc2, b1, b2, eps};
  pdl_launch(raster_finalize_adam_kernel, dim3(grid_cap(c, m, 128)), dim3(128), 0, c->stream, m, cl->s_min_mm, cl->rho_raw, cl->pos, cl->scale_raw, cl->rot, vsum, groups, g->rho_raw, g->pos, g->scale_raw,
      g->rot, st ? st->grad2d_norm_accum : nullptr, st ? st->grad_count : nullptr, st ? st->grad3d_accum : nullptr,
      *adam, ap, total, lambda_ssim, lambda_tv);
}

void launch_voxel_chain(Ctx* c, const sct_cloud& cl, const int32_t* offset, const int32_t* count,
                        const float4* pair_stats, sct_grads* g, int64_t n_bricks) {
  if (cl.m == 0) return;
  double* sums = nullptr;
  if (n_bricks >= 0 && n_bricks <= 512) {  // few pairs per kernel: summed in the chain thread, one launch
    KScope _ks(c, "K8_voxel_chain");
    pdl_launch(voxel_chain_kernel, dim3(grid_cap(c, cl.m, 128)), dim3(128), 0, c->stream, cl.m, cl.s_min_mm, cl.rho_raw, cl.pos,
                                                                     cl.scale_raw, cl.rot, offset, count, pair_stats,
                                                                     nullptr, g->rho_raw, g->pos, g->scale_raw, g->rot);
    return;
  }
  if (dev_alloc(c, (void**)&sums, 10 * cl.m * sizeof(double)) != SCT_OK) return;
  {
    KScope _ks(c, "K8_voxel_pair_sum");
    pdl_launch(voxel_pair_sum_kernel, dim3(grid_cap(c, 8 * cl.m, 256)), dim3(256), 0, c->stream, cl.m, offset, count, pair_stats,
                                                                              sums);
  }
  {
    KScope _ks(c, "K8_voxel_chain");
    pdl_launch(voxel_chain_kernel, dim3(grid_cap(c, cl.m, 128)), dim3(128), 0, c->stream, cl.m, cl.s_min_mm, cl.rho_raw, cl.pos,
                                                                     cl.scale_raw, cl.rot, offset, count, pair_stats,
                                                                     sums, g->rho_raw, g->pos, g->scale_raw, g->rot);
  }
  dev_free(c, sums);
}

}  // namespace sct
