// Adaptive density control on the device:
// trainer.cpp:167-230 — prune kernels with rho < threshold, then for kernels
// with mean screen-space gradient above threshold clone (small kernels: parent
// and copy share the density, the copy moves down the accumulated position
// gradient by the mean scale) or split (large kernels: two children with
// scales / split_factor at positions sampled from the parent's Gaussian).
// GaussianCloud::remove_kernels (gaussian_cloud.cpp:89-110) becomes an
// order-preserving stream compaction (exclusive scan of the keep flags),
// add_kernel (:48-72) an append in parent order with zero Adam state, and the
// statistics are reset.
//
// Random draws: the split positions use 6 standard-normal draws per split
// kernel, supplied by the caller in the reference's consumption order (per
// split kernel, per child: the z, y, x draws — GCC evaluates the Vec3
// constructor arguments right to left), so a host-seeded std::mt19937_64
// stream reproduces the reference exactly.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "fp64_math.cuh"
#include "sct_internal.cuh"

namespace sct {

namespace {

__device__ __forceinline__ double d_act_density_inv(double rho) {  // gaussian_cloud.cpp:15-20
  return rho > 30.0 ? rho : rho + log1p(-exp(-rho));
}

struct ACParams {
  double prune, densify, size_thr, split_factor, s_min;
};

// action: 0 none, 1 clone, 2 split; keep_out: parent survives; n_new: children
__global__ void ac_classify_kernel(long long m, const float* __restrict__ rho_raw, const float* __restrict__ scale_raw,
                                   const float* __restrict__ norm_acc, const int32_t* __restrict__ count,
                                   ACParams P, uint8_t* __restrict__ action, int32_t* __restrict__ keep_out,
                                   int32_t* __restrict__ n_new, int32_t* __restrict__ is_split) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const double rho = d_act_density((double)rho_raw[i]);
    int a = 0;
    const bool keep = !(rho < P.prune);
    if (keep && count[i] != 0) {
      const double mean_grad = (double)norm_acc[i] / count[i];
      const double rho_half = 0.5 * rho;
      if (mean_grad > P.densify && rho_half > 0.0) {
        double smax = 0.0;
        for (int k = 0; k < 3; ++k) smax = fmax(smax, P.s_min + exp((double)scale_raw[3 * i + k]));
        a = smax <= P.size_thr ? 1 : 2;
      }
    }
    action[i] = (uint8_t)a;
    keep_out[i] = keep && a != 2;
    n_new[i] = a == 1 ? 1 : (a == 2 ? 2 : 0);
    is_split[i] = a == 2;
  }
}

__global__ void ac_apply_kernel(long long m, long long m_kept, sct_cloud in, sct_adam_state ain,
                                const float* __restrict__ g3d, const uint8_t* __restrict__ action,
                                const int32_t* __restrict__ keep_out, const int32_t* __restrict__ keep_pos,
                                const int32_t* __restrict__ new_pos, const int32_t* __restrict__ split_ord,
                                const double* __restrict__ gauss, ACParams P, sct_cloud out, sct_adam_state aout) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int a = action[i];
    const double rho = d_act_density((double)in.rho_raw[i]);
    const double rho_half = 0.5 * rho;
    if (keep_out[i]) {  // remove_kernels: order-preserving compaction of params and Adam state
      const long long o = keep_pos[i];
      out.rho_raw[o] = a == 1 ? (float)d_act_density_inv(rho_half) : in.rho_raw[i];  // clone halves the parent
      for (int k = 0; k < 3; ++k) {
        out.pos[3 * o + k] = in.pos[3 * i + k];
        out.scale_raw[3 * o + k] = in.scale_raw[3 * i + k];
        aout.m_pos[3 * o + k] = ain.m_pos[3 * i + k];
        aout.v_pos[3 * o + k] = ain.v_pos[3 * i + k];
        aout.m_scale[3 * o + k] = ain.m_scale[3 * i + k];
        aout.v_scale[3 * o + k] = ain.v_scale[3 * i + k];
      }
      for (int k = 0; k < 4; ++k) {
        out.rot[4 * o + k] = in.rot[4 * i + k];
        aout.m_rot[4 * o + k] = ain.m_rot[4 * i + k];
        aout.v_rot[4 * o + k] = ain.v_rot[4 * i + k];
      }
      aout.m_rho[o] = ain.m_rho[i];
      aout.v_rho[o] = ain.v_rho[i];
    }
    if (a == 0) continue;
    // children: add_kernel(activated values) -> raw, zero Adam state
    double q[4], qr[4];
    {
      for (int k = 0; k < 4; ++k) qr[k] = (double)in.rot[4 * i + k];
      const double n1 = sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
      double q1[4];
      for (int k = 0; k < 4; ++k) q1[k] = qr[k] / n1;  // kernel(i).rotation
      const double n2 = sqrt(q1[0] * q1[0] + q1[1] * q1[1] + q1[2] * q1[2] + q1[3] * q1[3]);
      for (int k = 0; k < 4; ++k) q[k] = q1[k] / n2;  // add_kernel normalises again
    }
    double s[3], p[3];
    for (int k = 0; k < 3; ++k) {
      s[k] = P.s_min + exp((double)in.scale_raw[3 * i + k]);
      p[k] = (double)in.pos[3 * i + k];
    }
    const int nc = a == 1 ? 1 : 2;
    for (int c = 0; c < nc; ++c) {
      const long long o = m_kept + new_pos[i] + c;
      double cp[3], cs[3];
      if (a == 1) {  // clone: displaced down the accumulated position gradient (trainer.cpp:197-208)
        const double gd[3] = {(double)g3d[3 * i], (double)g3d[3 * i + 1], (double)g3d[3 * i + 2]};
        const double norm = sqrt(gd[0] * gd[0] + gd[1] * gd[1] + gd[2] * gd[2]);
        const double smean = (s[0] + s[1] + s[2]) / 3.0;
        for (int k = 0; k < 3; ++k) {
          cp[k] = norm > 0.0 ? p[k] - (smean / norm) * gd[k] : p[k];
          cs[k] = s[k];
        }
      } else {  // split (trainer.cpp:209-223)
        const dM3 R = d_rotation_matrix(qr);  // rotation_matrix() of the raw quaternion
        const double* g = gauss + 6 * (long long)split_ord[i] + 3 * c;
        const double local[3] = {g[2] * s[0], g[1] * s[1], g[0] * s[2]};
        for (int k = 0; k < 3; ++k) {
          cp[k] = p[k] + (R.m[k][0] * local[0] + R.m[k][1] * local[1] + R.m[k][2] * local[2]);
          cs[k] = fmax(s[k] / P.split_factor, P.s_min * (1.0 + 1e-6));
        }
      }
      out.rho_raw[o] = (float)d_act_density_inv(rho_half);
      aout.m_rho[o] = 0.f;
      aout.v_rho[o] = 0.f;
      for (int k = 0; k < 3; ++k) {
        out.pos[3 * o + k] = (float)cp[k];
        out.scale_raw[3 * o + k] = (float)log(cs[k] - P.s_min);
        aout.m_pos[3 * o + k] = aout.v_pos[3 * o + k] = 0.f;
        aout.m_scale[3 * o + k] = aout.v_scale[3 * o + k] = 0.f;
      }
      for (int k = 0; k < 4; ++k) {
        out.rot[4 * o + k] = (float)q[k];
        aout.m_rot[4 * o + k] = aout.v_rot[4 * o + k] = 0.f;
      }
    }
  }
}

int grid_cap(Ctx* c, long long n, int block) {
  long long b = (n + block - 1) / block;
  const long long cap = (long long)c->sm_count * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

}  // namespace sct

using namespace sct;

struct sct_ac_plan {
  Ctx* ctx = nullptr;
  int64_t m = 0, m_kept = 0, n_new = 0, n_split = 0;
  int32_t counts[3] = {0, 0, 0};  // pruned, cloned, split
  ACParams P{};
  uint8_t* action = nullptr;
  int32_t *keep_out = nullptr, *keep_pos = nullptr, *n_new_arr = nullptr, *new_pos = nullptr;
  int32_t *is_split = nullptr, *split_ord = nullptr;
};

static void ac_release(sct_ac_plan* p) {
  Ctx* c = p->ctx;
  dev_free(c, p->action);
  dev_free(c, p->keep_out);
  dev_free(c, p->keep_pos);
  dev_free(c, p->n_new_arr);
  dev_free(c, p->new_pos);
  dev_free(c, p->is_split);
  dev_free(c, p->split_ord);
}

static int ac_scan(Ctx* c, int32_t* in, int32_t* out, int64_t n, int64_t* total) {
  // exclusive scan of in[0..n) with the total, via the n+1-element trick
  SCT_CUDA_TRY(cudaMemsetAsync(in + n, 0, sizeof(int32_t), c->stream));
  size_t tmp = 0;
  SCT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n + 1, c->stream));
  SCT_TRY(ensure_cub_tmp(c, tmp));
  tmp = c->cub_tmp_bytes;
  SCT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(c->cub_tmp, tmp, in, out, n + 1, c->stream));
  int32_t t = 0;
  SCT_CUDA_TRY(cudaMemcpyAsync(&t, out + n, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  *total = t;
  return SCT_OK;
}

extern "C" {

int sct_adaptive_plan(sct_ctx* c, const sct_cloud* cloud, const sct_stats* stats, double prune_density_threshold,
                      double densify_grad_threshold, double split_scale_threshold_frac, double split_factor,
                      const double extent_size_mm[3], sct_ac_plan** plan, int64_t* new_m, int64_t* n_split,
                      int32_t counts[3]) {
  if (!c || !cloud || !stats || !plan || !extent_size_mm) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  if (!(split_factor > 1.0)) {
    set_error("ConfigError: train: split_factor must be > 1");
    return SCT_ERR_CONFIG;
  }
  auto* p = new sct_ac_plan();
  p->ctx = c;
  p->m = cloud->m;
  p->P.prune = prune_density_threshold;
  p->P.densify = densify_grad_threshold;
  p->P.size_thr =
      split_scale_threshold_frac * fmax(extent_size_mm[0], fmax(extent_size_mm[1], extent_size_mm[2]));
  p->P.split_factor = split_factor;
  p->P.s_min = cloud->s_min_mm;
  const int64_t m = cloud->m;
  int rc = SCT_OK;
  auto fail = [&](int r) {
    ac_release(p);
    delete p;
    return r;
  };
  if ((rc = dev_alloc(c, (void**)&p->action, m + 1))) return fail(rc);
  int32_t** arrs[6] = {&p->keep_out, &p->keep_pos, &p->n_new_arr, &p->new_pos, &p->is_split, &p->split_ord};
  for (auto* a : arrs)
    if ((rc = dev_alloc(c, (void**)a, (m + 1) * sizeof(int32_t)))) return fail(rc);
  if (m > 0) {
    KScope _ks(c, "AC_classify");
    ac_classify_kernel<<<grid_cap(c, m, 256), 256, 0, c->stream>>>(
        m, cloud->rho_raw, cloud->scale_raw, stats->grad2d_norm_accum, stats->grad_count, p->P, p->action,
        p->keep_out, p->n_new_arr, p->is_split);
  }
  int64_t kept = 0, nn = 0, ns = 0;
  if ((rc = ac_scan(c, p->keep_out, p->keep_pos, m, &kept))) return fail(rc);
  if ((rc = ac_scan(c, p->n_new_arr, p->new_pos, m, &nn))) return fail(rc);
  if ((rc = ac_scan(c, p->is_split, p->split_ord, m, &ns))) return fail(rc);
  p->m_kept = kept;
  p->n_new = nn;
  p->n_split = ns;
  // counts: pruned = m - kept - split; cloned = n_new - 2 split
  p->counts[2] = (int32_t)ns;
  p->counts[1] = (int32_t)(nn - 2 * ns);
  p->counts[0] = (int32_t)(m - kept - ns);
  if (new_m) *new_m = kept + nn;
  if (n_split) *n_split = ns;
  if (counts)
    for (int a = 0; a < 3; ++a) counts[a] = p->counts[a];
  *plan = p;
  return SCT_OK;
}

int sct_adaptive_apply(sct_ctx* c, sct_ac_plan* p, const sct_cloud* cloud, const sct_adam_state* adam,
                       const float* grad3d_accum, const double* gauss, sct_cloud* out, sct_adam_state* out_adam) {
  if (!c || !p || !cloud || !adam || !out || !out_adam || !grad3d_accum) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  if (p->n_split > 0 && !gauss) {
    set_error("ConfigError: adaptive control: split kernels need 6 normal draws each");
    return SCT_ERR_CONFIG;
  }
  if (p->m > 0) {
    KScope _ks(c, "AC_apply");
    ac_apply_kernel<<<grid_cap(c, p->m, 256), 256, 0, c->stream>>>(
        p->m, p->m_kept, *cloud, *adam, grad3d_accum, p->action, p->keep_out, p->keep_pos, p->new_pos,
        p->split_ord, gauss, p->P, *out, *out_adam);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_adaptive_free(sct_ac_plan* p) {
  if (!p) return SCT_OK;
  ac_release(p);
  delete p;
  return SCT_OK;
}

}  // extern "C"
