// Adam update of one kernel's 11 parameters + quaternion renormalisation
// (trainer.cpp:144-163,310-319, gaussian_cloud.cpp:112-117), shared by the Adam
// kernel (optim.cu) and the native train step's fused finalize + Adam
// (chain.cu). Every operation is an explicit round-to-nearest intrinsic, so the
// two kernels (and translation units) produce bitwise the same parameters.
#pragma once
#include <cuda_runtime.h>

#include "splatct_gpu.h"

namespace sct {

__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, float lr, float bc1, float bc2,
                                      float b1, float b2, float eps) {
  m = __fmaf_rn(b1, m, __fmul_rn(1.f - b1, g));
  v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(1.f - b2, g), g));
  const float mhat = __fdiv_rn(m, bc1);
  const float vhat = __fdiv_rn(v, bc2);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(lr, mhat), __fadd_rn(__fsqrt_rn(vhat), eps)));
}

struct AdamParams {
  float lr_pos, lr_rho, lr_sc, lr_rot, bc1, bc2, b1, b2, eps;
};

// kernel i with gradients g = {rho, pos[3], scale[3], rot[4]}
__device__ __forceinline__ void adam_kernel_update(long long i, float* __restrict__ rho, float* __restrict__ pos,
                                                   float* __restrict__ sc, float* __restrict__ rot,
                                                   const sct_adam_state& st, const float g[11], const AdamParams& a) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const long long j = 3 * i + k;
    float p = pos[j], mm = st.m_pos[j], vv = st.v_pos[j];
    adam1(p, mm, vv, g[1 + k], a.lr_pos, a.bc1, a.bc2, a.b1, a.b2, a.eps);
    pos[j] = p;
    st.m_pos[j] = mm;
    st.v_pos[j] = vv;
  }
  {
    float p = rho[i], mm = st.m_rho[i], vv = st.v_rho[i];
    adam1(p, mm, vv, g[0], a.lr_rho, a.bc1, a.bc2, a.b1, a.b2, a.eps);
    rho[i] = p;
    st.m_rho[i] = mm;
    st.v_rho[i] = vv;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const long long j = 3 * i + k;
    float p = sc[j], mm = st.m_scale[j], vv = st.v_scale[j];
    adam1(p, mm, vv, g[4 + k], a.lr_sc, a.bc1, a.bc2, a.b1, a.b2, a.eps);
    sc[j] = p;
    st.m_scale[j] = mm;
    st.v_scale[j] = vv;
  }
  float q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long j = 4 * i + k;
    float p = rot[j], mm = st.m_rot[j], vv = st.v_rot[j];
    adam1(p, mm, vv, g[7 + k], a.lr_rot, a.bc1, a.bc2, a.b1, a.b2, a.eps);
    q[k] = p;
    st.m_rot[j] = mm;
    st.v_rot[j] = vv;
  }
  const float n = __fsqrt_rn(__fmaf_rn(q[3], q[3], __fmaf_rn(q[2], q[2], __fmaf_rn(q[1], q[1], __fmul_rn(q[0], q[0])))));
#pragma unroll
  for (int k = 0; k < 4; ++k) rot[4 * i + k] = __fdiv_rn(q[k], n);
}

// total = (l1 + lambda_ssim dssim) + lambda_tv tv with separately rounded
// products, as the host-side composition (trainer.cpp:302-303)
__device__ __forceinline__ void train_total(double* total, double lambda_ssim, double lambda_tv) {
  total[3] = __dadd_rn(__dadd_rn(total[0], __dmul_rn(lambda_ssim, total[1])), __dmul_rn(lambda_tv, total[2]));
}

}  // namespace sct
