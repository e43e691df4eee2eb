// Layout probe for the tcgen05 primitives in csrc/tcgen05.cuh (diagnostic
// tool, not product): one CTA computes D[128][16] = A[128][256] . B[16][256]^T
// with A written to TMEM by the SIMT lanes (row i = TMEM lane i, k pairs
// packed per 32-bit column), B in shared memory in the canonical K-major
// no-swizzle layout, 16 MMAs of K = 16, and compares against the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2405_20693_b200/csrc tools/tc_probe.cu -o tc_probe
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tcgen05.cuh"

using namespace sct;

__global__ void probe(const __half* A, const __half* B, float* D, uint32_t lbo, uint32_t sbo, int swap_half) {
  __shared__ __align__(1024) __half sB[16 * 256];
  __shared__ uint32_t s_taddr;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  // B[n][k] -> ((k / 8) * 2 + n / 8) * 128 B + (n % 8) * 16 B + (k % 8) * 2 B
  for (int e = tid; e < 16 * 256; e += blockDim.x) {
    const int n = e / 256, k = e % 256;
    const int off = (((k >> 3) * 2 + (n >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2) / 2;
    sB[off] = B[e];
  }
  if (warp == 0) {
    tc::tmem_alloc(&s_taddr, 256);
    tc::tmem_relinquish();
  }
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init_fence();
  }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = s_taddr;
  const uint32_t lane_base = base + ((uint32_t)(32 * warp) << 16);
  // row tid of A -> TMEM lane tid, columns [0, 128)
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) {
      const int k = 2 * (c0 + j);
      __half lo = A[tid * 256 + k], hi = A[tid * 256 + k + 1];
      if (swap_half) { __half t = lo; lo = hi; hi = t; }
      v[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    tc::tmem_st16(lane_base + c0, v);
  }
  tc::tmem_wait_st();
  tc::fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    tc::fence_after_sync();
    const uint32_t idesc = tc::idesc_f16_f32(128, 16);
    for (int j = 0; j < 16; ++j) {
      const uint64_t bd = tc::smem_desc_kmajor(reinterpret_cast<const char*>(sB) + 512 * j, lbo, sbo);
      tc::mma_f16_ts(base + 128, base + 8 * j, bd, idesc, j > 0);
    }
    tc::commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  uint32_t d[16];
  tc::tmem_ld16(lane_base + 128, d);
  tc::tmem_wait_ld();
  for (int n = 0; n < 16; ++n) D[tid * 16 + n] = __uint_as_float(d[n]);
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 256);
}

int main() {
  std::vector<__half> A(128 * 256), B(16 * 256);
  std::vector<float> Af(A.size()), Bf(B.size());
  srand(1);
  for (size_t i = 0; i < A.size(); ++i) { A[i] = __float2half((rand() % 17 - 8) / 8.f); Af[i] = __half2float(A[i]); }
  for (size_t i = 0; i < B.size(); ++i) { B[i] = __float2half((rand() % 17 - 8) / 4.f); Bf[i] = __half2float(B[i]); }
  std::vector<double> ref(128 * 16, 0.0);
  for (int i = 0; i < 128; ++i)
    for (int n = 0; n < 16; ++n)
      for (int k = 0; k < 256; ++k) ref[i * 16 + n] += (double)Af[i * 256 + k] * Bf[n * 256 + k];
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, 128 * 16 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  struct V { uint32_t lbo, sbo; int swap; } vs[] = {{256, 128, 0}, {128, 256, 0}, {256, 128, 1}, {128, 256, 1}};
  int best = -1;
  for (int t = 0; t < 4; ++t) {
    cudaMemset(dD, 0, 128 * 16 * 4);
    probe<<<1, 128>>>(dA, dB, dD, vs[t].lbo, vs[t].sbo, vs[t].swap);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(128 * 16);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0.0, mx = 0.0;
    for (size_t i = 0; i < D.size(); ++i) { err = fmax(err, fabs(D[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); }
    printf("variant lbo=%u sbo=%u swap=%d: %s max abs err %.3g (max |ref| %.3g) D[0][0..3]=%g %g %g %g ref %g %g %g %g\n",
           vs[t].lbo, vs[t].sbo, vs[t].swap, cudaGetErrorString(e), err, mx, D[0], D[1], D[2], D[3], ref[0], ref[1],
           ref[2], ref[3]);
    if (e != cudaSuccess) return 1;
    if (err < 1e-3 && best < 0) best = t;
  }
  printf("PROBE %s (variant %d)\n", best >= 0 ? "OK" : "FAILED", best);
  return best == 0 ? 0 : 2;
}
