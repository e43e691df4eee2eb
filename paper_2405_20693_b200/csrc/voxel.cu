// Voxelizer FP32 hot kernels (sm_100a).
//
//   K6 voxel_emit   — brick keys for every covered 8^3 brick, Gaussian-major
//                     (voxelizer.cpp:82-85; brick id (tz*By+ty)*Bx+tx, :45-47)
//   K7 voxel_eval   — V(x,y,z) = sum_list rho * exp(-1/2 d^T Q d) at voxel
//                     centres (voxelizer.cpp:115-136)
//   K8 voxel stats  — per (brick, kernel) s0, s1 (3), s2 (6)
//                     (voxelizer.cpp:158-190)
//
// Voxel offsets are formed as (brick's first voxel centre - kernel position)
// in FP64 once per (brick, kernel) pair, then stepped in FP32 by the spacing,
// so the FP32 distance error stays at the level of one rounding of d.
#include <cuda_runtime.h>

#include "sct_internal.cuh"

namespace sct {

__device__ __forceinline__ float ex2v(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

namespace {

__global__ void __launch_bounds__(256) voxel_emit_kernel(long long m, const short4* __restrict__ lo,
                                                         const short4* __restrict__ hi,
                                                         const int32_t* __restrict__ offset, int bx, int by,
                                                         uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    int32_t o = offset[i];
    if (offset[i + 1] == o) continue;
    const short4 a = lo[i], b = hi[i];
    for (int tz = a.z; tz <= b.z; ++tz)
      for (int ty = a.y; ty <= b.y; ++ty)
        for (int tx = a.x; tx <= b.x; ++tx) {
          keys[o] = (uint32_t)((tz * by + ty) * bx + tx);
          vals[o] = (int32_t)i;
          ++o;
        }
  }
}

struct BrickGeo {
  int3 dims;
  double3 origin;
  double3 spacing;
  float3 spf;
  int bx, by, zb0;
};

__device__ __forceinline__ void brick_of(const BrickGeo& G, int b, int& tx, int& ty, int& tz) {
  tx = b % G.bx;
  const int r = b / G.bx;
  ty = r % G.by;
  tz = G.zb0 + r / G.by;
}

// K7: one 128-thread CTA per brick of the slab; thread = one (y,z) row, 4 x-voxels.
constexpr int kEvalThreads = 128;
__global__ void __launch_bounds__(kEvalThreads) voxel_eval_kernel(BrickGeo G, const int2* __restrict__ ranges,
                                                                  const int32_t* __restrict__ vals,
                                                                  const float4* __restrict__ rec,
                                                                  float* __restrict__ vol) {
  __shared__ float4 sA[kEvalThreads];  // base offset xyz, rho
  __shared__ float4 sB[kEvalThreads];  // Qxx Qyy Qzz
  __shared__ float4 sC[kEvalThreads];  // Qxy Qxz Qyz
  int tx, ty, tz;
  brick_of(G, blockIdx.x, tx, ty, tz);
  const int brick = (tz * G.by + ty) * G.bx + tx;
  const int2 rg = ranges[brick];
  const double c0x = G.origin.x + ((double)(tx * kTileVox) + 0.5) * G.spacing.x;
  const double c0y = G.origin.y + ((double)(ty * kTileVox) + 0.5) * G.spacing.y;
  const double c0z = G.origin.z + ((double)(tz * kTileVox) + 0.5) * G.spacing.z;
  const int row = threadIdx.x >> 1;
  const int ly = row & 7, lz = row >> 3;
  const int lx0 = (threadIdx.x & 1) * 4;
  const float fy = (float)ly * G.spf.y, fz = (float)lz * G.spf.z;
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  for (int base = rg.x; base < rg.y; base += kEvalThreads) {
    const int n = min(kEvalThreads, rg.y - base);
    __syncthreads();
    if ((int)threadIdx.x < n) {
      const long long i = vals[base + threadIdx.x];
      const float4 a = rec[3 * i];
      sA[threadIdx.x] = make_float4((float)(c0x - (double)a.x), (float)(c0y - (double)a.y),
                                    (float)(c0z - (double)a.z), a.w);
      sB[threadIdx.x] = rec[3 * i + 1];
      sC[threadIdx.x] = rec[3 * i + 2];
    }
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < n; ++j) {
      const float4 a = sA[j];
      const float4 q = sB[j];
      const float4 o = sC[j];
      const float dy = a.y + fy;
      const float dz = a.z + fz;
      const float c0 = fmaf(q.y * dy, dy, fmaf(q.z * dz, dz, o.z * dy * dz));
      const float c1 = fmaf(o.x, dy, o.y * dz);
      float dx, t;
      dx = fmaf((float)(lx0 + 0), G.spf.x, a.x); t = fmaf(q.x, dx, c1); acc0 = fmaf(a.w, ex2v(fmaf(dx, t, c0)), acc0);
      dx = fmaf((float)(lx0 + 1), G.spf.x, a.x); t = fmaf(q.x, dx, c1); acc1 = fmaf(a.w, ex2v(fmaf(dx, t, c0)), acc1);
      dx = fmaf((float)(lx0 + 2), G.spf.x, a.x); t = fmaf(q.x, dx, c1); acc2 = fmaf(a.w, ex2v(fmaf(dx, t, c0)), acc2);
      dx = fmaf((float)(lx0 + 3), G.spf.x, a.x); t = fmaf(q.x, dx, c1); acc3 = fmaf(a.w, ex2v(fmaf(dx, t, c0)), acc3);
    }
  }
  const int y = ty * kTileVox + ly, z = tz * kTileVox + lz, x0 = tx * kTileVox + lx0;
  if (y < G.dims.y && z < G.dims.z) {
    float* out = vol + ((long long)z * G.dims.y + y) * G.dims.x;
    if (x0 + 3 < G.dims.x && (G.dims.x & 3) == 0) {
      *reinterpret_cast<float4*>(out + x0) = make_float4(acc0, acc1, acc2, acc3);
    } else {
      if (x0 < G.dims.x) out[x0] = acc0;
      if (x0 + 1 < G.dims.x) out[x0 + 1] = acc1;
      if (x0 + 2 < G.dims.x) out[x0 + 2] = acc2;
      if (x0 + 3 < G.dims.x) out[x0 + 3] = acc3;
    }
  }
}

// K8: Gaussian-major backward statistics; 16 lanes per kernel, each lane four
// (y,z) rows of 8 voxels with the upstream gradient held in registers.
constexpr int kVBwdThreads = 256;
__global__ void __launch_bounds__(kVBwdThreads) voxel_backward_stats_kernel(
    BrickGeo G, const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    const short4* __restrict__ lo, const short4* __restrict__ hi, const int32_t* __restrict__ offset,
    const float* __restrict__ dL, float4* __restrict__ pair_stats) {
  int tx, ty, tz;
  brick_of(G, blockIdx.x, tx, ty, tz);
  const int brick = (tz * G.by + ty) * G.bx + tx;
  const int2 rg = ranges[brick];
  if (rg.y <= rg.x) return;
  const double c0x = G.origin.x + ((double)(tx * kTileVox) + 0.5) * G.spacing.x;
  const double c0y = G.origin.y + ((double)(ty * kTileVox) + 0.5) * G.spacing.y;
  const double c0z = G.origin.z + ((double)(tz * kTileVox) + 0.5) * G.spacing.z;
  const int lane16 = threadIdx.x & 15;
  const int group = threadIdx.x >> 4;
  const int ly = lane16 & 7;
  const int lz0 = lane16 >> 3;  // rows z = lz0 + 2*j, j = 0..3
  const int y = ty * kTileVox + ly;
  const int x0 = tx * kTileVox;
  float g[4][kTileVox];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int z = tz * kTileVox + lz0 + 2 * j;
    const bool rowok = y < G.dims.y && z < G.dims.z;
    const float* src = dL + ((long long)z * G.dims.y + y) * G.dims.x + x0;
#pragma unroll
    for (int c = 0; c < kTileVox; ++c) g[j][c] = (rowok && x0 + c < G.dims.x) ? __ldg(src + c) : 0.f;
  }
  const float fy = (float)ly * G.spf.y;
  for (int base = rg.x; base < rg.y; base += 16) {
    const int jj = base + group;
    const bool valid = jj < rg.y;
    float s[10];
#pragma unroll
    for (int a = 0; a < 10; ++a) s[a] = 0.f;
    long long i = 0;
    if (valid) {
      i = vals[jj];
      const float4 a = __ldg(rec + 3 * i);
      const float4 q = __ldg(rec + 3 * i + 1);
      const float4 o = __ldg(rec + 3 * i + 2);
      const float bx = (float)(c0x - (double)a.x);
      const float dy = (float)(c0y - (double)a.y) + fy;
      const float bz = (float)(c0z - (double)a.z);
      const float qyy_dy2 = q.y * dy * dy;
      const float oxy_dy = o.x * dy;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float dz = fmaf((float)(lz0 + 2 * j), G.spf.z, bz);
        const float c0 = fmaf(q.z * dz, dz, fmaf(o.z * dy, dz, qyy_dy2));
        const float c1 = fmaf(o.y, dz, oxy_dy);
        float r0 = 0.f, rx = 0.f, rxx = 0.f;
#pragma unroll
        for (int c = 0; c < kTileVox; ++c) {
          const float dx = fmaf((float)c, G.spf.x, bx);
          const float t = fmaf(q.x, dx, c1);
          const float ge = g[j][c] * ex2v(fmaf(dx, t, c0));
          r0 += ge;
          const float gx = ge * dx;
          rx += gx;
          rxx = fmaf(gx, dx, rxx);
        }
        s[0] += r0;            // s0
        s[1] += rx;            // s1.x
        s[2] += dy * r0;       // s1.y
        s[3] += dz * r0;       // s1.z
        s[4] += rxx;           // s2.xx
        s[5] += dy * dy * r0;  // s2.yy
        s[6] += dz * dz * r0;  // s2.zz
        s[7] += dy * rx;       // s2.xy
        s[8] += dz * rx;       // s2.xz
        s[9] += dy * dz * r0;  // s2.yz
      }
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1)
#pragma unroll
      for (int a = 0; a < 10; ++a) s[a] += __shfl_xor_sync(0xffffffffu, s[a], off);
    if (valid && lane16 == 0) {
      const short4 l = lo[i], h = hi[i];
      const int nx = h.x - l.x + 1, ny = h.y - l.y + 1;
      const long long slot = offset[i] + ((tz - l.z) * ny + (ty - l.y)) * nx + (tx - l.x);
      pair_stats[3 * slot + 0] = make_float4(s[0], s[1], s[2], s[3]);
      pair_stats[3 * slot + 1] = make_float4(s[4], s[5], s[6], s[7]);
      pair_stats[3 * slot + 2] = make_float4(s[8], s[9], 0.f, 0.f);
    }
  }
}

BrickGeo make_geo(const sct_grid& g, int zb0, int bx, int by) {
  BrickGeo G;
  G.dims = make_int3(g.dims[0], g.dims[1], g.dims[2]);
  G.origin = make_double3(g.origin_mm[0], g.origin_mm[1], g.origin_mm[2]);
  G.spacing = make_double3(g.spacing_mm[0], g.spacing_mm[1], g.spacing_mm[2]);
  G.spf = make_float3((float)g.spacing_mm[0], (float)g.spacing_mm[1], (float)g.spacing_mm[2]);
  G.bx = bx;
  G.by = by;
  G.zb0 = zb0;
  return G;
}

}  // namespace

void launch_voxel_emit(Ctx* c, int64_t m, const short4* lo, const short4* hi, const int32_t* offset,
                       int32_t bricks_x, int32_t bricks_y, uint32_t* keys, int32_t* vals) {
  if (m == 0) return;
  long long b = (m + 255) / 256;
  if (b > (long long)c->sm_count * 16) b = (long long)c->sm_count * 16;
  {
    KScope _ks(c, "K6_voxel_emit");
    voxel_emit_kernel<<<(int)b, 256, 0, c->stream>>>(m, lo, hi, offset, bricks_x, bricks_y, keys, vals);
  }
}

void launch_voxel_eval(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x, int32_t bricks_y,
                       const int2* ranges, const int32_t* vals, const float4* rec, const sct_cloud&, float* vol) {
  const long long nb = (long long)bricks_x * bricks_y * (zb1 - zb0);
  if (nb <= 0) return;
  {
    KScope _ks(c, "K7_voxel_eval");
    voxel_eval_kernel<<<(unsigned)nb, kEvalThreads, 0, c->stream>>>(make_geo(g, zb0, bricks_x, bricks_y), ranges,
                                                                     vals, rec, vol);
  }
}

void launch_voxel_backward_stats(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x,
                                 int32_t bricks_y, const int2* ranges, const int32_t* vals, const float4* rec,
                                 const short4* lo, const short4* hi, const int32_t* offset, const sct_cloud&,
                                 const float* dL, float4* pair_stats) {
  const long long nb = (long long)bricks_x * bricks_y * (zb1 - zb0);
  if (nb <= 0) return;
  {
    KScope _ks(c, "K8_voxel_backward_stats");
    voxel_backward_stats_kernel<<<(unsigned)nb, kVBwdThreads, 0, c->stream>>>(
        make_geo(g, zb0, bricks_x, bricks_y), ranges, vals, rec, lo, hi, offset, dL, pair_stats);
  }
}

}  // namespace sct
