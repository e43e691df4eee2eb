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
//
// Along x the exponential uses the same 4-voxel ratio recurrence as the
// rasterizer (raster.cu, run4): with A = Qxx*sx^2 (log2 units per voxel^2) the
// ratio between neighbouring voxels changes by K = 2^(2A). Unlike the
// rasterizer there is no 0.3 px low-pass floor, so a kernel can be far
// narrower than a voxel; the recurrence is used only when A >= -8 (then, as in
// DESIGN.md §K3, a run can only lose values below 2^-29 of rho) and narrow
// kernels take the direct one-MUFU-per-voxel path. The branch is uniform
// across the CTA (all lanes evaluate the same kernel at the same time).
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
  long long n_bricks;  // bricks in the slab
};

__device__ __forceinline__ void brick_of(const BrickGeo& G, long long b, int& tx, int& ty, int& tz) {
  tx = (int)(b % G.bx);
  const long long r = b / G.bx;
  ty = (int)(r % G.by);
  tz = G.zb0 + (int)(r / G.by);
}

// 8 voxel values along x for one row: E'(c) = 2^(L(dx0 + c*sx) + 64), c = 0..7.
// rec_ok: use two 4-voxel ratio runs; otherwise one MUFU per voxel.
__device__ __forceinline__ void row8(float e[8], bool rec_ok, float dx0, float sx, float qxx, float c1, float c0o,
                                     float K) {
  if (rec_ok) {
    const float qs = qxx * sx;
    const float dbase = fmaf(c1, sx, qs * sx);  // D(dx) = 2 qxx sx dx + c1 sx + qxx sx^2
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float dx = fmaf(4.f * h, sx, dx0);
      const float t = fmaf(qxx, dx, c1);
      float E = ex2v(fmaf(dx, t, c0o));
      float R = ex2v(fminf(fmaf(2.f * qs, dx, dbase), 126.f));
      e[4 * h] = E;
      E *= R;
      R *= K;
      e[4 * h + 1] = E;
      E *= R;
      R *= K;
      e[4 * h + 2] = E;
      e[4 * h + 3] = E * R;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float dx = fmaf((float)c, sx, dx0);
      e[c] = ex2v(fmaf(dx, fmaf(qxx, dx, c1), c0o));
    }
  }
}

// K7: one warp per brick, four bricks per CTA; lane = rows (y, z) and (y, z+4),
// 8 voxels each. Each warp stages its brick list 32 records at a time through
// its own shared memory, prefetching the next chunk into registers.
constexpr int kEvalWarps = 4;
__global__ void __launch_bounds__(32 * kEvalWarps) voxel_eval_kernel(BrickGeo G, const int2* __restrict__ ranges,
                                                                     const int32_t* __restrict__ vals,
                                                                     const float4* __restrict__ rec,
                                                                     float* __restrict__ vol) {
  __shared__ float4 sA[kEvalWarps][32];  // base offset xyz, rho*2^-64
  __shared__ float4 sB[kEvalWarps][32];  // Qxx Qyy Qzz K
  __shared__ float4 sC[kEvalWarps][32];  // Qxy Qxz Qyz
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long b = (long long)blockIdx.x * kEvalWarps + warp;
  if (b >= G.n_bricks) return;
  int tx, ty, tz;
  brick_of(G, b, tx, ty, tz);
  const int brick = (tz * G.by + ty) * G.bx + tx;
  const int2 rg = ranges[brick];
  const double c0x = G.origin.x + ((double)(tx * kTileVox) + 0.5) * G.spacing.x;
  const double c0y = G.origin.y + ((double)(ty * kTileVox) + 0.5) * G.spacing.y;
  const double c0z = G.origin.z + ((double)(tz * kTileVox) + 0.5) * G.spacing.z;
  const int ly = lane & 7, lz = lane >> 3;  // rows (ly, lz) and (ly, lz + 4)
  const float fy = (float)ly * G.spf.y;
  const float fz0 = (float)lz * G.spf.z, fz1 = (float)(lz + 4) * G.spf.z;
  float acc[2][8];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
  float4 na = make_float4(0.f, 0.f, 0.f, 0.f), nb = na, nc = na;
  auto fetch = [&](int p) {
    const long long i = vals[p];
    const float4 a = __ldg(rec + 3 * i);
    na = make_float4((float)(c0x - (double)a.x), (float)(c0y - (double)a.y), (float)(c0z - (double)a.z),
                     a.w * 0x1p-64f);
    nb = __ldg(rec + 3 * i + 1);
    nc = __ldg(rec + 3 * i + 2);
  };
  if (rg.x + lane < rg.y) fetch(rg.x + lane);
  for (int base = rg.x; base < rg.y; base += 32) {
    const int n = min(32, rg.y - base);
    __syncwarp();
    sA[warp][lane] = na;
    sB[warp][lane] = nb;
    sC[warp][lane] = nc;
    __syncwarp();
    if (base + 32 + lane < rg.y) fetch(base + 32 + lane);
    for (int j = 0; j < n; ++j) {
      const float4 a = sA[warp][j];
      const float4 q = sB[warp][j];
      const float4 o = sC[warp][j];
      const bool rec_ok = q.x * G.spf.x * G.spf.x >= -8.f;
      const float dy = a.y + fy;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float dz = a.z + (r ? fz1 : fz0);
        const float c0o = fmaf(q.y * dy, dy, fmaf(q.z * dz, dz, fmaf(o.z * dy, dz, 64.f)));
        const float c1 = fmaf(o.x, dy, o.y * dz);
        float e[8];
        row8(e, rec_ok, a.x, G.spf.x, q.x, c1, c0o, q.w);
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a.w, e[c], acc[r][c]);
      }
    }
  }
  const int y = ty * kTileVox + ly, x0 = tx * kTileVox;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int z = tz * kTileVox + lz + 4 * r;
    if (y >= G.dims.y || z >= G.dims.z) continue;
    float* out = vol + ((long long)z * G.dims.y + y) * G.dims.x + x0;
    if (x0 + 7 < G.dims.x && (G.dims.x & 3) == 0) {
      reinterpret_cast<float4*>(out)[0] = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      reinterpret_cast<float4*>(out)[1] = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (x0 + c < G.dims.x) out[c] = acc[r][c];
    }
  }
}

// K8: Gaussian-major backward statistics; 16 lanes per kernel, lane = four
// (y,z) rows of 8 voxels with the upstream gradient in registers (pre-scaled
// by 2^-64). Per row: the x-moments R0 = sum F, R1 = sum c' F, R2 = sum c'^2 F
// (F = g E, c' = x - 3.5, columns paired c <-> 7-c) give the row's share of
// the 10 statistics; the 16 lanes' partials are combined by a 4-step shuffle
// reduce-scatter and lanes 0..9 store the pair's 10 values.
constexpr int kVBwdThreads = 256;
__global__ void __launch_bounds__(kVBwdThreads, 3) voxel_backward_stats_kernel(
    BrickGeo G, const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    const short4* __restrict__ lo, const short4* __restrict__ hi, const int32_t* __restrict__ offset,
    const float* __restrict__ dL, float* __restrict__ pair_stats) {
  int tx, ty, tz;
  brick_of(G, blockIdx.x, tx, ty, tz);
  const int brick = (tz * G.by + ty) * G.bx + tx;
  const int2 rg = ranges[brick];
  if (rg.y <= rg.x) return;
  const double c0x = G.origin.x + ((double)(tx * kTileVox) + 0.5) * G.spacing.x;
  const double c0y = G.origin.y + ((double)(ty * kTileVox) + 0.5) * G.spacing.y;
  const double c0z = G.origin.z + ((double)(tz * kTileVox) + 0.5) * G.spacing.z;
  const int s = threadIdx.x & 15;
  const int group = threadIdx.x >> 4;
  const int ly = s & 7;
  const int lz0 = s >> 3;  // rows z = lz0 + 2*j, j = 0..3
  const int y = ty * kTileVox + ly;
  const int x0 = tx * kTileVox;
  float g[4][kTileVox];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int z = tz * kTileVox + lz0 + 2 * j;
    const bool rowok = y < G.dims.y && z < G.dims.z;
    const float* src = dL + ((long long)z * G.dims.y + y) * G.dims.x + x0;
#pragma unroll
    for (int c = 0; c < kTileVox; ++c)
      g[j][c] = (rowok && x0 + c < G.dims.x) ? __ldg(src + c) * 0x1p-64f : 0.f;
  }
  const float fy = (float)ly * G.spf.y;
  const float sx = G.spf.x;
  for (int base = rg.x; base < rg.y; base += kVBwdThreads / 16) {
    const int jj = base + group;
    const bool valid = jj < rg.y;
    float v[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) v[a] = 0.f;
    long long i = 0;
    if (valid) {
      i = vals[jj];
      const float4 a = __ldg(rec + 3 * i);
      const float4 q = __ldg(rec + 3 * i + 1);
      const float4 o = __ldg(rec + 3 * i + 2);
      const bool rec_ok = q.x * sx * sx >= -8.f;
      const float bx = (float)(c0x - (double)a.x);
      const float dy = (float)(c0y - (double)a.y) + fy;
      const float bz = (float)(c0z - (double)a.z);
      const float dxm = fmaf(3.5f, sx, bx);  // x offset of the row centre
      const float qyy_dy2 = fmaf(q.y * dy, dy, 64.f);
      const float oxy_dy = o.x * dy;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float dz = fmaf((float)(lz0 + 2 * j), G.spf.z, bz);
        const float c0o = fmaf(q.z * dz, dz, fmaf(o.z * dy, dz, qyy_dy2));
        const float c1 = fmaf(o.y, dz, oxy_dy);
        float e[8];
        row8(e, rec_ok, bx, sx, q.x, c1, c0o, q.w);
        float R0 = 0.f, R1 = 0.f, R2 = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float cp = (float)c - 3.5f;
          const float fa = g[j][c] * e[c];
          const float fb = g[j][7 - c] * e[7 - c];
          const float sm = fa + fb;
          R0 += sm;
          R1 = fmaf(fa - fb, cp, R1);
          R2 = fmaf(sm, cp * cp, R2);
        }
        // sum F dx = dxm R0 + sx R1; sum F dx^2 = dxm^2 R0 + 2 dxm sx R1 + sx^2 R2
        const float R1s = sx * R1;
        const float rx = fmaf(dxm, R0, R1s);
        const float rxx = fmaf(dxm, fmaf(dxm, R0, 2.f * R1s), sx * sx * R2);
        v[0] += R0;                      // s0
        v[1] += rx;                      // s1.x
        v[2] = fmaf(dy, R0, v[2]);       // s1.y
        v[3] = fmaf(dz, R0, v[3]);       // s1.z
        v[4] += rxx;                     // s2.xx
        v[5] = fmaf(dy * dy, R0, v[5]);  // s2.yy
        v[6] = fmaf(dz * dz, R0, v[6]);  // s2.zz
        v[7] = fmaf(dy, rx, v[7]);       // s2.xy
        v[8] = fmaf(dz, rx, v[8]);       // s2.xz
        v[9] = fmaf(dy * dz, R0, v[9]);  // s2.yz
      }
    }
    // reduce-scatter over the 16 lanes of the group: lane s ends with total[s]
#pragma unroll
    for (int off = 8, width = 16; off >= 1; off >>= 1, width >>= 1) {
      const bool up = s & off;
#pragma unroll
      for (int k = 0; k < width / 2; ++k) {
        const float send = up ? v[k] : v[k + width / 2];
        const float keep = up ? v[k + width / 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    if (valid && s < 10) {
      const short4 l = lo[i], h = hi[i];
      const int nx = h.x - l.x + 1, ny = h.y - l.y + 1;
      const long long slot = offset[i] + ((tz - l.z) * ny + (ty - l.y)) * nx + (tx - l.x);
      pair_stats[12 * slot + s] = v[0];
    }
  }
}

BrickGeo make_geo(const sct_grid& g, int zb0, int zb1, int bx, int by) {
  BrickGeo G;
  G.dims = make_int3(g.dims[0], g.dims[1], g.dims[2]);
  G.origin = make_double3(g.origin_mm[0], g.origin_mm[1], g.origin_mm[2]);
  G.spacing = make_double3(g.spacing_mm[0], g.spacing_mm[1], g.spacing_mm[2]);
  G.spf = make_float3((float)g.spacing_mm[0], (float)g.spacing_mm[1], (float)g.spacing_mm[2]);
  G.bx = bx;
  G.by = by;
  G.zb0 = zb0;
  G.n_bricks = (long long)bx * by * (zb1 - zb0);
  return G;
}

}  // namespace

void launch_voxel_emit(Ctx* c, int64_t m, const short4* lo, const short4* hi, const int32_t* offset,
                       int32_t bricks_x, int32_t bricks_y, uint32_t* keys, int32_t* vals) {
  if (m == 0) return;
  long long b = (m + 255) / 256;
  if (b > (long long)c->sm_count * 16) b = (long long)c->sm_count * 16;
  KScope _ks(c, "K6_voxel_emit");
  voxel_emit_kernel<<<(int)b, 256, 0, c->stream>>>(m, lo, hi, offset, bricks_x, bricks_y, keys, vals);
}

void launch_voxel_eval(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x, int32_t bricks_y,
                       const int2* ranges, const int32_t* vals, const float4* rec, const sct_cloud&, float* vol) {
  const long long nb = (long long)bricks_x * bricks_y * (zb1 - zb0);
  if (nb <= 0) return;
  KScope _ks(c, "K7_voxel_eval");
  voxel_eval_kernel<<<(unsigned)((nb + kEvalWarps - 1) / kEvalWarps), 32 * kEvalWarps, 0, c->stream>>>(
      make_geo(g, zb0, zb1, bricks_x, bricks_y), ranges, vals, rec, vol);
}

void launch_voxel_backward_stats(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x,
                                 int32_t bricks_y, const int2* ranges, const int32_t* vals, const float4* rec,
                                 const short4* lo, const short4* hi, const int32_t* offset, const sct_cloud&,
                                 const float* dL, float4* pair_stats) {
  const long long nb = (long long)bricks_x * bricks_y * (zb1 - zb0);
  if (nb <= 0) return;
  KScope _ks(c, "K8_voxel_backward_stats");
  voxel_backward_stats_kernel<<<(unsigned)nb, kVBwdThreads, 0, c->stream>>>(
      make_geo(g, zb0, zb1, bricks_x, bricks_y), ranges, vals, rec, lo, hi, offset, dL,
      reinterpret_cast<float*>(pair_stats));
}

}  // namespace sct
