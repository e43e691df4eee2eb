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
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <type_traits>

#include <cstdlib>
#include <string>

#include "sct_internal.cuh"

namespace sct {

__device__ __forceinline__ float ex2v(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

namespace {

// Warp-cooperative emission (as raster_emit): a warp owns 32 consecutive
// kernels, whose pairs form one contiguous output range; lanes stride over it
// (coalesced stores) and find their kernel by a 5-step binary search over the
// 32 offsets held in the lanes. Bricks of a kernel in z, y, x order
// (voxelizer.cpp:82-85), i.e. ascending brick id; 16-bit keys when they fit.
template <typename KeyT>
__global__ void __launch_bounds__(256) voxel_emit_kernel(long long m, const short4* __restrict__ lo,
                                                         const short4* __restrict__ hi,
                                                         const int32_t* __restrict__ offset, int bx, int by,
                                                         KeyT* __restrict__ keys, int32_t* __restrict__ vals,
                                                         long long cap) {
  pdl_prologue();
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w0 = (blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < m;
       w0 += warps * 32) {
    const long long it = w0 + lane;
    const int32_t o_l = it < m ? offset[it] : offset[m];
    const long long last = min(w0 + 32, m);
    const int32_t o_end = offset[last];
    short4 a = make_short4(0, 0, 0, 0), b = make_short4(-1, -1, -1, -1);
    if (it < m) {
      a = lo[it];
      b = hi[it];
    }
    const int axy = ((int)(unsigned short)a.x) | ((int)a.y << 16);
    const int nxy = ((b.x - a.x + 1) & 0xffff) | ((b.y - a.y + 1) << 16);
    const int az = a.z;
    const int32_t o_0 = __shfl_sync(0xffffffffu, o_l, 0);
    for (int32_t p0 = o_0; p0 < o_end; p0 += 32) {
      const int32_t p = p0 + lane;
      int j = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int32_t oj = __shfl_sync(0xffffffffu, o_l, j + step);
        if (j + step < 32 && oj <= p) j += step;
      }
      const int32_t oj = __shfl_sync(0xffffffffu, o_l, j);
      const int jxy = __shfl_sync(0xffffffffu, axy, j);
      const int jn = __shfl_sync(0xffffffffu, nxy, j);
      const int jz = __shfl_sync(0xffffffffu, az, j);
      if (p < o_end && p < cap) {  // cap: capacity-mode buffers (the overflow is flagged by the count check)
        const int x0 = (short)(jxy & 0xffff), y0 = (short)(jxy >> 16);
        const int nx = jn & 0xffff, ny = jn >> 16;
        const int rank = p - oj;
        const int tx = x0 + rank % nx;
        const int r2 = rank / nx;
        const int ty = y0 + r2 % ny, tz = jz + r2 / ny;
        keys[p] = (KeyT)((tz * by + ty) * bx + tx);
        vals[p] = (int32_t)(w0 + j);
      }
    }
  }
}

// [start, end) of each key's run in the sorted pairs (key = slot)
template <typename KeyT>
__global__ void __launch_bounds__(256) key_ranges_kernel(long long n_pairs, const KeyT* __restrict__ keys,
                                                         int2* __restrict__ ranges, long long n_keys) {
  pdl_prologue();
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n_pairs;
       p += (long long)gridDim.x * blockDim.x) {
    const KeyT k = keys[p];
    if ((long long)k >= n_keys) continue;  // capacity-mode padding (sorted last)
    if (p == 0) ranges[k].x = 0;
    if (p == n_pairs - 1) {
      ranges[k].y = (int)n_pairs;
    } else {
      const KeyT k2 = keys[p + 1];
      if (k2 != k) {
        ranges[k].y = (int)(p + 1);
        if ((long long)k2 < n_keys) ranges[k2].x = (int)(p + 1);
      }
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
// kRun8: a single 8-voxel run when Qxx sx^2 >= -1.5 (the bound of raster.cu's
// run8 with the +64 offset; used by the forward, whose branch is warp-uniform).
template <bool kRun8 = false>
__device__ __forceinline__ void row8(float e[8], bool rec_ok, float dx0, float sx, float qxx, float c1, float c0o,
                                     float K) {
  if (kRun8 && qxx * sx * sx >= -1.5f) {
    const float qs = qxx * sx;
    const float t = fmaf(qxx, dx0, c1);
    float E = ex2v(fmaf(dx0, t, c0o));
    float R = ex2v(fminf(fmaf(2.f * qs, dx0, fmaf(c1, sx, qs * sx)), 126.f));
    e[0] = E;
#pragma unroll
    for (int c = 1; c < 8; ++c) {
      E *= R;
      if (c < 7) R *= K;
      e[c] = E;
    }
  } else if (rec_ok) {
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

// row8's two 4-voxel runs for two kernels at once (K8: kernels gq and gq + 8
// of a chunk, each with its own x geometry) in packed FP32x2
__device__ __forceinline__ void run4x2v(float2 e[8], float2 dx0, float sx, float2 qxx, float2 c1, float2 c0o,
                                        float2 K) {
  const float2 s2 = make_float2(sx, sx);
  const float2 qs = __fmul2_rn(qxx, s2);
  const float2 dbase = __ffma2_rn(c1, s2, __fmul2_rn(qs, s2));  // D(dx) = 2 qxx sx dx + c1 sx + qxx sx^2
  const float2 qs2 = __fmul2_rn(make_float2(2.f, 2.f), qs);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float2 dx = __ffma2_rn(make_float2(4.f * h, 4.f * h), s2, dx0);
    const float2 t = __ffma2_rn(qxx, dx, c1);
    const float2 L = __ffma2_rn(dx, t, c0o);
    const float2 D = __ffma2_rn(qs2, dx, dbase);
    float2 E = make_float2(ex2v(L.x), ex2v(L.y));
    float2 R = make_float2(ex2v(fminf(D.x, 126.f)), ex2v(fminf(D.y, 126.f)));
    e[4 * h] = E;
    E = __fmul2_rn(E, R);
    R = __fmul2_rn(R, K);
    e[4 * h + 1] = E;
    E = __fmul2_rn(E, R);
    R = __fmul2_rn(R, K);
    e[4 * h + 2] = E;
    e[4 * h + 3] = __fmul2_rn(E, R);
  }
}

// one 8-voxel run for two kernels at once (K8, warp-uniform when every
// kernel of the chunk has Qxx sx^2 >= -1.25: with the +15 offset no value
// above 2^-11 of the kernel's peak — binary16 E's resolution — can sit in a
// run whose first voxel flushes; the derivation is at raster.cu's K4 8-run)
__device__ __forceinline__ void run8x2v(float2 e[8], float2 dx0, float sx, float2 qxx, float2 c1, float2 c0o,
                                        float2 K) {
  const float2 s2 = make_float2(sx, sx);
  const float2 qs = __fmul2_rn(qxx, s2);
  const float2 t = __ffma2_rn(qxx, dx0, c1);
  const float2 L = __ffma2_rn(dx0, t, c0o);
  const float2 D = __ffma2_rn(__fmul2_rn(make_float2(2.f, 2.f), qs), dx0, __ffma2_rn(c1, s2, __fmul2_rn(qs, s2)));
  float2 E = make_float2(ex2v(L.x), ex2v(L.y));
  float2 R = make_float2(ex2v(fminf(D.x, 126.f)), ex2v(fminf(D.y, 126.f)));
  e[0] = E;
#pragma unroll
  for (int c = 1; c < 8; ++c) {
    E = __fmul2_rn(E, R);
    if (c < 7) R = __fmul2_rn(R, K);
    e[c] = E;
  }
}

// row8 for two rows of one kernel at once (rows z and z + 4 of a lane: same
// x geometry, their own c1 / c0o) in packed FP32x2 arithmetic (FFMA2 / FMUL2
// on sm_100); element r of every float2 is exactly row8's value for row r.
__device__ __forceinline__ void row8x2(float2 e[8], bool rec_ok, float dx0, float sx, float qxx, float2 c1,
                                       float2 c0o, float K) {
  const float2 K2 = make_float2(K, K), q2 = make_float2(qxx, qxx);
  if (qxx * sx * sx >= -1.5f) {
    const float qs = qxx * sx;
    const float2 d0 = make_float2(dx0, dx0);
    const float2 t = __ffma2_rn(q2, d0, c1);
    const float2 L = __ffma2_rn(d0, t, c0o);
    const float2 D = __ffma2_rn(make_float2(2.f * qs, 2.f * qs), d0,
                                __ffma2_rn(c1, make_float2(sx, sx), make_float2(qs * sx, qs * sx)));
    float2 E = make_float2(ex2v(L.x), ex2v(L.y));
    float2 R = make_float2(ex2v(fminf(D.x, 126.f)), ex2v(fminf(D.y, 126.f)));
    e[0] = E;
#pragma unroll
    for (int c = 1; c < 8; ++c) {
      E = __fmul2_rn(E, R);
      if (c < 7) R = __fmul2_rn(R, K2);
      e[c] = E;
    }
  } else if (rec_ok) {
    const float qs = qxx * sx;
    const float2 dbase = __ffma2_rn(c1, make_float2(sx, sx), make_float2(qs * sx, qs * sx));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float dxs = fmaf(4.f * h, sx, dx0);
      const float2 dx = make_float2(dxs, dxs);
      const float2 t = __ffma2_rn(q2, dx, c1);
      const float2 L = __ffma2_rn(dx, t, c0o);
      const float2 D = __ffma2_rn(make_float2(2.f * qs, 2.f * qs), dx, dbase);
      float2 E = make_float2(ex2v(L.x), ex2v(L.y));
      float2 R = make_float2(ex2v(fminf(D.x, 126.f)), ex2v(fminf(D.y, 126.f)));
      e[4 * h] = E;
      E = __fmul2_rn(E, R);
      R = __fmul2_rn(R, K2);
      e[4 * h + 1] = E;
      E = __fmul2_rn(E, R);
      R = __fmul2_rn(R, K2);
      e[4 * h + 2] = E;
      e[4 * h + 3] = __fmul2_rn(E, R);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float dxs = fmaf((float)c, sx, dx0);
      const float2 dx = make_float2(dxs, dxs);
      const float2 L = __ffma2_rn(dx, __ffma2_rn(q2, dx, c1), c0o);
      e[c] = make_float2(ex2v(L.x), ex2v(L.y));
    }
  }
}

// K7: one warp per brick, four bricks per CTA; lane = rows (y, z) and (y, z+4),
// 8 voxels each. Each warp stages its brick list 32 records at a time through
// its own shared memory, prefetching the next chunk into registers.
constexpr int kEvalWarps = 4;
__global__ void __launch_bounds__(32 * kEvalWarps) voxel_eval_kernel(BrickGeo G, const int2* __restrict__ ranges,
                                                                     const int32_t* __restrict__ vals,
                                                                     const float4* __restrict__ rec, int splits,
                                                                     float* __restrict__ partial,
                                                                     float* __restrict__ vol) {
  pdl_prologue();
  __shared__ float4 sA[kEvalWarps][32];  // base offset xyz, rho*2^-64
  __shared__ float4 sB[kEvalWarps][32];  // Qxx Qyy Qzz K
  __shared__ float4 sC[kEvalWarps][32];  // Qxy Qxz Qyz
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * kEvalWarps + warp;
  const long long b = gw / splits;
  const int part = (int)(gw % splits);
  if (b >= G.n_bricks) return;
  int tx, ty, tz;
  brick_of(G, b, tx, ty, tz);
  const int brick = (tz * G.by + ty) * G.bx + tx;
  int2 rg = ranges[brick];
  SCT_DCHECK(0 <= rg.x && rg.x <= rg.y);
  if (splits > 1) {  // small grids: several warps per brick list, summed by voxel_reduce
    const int len = rg.y - rg.x, s0 = rg.x;
    rg.x = s0 + (int)((long long)len * part / splits);
    rg.y = s0 + (int)((long long)len * (part + 1) / splits);
    vol = partial + (long long)part * G.dims.x * G.dims.y * G.dims.z;
  }
  const double c0x = G.origin.x + ((double)(tx * kTileVox) + 0.5) * G.spacing.x;
  const double c0y = G.origin.y + ((double)(ty * kTileVox) + 0.5) * G.spacing.y;
  const double c0z = G.origin.z + ((double)(tz * kTileVox) + 0.5) * G.spacing.z;
  const int ly = lane & 7, lz = lane >> 3;  // rows (ly, lz) and (ly, lz + 4)
  const float fy = (float)ly * G.spf.y;
  const float fz0 = (float)lz * G.spf.z, fz1 = (float)(lz + 4) * G.spf.z;
  float2 acc2[8];  // (row z, row z + 4) per column
#pragma unroll
  for (int c = 0; c < 8; ++c) acc2[c] = make_float2(0.f, 0.f);
  const float2 fz = make_float2(fz0, fz1);
  float4 na = make_float4(0.f, 0.f, 0.f, 0.f), nb = na, nc = na;
  auto fetch = [&](int p) {
    const long long i = vals[p];
    SCT_DCHECK(i >= 0);
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
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
      const float4 a = sA[warp][j];
      const float4 q = sB[warp][j];
      const float4 o = sC[warp][j];
      const bool rec_ok = q.x * G.spf.x * G.spf.x >= -8.f;
      const float dy = a.y + fy;
      // both rows together: per element the scalar path's operations
      const float2 dz = __fadd2_rn(make_float2(a.z, a.z), fz);
      const float ody = o.z * dy, qdy = q.y * dy;
      const float2 c0o = __ffma2_rn(make_float2(qdy, qdy), make_float2(dy, dy),
                                    __ffma2_rn(__fmul2_rn(make_float2(q.z, q.z), dz), dz,
                                               __ffma2_rn(make_float2(ody, ody), dz, make_float2(64.f, 64.f))));
      const float2 c1 = __ffma2_rn(make_float2(o.x, o.x), make_float2(dy, dy),
                                   __fmul2_rn(make_float2(o.y, o.y), dz));
      float2 e[8];
      row8x2(e, rec_ok, a.x, G.spf.x, q.x, c1, c0o, q.w);
#pragma unroll
      for (int c = 0; c < 8; ++c) acc2[c] = __ffma2_rn(make_float2(a.w, a.w), e[c], acc2[c]);
    }
  }
  float acc[2][8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    acc[0][c] = acc2[c].x;
    acc[1][c] = acc2[c].y;
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
  pdl_prologue();
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

// K8 (tensor-core form), the voxel analogue of the rasterizer's moment GEMM
// (raster.cu, K4): with brick-centred voxel coordinates c' = index - 3.5 and
// the kernel's offset o = brick centre - kernel position, d = s*c' + o per
// axis, so the 10 statistics follow from the moments
// M[kernel][n] = sum_voxels E * g * {1, cx, cy, cz, cx^2, cy^2, cz^2, cxcy, cxcz, cycz}
// by a binomial shift. E comes from the x-recurrence (row8, +15 exponent
// offset so it fits binary16; values below 2^-29 of a kernel's peak lose
// precision) written straight into m16n8k16 A fragments; G (per brick: the
// upstream gradient times the 10 monomials, two n8 tiles) is split into hi + lo
// binary16 parts after a per-brick power-of-two scale. Lane t of a quad owns
// the x-row 4q + t (y = row & 7, z = row >> 3) of row quad q for kernels gq and
// gq + 8; slice 2q + h maps k = 2t, 2t+1 to x = 4h + {0, 1} and k = 2t+8, 2t+9
// to x = 4h + {2, 3}.
constexpr int kVMmaWarps = 4;

__device__ __forceinline__ void vmma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo_k, float hi_k) {
  const __half2 h = __floats2half2_rn(lo_k, hi_k);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__global__ void __launch_bounds__(32 * kVMmaWarps, 7) voxel_backward_mma_kernel(
    BrickGeo G, const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    const short4* __restrict__ lo, const short4* __restrict__ hi, const int32_t* __restrict__ offset,
    const float* __restrict__ dL, float* __restrict__ pair_stats, int parts) {
  pdl_prologue();
  // B fragments [slice][lane] = {hi k0-1, hi k8-9, lo k0-1, lo k8-9}: n tile 0
  // (moments 0-7) for all lanes; n tile 1 holds moments 8, 9 only (lanes 0-7)
  __shared__ uint4 s_g[32][32];
  __shared__ uint4 s_g1[32][8];
  __shared__ float s_gmax[kVMmaWarps];
  int tx, ty, tz;
  brick_of(G, blockIdx.x / parts, tx, ty, tz);
  const int brick = (tz * G.by + ty) * G.bx + tx;
  int2 rg = ranges[brick];
  SCT_DCHECK(0 <= rg.x && rg.x <= rg.y);
  if (parts > 1) {  // part of the list (small grids)
    const int len = rg.y - rg.x, s0 = rg.x, part = blockIdx.x % parts;
    rg.x = s0 + (int)((long long)len * part / parts);
    rg.y = s0 + (int)((long long)len * (part + 1) / parts);
  }
  if (rg.y <= rg.x) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane & 3, gq = lane >> 2;
  const int x0 = tx * kTileVox, y0 = ty * kTileVox, z0 = tz * kTileVox;
  auto grad = [&](int x, int y, int z) -> float {
    const int X = x0 + x, Y = y0 + y, Z = z0 + z;
    return (X < G.dims.x && Y < G.dims.y && Z < G.dims.z)
               ? __ldg(dL + ((long long)Z * G.dims.y + Y) * G.dims.x + X)
               : 0.f;
  };
  // --- per-brick scale: largest |G| = gmax * 12.25 * 2^-15 * S <= 2^14
  float gm = 0.f;
  for (int v = threadIdx.x; v < 512; v += 32 * kVMmaWarps) gm = fmaxf(gm, fabsf(grad(v & 7, (v >> 3) & 7, v >> 6)));
  gm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(gm)));
  if (lane == 0) s_gmax[warp] = gm;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kVMmaWarps; ++k) gm = fmaxf(gm, s_gmax[k]);
  const float S = gm > 0.f ? exp2f(floorf(log2f(16384.f / (gm * 12.25f * 0x1p-15f)))) : 1.f;
  const float gscale = 0x1p-15f * S, inv_s = 1.f / S;
  // --- G fragments: each thread produces voxel pairs (adjacent k) for all 16 moments
  for (int pp = threadIdx.x; pp < 256; pp += 32 * kVMmaWarps) {
    const int s = pp >> 3, j = pp & 7;
    const int tp = j >> 1, part = j & 1;
    const int q = s >> 1, h = s & 1;
    const int r = 4 * q + tp;
    const int y = r & 7, z = r >> 3;
    const int xa = 4 * h + 2 * part;
    float ph[2][16];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float g = grad(xa + e, y, z) * gscale;
      const float cx = (float)(xa + e) - 3.5f, cy = (float)y - 3.5f, cz = (float)z - 3.5f;
      ph[e][0] = g;
      ph[e][1] = g * cx;
      ph[e][2] = g * cy;
      ph[e][3] = g * cz;
      ph[e][4] = g * cx * cx;
      ph[e][5] = g * cy * cy;
      ph[e][6] = g * cz * cz;
      ph[e][7] = g * cx * cy;
      ph[e][8] = g * cx * cz;
      ph[e][9] = g * cy * cz;
#pragma unroll
      for (int n = 10; n < 16; ++n) ph[e][n] = 0.f;
    }
#pragma unroll
    for (int n = 0; n < 10; ++n) {  // moments 10..15 are zero: not stored
      const __half2 hv = __floats2half2_rn(ph[0][n], ph[1][n]);
      const float2 f = __half22float2(hv);
      const uint32_t hb = *reinterpret_cast<const uint32_t*>(&hv);
      const uint32_t lb = pack_h2(ph[0][n] - f.x, ph[1][n] - f.y);
      uint32_t* dst = reinterpret_cast<uint32_t*>(n < 8 ? &s_g[s][n * 4 + tp] : &s_g1[s][(n - 8) * 4 + tp]);
      dst[part] = hb;
      dst[2 + part] = lb;
    }
  }
  __syncthreads();
  const double c0x = G.origin.x + ((double)x0 + 0.5) * G.spacing.x;
  const double c0y = G.origin.y + ((double)y0 + 0.5) * G.spacing.y;
  const double c0z = G.origin.z + ((double)z0 + 0.5) * G.spacing.z;
  const float sx = G.spf.x, sy = G.spf.y, sz = G.spf.z;
  const int n_list = rg.y - rg.x;
  for (int cb = 16 * warp; cb < n_list; cb += 16 * kVMmaWarps) {
    float bxk[2], byk[2], bzk[2];
    float4 qk[2], okk[2];
    bool valid[2], rec_ok[2];
    long long itk[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int e = cb + gq + 8 * k;
      valid[k] = e < n_list;
      itk[k] = valid[k] ? vals[rg.x + e] : 0;
      const float4 a = __ldg(rec + 3 * itk[k]);
      qk[k] = __ldg(rec + 3 * itk[k] + 1);
      okk[k] = __ldg(rec + 3 * itk[k] + 2);
      bxk[k] = (float)(c0x - (double)a.x);
      byk[k] = (float)(c0y - (double)a.y);
      bzk[k] = (float)(c0z - (double)a.z);
      rec_ok[k] = qk[k].x * sx * sx >= -8.f;
    }
    const float2 bx2 = make_float2(bxk[0], bxk[1]), by2 = make_float2(byk[0], byk[1]);
    const float2 bz2 = make_float2(bzk[0], bzk[1]);
    const float2 qx2 = make_float2(qk[0].x, qk[1].x), qy2 = make_float2(qk[0].y, qk[1].y);
    const float2 qz2 = make_float2(qk[0].z, qk[1].z), K2 = make_float2(qk[0].w, qk[1].w);
    const float2 ox2 = make_float2(okk[0].x, okk[1].x), oy2 = make_float2(okk[0].y, okk[1].y);
    const float2 oz2 = make_float2(okk[0].z, okk[1].z), c15 = make_float2(15.f, 15.f);
    const bool r8 = __all_sync(0xffffffffu, qk[0].x * sx * sx >= -1.25f && qk[1].x * sx * sx >= -1.25f);
    float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
    // the +15 exponent offset, or -1e30 for a slot past the list (E = 0)
    const float2 off = make_float2(valid[0] ? 15.f : -1e30f, valid[1] ? 15.f : -1e30f);
    // the 16 voxel rows; the 8-run mode chosen once per chunk (warp-uniform)
    auto rows = [&](auto mode) {
      constexpr bool kR8 = decltype(mode)::value;
#pragma unroll 4
      for (int q = 0; q < 16; ++q) {
        const int r = 4 * q + t;
        const float fy = (float)(r & 7) * sy, fz = (float)(r >> 3) * sz;
        float E[2][8];
        {  // kernels gq (.x) and gq + 8 (.y) in packed FP32x2; elementwise the scalar row8
          const float2 dy = __fadd2_rn(by2, make_float2(fy, fy)), dz = __fadd2_rn(bz2, make_float2(fz, fz));
          const float2 c0o = __ffma2_rn(__fmul2_rn(qy2, dy), dy,
                                        __ffma2_rn(__fmul2_rn(qz2, dz), dz, __ffma2_rn(__fmul2_rn(oz2, dy), dz, off)));
          const float2 c1 = __ffma2_rn(ox2, dy, __fmul2_rn(oy2, dz));
          if (kR8) {
            float2 e[8];
            run8x2v(e, bx2, sx, qx2, c1, c0o, K2);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              E[0][i] = e[i].x;
              E[1][i] = e[i].y;
            }
          } else if (rec_ok[0] && rec_ok[1]) {
            float2 e[8];
            run4x2v(e, bx2, sx, qx2, c1, c0o, K2);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              E[0][i] = e[i].x;
              E[1][i] = e[i].y;
            }
          } else {
            row8(E[0], rec_ok[0], bxk[0], sx, qk[0].x, c1.x, c0o.x, qk[0].w);
            row8(E[1], rec_ok[1], bxk[1], sx, qk[1].x, c1.y, c0o.y, qk[1].w);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t a0 = pack_h2(E[0][4 * h], E[0][4 * h + 1]);
          const uint32_t a1 = pack_h2(E[1][4 * h], E[1][4 * h + 1]);
          const uint32_t a2 = pack_h2(E[0][4 * h + 2], E[0][4 * h + 3]);
          const uint32_t a3 = pack_h2(E[1][4 * h + 2], E[1][4 * h + 3]);
          const uint4 g0 = s_g[2 * q + h][lane];
          const uint4 g1 = lane < 8 ? s_g1[2 * q + h][lane] : make_uint4(0u, 0u, 0u, 0u);
          vmma_f16(acc0, a0, a1, a2, a3, g0.x, g0.y);
          vmma_f16(acc0, a0, a1, a2, a3, g0.z, g0.w);
          vmma_f16(acc1, a0, a1, a2, a3, g1.x, g1.y);
          vmma_f16(acc1, a0, a1, a2, a3, g1.z, g1.w);
        }
      }
    };
    if (r8) rows(std::true_type{});
    else rows(std::false_type{});
    // acc0: moments 2t, 2t+1 (c0,c1: kernel gq; c2,c3: kernel gq + 8); acc1: moments 8 + 2t, 9 + 2t
    const int base = lane & ~3;
    const bool second = t == 1;
    float m[10];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float x0v = __shfl_sync(0xffffffffu, acc0[0], base + k);
      const float x1v = __shfl_sync(0xffffffffu, acc0[1], base + k);
      const float y0v = __shfl_sync(0xffffffffu, acc0[2], base + k);
      const float y1v = __shfl_sync(0xffffffffu, acc0[3], base + k);
      m[2 * k] = (second ? y0v : x0v) * inv_s;
      m[2 * k + 1] = (second ? y1v : x1v) * inv_s;
    }
    {
      const float x0v = __shfl_sync(0xffffffffu, acc1[0], base);
      const float x1v = __shfl_sync(0xffffffffu, acc1[1], base);
      const float y0v = __shfl_sync(0xffffffffu, acc1[2], base);
      const float y1v = __shfl_sync(0xffffffffu, acc1[3], base);
      m[8] = (second ? y0v : x0v) * inv_s;
      m[9] = (second ? y1v : x1v) * inv_s;
    }
    const int kk = second ? 1 : 0;
    if (t < 2 && (kk ? valid[1] : valid[0])) {
      const float ox = fmaf(3.5f, sx, kk ? bxk[1] : bxk[0]);
      const float oy = fmaf(3.5f, sy, kk ? byk[1] : byk[0]);
      const float oz = fmaf(3.5f, sz, kk ? bzk[1] : bzk[0]);
      const long long i = kk ? itk[1] : itk[0];
      float v[10];
      v[0] = m[0];
      v[1] = fmaf(ox, m[0], sx * m[1]);
      v[2] = fmaf(oy, m[0], sy * m[2]);
      v[3] = fmaf(oz, m[0], sz * m[3]);
      v[4] = fmaf(ox, fmaf(ox, m[0], 2.f * sx * m[1]), sx * sx * m[4]);
      v[5] = fmaf(oy, fmaf(oy, m[0], 2.f * sy * m[2]), sy * sy * m[5]);
      v[6] = fmaf(oz, fmaf(oz, m[0], 2.f * sz * m[3]), sz * sz * m[6]);
      v[7] = fmaf(ox, fmaf(oy, m[0], sy * m[2]), fmaf(oy * sx, m[1], sx * sy * m[7]));
      v[8] = fmaf(ox, fmaf(oz, m[0], sz * m[3]), fmaf(oz * sx, m[1], sx * sz * m[8]));
      v[9] = fmaf(oy, fmaf(oz, m[0], sz * m[3]), fmaf(oz * sy, m[2], sy * sz * m[9]));
      const short4 l = lo[i], hh = hi[i];
      const int nx = hh.x - l.x + 1, ny = hh.y - l.y + 1;
      const long long slot = offset[i] + ((tz - l.z) * ny + (ty - l.y)) * nx + (tx - l.x);
      float4* dst = reinterpret_cast<float4*>(pair_stats + 12 * slot);
      dst[0] = make_float4(v[0], v[1], v[2], v[3]);
      dst[1] = make_float4(v[4], v[5], v[6], v[7]);
      *reinterpret_cast<float2*>(dst + 2) = make_float2(v[8], v[9]);
    }
  }
}

// vol[i] = sum over parts (in part order) of the split evaluation's partials
__global__ void __launch_bounds__(256) voxel_reduce_kernel(const float* __restrict__ partial, int splits,
                                                           long long stride, long long n, float* __restrict__ vol) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < splits; ++p) s += partial[(long long)p * stride + i];
    vol[i] = s;
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
                       int32_t bricks_x, int32_t bricks_y, void* keys, bool keys16, int32_t* vals, int64_t cap) {
  if (m == 0) return;
  long long b = (m + 255) / 256;
  if (b > (long long)c->sm_count * 16) b = (long long)c->sm_count * 16;
  KScope _ks(c, "K6_voxel_emit");
  if (keys16)
    pdl_launch(voxel_emit_kernel<uint16_t>, dim3((int)b), dim3(256), 0, c->stream, m, lo, hi, offset, bricks_x, bricks_y,
                                                               static_cast<uint16_t*>(keys), vals, (long long)cap);
  else
    pdl_launch(voxel_emit_kernel<uint32_t>, dim3((int)b), dim3(256), 0, c->stream, m, lo, hi, offset, bricks_x, bricks_y,
                                                               static_cast<uint32_t*>(keys), vals, (long long)cap);
}

void launch_key_ranges(Ctx* c, int64_t n_pairs, const void* keys, bool keys16, int2* ranges, int64_t n_keys) {
  if (n_pairs == 0) return;
  long long b = (n_pairs + 255) / 256;
  if (b > (long long)c->sm_count * 16) b = (long long)c->sm_count * 16;
  KScope _ks(c, "K2_ranges");
  if (keys16)
    pdl_launch(key_ranges_kernel<uint16_t>, dim3((int)b), dim3(256), 0, c->stream, n_pairs, static_cast<const uint16_t*>(keys), ranges,
                                                                (long long)n_keys);
  else
    pdl_launch(key_ranges_kernel<uint32_t>, dim3((int)b), dim3(256), 0, c->stream, n_pairs, static_cast<const uint32_t*>(keys), ranges,
                                                                (long long)n_keys);
}

void launch_voxel_eval(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x, int32_t bricks_y,
                       const int2* ranges, const int32_t* vals, const float4* rec, const sct_cloud&,
                       int64_t n_pairs, float* vol) {
  const long long nb = (long long)bricks_x * bricks_y * (zb1 - zb0);
  if (nb <= 0) return;
  // small grids (the train step's 32^3 TV sub-volume has 64 bricks): split
  // each brick list over several warps, then sum. The split depends on the
  // full grid only, so z-slab calls compute every brick exactly as the
  // full-grid call does (slab volumes compose bit-exactly).
  (void)n_pairs;
  const long long nb_full =
      (long long)bricks_x * bricks_y * (((long long)g.dims[2] + kTileVox - 1) / kTileVox);
  int splits = 1;
  while (splits < 16 && nb_full * splits * 2 <= (long long)c->sm_count * 32) splits *= 2;
  if (const char* e = std::getenv("SCT_K7_SPLITS")) splits = std::max(1, std::min(16, atoi(e)));
  const long long nvox = (long long)g.dims[0] * g.dims[1] * g.dims[2];
  float* partial = nullptr;
  // (every part writes every voxel of its slab bricks, so no clearing is needed)
  if (splits > 1 && stage_buf(c, 25, sizeof(float) * (size_t)nvox * splits, (void**)&partial) != SCT_OK) return;
  {
    KScope _ks(c, "K7_voxel_eval");
    const long long warps = nb * splits;
    pdl_launch(voxel_eval_kernel, dim3((unsigned)((warps + kEvalWarps - 1) / kEvalWarps)), dim3(32 * kEvalWarps), 0, c->stream, make_geo(g, zb0, zb1, bricks_x, bricks_y), ranges, vals, rec, splits, partial, vol);
  }
  if (splits > 1) {
    KScope _ks(c, "K7_reduce");
    const long long z0 = (long long)zb0 * kTileVox, z1 = std::min<long long>((long long)zb1 * kTileVox, g.dims[2]);
    const long long plane = (long long)g.dims[0] * g.dims[1];
    const long long n = (z1 - z0) * plane;
    if (n > 0)
      pdl_launch(voxel_reduce_kernel, dim3((unsigned)std::min<long long>((n + 255) / 256, (long long)c->sm_count * 16)), dim3(256), 0, c->stream, partial + z0 * plane, splits, nvox, n, vol + z0 * plane);
  }
}

void launch_voxel_backward_stats(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x,
                                 int32_t bricks_y, const int2* ranges, const int32_t* vals, const float4* rec,
                                 const short4* lo, const short4* hi, const int32_t* offset, const sct_cloud&,
                                 int64_t n_pairs, const float* dL, float4* pair_stats) {
  const long long nb = (long long)bricks_x * bricks_y * (zb1 - zb0);
  if (nb <= 0) return;
  // small grids (the train step's TV sub-volume: 64 bricks): several CTAs per
  // list (>= 64 kernels each; pair statistics are independent) until the grid
  // fills the CTA slots (7 per SM)
  const double avg_len = (double)n_pairs / (double)nb;
  int parts = 1;
  // small grids (the train step's TV sub-grid): up to 32 parts of >= 16 kernels
  // on average while the grid stays within ~8 waves; large grids keep one CTA per brick
  while (parts < 32 && nb * parts * 2 <= (long long)c->sm_count * 56 && avg_len / (2 * parts) >= 16.0) parts *= 2;
  // SCT_K8=simt selects the FP32 SIMT statistics kernel; default: tensor-core moments
  static const bool simt = [] {
    const char* e = std::getenv("SCT_K8");
    return e && std::string(e) == "simt";
  }();
  KScope _ks(c, "K8_voxel_backward_stats");
  if (simt)
    pdl_launch(voxel_backward_stats_kernel, dim3((unsigned)nb), dim3(kVBwdThreads), 0, c->stream, make_geo(g, zb0, zb1, bricks_x, bricks_y), ranges, vals, rec, lo, hi, offset, dL,
        reinterpret_cast<float*>(pair_stats));
  else
    pdl_launch(voxel_backward_mma_kernel, dim3((unsigned)(nb * parts)), dim3(32 * kVMmaWarps), 0, c->stream, make_geo(g, zb0, zb1, bricks_x, bricks_y), ranges, vals, rec, lo, hi, offset, dL,
        reinterpret_cast<float*>(pair_stats), parts);
}

}  // namespace sct
