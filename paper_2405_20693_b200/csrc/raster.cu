// Rasterizer FP32 hot kernels (sm_100a).
//
//   K2 raster_emit      — (view,tile) keys for every covered tile of every
//                         visible item, Gaussian-major (rasterizer.cpp:127-132)
//   K2 ranges           — per-(view,tile) [start,end) of the sorted pairs
//   K3 composite        — I(u,v) = sum_list amp * exp(-1/2 d^T conic d)
//                         (rasterizer.cpp:135-155), list order, fp32
//   K4 backward stats   — per (tile, kernel) sufficient statistics
//                         s0, s1 (2), s2 (3) (rasterizer.cpp:207-243)
//
// Records are log2-prescaled: exp(-1/2 d^T Q d) = exp2(A dx^2 + B dx dy + C dy^2),
// so each Gaussian-pixel evaluation is 3 FP32 ops + one MUFU.EX2.
#include <cuda_runtime.h>

#include "sct_internal.cuh"

namespace sct {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

namespace {

__global__ void __launch_bounds__(256) raster_emit_kernel(long long n_items, long long m,
                                                          const short4* __restrict__ rect,
                                                          const int32_t* __restrict__ offset, int tiles_x,
                                                          int tile_bits, uint32_t* __restrict__ keys,
                                                          int32_t* __restrict__ vals) {
  for (long long item = blockIdx.x * (long long)blockDim.x + threadIdx.x; item < n_items;
       item += (long long)gridDim.x * blockDim.x) {
    const int32_t o0 = offset[item];
    const int32_t o1 = offset[item + 1];
    if (o1 == o0) continue;
    const short4 r = rect[item];
    const uint32_t vbase = (uint32_t)(item / m) << tile_bits;
    int32_t o = o0;
    for (int ty = r.z; ty <= r.w; ++ty)
      for (int tx = r.x; tx <= r.y; ++tx) {
        keys[o] = vbase | (uint32_t)(ty * tiles_x + tx);
        vals[o] = (int32_t)item;
        ++o;
      }
  }
}

__global__ void __launch_bounds__(256) ranges_kernel(long long n_pairs, const uint32_t* __restrict__ keys,
                                                     int tile_bits, long long tiles_per_view,
                                                     int2* __restrict__ ranges) {
  const uint32_t mask = (1u << tile_bits) - 1u;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n_pairs;
       p += (long long)gridDim.x * blockDim.x) {
    const uint32_t k = keys[p];
    const long long slot = (long long)(k >> tile_bits) * tiles_per_view + (k & mask);
    if (p == 0 || keys[p - 1] != k) ranges[slot].x = (int)p;
    if (p == n_pairs - 1 || keys[p + 1] != k) ranges[slot].y = (int)(p + 1);
  }
}

// K3: one 64-thread CTA per (tile, view); thread = 1 row x 4 columns.
// Records for the tile list are staged through shared memory 64 at a time
// (coalesced float4 gathers); every thread then reads them as broadcasts.
constexpr int kCompThreads = 64;
__global__ void __launch_bounds__(kCompThreads) composite_kernel(
    const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    int tiles_x, int tiles_per_view, int W, int H, float* __restrict__ images) {
  __shared__ float4 s0[kCompThreads];
  __shared__ float4 s1[kCompThreads];
  const int tile = blockIdx.x;
  const int view = blockIdx.y;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int row = threadIdx.x >> 2;
  const int col0 = (threadIdx.x & 3) * 4;
  const int u0 = tx * kTilePx + col0;
  const int v = ty * kTilePx + row;
  const float py = (float)v + 0.5f;
  const float px0 = (float)u0 + 0.5f;
  const int2 rg = ranges[(long long)view * tiles_per_view + tile];
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  for (int base = rg.x; base < rg.y; base += kCompThreads) {
    const int n = min(kCompThreads, rg.y - base);
    __syncthreads();
    if ((int)threadIdx.x < n) {
      const long long item = vals[base + threadIdx.x];
      s0[threadIdx.x] = rec[2 * item];
      s1[threadIdx.x] = rec[2 * item + 1];
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
      const float4 a = s0[j];  // cx cy amp
      const float4 b = s1[j];  // A B C
      const float dy = py - a.y;
      const float bdy = b.y * dy;
      const float cdy2 = b.z * dy * dy;
      const float dx = px0 - a.x;
      float d, t;
      d = dx;        t = fmaf(b.x, d, bdy); acc0 = fmaf(a.z, ex2(fmaf(d, t, cdy2)), acc0);
      d = dx + 1.f;  t = fmaf(b.x, d, bdy); acc1 = fmaf(a.z, ex2(fmaf(d, t, cdy2)), acc1);
      d = dx + 2.f;  t = fmaf(b.x, d, bdy); acc2 = fmaf(a.z, ex2(fmaf(d, t, cdy2)), acc2);
      d = dx + 3.f;  t = fmaf(b.x, d, bdy); acc3 = fmaf(a.z, ex2(fmaf(d, t, cdy2)), acc3);
    }
  }
  if (v < H) {
    float* out = images + ((long long)view * H + v) * W;
    if (u0 + 3 < W && (W & 3) == 0) {
      *reinterpret_cast<float4*>(out + u0) = make_float4(acc0, acc1, acc2, acc3);
    } else {
      if (u0 < W) out[u0] = acc0;
      if (u0 + 1 < W) out[u0 + 1] = acc1;
      if (u0 + 2 < W) out[u0 + 2] = acc2;
      if (u0 + 3 < W) out[u0 + 3] = acc3;
    }
  }
}

// K4: Gaussian-major backward statistics. One 256-thread CTA per non-empty
// (tile, view). Sixteen lanes share a Gaussian, one pixel row each, so the
// sums over a row stay in registers; the 16 partials are combined with warp
// shuffles and written once per (tile, Gaussian) pair into that pair's slot
// (slot = item's scan offset + rank of this tile in its rectangle), which the
// chain kernel later reduces in the reference's fixed tile order
// (rasterizer.cpp:245-257) — deterministic, no atomics.
constexpr int kBwdThreads = 256;
__global__ void __launch_bounds__(kBwdThreads) backward_stats_kernel(
    const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    const short4* __restrict__ rect, const int32_t* __restrict__ offset, int tiles_x, int tiles_per_view, int W,
    int H, const float* __restrict__ dL, float4* __restrict__ pair_stats) {
  const int tile = blockIdx.x;
  const int view = blockIdx.y;
  const int2 rg = ranges[(long long)view * tiles_per_view + tile];
  if (rg.y <= rg.x) return;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lane16 = threadIdx.x & 15;
  const int group = threadIdx.x >> 4;
  const int v = ty * kTilePx + lane16;
  const int u0 = tx * kTilePx;
  // upstream gradient of this thread's pixel row, in registers
  float g[kTilePx];
  const float* drow = dL + ((long long)view * H + v) * W + u0;
#pragma unroll
  for (int c = 0; c < kTilePx; ++c) g[c] = (v < H && u0 + c < W) ? __ldg(drow + c) : 0.f;
  const float py = (float)v + 0.5f;
  const float px0 = (float)u0 + 0.5f;
  for (int base = rg.x; base < rg.y; base += 16) {
    const int j = base + group;
    const bool valid = j < rg.y;
    float st0 = 0.f, st1 = 0.f, st2 = 0.f, st3 = 0.f, st4 = 0.f, st5 = 0.f;
    long long item = 0;
    if (valid) {
      item = vals[j];
      const float4 a = __ldg(rec + 2 * item);
      const float4 b = __ldg(rec + 2 * item + 1);
      const float dy = py - a.y;
      const float bdy = b.y * dy;
      const float cdy2 = b.z * dy * dy;
      const float dx0 = px0 - a.x;
      float r0 = 0.f, rx = 0.f, rxx = 0.f;
#pragma unroll
      for (int c = 0; c < kTilePx; ++c) {
        const float dx = dx0 + (float)c;
        const float t = fmaf(b.x, dx, bdy);
        const float ge = g[c] * ex2(fmaf(dx, t, cdy2));
        r0 += ge;
        const float gx = ge * dx;
        rx += gx;
        rxx = fmaf(gx, dx, rxx);
      }
      st0 = r0;            // s0
      st1 = rx;            // s1.x
      st2 = dy * r0;       // s1.y
      st3 = rxx;           // s2.xx
      st4 = dy * dy * r0;  // s2.yy
      st5 = dy * rx;       // s2.xy
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
      st0 += __shfl_xor_sync(0xffffffffu, st0, off);
      st1 += __shfl_xor_sync(0xffffffffu, st1, off);
      st2 += __shfl_xor_sync(0xffffffffu, st2, off);
      st3 += __shfl_xor_sync(0xffffffffu, st3, off);
      st4 += __shfl_xor_sync(0xffffffffu, st4, off);
      st5 += __shfl_xor_sync(0xffffffffu, st5, off);
    }
    if (valid && lane16 == 0) {
      const short4 r = rect[item];
      const int slot = offset[item] + (ty - r.z) * (r.y - r.x + 1) + (tx - r.x);
      pair_stats[2 * (long long)slot] = make_float4(st0, st1, st2, st3);
      pair_stats[2 * (long long)slot + 1] = make_float4(st4, st5, 0.f, 0.f);
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

void launch_raster_emit(Ctx* c, int64_t n_items, int64_t m, const short4* rect, const int32_t* offset,
                        int tiles_x, int tile_bits, uint32_t* keys, int32_t* vals) {
  if (n_items == 0) return;
  {
    KScope _ks(c, "K2_raster_emit");
    raster_emit_kernel<<<grid_cap(c, n_items, 256), 256, 0, c->stream>>>(n_items, m, rect, offset, tiles_x,
                                                                        tile_bits, keys, vals);
  }
}

void launch_ranges(Ctx* c, int64_t n_pairs, const uint32_t* keys, int tile_bits, int64_t tiles_per_view,
                   int2* ranges) {
  if (n_pairs == 0) return;
  {
    KScope _ks(c, "K2_ranges");
    ranges_kernel<<<grid_cap(c, n_pairs, 256), 256, 0, c->stream>>>(n_pairs, keys, tile_bits, tiles_per_view,
                                                                    ranges);
  }
}

void launch_raster_composite(Ctx* c, const sct_fwd* s, float* images) {
  const int T = s->det.tiles_x * s->det.tiles_y;
  dim3 grid(T, s->n_views);
  {
    KScope _ks(c, "K3_composite");
    composite_kernel<<<grid, kCompThreads, 0, c->stream>>>(s->d_ranges, s->d_vals, s->d_rec, s->det.tiles_x, T,
                                                           s->det.w, s->det.h, images);
  }
}

void launch_raster_backward_stats(Ctx* c, const sct_fwd* s, const float* dL, float4* pair_stats) {
  if (s->n_pairs == 0) return;
  const int T = s->det.tiles_x * s->det.tiles_y;
  dim3 grid(T, s->n_views);
  {
    KScope _ks(c, "K4_backward_stats");
    backward_stats_kernel<<<grid, kBwdThreads, 0, c->stream>>>(s->d_ranges, s->d_vals, s->d_rec, s->d_rect,
                                                               s->d_offset, s->det.tiles_x, T, s->det.w, s->det.h,
                                                               dL, pair_stats);
  }
}

}  // namespace sct
