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
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "sct_internal.cuh"
#include "tcgen05.cuh"

namespace sct {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Asynchronous global -> shared copies (LDGSTS): staged data never passes
// through registers.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

constexpr int kBwdChunk = 256;  // tile-list entries staged per chunk in K4

namespace {

// Keys are the tile index only (16-bit when it fits): pairs are emitted
// view-major, so a stable sort on the tile groups them by (tile, view) and the
// view is recovered from the item (value) in the range scan.
template <typename KeyT>
__global__ void __launch_bounds__(256) raster_emit_kernel(long long n_items, const short4* __restrict__ rect,
                                                          const int32_t* __restrict__ offset, int tiles_x,
                                                          KeyT* __restrict__ keys, int32_t* __restrict__ vals) {
  pdl_prologue();
  // Warp-cooperative: a warp owns 32 consecutive items, whose pairs occupy one
  // contiguous output range (exclusive-scan order); lanes stride over that
  // range so the key/value stores are coalesced. Each output slot finds its
  // item by a 5-step binary search over the 32 offsets held in the lanes.
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w0 = (blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < n_items;
       w0 += warps * 32) {
    const long long it = w0 + lane;
    const int32_t o_l = it < n_items ? offset[it] : offset[n_items];
    const long long last = min(w0 + 32, n_items);
    const int32_t o_end = offset[last];
    short4 r = make_short4(0, -1, 0, -1);
    if (it < n_items) r = rect[it];
    const int rxy = ((int)(unsigned short)r.x) | ((int)r.y << 16);
    const int rzw = ((int)(unsigned short)r.z) | ((int)r.w << 16);
    const float inv_nx_l = 1.f / (float)max(r.y - r.x + 1, 1);  // rank -> (row, col) by reciprocal
    const int32_t o_0 = __shfl_sync(0xffffffffu, o_l, 0);
    for (int32_t p0 = o_0; p0 < o_end; p0 += 32) {
      const int32_t p = p0 + lane;
      // largest j with offset[w0+j] <= p
      int j = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int32_t oj = __shfl_sync(0xffffffffu, o_l, j + step);
        if (j + step < 32 && oj <= p) j += step;
      }
      const int32_t oj = __shfl_sync(0xffffffffu, o_l, j);
      const int jxy = __shfl_sync(0xffffffffu, rxy, j);
      const int jzw = __shfl_sync(0xffffffffu, rzw, j);
      const float inv_nx = __shfl_sync(0xffffffffu, inv_nx_l, j);
      if (p < o_end) {
        const int x0 = (short)(jxy & 0xffff), x1 = (short)(jxy >> 16), y0 = (short)(jzw & 0xffff);
        const int nx = x1 - x0 + 1;
        const int rank = p - oj;
        int q = (int)((float)rank * inv_nx);  // rank < 2^24: off by at most one, corrected exactly
        if (q * nx > rank) --q;
        if ((q + 1) * nx <= rank) ++q;
        const int ty = y0 + q, tx = x0 + (rank - q * nx);
        const long long item = w0 + j;
        keys[p] = (KeyT)(ty * tiles_x + tx);
        vals[p] = (int32_t)item;
      }
    }
  }
}


// ---------------------------------------------------------------------------
// K2 binning as one stable counting scatter (replaces emit + radix sort +
// ranges when the tile table fits in shared memory). The reference's lists
// (rasterizer.cpp:119-132) are, per (view, tile), the visible kernels in
// ascending index; items are view-major (item = view * m + kernel), so the
// target order is (tile, view, kernel) — a stable counting sort on the tile.
//   bin_count:   block (chunk c, view v) of consecutive items counts the
//                pairs per tile -> H[tile][view][chunk];
//   exclusive scan of H (cub) -> S: S[t][v][c] is where block (v, c)'s pairs
//                of tile t start; S[t][v][0] .. S[t][v+1][0] is list (v, t);
//   bin_scatter: the block recounts per warp (4 contiguous warp ranges),
//                prefixes the warps per tile, then each warp walks its items
//                32 at a time in item order: the rank of a lane's pair in tile
//                (tx, ty) among the round's earlier lanes is
//                popc(colmask[tx] & rowmask[ty] & lanes_below) — rectangles are
//                products of a column and a row range, so two 32-bit masks per
//                tile column / row give the exact stable rank;
//   bin_ranges:  (view, tile) ranges straight from S.
constexpr int kBinWarps = 4;
// SCT_SCATTER_SBOX=1: the scatter keeps its chunk's boxes in shared memory
// between the count and the write phase; 0: it re-reads them (L2) and needs
// only the tables, so more blocks fit per SM (default: cfg3 0.355 -> 0.297 ms,
// occupancy limited by registers instead of shared memory)
#ifndef SCT_SCATTER_SBOX
#define SCT_SCATTER_SBOX 0
#endif
// shared memory of the scatter: 4 warps x (tile counters + column and row
// masks) words + a chunk of rectangles (>= 256)
constexpr int64_t kScatterSmem = 225 * 1024;

// Item boxes in tile units, inclusive: the raster's rect (tx0, tx1, ty0, ty1)
// (hi == nullptr, one tile layer) or the voxelizer's brick box lo = (x0, y0,
// z0), hi = (x1, y1, z1). Tile id = (z * tiles_y + y) * tiles_x + x.
struct Box {
  int x0, x1, y0, y1, z0, z1;
};
__device__ __forceinline__ Box load_box(const short4* __restrict__ a, const short4* __restrict__ b, long long i,
                                        bool valid) {
  Box r{0, -1, 0, -1, 0, -1};
  if (!valid) return r;
  const short4 p = __ldg(a + i);
  if (!b) return Box{p.x, p.y, p.z, p.w, 0, 0};
  const short4 q = __ldg(b + i);
  return Box{p.x, q.x, p.y, q.y, p.z, q.z};
}
__device__ __forceinline__ bool box_empty(const Box& r) { return r.x1 < r.x0 || r.y1 < r.y0 || r.z1 < r.z0; }

__global__ void __launch_bounds__(256) bin_count_kernel(const short4* __restrict__ rect, const short4* __restrict__ hi,
                                                        long long m, int chunk, int T, int tiles_x, int tiles_y,
                                                        int32_t* __restrict__ H) {
  pdl_prologue();
  extern __shared__ uint32_t hist[];
  const int c = blockIdx.x, v = blockIdx.y;
  for (int t = threadIdx.x; t < T; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  const long long i0 = (long long)v * m + (long long)c * chunk;
  const long long i1 = (long long)v * m + min((long long)(c + 1) * chunk, m);
  // four boxes in flight per thread (the loop is latency-bound otherwise)
  for (long long i = i0 + threadIdx.x; i < i1; i += 4 * blockDim.x) {
    Box r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) r[k] = load_box(rect, hi, i + k * blockDim.x, i + k * blockDim.x < i1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (box_empty(r[k])) continue;
      for (int tz = r[k].z0; tz <= r[k].z1; ++tz)
        for (int ty = r[k].y0; ty <= r[k].y1; ++ty)
          for (int tx = r[k].x0; tx <= r[k].x1; ++tx) atomicAdd(&hist[(tz * tiles_y + ty) * tiles_x + tx], 1u);
    }
  }
  __syncthreads();
  int32_t* h = H + ((long long)v * gridDim.x + c) * T;  // block-major [view][chunk][tile], coalesced
  for (int t = threadIdx.x; t < T; t += blockDim.x) h[t] = (int32_t)hist[t];
}

// Exclusive prefix of the counts in (tile, view, chunk) order from the
// block-major table H[b][t] (b = view * chunks + chunk): S = TB[t] + P[b][t]
// with P the exclusive prefix down each tile column and TB the exclusive
// prefix of the column totals. Columns are scanned in row segments of
// kSegRows rows (pass 1 segment sums, pass 2 segment prefixes + column
// totals + tile bases, pass 3 apply); every access is coalesced across tiles.
constexpr int kSegRows = 64;
__global__ void __launch_bounds__(256) bin_colsum_kernel(const int32_t* __restrict__ H, int n_rows, int T,
                                                         int32_t* __restrict__ seg) {
  pdl_prologue();
  const int t = blockIdx.x * blockDim.x + threadIdx.x, g = blockIdx.y;
  if (t >= T) return;
  const int r0 = g * kSegRows, r1 = min(n_rows, r0 + kSegRows);
  int32_t acc = 0;
#pragma unroll 8
  for (int r = r0; r < r1; ++r) acc += H[(long long)r * T + t];
  seg[(long long)g * T + t] = acc;
}
__global__ void __launch_bounds__(256) bin_segscan_kernel(int32_t* __restrict__ seg, int n_seg, int T,
                                                          int32_t* __restrict__ coltot) {
  pdl_prologue();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  // 16 loads in flight before the in-place stores (a load after a store to
  // the same array is not hoisted: one L2 round trip per segment otherwise,
  // 34 us at cfg3's 115 segments)
  int32_t run = 0;
  for (int g0 = 0; g0 < n_seg; g0 += 16) {
    int32_t x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = g0 + k < n_seg ? seg[(long long)(g0 + k) * T + t] : 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (g0 + k < n_seg) seg[(long long)(g0 + k) * T + t] = run;
      run += x[k];
    }
  }
  coltot[t] = run;
}
// one block: exclusive prefix of the column totals -> tile_base[0..T], tile_base[T] = pairs
__global__ void __launch_bounds__(1024) bin_tilebase_kernel(const int32_t* __restrict__ coltot, int T,
                                                            int32_t* __restrict__ tile_base, long long cap,
                                                            int* __restrict__ overflow, int32_t* __restrict__ total) {
  pdl_prologue();
  __shared__ int32_t part[1024];
  const int per = (T + blockDim.x - 1) / blockDim.x;
  const int t0 = min(T, (int)threadIdx.x * per), t1 = min(T, t0 + per);
  int32_t mine = 0;
  for (int t = t0; t < t1; ++t) mine += coltot[t];
  part[threadIdx.x] = mine;
  __syncthreads();
  for (int d = 1; d < (int)blockDim.x; d <<= 1) {  // Hillis-Steele inclusive scan
    const int32_t y = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0;
    __syncthreads();
    part[threadIdx.x] += y;
    __syncthreads();
  }
  int32_t run = part[threadIdx.x] - mine;
  for (int t = t0; t < t1; ++t) {
    tile_base[t] = run;
    run += coltot[t];
  }
  if (threadIdx.x == blockDim.x - 1) {
    tile_base[T] = part[threadIdx.x];
    if (total) *total = (long long)part[threadIdx.x] > cap ? 0 : part[threadIdx.x];  // overflow: emptied
    if ((long long)part[threadIdx.x] > cap) atomicOr(overflow, 1);
  }
}

// The three scan passes + tile bases in one CTA for small tables (the train
// step's single view, small TV grids): T <= 1024 columns, kSmallScanThreads / T
// threads per column, each owning a contiguous row segment; segment sums ->
// column totals -> exclusive scan of the totals -> in-place exclusive prefix.
constexpr int kSmallScanThreads = 1024;
constexpr long long kSmallScanEntries = 1ll << 18;
__global__ void __launch_bounds__(kSmallScanThreads) bin_scan_small_kernel(int32_t* __restrict__ H, int n_rows,
                                                                           int T, int32_t* __restrict__ tile_base,
                                                                           long long cap, int* __restrict__ overflow,
                                                                           int32_t* __restrict__ total) {
  pdl_prologue();
  using Scan = cub::BlockScan<int32_t, kSmallScanThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int32_t seg_sum[kSmallScanThreads];
  __shared__ int32_t col[kSmallScanThreads + 1];
  const int S = kSmallScanThreads / T;  // threads (segments) per column
  const int tid = threadIdx.x;
  const int t = tid % T, j = tid / T;
  const bool active = j < S;
  const int per = (n_rows + S - 1) / S;
  const int r0 = min(n_rows, j * per), r1 = min(n_rows, r0 + per);
  int32_t mine = 0;
  if (active) {
#pragma unroll 8
    for (int r = r0; r < r1; ++r) mine += H[(long long)r * T + t];
  }
  seg_sum[tid] = mine;
  __syncthreads();
  int32_t c = 0;  // column total = its segments in order
  if (tid < T)
    for (int k = 0; k < S; ++k) c += seg_sum[k * T + tid];
  int32_t base = 0, run_total = 0;
  Scan(scan_tmp).ExclusiveSum(c, base, run_total);  // exclusive scan of the (<= 1024) column totals
  if (tid < T) col[tid] = base;
  if (tid == 0) {
    col[T] = run_total;
    if (total) *total = (long long)run_total > cap ? 0 : run_total;  // overflow: emptied
    if ((long long)run_total > cap) atomicOr(overflow, 1);
  }
  __syncthreads();
  for (int k = tid; k <= T; k += kSmallScanThreads) tile_base[k] = col[k];
  if (active) {
    int32_t run = col[t];
    for (int k = 0; k < j; ++k) run += seg_sum[k * T + t];
    for (int rb = r0; rb < r1; rb += 8) {  // 8 loads in flight before the in-place stores
      int32_t x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = rb + k < r1 ? H[(long long)(rb + k) * T + t] : 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (rb + k < r1) H[(long long)(rb + k) * T + t] = run;
        run += x[k];
      }
    }
  }
}

// capacity mode: a count scan whose total exceeds the pair buffers raises the
// overflow word and empties every item (zero counts and offsets, empty boxes),
// so no later kernel touches a pair slot beyond the buffers; the call's results
// are then empty, and the caller learns of it from sct_ctx_take_overflow.
__global__ void __launch_bounds__(256) capacity_guard_kernel(int32_t* __restrict__ count, int32_t* __restrict__ offset,
                                                             long long n, short4* __restrict__ box_a,
                                                             short4* __restrict__ box_b,
                                                             const long long* __restrict__ sum64, long long cap,
                                                             int* __restrict__ overflow) {
  pdl_prologue();
  // sum64 == nullptr: the int32 scan cannot have wrapped, offset[n] is the total
  const long long total = sum64 ? *sum64 : (long long)offset[n];
  if (total <= cap && offset[n] >= 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(overflow, 1);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n; i += (long long)gridDim.x * blockDim.x) {
    offset[i] = 0;
    if (i == n) continue;
    count[i] = 0;
    if (box_b) {  // voxel brick box: hi < lo
      const short4 a = box_a[i];
      box_b[i] = make_short4((short)(a.x - 1), (short)(a.y - 1), (short)(a.z - 1), 0);
    } else {
      box_a[i] = make_short4(1, 0, 1, 0);  // raster rect: tx1 < tx0
    }
  }
}
__global__ void __launch_bounds__(256) bin_apply_kernel(int32_t* __restrict__ H, const int32_t* __restrict__ seg,
                                                        const int32_t* __restrict__ tile_base, int n_rows, int T) {
  pdl_prologue();
  const int t = blockIdx.x * blockDim.x + threadIdx.x, g = blockIdx.y;
  if (t >= T) return;
  const int r0 = g * kSegRows, r1 = min(n_rows, r0 + kSegRows);
  int32_t run = tile_base[t] + seg[(long long)g * T + t];
  // 16 loads in flight before the in-place stores (H becomes S)
  for (int rb = r0; rb < r1; rb += 16) {
    int32_t x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = rb + k < r1 ? H[(long long)(rb + k) * T + t] : 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (rb + k < r1) H[(long long)(rb + k) * T + t] = run;
      run += x[k];
    }
  }
}

__global__ void __launch_bounds__(32 * kBinWarps) bin_scatter_kernel(const short4* __restrict__ rect,
                                                                     const short4* __restrict__ hi, long long m,
                                                                     int chunk, int T, int tiles_x, int tiles_y,
                                                                     int tiles_z, const int32_t* __restrict__ S,
                                                                     int32_t* __restrict__ vals, uint32_t cap,
                                                                     int v_off) {
  pdl_prologue();
  extern __shared__ uint32_t sm[];
  uint32_t* cnt = sm;                              // [kBinWarps][T]
  uint32_t* colm = sm + kBinWarps * T;             // [kBinWarps][tiles_x]
  uint32_t* rowm = colm + kBinWarps * tiles_x;     // [kBinWarps][tiles_y]
  uint32_t* laym = rowm + kBinWarps * tiles_y;     // [kBinWarps][tiles_z]
  short4* sbox = reinterpret_cast<short4*>(laym + kBinWarps * tiles_z);  // [chunk][2] the block's boxes
  const int c = blockIdx.x, v = blockIdx.y + v_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long i0 = (long long)v * m + (long long)c * chunk;
  const long long i1 = (long long)v * m + min((long long)(c + 1) * chunk, m);
  const long long per = (((i1 - i0) + kBinWarps * 32 - 1) / (kBinWarps * 32)) * 32;  // items per warp
  const long long w0 = i0 + warp * per, w1 = min(w0 + per, i1);
  uint32_t* mycnt = cnt + warp * T;
  uint32_t* mycol = colm + warp * tiles_x;
  uint32_t* myrow = rowm + warp * tiles_y;
  uint32_t* mylay = laym + warp * tiles_z;
  for (int t = threadIdx.x; t < kBinWarps * T; t += blockDim.x) cnt[t] = 0;
  __syncthreads();
  // phase A: per-warp tile counts; the boxes are kept in shared memory for
  // phase C (four loads in flight per lane)
  for (long long i = w0 + lane; i < w1; i += 4 * 32) {
    Box r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) r[k] = load_box(rect, hi, i + 32 * k, i + 32 * k < w1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i + 32 * k >= w1) continue;
      if (SCT_SCATTER_SBOX) {
        sbox[2 * (i + 32 * k - i0)] = make_short4(r[k].x0, r[k].x1, r[k].y0, r[k].y1);
        sbox[2 * (i + 32 * k - i0) + 1] = make_short4(r[k].z0, r[k].z1, 0, 0);
      }
      if (box_empty(r[k])) continue;
      for (int tz = r[k].z0; tz <= r[k].z1; ++tz)
        for (int ty = r[k].y0; ty <= r[k].y1; ++ty)
          for (int tx = r[k].x0; tx <= r[k].x1; ++tx)
            atomicAdd(&mycnt[(tz * tiles_y + ty) * tiles_x + tx], 1u);
    }
  }
  __syncthreads();
  // phase B: per tile, the block's global start plus the earlier warps' counts
  const int32_t* sb = S + ((long long)v * gridDim.x + c) * T;  // gridDim.x = chunks
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    uint32_t run = (uint32_t)sb[t];
#pragma unroll
    for (int w = 0; w < kBinWarps; ++w) {
      const uint32_t x = cnt[w * T + t];
      cnt[w * T + t] = run;
      run += x;
    }
  }
  __syncthreads();
  // phase C: rounds of 32 items in item order; a box is the product of a
  // column, a row and a layer range, so the stable rank of a pair among the
  // round's earlier items is popc(colmask & rowmask & layermask & lanes_below)
  const uint32_t below = (1u << lane) - 1u;
  for (long long base = w0; base < w1; base += 32) {
    const long long i = base + lane;
    Box r{0, -1, 0, -1, 0, -1};
    if (SCT_SCATTER_SBOX) {
      if (i < w1) {
        const short4 p = sbox[2 * (i - i0)], q = sbox[2 * (i - i0) + 1];
        r = Box{p.x, p.y, p.z, p.w, q.x, q.y};
      }
    } else {
      r = load_box(rect, hi, i, i < w1);
    }
    for (int k = lane; k < tiles_x; k += 32) mycol[k] = 0;
    for (int k = lane; k < tiles_y; k += 32) myrow[k] = 0;
    for (int k = lane; k < tiles_z; k += 32) mylay[k] = 0;
    __syncwarp();
    const uint32_t bit = 1u << lane;
    const bool any = !box_empty(r);
    if (any) {
      for (int tx = r.x0; tx <= r.x1; ++tx) atomicOr(&mycol[tx], bit);
      for (int ty = r.y0; ty <= r.y1; ++ty) atomicOr(&myrow[ty], bit);
      for (int tz = r.z0; tz <= r.z1; ++tz) atomicOr(&mylay[tz], bit);
    }
    __syncwarp();
    if (any) {
      for (int tz = r.z0; tz <= r.z1; ++tz) {
        const uint32_t lm = mylay[tz] & below;
        for (int ty = r.y0; ty <= r.y1; ++ty) {
          const uint32_t rm = myrow[ty] & lm;
          for (int tx = r.x0; tx <= r.x1; ++tx) {
            const int t = (tz * tiles_y + ty) * tiles_x + tx;
            const uint32_t pos = mycnt[t] + __popc(mycol[tx] & rm);
            if (pos < cap) vals[pos] = (int32_t)i;  // beyond: capacity overflow (flagged by bin_tilebase)
          }
        }
      }
    }
    __syncwarp();
    if (any)
      for (int tz = r.z0; tz <= r.z1; ++tz)
        for (int ty = r.y0; ty <= r.y1; ++ty)
          for (int tx = r.x0; tx <= r.x1; ++tx) atomicAdd(&mycnt[(tz * tiles_y + ty) * tiles_x + tx], 1u);
    __syncwarp();
  }
}

// (view, tile) list = [S[v][0][t], S[v+1][0][t]) with S[V][0][t] = the next tile's
// base (tile_base[t + 1]).
__global__ void __launch_bounds__(256) bin_ranges_kernel(const int32_t* __restrict__ S,
                                                         const int32_t* __restrict__ tile_base, int n_chunks,
                                                         int n_views, int T, int2* __restrict__ ranges,
                                                         long long cap) {
  pdl_prologue();
  const long long n = (long long)n_views * T;
  // capacity overflow (flagged by the column scan): empty lists, so nothing
  // downstream reads past the cap-sized pair buffer
  const bool over = (long long)tile_base[T] > cap;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(k / T), t = (int)(k % T);
    const int32_t a = S[(long long)v * n_chunks * T + t];
    const int32_t b = v + 1 < n_views ? S[(long long)(v + 1) * n_chunks * T + t] : tile_base[t + 1];
    SCT_DCHECK(over || (0 <= a && a <= b && b <= tile_base[T]));
    ranges[k] = over ? make_int2(0, 0) : make_int2(a, b);
  }
}

// (view, tile) ranges of the sorted raster pairs: tile from the key, view
// from the item (item = view * m + kernel; quotient by a float reciprocal
// with an exact integer correction). Pair p closes the range at p and opens
// the one at p + 1 when the slot changes.
__device__ __forceinline__ int div_m(int x, int m, float inv_m) {
  int q = (int)((float)x * inv_m);
  if ((long long)q * m > x) --q;
  if ((long long)(q + 1) * m <= x) ++q;
  return q;
}
// Eight consecutive pairs per thread (16/32-byte vector loads of the keys
// and items, the next group's first pair for the closing test), so each
// thread has several loads in flight: the scalar form was latency-bound at a
// quarter of the HBM rate.
template <typename KeyT>
__global__ void __launch_bounds__(256) raster_ranges_kernel(long long n_pairs, const KeyT* __restrict__ keys,
                                                            const int32_t* __restrict__ vals, int m, float inv_m,
                                                            long long tiles_per_view, int2* __restrict__ ranges) {
  pdl_prologue();
  const long long groups = (n_pairs + 7) / 8;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < groups;
       g += (long long)gridDim.x * blockDim.x) {
    const long long p0 = 8 * g;
    KeyT k[9];
    int32_t v[9];
    if (p0 + 8 <= n_pairs) {
      if (sizeof(KeyT) == 2) {
        const uint4 kv = *reinterpret_cast<const uint4*>(keys + p0);
        const uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          k[2 * i] = (KeyT)(w[i] & 0xffffu);
          k[2 * i + 1] = (KeyT)(w[i] >> 16);
        }
      } else {
        const uint4 k0 = *reinterpret_cast<const uint4*>(keys + p0);
        const uint4 k1 = *reinterpret_cast<const uint4*>(keys + p0 + 4);
        k[0] = (KeyT)k0.x, k[1] = (KeyT)k0.y, k[2] = (KeyT)k0.z, k[3] = (KeyT)k0.w;
        k[4] = (KeyT)k1.x, k[5] = (KeyT)k1.y, k[6] = (KeyT)k1.z, k[7] = (KeyT)k1.w;
      }
      const int4 v0 = *reinterpret_cast<const int4*>(vals + p0);
      const int4 v1 = *reinterpret_cast<const int4*>(vals + p0 + 4);
      v[0] = v0.x, v[1] = v0.y, v[2] = v0.z, v[3] = v0.w;
      v[4] = v1.x, v[5] = v1.y, v[6] = v1.z, v[7] = v1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        k[i] = p0 + i < n_pairs ? keys[p0 + i] : (KeyT)0;
        v[i] = p0 + i < n_pairs ? vals[p0 + i] : 0;
      }
    }
    const bool has_next = p0 + 8 < n_pairs;
    k[8] = has_next ? keys[p0 + 8] : (KeyT)0;
    v[8] = has_next ? vals[p0 + 8] : 0;
    long long slot[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) slot[i] = (long long)div_m(v[i], m, inv_m) * tiles_per_view + k[i];
    if (p0 == 0) ranges[slot[0]].x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const long long p = p0 + i;
      if (p >= n_pairs) break;
      if (p == n_pairs - 1) {
        ranges[slot[i]].y = (int)n_pairs;
      } else if (slot[i + 1] != slot[i]) {
        ranges[slot[i]].y = (int)(p + 1);
        ranges[slot[i + 1]].x = (int)(p + 1);
      }
    }
  }
}

// Gaussian-pixel evaluation along a run of 4 pixels of one row.
// The exponent is carried with a +64 offset: E' = 2^(L + 64), L <= 0, so one
// MUFU.EX2 gives the first pixel and one more the ratio to the next pixel,
// R = 2^(L(dx+1) - L(dx)) = 2^(2A dx + A + B dy); later ratios follow from
// R *= K, K = 2^(2A). Two MUFU per 4 GPE instead of four. The ratio argument
// is clamped at 126: when it would exceed that, L(dx) < -126 already and every
// pixel value it could feed is below 2^-29 of the amplitude;
// likewise a run whose first E' flushes to zero (L < -190) only holds values
// below 2^-29 * amp. The amplitude (records) or upstream gradient (backward)
// carries the matching 2^-64.
struct Run4 {
  float e0, e1, e2, e3;
};
__device__ __forceinline__ Run4 run4(float dx, float A, float A2, float bdy, float apb, float cdy2o, float K) {
  const float t = fmaf(A, dx, bdy);
  const float L = fmaf(dx, t, cdy2o);
  const float D = fmaf(A2, dx, apb);
  float E = ex2(L);
  float R = ex2(fminf(D, 126.f));
  Run4 r;
  r.e0 = E;
  E *= R;
  R *= K;
  r.e1 = E;
  E *= R;
  R *= K;
  r.e2 = E;
  r.e3 = E * R;
  return r;
}

// Eight pixels from one pair of MUFU ops (run8x2 below; 19 instead of 22 + 1
// instructions for two 4-runs). Along a row L(x) = -a (x - x*)^2 + L*, a = |A|;
// a pixel that matters (L >= -24: 2^-24 of the kernel's amplitude) sits within
// sqrt(24 / a) of x*, so the run's first pixel is at most 49 a + 14 sqrt(24 a)
// below it. It must stay above the ftz floor: -190 with K3's +64 offset
// (a <= 1.6); narrower kernels take two 4-runs (a warp-uniform branch in K3).
constexpr float kRun8MaxA_K3 = 1.5f;

// Narrow kernels (rasterizer.cpp:44-50,151 with a small or zero low-pass:
// projected sigma below ~0.25 px) fall by orders of magnitude between
// neighbouring pixels, and a 4-run's recurrence can lose its peak: a pixel p
// that matters (L(p) >= -T, 2^-T of the amplitude) has a run head with
// L(first) >= -T - 9a - 6 sqrt(T a), which must stay above the ftz floor
// (-190 with K3's +64 offset, T = 24; -141 with K4's +15, T = 10). That holds
// for a = |A| <= 8.5 (K3) and <= 8.25 (K4); the default 0.3 px low-pass keeps
// a <= 0.5 log2(e) / 0.09 = 8.01. Beyond those bounds the kernels take a
// direct evaluation, one MUFU.EX2 per pixel (warp-uniform branch).
constexpr float kRun4MaxA_K3 = 8.5f;
constexpr float kRun4MaxA_K4 = 8.25f;

// Direct evaluation of 8 consecutive pixels of a row for two kernels:
// E(dx + k) = 2^(L(dx + k)), L = (A x + B dy) x + (C dy^2 + offset).
__device__ __forceinline__ void direct8x2(float2 e[8], float2 dx, float2 A, float2 bdy, float2 cdy2o) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float2 x = __fadd2_rn(dx, make_float2((float)k, (float)k));
    const float2 L = __ffma2_rn(x, __ffma2_rn(A, x, bdy), cdy2o);
    e[k] = make_float2(ex2(L.x), ex2(L.y));
  }
}

// Two kernels at once in packed FP32x2 arithmetic (FFMA2 / FMUL2 / FADD2 on
// sm_100): element i of every float2 belongs to kernel i of the pair and is
// computed with exactly the scalar path's operations and rounding (run4's; an
// 8-run continues the same recurrence); one instruction issues both.
__device__ __forceinline__ void run4x2(float2 e[4], float2 dx, float2 A, float2 A2, float2 bdy, float2 apb,
                                       float2 cdy2o, float2 K) {
  const float2 t = __ffma2_rn(A, dx, bdy);
  const float2 L = __ffma2_rn(dx, t, cdy2o);
  const float2 D = __ffma2_rn(A2, dx, apb);
  float2 E = make_float2(ex2(L.x), ex2(L.y));
  float2 R = make_float2(ex2(fminf(D.x, 126.f)), ex2(fminf(D.y, 126.f)));
  e[0] = E;
  E = __fmul2_rn(E, R);
  R = __fmul2_rn(R, K);
  e[1] = E;
  E = __fmul2_rn(E, R);
  R = __fmul2_rn(R, K);
  e[2] = E;
  e[3] = __fmul2_rn(E, R);
}

__device__ __forceinline__ void run8x2(float2 e[8], float2 dx, float2 A, float2 A2, float2 bdy, float2 apb,
                                       float2 cdy2o, float2 K) {
  const float2 t = __ffma2_rn(A, dx, bdy);
  const float2 L = __ffma2_rn(dx, t, cdy2o);
  const float2 D = __ffma2_rn(A2, dx, apb);
  float2 E = make_float2(ex2(L.x), ex2(L.y));
  float2 R = make_float2(ex2(fminf(D.x, 126.f)), ex2(fminf(D.y, 126.f)));
  e[0] = E;
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    E = __fmul2_rn(E, R);
    if (k < 7) R = __fmul2_rn(R, K);
    e[k] = E;
  }
}

// K3: one warp per work item = one part of one (view, tile) list; lane = 1
// row x 8 columns (two 4-pixel runs sharing the per-row setup). Lists longer
// than kPart kernels are cut into parts of kPart (K3Work): every work item is
// short, so the persistent warps stay balanced and finish the items in claim
// order (which the host-buffer path relies on to publish view units early).
// A one-part list is accumulated straight into the image; a part of a longer
// list writes its 16x16 partial tile, and the last part to finish sums the
// parts in part order (fixed, so the result does not depend on timing) and
// writes the image tile. Persistent: each warp takes the next item from a
// global counter and stages the list through shared memory 32 records at a
// time (one coalesced gather per lane), synchronising only itself; the next
// chunk's records are fetched while the current chunk is evaluated.
constexpr int kCompWarps = 4;
__global__ void __launch_bounds__(32 * kCompWarps) composite_kernel(
    const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    int tiles_x, int tiles_per_view, int W, int H, const int4* __restrict__ items, const int* __restrict__ n_items,
    int part_len, int* __restrict__ work, int* __restrict__ tile_cnt, float* __restrict__ partial,
    float* __restrict__ images, UnitSync us, const int* __restrict__ item_lo, const int* __restrict__ item_hi) {
  pdl_prologue();
  // a chunk's 32 records as 16 kernel pairs, fields interleaved so that one
  // LDS.128 yields two float2 operands: [pair][0] = (cx0, cx1, cy0, cy1),
  // [1] = (amp0, amp1, K0, K1), [2] = (A0, A1, B0, B1), [3] = (C0, C1, 2A0, 2A1)
  __shared__ float4 sp[kCompWarps][16][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = lane >> 1;
  // the items [lo, hi): all of them, or one view part of the host path
  const int lo = item_lo ? *item_lo : 0;
  const int total = item_hi ? *item_hi : *n_items;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(work, 1) + lo;
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= total) break;
    const int4 it = items[c];  // (view * T + tile, part, parts, first item of the list)
    SCT_DCHECK(c >= 0 && it.x >= 0 && it.y >= 0 && it.y < it.z && it.w >= 0 && it.w <= c);
    if (us.stamp && lane == 0) atomicMin(us.stamp + Ctx::kMaxUnits, (unsigned long long)global_ns());
    const int w = it.x, part = it.y, parts = it.z;
    const int view = w / tiles_per_view;
    const int tile = w % tiles_per_view;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int u0 = tx * kTilePx + (lane & 1) * 8;
    const int v = ty * kTilePx + row;
    const float py = (float)v + 0.5f;
    const float px0 = (float)u0 + 0.5f;
    int2 rg = ranges[w];
    SCT_DCHECK(0 <= rg.x && rg.x <= rg.y);
    rg.x += part * part_len;
    rg.y = min(rg.y, rg.x + part_len);
    SCT_DCHECK(rg.x <= rg.y);
    // even and odd kernels of the list accumulate in the two halves of acc2
    float2 acc2[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc2[k] = make_float2(0.f, 0.f);
    float4 na = make_float4(0.f, 0.f, 0.f, 0.f), nb = na;  // past the list: amplitude 0
    if (rg.x + lane < rg.y) {
      const long long item = vals[rg.x + lane];
      SCT_DCHECK(item >= 0);
      na = __ldg(rec + 2 * item);
      nb = __ldg(rec + 2 * item + 1);
    }
    const float2 py2 = make_float2(py, py), px2 = make_float2(px0, px0);
    const float2 c64 = make_float2(64.f, 64.f), neg = make_float2(-1.f, -1.f);
    for (int base = rg.x; base < rg.y; base += 32) {
      const int n = min(32, rg.y - base);
      __syncwarp();
      {
        float* d = reinterpret_cast<float*>(&sp[warp][lane >> 1][0]) + (lane & 1);
        d[0] = na.x;  d[2] = na.y;  d[4] = na.z;  d[6] = na.w;
        d[8] = nb.x;  d[10] = nb.y; d[12] = nb.z; d[14] = nb.w;
      }
      __syncwarp();
      na = make_float4(0.f, 0.f, 0.f, 0.f);
      nb = na;
      if (base + 32 + lane < rg.y) {  // prefetch the next chunk
        const long long item = vals[base + 32 + lane];
        na = __ldg(rec + 2 * item);
        nb = __ldg(rec + 2 * item + 1);
      }
#pragma unroll 8
      for (int j = 0; j < (n + 1) >> 1; ++j) {  // an odd list's last pair has a zero-amplitude twin
        const float4 p0 = sp[warp][j][0], p1 = sp[warp][j][1], p2 = sp[warp][j][2], p3 = sp[warp][j][3];
        const float2 cx = make_float2(p0.x, p0.y), cy = make_float2(p0.z, p0.w);
        const float2 amp = make_float2(p1.x, p1.y), K = make_float2(p1.z, p1.w);
        const float2 A = make_float2(p2.x, p2.y), B = make_float2(p2.z, p2.w);
        const float2 Cc = make_float2(p3.x, p3.y), A2 = make_float2(p3.z, p3.w);
        const float2 dy = __ffma2_rn(neg, cy, py2);  // py - cy
        const float2 bdy = __fmul2_rn(B, dy);
        const float2 apb = __fadd2_rn(A, bdy);
        const float2 cdy2o = __ffma2_rn(__fmul2_rn(Cc, dy), dy, c64);
        const float2 dx = __ffma2_rn(neg, cx, px2);  // px0 - cx
        float2 e[8];
        const float amax = fmaxf(fabsf(A.x), fabsf(A.y));  // warp-uniform: one kernel pair per step
        if (amax <= kRun8MaxA_K3) {
          run8x2(e, dx, A, A2, bdy, apb, cdy2o, K);
        } else if (amax <= kRun4MaxA_K3) {
          run4x2(e, dx, A, A2, bdy, apb, cdy2o, K);
          run4x2(e + 4, __fadd2_rn(dx, make_float2(4.f, 4.f)), A, A2, bdy, apb, cdy2o, K);
        } else {
          direct8x2(e, dx, A, bdy, cdy2o);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc2[k] = __ffma2_rn(amp, e[k], acc2[k]);
      }
    }
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = acc2[k].x + acc2[k].y;
    if (parts > 1) {
      // partial tile of this part (lane: row, 8 columns), then the last part sums all parts in order
      float4* mine = reinterpret_cast<float4*>(partial + (long long)(it.w + part) * 256) + 2 * lane;
      mine[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      mine[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      __threadfence();
      __syncwarp();
      int done = 0;
      if (lane == 0) {
        const int old = atomicAdd(tile_cnt + it.w, 1);
        SCT_DCHECK(old < parts);  // each part of the list counts once; the last one resets
        done = old == parts - 1;
        if (done) tile_cnt[it.w] = 0;  // ready for the next launch
      }
      done = __shfl_sync(0xffffffffu, done, 0);
      if (!done) continue;
      __threadfence();
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.f;
      for (int q = 0; q < parts; ++q) {
        const float4* src = reinterpret_cast<const float4*>(partial + (long long)(it.w + q) * 256) + 2 * lane;
        const float4 p0 = __ldcg(src), p1 = __ldcg(src + 1);
        acc[0] += p0.x;
        acc[1] += p0.y;
        acc[2] += p0.z;
        acc[3] += p0.w;
        acc[4] += p1.x;
        acc[5] += p1.y;
        acc[6] += p1.z;
        acc[7] += p1.w;
      }
    }
    if (v < H) {
      float* out = images + ((long long)view * H + v) * W;
      if (u0 + 7 < W && (W & 3) == 0) {
        *reinterpret_cast<float4*>(out + u0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4*>(out + u0 + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (u0 + k < W) out[u0 + k] = acc[k];
      }
    }
    if (us.done) {  // host path: publish the view unit once all its tiles are written
      __threadfence();
      __syncwarp();
      if (lane == 0) unit_signal(us, unit_of_view(view, us.n_views, us.units));
    }
  }
}

// Work items of K3 in the given (view, tile) order: list i of length n gets
// max(1, ceil(n / part_len)) consecutive items (exclusive scan `first`).
__global__ void __launch_bounds__(256) k3_parts_kernel(const int2* __restrict__ ranges, const int* __restrict__ order,
                                                       int n, int part_len, int* __restrict__ count) {
  pdl_prologue();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int2 r = ranges[order[i]];
    count[i] = max(1, (r.y - r.x + part_len - 1) / part_len);
  }
}

// k3_parts + the scan in one CTA, for small list counts (n <= kSmallWork; the
// train step and 8-rank shards): thread t takes the lists [t * per, (t + 1) *
// per) of the order in two passes (part counts, then after the block scan the
// first item of each list). The items themselves are written by the
// multi-CTA k3_items_kernel: from one SM the scattered 16-byte item stores
// were the bottleneck (34 us for the 10-view shard's 26k items).
constexpr int kSmallWorkThreads = 1024, kSmallWork = 16 * kSmallWorkThreads;
__global__ void __launch_bounds__(kSmallWorkThreads) k3_first_small_kernel(const int2* __restrict__ ranges,
                                                                           const int* __restrict__ order, int n,
                                                                           int part_len, int* __restrict__ count,
                                                                           int* __restrict__ first) {
  pdl_prologue();
  using Scan = cub::BlockScan<int, kSmallWorkThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int per = (n + kSmallWorkThreads - 1) / kSmallWorkThreads;
  const int i0 = min(n, (int)threadIdx.x * per), i1 = min(n, i0 + per);
  auto parts_of = [&](int w) {
    const int2 r = ranges[w];
    return max(1, (r.y - r.x + part_len - 1) / part_len);
  };
  int mine = 0;
#pragma unroll 4
  for (int i = i0; i < i1; ++i) {
    const int k = parts_of(order[i]);
    count[i] = k;
    mine += k;
  }
  int f = 0;
  Scan(tmp).ExclusiveSum(mine, f);
  for (int i = i0; i < i1; ++i) {
    first[i] = f;
    f += count[i];
  }
}

// K3 work items for larger list counts in two multi-CTA passes (replacing
// k3_parts + CUB's two-kernel scan + k3_items): per 1024-list block the part
// counts and their sum, then each block's base (the earlier blocks' sums), a
// block scan, the lists' first items and the items themselves.
constexpr int kK3Block = 1024;
__global__ void __launch_bounds__(kK3Block) k3_block_parts_kernel(const int2* __restrict__ ranges,
                                                                  const int* __restrict__ order, int n, int part_len,
                                                                  int* __restrict__ count, int* __restrict__ bsum) {
  pdl_prologue();
  using Reduce = cub::BlockReduce<int, kK3Block>;
  __shared__ typename Reduce::TempStorage tmp;
  const int i = blockIdx.x * kK3Block + threadIdx.x;
  int k = 0;
  if (i < n) {
    const int2 r = ranges[order[i]];
    k = max(1, (r.y - r.x + part_len - 1) / part_len);
    count[i] = k;
  }
  const int sum = Reduce(tmp).Sum(k);
  if (threadIdx.x == 0) bsum[blockIdx.x] = sum;
}
__global__ void __launch_bounds__(kK3Block) k3_block_items_kernel(const int* __restrict__ order,
                                                                  const int* __restrict__ count, int n,
                                                                  const int* __restrict__ bsum, int* __restrict__ first,
                                                                  int4* __restrict__ items, int* __restrict__ n_items,
                                                                  int* __restrict__ tile_cnt, long long max_items) {
  pdl_prologue();
  using Scan = cub::BlockScan<int, kK3Block>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  if (threadIdx.x < 32) {  // sum of the earlier blocks (fixed order: lane-strided, then a shuffle tree)
    int b = 0;
    for (int j = threadIdx.x; j < (int)blockIdx.x; j += 32) b += bsum[j];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if (threadIdx.x == 0) s_base = b;
  }
  const int i = blockIdx.x * kK3Block + threadIdx.x;
  const int k = i < n ? count[i] : 0;
  int f = 0;
  Scan(tmp).ExclusiveSum(k, f);
  __syncthreads();
  f += s_base;
  if (i < n) {
    const int w = order[i];
    first[i] = f;
    for (int p = 0; p < k; ++p) items[f + p] = make_int4(w, p, k, f);
    if (i == n - 1) *n_items = f + k;
  }
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < max_items;
       j += (long long)gridDim.x * blockDim.x)
    tile_cnt[j] = 0;
}

// the items of every list, and the reset of K3's per-item tile counters
__global__ void __launch_bounds__(256) k3_items_kernel(const int* __restrict__ order, const int* __restrict__ count,
                                                       const int* __restrict__ first, int n,
                                                       int4* __restrict__ items, int* __restrict__ n_items,
                                                       int* __restrict__ tile_cnt, long long max_items) {
  pdl_prologue();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int)stride) {
    const int k = count[i], f = first[i], w = order[i];
    for (int p = 0; p < k; ++p) items[f + p] = make_int4(w, p, k, f);
    if (i == n - 1) *n_items = f + k;
  }
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < max_items; j += stride) tile_cnt[j] = 0;
}

// K4: Gaussian-major backward statistics. One 256-thread CTA per non-empty
// (tile, view). Eight lanes share a Gaussian; lane s owns pixel rows s and
// s+8 with their upstream gradient in registers, so per pixel the work is the
// run4 exponential plus three FMAs accumulating column moments
// R0 = sum g E, R1 = sum g E c', R2 = sum g E c'^2 (c' = column - 7.5); the
// row's s0, s1, s2 follow from them. The 8 lanes' partial statistics are
// combined with a 3-step shuffle reduce-scatter (7 shuffles for 6 values) and
// lanes 0..5 write the (tile, Gaussian) pair's 6 values as one 32-byte sector
// into the pair's slot (item scan offset + rank of this tile in its
// rectangle). The chain kernel reduces slots in the reference's fixed tile
// order (rasterizer.cpp:245-257): deterministic, no atomics.
constexpr int kBwdThreads = 256;
__global__ void __launch_bounds__(kBwdThreads, 4) backward_stats_kernel(
    const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    const short4* __restrict__ rect, const int32_t* __restrict__ offset, int tiles_x, int tiles_per_view, int W,
    int H, int view0, const float* __restrict__ dL, float* __restrict__ pair_stats, float* __restrict__ item_stats) {
  pdl_prologue();
  const int tile = blockIdx.x;
  const int view = view0 + blockIdx.y;
  const int2 rg = ranges[(long long)view * tiles_per_view + tile];
  if (rg.y <= rg.x) return;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int s = threadIdx.x & 7;
  const int group = threadIdx.x >> 3;
  const int u0 = tx * kTilePx;
  float g[2][kTilePx];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int v = ty * kTilePx + s + 8 * r;
    const float* drow = dL + ((long long)view * H + v) * W + u0;
#pragma unroll
    for (int c = 0; c < kTilePx; ++c) g[r][c] = (v < H && u0 + c < W) ? __ldg(drow + c) * 0x1p-64f : 0.f;
  }
  const float py0 = (float)(ty * kTilePx + s) + 0.5f;
  const float px0 = (float)u0 + 0.5f;
  const bool b2 = s & 4, b1 = s & 2, b0 = s & 1;
  // The tile list is processed in chunks of kBwdChunk entries (item indices
  // loaded coalesced into shared memory), 32 kernels per pass. Warp 0 stages
  // the NEXT pass's records, rectangles and scan offsets with cp.async
  // (global -> shared, no registers held) while all warps evaluate the
  // current pass from the other buffer.
  constexpr int kPass = kBwdThreads / 8;  // kernels per pass
  __shared__ int s_items[kBwdChunk];
  __shared__ float4 s_rec[2][kPass][2];
  __shared__ short4 s_rect[2][kPass];
  __shared__ int s_off[2][kPass];
  const int tid = threadIdx.x;
  const int n_list = rg.y - rg.x;
  auto stage = [&](int buf, int p, int cn) {  // called by warp 0 only
    const int e = p * kPass + tid;
    if (e < cn) {
      const long long it = s_items[e];
      cp_async16(&s_rec[buf][tid][0], rec + 2 * it);
      cp_async16(&s_rec[buf][tid][1], rec + 2 * it + 1);
      cp_async8(&s_rect[buf][tid], rect + it);
      cp_async4(&s_off[buf][tid], offset + it);
    }
    cp_async_commit();
  };
  for (int cb = 0; cb < n_list; cb += kBwdChunk) {
    const int cn = min(kBwdChunk, n_list - cb);
    __syncthreads();  // previous chunk finished with s_items / buffers
    if (tid < cn) s_items[tid] = vals[rg.x + cb + tid];
    __syncthreads();
    if (tid < 32) {
      stage(0, 0, cn);
      cp_async_wait_all();
    }
    __syncthreads();
    const int npass = (cn + kPass - 1) / kPass;
  for (int p = 0; p < npass; ++p) {
    if (tid < 32 && p + 1 < npass) stage((p + 1) & 1, p + 1, cn);
    const int buf = p & 1;
    const bool valid = p * kPass + group < cn;
    float st[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) st[k] = 0.f;
    if (valid) {
      const float4 a = s_rec[buf][group][0];
      const float4 b = s_rec[buf][group][1];
      const float dx0 = px0 - a.x;
      const float dxm = dx0 + 7.5f;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float dy = py0 + 8.f * r - a.y;
        const float bdy = b.y * dy;
        const float apb = b.x + bdy;
        const float cdy2o = fmaf(b.z * dy, dy, 64.f);
        // Columns c and 15-c have opposite c' = c - 7.5, so with s = F_c + F_15-c
        // and d = F_c - F_15-c (F = g E): R0 += s, R1 += c' d, R2 += c'^2 s —
        // 7 instead of 8 ops per column pair. Runs 0/3 and 1/2 are paired.
        float R0 = 0.f, R1 = 0.f, R2 = 0.f;
        const bool narrow = fabsf(b.x) > kRun4MaxA_K4;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          Run4 lo, hi;
          if (!narrow) {
            lo = run4(dx0 + 4.f * q, b.x, b.w, bdy, apb, cdy2o, a.w);
            hi = run4(dx0 + 4.f * (3 - q), b.x, b.w, bdy, apb, cdy2o, a.w);
          } else {  // direct evaluation (see kRun4MaxA_K4)
            float ev[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float xl = dx0 + (float)(4 * q + k), xh = dx0 + (float)(4 * (3 - q) + k);
              ev[k] = ex2(fmaf(xl, fmaf(b.x, xl, bdy), cdy2o));
              ev[4 + k] = ex2(fmaf(xh, fmaf(b.x, xh, bdy), cdy2o));
            }
            lo = Run4{ev[0], ev[1], ev[2], ev[3]};
            hi = Run4{ev[4], ev[5], ev[6], ev[7]};
          }
          const float el[4] = {lo.e0, lo.e1, lo.e2, lo.e3};
          const float eh[4] = {hi.e0, hi.e1, hi.e2, hi.e3};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int c = 4 * q + k;           // 0..7
            const float cp = (float)c - 7.5f;  // c' of column c; column 15-c has -c'
            const float fa = g[r][c] * el[k];
            const float fb = g[r][15 - c] * eh[3 - k];
            const float s = fa + fb;
            R0 += s;
            R1 = fmaf(fa - fb, cp, R1);
            R2 = fmaf(s, cp * cp, R2);
          }
        }
        // sum ge dx = dxm R0 + R1, sum ge dx^2 = dxm^2 R0 + 2 dxm R1 + R2
        const float rx = fmaf(dxm, R0, R1);
        const float rxx = fmaf(dxm, fmaf(dxm, R0, 2.f * R1), R2);
        st[0] += R0;                      // s0
        st[1] += rx;                      // s1.x
        st[2] = fmaf(dy, R0, st[2]);      // s1.y
        st[3] += rxx;                     // s2.xx
        st[4] = fmaf(dy * dy, R0, st[4]); // s2.yy
        st[5] = fmaf(dy, rx, st[5]);      // s2.xy
      }
    }
    // reduce-scatter over the 8 lanes of the group: lane s ends with total[s]
    float w[4], x[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float send = b2 ? st[k] : st[k + 4];
      const float keep = b2 ? st[k + 4] : st[k];
      w[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float send = b1 ? w[k] : w[k + 2];
      const float keep = b1 ? w[k + 2] : w[k];
      x[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    const float send = b0 ? x[0] : x[1];
    const float keep = b0 ? x[1] : x[0];
    const float tot = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    if (valid && s < 6) {
      if (item_stats) {
        // parallel-atomic mode: the shuffle-reduced pair
        // statistics go straight into the item's 6 accumulators
        atomicAdd(item_stats + 8 * (long long)s_items[p * kPass + group] + s, tot);
      } else {
        const short4 r = s_rect[buf][group];
        const int slot = s_off[buf][group] + (ty - r.z) * (r.y - r.x + 1) + (tx - r.x);
        pair_stats[8 * (long long)slot + s] = tot;
      }
    }
    if (tid < 32) cp_async_wait_all();
    __syncthreads();  // next buffer visible; this buffer free for re-staging
  }
  }
}

// ---------------------------------------------------------------------------
// K4 (tensor-core form). The six statistics of a (tile, kernel) pair are
// linear in the upstream gradient: with tile-centred pixel offsets
// c' = col - 7.5, r' = row - 7.5 and the kernel's offset (ox, oy) = tile centre
// - projected centre, dx = c' + ox and dy = r' + oy, so
//   s0 = M0, s1x = M1 + ox M0, s1y = M2 + oy M0, s2xx = M3 + 2 ox M1 + ox^2 M0,
//   s2yy = M4 + 2 oy M2 + oy^2 M0, s2xy = M5 + ox M2 + oy M1 + ox oy M0,
// where M = E G: E[kernel][pixel] = exp(-1/2 d^T Q d) and
// G[pixel][n] = g(pixel) * {1, c', r', c'^2, r'^2, c'r', 0, 0}. G is fixed per
// tile, so a tile list is a [list x 256] x [256 x 8] product: the SIMT lanes
// produce E with the exp2 recurrence directly in mma.m16n8k16 A-fragment
// order, and the moment accumulation plus the cross-lane reduction (about 60 %
// of the former per-pixel instructions) move onto the tensor cores.
//
// Precision: E is rounded to binary16 (it carries a +15 exponent offset, so
// it spans (0, 2^15]; values below 2^-29 of a kernel's peak lose precision
// and are negligible), G is split into hi + lo binary16 parts after a per-tile
// power-of-two scale S that puts its largest entry near 2^14, and the MMA
// accumulates in FP32. E's rounding (2^-11, zero mean) is the only error of
// note: 2e-4 relative on the gradients against the FP64 oracle (bar 1e-3).
// Measured alternatives (tools/k4_variants.sh, cfg3): FP32 SIMT 2.90 ms;
// TF32 E with split G 2.43 ms (same error); fully split TF32 3.20 ms (1e-5);
// TF32 with unsplit G 2.00 ms but 8e-3 error — the binomial shift above
// amplifies G's rounding for kernels centred outside the tile.
// mma.sync is the right instruction: the A operand is produced in registers
// (tcgen05 would need it staged through shared memory), and the tensor pipe
// is ~30 % busy — E's SIMT evaluation is the limiter.
//
// Fragment mapping (lane = 4 gq + t): lane t of a quad owns row 2q + (t >> 1),
// columns 8 (t & 1) .. +7 of row pair q, for kernels gq and gq + 8 of the
// current 16-kernel chunk. Slice s = 2q + h (k = 16 pixels) maps k = 2t, 2t+1
// to columns 8 (t & 1) + 4h + {0, 1} and k = 2t+8, 2t+9 to + {2, 3}, so the
// A fragment of a slice is one 4-pixel run per kernel. B fragments (G hi/lo)
// are built per tile in shared memory, in fragment order.
//
// One CTA of kMmaWarps warps per non-empty (view, tile): the warps share the
// tile's G and take interleaved 16-kernel chunks of the list.
// Separate accumulators for the hi and lo MMA chains, and 2 warps per CTA for
// large workloads (1.80 -> 1.77 ms at cfg3; 4 / 8 warps: 1.80 / 1.92 ms) but 4
// when lists are split into parts (small workloads: the longest lists bound
// the kernel and more warps per list finish them sooner)
#ifndef SCT_K4_WARPS
#define SCT_K4_WARPS 2
#endif
#ifndef SCT_K4_ACC2
#define SCT_K4_ACC2 1
#endif
#ifndef SCT_K4_REC16
#define SCT_K4_REC16 0
#endif
constexpr int kMmaWarpsLarge = SCT_K4_WARPS, kMmaWarpsSmall = 4;
#ifndef SCT_K4_LARGE_LISTS
#define SCT_K4_LARGE_LISTS 32768
#endif
constexpr long long kK4LargeLists = SCT_K4_LARGE_LISTS;  // (view, tile) lists from which 2-warp CTAs pay

__device__ __forceinline__ void mma_f16(float (&d)[4], __half2 a0, __half2 a1, __half2 a2, __half2 a3, uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(*reinterpret_cast<uint32_t*>(&a0)), "r"(*reinterpret_cast<uint32_t*>(&a1)),
        "r"(*reinterpret_cast<uint32_t*>(&a2)), "r"(*reinterpret_cast<uint32_t*>(&a3)), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

template <int kMmaWarps>
__global__ void __launch_bounds__(32 * kMmaWarps, 32 / kMmaWarps) backward_stats_mma_kernel(
    const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    const short4* __restrict__ rect, const int32_t* __restrict__ offset, int tiles_x, int tiles_per_view, int W,
    int H, int view0, const int* __restrict__ order, int parts, const float* __restrict__ dL,
    float* __restrict__ pair_stats,
    float* __restrict__ item_stats, UnitSync us) {
  pdl_prologue();
  __shared__ uint4 s_g[16][32];  // [slice][lane] = {hi k0-1, hi k8-9, lo k0-1, lo k8-9}
  __shared__ float s_gmax[kMmaWarps];
  // per-warp double buffer of the 16 records (and items) of a chunk, filled
  // by cp.async one chunk ahead (no registers held across the chunk's work);
  // kernels gq and gq + 8 form pair gq with their fields interleaved, so one
  // LDS.128 yields two float2 operands: [pair][0] = (cx, cx', cy, cy'),
  // [1] = (amp, amp', K, K'), [2] = (A, A', B, B'), [3] = (C, C', 2A, 2A')
  __shared__ __align__(16) float4 s_rec[kMmaWarps][2][8][4];
  __shared__ int s_it[kMmaWarps][2][16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane & 3, gq = lane >> 2;
  const float px_off = (float)(8 * (t & 1)) + 0.5f;
  const float py_off = (float)(t >> 1) + 0.5f;
  {
    const int w = order[blockIdx.x / parts];  // blocks dispatched longest lists first (tile_order)
    const int part = blockIdx.x % parts;
    const int tile = w % tiles_per_view;
    const int view = view0 + w / tiles_per_view;
    // host path: wait for this view unit's upstream gradient (H2D copy on the copy stream)
    const int unit = (us.ready || us.done) ? unit_of_view(view, us.n_views, us.units) : 0;
    if (us.ready) {
      if (threadIdx.x == 0) unit_wait(us, unit);
      __syncthreads();
    }
    int2 rg = ranges[(long long)view * tiles_per_view + tile];
    if (parts > 1) {  // small workloads: several CTAs share a list (pair statistics are independent)
      const int len = rg.y - rg.x, s0 = rg.x;
      rg.x = s0 + (int)((long long)len * part / parts);
      rg.y = s0 + (int)((long long)len * (part + 1) / parts);
    }
    SCT_DCHECK(0 <= rg.x && rg.x <= rg.y);
    if (rg.y <= rg.x) {
      if (threadIdx.x == 0) unit_signal(us, unit);
      return;
    }
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int u0 = tx * kTilePx, v0 = ty * kTilePx;
    const float* dtile = dL + ((long long)view * H + v0) * W + u0;
    // host path: the copy engine is still writing later units of dL while this
    // kernel runs, so the non-coherent (read-only for the whole kernel) path
    // must not be used for it; L2-coherent loads instead (ld.global.cg)
    const bool streamed = us.ready != nullptr;
    auto ld_dl = [streamed](const float* p) { return streamed ? __ldcg(p) : __ldg(p); };
    // --- G fragments of this tile: per-tile power-of-two scale first
    float gm = 0.f;
#pragma unroll
    for (int i = 0; i < 256 / (32 * kMmaWarps); ++i) {
      const int p = threadIdx.x + 32 * kMmaWarps * i;
      const int c = p & 15, r = p >> 4;
      if (v0 + r < H && u0 + c < W) gm = fmaxf(gm, fabsf(ld_dl(dtile + (long long)r * W + c)));
    }
    gm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(gm)));
    if (lane == 0) s_gmax[warp] = gm;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kMmaWarps; ++k) gm = fmaxf(gm, s_gmax[k]);
    // largest |G| = gm * 56.25 * 2^-15 * S <= 2^14 (the 2^-15 matches E's offset)
    const float S = gm > 0.f ? exp2f(floorf(log2f(16384.f / (gm * 56.25f * 0x1p-15f)))) : 1.f;
    const float gscale = 0x1p-15f * S, inv_s = 1.f / S;
    {
      const int n = gq;  // this lane's B column (moment)
#pragma unroll 4
      for (int s = warp; s < 16; s += kMmaWarps) {
        const int q = s >> 1, h = s & 1;
        const int r = 2 * q + (t >> 1);
        float gv[4];  // k = 2t, 2t+1, 2t+8, 2t+9 -> columns c0 + 4h + {0, 1, 2, 3}
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c = 8 * (t & 1) + 4 * h + i;
          const float g = (v0 + r < H && u0 + c < W) ? ld_dl(dtile + (long long)r * W + c) * gscale : 0.f;
          const float cp = (float)c - 7.5f, rp = (float)r - 7.5f;
          const float phi = n == 0 ? 1.f : n == 1 ? cp : n == 2 ? rp : n == 3 ? cp * cp : n == 4 ? rp * rp
                          : n == 5 ? cp * rp : 0.f;
          gv[i] = g * phi;
        }
        const __half2 h01 = __floats2half2_rn(gv[0], gv[1]), h23 = __floats2half2_rn(gv[2], gv[3]);
        const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
        s_g[s][lane] = make_uint4(h2_bits(h01), h2_bits(h23),
                                        h2_bits(__floats2half2_rn(gv[0] - f01.x, gv[1] - f01.y)),
                                        h2_bits(__floats2half2_rn(gv[2] - f23.x, gv[3] - f23.y)));
      }
    }
    __syncthreads();
    const float px0 = (float)u0 + px_off;
    const float py_base = (float)v0 + py_off;
    const int n_list = rg.y - rg.x;
    // records of a chunk: lane l copies floats 4 (l & 1) .. +3 of kernel
    // (l >> 1)'s record into its pair slot with 4-byte cp.async, one chunk
    // ahead; the item index of the chunk after that is loaded meanwhile
    // (two-deep pipeline); lane quads then read their pair gq
    constexpr int kStride = 16 * kMmaWarps;
    const int ck = lane >> 1, ch = lane & 1;
    auto load_idx = [&](int cb) {
      const int v = cb + ck < n_list ? vals[rg.x + cb + ck] : -1;
      SCT_DCHECK(cb + ck >= n_list || v >= 0);
      return v;
    };
    auto issue = [&](int buf, int it) {
#if SCT_K4_REC16
      // plain layout [kernel][2] float4: one 16-byte cp.async per lane
      float4* d16 = reinterpret_cast<float4*>(&s_rec[warp][buf][0][0]) + 2 * ck + ch;
      if (it >= 0) {
        cp_async16(d16, rec + 2 * (long long)it + ch);
      } else {
        *d16 = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (ch == 0) s_it[warp][buf][ck] = it;
      cp_async_commit();
      return;
#endif
      float* d = reinterpret_cast<float*>(&s_rec[warp][buf][ck & 7][0]) + (ck >> 3);
      if (it >= 0) {
        const float* src = reinterpret_cast<const float*>(rec + 2 * (long long)it) + 4 * ch;
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async4(d + 2 * (4 * ch + i), src + i);
      } else {  // past the list (masked by `ok`): any finite record
#pragma unroll
        for (int i = 0; i < 4; ++i) d[2 * (4 * ch + i)] = 0.f;
      }
      if (ch == 0) s_it[warp][buf][ck] = it;
      cp_async_commit();
    };
    int next_it = load_idx(16 * warp);
    issue(0, next_it);
    next_it = load_idx(16 * warp + kStride);
    int buf = 0;
    for (int cb = 16 * warp; cb < n_list; cb += kStride, buf ^= 1) {
      if (cb + kStride < n_list) {
        issue(buf ^ 1, next_it);
        next_it = load_idx(cb + 2 * kStride);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
#if SCT_K4_REC16
      const float4* rk = reinterpret_cast<const float4*>(&s_rec[warp][buf][0][0]);
      const float4 ra0 = rk[2 * gq], ra1 = rk[2 * gq + 1], rb0 = rk[2 * gq + 16], rb1 = rk[2 * gq + 17];
      const float4 f0 = make_float4(ra0.x, rb0.x, ra0.y, rb0.y), f1 = make_float4(ra0.z, rb0.z, ra0.w, rb0.w);
      const float4 f2 = make_float4(ra1.x, rb1.x, ra1.y, rb1.y), f3 = make_float4(ra1.z, rb1.z, ra1.w, rb1.w);
#else
      const float4 f0 = s_rec[warp][buf][gq][0], f1 = s_rec[warp][buf][gq][1];
      const float4 f2 = s_rec[warp][buf][gq][2], f3 = s_rec[warp][buf][gq][3];
#endif
      // kernels gq (.x) and gq + 8 (.y), evaluated together in FP32x2
      const float2 cy = make_float2(f0.z, f0.w), K = make_float2(f1.z, f1.w);
      const float2 A = make_float2(f2.x, f2.y), B = make_float2(f2.z, f2.w);
      const float2 Cc = make_float2(f3.x, f3.y), A2 = make_float2(f3.z, f3.w);
      const float2 dx = __ffma2_rn(make_float2(-1.f, -1.f), make_float2(f0.x, f0.y), make_float2(px0, px0));
      const float2 dx4 = __fadd2_rn(dx, make_float2(4.f, 4.f));
      const bool ok[2] = {cb + gq < n_list, cb + gq + 8 < n_list};
      // one 8-run per row when every kernel of the chunk is wide enough
      // (warp-uniform). With the +15 offset E' flushes below L = -141. A
      // pixel p of the run with L(p) >= -11 (2^-11 of the peak: binary16 E's
      // own rounding) has L(first) >= L(p) - 49a - 14a|p - x*| >= -11 - 49a -
      // 14 sqrt(11 a) >= -125 for a = |A| <= 1.25: no value above binary16
      // resolution is lost. (K3's +64 offset allows 1.5 at the 2^-24 level.)
      const bool r8 = __all_sync(0xffffffffu, fabsf(A.x) <= 1.25f && fabsf(A.y) <= 1.25f);
      const bool direct =
          __any_sync(0xffffffffu, fabsf(A.x) > kRun4MaxA_K4 || fabsf(A.y) > kRun4MaxA_K4);
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#if SCT_K4_ACC2
      float acc2[4] = {0.f, 0.f, 0.f, 0.f};  // the lo parts: two independent MMA chains
#else
      float (&acc2)[4] = acc;
#endif
      // the +15 exponent offset, or -1e30 for a slot past the list (E = 0)
      const float2 off = make_float2(ok[0] ? 15.f : -1e30f, ok[1] ? 15.f : -1e30f);
      // the 8 row pairs, the run mode chosen once per chunk (warp-uniform)
      auto rows = [&](auto mode) {
        constexpr int kMode = decltype(mode)::value;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float py = py_base + 2.f * q;
          const float2 dy = __ffma2_rn(make_float2(-1.f, -1.f), cy, make_float2(py, py));
          const float2 bdy = __fmul2_rn(B, dy);
          const float2 apb = __fadd2_rn(A, bdy);
          const float2 cdy2o = __ffma2_rn(__fmul2_rn(Cc, dy), dy, off);
          float2 e[8];
          if (kMode == 0) {
            run8x2(e, dx, A, A2, bdy, apb, cdy2o, K);
          } else if (kMode == 1) {
            run4x2(e, dx, A, A2, bdy, apb, cdy2o, K);
            run4x2(e + 4, dx4, A, A2, bdy, apb, cdy2o, K);
          } else {
            direct8x2(e, dx, A, bdy, cdy2o);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // two m16n8k16 slices per row pair, four pixels each
            const uint4 gb = s_g[2 * q + h][lane];
            const __half2 a0 = __floats2half2_rn(e[4 * h].x, e[4 * h + 1].x);
            const __half2 a1 = __floats2half2_rn(e[4 * h].y, e[4 * h + 1].y);
            const __half2 a2 = __floats2half2_rn(e[4 * h + 2].x, e[4 * h + 3].x);
            const __half2 a3 = __floats2half2_rn(e[4 * h + 2].y, e[4 * h + 3].y);
            mma_f16(acc, a0, a1, a2, a3, gb.x, gb.y);
            mma_f16(acc2, a0, a1, a2, a3, gb.z, gb.w);
          }
        }
      };
      if (r8) rows(std::integral_constant<int, 0>{});
      else if (!direct) rows(std::integral_constant<int, 1>{});
      else rows(std::integral_constant<int, 2>{});
#if SCT_K4_ACC2
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] += acc2[k];
#endif
      // acc: c0,c1 = moments 2t, 2t+1 of kernel gq; c2,c3 = of kernel gq + 8.
      // Lane t = 0 finishes kernel gq, lane t = 1 kernel gq + 8.
      const int base = lane & ~3;
      float m[6];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float x0 = __shfl_sync(0xffffffffu, acc[0], base + k);
        const float x1 = __shfl_sync(0xffffffffu, acc[1], base + k);
        const float y0 = __shfl_sync(0xffffffffu, acc[2], base + k);
        const float y1 = __shfl_sync(0xffffffffu, acc[3], base + k);
        m[2 * k] = (t == 1 ? y0 : x0) * inv_s;
        m[2 * k + 1] = (t == 1 ? y1 : x1) * inv_s;
      }
      const int kk = t == 1 ? 1 : 0;
      const int e = cb + gq + 8 * kk;
      if (t < 2 && e < n_list) {
        const float ox = (float)(u0 + 8) - (kk ? f0.y : f0.x);
        const float oy = (float)(v0 + 8) - (kk ? f0.w : f0.z);
        float st[6];
        st[0] = m[0];
        st[1] = fmaf(ox, m[0], m[1]);
        st[2] = fmaf(oy, m[0], m[2]);
        st[3] = fmaf(ox, fmaf(ox, m[0], 2.f * m[1]), m[3]);
        st[4] = fmaf(oy, fmaf(oy, m[0], 2.f * m[2]), m[4]);
        st[5] = fmaf(ox, fmaf(oy, m[0], m[2]), fmaf(oy, m[1], m[5]));
        const long long it = s_it[warp][buf][gq + 8 * kk];
        if (item_stats) {  // vector reductions (sm_90+): 2 instead of 6 L1 wavefronts per pair
          float4* dst = reinterpret_cast<float4*>(item_stats + 8 * it);
          atomicAdd(dst, make_float4(st[0], st[1], st[2], st[3]));
          atomicAdd(reinterpret_cast<float2*>(dst + 1), make_float2(st[4], st[5]));
        } else {
          const short4 r = rect[it];
          const long long slot = offset[it] + (ty - r.z) * (r.y - r.x + 1) + (tx - r.x);
          float4* dst = reinterpret_cast<float4*>(pair_stats + 8 * slot);
          dst[0] = make_float4(st[0], st[1], st[2], st[3]);
          *reinterpret_cast<float2*>(dst + 1) = make_float2(st[4], st[5]);
        }
      }
      __syncwarp();  // the next chunk's copy overwrites this buffer
    }
    if (us.done) {  // host path: publish the unit to the chain stream once all its lists are done
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) unit_signal(us, unit);
    }
  }
}

// K4 on the 5th-generation tensor cores (tcgen05 + TMEM): SCT_K4=tc. Measured at
// parity with the mma.sync form at cfg3 (1.91 vs 1.88 ms, DESIGN.md §3 "K4"): K4 is
// bound by issuing the E evaluation, which both forms share, not by the MMA; the
// mma.sync form stays the default and serves the host-buffer (unit-pipelined) path.
// Same product M = E G as above, transposed onto the Blackwell datapath:
//   * thread = kernel: a CTA holds 128 kernels of a (view, tile) list per chunk,
//     kernel i of the chunk owning TMEM lane i. Each thread evaluates its
//     kernel's E over the tile (exp2 recurrence, rows 2q and 2q+1 packed in
//     FP32x2) and stores it as binary16 pairs straight into tensor memory
//     (tcgen05.st): A[kernel][pixel], one row pair (16 columns) per buffer,
//     kTcABuf buffers in flight;
//   * G (hi/lo binary16, moments n = 0..5 hi, 8..13 lo) sits in shared memory
//     in the canonical K-major no-swizzle layout, built once per tile;
//   * a fifth warp issues tcgen05.mma kind::f16 M=128 N=16 K=16 (two per row
//     pair, FP32 accumulate in TMEM, D double-buffered per chunk) and
//     tcgen05.commit releases the A buffer / publishes D through mbarriers;
//   * each thread reads its kernel's 16 accumulator columns (tcgen05.ld) and
//     applies the binomial shift: no fragment shuffles, no B-fragment LDS.
//     The epilogue of chunk c runs in the middle of chunk c + 1, when its
//     MMAs have long completed.
// Records and list indices are staged per thread with cp.async (one and two
// chunks ahead; each thread reads back only what it copied itself).
// Numerics are those of the mma.sync form (same E, same G split, FP32 accumulate).
// Persistent CTAs take (list, part) work items from a global counter in the
// given order; empty lists are skipped by the claiming thread.
constexpr int kTcWarps = 4;  // compute warps (128 TMEM lanes)
constexpr int kTcThreads = 32 * (kTcWarps + 1);
constexpr int kTcABuf = 4;  // row-pair A buffers (16 TMEM columns each)
constexpr uint32_t kTcDCol = 16 * kTcABuf;
constexpr uint32_t kTcCols = 128;  // A 4 x 16, D 2 x 16 (+ 32 spare)
#ifndef SCT_K4TC_CTAS
#define SCT_K4TC_CTAS 4
#endif
constexpr int kTcCtas = SCT_K4TC_CTAS;  // CTAs per SM (kTcCols TMEM columns each, <= 512 per SM)
static_assert(kTcCtas * kTcCols <= 512, "TMEM columns per SM");
constexpr uint32_t kSleepNs = 0x100000;  // mbarrier waits: stay suspended until the phase completes

// byte offset of G[n][k] (moment n, pixel k) in the K-major no-swizzle layout:
// core matrix (k / 8, n / 8) of 8 rows x 16 bytes; LBO (next 8 pixels) = 256 B,
// SBO (next 8 moments) = 128 B; the K = 16 slice j starts at 512 j
__device__ __forceinline__ int g_off(int n, int k) { return ((k >> 3) * 2 + (n >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2; }

struct TcRow {  // per-kernel constants of the E evaluation (scalars: FFMA2 / FMUL2 take them as broadcast operands)
  float A, A2, B, C, K, dx, cy;
  bool ok;
};
__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }

// E of rows 2q (.x) and 2q+1 (.y), 16 columns, into A buffer q % kTcABuf.
// MODE 0: one 8-run per half row, 1: two 4-runs, 2: direct evaluation.
template <int MODE>
__device__ __forceinline__ void tc_row_pair(const TcRow& k, int q, float py0, uint32_t tl, uint64_t* aempty,
                                            uint64_t* afull, uint32_t parity, int lane) {
  const float py = py0 + (float)(2 * q);
  const float2 dy = make_float2(py - k.cy, py + 1.f - k.cy);
  const float2 bdy = __fmul2_rn(bc(k.B), dy);
  const float2 apb = __fadd2_rn(bc(k.A), bdy);
  float2 cdy2o = __ffma2_rn(__fmul2_rn(bc(k.C), dy), dy, make_float2(15.f, 15.f));
  if (!k.ok) cdy2o = make_float2(-1e30f, -1e30f);
  const int b = q % kTcABuf;
  tc::mbar_wait_sleep(&aempty[b], parity ^ 1, kSleepNs);
  tc::fence_after_sync();
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // columns 8h .. 8h+7
    float2 e[8];
    const float2 dxh = bc(k.dx + 8.f * h);
    if (MODE == 0) {
      run8x2(e, dxh, bc(k.A), bc(k.A2), bdy, apb, cdy2o, bc(k.K));
    } else if (MODE == 1) {
      run4x2(e, dxh, bc(k.A), bc(k.A2), bdy, apb, cdy2o, bc(k.K));
      run4x2(e + 4, bc(k.dx + 8.f * h + 4.f), bc(k.A), bc(k.A2), bdy, apb, cdy2o, bc(k.K));
    } else {
      direct8x2(e, dxh, bc(k.A), bdy, cdy2o);
    }
    uint32_t p0[4], p1[4];  // pixel pairs of row 2q (A columns 16b + 4h ..) / 2q+1 (16b + 8 + 4h ..)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      p0[j] = h2_bits(__floats2half2_rn(e[2 * j].x, e[2 * j + 1].x));
      p1[j] = h2_bits(__floats2half2_rn(e[2 * j].y, e[2 * j + 1].y));
    }
    tc::tmem_st4(tl + 16 * b + 4 * h, p0);
    tc::tmem_st4(tl + 16 * b + 8 + 4 * h, p1);
  }
  tc::tmem_wait_st();
  tc::fence_before_sync();
  __syncwarp();
  if (lane == 0) tc::mbar_arrive(&afull[b]);
}

template <int MODE>
__device__ __forceinline__ void tc_rows4(const TcRow& k, int q0, float py0, uint32_t tl, uint64_t* aempty,
                                         uint64_t* afull, uint32_t parity, int lane) {
#pragma unroll 1
  for (int q = q0; q < q0 + 4; ++q) tc_row_pair<MODE>(k, q, py0, tl, aempty, afull, parity, lane);
}

__global__ void __launch_bounds__(kTcThreads, kTcCtas) backward_stats_tc_kernel(
    const int2* __restrict__ ranges, const int32_t* __restrict__ vals, const float4* __restrict__ rec,
    const short4* __restrict__ rect, const int32_t* __restrict__ offset, int tiles_x, int tiles_per_view, int W,
    int H, int view0, const int* __restrict__ order, int parts, int n_work, int* __restrict__ work,
    const float* __restrict__ dL, float* __restrict__ pair_stats, float* __restrict__ item_stats, UnitSync us) {
  pdl_prologue();
  __shared__ __align__(1024) unsigned char s_g[16 * 256 * 2];
  __shared__ __align__(8) uint64_t bar_afull[kTcABuf], bar_aempty[kTcABuf], bar_dfull[2], bar_dempty[2];
  __shared__ __align__(16) float4 s_rec[2][32 * kTcWarps][2];  // per-thread staging (own slots)
  __shared__ int s_idx[2][32 * kTcWarps];
  __shared__ uint32_t s_taddr;
  __shared__ int4 s_item[2];  // current / next work item
  __shared__ float s_gmax[kTcWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool issuer = warp == kTcWarps;
  // zero moments 6, 7, 14, 15 once (never rewritten)
  for (int e = tid; e < 4 * 256; e += kTcThreads) {
    const int n = (e >> 8) < 2 ? 6 + (e >> 8) : 12 + (e >> 8), k = e & 255;
    *reinterpret_cast<__half*>(s_g + g_off(n, k)) = __float2half(0.f);
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) {
    tc::tmem_alloc(&s_taddr, kTcCols);
    tc::tmem_relinquish();
  }
  if (tid == 0) {
    for (int b = 0; b < kTcABuf; ++b) {
      tc::mbar_init(&bar_afull[b], kTcWarps);
      tc::mbar_init(&bar_aempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&bar_dfull[b], 1);
      tc::mbar_init(&bar_dempty[b], kTcWarps);
    }
    tc::mbar_init_fence();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = s_taddr;
  const uint32_t tlane = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  const uint32_t idesc = tc::idesc_f16_f32(128, 16);
  uint32_t ck = 0;  // chunks so far: A buffer uses (2 per chunk) and D buffer phases
  // claim the next non-empty (list, part) in the order: {work index, list, start, end};
  // empty lists are published right away (host path)
  auto claim = [&]() -> int4 {
    for (;;) {
      const int c = atomicAdd(work, 1);
      if (c >= n_work) return make_int4(-1, 0, 0, 0);
      const int w = order[c / parts], p = c % parts;
      const int2 rg = ranges[(long long)view0 * tiles_per_view + w];
      const int len = rg.y - rg.x;
      const int a0 = rg.x + (int)((long long)len * p / parts), a1 = rg.x + (int)((long long)len * (p + 1) / parts);
      if (a1 > a0) return make_int4(c, w, a0, a1);
      if (us.done) unit_signal(us, unit_of_view(view0 + w / tiles_per_view, us.n_views, us.units));
    }
  };
  const bool host_path = us.done != nullptr || us.ready != nullptr;
  if (tid == 0) {
    const int4 f = claim();
    if (f.x >= 0 && us.ready) unit_wait(us, unit_of_view(view0 + f.y / tiles_per_view, us.n_views, us.units));
    s_item[0] = f;
  }
  __syncthreads();
  for (int cur = 0;; cur ^= 1) {
    const int4 itm = s_item[cur];
    if (itm.x < 0) break;
    const int w = itm.y;
    const int tile = w % tiles_per_view, view = view0 + w / tiles_per_view;
    const int2 rg = make_int2(itm.z, itm.w);
    const int n_list = rg.y - rg.x;
    const int n_chunks = (n_list + 127) >> 7;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int u0 = tx * kTilePx, v0 = ty * kTilePx;
    if (issuer) {
      __syncthreads();  // G of this tile is ready
      // ---------------- MMA issue: per chunk, 8 row pairs x 2 K-slices into D[ck & 1]
      for (int ch = 0; ch < n_chunks; ++ch, ++ck) {
        const uint32_t d = ck & 1;
        tc::mbar_wait_sleep(&bar_dempty[d], ((ck >> 1) & 1) ^ 1, kSleepNs);
        tc::fence_after_sync();
        const uint32_t dt = tbase + kTcDCol + 16 * d;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int b = q % kTcABuf;
          const uint32_t use = 2 * ck + q / kTcABuf;  // uses of buffer b so far
          tc::mbar_wait_sleep(&bar_afull[b], use & 1, kSleepNs);
          tc::fence_after_sync();
          if (lane == 0) {
            const uint32_t at = tbase + 16 * b;
            tc::mma_f16_ts(dt, at, tc::smem_desc_kmajor(s_g + 512 * (2 * q), 256, 128), idesc, q > 0);
            tc::mma_f16_ts(dt, at + 8, tc::smem_desc_kmajor(s_g + 512 * (2 * q + 1), 256, 128), idesc, 1);
            tc::commit(&bar_aempty[b]);  // A buffer b free once these MMAs completed
            if (q == 7) tc::commit(&bar_dfull[d]);
          }
          __syncwarp();
        }
        if (ch == 0 && lane == 0) s_item[cur ^ 1] = claim();  // the next item, while this one runs
      }
    } else {
      // ---------------- G of this tile (per-tile power-of-two scale, hi/lo split)
      float inv_s;
      {
        const float* dtile = dL + ((long long)view * H + v0) * W + u0;
        const bool streamed = us.ready != nullptr;  // host path: L2-coherent loads (copies still landing)
        float g[2];
        float gm = 0.f;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int p = tid + 128 * i, r = p >> 4, cc = p & 15;
          const float* src = dtile + (long long)r * W + cc;
          g[i] = (v0 + r < H && u0 + cc < W) ? (streamed ? __ldcg(src) : __ldg(src)) : 0.f;
          gm = fmaxf(gm, fabsf(g[i]));
        }
        gm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(gm)));
        if (lane == 0) s_gmax[warp] = gm;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcWarps) : "memory");
#pragma unroll
        for (int k = 0; k < kTcWarps; ++k) gm = fmaxf(gm, s_gmax[k]);
        const float S = gm > 0.f ? exp2f(floorf(log2f(16384.f / (gm * 56.25f * 0x1p-15f)))) : 1.f;
        const float gscale = 0x1p-15f * S;
        inv_s = 1.f / S;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int p = tid + 128 * i, r = p >> 4, cc = p & 15;
          const float gs = g[i] * gscale, cp = (float)cc - 7.5f, rpf = (float)r - 7.5f;
          const float phi[6] = {1.f, cp, rpf, cp * cp, rpf * rpf, cp * rpf};
#pragma unroll
          for (int n = 0; n < 6; ++n) {
            const float v = gs * phi[n];
            const __half hi = __float2half_rn(v);
            *reinterpret_cast<__half*>(s_g + g_off(n, p)) = hi;
            *reinterpret_cast<__half*>(s_g + g_off(8 + n, p)) = __float2half_rn(v - __half2float(hi));
          }
        }
        tc::fence_proxy_async_smem();  // G -> visible to the tensor core
      }
      // prologue of the staging pipeline: index 0 (direct), record 0 and index 1 (cp.async)
      {
        const int it0 = tid < n_list ? vals[rg.x + tid] : -1;
        s_idx[0][tid] = it0;
        float4* dst = &s_rec[0][tid][0];
        if (it0 >= 0) {
          cp_async16(dst, rec + 2 * (long long)it0);
          cp_async16(dst + 1, rec + 2 * (long long)it0 + 1);
        } else {
          dst[0] = make_float4(0.f, 0.f, 0.f, 1.f);
          dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (128 + tid < n_list) cp_async4(&s_idx[1][tid], vals + rg.x + 128 + tid);
        else s_idx[1][tid] = -1;
        cp_async_commit();
      }
      __syncthreads();  // G ready for the issuer
      const float px0 = (float)u0 + 0.5f, py0 = (float)v0 + 0.5f;
      // pending epilogue (the previous chunk of this list)
      int pend_it = -1;
      float pend_cx = 0.f, pend_cy = 0.f;
      uint32_t pend_ck = 0;
      auto epilogue = [&]() {
        const uint32_t d = pend_ck & 1;
        tc::mbar_wait_sleep(&bar_dfull[d], (pend_ck >> 1) & 1, kSleepNs);
        tc::fence_after_sync();
        uint32_t acc[16];
        tc::tmem_ld16(tlane + kTcDCol + 16 * d, acc);
        tc::tmem_wait_ld();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bar_dempty[d]);
        if (pend_it < 0) return;
        float m[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) m[k] = (__uint_as_float(acc[k]) + __uint_as_float(acc[8 + k])) * inv_s;
        const float ox = (float)(u0 + 8) - pend_cx;
        const float oy = (float)(v0 + 8) - pend_cy;
        float st[6];
        st[0] = m[0];
        st[1] = fmaf(ox, m[0], m[1]);
        st[2] = fmaf(oy, m[0], m[2]);
        st[3] = fmaf(ox, fmaf(ox, m[0], 2.f * m[1]), m[3]);
        st[4] = fmaf(oy, fmaf(oy, m[0], 2.f * m[2]), m[4]);
        st[5] = fmaf(ox, fmaf(oy, m[0], m[2]), fmaf(oy, m[1], m[5]));
        if (item_stats) {
          float4* dst = reinterpret_cast<float4*>(item_stats + 8 * (long long)pend_it);
          atomicAdd(dst, make_float4(st[0], st[1], st[2], st[3]));
          atomicAdd(reinterpret_cast<float2*>(dst + 1), make_float2(st[4], st[5]));
        } else {
          const short4 r = rect[pend_it];
          const long long slot = offset[pend_it] + (ty - r.z) * (r.y - r.x + 1) + (tx - r.x);
          float4* dst = reinterpret_cast<float4*>(pair_stats + 8 * slot);
          dst[0] = make_float4(st[0], st[1], st[2], st[3]);
          *reinterpret_cast<float2*>(dst + 1) = make_float2(st[4], st[5]);
        }
      };
      for (int ch = 0; ch < n_chunks; ++ch, ++ck) {
        cp_async_wait_all();  // record ch, index ch + 1 (own slots)
        const int sb = ch & 1;
        const int it = s_idx[sb][tid];
        const float4 ra = s_rec[sb][tid][0], rb = s_rec[sb][tid][1];  // {cx, cy, amp, K}, {A, B, C, 2A}
        if (ch + 1 < n_chunks) {  // stage record ch + 1 and index ch + 2
          const int itn = s_idx[sb ^ 1][tid];
          float4* dst = &s_rec[sb ^ 1][tid][0];
          if (itn >= 0) {
            cp_async16(dst, rec + 2 * (long long)itn);
            cp_async16(dst + 1, rec + 2 * (long long)itn + 1);
          } else {
            dst[0] = make_float4(0.f, 0.f, 0.f, 1.f);
            dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          const int e2 = (ch + 2) * 128 + tid;
          if (e2 < n_list) cp_async4(&s_idx[sb][tid], vals + rg.x + e2);
          else s_idx[sb][tid] = -1;
          cp_async_commit();
        }
        TcRow k;
        k.A = rb.x;
        k.B = rb.y;
        k.C = rb.z;
        k.A2 = rb.w;
        k.K = ra.w;
        k.dx = px0 - ra.x;
        k.cy = ra.y;
        k.ok = it >= 0;
        const float aa = fabsf(rb.x);
        const int mode = __all_sync(0xffffffffu, aa <= 1.25f) ? 0 : __any_sync(0xffffffffu, aa > kRun4MaxA_K4) ? 2 : 1;
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {  // A-buffer use 2 ck + half: parity = half
          if (mode == 0) tc_rows4<0>(k, 4 * half, py0, tlane, bar_aempty, bar_afull, half, lane);
          else if (mode == 1) tc_rows4<1>(k, 4 * half, py0, tlane, bar_aempty, bar_afull, half, lane);
          else tc_rows4<2>(k, 4 * half, py0, tlane, bar_aempty, bar_afull, half, lane);
          if (half == 0 && ch > 0) epilogue();
        }
        pend_it = it;
        pend_cx = ra.x;
        pend_cy = ra.y;
        pend_ck = ck;
      }
      if (n_chunks > 0) epilogue();
      if (us.done) __threadfence();
    }
    // every chunk's accumulator was read (so every MMA reading G completed)
    // before the next tile's G overwrites it; the next item is in s_item[cur ^ 1]
    __syncthreads();
    if (host_path) {  // publish this list's unit, wait for the next one's upstream gradient
      if (tid == 0) {
        if (us.done) unit_signal(us, unit_of_view(view, us.n_views, us.units));
        const int4 nx = s_item[cur ^ 1];
        if (nx.x >= 0 && us.ready) unit_wait(us, unit_of_view(view0 + nx.y / tiles_per_view, us.n_views, us.units));
      }
      __syncthreads();
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTcCols);
}

int grid_cap(Ctx* c, long long n, int block) {
  long long b = (n + block - 1) / block;
  const long long cap = (long long)c->sm_count * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

void launch_raster_emit(Ctx* c, int64_t n_items, const short4* rect, const int32_t* offset, int tiles_x,
                        void* keys, bool keys16, int32_t* vals) {
  if (n_items == 0) return;
  KScope _ks(c, "K2_raster_emit");
  if (keys16)
    pdl_launch(raster_emit_kernel<uint16_t>, dim3(grid_cap(c, n_items, 256)), dim3(256), 0, c->stream, n_items, rect, offset, tiles_x, static_cast<uint16_t*>(keys), vals);
  else
    pdl_launch(raster_emit_kernel<uint32_t>, dim3(grid_cap(c, n_items, 256)), dim3(256), 0, c->stream, n_items, rect, offset, tiles_x, static_cast<uint32_t*>(keys), vals);
}

// Counting-scatter binning (bin_* kernels above). Needs the per-warp tile
// table in shared memory: T <= kMaxScatterTiles, else the caller keeps the
// radix-sort path. Returns false when not applicable.
static int64_t scatter_tables(int64_t tx, int64_t ty, int64_t tz) {
  return kBinWarps * (tx * ty * tz + tx + ty + tz) * (int64_t)sizeof(uint32_t);
}
bool bin_scatter_fits(int tiles_x, int tiles_y, int tiles_z) {
  const int64_t T = (int64_t)tiles_x * tiles_y * tiles_z;
  return scatter_tables(tiles_x, tiles_y, tiles_z) + 256 * 2 * (int64_t)sizeof(short4) <= kScatterSmem &&
         T * 4 <= 48 * 1024;  // bin_count's histogram (default shared limit)
}
bool raster_bin_scatter_fits(int tiles_x, int tiles_y) { return bin_scatter_fits(tiles_x, tiles_y, 1); }

// exclusive scan of count[0..n] into offset[0..n] (count[n] == 0) with the int64
// total into *sum64, in one CTA (small item counts: the train step's one view),
// and — capacity mode (cap > 0) — the capacity guard of capacity_guard_kernel
constexpr int kCountScanThreads = 1024;
__global__ void __launch_bounds__(kCountScanThreads) count_scan_small_kernel(int32_t* __restrict__ count,
                                                                             int32_t* __restrict__ offset, long long n,
                                                                             long long* __restrict__ sum64,
                                                                             long long cap, short4* __restrict__ box_a,
                                                                             short4* __restrict__ box_b,
                                                                             int* __restrict__ overflow) {
  pdl_prologue();
  using Scan = cub::BlockScan<long long, kCountScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long s_total;
  // tiles of 4 * kCountScanThreads entries: coalesced int4 loads, one block scan per tile
  constexpr int kTile = 4 * kCountScanThreads;
  long long carry = 0;
  for (long long t0 = 0; t0 <= n; t0 += kTile) {
    const long long i = t0 + 4 * (long long)threadIdx.x;
    int v[4];
    if (i + 3 <= n) {
      const int4 q = *reinterpret_cast<const int4*>(count + i);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = i + k <= n ? count[i + k] : 0;
    }
    long long ex = 0, tile_total = 0;
    Scan(tmp).ExclusiveSum((long long)v[0] + v[1] + v[2] + v[3], ex, tile_total);
    __syncthreads();  // temp storage reuse
    long long run = carry + ex;
    if (i + 3 <= n) {
      int4 o;
      o.x = (int32_t)run; run += v[0];
      o.y = (int32_t)run; run += v[1];
      o.z = (int32_t)run; run += v[2];
      o.w = (int32_t)run;
      *reinterpret_cast<int4*>(offset + i) = o;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i + k <= n) {
          offset[i + k] = (int32_t)run;
          run += v[k];
        }
    }
    carry += tile_total;
  }
  const long long total = carry;
  if (threadIdx.x == 0) {
    *sum64 = total;
    s_total = total;
  }
  __syncthreads();
  if (cap > 0 && s_total > cap) {  // as capacity_guard_kernel: empty every item
    if (threadIdx.x == 0) atomicOr(overflow, 1);
    for (long long i = threadIdx.x; i <= n; i += kCountScanThreads) {
      offset[i] = 0;
      if (i == n) continue;
      count[i] = 0;
      if (box_b) {
        const short4 a = box_a[i];
        box_b[i] = make_short4((short)(a.x - 1), (short)(a.y - 1), (short)(a.z - 1), 0);
      } else {
        box_a[i] = make_short4(1, 0, 1, 0);
      }
    }
  }
}

void launch_count_scan_small(Ctx* c, int32_t* count, int32_t* offset, int64_t n, int64_t cap, short4* box_a,
                             short4* box_b) {
  pdl_launch(count_scan_small_kernel, dim3(1), dim3(kCountScanThreads), 0, c->stream, count, offset, (long long)n, c->sum64,
                                                                  (long long)cap, box_a, box_b, c->overflow);
}

void launch_capacity_guard(Ctx* c, int32_t* count, int32_t* offset, int64_t n, short4* box_a, short4* box_b,
                           int64_t cap, bool no_wrap) {
  pdl_launch(capacity_guard_kernel, dim3(grid_cap(c, n + 1, 256)), dim3(256), 0, c->stream, count, offset, n, box_a, box_b, no_wrap ? nullptr : c->sum64, (long long)cap, c->overflow);
}

// Stable counting-scatter binning of n_views x m items with boxes (lo, hi)
// over a tiles_x x tiles_y x tiles_z tile grid (raster: hi == nullptr, one
// layer). cap: size of vals (pairs beyond it are dropped and flag
// c->overflow); total (nullable): device word receiving the pair count;
// ranges [n_views][T] (nullable when only the totals are needed).
int launch_bin_scatter(Ctx* c, int64_t n_views, int64_t m, int tiles_x, int tiles_y, int tiles_z, const short4* lo,
                       const short4* hi, int32_t* vals, int2* ranges, int64_t cap, int32_t* total,
                       int64_t scatter_views, BinDeferred** defer) {
  const int64_t T = (int64_t)tiles_x * tiles_y * tiles_z;
  if (m == 0 || n_views == 0) return SCT_OK;
  // chunk size: the count table H holds (V * chunks) x T entries (<= ~64M), and
  // the scatter keeps a chunk's boxes in shared memory next to its tables
  const int64_t target = 64ll << 20;
  static const int64_t min_chunk = [] {
    const char* e = std::getenv("SCT_BIN_CHUNK");
    return e ? std::max<int64_t>(256, atoll(e)) : 1024;
  }();
  const int64_t tables = scatter_tables(tiles_x, tiles_y, tiles_z);
  const int64_t max_chunk = ((kScatterSmem - tables) / (2 * (int64_t)sizeof(short4))) / 256 * 256;
  const int64_t need = (m * n_views * T + target - 1) / target;  // H within its budget
  int64_t chunk = std::max<int64_t>(min_chunk, need);
  // small workloads (the train step's single view): at least two blocks per SM
  const int64_t par = (m * n_views + 2 * c->sm_count - 1) / (2 * c->sm_count);
  chunk = std::max<int64_t>(need, std::min<int64_t>(chunk, std::max<int64_t>(256, par)));
  chunk = std::min<int64_t>(((chunk + 255) / 256) * 256, max_chunk);
  const int64_t n_chunks = (m + chunk - 1) / chunk;
  const int64_t rows = n_views * n_chunks;
  const int64_t n_seg = (rows + kSegRows - 1) / kSegRows;
  int32_t *H = nullptr, *seg = nullptr, *tb = nullptr;
  SCT_TRY(dev_alloc(c, (void**)&H, rows * T * sizeof(int32_t)));
  SCT_TRY(dev_alloc(c, (void**)&seg, n_seg * T * sizeof(int32_t)));
  SCT_TRY(dev_alloc(c, (void**)&tb, (2 * T + 1) * sizeof(int32_t)));
  int32_t* tb2 = tb + T;  // tile bases [T + 1]; tb[0..T) holds the column totals
  const dim3 grid((unsigned)n_chunks, (unsigned)n_views);
  {
    KScope _ks(c, "K2_bin_count");
    pdl_launch(bin_count_kernel, dim3(grid), dim3(256), T * sizeof(uint32_t), c->stream, lo, hi, m, (int)chunk, (int)T, tiles_x, tiles_y,
                                                                     H);
  }
  if (T <= kSmallScanThreads && rows * T <= kSmallScanEntries) {
    KScope _ks(c, "K2_bin_scan");
    pdl_launch(bin_scan_small_kernel, dim3(1), dim3(kSmallScanThreads), 0, c->stream, H, (int)rows, (int)T, tb2, (long long)cap,
                                                                  c->overflow, total);
  } else {
    KScope _ks(c, "K2_bin_scan");
    const dim3 g2((unsigned)((T + 255) / 256), (unsigned)n_seg);
    pdl_launch(bin_colsum_kernel, dim3(g2), dim3(256), 0, c->stream, H, (int)rows, (int)T, seg);
    pdl_launch(bin_segscan_kernel, dim3((unsigned)((T + 255) / 256)), dim3(256), 0, c->stream, seg, (int)n_seg, (int)T, tb);
    pdl_launch(bin_tilebase_kernel, dim3(1), dim3(1024), 0, c->stream, tb, (int)T, tb2, (long long)cap, c->overflow, total);
    pdl_launch(bin_apply_kernel, dim3(g2), dim3(256), 0, c->stream, H, seg, tb2, (int)rows, (int)T);
  }
  if (ranges) {  // from the scan alone: final before any pair is written
    KScope _ks(c, "K2_bin_ranges");
    pdl_launch(bin_ranges_kernel, dim3(grid_cap(c, n_views * T, 256)), dim3(256), 0, c->stream, H, tb2, (int)n_chunks, (int)n_views,
                                                                            (int)T, ranges, (long long)cap);
  }
  static bool attr = false;
  if (!attr) {
    SCT_CUDA_TRY(cudaFuncSetAttribute(bin_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kScatterSmem));
    attr = true;
  }
  const size_t smem = tables + (SCT_SCATTER_SBOX ? chunk * 2 * sizeof(short4) : 0);
  const int64_t v_now = (scatter_views > 0 && scatter_views < n_views && defer) ? scatter_views : n_views;
  {
    KScope _ks(c, "K2_bin_scatter");
    pdl_launch(bin_scatter_kernel, dim3(dim3((unsigned)n_chunks, (unsigned)v_now)), dim3(32 * kBinWarps), smem, c->stream, lo, hi, m, (int)chunk, (int)T, tiles_x, tiles_y, tiles_z, H, vals,
        (uint32_t)std::min<int64_t>(cap, UINT32_MAX), 0);
  }
  if (v_now < n_views) {  // the rest later (launch_bin_scatter_rest)
    auto* d = new BinDeferred();
    d->H = H;
    d->seg = seg;
    d->tb = tb;
    d->lo = lo;
    d->hi = hi;
    d->vals = vals;
    d->m = m;
    d->n_views = n_views;
    d->v0 = v_now;
    d->chunk = chunk;
    d->n_chunks = n_chunks;
    d->cap = cap;
    d->tiles_x = tiles_x;
    d->tiles_y = tiles_y;
    d->tiles_z = tiles_z;
    d->smem = smem;
    *defer = d;
    return SCT_OK;
  }
  dev_free(c, H);
  dev_free(c, seg);
  dev_free(c, tb);
  return SCT_OK;
}

int launch_bin_scatter_rest(Ctx* c, BinDeferred* d) {
  if (!d) return SCT_OK;
  const int64_t T = (int64_t)d->tiles_x * d->tiles_y * d->tiles_z;
  {
    KScope _ks(c, "K2_bin_scatter");
    pdl_launch(bin_scatter_kernel, dim3(dim3((unsigned)d->n_chunks, (unsigned)(d->n_views - d->v0))), dim3(32 * kBinWarps), d->smem, c->stream, d->lo, d->hi, d->m, (int)d->chunk, (int)T, d->tiles_x, d->tiles_y, d->tiles_z,
                                      d->H, d->vals, (uint32_t)std::min<int64_t>(d->cap, UINT32_MAX), (int)d->v0);
  }
  dev_free(c, d->H);
  dev_free(c, d->seg);
  dev_free(c, d->tb);
  delete d;
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int launch_raster_bin_scatter(Ctx* c, int64_t n_views, int64_t m, int tiles_x, int tiles_y, const short4* rect,
                              int32_t* vals, int2* ranges, int64_t n_pairs, int64_t cap, int32_t* total,
                              int64_t scatter_views, BinDeferred** defer) {
  if (n_pairs == 0) return SCT_OK;
  return launch_bin_scatter(c, n_views, m, tiles_x, tiles_y, 1, rect, nullptr, vals, ranges, cap, total,
                            scatter_views, defer);
}

void launch_raster_ranges(Ctx* c, int64_t n_pairs, const void* keys, bool keys16, const int32_t* vals, int64_t m,
                          int64_t tiles_per_view, int2* ranges) {
  if (n_pairs == 0) return;
  KScope _ks(c, "K2_ranges");
  if (keys16)
    pdl_launch(raster_ranges_kernel<uint16_t>, dim3(grid_cap(c, (n_pairs + 7) / 8, 256)), dim3(256), 0, c->stream, n_pairs, static_cast<const uint16_t*>(keys), vals, (int)m, 1.f / (float)m, tiles_per_view, ranges);
  else
    pdl_launch(raster_ranges_kernel<uint32_t>, dim3(grid_cap(c, (n_pairs + 7) / 8, 256)), dim3(256), 0, c->stream, n_pairs, static_cast<const uint32_t*>(keys), vals, (int)m, 1.f / (float)m, tiles_per_view, ranges);
}

// list order key: the length octave, descending, clamped to 4 bits (lists of
// >= 2^14 kernels share the first bucket)
__device__ __forceinline__ uint32_t order_key4(int len) {
  return 15u - (uint32_t)min(15, 32 - __clz(max(len, 0)));
}

// Longest-processing-time order of the (view, tile) lists of views
// [v0, v0 + nv): local indices sorted by descending list length, so that K3's
// persistent warps and K4's blocks start the long lists first and the kernels'
// tails consist of short lists. Cached in the context for the last range.
__global__ void __launch_bounds__(256) tile_order_keys_kernel(const int2* __restrict__ ranges, long long base,
                                                              int n, uint32_t* __restrict__ keys,
                                                              int32_t* __restrict__ idx) {
  pdl_prologue();
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < n; w += gridDim.x * blockDim.x) {
    const int2 r = ranges[base + w];
    // descending octave of the list length; the stable sort keeps the natural
    // (view-major, spatially coherent) order inside an octave for L2 locality
    keys[w] = order_key4(r.y - r.x);
    idx[w] = w;
  }
}

// tile_order_keys_kernel + the stable sort in one CTA, for small workloads
// (n <= kSmallOrder). The key is the length octave clamped to 4 bits (lists of
// >= 2^14 kernels share the first bucket), so the block sort is one radix pass.
constexpr int kSmallOrderThreads = 1024, kSmallOrderItems = 8;
constexpr int kSmallOrder = kSmallOrderThreads * kSmallOrderItems;
template <int kItems>
__global__ void __launch_bounds__(kSmallOrderThreads) tile_order_small_kernel(const int2* __restrict__ ranges,
                                                                              long long base, int n,
                                                                              int32_t* __restrict__ order) {
  pdl_prologue();
  using Sort = cub::BlockRadixSort<uint32_t, kSmallOrderThreads, kItems, int32_t>;
  __shared__ typename Sort::TempStorage tmp;
  uint32_t key[kItems];
  int32_t idx[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int w = threadIdx.x * kItems + i;  // blocked arrangement: input order = w
    if (w < n) {
      const int2 r = ranges[base + w];
      key[i] = order_key4(r.y - r.x);
    } else {
      key[i] = 15u;  // padding sorts after every real list (stable, larger index)
    }
    idx[i] = w;
  }
  Sort(tmp).Sort(key, idx, 0, 4);
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int w = threadIdx.x * kItems + i;
    if (w < n) order[w] = idx[i];
  }
}

// The same stable 16-bucket order for larger list counts in two multi-CTA
// passes (cfg3, 76 800 lists: 31 -> 11 us against the device-wide radix sort's
// four launches; the 8-rank shard's 10 240: 28 -> 9 us, a one-CTA counting sort
// took 16):
// pass 1 counts each 1024-list block's buckets, pass 2 ranks every list — the
// bucket start over all blocks, the earlier blocks' and earlier warps' counts
// of its bucket, and its rank among the warp's lanes of the same bucket
// (__match_any_sync) — and writes it to its stable position.
constexpr int kOrderBlock = 1024;
__global__ void __launch_bounds__(kOrderBlock) tile_order_hist_kernel(const int2* __restrict__ ranges, long long base,
                                                                      int n, int32_t* __restrict__ hist) {
  pdl_prologue();
  __shared__ int32_t h[16];
  if (threadIdx.x < 16) h[threadIdx.x] = 0;
  __syncthreads();
  const int w = blockIdx.x * kOrderBlock + threadIdx.x;
  if (w < n) {
    const int2 r = ranges[base + w];
    atomicAdd(&h[order_key4(r.y - r.x)], 1);
  }
  __syncthreads();
  if (threadIdx.x < 16) hist[blockIdx.x * 16 + threadIdx.x] = h[threadIdx.x];
}
__global__ void __launch_bounds__(kOrderBlock) tile_order_rank_kernel(const int2* __restrict__ ranges, long long base,
                                                                      int n, const int32_t* __restrict__ hist,
                                                                      int32_t* __restrict__ order) {
  pdl_prologue();
  __shared__ int32_t s_base[16];
  __shared__ int32_t s_wc[kOrderBlock / 32][16];  // per-warp bucket counts, then their exclusive prefix
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = blockIdx.x * kOrderBlock + threadIdx.x;
  if (warp == 0) {  // bucket starts over all blocks + this bucket's count in earlier blocks
    int tot = 0, before = 0;
    if (lane < 16)
      for (int b = 0; b < (int)gridDim.x; ++b) {
        const int v = hist[b * 16 + lane];
        tot += v;
        if (b < (int)blockIdx.x) before += v;
      }
    int incl = tot;
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane < 16) s_base[lane] = incl - tot + before;
  }
  for (int i = threadIdx.x; i < (kOrderBlock / 32) * 16; i += blockDim.x) (&s_wc[0][0])[i] = 0;
  __syncthreads();
  uint32_t key = 16;  // past the end: no bucket
  if (w < n) {
    const int2 r = ranges[base + w];
    key = order_key4(r.y - r.x);
  }
  const uint32_t same = __match_any_sync(0xffffffffu, key);
  const int rank = __popc(same & ((1u << lane) - 1u));
  if (key < 16 && rank == 0) s_wc[warp][key] = __popc(same);
  __syncthreads();
  if (threadIdx.x < 16) {  // exclusive prefix over the warps, per bucket
    int run = 0;
    for (int k = 0; k < kOrderBlock / 32; ++k) {
      const int v = s_wc[k][threadIdx.x];
      s_wc[k][threadIdx.x] = run;
      run += v;
    }
  }
  __syncthreads();
  if (key < 16) order[s_base[key] + s_wc[warp][key] + rank] = w;
}

// keys for the chunked order: (chunk of the view, descending length octave)
__global__ void __launch_bounds__(256) tile_order_chunk_keys_kernel(const int2* __restrict__ ranges, int n,
                                                                    int tiles_per_view, int n_views, int chunks,
                                                                    uint32_t* __restrict__ keys,
                                                                    int32_t* __restrict__ idx) {
  pdl_prologue();
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < n; w += gridDim.x * blockDim.x) {
    const int2 r = ranges[w];
    const int v = w / tiles_per_view;
    int k = 0;  // chunk k holds views [V k / chunks, V (k + 1) / chunks)
    while (k + 1 < chunks && (long long)n_views * (k + 1) / chunks <= v) ++k;
    keys[w] = ((uint32_t)k << 5) | (31u - (uint32_t)(32 - __clz(max(r.y - r.x, 0))));
    idx[w] = w;
  }
}

static const int* tile_order(Ctx* c, const sct_fwd* s, int v0, int nv) {
  const int T = s->det.tiles_x * s->det.tiles_y;
  const int n = T * nv;
  char* buf = nullptr;
  if (stage_buf(c, 22, (size_t)4 * n * sizeof(uint32_t), (void**)&buf) != SCT_OK) return nullptr;
  uint32_t* k0 = reinterpret_cast<uint32_t*>(buf);
  uint32_t* k1 = k0 + n;
  int32_t* i0 = reinterpret_cast<int32_t*>(k1 + n);
  int32_t* i1 = i0 + n;
  KScope _ks(c, "K2_tile_order");
  if (n <= kSmallOrder) {  // one CTA instead of the device-wide sort's launches (train step: 256 lists)
    // items per thread sized to n (the 256-list train step sorts 1024 keys)
    if (n <= kSmallOrderThreads)
      pdl_launch(tile_order_small_kernel<1>, dim3(1), dim3(kSmallOrderThreads), 0, c->stream, s->d_ranges, (long long)v0 * T, n, i0);
    else if (n <= 4 * kSmallOrderThreads)
      pdl_launch(tile_order_small_kernel<4>, dim3(1), dim3(kSmallOrderThreads), 0, c->stream, s->d_ranges, (long long)v0 * T, n, i0);
    else
      pdl_launch(tile_order_small_kernel<kSmallOrderItems>, dim3(1), dim3(kSmallOrderThreads), 0, c->stream, s->d_ranges, (long long)v0 * T, n, i0);
    ++c->order_gen;
    return i0;
  }
  static const bool mid_ok = [] {  // SCT_ORDER_MID=0 (diagnostic): the device-wide radix sort instead
    const char* e = std::getenv("SCT_ORDER_MID");
    return !(e && atoi(e) == 0);
  }();
  if (mid_ok) {  // two multi-CTA passes (SCT_ORDER_MID=0: the device-wide radix sort below)
    const int nb = (n + kOrderBlock - 1) / kOrderBlock;
    int32_t* hist = reinterpret_cast<int32_t*>(k1);  // nb * 16 <= n entries
    pdl_launch(tile_order_hist_kernel, dim3(nb), dim3(kOrderBlock), 0, c->stream, s->d_ranges, (long long)v0 * T, n,
               hist);
    pdl_launch(tile_order_rank_kernel, dim3(nb), dim3(kOrderBlock), 0, c->stream, s->d_ranges, (long long)v0 * T, n,
               (const int32_t*)hist, i0);
    ++c->order_gen;
    return i0;
  }
  pdl_launch(tile_order_keys_kernel, dim3(grid_cap(c, n, 256)), dim3(256), 0, c->stream, s->d_ranges, (long long)v0 * T, n, k0, i0);
  cub::DoubleBuffer<uint32_t> keys(k0, k1);
  cub::DoubleBuffer<int32_t> vals(i0, i1);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, vals, n, 0, 4, c->stream);
  if (ensure_cub_tmp(c, tmp) != SCT_OK) return nullptr;
  tmp = c->cub_tmp_bytes;
  cub::DeviceRadixSort::SortPairs(c->cub_tmp, tmp, keys, vals, n, 0, 4, c->stream);
  ++c->order_gen;
  return vals.Current();
}

static const int* cached_tile_order(Ctx* c, const sct_fwd* s, int v0, int nv) {
  if (c->order_id == s->id && c->order_v0 == v0 && c->order_nv == nv && c->order_ptr) return c->order_ptr;
  c->order_ptr = tile_order(c, s, v0, nv);
  c->order_id = s->id;
  c->order_v0 = v0;
  c->order_nv = nv;
  return c->order_ptr;
}

// (view unit, then longest lists first) order of all views: unit u holds
// views [V u / units, V (u + 1) / units) and precedes unit u + 1, so the
// kernels of the host-buffer path finish (and publish) units in order while
// each unit's own tail stays short. Cached like cached_tile_order
// (order_v0 = -1 marks a unit order of order_nv units).
static const int* unit_tile_order(Ctx* c, const sct_fwd* s, int units) {
  if (c->order_id == s->id && c->order_v0 == -1 && c->order_nv == units && c->order_ptr) return c->order_ptr;
  const int V = s->n_views;
  const int T = s->det.tiles_x * s->det.tiles_y;
  const int n = T * V;
  char* buf = nullptr;
  c->order_id = 0;
  if (stage_buf(c, 22, (size_t)4 * n * sizeof(uint32_t), (void**)&buf) != SCT_OK) return nullptr;
  uint32_t* k0 = reinterpret_cast<uint32_t*>(buf);
  uint32_t* k1 = k0 + n;
  int32_t* i0 = reinterpret_cast<int32_t*>(k1 + n);
  int32_t* i1 = i0 + n;
  {
    KScope _ks(c, "K2_tile_order");
    pdl_launch(tile_order_chunk_keys_kernel, dim3(grid_cap(c, n, 256)), dim3(256), 0, c->stream, s->d_ranges, n, T, V, units, k0, i0);
  }
  cub::DoubleBuffer<uint32_t> keys(k0, k1);
  cub::DoubleBuffer<int32_t> vals(i0, i1);
  size_t tmp = 0;
  int bits = 5;
  while ((1 << (bits - 5)) < units) ++bits;
  if (cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, vals, n, 0, bits, c->stream) != cudaSuccess ||
      ensure_cub_tmp(c, tmp) != SCT_OK)
    return nullptr;
  tmp = c->cub_tmp_bytes;
  if (cub::DeviceRadixSort::SortPairs(c->cub_tmp, tmp, keys, vals, n, 0, bits, c->stream) != cudaSuccess)
    return nullptr;
  c->order_ptr = vals.Current();
  ++c->order_gen;
  c->order_id = s->id;
  c->order_v0 = -1;
  c->order_nv = units;
  return c->order_ptr;
}

enum class K4Impl { kTc, kMma, kSimt };
// SCT_K4 selects the statistics kernel: "mma" (default: mma.sync f16, FP32
// accumulate), "tc" (tcgen05 + TMEM; device-resident calls only), "simt" (FP32
// SIMT, no tensor cores: the reference-order arithmetic)
static K4Impl k4_impl() {
  static const K4Impl impl = [] {
    const char* e = std::getenv("SCT_K4");
    const std::string v = e ? e : "";
    return v == "simt" ? K4Impl::kSimt : v == "tc" ? K4Impl::kTc : K4Impl::kMma;
  }();
  return impl;
}
static bool k4_simt() { return k4_impl() == K4Impl::kSimt; }

static int composite_per_sm() {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, composite_kernel, 32 * kCompWarps, 0);
    if (per_sm < 1) per_sm = 1;
  }
  return per_sm;
}

// Part length of K3's work items, decided per forward state (so the device
// and host-buffer paths cut, and therefore sum, every list identically):
// 256 kernels, halved (down to 32) while the state has fewer items than twice
// the GPU's warp slots (small workloads: the train step renders one view).
// Measured at cfg3 (B200, scalar K3): 1.37 ms at 256 and 512, 1.40 at 128,
// 1.47 at 64, 1.54 uncut; the longest item of the unit-ordered host path
// takes 0.2 ms at 256 vs 0.4 at 512, which sets when the first D2H copy can
// start. With the FP32x2 K3: 1.20 ms at 256, 1.185 at 512, but e2e 13.0k vs
// 12.4-12.6k projections/s, so 256 stays.
static int composite_part_len(Ctx* c, const sct_fwd* s) {
  if (const char* e = std::getenv("SCT_K3_PART")) return std::max(32, atoi(e));
  const long long lists = (long long)s->det.tiles_x * s->det.tiles_y * s->n_views;
  const long long slots = (long long)c->sm_count * composite_per_sm() * kCompWarps;
  int len = 256;
  while (len > 32 && lists + s->n_pairs / len < 2 * slots) len /= 2;
  return len;
}

// K3 work items of a (view, tile) order: per list max(1, ceil(n / part_len))
// items (scan of the counts), plus the partial tiles and the per-list
// counters of the last-part reduction (slot 27: counts, firsts, items, the
// item count, counters; slot 24: partial tiles).
struct K3Work {
  const int4* items = nullptr;
  const int* first = nullptr;  // first item of each list (order position)
  const int* n_items = nullptr;
  int* tile_cnt = nullptr;
  float* partial = nullptr;
  int part_len = 0;
  long long max_items = 0;  // host-side bound of *n_items
};

// ranges: the lists the order's indices refer to (s->d_ranges + T v0 for a
// view-range order). Cached: rebuilt only when the order (generation), the
// part length or the list count changed.
static bool k3_two_pass() {  // SCT_K3_TWOPASS=0 (diagnostic): k3_parts + CUB scan + k3_items
  static const bool on = [] {
    const char* e = std::getenv("SCT_K3_TWOPASS");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
static int list_work(Ctx* c, const sct_fwd* s, const int* order, const int2* ranges, int n, int part_len,
                     K3Work& kw) {
  kw.part_len = part_len;
  Ctx::ItemsKey& key = c->items_key;
  const int slot = 27;
  const long long max_items = (long long)n + s->n_pairs / kw.part_len + 1;
  char* buf = nullptr;
  const size_t n4 = ((size_t)n + 3) & ~(size_t)3;  // int4 alignment of the item array
  const size_t bytes = sizeof(int) * (2 * n4 + 4) + sizeof(int4) * max_items + sizeof(int) * max_items;
  const bool hit = key.gen == c->order_gen && key.part == kw.part_len && key.n == n;
  SCT_TRY(stage_buf(c, slot, bytes, (void**)&buf));
  int* count = reinterpret_cast<int*>(buf);
  int* first = count + n4;
  int* n_items = first + n4;
  int4* items = reinterpret_cast<int4*>(n_items + 4);
  int* tile_cnt = reinterpret_cast<int*>(items + max_items);
  SCT_TRY(stage_buf(c, 24, sizeof(float) * 256 * (size_t)max_items, (void**)&kw.partial));
  kw.items = items;
  kw.first = first;
  kw.n_items = n_items;
  kw.tile_cnt = tile_cnt;
  kw.max_items = max_items;
  if (hit) return SCT_OK;  // (K3's last parts leave the counters zeroed)
  key.gen = 0;
  {
    KScope _ks(c, "K2_k3_items");
    // the one-CTA scan up to 4096 lists (train step: 256); beyond, the
    // multi-CTA parts + CUB scan (10-view shard, 10 240 lists: 19 vs 24 us)
    static const int small_max = [] {  // SCT_K3_SMALL (diagnostic): the one-CTA scan's list-count limit
      const char* e = std::getenv("SCT_K3_SMALL");
      return e ? std::min(kSmallWork, atoi(e)) : 4096;
    }();
    if (n <= small_max) {
      pdl_launch(k3_first_small_kernel, dim3(1), dim3(kSmallWorkThreads), 0, c->stream, ranges, order, n, kw.part_len, count, first);
    } else if (k3_two_pass()) {
      const int nb = (n + kK3Block - 1) / kK3Block;
      int* bsum = nullptr;
      SCT_TRY(stage_buf(c, 26, sizeof(int) * (size_t)nb, (void**)&bsum));
      pdl_launch(k3_block_parts_kernel, dim3(nb), dim3(kK3Block), 0, c->stream, ranges, order, n, kw.part_len, count,
                 bsum);
      pdl_launch(k3_block_items_kernel, dim3(nb), dim3(kK3Block), 0, c->stream, (const int*)order, (const int*)count,
                 n, (const int*)bsum, first, items, n_items, tile_cnt, max_items);
      key.gen = c->order_gen;
      key.part = kw.part_len;
      key.n = n;
      return SCT_OK;
    } else {
      pdl_launch(k3_parts_kernel, dim3(grid_cap(c, n, 256)), dim3(256), 0, c->stream, ranges, order, n, kw.part_len, count);
      size_t tmp = 0;
      SCT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, count, first, n, c->stream));
      SCT_TRY(ensure_cub_tmp(c, tmp));
      tmp = c->cub_tmp_bytes;
      SCT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(c->cub_tmp, tmp, count, first, n, c->stream));
    }
    pdl_launch(k3_items_kernel, dim3(grid_cap(c, std::max<long long>(n, max_items / 4), 256)), dim3(256), 0, c->stream, order, count, first, n, items, n_items, tile_cnt, max_items);
  }
  key.gen = c->order_gen;
  key.part = kw.part_len;
  key.n = n;
  return SCT_OK;
}

static int composite_launch(Ctx* c, const sct_fwd* s, const int* order, float* images, const UnitSync& us,
                            int pos0 = 0, int pos1 = -1) {
  const int T = s->det.tiles_x * s->det.tiles_y;
  const int n = T * s->n_views;
  if (!order) {
    set_error("CUDA error: tile order");
    return SCT_ERR_CUDA;
  }
  K3Work kw;
  SCT_TRY(list_work(c, s, order, s->d_ranges, n, composite_part_len(c, s), kw));
  int* work = nullptr;
  SCT_TRY(stage_buf(c, 20, sizeof(int) * 4, (void**)&work));
  SCT_TRY(launch_zero(c, work, sizeof(int)));
  const int blocks = (int)std::min<long long>((long long)c->sm_count * composite_per_sm(),
                                              (kw.max_items + kCompWarps - 1) / kCompWarps);
  KScope _ks(c, "K3_composite");
  pdl_launch(composite_kernel, dim3(blocks), dim3(32 * kCompWarps), 0, c->stream, s->d_ranges, s->d_vals, s->d_rec, s->det.tiles_x, T,
                                                              s->det.w, s->det.h, kw.items, kw.n_items, kw.part_len,
                                                              work, kw.tile_cnt, kw.partial, images, us,
                                                              pos0 > 0 ? kw.first + pos0 : nullptr,
                                                              pos1 >= 0 && pos1 < n ? kw.first + pos1 : nullptr);
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

// All views of the forward state, longest lists first.
void launch_raster_composite(Ctx* c, const sct_fwd* s, float* images) {
  if (s->n_views <= 0) return;
  composite_launch(c, s, cached_tile_order(c, s, 0, s->n_views), images, UnitSync{});
}

bool raster_units_supported(Ctx* c, const sct_fwd* s) { return !k4_simt(); }

// Host-buffer forward: one composite over all views in unit order; the last
// finished tile of unit u publishes unit_flags[u] (the copy stream waits on
// it), so the D2H copies overlap the composite.
int launch_raster_composite_units(Ctx* c, const sct_fwd* s, float* images, UnitSync us, int pos0, int pos1) {
  us.per_view = s->det.tiles_x * s->det.tiles_y;
  return composite_launch(c, s, unit_tile_order(c, s, us.units), images, us, pos0, pos1);
}

void launch_raster_backward_stats(Ctx* c, const sct_fwd* s, const float* dL, float4* pair_stats, int v0, int nv,
                                  float* item_stats, const UnitSync* us) {
  if (s->n_pairs == 0) return;
  if (nv <= 0) nv = s->n_views - v0;
  if (nv <= 0) return;
  const int T = s->det.tiles_x * s->det.tiles_y;
  dim3 grid(T, nv);
  const bool simt = k4_simt();
  KScope _ks(c, "K4_backward_stats");
  float* ps = reinterpret_cast<float*>(pair_stats);
  if (simt) {
    pdl_launch(backward_stats_kernel, dim3(grid), dim3(kBwdThreads), 0, c->stream, s->d_ranges, s->d_vals, s->d_rec, s->d_rect,
                                                               s->d_offset, s->det.tiles_x, T, s->det.w, s->det.h,
                                                               v0, dL, ps, item_stats);
    return;
  }
  if (us) {  // host path: all views in unit order, each unit waiting for its H2D copy
    v0 = 0;
    nv = s->n_views;
  }
  // SCT_K4_UNIT_ORDER=N (diagnostic): the device path in the host path's N-unit order
  static const int dbg_units = [] {
    const char* e = std::getenv("SCT_K4_UNIT_ORDER");
    return e ? atoi(e) : 0;
  }();
  const int* order = us ? unit_tile_order(c, s, us->units)
                        : (dbg_units > 0 && v0 == 0 && nv == s->n_views ? unit_tile_order(c, s, dbg_units)
                                                                        : cached_tile_order(c, s, v0, nv));
  if (!order) return;
  // small workloads: several CTAs per list (>= 16 kernels each on average,
  // up to 16 parts) while the grid stays within ~8 waves of 4-warp CTAs: the
  // longest lists bound the kernel (cfg2 train step, one view of 256 tiles:
  // 1 / 2 / 4 / 8 / 16 parts -> 188 / 56 / 37 / 30 / 28 us); large workloads
  // (cfg3 and its 8-rank shards) keep one CTA per list
  const long long total = (long long)T * nv;
  const double avg_len = total > 0 ? (double)s->n_pairs / (double)total : 0.0;
  int parts = 1;
  while (parts < 16 && total * parts * 2 <= (long long)c->sm_count * 64 && avg_len / (2 * parts) >= 16.0) parts *= 2;
  static const int forced_parts = [] {  // SCT_K4_PARTS (diagnostic): force the parts per list
    const char* e = std::getenv("SCT_K4_PARTS");
    return e ? std::max(1, std::min(64, atoi(e))) : 0;
  }();
  if (forced_parts && !us) parts = forced_parts;
  UnitSync ks = us ? *us : UnitSync{};
  ks.per_view = T * parts;
  if (k4_impl() == K4Impl::kTc && !ks.ready && !ks.done) {
    int* work = nullptr;
    if (stage_buf(c, 20, sizeof(int) * 4, (void**)&work) != SCT_OK) return;
    cudaMemsetAsync(work + 1, 0, sizeof(int), c->stream);
    const long long n_work = total * parts;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((long long)c->sm_count * kTcCtas, n_work));
    pdl_launch(backward_stats_tc_kernel, dim3(blocks), dim3(kTcThreads), 0, c->stream, s->d_ranges, s->d_vals, s->d_rec, s->d_rect, s->d_offset, s->det.tiles_x, T, s->det.w, s->det.h, v0, order,
        parts, (int)n_work, work + 1, dL, ps, item_stats, ks);
    return;
  }
  // 2-warp CTAs only for large workloads: with fewer lists the longest list,
  // worked by one CTA, becomes the kernel's tail (8-rank cfg3 shard, 10 views:
  // 344 us with 2 warps vs 272 with 4; all 75 views: 1.77 vs 1.80 ms)
  static const int forced_w = [] {  // SCT_K4_W=2|4 (diagnostic)
    const char* e = std::getenv("SCT_K4_W");
    return e ? atoi(e) : 0;
  }();
  const bool wide = forced_w ? forced_w == 4 : (parts > 1 || total < kK4LargeLists);
  if (wide)
    pdl_launch(backward_stats_mma_kernel<kMmaWarpsSmall>, dim3((unsigned)(total * parts)), dim3(32 * kMmaWarpsSmall), 0, c->stream, s->d_ranges, s->d_vals, s->d_rec, s->d_rect, s->d_offset, s->det.tiles_x, T, s->det.w, s->det.h, v0, order,
        parts, dL, ps, item_stats, ks);
  else
    pdl_launch(backward_stats_mma_kernel<kMmaWarpsLarge>, dim3((unsigned)(total * parts)), dim3(32 * kMmaWarpsLarge), 0, c->stream, s->d_ranges, s->d_vals, s->d_rec, s->d_rect, s->d_offset, s->det.tiles_x, T, s->det.w, s->det.h, v0, order,
        parts, dL, ps, item_stats, ks);
}

}  // namespace sct
