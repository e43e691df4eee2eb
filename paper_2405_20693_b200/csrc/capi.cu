// C ABI (include/splatct_gpu.h): contexts, forward state, binning pipeline
// (scan -> emit -> stable radix sort -> ranges) and the host-buffer entry points.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "sct_internal.cuh"

namespace sct {

static thread_local std::string g_last_error;

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SCT_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
void set_error(const std::string& msg) { g_last_error = msg; }

DetParams make_det(const sct_scanner& s) {  // geometry.cpp:88-98
  DetParams d;
  d.w = s.det_res_px[0];
  d.h = s.det_res_px[1];
  d.parallel = s.parallel_beam != 0;
  d.fx = d.parallel ? d.w / s.det_size_mm[0] : s.l_sd_mm * d.w / s.det_size_mm[0];
  d.fy = d.parallel ? d.h / s.det_size_mm[1] : s.l_sd_mm * d.h / s.det_size_mm[1];
  d.cx = 0.5 * d.w;
  d.cy = 0.5 * d.h;
  d.near_clip = s.near_clip_mm > 0.0 ? s.near_clip_mm : 0.01 * s.l_so_mm;
  d.tiles_x = (d.w + kTilePx - 1) / kTilePx;
  d.tiles_y = (d.h + kTilePx - 1) / kTilePx;
  return d;
}

ViewParams make_view(const sct_scanner& s, double theta) {  // geometry.cpp:76-86
  const double sn = std::sin(theta), cs = std::cos(theta);
  ViewParams v;
  const double r[9] = {-sn, cs, 0.0, 0.0, 0.0, -1.0, -cs, -sn, 0.0};
  for (int i = 0; i < 9; ++i) v.rot[i] = r[i];
  v.t[0] = 0.0;
  v.t[1] = 0.0;
  v.t[2] = s.l_so_mm;
  return v;
}

RasterParams make_raster(const sct_raster_opts& o) {
  RasterParams r;
  r.mode = o.mode;
  r.dilation_compensation = o.dilation_compensation;
  r.freeze_jacobian = o.freeze_jacobian;
  r.eps2 = o.lowpass_eps_px * o.lowpass_eps_px;
  r.cull = o.cull_mahalanobis;
  return r;
}

KScope::KScope(Ctx* ctx, const char* name, bool engine_kernel, cudaStream_t stream)
    : c(ctx), st(stream ? stream : ctx->stream) {
  if (engine_kernel) c->launches++;
  if (!c->timing) return;
  TimingRec r;
  r.name = name;
  for (cudaEvent_t* e : {&r.a, &r.b}) {
    if (!c->pool.empty()) {
      *e = c->pool.back();
      c->pool.pop_back();
    } else {
      cudaEventCreate(e);
    }
  }
  cudaEventRecord(r.a, st);
  idx = (int)c->recs.size();
  c->recs.push_back(r);
}
KScope::~KScope() {
  if (idx >= 0) cudaEventRecord(c->recs[idx].b, st);
}

int dev_alloc(Ctx* c, void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 16;
  SCT_CUDA_TRY(cudaMallocAsync(p, bytes, c->stream));
  return SCT_OK;
}
void dev_free(Ctx* c, void* p) {
  if (p) cudaFreeAsync(p, c->stream);
}
int stage_buf(Ctx* c, int slot, size_t bytes, void** p) {
  if (bytes > c->stage_bytes[slot]) {
    if (c->stage[slot]) cudaFreeAsync(c->stage[slot], c->stream);
    c->stage[slot] = nullptr;
    c->stage_bytes[slot] = 0;
    SCT_CUDA_TRY(cudaMallocAsync(&c->stage[slot], bytes, c->stream));
    c->stage_bytes[slot] = bytes;
  }
  *p = c->stage[slot];
  return SCT_OK;
}

// Staging slots are (re)allocated in `stream` order from the stream-ordered
// pool; before another stream (the copy stream) touches them, it must be
// ordered after those allocations (and after any cudaFreeAsync of the slot's
// previous block).
int stage_publish(Ctx* c, cudaStream_t other) {
  SCT_CUDA_TRY(cudaEventRecord(c->ev_stage, c->stream));
  SCT_CUDA_TRY(cudaStreamWaitEvent(other, c->ev_stage, 0));
  return SCT_OK;
}

int ensure_cub_tmp(Ctx* c, size_t bytes) {
  if (bytes <= c->cub_tmp_bytes) return SCT_OK;
  if (c->cub_tmp) cudaFreeAsync(c->cub_tmp, c->stream);
  c->cub_tmp = nullptr;
  const size_t b = bytes + bytes / 4 + 4096;
  SCT_CUDA_TRY(cudaMallocAsync(&c->cub_tmp, b, c->stream));
  c->cub_tmp_bytes = b;
  return SCT_OK;
}

static int bits_for(uint64_t n) {  // smallest b with 2^b >= n (n >= 1)
  int b = 0;
  while ((1ull << b) < n) ++b;
  return b;
}

// exclusive scan of count[0..n] (count[n] == 0) into offset[0..n]; returns offset[n].
// The total is first summed in int64 (cub Reduce into a 64-bit output): an
// int32 total between 2^31 and 2^32 + 2^31 would wrap to a plausible value.
// cap > 0 (capacity mode): no host readback — *total = cap, and a device guard
// flags c->overflow and empties the items (boxes box_a / box_b) when the pairs
// exceed it (launch_capacity_guard).
// the one-CTA count scan measured slower than CUB's two passes at the train
// step's 50k items (29 vs 13 us: one CTA walks the tiles at memory latency),
// so it only takes tiny inputs
constexpr int64_t kCountScanSmallUse = 4096;
// max_per_item > 0: no item counts more than that, so when (n + 1) * max_per_item
// fits in int32 the int32 scan cannot wrap and the int64 reduction is skipped
// (two launches fewer: the train step's single-view and TV binnings)
static int scan_counts(Ctx* c, int32_t* count, int32_t* offset, int64_t n, int64_t* total, int64_t cap = 0,
                       short4* box_a = nullptr, short4* box_b = nullptr, int64_t max_per_item = 0) {
  const bool no_wrap = max_per_item > 0 && (n + 1) * max_per_item < (int64_t)INT32_MAX;
  SCT_TRY(launch_zero(c, count + n, sizeof(int32_t)));
  if (n + 1 <= kCountScanSmallUse) {  // one CTA: scan, int64 total and capacity guard
    {
      KScope _ks(c, "K2_scan(cub)", false);
      launch_count_scan_small(c, count, offset, n, cap, box_a, box_b);
    }
    if (cap > 0) {
      *total = cap;
      return SCT_OK;
    }
    SCT_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(c->pinned_count) + 64, c->sum64, sizeof(long long),
                                 cudaMemcpyDeviceToHost, c->stream));
  } else {
    long long* d_sum = c->sum64;
    size_t tmp = 0;
    if (!no_wrap) {
      SCT_CUDA_TRY(cub::DeviceReduce::Sum(nullptr, tmp, count, d_sum, n + 1, c->stream));
      SCT_TRY(ensure_cub_tmp(c, tmp));
      tmp = c->cub_tmp_bytes;
      SCT_CUDA_TRY(cub::DeviceReduce::Sum(c->cub_tmp, tmp, count, d_sum, n + 1, c->stream));
      SCT_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(c->pinned_count) + 64, d_sum, sizeof(long long),
                                   cudaMemcpyDeviceToHost, c->stream));
    }
    tmp = 0;
    SCT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, count, offset, n + 1, c->stream));
    SCT_TRY(ensure_cub_tmp(c, tmp));
    tmp = c->cub_tmp_bytes;
    {
      KScope _ks(c, "K2_scan(cub)", false);
      SCT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(c->cub_tmp, tmp, count, offset, n + 1, c->stream));
    }
    if (cap > 0) {
      launch_capacity_guard(c, count, offset, n, box_a, box_b, cap, no_wrap);
      *total = cap;
      return SCT_OK;
    }
  }
  int32_t t = 0;
  long long t64 = 0;
  SCT_CUDA_TRY(cudaMemcpyAsync(c->pinned_count, offset + n, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  std::memcpy(&t, c->pinned_count, sizeof(int32_t));
  if (no_wrap)
    t64 = t;
  else
    std::memcpy(&t64, reinterpret_cast<char*>(c->pinned_count) + 64, sizeof(long long));
  if (t64 > INT32_MAX || t < 0) {
    set_error("DataError: more than 2^31-1 (tile, kernel) pairs in one call; split the views into batches");
    return SCT_ERR_DATA;
  }
  *total = t;
  return SCT_OK;
}

// stable LSD radix sort of (key, value) pairs on key bits [0, end_bit)
template <typename KeyT>
static int sort_pairs(Ctx* c, KeyT*& keys, int32_t*& vals, int64_t n, int end_bit) {
  if (n == 0) return SCT_OK;
  KeyT* k2 = nullptr;
  int32_t* v2 = nullptr;
  SCT_TRY(dev_alloc(c, (void**)&k2, n * sizeof(KeyT)));
  SCT_TRY(dev_alloc(c, (void**)&v2, n * sizeof(int32_t)));
  size_t tmp = 0;
  SCT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, k2, vals, v2, (int)n, 0, end_bit, c->stream));
  SCT_TRY(ensure_cub_tmp(c, tmp));
  tmp = c->cub_tmp_bytes;
  {
    KScope _ks(c, "K2_sort(cub)", false);
    SCT_CUDA_TRY(
        cub::DeviceRadixSort::SortPairs(c->cub_tmp, tmp, keys, k2, vals, v2, (int)n, 0, end_bit, c->stream));
  }
  dev_free(c, keys);
  dev_free(c, vals);
  keys = k2;
  vals = v2;
  return SCT_OK;
}

static int check_cloud(const sct_cloud* cl) {
  if (!cl || cl->m < 0) {
    set_error("ConfigError: null or negative-size cloud");
    return SCT_ERR_CONFIG;
  }
  if (cl->m > 0 && (!cl->rho_raw || !cl->pos || !cl->scale_raw || !cl->rot)) {
    set_error("ConfigError: cloud has null parameter arrays");
    return SCT_ERR_CONFIG;
  }
  if (cl->m > (int64_t)INT32_MAX) {
    set_error("ConfigError: more than 2^31-1 kernels");
    return SCT_ERR_CONFIG;
  }
  return SCT_OK;
}

static int check_scanner(const sct_scanner* s) {
  if (!s || s->det_res_px[0] <= 0 || s->det_res_px[1] <= 0 || !(s->det_size_mm[0] > 0.0) ||
      !(s->det_size_mm[1] > 0.0) || !(s->l_so_mm > 0.0) || !(s->l_sd_mm > s->l_so_mm)) {
    set_error("ConfigError: scanner: invalid detector resolution/size or distances (geometry.cpp:26-34)");
    return SCT_ERR_CONFIG;
  }
  if (s->det_res_px[0] > 32767 * kTilePx || s->det_res_px[1] > 32767 * kTilePx) {
    set_error("ConfigError: detector too large");
    return SCT_ERR_CONFIG;
  }
  return SCT_OK;
}

static int check_grid(const sct_grid* g) {
  if (!g || g->dims[0] <= 0 || g->dims[1] <= 0 || g->dims[2] <= 0 || !(g->spacing_mm[0] > 0.0) ||
      !(g->spacing_mm[1] > 0.0) || !(g->spacing_mm[2] > 0.0)) {
    set_error("ConfigError: grid dims and spacing must be positive");
    return SCT_ERR_CONFIG;
  }
  const uint64_t nb = (uint64_t)((g->dims[0] + 7) / 8) * ((g->dims[1] + 7) / 8) * ((g->dims[2] + 7) / 8);
  if (nb >= (1ull << 31)) {
    set_error("ConfigError: grid too large");
    return SCT_ERR_CONFIG;
  }
  return SCT_OK;
}

// ------------------------------------------------------------------ voxel binning
struct VoxelBins {
  int32_t bx = 0, by = 0, bz = 0, zb0 = 0, zb1 = 0;
  int64_t n_pairs = 0;
  float4* rec = nullptr;
  short4* lo = nullptr;
  short4* hi = nullptr;
  int32_t* count = nullptr;
  int32_t* offset = nullptr;
  void* keys = nullptr;  // brick ids, uint16 when they fit
  int32_t* vals = nullptr;
  int2* ranges = nullptr;
  void release(Ctx* c) {
    dev_free(c, rec);
    dev_free(c, lo);
    dev_free(c, hi);
    dev_free(c, count);
    dev_free(c, offset);
    dev_free(c, keys);
    dev_free(c, vals);
    dev_free(c, ranges);
    rec = nullptr;
    lo = hi = nullptr;
    count = offset = nullptr;
    keys = nullptr;
    vals = nullptr;
    ranges = nullptr;
  }
};

static int voxel_bin(Ctx* c, const sct_cloud& cl, const sct_grid& g, double cull, int32_t zb0, int32_t zb1,
                     VoxelBins& b) {
  b.bx = (g.dims[0] + kTileVox - 1) / kTileVox;
  b.by = (g.dims[1] + kTileVox - 1) / kTileVox;
  b.bz = (g.dims[2] + kTileVox - 1) / kTileVox;
  b.zb0 = zb0 < 0 ? 0 : (zb0 > b.bz ? b.bz : zb0);
  b.zb1 = zb1 > b.bz ? b.bz : (zb1 < b.zb0 ? b.zb0 : zb1);
  const int64_t m = cl.m;
  const int64_t nbr = (int64_t)b.bx * b.by * b.bz;
  SCT_TRY(dev_alloc(c, (void**)&b.rec, 3 * m * sizeof(float4)));
  SCT_TRY(dev_alloc(c, (void**)&b.lo, m * sizeof(short4)));
  SCT_TRY(dev_alloc(c, (void**)&b.hi, m * sizeof(short4)));
  SCT_TRY(dev_alloc(c, (void**)&b.count, (m + 1) * sizeof(int32_t)));
  SCT_TRY(dev_alloc(c, (void**)&b.offset, (m + 1) * sizeof(int32_t)));
  SCT_TRY(dev_alloc(c, (void**)&b.ranges, nbr * sizeof(int2)));
  // the counting scatter writes every brick range from its scan (m > 0)
  const bool scatter = bin_scatter_fits(b.bx, b.by, b.bz);
  if (!scatter || m == 0) SCT_CUDA_TRY(cudaMemsetAsync(b.ranges, 0, nbr * sizeof(int2), c->stream));
  launch_voxel_preprocess(c, cl, g, cull, b.zb0, b.zb1, b.bx, b.by, b.rec, b.lo, b.hi, b.count);
  // Brick lists: the stable counting scatter (raster.cu launch_bin_scatter)
  // when the brick table fits in shared memory, else emit + radix sort.
  // Capacity mode (sct_ctx_set_capacity): no host readback of the pair count;
  // the buffers hold cap pairs (sort path: the unused tail carries a padding
  // key beyond every brick id, so it sorts last and the range scan skips it).
  const int64_t cap = c->cap_voxel;
  SCT_TRY(scan_counts(c, b.count, b.offset, m, &b.n_pairs, cap, b.lo, b.hi, (int64_t)b.bx * b.by * b.bz));
  if (scatter) {
    SCT_TRY(dev_alloc(c, (void**)&b.vals, std::max<int64_t>(b.n_pairs, 1) * sizeof(int32_t)));
    SCT_TRY(launch_bin_scatter(c, 1, m, b.bx, b.by, b.bz, b.lo, b.hi, b.vals, b.ranges, b.n_pairs, nullptr));
    SCT_CUDA_TRY(cudaGetLastError());
    return SCT_OK;
  }
  const int bits = bits_for((uint64_t)(cap > 0 ? nbr + 1 : nbr));
  const bool k16 = bits <= 16;
  const size_t ksz = k16 ? sizeof(uint16_t) : sizeof(uint32_t);
  SCT_TRY(dev_alloc(c, &b.keys, std::max<int64_t>(b.n_pairs, 1) * ksz));
  SCT_TRY(dev_alloc(c, (void**)&b.vals, std::max<int64_t>(b.n_pairs, 1) * sizeof(int32_t)));
  if (cap > 0) {
    SCT_CUDA_TRY(cudaMemsetAsync(b.keys, 0xff, b.n_pairs * ksz, c->stream));
    SCT_CUDA_TRY(cudaMemsetAsync(b.vals, 0, b.n_pairs * sizeof(int32_t), c->stream));
  }
  launch_voxel_emit(c, m, b.lo, b.hi, b.offset, b.bx, b.by, b.keys, k16, b.vals, cap > 0 ? cap : INT64_MAX);
  if (bits > 0) {
    if (k16) {
      uint16_t* kp = static_cast<uint16_t*>(b.keys);
      SCT_TRY(sort_pairs(c, kp, b.vals, b.n_pairs, bits));
      b.keys = kp;
    } else {
      uint32_t* kp = static_cast<uint32_t*>(b.keys);
      SCT_TRY(sort_pairs(c, kp, b.vals, b.n_pairs, bits));
      b.keys = kp;
    }
  }
  launch_key_ranges(c, b.n_pairs, b.keys, k16, b.ranges, nbr);
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

}  // namespace sct

namespace sct {
namespace {
// Forward-state initialisation in one launch: the view matrices arrive as a
// kernel parameter (no pageable host->device copy, whose copy-engine round trip
// costs more than a launch), the tile ranges are zeroed and the capacity-mode
// pair total reset.
constexpr int kViewPack = 16;
struct ViewPack {
  ViewParams v[kViewPack];
};
__global__ void fwd_init_kernel(ViewPack p, int nv, ViewParams* dst, int2* ranges, int64_t n_ranges, int32_t* total) {
  pdl_prologue();
  if (blockIdx.x == 0 && threadIdx.x < nv) dst[threadIdx.x] = p.v[threadIdx.x];
  if (total && blockIdx.x == 0 && threadIdx.x == 0) *total = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_ranges; i += (int64_t)gridDim.x * blockDim.x)
    ranges[i] = make_int2(0, 0);
}

__global__ void __launch_bounds__(256) zero_kernel(uint32_t* __restrict__ p, long long n_words) {
  pdl_prologue();
  const long long n4 = (reinterpret_cast<uintptr_t>(p) & 15) == 0 ? n_words / 4 : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  uint4* p4 = reinterpret_cast<uint4*>(p);
  for (long long i = t; i < n4; i += stride) p4[i] = make_uint4(0u, 0u, 0u, 0u);
  for (long long i = 4 * n4 + t; i < n_words; i += stride) p[i] = 0u;
}

int fwd_init(Ctx* c, const std::vector<ViewParams>& hv, ViewParams* d_views, int2* ranges, int64_t n_ranges,
             int32_t* total) {
  for (size_t v0 = 0; v0 < hv.size() || v0 == 0; v0 += kViewPack) {
    ViewPack p;
    const int nv = (int)std::min<size_t>(kViewPack, hv.size() - v0);
    for (int k = 0; k < nv; ++k) p.v[k] = hv[v0 + k];
    const bool first = v0 == 0;
    const int grid = first ? (int)std::max<int64_t>(1, std::min<int64_t>((n_ranges + 255) / 256, 4 * c->sm_count)) : 1;
    pdl_launch(fwd_init_kernel, dim3(grid), dim3(256), 0, c->stream, p, nv, d_views + v0, ranges, first ? n_ranges : 0,
                                                 first ? total : nullptr);
    ++c->launches;
    if (hv.empty()) break;
  }
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}
}  // namespace

int launch_zero(Ctx* c, void* p, size_t bytes) {
  const long long words = (long long)(bytes / 4);
  if (words == 0) return SCT_OK;
  const long long b = std::min<long long>((words / 4 + 255) / 256 + 1, (long long)c->sm_count * 8);
  pdl_launch(zero_kernel, dim3((unsigned)b), dim3(256), 0, c->stream, static_cast<uint32_t*>(p), words);
  ++c->launches;
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}
}  // namespace sct

using namespace sct;

// the per-item offsets of a state binned without them (atomic-mode forward)
// when a deterministic backward needs its slots
static int ensure_item_offsets(Ctx* c, sct_fwd* s) {
  if (s->offsets_ready) return SCT_OK;
  int64_t total = 0;
  SCT_TRY(scan_counts(c, s->d_count, s->d_offset, s->n_items, &total, s->n_pairs, s->d_rect, nullptr,
                      (int64_t)s->det.tiles_x * s->det.tiles_y));
  s->offsets_ready = true;
  return SCT_OK;
}

static void free_state_buffers(sct_fwd* s) {
  Ctx* c = s->ctx;
  if (s->defer) {  // a split scatter never completed (error path)
    dev_free(c, s->defer->H);
    dev_free(c, s->defer->seg);
    dev_free(c, s->defer->tb);
    delete s->defer;
    s->defer = nullptr;
  }
  dev_free(c, s->d_views);
  dev_free(c, s->d_rec);
  dev_free(c, s->d_rect);
  dev_free(c, s->d_count);
  dev_free(c, s->d_offset);
  dev_free(c, s->d_vis);
  dev_free(c, s->d_keys);
  dev_free(c, s->d_vals);
  dev_free(c, s->d_total);
  dev_free(c, s->d_ranges);
  dev_free(c, s->d_prep);
}

extern "C" {

const char* sct_last_error(void) { return g_last_error.c_str(); }
const char* sct_version(void) { return "splatct-b200 0.1 (sm_100a)"; }

int sct_ctx_create(int device, void* stream, sct_ctx** out) {
  if (!out) return SCT_ERR_CONFIG;
  *out = nullptr;
  SCT_CUDA_TRY(cudaSetDevice(device));
  auto* c = new sct_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
    c->sm_count = sms;
  // keep freed blocks in the stream-ordered pool: steady-state calls do not
  // return memory to the driver
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // Pre-grow the pool (SCT_POOL_RESERVE_MB, default 12288): growing it maps
    // new physical memory, which on the GPU VMs stalls the calling thread for
    // up to hundreds of ms — paid here once instead of inside the first steps
    // (measured: steps 2-9 after a sync ran 7-650 ms instead of 5.3 ms).
    size_t mb = 12288;
    if (const char* e = std::getenv("SCT_POOL_RESERVE_MB")) mb = (size_t)std::max(0L, atol(e));
    uint64_t have = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have);
    if (mb > 0 && have < (uint64_t)mb << 20) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const size_t want = std::min<size_t>((size_t)mb << 20, free_b / 4);
      void* p = nullptr;
      if (want > 0 && cudaMallocAsync(&p, want, (cudaStream_t)stream) == cudaSuccess) {
        cudaFreeAsync(p, (cudaStream_t)stream);
        cudaStreamSynchronize((cudaStream_t)stream);
      }
      cudaGetLastError();
    }
  }
  if (cudaMallocHost((void**)&c->pinned_count, 128) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    set_error("CUDA error: context host allocations failed");
    return SCT_ERR_CUDA;
  }
  for (int a = 0; a < Ctx::kChunkEvents; ++a) {
    cudaEventCreateWithFlags(&c->ev_compute[a], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_copy[a], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_stage, cudaEventDisableTiming);
  // unit signal words: 3 flag arrays, 2 counter arrays, the error word
  // (device memory: kernel-side polls of mapped host words cost a PCIe read
  // each, measured 50x slower for K4)
  char* u = nullptr;
  const size_t words = (6 * Ctx::kMaxUnits * sizeof(uint32_t) + 15) & ~size_t(15);
  if (cudaMalloc((void**)&u, words + 32) != cudaSuccess || cudaMemset(u, 0, words + 32) != cudaSuccess) {
    sct_ctx_destroy(c);
    set_error("CUDA error: context signal allocation failed");
    return SCT_ERR_CUDA;
  }
  c->unit_flags = reinterpret_cast<uint32_t*>(u);
  c->unit_done = reinterpret_cast<int*>(c->unit_flags + 3 * Ctx::kMaxUnits);
  c->unit_err = c->unit_done + 2 * Ctx::kMaxUnits;
  c->sum64 = reinterpret_cast<long long*>(u + words);
  c->overflow = reinterpret_cast<int*>(u + words + 8);
  c->fin_counter = reinterpret_cast<int*>(u + words + 16);
  *out = c;
  return SCT_OK;
}

int sct_ctx_destroy(sct_ctx* c) {
  if (!c) return SCT_OK;
  cudaStreamSynchronize(c->stream);
  comm_release(c);
  if (c->cub_tmp) cudaFree(c->cub_tmp);
  for (int a = 0; a < Ctx::kStageSlots; ++a)
    if (c->stage[a]) cudaFree(c->stage[a]);
  if (c->pinned_count) cudaFreeHost(c->pinned_count);
  for (int a = 0; a < Ctx::kChunkEvents; ++a) {
    if (c->ev_compute[a]) cudaEventDestroy(c->ev_compute[a]);
    if (c->ev_copy[a]) cudaEventDestroy(c->ev_copy[a]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_stage) cudaEventDestroy(c->ev_stage);
  if (c->unit_flags) cudaFree(c->unit_flags);
  delete c;
  return SCT_OK;
}

int sct_ctx_set_stream(sct_ctx* c, void* stream) {
  if (!c) return SCT_ERR_CONFIG;
  c->stream = (cudaStream_t)stream;
  return SCT_OK;
}

int sct_ctx_sync(sct_ctx* c) {
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_ctx_set_capacity(sct_ctx* c, int64_t raster_pairs, int64_t voxel_pairs) {
  if (!c || raster_pairs < 0 || voxel_pairs < 0 || raster_pairs > INT32_MAX || voxel_pairs > INT32_MAX) {
    set_error("ConfigError: capacities must be in [0, 2^31)");
    return SCT_ERR_CONFIG;
  }
  c->cap_raster = raster_pairs;
  c->cap_voxel = voxel_pairs;
  return SCT_OK;
}

int sct_ctx_take_overflow(sct_ctx* c, int32_t* overflowed) {
  if (!c || !overflowed) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  int h = 0;
  SCT_CUDA_TRY(cudaMemcpyAsync(&h, c->overflow, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (h) SCT_CUDA_TRY(cudaMemsetAsync(c->overflow, 0, sizeof(int), c->stream));
  *overflowed = h;
  return SCT_OK;
}

int sct_ctx_set_deterministic(sct_ctx* c, int d) {
  c->deterministic = d != 0;
  return SCT_OK;
}

int64_t sct_ctx_kernel_launches(const sct_ctx* c) { return c ? c->launches : 0; }

int sct_ctx_set_timing(sct_ctx* c, int enable) {
  if (!c) return SCT_ERR_CONFIG;
  c->timing = enable != 0;
  return SCT_OK;
}

// JSON {"kernel": [total_ms, launches], ...}; synchronises, then resets.
int sct_ctx_timing_report(sct_ctx* c, char* buf, int32_t buflen) {
  if (!c || !buf || buflen < 3) return SCT_ERR_CONFIG;
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  std::vector<std::pair<std::string, std::pair<double, int64_t>>> agg;
  for (auto& r : c->recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& a : agg)
      if (a.first == r.name) {
        a.second.first += ms;
        a.second.second += 1;
        found = true;
      }
    if (!found) agg.push_back({r.name, {ms, 1}});
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->recs.clear();
  std::string out = "{";
  for (size_t i = 0; i < agg.size(); ++i) {
    char tmp[256];
    snprintf(tmp, sizeof(tmp), "%s\"%s\": [%.6f, %lld]", i ? ", " : "", agg[i].first.c_str(), agg[i].second.first,
             (long long)agg[i].second.second);
    out += tmp;
  }
  out += "}";
  if ((int32_t)out.size() + 1 > buflen) {
    set_error("ConfigError: timing report buffer too small");
    return SCT_ERR_CONFIG;
  }
  std::memcpy(buf, out.c_str(), out.size() + 1);
  return SCT_OK;
}

double sct_lr_at(double lr_init, double final_ratio, int32_t t, int32_t iters) {  // trainer.cpp:34-36
  return lr_init * std::pow(final_ratio, static_cast<double>(t) / iters);
}

// ------------------------------------------------------------------ rasterizer
int sct_render_fwd(sct_ctx* c, const sct_cloud* cloud, const sct_scanner* scanner, const double* thetas,
                   int32_t n_views, const sct_raster_opts* opts, float* images, sct_fwd** state) {
  if (!c || !state || !opts) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  *state = nullptr;
  SCT_TRY(check_cloud(cloud));
  SCT_TRY(check_scanner(scanner));
  if (n_views < 1 || n_views > 65535 || !thetas) {
    set_error("ConfigError: need 1..65535 views");
    return SCT_ERR_CONFIG;
  }
  for (int v = 0; v < n_views; ++v)
    if (!std::isfinite(thetas[v])) {
      set_error("ConfigError: scanner: non-finite view angle");
      return SCT_ERR_CONFIG;
    }
  auto* s = new sct_fwd();
  s->ctx = c;
  s->id = c->next_fwd_id++;
  s->n_views = n_views;
  s->m = cloud->m;
  s->det = make_det(*scanner);
  s->rp = make_raster(*opts);
  s->opts = *opts;
  s->scanner = *scanner;
  s->s_min = cloud->s_min_mm;
  s->thetas.assign(thetas, thetas + n_views);
  const int64_t T = (int64_t)s->det.tiles_x * s->det.tiles_y;
  s->tile_bits = bits_for((uint64_t)T);
  if (s->tile_bits > 31 || s->m * (int64_t)n_views > INT32_MAX) {
    delete s;
    set_error("ConfigError: more than 2^31 (view, kernel) items or tiles; split the views into batches");
    return SCT_ERR_CONFIG;
  }
  s->n_items = s->m * n_views;
  int rc = SCT_OK;
  auto fail = [&](int r) {
    free_state_buffers(s);
    delete s;
    return r;
  };
  std::vector<ViewParams> hv(n_views);
  for (int v = 0; v < n_views; ++v) hv[v] = make_view(*scanner, thetas[v]);
  if ((rc = dev_alloc(c, (void**)&s->d_views, n_views * sizeof(ViewParams)))) return fail(rc);
  const int64_t ni = s->n_items;
  if ((rc = dev_alloc(c, (void**)&s->d_rec, 2 * ni * sizeof(float4)))) return fail(rc);
  if ((rc = dev_alloc(c, (void**)&s->d_rect, ni * sizeof(short4)))) return fail(rc);
  if ((rc = dev_alloc(c, (void**)&s->d_count, (ni + 1) * sizeof(int32_t)))) return fail(rc);
  if ((rc = dev_alloc(c, (void**)&s->d_offset, (ni + 1) * sizeof(int32_t)))) return fail(rc);
  if ((rc = dev_alloc(c, (void**)&s->d_vis, ni + 1))) return fail(rc);
  if ((rc = dev_alloc(c, (void**)&s->d_ranges, n_views * T * sizeof(int2)))) return fail(rc);
  // capacity mode: sync-free when the counting scatter applies (the radix
  // sort needs the exact count on the host)
  const bool scatter = raster_bin_scatter_fits(s->det.tiles_x, s->det.tiles_y);
  const int64_t cap = (c->cap_raster > 0 && scatter) ? c->cap_raster : 0;
  if (cap > 0 && (rc = dev_alloc(c, (void**)&s->d_total, sizeof(int32_t)))) return fail(rc);
  if ((rc = fwd_init(c, hv, s->d_views, s->d_ranges, n_views * T, s->d_total))) return fail(rc);
  if ((rc = dev_alloc(c, (void**)&s->d_prep, kPrepStride * s->m * sizeof(double)))) return fail(rc);
  launch_gauss_prep(c, *cloud, s->d_prep);
  launch_raster_preprocess(c, *cloud, s->d_prep, s->d_views, n_views, s->det, s->rp, s->d_rec, s->d_rect,
                           s->d_count, s->d_vis);
  // Binning: one stable counting scatter straight into (tile, view, kernel)
  // order when the tile table fits in shared memory (raster.cu bin_*), else
  // emit + radix sort. SCT_BIN=sort forces the latter.
  static const bool force_sort = [] {
    const char* e = std::getenv("SCT_BIN");
    return e && std::string(e) == "sort";
  }();
  // The per-item pair offsets (scan of the counts) serve the deterministic
  // backward's slots, the emit + sort path and the exact host-side count. A
  // sync-free scatter binning in the parallel-atomic mode needs none of them:
  // the column scan yields the total and flags an overflow, and the ranges
  // come out empty then (bin_ranges_kernel), so the scan is deferred to a
  // deterministic backward of this state, if one ever runs.
  if (cap > 0 && scatter && !force_sort && !c->deterministic) {
    s->n_pairs = cap;
    s->offsets_ready = false;
  } else if ((rc = scan_counts(c, s->d_count, s->d_offset, ni, &s->n_pairs, cap, s->d_rect, nullptr,
                               (int64_t)s->det.tiles_x * s->det.tiles_y))) {
    return fail(rc);
  }
  if (cap > 0) s->exact = false;
  if ((!force_sort || cap > 0) && scatter) {
    if ((rc = dev_alloc(c, (void**)&s->d_vals, std::max<int64_t>(s->n_pairs, 1) * sizeof(int32_t)))) return fail(rc);
    const int64_t split = images ? -1 : c->fwd_split_views;  // host path: the rest after the first composite
    if ((rc = launch_raster_bin_scatter(c, n_views, s->m, s->det.tiles_x, s->det.tiles_y, s->d_rect, s->d_vals,
                                        s->d_ranges, s->n_pairs, s->n_pairs, s->d_total, split, &s->defer)))
      return fail(rc);
#if SCT_CHECKED
    if (std::getenv("SCT_DCHECK_SELFTEST")) {  // checked build only: an invalid list range K3 must reject
      static const int2 bad = make_int2(1, 0);
      cudaMemcpyAsync(s->d_ranges, &bad, sizeof(int2), cudaMemcpyHostToDevice, c->stream);
      cudaStreamSynchronize(c->stream);
    }
#endif
    if (images) launch_raster_composite(c, s, images);
    if (cudaGetLastError() != cudaSuccess) {
      set_error("CUDA error: kernel launch in sct_render_fwd");
      return fail(SCT_ERR_CUDA);
    }
    *state = s;
    return SCT_OK;
  }
  // Pairs are emitted view-major (and kernel-ascending within a view), so a
  // STABLE sort on the tile bits alone already groups them by (tile, view)
  // with each list ascending in kernel index: fewer radix passes than the
  // full (view, tile) key, and 16-bit keys whenever the tile index fits.
  const bool k16 = s->tile_bits <= 16;
  const size_t ksz = k16 ? sizeof(uint16_t) : sizeof(uint32_t);
  if ((rc = dev_alloc(c, &s->d_keys, s->n_pairs * ksz))) return fail(rc);
  if ((rc = dev_alloc(c, (void**)&s->d_vals, s->n_pairs * sizeof(int32_t)))) return fail(rc);
  launch_raster_emit(c, ni, s->d_rect, s->d_offset, s->det.tiles_x, s->d_keys, k16, s->d_vals);
  if (s->tile_bits > 0) {
    if (k16) {
      uint16_t* kp = static_cast<uint16_t*>(s->d_keys);
      rc = sort_pairs(c, kp, s->d_vals, s->n_pairs, s->tile_bits);
      s->d_keys = kp;
    } else {
      uint32_t* kp = static_cast<uint32_t*>(s->d_keys);
      rc = sort_pairs(c, kp, s->d_vals, s->n_pairs, s->tile_bits);
      s->d_keys = kp;
    }
    if (rc) return fail(rc);
  }
  launch_raster_ranges(c, s->n_pairs, s->d_keys, k16, s->d_vals, s->m, T, s->d_ranges);
  if (images) launch_raster_composite(c, s, images);
  if (cudaGetLastError() != cudaSuccess) {
    set_error("CUDA error: kernel launch in sct_render_fwd");
    return fail(SCT_ERR_CUDA);
  }
  *state = s;
  return SCT_OK;
}

// chunks > 0: the upstream gradient arrives in `chunks` view chunks, chunk k
// signalled by ctx->ev_copy[k]; K4 for chunk k waits only for its own copy.
int sct_render_bwd_chunked(sct_ctx* c, sct_fwd* s, const sct_cloud* cloud, const float* dL, sct_grads* grads,
                         sct_stats* stats, int chunks, double** defer_vsum, int* defer_groups) {
  if (defer_vsum) *defer_vsum = nullptr;
  if (!c || !s || !grads || !dL) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(check_cloud(cloud));
  if (cloud->m != s->m) {
    set_error("DimMismatch: render_backward: cloud size differs from the forward state");
    return SCT_ERR_DATA;
  }
  if (s->n_items == 0) return SCT_OK;
  float4* pair_stats = nullptr;
  double* vsum = nullptr;
  // deterministic (default): per-(tile, kernel) slots reduced in the
  // reference's fixed tile order; otherwise the parallel-atomic mode of
  // SPEC.md:224-226 accumulates straight into 8-float per-item records.
  // (grow-only context buffers: slot 14 statistics, slot 15 item outputs)
  const bool atomic = !c->deterministic;
  if (!atomic) SCT_TRY(ensure_item_offsets(c, s));
  float* item_stats = nullptr;
  if (atomic) {
    SCT_TRY(stage_buf(c, 14, 8 * s->n_items * sizeof(float), (void**)&item_stats));
    SCT_TRY(launch_zero(c, item_stats, 8 * s->n_items * sizeof(float)));
  } else {
    SCT_TRY(stage_buf(c, 14, 2 * s->n_pairs * sizeof(float4), (void**)&pair_stats));
  }
  const int nch = chunks > 0 ? chunks : 1;
  SCT_TRY(stage_buf(c, 15, chain_sums_bytes(s, nch), (void**)&vsum));
  // View chunks pipeline the two backward stages: the statistics kernel of
  // chunk k+1 (FP32, issue-bound) runs on the main stream while the FP64
  // chain of chunk k (latency-bound) runs on the aux stream; items of view v
  // only receive statistics from tiles of view v, so chunk k's chain needs
  // nothing from later chunks.
  // (measured on B200 at cfg3: the overlap is neutral when the upstream
  // gradient is already resident — the issue-bound K4 yields the slots K5
  // takes — and pays off on the host-buffer path, where it also hides the
  // chunked H2D copies; so it is used there only)
  const float4* chain_src = atomic ? reinterpret_cast<const float4*>(item_stats) : pair_stats;
  for (int k = 0; k < nch; ++k) {
    const int v0 = (int)((int64_t)s->n_views * k / nch), v1 = (int)((int64_t)s->n_views * (k + 1) / nch);
    if (chunks > 0) SCT_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_copy[k], 0));
    launch_raster_backward_stats(c, s, dL, pair_stats, v0, v1 - v0, item_stats);
    if (nch > 1) {
      SCT_CUDA_TRY(cudaEventRecord(c->ev_compute[k], c->stream));
      SCT_CUDA_TRY(cudaStreamWaitEvent(c->aux_stream, c->ev_compute[k], 0));
      launch_raster_chain(c, s, *cloud, chain_src, vsum + k * chain_sums_bytes(s, 1) / 8, atomic, v0, v1,
                          c->aux_stream);
    } else {
      launch_raster_chain(c, s, *cloud, chain_src, vsum, atomic);
    }
  }
  if (nch > 1) {
    SCT_CUDA_TRY(cudaEventRecord(c->ev_join, c->aux_stream));
    SCT_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  }
  if (defer_vsum) {
    *defer_vsum = vsum;
    if (defer_groups) *defer_groups = nch;
    SCT_CUDA_TRY(cudaGetLastError());
    return SCT_OK;
  }
  launch_raster_finalize(c, s, *cloud, vsum, nch, grads, stats);
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

// ------------------------------------------------------------------ view units
// Stream memory operations (driver entry points, resolved through the
// runtime): a stream waits until a device word reaches the call's epoch, or
// writes it. Used by the host-buffer entry points so that one kernel over all
// views overlaps the per-unit copies; SCT_HOST_UNITS=0 selects the chunked
// multi-launch path instead.
typedef CUresult (*PfnStreamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamMemOps {
  PfnStreamValue32 wait = nullptr, write = nullptr;
};
static const StreamMemOps& memops() {
  static const StreamMemOps m = [] {
    StreamMemOps r;
    if (const char* e = std::getenv("SCT_HOST_UNITS"))
      if (atoi(e) == 0) return r;
    void* w = nullptr;
    void* x = nullptr;
    cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = q1;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &x, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && x) {
      r.wait = reinterpret_cast<PfnStreamValue32>(w);
      r.write = reinterpret_cast<PfnStreamValue32>(x);
    }
    cudaGetLastError();
    return r;
  }();
  return m;
}

static int stream_wait_flag(cudaStream_t st, const uint32_t* flag, uint32_t epoch) {
  if (memops().wait((CUstream)st, (CUdeviceptr)flag, epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
    set_error("CUDA error: cuStreamWaitValue32");
    return SCT_ERR_CUDA;
  }
  return SCT_OK;
}

static int stream_write_flag(cudaStream_t st, uint32_t* flag, uint32_t epoch) {
  if (memops().write((CUstream)st, (CUdeviceptr)flag, epoch, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
    set_error("CUDA error: cuStreamWriteValue32");
    return SCT_ERR_CUDA;
  }
  return SCT_OK;
}

// view units of a host transfer of `bytes` over n_views views: ~4 MB each
// SCT_HOST_SPLIT=0 keeps the forward host path's binning in one piece
static bool host_split_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SCT_HOST_SPLIT");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

static int host_units(int n_views, size_t bytes) {
  if (const char* e = std::getenv("SCT_UNIT_KB")) {
    const size_t per = (size_t)std::max(1, atoi(e)) << 10;
    return (int)std::max<size_t>(1, std::min<size_t>({(bytes + per - 1) / per, (size_t)n_views,
                                                       (size_t)Ctx::kMaxUnits}));
  }
  const size_t per = 4u << 20;
  return (int)std::max<size_t>(1, std::min<size_t>({(bytes + per - 1) / per, (size_t)n_views,
                                                     (size_t)Ctx::kMaxUnits}));
}

// SCT_UNIT_DEBUG: timing events at named points of the host-buffer paths,
// printed (ms after the first mark) at the end of the call
struct DbgMarks {
  bool on = std::getenv("SCT_UNIT_DEBUG") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void mark(cudaStream_t st, const std::string& name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.emplace_back(name, e);
  }
  void report(const char* what) {
    if (!on || ev.empty()) return;
    cudaDeviceSynchronize();
    std::fprintf(stderr, "[%s]", what);
    for (auto& p : ev) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[0].second, p.second);
      std::fprintf(stderr, " %s=%.3f", p.first.c_str(), t);
    }
    std::fprintf(stderr, "\n");
    for (auto& p : ev) cudaEventDestroy(p.second);
    ev.clear();
  }
};
static DbgMarks g_dbg;

// the error word of a kernel-side unit wait (read after the call's stream sync)
static int check_unit_err(Ctx* c) {
  int32_t* h = reinterpret_cast<int32_t*>(c->pinned_count) + 8;
  if (*h) {
    *h = 0;
    cudaMemsetAsync(c->unit_err, 0, sizeof(int), c->stream);
    cudaStreamSynchronize(c->stream);
    set_error("CUDA error: a view-unit wait timed out (host-buffer backward)");
    return SCT_ERR_CUDA;
  }
  return SCT_OK;
}

// chain groups of the units backward (measured at cfg3 with the fused view-sum
// chain, e2e per step: 1 / 2 / 4 groups 5.56 / 5.37 / 5.48 ms; a high-priority
// chain stream starts the groups earlier but slows K4 by as much)
static const int kChainGroups = [] {
  const char* e = std::getenv("SCT_CHAIN_GROUPS");
  return e ? std::max(1, atoi(e)) : 2;
}();

// Backward with the upstream gradient landing in view units (unit_flags[1][u]
// written by the copy stream): one K4 over all views waits per unit and
// publishes unit_flags[2][u]; the FP64 chain runs on the aux stream in groups
// of units, each group starting when its units' statistics are published.
static int render_bwd_units(Ctx* c, sct_fwd* s, const sct_cloud* cloud, const float* dL, sct_grads* grads,
                            sct_stats* stats, int units, uint32_t epoch, cudaEvent_t cloud_ready,
                            cudaEvent_t grads_ready) {
  SCT_TRY(check_cloud(cloud));
  if (cloud->m != s->m) {
    set_error("DimMismatch: render_backward: cloud size differs from the forward state");
    return SCT_ERR_DATA;
  }
  if (s->n_items == 0) return SCT_OK;
  const bool atomic = !c->deterministic;
  if (!atomic) SCT_TRY(ensure_item_offsets(c, s));
  float4* pair_stats = nullptr;
  float* item_stats = nullptr;
  double* vsum = nullptr;
  if (atomic) {
    SCT_TRY(stage_buf(c, 14, 8 * s->n_items * sizeof(float), (void**)&item_stats));
    SCT_CUDA_TRY(cudaMemsetAsync(item_stats, 0, 8 * s->n_items * sizeof(float), c->stream));
  } else {
    SCT_TRY(stage_buf(c, 14, 2 * s->n_pairs * sizeof(float4), (void**)&pair_stats));
  }
  const int groups = std::min(units, kChainGroups);
  SCT_TRY(stage_buf(c, 15, chain_sums_bytes(s, groups), (void**)&vsum));
  uint32_t* ready = c->unit_flags + Ctx::kMaxUnits;
  uint32_t* k4_done = c->unit_flags + 2 * Ctx::kMaxUnits;
  int* counters = c->unit_done + Ctx::kMaxUnits;
  SCT_CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(int) * units, c->stream));
  SCT_CUDA_TRY(cudaEventRecord(c->ev_join, c->stream));  // the chain stream sees the zeroing
  SCT_CUDA_TRY(cudaStreamWaitEvent(c->aux_stream, c->ev_join, 0));
  SCT_CUDA_TRY(cudaStreamWaitEvent(c->aux_stream, cloud_ready, 0));
  UnitSync us;
  us.ready = ready;
  us.done_flag = k4_done;
  us.done = counters;
  us.err = c->unit_err;
  us.epoch = epoch;
  us.units = units;
  us.n_views = s->n_views;
  g_dbg.mark(c->stream, "k4_start");
  launch_raster_backward_stats(c, s, dL, pair_stats, 0, 0, item_stats, &us);
  g_dbg.mark(c->stream, "k4_end");
  SCT_CUDA_TRY(cudaGetLastError());
  // a lost kernel-side signal only delays the chain to the end of K4
  for (int u = 0; u < units; ++u) SCT_TRY(stream_write_flag(c->stream, k4_done + u, epoch));
  const float4* chain_src = atomic ? reinterpret_cast<const float4*>(item_stats) : pair_stats;
  for (int g = 0; g < groups; ++g) {
    const int u0 = units * g / groups, u1 = units * (g + 1) / groups;
    for (int u = u0; u < u1; ++u) SCT_TRY(stream_wait_flag(c->aux_stream, k4_done + u, epoch));
    const int64_t v0 = (int64_t)s->n_views * u0 / units, v1 = (int64_t)s->n_views * u1 / units;
    g_dbg.mark(c->aux_stream, "chain" + std::to_string(g) + "_start");
    launch_raster_chain(c, s, *cloud, chain_src, vsum + g * chain_sums_bytes(s, 1) / 8, atomic, (int)v0, (int)v1,
                        c->aux_stream);
  }
  SCT_CUDA_TRY(cudaEventRecord(c->ev_join, c->aux_stream));
  SCT_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  g_dbg.mark(c->stream, "chain_end");
  SCT_CUDA_TRY(cudaStreamWaitEvent(c->stream, grads_ready, 0));
  launch_raster_finalize(c, s, *cloud, vsum, groups, grads, stats);
  g_dbg.mark(c->stream, "finalize_end");
  SCT_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<int32_t*>(c->pinned_count) + 8, c->unit_err, sizeof(int32_t),
                               cudaMemcpyDeviceToHost, c->stream));
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_render_bwd(sct_ctx* c, sct_fwd* s, const sct_cloud* cloud, const float* dL, sct_grads* grads,
                   sct_stats* stats) {
  return sct_render_bwd_chunked(c, s, cloud, dL, grads, stats, 0);
}

int sct_fwd_free(sct_fwd* s) {
  if (!s) return SCT_OK;
  free_state_buffers(s);
  delete s;
  return SCT_OK;
}

// the pair count of a state (a device read in capacity mode)
static int64_t state_pairs(sct_fwd* s) {
  if (s->exact || !s->d_total) return s->n_pairs;
  int32_t t = 0;
  if (cudaMemcpyAsync(&t, s->d_total, sizeof(int32_t), cudaMemcpyDeviceToHost, s->ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(s->ctx->stream) != cudaSuccess)
    return s->n_pairs;
  return t;
}

// Algorithmic work of a forward state: GPE = sum over (view, tile) of
// |tile list| x pixels inside the detector for that tile (the trip count of
// rasterizer.cpp:144-153, identical for rasterizer.cpp:225-241).
int sct_fwd_work(sct_fwd* s, int64_t* gpe, int64_t* n_pairs) {
  if (!s) return SCT_ERR_CONFIG;
  const int64_t T = (int64_t)s->det.tiles_x * s->det.tiles_y;
  std::vector<int2> r(T * s->n_views);
  SCT_CUDA_TRY(cudaMemcpyAsync(r.data(), s->d_ranges, r.size() * sizeof(int2), cudaMemcpyDeviceToHost,
                               s->ctx->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(s->ctx->stream));
  int64_t g = 0;
  for (int64_t k = 0; k < (int64_t)r.size(); ++k) {
    const int64_t t = k % T;
    const int tx = (int)(t % s->det.tiles_x), ty = (int)(t / s->det.tiles_x);
    const int pw = std::min(kTilePx, s->det.w - tx * kTilePx), ph = std::min(kTilePx, s->det.h - ty * kTilePx);
    g += (int64_t)(r[k].y - r[k].x) * pw * ph;
  }
  if (gpe) *gpe = g;
  if (n_pairs) *n_pairs = state_pairs(s);
  return SCT_OK;
}

int sct_fwd_info(sct_fwd* s, int64_t* n_pairs, int32_t* tiles_x, int32_t* tiles_y, int64_t* n_visible) {
  if (!s) return SCT_ERR_CONFIG;
  if (n_pairs) *n_pairs = state_pairs(s);
  if (tiles_x) *tiles_x = s->det.tiles_x;
  if (tiles_y) *tiles_y = s->det.tiles_y;
  if (n_visible) {
    std::vector<uint8_t> v(s->n_items);
    SCT_CUDA_TRY(cudaMemcpyAsync(v.data(), s->d_vis, s->n_items, cudaMemcpyDeviceToHost, s->ctx->stream));
    SCT_CUDA_TRY(cudaStreamSynchronize(s->ctx->stream));
    int64_t n = 0;
    for (uint8_t x : v) n += x;
    *n_visible = n;
  }
  return SCT_OK;
}

int sct_fwd_tile_lists(sct_fwd* s, int32_t view, int64_t* offsets, int32_t* kernel_idx) {
  if (!s || view < 0 || view >= s->n_views || !offsets) {
    set_error("ConfigError: bad view");
    return SCT_ERR_CONFIG;
  }
  Ctx* c = s->ctx;
  const int64_t T = (int64_t)s->det.tiles_x * s->det.tiles_y;
  std::vector<int2> r(T);
  SCT_CUDA_TRY(cudaMemcpyAsync(r.data(), s->d_ranges + view * T, T * sizeof(int2), cudaMemcpyDeviceToHost,
                               c->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  int64_t o = 0;
  for (int64_t t = 0; t < T; ++t) {
    offsets[t] = o;
    o += r[t].y > r[t].x ? r[t].y - r[t].x : 0;
  }
  offsets[T] = o;
  if (kernel_idx && o > 0) {
    // pairs are sorted tile-major; gather this view's sub-range of every tile
    std::vector<int32_t> all(s->n_pairs);
    SCT_CUDA_TRY(cudaMemcpyAsync(all.data(), s->d_vals, s->n_pairs * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 c->stream));
    SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const int64_t base = (int64_t)view * s->m;
    for (int64_t t = 0; t < T; ++t)
      for (int64_t k = r[t].x; k < r[t].y; ++k) kernel_idx[offsets[t] + (k - r[t].x)] = (int32_t)(all[k] - base);
  }
  return SCT_OK;
}

int sct_project_kernels(sct_ctx* c, const sct_cloud* cloud, const sct_scanner* scanner, double theta,
                        const sct_raster_opts* opts, int32_t* visible, double* rec) {
  SCT_TRY(check_cloud(cloud));
  SCT_TRY(check_scanner(scanner));
  const int64_t m = cloud->m;
  if (m == 0) return SCT_OK;
  ViewParams hv = make_view(*scanner, theta);
  ViewParams* dv = nullptr;
  int32_t* dvis = nullptr;
  double* drec = nullptr;
  SCT_TRY(dev_alloc(c, (void**)&dv, sizeof(ViewParams)));
  SCT_TRY(dev_alloc(c, (void**)&dvis, m * sizeof(int32_t)));
  SCT_TRY(dev_alloc(c, (void**)&drec, 11 * m * sizeof(double)));
  SCT_CUDA_TRY(cudaMemcpyAsync(dv, &hv, sizeof(hv), cudaMemcpyHostToDevice, c->stream));
  launch_project_export(c, *cloud, dv, make_det(*scanner), make_raster(*opts), dvis, drec);
  SCT_CUDA_TRY(cudaMemcpyAsync(visible, dvis, m * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  SCT_CUDA_TRY(cudaMemcpyAsync(rec, drec, 11 * m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  dev_free(c, dv);
  dev_free(c, dvis);
  dev_free(c, drec);
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SCT_OK;
}

// ---- host-buffer variants ----------------------------------------------------
// Number of view chunks of the backward's upstream-gradient copy when stream
// memory operations are unavailable, at most Ctx::kChunkEvents: ~20 MB per
// chunk (4 at cfg3, measured best).
static int host_chunks(size_t bytes, bool /*forward*/) {
  if (const char* e = std::getenv("SCT_HOST_CHUNKS")) return std::max(1, std::min(atoi(e), Ctx::kChunkEvents));
  const size_t per = 20u << 20;
  size_t k = (bytes + per - 1) / per;
  if (k < 1) k = 1;
  if (k > (size_t)Ctx::kChunkEvents) k = Ctx::kChunkEvents;
  return (int)k;
}

// Staging slots: 0-3 cloud arrays, 4 images, 5 upstream gradient, 6-9 grads,
// 10-12 stats, 13 volume.
static int upload_cloud(Ctx* c, const sct_cloud* h, sct_cloud* d, cudaStream_t st = nullptr) {
  if (!st) st = c->stream;
  *d = *h;
  const int64_t m = h->m;
  float** dst[4] = {&d->rho_raw, &d->pos, &d->scale_raw, &d->rot};
  float* src[4] = {h->rho_raw, h->pos, h->scale_raw, h->rot};
  const int64_t n[4] = {m, 3 * m, 3 * m, 4 * m};
  for (int a = 0; a < 4; ++a) {
    SCT_TRY(stage_buf(c, a, n[a] * sizeof(float), (void**)dst[a]));
    SCT_CUDA_TRY(cudaMemcpyAsync(*dst[a], src[a], n[a] * sizeof(float), cudaMemcpyHostToDevice, st));
  }
  return SCT_OK;
}

int sct_render_fwd_host(sct_ctx* c, const sct_cloud* cloud_host, const sct_scanner* scanner, const double* thetas,
                        int32_t n_views, const sct_raster_opts* opts, float* images_host, sct_fwd** state) {
  SCT_TRY(check_cloud(cloud_host));
  SCT_TRY(check_scanner(scanner));
  if (n_views < 1) {
    set_error("ConfigError: need at least one view");
    return SCT_ERR_CONFIG;
  }
  sct_cloud d;
  g_dbg.mark(c->stream, "start");
  SCT_TRY(upload_cloud(c, cloud_host, &d));
  const size_t px = (size_t)scanner->det_res_px[0] * scanner->det_res_px[1];
  float* dimg = nullptr;
  SCT_TRY(stage_buf(c, 4, n_views * px * sizeof(float), (void**)&dimg));
  SCT_TRY(stage_publish(c, c->copy_stream));
  // binning for all views, then one composite whose view units are copied
  // to the host (copy stream) as they complete. With stream memory operations
  // the binning's last pass (the counting scatter) is split at a unit
  // boundary near the middle: the composite of the first views starts — and
  // their copies with it — while the scatter of the remaining views runs
  // after it (sct_render_fwd leaves that half pending in the state).
  const bool units_ok = memops().wait && images_host != nullptr;
  const int units = host_units(n_views, n_views * px * sizeof(float));
  const int u_split = units / 2;
  const int v_split = (int)((int64_t)n_views * u_split / units);
  c->fwd_split_views = (units_ok && host_split_enabled() && u_split > 0 && v_split > 0 && v_split < n_views)
                           ? v_split
                           : -1;
  int rc = sct_render_fwd(c, &d, scanner, thetas, n_views, opts, nullptr, state);
  c->fwd_split_views = -1;
  if (rc != SCT_OK) return rc;
  g_dbg.mark(c->stream, "binned");
  if (units_ok && (*state)->n_pairs > 0 && raster_units_supported(c, *state)) {
    // one composite over all views; unit u's D2H copy starts when the
    // composite publishes unit_flags[0][u] (and at the latest after the
    // kernel, which re-publishes every unit)
    const uint32_t epoch = ++c->epoch;
    SCT_CUDA_TRY(cudaMemsetAsync(c->unit_done, 0, sizeof(int) * units, c->stream));
    UnitSync us;
    us.done_flag = c->unit_flags;
    us.done = c->unit_done;
    us.epoch = epoch;
    us.units = units;
    us.n_views = n_views;
    static const bool dbg = std::getenv("SCT_UNIT_DEBUG") != nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr, ec[Ctx::kMaxUnits] = {};
    unsigned long long* stamp = nullptr;
    if (dbg) {
      cudaMalloc((void**)&stamp, (Ctx::kMaxUnits + 1) * sizeof(unsigned long long));
      cudaMemset(stamp, 0xff, (Ctx::kMaxUnits + 1) * sizeof(unsigned long long));
      us.stamp = stamp;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int u = 0; u < units; ++u) cudaEventCreate(&ec[u]);
      cudaEventRecord(e0, c->stream);
    }
    if ((*state)->defer) {  // views [0, v_split): composite; then the rest of the scatter and its composite
      const int T = (*state)->det.tiles_x * (*state)->det.tiles_y;
      SCT_TRY(launch_raster_composite_units(c, *state, dimg, us, 0, T * v_split));
      g_dbg.mark(c->stream, "comp1");
      sct::BinDeferred* rest = (*state)->defer;
      (*state)->defer = nullptr;
      SCT_TRY(launch_bin_scatter_rest(c, rest));
      g_dbg.mark(c->stream, "scatter2");
      SCT_TRY(launch_raster_composite_units(c, *state, dimg, us, T * v_split, -1));
      g_dbg.mark(c->stream, "comp2");
    } else {
      SCT_TRY(launch_raster_composite_units(c, *state, dimg, us));
    }
    if (dbg) cudaEventRecord(e1, c->stream);
    for (int u = 0; u < units; ++u) SCT_TRY(stream_write_flag(c->stream, c->unit_flags + u, epoch));
    for (int u = 0; u < units; ++u) {
      const int v0 = (int)((int64_t)n_views * u / units), v1 = (int)((int64_t)n_views * (u + 1) / units);
      SCT_TRY(stream_wait_flag(c->copy_stream, c->unit_flags + u, epoch));
      SCT_CUDA_TRY(cudaMemcpyAsync(images_host + v0 * px, dimg + v0 * px, (v1 - v0) * px * sizeof(float),
                                   cudaMemcpyDeviceToHost, c->copy_stream));
      if (dbg) cudaEventRecord(ec[u], c->copy_stream);
      if (u == 0 || u == units / 2 || u == units - 1) g_dbg.mark(c->copy_stream, "d2h" + std::to_string(u));
    }
    SCT_CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
    SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (dbg) {
      float k = 0.f;
      cudaEventElapsedTime(&k, e0, e1);
      std::fprintf(stderr, "[units] composite %.3f ms; copies done at", k);
      for (int u = 0; u < units; ++u) {
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, ec[u]);
        std::fprintf(stderr, " %.3f", t);
        cudaEventDestroy(ec[u]);
      }
      std::fprintf(stderr, "\n");
      unsigned long long hs[Ctx::kMaxUnits + 1];
      cudaMemcpy(hs, stamp, sizeof(hs), cudaMemcpyDeviceToHost);
      std::fprintf(stderr, "[units] published at (ms after the first claim)");
      for (int u = 0; u < units; ++u)
        std::fprintf(stderr, " %.3f", 1e-6 * (double)(hs[u] - hs[Ctx::kMaxUnits]));
      std::fprintf(stderr, "\n");
      cudaFree(stamp);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    g_dbg.report("fwd_host");
    return SCT_OK;
  }
  // without stream memory operations: one composite, then one copy
  if ((*state)->defer) {
    sct::BinDeferred* rest = (*state)->defer;
    (*state)->defer = nullptr;
    SCT_TRY(launch_bin_scatter_rest(c, rest));
  }
  if ((*state)->n_pairs > 0)
    launch_raster_composite(c, *state, dimg);
  else
    SCT_CUDA_TRY(cudaMemsetAsync(dimg, 0, n_views * px * sizeof(float), c->stream));
  if (images_host)
    SCT_CUDA_TRY(cudaMemcpyAsync(images_host, dimg, n_views * px * sizeof(float), cudaMemcpyDeviceToHost,
                                 c->stream));
  SCT_CUDA_TRY(cudaGetLastError());
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return rc;
}

// sct_project_kernels with the cloud in host memory (the C++ drop-in's
// RenderedProjection::visible / project_kernels)
int sct_project_kernels_host(sct_ctx* c, const sct_cloud* cloud_host, const sct_scanner* scanner, double theta,
                             const sct_raster_opts* opts, int32_t* visible, double* rec) {
  SCT_TRY(check_cloud(cloud_host));
  if (cloud_host->m == 0) return SCT_OK;
  sct_cloud d;
  SCT_TRY(upload_cloud(c, cloud_host, &d));
  return sct_project_kernels(c, &d, scanner, theta, opts, visible, rec);
}

int sct_render_bwd_host(sct_ctx* c, sct_fwd* s, const sct_cloud* cloud_host, const float* dL_host,
                        sct_grads* grads_host, sct_stats* stats_host) {
  if (!s || !grads_host || !dL_host) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(check_cloud(cloud_host));
  sct_cloud d;
  g_dbg.mark(c->stream, "start");
  const int64_t m = cloud_host->m;
  const size_t px = (size_t)s->det.w * s->det.h;
  float* ddl = nullptr;
  SCT_TRY(stage_buf(c, 5, s->n_views * px * sizeof(float), (void**)&ddl));
  // every staging slot this call touches is sized here, on the main stream,
  // and the copy stream is ordered after those allocations (stage_publish)
  {
    void* tmp = nullptr;
    const int64_t na[4] = {m, 3 * m, 3 * m, 4 * m};
    for (int a = 0; a < 4; ++a) SCT_TRY(stage_buf(c, a, na[a] * sizeof(float), &tmp));
    for (int a = 0; a < 4; ++a) SCT_TRY(stage_buf(c, 6 + a, na[a] * sizeof(float), &tmp));
    if (stats_host) {
      const size_t sz[3] = {m * sizeof(float), m * sizeof(int32_t), 3 * m * sizeof(float)};
      for (int a = 0; a < 3; ++a) SCT_TRY(stage_buf(c, 10 + a, sz[a], &tmp));
    }
    SCT_TRY(stage_publish(c, c->copy_stream));
  }
  // units path: every H2D copy on the copy stream, in the order the GPU
  // needs the data — upstream-gradient unit 0 (K4 starts on it), the cloud
  // (the FP64 chain), the other units (K4 waits per unit, unit_flags[1]), the
  // caller's running sums (finalize). Chunked path: the cloud and the sums on
  // the main stream, K4 for chunk k once chunk k has landed.
  const bool units_path = memops().wait && s->n_items > 0 && raster_units_supported(c, s);
  const int units = units_path ? host_units(s->n_views, s->n_views * px * sizeof(float)) : 0;
  const uint32_t epoch = units_path ? ++c->epoch : 0;
  cudaStream_t up_stream = units_path ? c->copy_stream : c->stream;
  if (!units_path) SCT_TRY(upload_cloud(c, cloud_host, &d));
  for (int u = 0; u < units; ++u) {
    const int v0 = (int)((int64_t)s->n_views * u / units), v1 = (int)((int64_t)s->n_views * (u + 1) / units);
    SCT_CUDA_TRY(cudaMemcpyAsync(ddl + v0 * px, dL_host + v0 * px, (v1 - v0) * px * sizeof(float),
                                 cudaMemcpyHostToDevice, c->copy_stream));
    SCT_TRY(stream_write_flag(c->copy_stream, c->unit_flags + Ctx::kMaxUnits + u, epoch));
    if (u == 0 || u == units - 1) g_dbg.mark(c->copy_stream, "dl" + std::to_string(u));
    if (u == 0) {
      SCT_TRY(upload_cloud(c, cloud_host, &d, c->copy_stream));
      SCT_CUDA_TRY(cudaEventRecord(c->ev_copy[0], c->copy_stream));
    }
  }
  const int chunks =
      units_path ? 0 : std::min<int>(s->n_views, host_chunks(s->n_views * px * sizeof(float), false));
  for (int k = 0; k < chunks; ++k) {
    const int v0 = (int)((int64_t)s->n_views * k / chunks), v1 = (int)((int64_t)s->n_views * (k + 1) / chunks);
    SCT_CUDA_TRY(cudaMemcpyAsync(ddl + v0 * px, dL_host + v0 * px, (v1 - v0) * px * sizeof(float),
                                 cudaMemcpyHostToDevice, c->copy_stream));
    SCT_CUDA_TRY(cudaEventRecord(c->ev_copy[k], c->copy_stream));
  }
  // accumulate semantics: bring the caller's running sums to the device
  sct_grads dg;
  float** gd[4] = {&dg.rho_raw, &dg.pos, &dg.scale_raw, &dg.rot};
  float* gh[4] = {grads_host->rho_raw, grads_host->pos, grads_host->scale_raw, grads_host->rot};
  const int64_t n[4] = {m, 3 * m, 3 * m, 4 * m};
  for (int a = 0; a < 4; ++a) {
    SCT_TRY(stage_buf(c, 6 + a, n[a] * sizeof(float), (void**)gd[a]));
    SCT_CUDA_TRY(cudaMemcpyAsync(*gd[a], gh[a], n[a] * sizeof(float), cudaMemcpyHostToDevice, up_stream));
  }
  sct_stats dst{};
  void* sh[3] = {};
  void** sd[3] = {(void**)&dst.grad2d_norm_accum, (void**)&dst.grad_count, (void**)&dst.grad3d_accum};
  const size_t sb[3] = {m * sizeof(float), m * sizeof(int32_t), 3 * m * sizeof(float)};
  if (stats_host) {
    sh[0] = stats_host->grad2d_norm_accum;
    sh[1] = stats_host->grad_count;
    sh[2] = stats_host->grad3d_accum;
    for (int a = 0; a < 3; ++a) {
      SCT_TRY(stage_buf(c, 10 + a, sb[a], sd[a]));
      SCT_CUDA_TRY(cudaMemcpyAsync(*sd[a], sh[a], sb[a], cudaMemcpyHostToDevice, up_stream));
    }
  }
  if (units_path) SCT_CUDA_TRY(cudaEventRecord(c->ev_copy[1], c->copy_stream));
  g_dbg.mark(up_stream, "grads_up");
  int rc = units_path ? render_bwd_units(c, s, &d, ddl, &dg, stats_host ? &dst : nullptr, units, epoch,
                                         c->ev_copy[0], c->ev_copy[1])
                      : sct_render_bwd_chunked(c, s, &d, ddl, &dg, stats_host ? &dst : nullptr, chunks);
  if (rc == SCT_OK && units_path) {
    // a timed-out unit wait leaves the device sums incomplete: check the error
    // word before anything is copied into the caller's accumulate buffers
    SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    rc = check_unit_err(c);
  }
  if (rc == SCT_OK) {
    for (int a = 0; a < 4; ++a)
      SCT_CUDA_TRY(cudaMemcpyAsync(gh[a], *gd[a], n[a] * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    if (stats_host)
      for (int a = 0; a < 3; ++a)
        SCT_CUDA_TRY(cudaMemcpyAsync(sh[a], *sd[a], sb[a], cudaMemcpyDeviceToHost, c->stream));
  }
  g_dbg.mark(c->stream, "grads_down");
  SCT_CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  g_dbg.report("bwd_host");
  return rc;
}

// ------------------------------------------------------------------ voxelizer
int sct_voxelize_fwd(sct_ctx* c, const sct_cloud* cloud, const sct_grid* grid, double cull, int32_t zb0, int32_t zb1,
                     float* vol) {
  SCT_TRY(check_cloud(cloud));
  SCT_TRY(check_grid(grid));
  VoxelBins b;
  int rc = voxel_bin(c, *cloud, *grid, cull, zb0, zb1, b);
  if (rc == SCT_OK)
    launch_voxel_eval(c, *grid, b.zb0, b.zb1, b.bx, b.by, b.ranges, b.vals, b.rec, *cloud, b.n_pairs, vol);
  b.release(c);
  if (rc == SCT_OK && cudaGetLastError() != cudaSuccess) {
    set_error("CUDA error: kernel launch in sct_voxelize_fwd");
    rc = SCT_ERR_CUDA;
  }
  return rc;
}

int sct_voxelize_bwd(sct_ctx* c, const sct_cloud* cloud, const sct_grid* grid, double cull, int32_t zb0, int32_t zb1,
                     const float* dL, sct_grads* grads) {
  SCT_TRY(check_cloud(cloud));
  SCT_TRY(check_grid(grid));
  if (!grads || !dL) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  VoxelBins b;
  int rc = voxel_bin(c, *cloud, *grid, cull, zb0, zb1, b);
  float4* ps = nullptr;
  if (rc == SCT_OK) rc = dev_alloc(c, (void**)&ps, 3 * b.n_pairs * sizeof(float4));
  if (rc == SCT_OK) {
    launch_voxel_backward_stats(c, *grid, b.zb0, b.zb1, b.bx, b.by, b.ranges, b.vals, b.rec, b.lo, b.hi, b.offset,
                                *cloud, b.n_pairs, dL, ps);
    launch_voxel_chain(c, *cloud, b.offset, b.count, ps, grads, (int64_t)b.bx * b.by * (b.zb1 - b.zb0));
  }
  dev_free(c, ps);
  b.release(c);
  if (rc == SCT_OK && cudaGetLastError() != cudaSuccess) {
    set_error("CUDA error: kernel launch in sct_voxelize_bwd");
    rc = SCT_ERR_CUDA;
  }
  return rc;
}

// Forward + backward sharing one binning (the reference re-bins in
// voxelize_backward, voxelizer.cpp:145, because it keeps no state; the brick
// lists depend only on the cloud, grid, cull and slab, so they are reused).
struct sct_vox_state {
  sct_ctx* ctx = nullptr;
  VoxelBins b;
  sct_grid grid{};
  double cull = 0.0;
  int64_t m = 0;
};

int sct_voxelize_fwd_state(sct_ctx* c, const sct_cloud* cloud, const sct_grid* grid, double cull, int32_t zb0,
                           int32_t zb1, float* vol, sct_vox_state** state) {
  SCT_TRY(check_cloud(cloud));
  SCT_TRY(check_grid(grid));
  if (!state) {
    set_error("ConfigError: null state pointer");
    return SCT_ERR_CONFIG;
  }
  auto* s = new sct_vox_state();
  s->ctx = c;
  s->grid = *grid;
  s->cull = cull;
  s->m = cloud->m;
  int rc = voxel_bin(c, *cloud, *grid, cull, zb0, zb1, s->b);
  if (rc == SCT_OK && vol)
    launch_voxel_eval(c, *grid, s->b.zb0, s->b.zb1, s->b.bx, s->b.by, s->b.ranges, s->b.vals, s->b.rec, *cloud,
                      s->b.n_pairs, vol);
  if (rc == SCT_OK && cudaGetLastError() != cudaSuccess) {
    set_error("CUDA error: kernel launch in sct_voxelize_fwd_state");
    rc = SCT_ERR_CUDA;
  }
  if (rc != SCT_OK) {
    s->b.release(c);
    delete s;
    return rc;
  }
  *state = s;
  return SCT_OK;
}

int sct_voxelize_bwd_state(sct_ctx* c, sct_vox_state* s, const sct_cloud* cloud, const float* dL,
                           sct_grads* grads) {
  SCT_TRY(check_cloud(cloud));
  if (!s || !grads || !dL) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  if (cloud->m != s->m) {
    set_error("DimMismatch: voxelize_backward: cloud size differs from the forward state");
    return SCT_ERR_DATA;
  }
  float4* ps = nullptr;
  SCT_TRY(dev_alloc(c, (void**)&ps, 3 * s->b.n_pairs * sizeof(float4)));
  launch_voxel_backward_stats(c, s->grid, s->b.zb0, s->b.zb1, s->b.bx, s->b.by, s->b.ranges, s->b.vals, s->b.rec,
                              s->b.lo, s->b.hi, s->b.offset, *cloud, s->b.n_pairs, dL, ps);
  launch_voxel_chain(c, *cloud, s->b.offset, s->b.count, ps, grads,
                     (int64_t)s->b.bx * s->b.by * (s->b.zb1 - s->b.zb0));
  dev_free(c, ps);
  if (cudaGetLastError() != cudaSuccess) {
    set_error("CUDA error: kernel launch in sct_voxelize_bwd_state");
    return SCT_ERR_CUDA;
  }
  return SCT_OK;
}

int sct_vox_free(sct_vox_state* s) {
  if (!s) return SCT_OK;
  s->b.release(s->ctx);
  delete s;
  return SCT_OK;
}

int sct_voxel_bins(sct_ctx* c, const sct_cloud* cloud, const sct_grid* grid, double cull, int64_t* n_pairs,
                   int64_t* offsets, int32_t* kernel_idx) {
  SCT_TRY(check_cloud(cloud));
  SCT_TRY(check_grid(grid));
  VoxelBins b;
  int rc = voxel_bin(c, *cloud, *grid, cull, 0, INT32_MAX, b);
  if (rc == SCT_OK) {
    const int64_t nbr = (int64_t)b.bx * b.by * b.bz;
    if (n_pairs) *n_pairs = b.n_pairs;
    if (offsets) {
      std::vector<int2> r(nbr);
      cudaMemcpyAsync(r.data(), b.ranges, nbr * sizeof(int2), cudaMemcpyDeviceToHost, c->stream);
      cudaStreamSynchronize(c->stream);
      int64_t o = 0;
      for (int64_t t = 0; t < nbr; ++t) {
        offsets[t] = o;
        o += r[t].y > r[t].x ? r[t].y - r[t].x : 0;
      }
      offsets[nbr] = o;
    }
    if (kernel_idx && b.n_pairs > 0) {
      cudaMemcpyAsync(kernel_idx, b.vals, b.n_pairs * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream);
      cudaStreamSynchronize(c->stream);
    }
  }
  b.release(c);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess && rc == SCT_OK) {
    set_error("CUDA error in sct_voxel_bins");
    rc = SCT_ERR_CUDA;
  }
  return rc;
}

// VGE = sum over bricks of |brick list| x voxels of the brick inside the grid
// (trip count of voxelizer.cpp:125-133 and :169-188).
int sct_voxel_work(sct_ctx* c, const sct_cloud* cloud, const sct_grid* grid, double cull, int64_t* vge,
                   int64_t* n_pairs) {
  SCT_TRY(check_cloud(cloud));
  SCT_TRY(check_grid(grid));
  VoxelBins b;
  int rc = voxel_bin(c, *cloud, *grid, cull, 0, INT32_MAX, b);
  if (rc == SCT_OK) {
    const int64_t nbr = (int64_t)b.bx * b.by * b.bz;
    std::vector<int2> r(nbr);
    cudaMemcpyAsync(r.data(), b.ranges, nbr * sizeof(int2), cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    int64_t g = 0;
    for (int64_t t = 0; t < nbr; ++t) {
      const int tx = (int)(t % b.bx), ty = (int)((t / b.bx) % b.by), tz = (int)(t / ((int64_t)b.bx * b.by));
      const int64_t nv = (int64_t)std::min(kTileVox, grid->dims[0] - tx * kTileVox) *
                         std::min(kTileVox, grid->dims[1] - ty * kTileVox) *
                         std::min(kTileVox, grid->dims[2] - tz * kTileVox);
      g += (int64_t)(r[t].y - r[t].x) * nv;
    }
    if (vge) *vge = g;
    if (n_pairs) *n_pairs = b.n_pairs;
  }
  b.release(c);
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return rc;
}

int sct_voxelize_fwd_host(sct_ctx* c, const sct_cloud* cloud_host, const sct_grid* grid, double cull,
                          float* vol_host) {
  SCT_TRY(check_cloud(cloud_host));
  SCT_TRY(check_grid(grid));
  sct_cloud d;
  SCT_TRY(upload_cloud(c, cloud_host, &d));
  const size_t nv = (size_t)grid->dims[0] * grid->dims[1] * grid->dims[2];
  float* dv = nullptr;
  SCT_TRY(stage_buf(c, 13, nv * sizeof(float), (void**)&dv));
  int rc = sct_voxelize_fwd(c, &d, grid, cull, 0, INT32_MAX, dv);
  if (rc == SCT_OK)
    if (cudaMemcpyAsync(vol_host, dv, nv * sizeof(float), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) {
      set_error("CUDA error: volume download");
      rc = SCT_ERR_CUDA;
    }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess && rc == SCT_OK) rc = SCT_ERR_CUDA;
  return rc;
}

int sct_voxelize_bwd_host(sct_ctx* c, const sct_cloud* cloud_host, const sct_grid* grid, double cull,
                          const float* dL_host, sct_grads* grads_host) {
  SCT_TRY(check_cloud(cloud_host));
  SCT_TRY(check_grid(grid));
  if (!dL_host || !grads_host) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  sct_cloud d;
  SCT_TRY(upload_cloud(c, cloud_host, &d));
  const int64_t m = cloud_host->m;
  const size_t nv = (size_t)grid->dims[0] * grid->dims[1] * grid->dims[2];
  float* ddl = nullptr;
  SCT_TRY(stage_buf(c, 13, nv * sizeof(float), (void**)&ddl));
  SCT_CUDA_TRY(cudaMemcpyAsync(ddl, dL_host, nv * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  sct_grads dg;
  float** gd[4] = {&dg.rho_raw, &dg.pos, &dg.scale_raw, &dg.rot};
  float* gh[4] = {grads_host->rho_raw, grads_host->pos, grads_host->scale_raw, grads_host->rot};
  const int64_t n[4] = {m, 3 * m, 3 * m, 4 * m};
  for (int a = 0; a < 4; ++a) {
    SCT_TRY(stage_buf(c, 6 + a, n[a] * sizeof(float), (void**)gd[a]));
    SCT_CUDA_TRY(cudaMemcpyAsync(*gd[a], gh[a], n[a] * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  }
  int rc = sct_voxelize_bwd(c, &d, grid, cull, 0, INT32_MAX, ddl, &dg);
  if (rc == SCT_OK)
    for (int a = 0; a < 4; ++a)
      SCT_CUDA_TRY(cudaMemcpyAsync(gh[a], *gd[a], n[a] * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  SCT_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return rc;
}

// ------------------------------------------------------------------ objectives / optimizer
int sct_tv3d(sct_ctx* c, const float* vol, const int32_t dims[3], float lambda, double* value, float* grad) {
  if (!dims || dims[0] < 2 || dims[1] < 2 || dims[2] < 2) {
    set_error("DimMismatch: tv3d_loss: need at least 2 voxels per axis");
    return SCT_ERR_DATA;
  }
  const long long n = (long long)dims[0] * dims[1] * dims[2];
  int nb = (int)((n + 255) / 256);
  if (nb > c->sm_count * 8) nb = c->sm_count * 8;
  double* partials = nullptr;
  SCT_TRY(dev_alloc(c, (void**)&partials, 3 * nb * sizeof(double)));
  launch_tv3d(c, vol, dims, lambda, value, grad, partials, nb);
  dev_free(c, partials);
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_photometric_loss(sct_ctx* c, const float* rendered, const float* measured, int32_t n, int32_t w, int32_t h,
                         float render_scale, float lambda_ssim, float grad_scale, double* values, float* dL) {
  SCT_TRY(photometric_loss(c, rendered, measured, n, w, h, render_scale, lambda_ssim, grad_scale, values, dL));
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

int sct_adam_step(sct_ctx* c, sct_cloud* p, sct_adam_state* st, const sct_grads* g, int32_t t, const double lr[4],
                  double beta1, double beta2, double eps) {
  if (!p || !st || !g || t < 1) {
    set_error("ConfigError: adam: null argument or step < 1");
    return SCT_ERR_CONFIG;
  }
  const double bc1 = 1.0 - std::pow(beta1, t);  // trainer.cpp:152-153
  const double bc2 = 1.0 - std::pow(beta2, t);
  const float lrf[4] = {(float)lr[0], (float)lr[1], (float)lr[2], (float)lr[3]};
  launch_adam(c, p, st, g, lrf, (float)bc1, (float)bc2, (float)beta1, (float)beta2, (float)eps);
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

}  // extern "C"

extern "C" {
// Diagnostics: cudaPointerGetAttributes(ptr).type as seen by the engine's
// runtime (0 unregistered, 1 host/pinned, 2 device, 3 managed).
int sct_debug_pointer_type(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return (int)a.type;
}
// Page-locked host allocation through the engine's runtime (for callers that
// want the host-buffer entry points to run at full copy bandwidth).
int sct_host_alloc(void** p, size_t bytes) {
  SCT_CUDA_TRY(cudaMallocHost(p, bytes));
  return SCT_OK;
}
int sct_host_free(void* p) {
  SCT_CUDA_TRY(cudaFreeHost(p));
  return SCT_OK;
}
}
