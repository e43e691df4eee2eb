// Internal declarations shared by the engine's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "splatct_gpu.h"

// Checked build (make checked -> libsplatct_b200_checked.so, loaded with
// SCT_CHECKED=1): device-side invariant checks on the cross-CTA protocols and
// every gathered index — list ranges, pair and item indices, the K3 last-part
// and view-unit counters, the work counter. A failed check prints its
// condition and traps (the launch fails, the process sees a CUDA error). It
// stands in for compute-sanitizer, which this GPU pool does not run.
#ifndef SCT_CHECKED
#define SCT_CHECKED 0
#endif
#if SCT_CHECKED
#include <cstdio>
#define SCT_DCHECK(cond)                                                                \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("SCT_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                        \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define SCT_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace sct {

constexpr int kTilePx = 16;   // common.hpp:24 kImageTilePx
constexpr int kTileVox = 8;   // common.hpp:25 kVolumeTileVox
constexpr double kLog2e = 1.4426950408889634;
constexpr double kPi = 3.14159265358979323846;  // M_PI
// per-Gaussian prep record (doubles): Sigma (9, d_covariance order) | rho |
// Sigma^-1 (xx xy xz yy yz zz) | det Sigma | pad
constexpr int kPrepStride = 18;

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
struct Status {
  int code = SCT_OK;
};
#define SCT_CUDA_TRY(expr)                                                                 \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      ::sct::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " +     \
                       __FILE__ + ":" + std::to_string(__LINE__) + " (" #expr ")");       \
      return SCT_ERR_CUDA;                                                                 \
    }                                                                                      \
  } while (0)
#define SCT_TRY(expr)          \
  do {                         \
    int _rc = (expr);          \
    if (_rc != SCT_OK) return _rc; \
  } while (0)

// ------------------------------------------------------------------ geometry
// Per-view constants computed on the host in double (geometry.cpp:76-98).
struct ViewParams {
  double rot[9];  // W row-major
  double t[3];
};
struct DetParams {
  double fx, fy, cx, cy;
  int32_t w, h;
  double near_clip;
  int32_t tiles_x, tiles_y;
  int32_t parallel;  // parallel-beam extension: phi(p) = (fx x + cx, fy y + cy, z)
};
DetParams make_det(const sct_scanner& s);
ViewParams make_view(const sct_scanner& s, double theta);

// Raster options as device-friendly POD.
struct RasterParams {
  int32_t mode;
  int32_t dilation_compensation;
  int32_t freeze_jacobian;
  double eps2;      // lowpass_eps_px^2
  double cull;      // cull_mahalanobis
};
RasterParams make_raster(const sct_raster_opts& o);

// ------------------------------------------------------------------ device buffers
// Stream-ordered device allocation (cudaMallocAsync on the context stream; the
// pool keeps freed blocks, so steady-state calls allocate nothing from the driver).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// ------------------------------------------------------------------ context
struct TimingRec {
  const char* name;
  cudaEvent_t a, b;
};

struct Ctx {
  // per-kernel CUDA-event timing (sct_ctx_set_timing); events bracket each
  // engine launch on the context stream
  bool timing = false;
  std::vector<TimingRec> recs;
  std::vector<cudaEvent_t> pool;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool deterministic = true;
  int64_t launches = 0;
  // sct_render_fwd_host: scatter only views [0, fwd_split_views) inside
  // sct_render_fwd and leave the rest pending in the state (-1: no split)
  int64_t fwd_split_views = -1;
  // grow-only scratch reused across calls
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  int64_t* pinned_count = nullptr;  // small pinned host words (128 B) for D2H of counts
  long long* sum64 = nullptr;       // device word: int64 total of a count scan
  // sync-free binning (sct_ctx_set_capacity): pair buffers of a fixed capacity
  // instead of a host readback of the pair count; a device overflow word is
  // set when a call's pairs exceed it (sct_ctx_take_overflow)
  int64_t cap_raster = 0, cap_voxel = 0;
  int* overflow = nullptr;
  int* fin_counter = nullptr;  // [2] self-resetting last-block counters (photometric loss, TV)
  int sm_count = 148;
  // copy stream + events for the host-buffer entry points (H2D/D2H of view
  // chunks overlap the compute of neighbouring chunks)
  cudaStream_t copy_stream = nullptr;
  // second compute stream: the FP64 chain of view chunk k runs on it while
  // the statistics kernel of chunk k+1 runs on the main stream
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t ev_join = nullptr;
  cudaEvent_t ev_stage = nullptr;  // staging slots (re)allocated on `stream`, before another stream uses them
  static constexpr int kChunkEvents = 16;
  cudaEvent_t ev_compute[kChunkEvents] = {};
  cudaEvent_t ev_copy[kChunkEvents] = {};
  // grow-only device staging buffers of the host-buffer entry points (a
  // context serialises its calls, so a slot is free again at the next call)
  // slots: 0-13 host-path staging, 14/15 backward statistics, 16/17 NCCL
  // scratch, 18/19 fixtures, 20 K3 work counter, 22 tile order, 23 photometric
  // partials, 24 K3 partial tiles, 25 K7 partials, 27 K3 work items, 28-31 the
  // native train step's image / dL / volume / TV gradient
  static constexpr int kStageSlots = 32;
  void* stage[kStageSlots] = {};
  size_t stage_bytes[kStageSlots] = {};
  // longest-first (view, tile) order of the last forward state / view range
  // (raster.cu tile_order), keyed by the state's id
  uint64_t next_fwd_id = 1;
  uint64_t order_id = 0;
  int order_v0 = -1, order_nv = -1;
  const int* order_ptr = nullptr;
  uint64_t order_gen = 0;  // bumped whenever slot 22 receives a new order
  // K3's work items (raster.cu list_work, slot 27) were built from this order
  // generation with this part length and list count
  struct ItemsKey {
    uint64_t gen = 0;
    int part = 0, n = 0;
  } items_key;
  // NCCL communicator of the *_allreduce entry points (comm.cu): an
  // ncclComm_t, owned by the context when made by sct_ctx_comm_init
  void* comm = nullptr;
  bool comm_owned = false;
  // view-unit signals of the host-buffer entry points (stream memory
  // operations, see UnitSync): epoch-stamped flags in device memory, written
  // by kernels or by the copy stream and waited on by streams or kernels.
  // Flags are never reset: a wait compares against the call's epoch.
  static constexpr int kMaxUnits = 64;
  uint32_t* unit_flags = nullptr;  // [3][kMaxUnits] mapped host: composite done, dL landed, K4 done
  int* unit_done = nullptr;        // [2][kMaxUnits] finished-list counters
  int* unit_err = nullptr;         // a kernel-side wait timed out
  uint32_t epoch = 0;
};

// Per-unit (contiguous view range) wait / signal of one kernel launch.
// Unit u holds views [V u / units, V (u + 1) / units).
struct UnitSync {
  const uint32_t* ready = nullptr;  // wait until ready[u] >= epoch before reading unit u's input
  uint32_t* done_flag = nullptr;    // done_flag[u] = epoch once all of unit u's lists are finished
  int* done = nullptr;              // finished-list counters (zeroed before the launch)
  int* err = nullptr;
  uint32_t epoch = 0;
  int units = 0, n_views = 0;
  int per_view = 0;  // lists (x parts) per view
  unsigned long long* stamp = nullptr;  // SCT_UNIT_DEBUG: [u] publish time, [kMaxUnits] first claim (K3)
};

#ifdef __CUDACC__
__device__ __forceinline__ int unit_of_view(int v, int n_views, int units) {
  int k = 0;
  while (k + 1 < units && (long long)n_views * (k + 1) / units <= v) ++k;
  return k;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// one thread: spin until unit u's input has landed (bounded: after 2 s the
// error word is set and the kernel proceeds, so a lost signal cannot hang)
__device__ __forceinline__ void unit_wait(const UnitSync& us, int u) {
  if (!us.ready) return;
  const uint64_t t0 = global_ns();
  while ((int)(ld_acquire_sys(us.ready + u) - us.epoch) < 0) {
    __nanosleep(128);
    if (global_ns() - t0 > 2000000000ull) {
      atomicExch(us.err, 1);
      break;
    }
  }
}

// one thread, after every writer of the finished list fenced and met it at a
// barrier: count the list; the last list of the unit publishes the flag
__device__ __forceinline__ void unit_signal(const UnitSync& us, int u) {
  if (!us.done) return;
  const int v0 = (int)((long long)us.n_views * u / us.units);
  const int v1 = (int)((long long)us.n_views * (u + 1) / us.units);
  SCT_DCHECK(u >= 0 && u < us.units);
  const int old = atomicAdd(us.done + u, 1);
  SCT_DCHECK(old < us.per_view * (v1 - v0));  // every list of the unit signals exactly once
  if (old == us.per_view * (v1 - v0) - 1) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(us.done_flag + u), "r"(us.epoch) : "memory");
    if (us.stamp) us.stamp[u] = global_ns();
  }
}
#endif
void comm_release(Ctx* c);
int stage_buf(Ctx* c, int slot, size_t bytes, void** p);

int ensure_cub_tmp(Ctx* c, size_t bytes);

// Programmatic dependent launch (sm_90+): every engine kernel is launched with
// programmatic stream serialisation (pdl_launch) and begins with
// pdl_prologue(): it lets the next kernel of the stream be scheduled once all
// of its own blocks are running, then waits until the previous kernel has
// completed and its writes are visible. So a dependent kernel's launch and
// block ramp overlap its predecessor's tail instead of following it — the
// train step is a chain of ~30 small dependent kernels. (Both instructions
// are no-ops for a kernel launched without the attribute; SCT_PDL=0 launches
// without it.)
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
#endif
bool pdl_enabled();
// zero `bytes` (a multiple of 4) at p with a PDL-launched kernel instead of a
// cudaMemsetAsync, which would break the dependent-launch chain
int launch_zero(Ctx* c, void* p, size_t bytes);
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// RAII scope recording a start/stop event pair around one kernel launch when
// timing is enabled; also counts the launch.
struct KScope {
  Ctx* c;
  int idx = -1;
  cudaStream_t st;
  KScope(Ctx* ctx, const char* name, bool engine_kernel = true, cudaStream_t stream = nullptr);
  ~KScope();
};
int dev_alloc(Ctx* c, void** p, size_t bytes);
void dev_free(Ctx* c, void* p);

}  // namespace sct

// Forward state (opaque to callers).
namespace sct {
// a counting scatter split at a view (raster.cu): the count table and tile
// bases stay alive until the remaining views are scattered
struct BinDeferred {
  int32_t* H = nullptr;
  int32_t* seg = nullptr;
  int32_t* tb = nullptr;
  const short4* lo = nullptr;
  const short4* hi = nullptr;
  int32_t* vals = nullptr;
  int64_t m = 0, n_views = 0, v0 = 0, chunk = 0, n_chunks = 0, cap = 0;
  int tiles_x = 0, tiles_y = 0, tiles_z = 0;
  size_t smem = 0;
};
}  // namespace sct

struct sct_fwd {
  sct::Ctx* ctx = nullptr;
  uint64_t id = 0;  // unique per context (tile-order cache key)
  int32_t n_views = 0;
  int64_t m = 0;
  sct::DetParams det{};
  sct::RasterParams rp{};
  sct_raster_opts opts{};
  sct_scanner scanner{};
  double s_min = 0.0;
  std::vector<double> thetas;
  int32_t tile_bits = 0;
  int64_t n_pairs = 0;
  int64_t n_items = 0;
  // device buffers
  sct::ViewParams* d_views = nullptr;  // [V]
  float4* d_rec = nullptr;             // [items][2]: {cx,cy,amp,-}, {A,B,C,-} (log2-scaled conic)
  short4* d_rect = nullptr;            // [items] tx0,tx1,ty0,ty1 (tx0>tx1 => empty)
  int32_t* d_count = nullptr;          // [items] tiles covered
  int32_t* d_offset = nullptr;         // [items+1] exclusive scan of count
  uint8_t* d_vis = nullptr;            // [items] visible flag
  void* d_keys = nullptr;              // [pairs] sorted tile keys (uint16 if tile_bits <= 16, else uint32)
  int32_t* d_vals = nullptr;           // [pairs] sorted item index
  bool exact = true;                   // n_pairs is the pair count (else the capacity; count in d_total)
  bool offsets_ready = true;           // d_offset holds the per-item pair offsets (ensure_item_offsets)
  int32_t* d_total = nullptr;          // [1] pair count on the device (capacity mode)
  int2* d_ranges = nullptr;            // [V*T] [start,end) into sorted pairs
  double* d_prep = nullptr;            // [kPrepStride][m] (SoA) Sigma (9), rho, Sigma^-1 (6), det, FP64
  // host path: the counting scatter of views [defer.v0, V) still pending
  // (sct_render_fwd_host composites the first views while it runs)
  sct::BinDeferred* defer = nullptr;
};

struct sct_ctx : public sct::Ctx {};

// render backward with optional view-chunk pipelining (capi.cu; chunks = 0:
// the device-resident path); shared by the plain and the NCCL entry points
// defer_vsum != nullptr: stop before the finalize and hand back the chain's
// view-range partials (staging slot 15) and their count (the native train step
// finalizes them inside its Adam kernel); *defer_vsum = nullptr: no visible item
extern "C" int sct_render_bwd_chunked(sct_ctx* c, sct_fwd* s, const sct_cloud* cloud, const float* dL,
                                      sct_grads* grads, sct_stats* stats, int chunks,
                                      double** defer_vsum = nullptr, int* defer_groups = nullptr);

// ------------------------------------------------------------------ kernel entry points
namespace sct {
// binning preprocess (FP64, compiled with -fmad=false: bit-exact vs oracle)
void launch_gauss_prep(Ctx* c, const sct_cloud& cl, double* prep);
void launch_raster_preprocess(Ctx* c, const sct_cloud& cl, const double* prep, const ViewParams* d_views,
                              int n_views, const DetParams& det, const RasterParams& rp, float4* rec, short4* rect,
                              int32_t* count, uint8_t* vis);
void launch_voxel_preprocess(Ctx* c, const sct_cloud& cl, const sct_grid& g, double cull, int32_t zb0,
                             int32_t zb1, int32_t bricks_x, int32_t bricks_y, float4* rec, short4* rect_lo,
                             short4* rect_hi, int32_t* count);
// FP32 hot kernels
void launch_raster_emit(Ctx* c, int64_t n_items, const short4* rect, const int32_t* offset, int tiles_x,
                        void* keys, bool keys16, int32_t* vals);
bool raster_bin_scatter_fits(int tiles_x, int tiles_y);
// the second half of a split counting scatter: views [v0, n_views) of a binning
// whose count / scan / ranges are done (launch_bin_scatter with scatter_views)
int launch_bin_scatter_rest(Ctx* c, BinDeferred* d);
// scatter_views in (0, n_views): scatter only views [0, scatter_views) now and
// leave the rest in *defer (ranges of all views are final either way)
int launch_raster_bin_scatter(Ctx* c, int64_t n_views, int64_t m, int tiles_x, int tiles_y, const short4* rect,
                              int32_t* vals, int2* ranges, int64_t n_pairs, int64_t cap, int32_t* total,
                              int64_t scatter_views = -1, BinDeferred** defer = nullptr);
// one-CTA count scan for n + 1 <= kCountScanSmall: offsets, int64 total into
// c->sum64, and the capacity guard when cap > 0
constexpr int64_t kCountScanSmall = 1 << 16;
void launch_count_scan_small(Ctx* c, int32_t* count, int32_t* offset, int64_t n, int64_t cap, short4* box_a,
                             short4* box_b);
void launch_capacity_guard(Ctx* c, int32_t* count, int32_t* offset, int64_t n, short4* box_a, short4* box_b,
                           int64_t cap,
                           bool no_wrap = false);
bool bin_scatter_fits(int tiles_x, int tiles_y, int tiles_z);
int launch_bin_scatter(Ctx* c, int64_t n_views, int64_t m, int tiles_x, int tiles_y, int tiles_z, const short4* lo,
                       const short4* hi, int32_t* vals, int2* ranges, int64_t cap, int32_t* total,
                       int64_t scatter_views = -1, BinDeferred** defer = nullptr);
void launch_raster_ranges(Ctx* c, int64_t n_pairs, const void* keys, bool keys16, const int32_t* vals, int64_t m,
                          int64_t tiles_per_view, int2* ranges);
void launch_raster_composite(Ctx* c, const sct_fwd* s, float* images);
// unit-signalled host path (UnitSync): one composite / one K4 over all views
bool raster_units_supported(Ctx* c, const sct_fwd* s);
// items of the order positions [pos0, pos1) only (pos1 < 0: to the end)
int launch_raster_composite_units(Ctx* c, const sct_fwd* s, float* images, UnitSync us, int pos0 = 0,
                                  int pos1 = -1);
// item_stats != nullptr: parallel-atomic mode, 8 floats per item accumulated
// with atomics instead of per-pair slots; us != nullptr: all views, waiting
// for and publishing view units
void launch_raster_backward_stats(Ctx* c, const sct_fwd* s, const float* dL, float4* pair_stats, int v0 = 0,
                                  int nv = 0, float* item_stats = nullptr, const UnitSync* us = nullptr);
void launch_voxel_emit(Ctx* c, int64_t m, const short4* lo, const short4* hi, const int32_t* offset,
                       int32_t bricks_x, int32_t bricks_y, void* keys, bool keys16, int32_t* vals,
                       int64_t cap = INT64_MAX);
// keys >= n_keys are capacity-mode padding (sorted after every real key) and are skipped
void launch_key_ranges(Ctx* c, int64_t n_pairs, const void* keys, bool keys16, int2* ranges,
                       int64_t n_keys = INT64_MAX);
void launch_voxel_eval(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x,
                       int32_t bricks_y, const int2* ranges, const int32_t* vals, const float4* rec,
                       const sct_cloud& cl, int64_t n_pairs, float* vol);
void launch_voxel_backward_stats(Ctx* c, const sct_grid& g, int32_t zb0, int32_t zb1, int32_t bricks_x,
                                 int32_t bricks_y, const int2* ranges, const int32_t* vals,
                                 const float4* rec, const short4* lo, const short4* hi,
                                 const int32_t* offset, const sct_cloud& cl, int64_t n_pairs, const float* dL,
                                 float4* pair_stats);
// FP64 chain rules
// per_item: pair_stats holds one pre-summed 8-float record per item (atomic mode).
// The chain of views [v0, v1) writes one view-range partial (chain_sums_bytes(s, 1))
// at vsum; finalize sums `groups` consecutive partials in order.
int64_t chain_sums_bytes(const sct_fwd* s, int groups);
void launch_raster_chain(Ctx* c, const sct_fwd* s, const sct_cloud& cl, const float4* pair_stats, double* vsum,
                         bool per_item = false, int v0 = 0, int v1 = -1, cudaStream_t stream = nullptr);
void launch_raster_finalize(Ctx* c, const sct_fwd* s, const sct_cloud& cl, const double* vsum, int groups,
                            sct_grads* g, sct_stats* st);
// the finalize fused with Adam (native train step): grads already hold the TV
// contribution; the raster part is added per kernel, the statistics updated, and
// the Adam step (+ quaternion renormalisation, + the total loss) applied at once.
// vsum == nullptr: no raster contribution this iteration
void launch_raster_finalize_adam(Ctx* c, int64_t m, const sct_fwd* s, sct_cloud* cl, const double* vsum, int groups,
                                 const sct_grads* g, sct_stats* st, sct_adam_state* adam, const float lr[4],
                                 float bc1, float bc2, float b1, float b2, float eps, double* total,
                                 double lambda_ssim, double lambda_tv);
// n_bricks: bricks of the binned grid; small grids (the train step's TV
// sub-grid) sum each kernel's few pairs inside the chain instead of a separate
// 8-lanes-per-kernel pass
void launch_voxel_chain(Ctx* c, const sct_cloud& cl, const int32_t* offset, const int32_t* count,
                        const float4* pair_stats, sct_grads* g, int64_t n_bricks = -1);
// project_kernel export (FP64)
void launch_project_export(Ctx* c, const sct_cloud& cl, const ViewParams* d_view, const DetParams& det,
                           const RasterParams& rp, int32_t* vis, double* rec);
// optimizer / objectives
void launch_tv3d(Ctx* c, const float* vol, const int32_t dims[3], float lambda, double* value, float* grad,
                 double* partials, int n_partials);
void launch_adam(Ctx* c, sct_cloud* p, sct_adam_state* st, const sct_grads* g, const float lr[4], float bc1,
                 float bc2, float beta1, float beta2, float eps, double* total = nullptr,
                 double lambda_ssim = 0.0, double lambda_tv = 0.0);
int photometric_loss(Ctx* c, const float* rendered, const float* measured, int n, int w, int h,
                     float render_scale, float lambda_ssim, float grad_scale, double* values, float* dL);
}  // namespace sct
