// NCCL-aware entry points (SURVEY.md §8b "NCCL-aware variants taking an
// ncclComm_t", §8e): the data-parallel exchange of the path is one sum over
// ranks of the per-kernel gradients (views are sharded across ranks, each rank
// holds the whole cloud; rasterizer.cpp:329-331 sums view contributions into
// one CloudGrads) and, for the voxelizer, of the z-slab partial gradients.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing the copy the
// process already loaded, e.g. torch's) so the C-ABI library itself carries no
// link-time NCCL dependency; only these entry points need it.
//
// Semantics: sct_allreduce_grads sums buffers in place across ranks. The
// *_allreduce backward variants keep the reference's accumulate contract on
// every rank: grads += sum over ranks of each rank's contribution (the
// contribution is produced into a zeroed scratch buffer, reduced as ONE
// contiguous 11*M-float collective, then added), so a caller can mix them
// with local accumulation exactly like render_backward / voxelize_backward.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "sct_internal.cuh"

namespace sct {
namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.err = std::string("NCCL library not found: ") + (e ? e : "dlopen failed");
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) api.err = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommCount, "ncclCommCount");
    sym(api.CommUserRank, "ncclCommUserRank");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = api.err.empty();
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SCT_OK;
  set_error(std::string("CudaError: NCCL ") + what + ": " + nccl().GetErrorString(r));
  return SCT_ERR_CUDA;
}

#define SCT_NCCL_TRY(expr, what)                    \
  do {                                              \
    int _r = ::sct::nccl_check((expr), what);       \
    if (_r != SCT_OK) return _r;                    \
  } while (0)

int need_comm(Ctx* c) {
  if (!nccl().ok) {
    set_error("CudaError: " + nccl().err);
    return SCT_ERR_CUDA;
  }
  if (!c->comm) {
    set_error("ConfigError: no communicator on this context (sct_ctx_comm_init / sct_ctx_set_comm)");
    return SCT_ERR_CONFIG;
  }
  return SCT_OK;
}

// grads += reduced contribution (scratch layout: rho[M] pos[3M] scale[3M] rot[4M]);
// stats likewise (norm[M] g3d[3M] as floats, counts[M] as int32)
__global__ void add_reduced_kernel(int64_t m, const float* __restrict__ g, sct_grads out, const float* __restrict__ st,
                                   const int32_t* __restrict__ cnt, sct_stats sout, bool with_stats) {
  const int64_t n = 11 * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = g[i];
    if (i < m)
      out.rho_raw[i] += v;
    else if (i < 4 * m)
      out.pos[i - m] += v;
    else if (i < 7 * m)
      out.scale_raw[i - 4 * m] += v;
    else
      out.rot[i - 7 * m] += v;
    if (with_stats && i < 4 * m) {
      if (i < m) {
        sout.grad2d_norm_accum[i] += st[i];
        sout.grad_count[i] += cnt[i];
      } else {
        sout.grad3d_accum[i - m] += st[i];
      }
    }
  }
}

int grid_for(Ctx* c, int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)c->sm_count * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// Scratch (context slots 16, 17): contribution buffers for the fused variants.
int scratch(Ctx* c, int64_t m, bool with_stats, float** g, float** st, int32_t** cnt, sct_grads* sg, sct_stats* ss) {
  SCT_TRY(stage_buf(c, 16, 11 * m * sizeof(float), (void**)g));
  SCT_CUDA_TRY(cudaMemsetAsync(*g, 0, 11 * m * sizeof(float), c->stream));
  sg->rho_raw = *g;
  sg->pos = *g + m;
  sg->scale_raw = *g + 4 * m;
  sg->rot = *g + 7 * m;
  if (with_stats) {
    char* b = nullptr;
    SCT_TRY(stage_buf(c, 17, 5 * m * sizeof(float), (void**)&b));
    SCT_CUDA_TRY(cudaMemsetAsync(b, 0, 5 * m * sizeof(float), c->stream));
    *st = reinterpret_cast<float*>(b);
    *cnt = reinterpret_cast<int32_t*>(b + 4 * m * sizeof(float));
    ss->grad2d_norm_accum = *st;
    ss->grad3d_accum = *st + m;
    ss->grad_count = *cnt;
  }
  return SCT_OK;
}

int reduce_and_add(Ctx* c, int64_t m, float* g, float* st, int32_t* cnt, sct_grads* grads, sct_stats* stats) {
  const auto& A = nccl();
  auto comm = static_cast<ncclComm_t>(c->comm);
  SCT_NCCL_TRY(A.GroupStart(), "group start");
  SCT_NCCL_TRY(A.AllReduce(g, g, 11 * m, ncclFloat32, ncclSum, comm, c->stream), "all-reduce (grads)");
  if (stats) {
    SCT_NCCL_TRY(A.AllReduce(st, st, 4 * m, ncclFloat32, ncclSum, comm, c->stream), "all-reduce (stats)");
    SCT_NCCL_TRY(A.AllReduce(cnt, cnt, m, ncclInt32, ncclSum, comm, c->stream), "all-reduce (counts)");
  }
  SCT_NCCL_TRY(A.GroupEnd(), "group end");
  {
    KScope _ks(c, "add_reduced");
    add_reduced_kernel<<<grid_for(c, 11 * m), 256, 0, c->stream>>>(m, g, *grads, st, cnt,
                                                                    stats ? *stats : sct_stats{}, stats != nullptr);
  }
  SCT_CUDA_TRY(cudaGetLastError());
  return SCT_OK;
}

}  // namespace

void comm_release(Ctx* c) {
  if (c->comm && c->comm_owned && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(c->comm));
  c->comm = nullptr;
  c->comm_owned = false;
}

}  // namespace sct

using namespace sct;

extern "C" {

int sct_nccl_unique_id(uint8_t id[128]) {
  if (!id) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  if (!nccl().ok) {
    set_error("CudaError: " + nccl().err);
    return SCT_ERR_CUDA;
  }
  ncclUniqueId u;
  SCT_NCCL_TRY(nccl().GetUniqueId(&u), "get unique id");
  static_assert(sizeof(u.internal) == 128, "NCCL unique id size");
  std::memcpy(id, u.internal, 128);
  return SCT_OK;
}

int sct_ctx_comm_init(sct_ctx* c, int32_t nranks, int32_t rank, const uint8_t id[128]) {
  if (!c || !id || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("ConfigError: comm init: bad rank / size / id");
    return SCT_ERR_CONFIG;
  }
  if (!nccl().ok) {
    set_error("CudaError: " + nccl().err);
    return SCT_ERR_CUDA;
  }
  SCT_CUDA_TRY(cudaSetDevice(c->device));
  comm_release(c);
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t comm = nullptr;
  SCT_NCCL_TRY(nccl().CommInitRank(&comm, nranks, u, rank), "comm init");
  c->comm = comm;
  c->comm_owned = true;
  return SCT_OK;
}

int sct_ctx_set_comm(sct_ctx* c, void* nccl_comm) {
  if (!c) return SCT_ERR_CONFIG;
  comm_release(c);
  c->comm = nccl_comm;
  c->comm_owned = false;
  return SCT_OK;
}

int sct_ctx_comm_info(sct_ctx* c, int32_t* nranks, int32_t* rank) {
  if (!c) return SCT_ERR_CONFIG;
  SCT_TRY(need_comm(c));
  int n = 0, r = 0;
  SCT_NCCL_TRY(nccl().CommCount(static_cast<ncclComm_t>(c->comm), &n), "comm count");
  SCT_NCCL_TRY(nccl().CommUserRank(static_cast<ncclComm_t>(c->comm), &r), "comm rank");
  if (nranks) *nranks = n;
  if (rank) *rank = r;
  return SCT_OK;
}

int sct_allreduce_grads(sct_ctx* c, int64_t m, sct_grads* grads, sct_stats* stats) {
  if (!c || !grads || m < 0) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(need_comm(c));
  if (m == 0) return SCT_OK;
  const auto& A = nccl();
  auto comm = static_cast<ncclComm_t>(c->comm);
  SCT_NCCL_TRY(A.GroupStart(), "group start");
  float* g[4] = {grads->rho_raw, grads->pos, grads->scale_raw, grads->rot};
  const int64_t w[4] = {1, 3, 3, 4};
  for (int a = 0; a < 4; ++a)
    SCT_NCCL_TRY(A.AllReduce(g[a], g[a], w[a] * m, ncclFloat32, ncclSum, comm, c->stream), "all-reduce (grads)");
  if (stats) {
    SCT_NCCL_TRY(A.AllReduce(stats->grad2d_norm_accum, stats->grad2d_norm_accum, m, ncclFloat32, ncclSum, comm,
                             c->stream), "all-reduce (stats)");
    SCT_NCCL_TRY(A.AllReduce(stats->grad3d_accum, stats->grad3d_accum, 3 * m, ncclFloat32, ncclSum, comm, c->stream),
                 "all-reduce (stats)");
    SCT_NCCL_TRY(A.AllReduce(stats->grad_count, stats->grad_count, m, ncclInt32, ncclSum, comm, c->stream),
                 "all-reduce (counts)");
  }
  SCT_NCCL_TRY(A.GroupEnd(), "group end");
  return SCT_OK;
}

int sct_render_bwd_allreduce(sct_ctx* c, sct_fwd* s, const sct_cloud* cloud, const float* dL, sct_grads* grads,
                             sct_stats* stats) {
  if (!c || !s || !cloud || !grads || !dL) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(need_comm(c));
  const int64_t m = cloud->m;
  if (m == 0) return SCT_OK;
  float *g = nullptr, *st = nullptr;
  int32_t* cnt = nullptr;
  sct_grads sg{};
  sct_stats ss{};
  SCT_TRY(scratch(c, m, stats != nullptr, &g, &st, &cnt, &sg, &ss));
  SCT_TRY(sct_render_bwd_chunked(c, s, cloud, dL, &sg, stats ? &ss : nullptr, 0));
  return reduce_and_add(c, m, g, st, cnt, grads, stats);
}

int sct_voxelize_bwd_allreduce(sct_ctx* c, const sct_cloud* cloud, const sct_grid* grid, double cull_mahalanobis,
                               int32_t z_brick_begin, int32_t z_brick_end, const float* dL_dvol, sct_grads* grads) {
  if (!c || !cloud || !grid || !grads || !dL_dvol) {
    set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  SCT_TRY(need_comm(c));
  const int64_t m = cloud->m;
  if (m == 0) return SCT_OK;
  float *g = nullptr, *st = nullptr;
  int32_t* cnt = nullptr;
  sct_grads sg{};
  sct_stats ss{};
  SCT_TRY(scratch(c, m, false, &g, &st, &cnt, &sg, &ss));
  SCT_TRY(sct_voxelize_bwd(c, cloud, grid, cull_mahalanobis, z_brick_begin, z_brick_end, dL_dvol, &sg));
  return reduce_and_add(c, m, g, st, cnt, grads, nullptr);
}

}  // extern "C"
