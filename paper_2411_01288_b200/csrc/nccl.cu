// nccl.cu -- the tensor-parallel collectives of the reference's two
// configurations (core/src/dist_sim.cpp), over NCCL for a C / C++ host.
//
// The reference simulates them in-process: all_gather_rows = rank-order row
// concatenation, all_reduce_sum = ascending-rank sum (dist_sim.cpp:127-176),
// run_data_centric all-gathers the hidden shards into the pipeline-shared
// cache (dist_sim.cpp:367-368, CacheError dist_sim.cpp:104-125) and
// all-reduces the gradients (dist_sim.cpp:397-399); run_model_centric
// all-gathers tokens / routing / g_y and all-reduces the partial y and g_x
// (dist_sim.cpp:478-530).  These entry points issue the same collectives
// with NCCL on the caller's stream (NVLink / NVSwitch on a B200 box).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): the library does not
// link it, so a process that already loaded NCCL (e.g. through PyTorch)
// shares that copy, and a host without NCCL still loads libhexamoe.so (these
// calls then fail with HXM_ERR_NCCL).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace hxm {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
#define HXM_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(sym(name))
    HXM_SYM(GetUniqueId, "ncclGetUniqueId");
    HXM_SYM(CommInitRank, "ncclCommInitRank");
    HXM_SYM(CommDestroy, "ncclCommDestroy");
    HXM_SYM(CommCount, "ncclCommCount");
    HXM_SYM(CommUserRank, "ncclCommUserRank");
    HXM_SYM(AllGather, "ncclAllGather");
    HXM_SYM(AllReduce, "ncclAllReduce");
    HXM_SYM(GroupStart, "ncclGroupStart");
    HXM_SYM(GroupEnd, "ncclGroupEnd");
    HXM_SYM(GetErrorString, "ncclGetErrorString");
#undef HXM_SYM
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.CommCount && a.CommUserRank &&
           a.AllGather && a.AllReduce && a.GroupStart && a.GroupEnd && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

hxm_status nccl_err(const char* what, ncclResult_t r) {
  const NcclApi& a = api();
  set_error(std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error"));
  return HXM_ERR_NCCL;
}

#define HXM_TRY_NCCL(what, expr)              \
  do {                                        \
    const ncclResult_t _r = (expr);           \
    if (_r != ncclSuccess) return nccl_err(what, _r); \
  } while (0)

hxm_status need_api() {
  const NcclApi& a = api();
  if (!a.ok) {
    set_error(a.why);
    return HXM_ERR_NCCL;
  }
  return HXM_OK;
}

hxm_status comm_size(void* comm, int* n, int* r) {
  if (!comm) return invalid_arg("nccl: null communicator");
  HXM_TRY_NCCL("ncclCommCount", api().CommCount(static_cast<ncclComm_t>(comm), n));
  HXM_TRY_NCCL("ncclCommUserRank", api().CommUserRank(static_cast<ncclComm_t>(comm), r));
  return HXM_OK;
}

size_t esz(int32_t dt) { return dt == HXM_BF16 ? 2 : 4; }

// the data-centric cache: one slot of shard-major w1 | b1 | w2, 256-B aligned
struct CacheLayout {
  size_t w1, b1, w2, total;
};
CacheLayout cache_layout(const hxm_layer_desc& d) {
  const size_t e = esz(d.dtype);
  CacheLayout c{};
  c.w1 = 0;
  c.b1 = align_up(static_cast<size_t>(d.n_experts * d.d_in * d.hidden) * e, 256);
  c.w2 = c.b1 + align_up(static_cast<size_t>(d.n_experts * d.hidden) * 4, 256);
  c.total = c.w2 + align_up(static_cast<size_t>(d.n_experts * d.hidden * d.d_out) * e, 256);
  return c;
}

}  // namespace
}  // namespace hxm

using namespace hxm;

extern "C" {

hxm_status hxm_nccl_get_unique_id(unsigned char id[128]) {
  HXM_RETURN_IF(need_api());
  if (!id) return invalid_arg("nccl: null id buffer");
  ncclUniqueId u;
  HXM_TRY_NCCL("ncclGetUniqueId", api().GetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, sizeof(u));
  return HXM_OK;
}

hxm_status hxm_nccl_comm_init(void** comm, int32_t n_ranks, const unsigned char id[128],
                              int32_t rank) {
  HXM_RETURN_IF(need_api());
  if (!comm || !id) return invalid_arg("nccl: null argument");
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks)
    return invalid_arg("nccl: rank must be in [0, n_ranks)");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  HXM_TRY_NCCL("ncclCommInitRank", api().CommInitRank(&c, n_ranks, u, rank));
  *comm = c;
  return HXM_OK;
}

hxm_status hxm_nccl_comm_destroy(void* comm) {
  HXM_RETURN_IF(need_api());
  if (!comm) return HXM_OK;
  HXM_TRY_NCCL("ncclCommDestroy", api().CommDestroy(static_cast<ncclComm_t>(comm)));
  return HXM_OK;
}

size_t hxm_dc_cache_bytes(const hxm_layer_desc* d) {
  if (!d || d->n_experts < 1 || d->hidden < 1) return 0;
  return cache_layout(*d).total;
}

hxm_status hxm_dc_cache_views(const hxm_layer_desc* d, void* cache, void** w1, float** b1,
                              void** w2) {
  if (!d || !cache || !w1 || !b1 || !w2) return invalid_arg("dc cache: null argument");
  const CacheLayout c = cache_layout(*d);
  char* base = static_cast<char*>(cache);
  *w1 = base + c.w1;
  *b1 = reinterpret_cast<float*>(base + c.b1);
  *w2 = base + c.w2;
  return HXM_OK;
}

hxm_status hxm_dc_fill_cache(void* comm, const hxm_layer_desc* d, const void* w1_shard,
                             const float* b1_shard, const void* w2_shard, void* cache,
                             size_t cache_bytes, hxm_stream_t stream) {
  HXM_RETURN_IF(need_api());
  if (!d || !w1_shard || !b1_shard || !w2_shard || !cache)
    return invalid_arg("dc_fill_cache: null argument");
  int P = 0, r = 0;
  HXM_RETURN_IF(comm_size(comm, &P, &r));
  if (d->hidden % P != 0) return invalid_arg("dc_fill_cache: H must split evenly over the ranks");
  const CacheLayout c = cache_layout(*d);
  if (cache_bytes < c.total) {  // PipelineSharedCache::fill, dist_sim.cpp:104-125
    set_error("pipeline-shared cache: layer parameters exceed cache capacity");
    return HXM_ERR_CACHE;
  }
  const size_t h = static_cast<size_t>(d->hidden / P), E = static_cast<size_t>(d->n_experts);
  const ncclDataType_t wt = d->dtype == HXM_BF16 ? ncclBfloat16 : ncclFloat32;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(cache);
  const NcclApi& a = api();
  ncclComm_t cm = static_cast<ncclComm_t>(comm);
  // rank-major gathers = the shard-major layout hxm_layer_desc.weight_shards reads
  HXM_TRY_NCCL("ncclGroupStart", a.GroupStart());
  HXM_TRY_NCCL("ncclAllGather w1", a.AllGather(w1_shard, base + c.w1, E * d->d_in * h, wt, cm, st));
  HXM_TRY_NCCL("ncclAllGather b1", a.AllGather(b1_shard, base + c.b1, E * h, ncclFloat32, cm, st));
  HXM_TRY_NCCL("ncclAllGather w2", a.AllGather(w2_shard, base + c.w2, E * h * d->d_out, wt, cm, st));
  HXM_TRY_NCCL("ncclGroupEnd", a.GroupEnd());
  return HXM_OK;
}

hxm_status hxm_dc_allreduce_grads(void* comm, const hxm_layer_desc* d, float* gw1, float* gb1,
                                  float* gw2, float* gb2, hxm_stream_t stream) {
  HXM_RETURN_IF(need_api());
  if (!d || !gw1 || !gb1 || !gw2) return invalid_arg("dc_allreduce_grads: null gradient");
  int P = 0, r = 0;
  HXM_RETURN_IF(comm_size(comm, &P, &r));
  const size_t E = static_cast<size_t>(d->n_experts), Di = d->d_in, H = d->hidden, Do = d->d_out;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const NcclApi& a = api();
  ncclComm_t cm = static_cast<ncclComm_t>(comm);
  HXM_TRY_NCCL("ncclGroupStart", a.GroupStart());
  HXM_TRY_NCCL("ncclAllReduce gw1", a.AllReduce(gw1, gw1, E * Di * H, ncclFloat32, ncclSum, cm, st));
  HXM_TRY_NCCL("ncclAllReduce gb1", a.AllReduce(gb1, gb1, E * H, ncclFloat32, ncclSum, cm, st));
  HXM_TRY_NCCL("ncclAllReduce gw2", a.AllReduce(gw2, gw2, E * H * Do, ncclFloat32, ncclSum, cm, st));
  if (gb2)
    HXM_TRY_NCCL("ncclAllReduce gb2", a.AllReduce(gb2, gb2, E * Do, ncclFloat32, ncclSum, cm, st));
  HXM_TRY_NCCL("ncclGroupEnd", a.GroupEnd());
  return HXM_OK;
}

hxm_status hxm_tp_allgather_rows(void* comm, const void* local, int64_t rows_per_rank,
                                 int64_t row_bytes, void* out, hxm_stream_t stream) {
  HXM_RETURN_IF(need_api());
  if (rows_per_rank < 0 || row_bytes < 0) return shape_error("tp_allgather_rows: negative extent");
  if ((!local || !out) && rows_per_rank * row_bytes > 0)
    return invalid_arg("tp_allgather_rows: null buffer");
  int P = 0, r = 0;
  HXM_RETURN_IF(comm_size(comm, &P, &r));
  HXM_TRY_NCCL("ncclAllGather rows",
               api().AllGather(local, out, static_cast<size_t>(rows_per_rank * row_bytes), ncclUint8,
                               static_cast<ncclComm_t>(comm), reinterpret_cast<cudaStream_t>(stream)));
  return HXM_OK;
}

hxm_status hxm_tp_allgather_assignments(void* comm, const int32_t* local, int64_t k,
                                        int64_t n_local, int32_t* out, hxm_stream_t stream) {
  HXM_RETURN_IF(need_api());
  if (k < 1 || n_local < 0) return shape_error("tp_allgather_assignments: bad extent");
  if ((!local || !out) && n_local > 0) return invalid_arg("tp_allgather_assignments: null buffer");
  int P = 0, r = 0;
  HXM_RETURN_IF(comm_size(comm, &P, &r));
  // RoutingChoice is k x N (choice-major): gather each choice's row so the
  // global routing keeps that layout, tokens in rank order
  const NcclApi& a = api();
  HXM_TRY_NCCL("ncclGroupStart", a.GroupStart());
  for (int64_t c = 0; c < k; ++c)
    HXM_TRY_NCCL("ncclAllGather assignments",
                 a.AllGather(local + c * n_local, out + c * n_local * P, static_cast<size_t>(n_local),
                             ncclInt32, static_cast<ncclComm_t>(comm),
                             reinterpret_cast<cudaStream_t>(stream)));
  HXM_TRY_NCCL("ncclGroupEnd", a.GroupEnd());
  return HXM_OK;
}

hxm_status hxm_tp_allreduce_sum(void* comm, float* buf, int64_t n_elems, hxm_stream_t stream) {
  HXM_RETURN_IF(need_api());
  if (n_elems < 0) return shape_error("tp_allreduce_sum: negative extent");
  if (!buf && n_elems > 0) return invalid_arg("tp_allreduce_sum: null buffer");
  int P = 0, r = 0;
  HXM_RETURN_IF(comm_size(comm, &P, &r));
  HXM_TRY_NCCL("ncclAllReduce",
               api().AllReduce(buf, buf, static_cast<size_t>(n_elems), ncclFloat32, ncclSum,
                               static_cast<ncclComm_t>(comm), reinterpret_cast<cudaStream_t>(stream)));
  return HXM_OK;
}

}  // extern "C"
