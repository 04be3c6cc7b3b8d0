// Distributed context: NCCL communicator over NVLink/NVSwitch, one process per
// GPU. libnccl.so.2 is bound lazily with dlopen so single-GPU use (and the
// CPU-only import checks) carry no NCCL dependency; when torch has already
// loaded its bundled NCCL the same library instance is reused.
#include <dlfcn.h>
#include <nccl.h>

#include "internal.cuh"

namespace {

struct NcclApi {
  bool loaded = false;
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.lib = h;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.loaded = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather;
  });
  if (!a.loaded) kt::fail(KTUNE_ERR_BACKEND, "libnccl.so.2 could not be loaded");
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    kt::fail(KTUNE_ERR_BACKEND, std::string(what) + ": " +
                                    (api().GetErrorString ? api().GetErrorString(r) : "nccl error"));
}

}  // namespace

void kt_nccl_destroy(ktune_ctx* ctx) {
  if (ctx->nccl) {
    api().CommDestroy((ncclComm_t)ctx->nccl);
    ctx->nccl = nullptr;
  }
}

namespace kt {
// In-place sum all-reduce on the context stream (no-op without a communicator).
void allreduce_sum(ktune_ctx* ctx, void* buf, size_t count, bool is_double) {
  if (ctx->hc_allreduce) {  // host transport: stage through pinned memory
    void* h = ctx->host(3, count * 8);
    KT_CUDA(cudaMemcpyAsync(h, buf, count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->hc_allreduce(h, (int64_t)count, is_double ? 1 : 0, ctx->hc_user) != 0)
      fail(KTUNE_ERR_BACKEND, "host all-reduce failed");
    KT_CUDA(cudaMemcpyAsync(buf, h, count * 8, cudaMemcpyHostToDevice, ctx->stream));
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  if (!ctx->nccl) return;
  nccl_check(api().AllReduce(buf, buf, count, is_double ? ncclFloat64 : ncclInt64, ncclSum,
                             (ncclComm_t)ctx->nccl, ctx->stream),
             "ncclAllReduce");
}
// Rank-ordered all-gather; `send` may alias recv + rank * bytes_per_rank (in place).
void allgather(ktune_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
  if (ctx->hc_allgather) {
    const size_t total = bytes_per_rank * (size_t)ctx->world;
    char* h = (char*)ctx->host(3, total + bytes_per_rank);
    char* hs = h + total;
    KT_CUDA(cudaMemcpyAsync(hs, send, bytes_per_rank, cudaMemcpyDeviceToHost, ctx->stream));
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->hc_allgather(hs, h, (int64_t)bytes_per_rank, ctx->hc_user) != 0)
      fail(KTUNE_ERR_BACKEND, "host all-gather failed");
    KT_CUDA(cudaMemcpyAsync(recv, h, total, cudaMemcpyHostToDevice, ctx->stream));
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  if (!ctx->nccl) {
    if (send != recv) KT_CUDA(cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  nccl_check(api().AllGather(send, recv, bytes_per_rank, ncclUint8, (ncclComm_t)ctx->nccl, ctx->stream),
             "ncclAllGather");
}
bool has_comm(const ktune_ctx* ctx) { return ctx->nccl || ctx->hc_allgather; }
}  // namespace kt

extern "C" {

int ktune_nccl_get_unique_id(void* out128) {
  return kt_guard(nullptr, [&] {
    ncclUniqueId id;
    nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int ktune_ctx_create_dist(int device, int rank, int world, const void* nccl_id, ktune_ctx** out) {
  ktune_ctx* ctx = nullptr;
  const int rc = kt_guard(nullptr, [&] {
    if (world < 1 || rank < 0 || rank >= world) kt::fail(KTUNE_ERR_CONFIG, "bad rank/world");
    int ndev = 0;
    KT_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) kt::fail(KTUNE_ERR_CONFIG, "no such CUDA device");
    KT_CUDA(cudaSetDevice(device));
    ctx = new ktune_ctx();
    ctx->device = device;
    ctx->rank = rank;
    ctx->world = world;
    KT_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    // keep stream-ordered allocations cached across calls (host-pointer paths
    // allocate trajectory-sized buffers per call)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (world > 1 || nccl_id) {  // a one-rank communicator (nccl_id given) exercises the sharded paths
      if (!nccl_id) kt::fail(KTUNE_ERR_CONFIG, "world > 1 needs an ncclUniqueId");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      ncclComm_t comm;
      nccl_check(api().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
      ctx->nccl = comm;
    }
  });
  if (rc != KTUNE_OK) {
    if (ctx) {
      if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
      delete ctx;
    }
    return rc;
  }
  *out = ctx;
  return KTUNE_OK;
}

int ktune_ctx_create_hostcomm(int device, int rank, int world, ktune_host_allreduce_fn allreduce,
                              ktune_host_allgather_fn allgather, void* user, ktune_ctx** out) {
  if (!allreduce || !allgather || world < 1 || rank < 0 || rank >= world) return KTUNE_ERR_CONFIG;
  ktune_ctx* ctx = nullptr;
  const int rc = ktune_ctx_create_dist(device, 0, 1, nullptr, &ctx);
  if (rc != KTUNE_OK) return rc;
  ctx->rank = rank;
  ctx->world = world;
  ctx->hc_allreduce = allreduce;
  ctx->hc_allgather = allgather;
  ctx->hc_user = user;
  *out = ctx;
  return KTUNE_OK;
}

}  // extern "C"
