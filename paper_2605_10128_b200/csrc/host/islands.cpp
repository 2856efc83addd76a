// Native multi-GPU exchange of the engine: one engine
// context per process / GPU, NCCL over NVLink / NVSwitch for the data path,
// no torch. Built on the public C ABI (pack / merge / shard kernels, all on
// the context's stream) plus ncclAllGather on the same stream, so the
// collective is ordered between the engine's kernels with no host sync.
//
//   island mode  (tg_islands_exchange / tg_islands_step): every rank runs its
//     own population; the archives are packed into fixed-layout device blobs,
//     allgathered and merged with Repertoire::insert semantics
//     (qd_optimizer.cpp:281-303), so all ranks end each exchange with the
//     same archive;
//   shard mode   (tg_islands_shard_step): the ranks share ONE population;
//     each evaluates its slice of the generation's lanes, the score slices are
//     allgathered and every rank inserts all lanes in lane order, so the
//     archive is bit-identical to a one-GPU run.
//
// NCCL is loaded with dlopen (the library torch already loaded, else
// libnccl.so.2 from the loader path): the engine itself has no link-time
// NCCL dependency, and a missing NCCL is a TG_CUDA_ERROR at tg_islands_create.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../../include/topopt_b200.h"

namespace tgb {
void set_last_error(const std::string& m);  // capi.cu: the message tg_last_error() returns
}

namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string error;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!n.get_unique_id || !n.comm_init_rank || !n.all_gather || !n.comm_destroy || !n.error_string)
      n.error = "libnccl.so.2 lacks a required symbol";
  });
  return n;
}

struct Failure : std::runtime_error {
  tg_status status;
  Failure(tg_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void ck_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Failure(TG_CUDA_ERROR, std::string(what) + ": " + nccl().error_string(r));
}
void ck_cuda(cudaError_t r, const char* what) {
  if (r != cudaSuccess) throw Failure(TG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(r));
}
void ck_tg(tg_status s) {
  if (s != TG_OK) throw Failure(s, tg_last_error());
}

template <class F>
tg_status guarded(F&& f) {
  try {
    f();
    return TG_OK;
  } catch (const Failure& e) {
    tgb::set_last_error(e.what());
    return e.status;
  } catch (const std::exception& e) {
    tgb::set_last_error(e.what());
    return TG_CUDA_ERROR;
  }
}

}  // namespace

struct tg_islands {
  tg_context* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  // device buffers, (re)sized lazily: archive blobs and score-slice blobs
  void* send = nullptr;
  void* recv = nullptr;
  size_t cap = 0;  // bytes of send; recv holds world * cap

  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (send) cudaFree(send);
    if (recv) cudaFree(recv);
    send = recv = nullptr;
    ck_cuda(cudaMalloc(&send, bytes), "cudaMalloc (island blob)");
    ck_cuda(cudaMalloc(&recv, bytes * static_cast<size_t>(world)), "cudaMalloc (island blobs)");
    cap = bytes;
  }
  void allgather(size_t bytes) {
    ck_nccl(nccl().all_gather(send, recv, bytes, ncclUint8, comm, stream), "ncclAllGather");
  }
};

extern "C" {

tg_status tg_islands_unique_id(uint8_t* id) {
  return guarded([&] {
    if (!nccl().error.empty()) throw Failure(TG_CUDA_ERROR, nccl().error);
    ncclUniqueId u;
    ck_nccl(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

tg_status tg_islands_create(tg_context* ctx, const uint8_t* id, int32_t rank, int32_t world, tg_islands** out) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world) throw Failure(TG_CONFIG_ERROR, "islands: rank outside [0, world)");
    if (!nccl().error.empty()) throw Failure(TG_CUDA_ERROR, nccl().error);
    auto* isl = new tg_islands;
    isl->ctx = ctx;
    isl->rank = rank;
    isl->world = world;
    isl->stream = static_cast<cudaStream_t>(tg_context_stream(ctx));
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    const ncclResult_t r = nccl().comm_init_rank(&isl->comm, world, u, rank);
    if (r != ncclSuccess) {
      delete isl;
      ck_nccl(r, "ncclCommInitRank");
    }
    *out = isl;
  });
}

void tg_islands_destroy(tg_islands* isl) {
  if (!isl) return;
  if (isl->stream) cudaStreamSynchronize(isl->stream);
  if (isl->comm) nccl().comm_destroy(isl->comm);
  if (isl->send) cudaFree(isl->send);
  if (isl->recv) cudaFree(isl->recv);
  delete isl;
}

tg_status tg_islands_exchange(tg_islands* isl) {
  return guarded([&] {
    int64_t bytes = 0;
    ck_tg(tg_archive_blob_bytes(isl->ctx, &bytes));
    isl->ensure(static_cast<size_t>(bytes));
    ck_tg(tg_archive_pack(isl->ctx, isl->send));
    isl->allgather(static_cast<size_t>(bytes));
    ck_tg(tg_archive_merge(isl->ctx, isl->recv, isl->world));
  });
}

tg_status tg_islands_step(tg_islands* isl, int32_t n, int32_t merge_every) {
  return guarded([&] {
    for (int32_t i = 0; i < n; ++i) {
      ck_tg(tg_qd_step(isl->ctx, 1));
      if (merge_every > 0 && (i + 1) % merge_every == 0) ck_tg(tg_islands_exchange(isl));
    }
  });
}

tg_status tg_islands_shard_step(tg_islands* isl, int32_t n, int32_t batch_size) {
  return guarded([&] {
    if (batch_size % isl->world) throw Failure(TG_CONFIG_ERROR, "batch does not split evenly over the ranks");
    const int32_t per = batch_size / isl->world, lo = isl->rank * per, hi = lo + per;
    int64_t bytes = 0;
    ck_tg(tg_qd_scores_blob_bytes(isl->ctx, per, &bytes));
    isl->ensure(static_cast<size_t>(bytes));
    for (int32_t i = 0; i < n; ++i) {
      ck_tg(tg_qd_generation_begin(isl->ctx));
      ck_tg(tg_qd_evaluate_lanes(isl->ctx, lo, hi));
      if (isl->world > 1) {
        ck_tg(tg_qd_scores_pack(isl->ctx, lo, hi, isl->send));
        isl->allgather(static_cast<size_t>(bytes));
        for (int32_t r = 0; r < isl->world; ++r)
          if (r != isl->rank)
            ck_tg(tg_qd_scores_unpack(isl->ctx, r * per, (r + 1) * per,
                                      static_cast<uint8_t*>(isl->recv) + static_cast<size_t>(r) * bytes));
      }
      ck_tg(tg_qd_generation_end(isl->ctx));
    }
  });
}

}  // extern "C"
