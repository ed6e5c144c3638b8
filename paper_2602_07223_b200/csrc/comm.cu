// comm.cu — the path's single collective: per-layer score exchange across KV-head shards.
//
// with KV heads of one layer on several GPUs, per-layer selection (the reference
// contract, selection.cpp:96 / SPEC.md:335) needs the column sums of ALL heads.  The verify kernel
// emits them as int64 fixed point, so the exchange is one ncclAllReduce(int64, sum) over the head
// group — exact and order-independent, hence the sharded selection is bit-identical to the
// single-GPU one.  The runner enqueues it between each layer's verify and select on the selection
// side stream (captured into the iteration graph with everything else).
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: the system copy or whichever the process
// already loaded, e.g. torch's), so the library itself has no link-time NCCL dependency.
#include <dlfcn.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>

#include "internal.h"

namespace {

// The NCCL C API subset used here (nccl.h, ABI-stable across 2.x).
typedef struct {
  char internal[128];
} nccl_unique_id_t;
typedef void* nccl_comm_t;
typedef int nccl_result_t;  // ncclSuccess == 0
enum { kNcclInt64 = 4, kNcclSum = 0 };

struct NcclApi {
  nccl_result_t (*get_unique_id)(nccl_unique_id_t*) = nullptr;
  nccl_result_t (*comm_init_rank)(nccl_comm_t*, int, nccl_unique_id_t, int) = nullptr;
  nccl_result_t (*comm_destroy)(nccl_comm_t) = nullptr;
  nccl_result_t (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  const char* (*get_error_string)(nccl_result_t) = nullptr;
  nccl_result_t (*comm_count)(nccl_comm_t, int*) = nullptr;
  nccl_result_t (*comm_user_rank)(nccl_comm_t, int*) = nullptr;
  nccl_result_t (*comm_get_async_error)(nccl_comm_t, nccl_result_t*) = nullptr;
  nccl_result_t (*comm_abort)(nccl_comm_t) = nullptr;
  bool ok = false;
  std::string err;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.get_error_string = reinterpret_cast<decltype(api.get_error_string)>(dlsym(h, "ncclGetErrorString"));
    api.comm_count = reinterpret_cast<decltype(api.comm_count)>(dlsym(h, "ncclCommCount"));
    api.comm_user_rank = reinterpret_cast<decltype(api.comm_user_rank)>(dlsym(h, "ncclCommUserRank"));
    api.comm_get_async_error = reinterpret_cast<decltype(api.comm_get_async_error)>(dlsym(h, "ncclCommGetAsyncError"));
    api.comm_abort = reinterpret_cast<decltype(api.comm_abort)>(dlsym(h, "ncclCommAbort"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.get_error_string &&
             api.comm_count && api.comm_user_rank && api.comm_get_async_error && api.comm_abort;
    if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

sa_status nccl_fail(nccl_result_t r, const char* where) {
  return sa::fail(SA_NCCL_ERROR, std::string(where) + ": " + nccl().get_error_string(r));
}

}  // namespace

struct sa_comm {
  nccl_comm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool aborted = false;
};

namespace {
constexpr nccl_result_t kNcclInProgress = 7;  // ncclInProgress (non-blocking communicators)

// Asynchronous NCCL errors (a peer died, a network failure): abort the communicator so no kernel of
// this rank waits on it forever, and report SA_NCCL_ERROR.
sa_status check_async(sa_comm* c) {
  if (!c || !c->comm) return SA_OK;
  if (c->aborted) return sa::fail(SA_NCCL_ERROR, "communicator was aborted after an earlier error");
  nccl_result_t ae = 0;
  nccl_result_t r = nccl().comm_get_async_error(c->comm, &ae);
  if (r != 0) return nccl_fail(r, "ncclCommGetAsyncError");
  if (ae != 0 && ae != kNcclInProgress) {
    nccl().comm_abort(c->comm);
    c->aborted = true;
    return nccl_fail(ae, "NCCL asynchronous error (communicator aborted)");
  }
  return SA_OK;
}
}  // namespace

namespace sa {
sa_status comm_allreduce_i64(sa_comm* c, long long* buf, size_t count, cudaStream_t s) {
  if (!c) return SA_OK;  // no communicator: nothing to exchange
  if (sa_status st = check_async(c)) return st;
  nccl_result_t r = nccl().all_reduce(buf, buf, count, kNcclInt64, kNcclSum, c->comm, s);
  return r == 0 ? SA_OK : nccl_fail(r, "ncclAllReduce");
}
}  // namespace sa

extern "C" {

SA_API sa_status sa_comm_unique_id(void* id_out_128) {
  if (!id_out_128) return sa::fail(SA_INVALID_ARGUMENT, "null argument");
  if (!nccl().ok) return sa::fail(SA_NCCL_ERROR, nccl().err);
  nccl_unique_id_t id;
  nccl_result_t r = nccl().get_unique_id(&id);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_out_128, id.internal, 128);
  return SA_OK;
}

SA_API sa_status sa_comm_create(const void* id_128, int32_t nranks, int32_t rank, sa_comm** out) {
  if (!id_128 || !out) return sa::fail(SA_INVALID_ARGUMENT, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return sa::fail(SA_INVALID_ARGUMENT, "rank / nranks out of range");
  *out = nullptr;
  auto* c = new sa_comm();
  c->nranks = nranks;
  c->rank = rank;
  {  // a one-rank group is a real (identity) NCCL communicator too: same code path as N > 1
    if (!nccl().ok) {
      delete c;
      return sa::fail(SA_NCCL_ERROR, nccl().err);
    }
    nccl_unique_id_t id;
    std::memcpy(id.internal, id_128, 128);
    nccl_result_t r = nccl().comm_init_rank(&c->comm, nranks, id, rank);
    if (r != 0) {
      delete c;
      return nccl_fail(r, "ncclCommInitRank");
    }
  }
  *out = c;
  return SA_OK;
}

SA_API sa_status sa_comm_info(const sa_comm* c, int32_t* nranks, int32_t* rank) {
  if (!c || !nranks || !rank) return sa::fail(SA_INVALID_ARGUMENT, "null argument");
  int n = 0, r = 0;
  if (nccl_result_t e = nccl().comm_count(c->comm, &n)) return nccl_fail(e, "ncclCommCount");
  if (nccl_result_t e = nccl().comm_user_rank(c->comm, &r)) return nccl_fail(e, "ncclCommUserRank");
  *nranks = n;
  *rank = r;
  return SA_OK;
}

SA_API sa_status sa_comm_check(sa_comm* c) {
  if (!c) return sa::fail(SA_INVALID_ARGUMENT, "null communicator");
  return check_async(c);
}

SA_API sa_status sa_comm_sync(sa_comm* c, void* stream, int64_t timeout_ms) {
  if (!c) return sa::fail(SA_INVALID_ARGUMENT, "null communicator");
  const auto t0 = std::chrono::steady_clock::now();
  auto s = static_cast<cudaStream_t>(stream);
  while (true) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return check_async(c);
    if (e != cudaErrorNotReady) return sa::cuda_fail(e, "sa_comm_sync");
    if (sa_status st = check_async(c)) return st;
    if (timeout_ms >= 0 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) {
      nccl().comm_abort(c->comm);  // a hung peer: unblock this rank's kernels
      c->aborted = true;
      return sa::fail(SA_NCCL_ERROR, "sa_comm_sync: timed out waiting for the stream (communicator aborted)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
}

SA_API sa_status sa_comm_destroy(sa_comm* c) {
  if (!c) return SA_OK;
  if (c->comm && !c->aborted) nccl().comm_destroy(c->comm);
  delete c;
  return SA_OK;
}

}  // extern "C"
