// NCCL gradient all-reduce (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../common.cuh"
#include "../memory.h"

namespace dgnn {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
  static const NcclApi a = [] {
    NcclApi r;
    void* h = nullptr;
    std::string tried;
    const char* env = std::getenv("DGNN_NCCL_LIB");
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (name == nullptr) continue;
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
      tried += std::string(" ") + name + ": " + dlerror() + ";";
    }
    if (h == nullptr) throw std::runtime_error("NCCL not found (" + tried + ")");
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (p == nullptr) throw std::runtime_error(std::string("NCCL symbol missing: ") + s);
      return p;
    };
    r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(sym("ncclGetUniqueId"));
    r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(sym("ncclCommInitRank"));
    r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(sym("ncclAllReduce"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(sym("ncclCommDestroy"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(sym("ncclGetErrorString"));
    return r;
  }();
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " + api().error_string(r));
}

}  // namespace

static_assert(sizeof(ncclUniqueId) == kCommIdBytes, "ncclUniqueId size");

void NcclComm::unique_id(uint8_t out[kCommIdBytes]) {
  ncclUniqueId id;
  nccl_check(api().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, kCommIdBytes);
}

NcclComm::NcclComm(const uint8_t id[kCommIdBytes], int world, int rank) : world_(world), rank_(rank) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("comm: rank out of range");
  ncclUniqueId uid;
  std::memcpy(&uid, id, kCommIdBytes);
  ncclComm_t c = nullptr;
  nccl_check(api().comm_init_rank(&c, world, uid, rank), "ncclCommInitRank");
  comm_ = c;
}

NcclComm::~NcclComm() {
  if (comm_) api().comm_destroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::allreduce_sum(float* data, int64_t n, cudaStream_t stream) {
  if (n <= 0) return;
  nccl_check(api().all_reduce(data, data, static_cast<size_t>(n), ncclFloat32, ncclSum,
                              static_cast<ncclComm_t>(comm_), stream),
             "ncclAllReduce");
}

double NcclComm::allreduce_max(double v, cudaStream_t stream) {
  cuda::DevArray<double> d(1, stream);
  DGNN_CUDA(cudaMemcpyAsync(d.get(), &v, sizeof(double), cudaMemcpyHostToDevice, stream));
  nccl_check(api().all_reduce(d.get(), d.get(), 1, ncclFloat64, ncclMax, static_cast<ncclComm_t>(comm_),
                              stream),
             "ncclAllReduce");
  double out = 0.0;
  DGNN_CUDA(cudaMemcpyAsync(&out, d.get(), sizeof(double), cudaMemcpyDeviceToHost, stream));
  DGNN_CUDA(cudaStreamSynchronize(stream));
  return out;
}

}  // namespace dgnn
