// Gradient all-reduce over NCCL for the snapshot-window-sharded trainer (the
// one collective of ReInc's communication-free placement: the flat fp32
// gradient sum once per optimizer step, ref src/distsim.cpp:248-260).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: the process's own copy
// when torch already loaded one, else the system library), so the library has
// no link-time NCCL dependency and a process never holds two NCCL instances.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dgnn {

constexpr int kCommIdBytes = 128;  // sizeof(ncclUniqueId)

class NcclComm {
 public:
  // Rank 0 makes the id; every rank passes the same bytes (exchanged by the
  // caller: a file, a socket or torch.distributed).
  static void unique_id(uint8_t out[kCommIdBytes]);
  NcclComm(const uint8_t id[kCommIdBytes], int world, int rank);
  ~NcclComm();
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;

  int world() const { return world_; }
  int rank() const { return rank_; }
  // in-place sum over ranks of n fp32 values, stream-ordered
  void allreduce_sum(float* data, int64_t n, cudaStream_t stream);
  // max over ranks of one fp64 value (device-timed epoch seconds), blocking
  double allreduce_max(double v, cudaStream_t stream);

 private:
  void* comm_ = nullptr;
  int world_, rank_;
};

}  // namespace dgnn
