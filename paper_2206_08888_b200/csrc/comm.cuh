// Transport of the PBT exchange between population shards: the fitness
// all-gather and the exploit weight copies.  NCCL over NVLink / NVSwitch on a multi-GPU box
// (NcclComm, libnccl resolved at run time so the library loads without it and shares the copy
// torch already loaded); a caller-supplied host transport (pbrl_comm_ops) for processes that
// share one device or have no NCCL (the CPU-side tests run it over gloo).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/pbrl_b200.h"

namespace pbrl {

struct P2P {
  int peer;
  bool send;
  float* dev;      // device buffer of `floats` floats on the comm's device
  uint64_t floats;
};

struct Comm {
  int rank = 0, world = 1, device = 0;
  virtual ~Comm() = default;
  // all-gather of `count` doubles per rank, host buffers: recv = [world][count]
  virtual void allgather_f64(const double* send, uint64_t count, double* recv, cudaStream_t s) = 0;
  // grouped point-to-point of device buffers, stream-ordered on s; returns when complete
  virtual void exchange(const std::vector<P2P>& ops, cudaStream_t s) = 0;
  // in-place sum over the ranks of a device float buffer, stream-ordered on s (the shared
  // critic's per-step gradient all-reduce)
  virtual void allreduce_f32(float* dev, uint64_t count, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
};

Comm* make_nccl_comm(const void* unique_id, int rank, int world, int device);
Comm* make_host_comm(const pbrl_comm_ops* ops, int rank, int world, int device);
void nccl_unique_id(void* out, size_t len);

}  // namespace pbrl
