// PBT exchange transports (comm.cuh).  The reference has no multi-device path at all; the
// exchange it would need is the one SURVEY.md §8(e) derives from pbt_evolve_trainer
// (evolve.hpp:169-213): fitness of every member on every rank, then the donor -> replaced
// weight copies.  NCCL is resolved with dlopen: a process that already loaded libnccl (torch
// does) reuses that copy, so two NCCL versions never meet in one address space, and the
// library itself loads on hosts without NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "comm.cuh"
#include "pop.cuh"

namespace pbrl {
namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    a.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch loaded, if any
    if (!a.so) a.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.so) a.so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!a.so) return a;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.so, name));
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllGather, "ncclAllGather");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  if (!api.so || !api.CommInitRank || !api.Send)
    PBRL_THROW(PBRL_E_NCCL, "libnccl.so.2 not found (NCCL transport unavailable)");
  return api;
}

#define NCCL_CHECK(x)                                                                     \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      PBRL_THROW(PBRL_E_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_));        \
  } while (0)

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  double* d_send = nullptr;
  double* d_recv = nullptr;
  uint64_t cap = 0;

  ~NcclComm() override {
    cudaSetDevice(device);
    if (comm) nccl().CommDestroy(comm);
    cudaFree(d_send);
    cudaFree(d_recv);
  }
  const char* kind() const override { return "nccl"; }

  void allgather_f64(const double* send, uint64_t count, double* recv, cudaStream_t s) override {
    if (count > cap) {
      cudaFree(d_send);
      cudaFree(d_recv);
      d_send = d_recv = nullptr;
      CUDA_CHECK(cudaMalloc(&d_send, count * 8));
      CUDA_CHECK(cudaMalloc(&d_recv, count * 8 * world));
      cap = count;
    }
    CUDA_CHECK(cudaMemcpyAsync(d_send, send, count * 8, cudaMemcpyHostToDevice, s));
    NCCL_CHECK(nccl().AllGather(d_send, d_recv, count, ncclFloat64, comm, s));
    CUDA_CHECK(cudaMemcpyAsync(recv, d_recv, count * 8 * world, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }

  void allreduce_f32(float* dev, uint64_t count, cudaStream_t s) override {
    if (!nccl().AllReduce) PBRL_THROW(PBRL_E_NCCL, "ncclAllReduce not found");
    NCCL_CHECK(nccl().AllReduce(dev, dev, count, ncclFloat32, ncclSum, comm, s));
  }

  void exchange(const std::vector<P2P>& ops, cudaStream_t s) override {
    if (ops.empty()) return;
    NCCL_CHECK(nccl().GroupStart());
    for (const P2P& op : ops) {
      if (op.send)
        NCCL_CHECK(nccl().Send(op.dev, op.floats, ncclFloat32, op.peer, comm, s));
      else
        NCCL_CHECK(nccl().Recv(op.dev, op.floats, ncclFloat32, op.peer, comm, s));
    }
    NCCL_CHECK(nccl().GroupEnd());
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
};

struct HostComm final : Comm {
  pbrl_comm_ops ops{};
  const char* kind() const override { return "host"; }

  void allgather_f64(const double* send, uint64_t count, double* recv, cudaStream_t) override {
    if (ops.allgather_f64(ops.ctx, send, count, recv) != 0)
      PBRL_THROW(PBRL_E_NCCL, "pbrl_comm_ops.allgather_f64 failed");
  }

  void allreduce_f32(float* dev, uint64_t count, cudaStream_t s) override {
    if (!ops.allreduce_f32) PBRL_THROW(PBRL_E_USAGE, "pbrl_comm_ops.allreduce_f32 not provided");
    std::vector<float> h(count);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), dev, count * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (ops.allreduce_f32(ops.ctx, h.data(), count) != 0)
      PBRL_THROW(PBRL_E_NCCL, "pbrl_comm_ops.allreduce_f32 failed");
    CUDA_CHECK(cudaMemcpyAsync(dev, h.data(), count * 4, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }

  // device blobs are staged through host memory around the caller's exchange callback
  void exchange(const std::vector<P2P>& v, cudaStream_t s) override {
    if (v.empty()) return;
    std::vector<std::vector<float>> host(v.size());
    std::vector<pbrl_p2p_op> hops(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
      host[i].resize(v[i].floats);
      if (v[i].send)
        CUDA_CHECK(cudaMemcpyAsync(host[i].data(), v[i].dev, v[i].floats * 4,
                                   cudaMemcpyDeviceToHost, s));
      hops[i] = pbrl_p2p_op{v[i].peer, v[i].send ? 1 : 0, host[i].data(), v[i].floats};
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (ops.exchange(ops.ctx, hops.data(), static_cast<uint32_t>(hops.size())) != 0)
      PBRL_THROW(PBRL_E_NCCL, "pbrl_comm_ops.exchange failed");
    for (size_t i = 0; i < v.size(); ++i) {
      if (!v[i].send)
        CUDA_CHECK(cudaMemcpyAsync(v[i].dev, host[i].data(), v[i].floats * 4,
                                   cudaMemcpyHostToDevice, s));
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
};

}  // namespace

void nccl_unique_id(void* out, size_t len) {
  if (len < sizeof(ncclUniqueId)) PBRL_THROW(PBRL_E_USAGE, "unique id buffer < 128 bytes");
  ncclUniqueId id;
  NCCL_CHECK(nccl().GetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
}

Comm* make_nccl_comm(const void* unique_id, int rank, int world, int device) {
  if (world < 1 || rank < 0 || rank >= world) PBRL_THROW(PBRL_E_USAGE, "comm: bad rank / world");
  auto* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  CUDA_CHECK(cudaSetDevice(device));
  ncclResult_t r = nccl().CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    c->comm = nullptr;
    delete c;
    PBRL_THROW(PBRL_E_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
  }
  return c;
}

Comm* make_host_comm(const pbrl_comm_ops* ops, int rank, int world, int device) {
  if (!ops || !ops->allgather_f64 || !ops->exchange)
    PBRL_THROW(PBRL_E_USAGE, "comm: pbrl_comm_ops needs allgather_f64 and exchange");
  if (world < 1 || rank < 0 || rank >= world) PBRL_THROW(PBRL_E_USAGE, "comm: bad rank / world");
  auto* c = new HostComm();
  c->ops = *ops;
  c->rank = rank;
  c->world = world;
  c->device = device;
  return c;
}

}  // namespace pbrl
