// Snapshot publication between the learner and the actors:
// SnapshotMailbox / ActorSnapshot (pipeline.hpp:31-83) and the actor-side refresh
// (actor_loop, pipeline.hpp:255-285), device-resident.
//
// The learner publishes the policy population of its handle into one of three device slots
// (a stream-ordered D2D copy on the learner's stream: the publish never waits for actors, and
// actors never see a half-written slot because a slot becomes `latest` only with its copy
// event recorded).  An actor thread owns its own population handle (same shapes / precision /
// member ids) and adopts a new version with pbrl_actor_refresh: it pins the latest slot, its
// stream waits for the slot's copy event, copies the slot into its policy arena and unpins.
// Acting then runs on the actor's handle and stream, concurrently with the learner's updates.
#include <condition_variable>
#include <cstring>
#include <mutex>

#include "pop_impl.cuh"

namespace pbrl {
namespace {

struct Slot {
  DBuf<float> policy;           // [n][stride_p], the learner's policy arena layout
  std::vector<double> explore;  // per-member exploration scales published with it
  cudaEvent_t ready = nullptr;  // the copy into this slot is complete
  uint64_t version = 0;
  int pins = 0;                 // actors copying out of this slot (or the learner writing it)
};

}  // namespace
}  // namespace pbrl

struct pbrl_mailbox {
  int device = 0;
  uint64_t n = 0, P = 0, stride = 0;
  pbrl::NetShape shape;
  std::mutex mu;
  std::condition_variable cv;
  pbrl::Slot slot[3];
  int latest = -1;
  uint64_t version = 0;
};

namespace pbrl {
namespace {
template <typename F>
int mb_guarded(F&& f) {
  try {
    f();
    return PBRL_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PBRL_E_USAGE;
  }
}

uint64_t fnv1a(const void* data, size_t bytes, uint64_t h) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}
}  // namespace

}  // namespace pbrl

using namespace pbrl;

extern "C" {

int pbrl_mailbox_create(pbrl_pop* learner, pbrl_mailbox** out) {
  return mb_guarded([&] {
    if (!learner || !out) PBRL_THROW(PBRL_E_USAGE, "mailbox_create: null argument");
    Pop* p = reinterpret_cast<Pop*>(learner);
    CUDA_CHECK(cudaSetDevice(p->device));
    auto* mb = new pbrl_mailbox();
    mb->device = p->device;
    mb->n = static_cast<uint64_t>(p->n);
    mb->P = p->pol.P;
    mb->stride = p->pol.stride;
    mb->shape = p->pol;
    try {
      for (auto& s : mb->slot) {
        s.policy.alloc(mb->n * mb->stride);
        CUDA_CHECK(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
      }
    } catch (...) {
      for (auto& s : mb->slot)
        if (s.ready) cudaEventDestroy(s.ready);
      delete mb;
      throw;
    }
    *out = mb;
  });
}

int pbrl_mailbox_destroy(pbrl_mailbox* mb) {
  return mb_guarded([&] {
    if (!mb) return;
    cudaSetDevice(mb->device);
    for (auto& s : mb->slot) {
      if (s.ready) {
        cudaEventSynchronize(s.ready);
        cudaEventDestroy(s.ready);
      }
    }
    delete mb;
  });
}

// SnapshotMailbox::publish (pipeline.hpp:56-65): a fresh immutable snapshot of the policy
// population + explore_std; returns the new version.  Called by the learner thread.
int pbrl_mailbox_publish(pbrl_mailbox* mb, pbrl_pop* learner, const double* explore_std,
                         uint64_t* version) {
  return mb_guarded([&] {
    if (!mb || !learner) PBRL_THROW(PBRL_E_USAGE, "mailbox_publish: null argument");
    Pop* p = reinterpret_cast<Pop*>(learner);
    if (static_cast<uint64_t>(p->n) != mb->n || p->pol.P != mb->P)
      PBRL_THROW(PBRL_E_SHAPE, "mailbox_publish: population shape differs from the mailbox's");
    CUDA_CHECK(cudaSetDevice(p->device));
    int w = -1;
    {
      std::unique_lock<std::mutex> lk(mb->mu);
      mb->cv.wait(lk, [&] {
        for (int i = 0; i < 3; ++i)
          if (i != mb->latest && mb->slot[i].pins == 0) return true;
        return false;
      });
      for (int i = 0; i < 3 && w < 0; ++i)
        if (i != mb->latest && mb->slot[i].pins == 0) w = i;
      mb->slot[w].pins = 1;  // being written
    }
    Slot& s = mb->slot[w];
    CUDA_CHECK(cudaMemcpyAsync(s.policy.p, p->pol_p.p, mb->n * mb->stride * 4,
                               cudaMemcpyDeviceToDevice, p->stream));
    CUDA_CHECK(cudaEventRecord(s.ready, p->stream));
    s.explore.assign(mb->n, 0.0);
    if (explore_std) std::memcpy(s.explore.data(), explore_std, mb->n * 8);
    std::lock_guard<std::mutex> lk(mb->mu);
    s.version = ++mb->version;
    s.pins = 0;
    mb->latest = w;
    if (version) *version = s.version;
    mb->cv.notify_all();
  });
}

int pbrl_mailbox_version(pbrl_mailbox* mb, uint64_t* version) {
  return mb_guarded([&] {
    if (!mb || !version) PBRL_THROW(PBRL_E_USAGE, "mailbox_version: null argument");
    std::lock_guard<std::mutex> lk(mb->mu);
    *version = mb->version;
  });
}

// actor_loop's refresh() (pipeline.hpp:270-279): adopt the newest snapshot if its version
// differs from the one this actor holds.  *version = the version now held (0: nothing
// published yet); explore_std (may be NULL) receives that snapshot's exploration scales.
int pbrl_actor_refresh(pbrl_pop* actor, pbrl_mailbox* mb, uint64_t* version,
                       double* explore_std) {
  return mb_guarded([&] {
    if (!actor || !mb) PBRL_THROW(PBRL_E_USAGE, "actor_refresh: null argument");
    Pop* p = reinterpret_cast<Pop*>(actor);
    if (static_cast<uint64_t>(p->n) != mb->n || p->pol.P != mb->P)
      PBRL_THROW(PBRL_E_SHAPE, "actor_refresh: actor population shape differs from the mailbox's");
    CUDA_CHECK(cudaSetDevice(p->device));
    int r = -1;
    {
      std::lock_guard<std::mutex> lk(mb->mu);
      if (mb->latest < 0) {
        if (version) *version = 0;
        return;
      }
      if (mb->slot[mb->latest].version != p->snap_version) {
        r = mb->latest;
        mb->slot[r].pins += 1;
      }
    }
    if (r >= 0) {
      Slot& s = mb->slot[r];
      try {
        CUDA_CHECK(cudaStreamWaitEvent(p->stream, s.ready, 0));
        CUDA_CHECK(cudaMemcpyAsync(p->pol_p.p, s.policy.p, mb->n * mb->stride * 4,
                                   cudaMemcpyDeviceToDevice, p->stream));
        p->sync();
      } catch (...) {
        std::lock_guard<std::mutex> lk(mb->mu);
        s.pins -= 1;
        mb->cv.notify_all();
        throw;
      }
      p->weights_dirty = true;
      p->weights_written_outside();
      p->snap_explore = s.explore;
      std::lock_guard<std::mutex> lk(mb->mu);
      p->snap_version = s.version;
      s.pins -= 1;
      mb->cv.notify_all();
    }
    if (version) *version = p->snap_version;
    if (explore_std && !p->snap_explore.empty())
      std::memcpy(explore_std, p->snap_explore.data(), mb->n * 8);
  });
}

// ActorSnapshot::compute_checksum (pipeline.hpp:38-47) of the latest snapshot: FNV-1a over
// every layer's weights [N][in][out] then biases [N][1][out], then explore_std.
int pbrl_mailbox_checksum(pbrl_mailbox* mb, uint64_t* version, uint64_t* checksum) {
  return mb_guarded([&] {
    if (!mb || !checksum) PBRL_THROW(PBRL_E_USAGE, "mailbox_checksum: null argument");
    CUDA_CHECK(cudaSetDevice(mb->device));
    int r;
    {
      std::lock_guard<std::mutex> lk(mb->mu);
      r = mb->latest;
      if (r < 0) PBRL_THROW(PBRL_E_NOT_READY, "mailbox_checksum: nothing published yet");
      mb->slot[r].pins += 1;
    }
    Slot& s = mb->slot[r];
    std::vector<float> h(mb->n * mb->stride);
    cudaError_t e = cudaEventSynchronize(s.ready);
    if (e == cudaSuccess)
      e = cudaMemcpy(h.data(), s.policy.p, h.size() * 4, cudaMemcpyDeviceToHost);
    uint64_t ver;
    std::vector<double> ex;
    {
      std::lock_guard<std::mutex> lk(mb->mu);
      ver = s.version;
      ex = s.explore;
      s.pins -= 1;
      mb->cv.notify_all();
    }
    if (e != cudaSuccess) PBRL_THROW(PBRL_E_CUDA, cudaGetErrorString(e));
    uint64_t hsh = 1469598103934665603ull;
    const NetShape& sh = mb->shape;
    for (int l = 0; l < sh.depth; ++l) {
      const size_t wc = static_cast<size_t>(sh.dims[l]) * sh.dims[l + 1];
      for (uint64_t m = 0; m < mb->n; ++m)
        hsh = fnv1a(h.data() + m * mb->stride + sh.woff[l], wc * 4, hsh);
      for (uint64_t m = 0; m < mb->n; ++m)
        hsh = fnv1a(h.data() + m * mb->stride + sh.boff[l], sh.dims[l + 1] * 4, hsh);
    }
    hsh = fnv1a(ex.data(), ex.size() * 8, hsh);
    if (version) *version = ver;
    *checksum = hsh;
  });
}

}  // extern "C"
