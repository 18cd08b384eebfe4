// extern "C" boundary (include/pbrl_b200.h): error mapping, member access, replay, PBT.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <unordered_map>

#include "comm.cuh"
#include "pop_impl.cuh"
#include "tc_gemm.cuh"

namespace pbrl {

std::atomic<uint64_t> g_launches{0};

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return PBRL_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = e.what();
    return PBRL_E_RESOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PBRL_E_USAGE;
  }
}

}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

namespace {

Pop* P(pbrl_pop* h) {
  if (!h) PBRL_THROW(PBRL_E_USAGE, "null population handle");
  Pop* p = reinterpret_cast<Pop*>(h);
  CUDA_CHECK(cudaSetDevice(p->device));
  return p;
}

void check_member(const Pop* p, uint64_t m, const char* what) {
  if (m >= static_cast<uint64_t>(p->n)) PBRL_THROW(PBRL_E_USAGE, std::string(what) + ": index out of range");
}

// member index of one network (a shared critic has ONE member, algos.hpp:197)
void check_net_member(const Pop* p, int net, uint64_t m, const char* what) {
  if (m >= static_cast<uint64_t>(p->net_members(net)))
    PBRL_THROW(PBRL_E_USAGE, std::string(what) + ": index out of range");
}

// per-member splitting / exchange of whole agents (slice_member, PBT copies) has no meaning for
// a shared critic (algos.hpp:427-429, copy_member's range check net_pop.hpp:193-195)
void check_independent(const Pop* p, const char* what) {
  if (p->shared)
    PBRL_THROW(PBRL_E_USAGE, std::string(what) + ": shared-critic state cannot be split per member");
}

// RngSequence (rng.hpp:74-95) on the host, used for the PBT hyper re-draws so they match the
// reference's glibc exp/log bit for bit.
struct Seq {
  uint64_t key, next;
  double uniform(double lo, double hi) {
    const double u = static_cast<double>(rng_bits(key, next++) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
  }
  double log_uniform(double lo, double hi) { return std::exp(uniform(std::log(lo), std::log(hi))); }
};

// Td3Prior / SacPrior::sample_member (evolve.hpp:31-73): the sampled fields, then the untuned
// fields reset to their defaults (set_member copies the whole one-member hyper).
void prior_draw(int algo, Seq& rng, double* h) {
  if (algo == PBRL_ALGO_TD3) {
    h[0] = rng.log_uniform(3e-5, 3e-3);
    h[1] = rng.log_uniform(3e-5, 3e-3);
    h[2] = rng.uniform(0.2, 1.0);
    h[3] = rng.uniform(0.0, 1.0);
    h[4] = rng.uniform(0.0, 1.0);
    h[6] = rng.uniform(0.9, 1.0);
    h[5] = 0.5;
    h[7] = 0.005;
  } else {
    h[0] = rng.log_uniform(3e-5, 3e-3);
    h[1] = rng.log_uniform(3e-5, 3e-3);
    h[2] = rng.log_uniform(3e-5, 3e-3);
    h[3] = rng.uniform(0.2, 2.0) * -1.0;  // SacPrior::default_target_entropy = -1
    h[4] = rng.uniform(0.1, 10.0);
    h[5] = rng.uniform(0.9, 1.0);
    h[6] = 0.005;
  }
}

void prior_sample(Pop* p, Seq& rng, uint64_t m) {
  double h[8];
  prior_draw(p->algo, rng, h);
  const int nf = p->algo == PBRL_ALGO_TD3 ? 8 : 7;
  for (int f = 0; f < nf; ++f) p->hyper[f][m] = h[f];
}
}  // namespace

float* Pop::net_row(int net, uint64_t member) {
  switch (net) {
    case PBRL_NET_POLICY: return pol_p.p + member * pol.stride;
    case PBRL_NET_POLICY_TARGET:
      if (algo != PBRL_ALGO_TD3) PBRL_THROW(PBRL_E_USAGE, "SAC has no policy target");
      return pol_t.p + member * pol.stride;
    case PBRL_NET_CRITIC1: return cri_p.p + member * cri.stride;
    case PBRL_NET_CRITIC2: return cri_p.p + (ncrit + member) * cri.stride;
    case PBRL_NET_CRITIC1_TARGET: return cri_t.p + member * cri.stride;
    case PBRL_NET_CRITIC2_TARGET: return cri_t.p + (ncrit + member) * cri.stride;
    default: PBRL_THROW(PBRL_E_USAGE, "unknown network id");
  }
}

const NetShape& Pop::net_shape(int net) const {
  return (net == PBRL_NET_POLICY || net == PBRL_NET_POLICY_TARGET) ? pol : cri;
}

// ---------------------------------------------------------------- PBRLNET1 (net_pop.hpp:224-304)
namespace {
constexpr char kNetMagic[8] = {'P', 'B', 'R', 'L', 'N', 'E', 'T', '1'};

template <typename V>
void put(std::ostream& os, const V& v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof(V));
}
template <typename V>
V get(std::istream& is) {
  V v{};
  is.read(reinterpret_cast<char*>(&v), sizeof(V));
  return v;
}

// the whole population of one network, member rows in flatten_member order
std::vector<float> net_rows(Pop* p, int net) {
  const NetShape& sh = p->net_shape(net);
  const int rows = p->net_members(net);
  std::vector<float> flat(static_cast<size_t>(rows) * sh.P);
  CUDA_CHECK(cudaMemcpy2DAsync(flat.data(), sh.P * 4, p->net_row(net, 0), sh.stride * 4,
                               sh.P * 4, rows, cudaMemcpyDeviceToHost, p->stream));
  p->sync();
  return flat;
}

// save_checkpoint (net_pop.hpp:245-261): magic, u32 value bytes, u64 N, u64 extent count,
// u64 extents, u8 output activation, f64 output scale, members flattened in index order
void save_net(Pop* p, int net, std::ostream& os) {
  const NetShape& sh = p->net_shape(net);
  const std::vector<float> flat = net_rows(p, net);
  os.write(kNetMagic, sizeof(kNetMagic));
  put<uint32_t>(os, 4);
  put<uint64_t>(os, static_cast<uint64_t>(p->net_members(net)));
  put<uint64_t>(os, static_cast<uint64_t>(sh.depth + 1));
  for (int l = 0; l <= sh.depth; ++l) put<uint64_t>(os, static_cast<uint64_t>(sh.dims[l]));
  put<uint8_t>(os, static_cast<uint8_t>(sh.out_act));
  put<double>(os, static_cast<double>(sh.out_scale));
  os.write(reinterpret_cast<const char*>(flat.data()),
           static_cast<std::streamsize>(flat.size() * 4));
}

// load_checkpoint (net_pop.hpp:262-304) from a stream: PBRLNET1 header checks, then the rows
void load_net(Pop* p, int net, std::istream& is) {
  const NetShape& sh = p->net_shape(net);
  float* dst0 = p->net_row(net, 0);
    char magic[8];
    is.read(magic, sizeof(magic));
    if (!is || std::memcmp(magic, kNetMagic, sizeof(magic)) != 0)
      PBRL_THROW(PBRL_E_CONFIG, "load_checkpoint: bad magic");
    const uint32_t prec = get<uint32_t>(is);
    if (prec != 4)
      PBRL_THROW(PBRL_E_CONFIG, "load_checkpoint: file stores " + std::to_string(prec * 8) +
                                    "-bit values but 32-bit was requested");
    const uint64_t fn = get<uint64_t>(is), nd = get<uint64_t>(is);
    const int rows = p->net_members(net);
    if (fn != static_cast<uint64_t>(rows))
      PBRL_THROW(PBRL_E_CONFIG, "load_checkpoint: population size " + std::to_string(fn) +
                                    " != " + std::to_string(rows));
    if (nd != static_cast<uint64_t>(sh.depth + 1))
      PBRL_THROW(PBRL_E_CONFIG, "load_checkpoint: network depth mismatch");
    for (int l = 0; l <= sh.depth; ++l)
      if (get<uint64_t>(is) != static_cast<uint64_t>(sh.dims[l]))
        PBRL_THROW(PBRL_E_CONFIG, "load_checkpoint: layer extents mismatch");
    const uint8_t act = get<uint8_t>(is);
    const double scale = get<double>(is);
    if (act != static_cast<uint8_t>(sh.out_act) ||
        static_cast<float>(scale) != sh.out_scale)
      PBRL_THROW(PBRL_E_CONFIG, "load_checkpoint: output activation / scale mismatch");
    std::vector<float> flat(static_cast<size_t>(rows) * sh.P);
    is.read(reinterpret_cast<char*>(flat.data()), static_cast<std::streamsize>(flat.size() * 4));
    if (!is) PBRL_THROW(PBRL_E_CONFIG, "load_checkpoint: truncated file");
    CUDA_CHECK(cudaMemcpy2DAsync(dst0, sh.stride * 4, flat.data(), sh.P * 4, sh.P * 4, rows,
                                 cudaMemcpyHostToDevice, p->stream));
  p->weights_dirty = true;
  p->weights_written_outside();
}
}  // namespace

}  // namespace pbrl

using namespace pbrl;

extern "C" {

int pbrl_save_checkpoint(pbrl_pop* pop, int net, const char* path) {
  return guarded([&] {
    Pop* p = P(pop);
    p->net_row(net, 0);  // validates the network id
    std::ofstream os(path ? path : "", std::ios::binary);
    if (!path || !os) PBRL_THROW(PBRL_E_CONFIG, std::string("save_checkpoint: cannot open ") + (path ? path : "(null)"));
    save_net(p, net, os);
    if (!os) PBRL_THROW(PBRL_E_RESOURCE, "save_checkpoint: write failed");
  });
}

// load_checkpoint (net_pop.hpp:264-296) into an existing population: the file's population
// size, extents, activation and scale must match this network (ConfigError otherwise, as the
// reference raises for a bad magic / precision / truncated file)
int pbrl_load_checkpoint(pbrl_pop* pop, int net, const char* path) {
  return guarded([&] {
    Pop* p = P(pop);
    p->net_row(net, 0);  // validates the network id
    std::ifstream is(path ? path : "", std::ios::binary);
    if (!path || !is) PBRL_THROW(PBRL_E_CONFIG, std::string("load_checkpoint: cannot open ") + (path ? path : "(null)"));
    load_net(p, net, is);
    p->sync();
  });
}

// serialize_state (algos.hpp:989-1015), TD3: six PBRLNET1 checkpoints, then per optimizer
// (policy, critic1, critic2) for every layer the weight AdamState (m, v, t) and then every
// layer's bias AdamState, then delay_acc and steps
int pbrl_serialize_state(pbrl_pop* pop, const char* path) {
  return guarded([&] {
    Pop* p = P(pop);
    if (p->algo != PBRL_ALGO_TD3) PBRL_THROW(PBRL_E_USAGE, "serialize_state: TD3 only (as the reference)");
    std::ofstream os(path ? path : "", std::ios::binary);
    if (!path || !os) PBRL_THROW(PBRL_E_CONFIG, std::string("serialize_state: cannot open ") + (path ? path : "(null)"));
    for (int net = 0; net < 6; ++net) save_net(p, net, os);
    const int n = p->n;
    // rows: the network's members (a shared critic has one)
    auto dump_adam = [&](const NetShape& sh, int rows, const float* m_arena,
                         const float* v_arena, const int64_t* t_dev) {
      const int n = rows;
      std::vector<float> m(static_cast<size_t>(n) * sh.P), v(m.size());
      std::vector<int64_t> t(n);
      CUDA_CHECK(cudaMemcpy2DAsync(m.data(), sh.P * 4, m_arena, sh.stride * 4, sh.P * 4, n,
                                   cudaMemcpyDeviceToHost, p->stream));
      CUDA_CHECK(cudaMemcpy2DAsync(v.data(), sh.P * 4, v_arena, sh.stride * 4, sh.P * 4, n,
                                   cudaMemcpyDeviceToHost, p->stream));
      CUDA_CHECK(cudaMemcpyAsync(t.data(), t_dev, 8 * n, cudaMemcpyDeviceToHost, p->stream));
      p->sync();
      auto seg = [&](const std::vector<float>& a, size_t off, size_t cnt) {
        for (int mm = 0; mm < n; ++mm)
          os.write(reinterpret_cast<const char*>(a.data() + static_cast<size_t>(mm) * sh.P + off),
                   static_cast<std::streamsize>(cnt * 4));
      };
      for (int pass = 0; pass < 2; ++pass) {  // weights of every layer, then biases
        for (int l = 0; l < sh.depth; ++l) {
          const size_t off = pass == 0 ? sh.woff[l] : sh.boff[l];
          const size_t cnt = static_cast<size_t>(sh.dims[l + 1]) * (pass == 0 ? sh.dims[l] : 1);
          seg(m, off, cnt);
          seg(v, off, cnt);
          os.write(reinterpret_cast<const char*>(t.data()), 8 * n);
        }
      }
    };
    const int nc = p->ncrit;
    dump_adam(p->pol, n, p->pol_m.p, p->pol_v.p, p->t_pol.p);
    dump_adam(p->cri, nc, p->cri_m.p, p->cri_v.p, p->t_cri.p);
    dump_adam(p->cri, nc, p->cri_m.p + static_cast<size_t>(nc) * p->cri.stride,
              p->cri_v.p + static_cast<size_t>(nc) * p->cri.stride, p->t_cri.p + nc);
    std::vector<double> acc(n);
    std::vector<uint64_t> steps(n);
    CUDA_CHECK(cudaMemcpyAsync(acc.data(), p->delay_acc.p, 8 * n, cudaMemcpyDeviceToHost, p->stream));
    CUDA_CHECK(cudaMemcpyAsync(steps.data(), p->steps.p, 8 * n, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
    os.write(reinterpret_cast<const char*>(acc.data()), 8 * n);
    os.write(reinterpret_cast<const char*>(steps.data()), 8 * n);
    if (!os) PBRL_THROW(PBRL_E_RESOURCE, "serialize_state: write failed");
  });
}

// The inverse of serialize_state (the reference writes it but has no loader): full-trainer
// resume of a TD3 population from that byte stream -- the six networks, every Adam moment and
// step counter, delay_acc and steps.  Extents are checked against this population.
int pbrl_deserialize_state(pbrl_pop* pop, const char* path) {
  return guarded([&] {
    Pop* p = P(pop);
    if (p->algo != PBRL_ALGO_TD3) PBRL_THROW(PBRL_E_USAGE, "deserialize_state: TD3 only (as serialize_state)");
    std::ifstream is(path ? path : "", std::ios::binary);
    if (!path || !is) PBRL_THROW(PBRL_E_CONFIG, std::string("deserialize_state: cannot open ") + (path ? path : "(null)"));
    for (int net = 0; net < 6; ++net) load_net(p, net, is);
    const int n = p->n;
    int64_t tmax = 0;
    auto load_adam = [&](const NetShape& sh, int rows, float* m_arena, float* v_arena,
                         int64_t* t_dev) {
      const int n = rows;
      std::vector<float> m(static_cast<size_t>(n) * sh.P), v(m.size());
      std::vector<int64_t> t(n), t0(n);
      bool first = true;
      auto seg = [&](std::vector<float>& a, size_t off, size_t cnt) {
        for (int mm = 0; mm < n; ++mm)
          is.read(reinterpret_cast<char*>(a.data() + static_cast<size_t>(mm) * sh.P + off),
                  static_cast<std::streamsize>(cnt * 4));
      };
      for (int pass = 0; pass < 2; ++pass) {
        for (int l = 0; l < sh.depth; ++l) {
          const size_t off = pass == 0 ? sh.woff[l] : sh.boff[l];
          const size_t cnt = static_cast<size_t>(sh.dims[l + 1]) * (pass == 0 ? sh.dims[l] : 1);
          seg(m, off, cnt);
          seg(v, off, cnt);
          is.read(reinterpret_cast<char*>(first ? t0.data() : t.data()), 8 * n);
          // MlpAdam steps every tensor of a network together (optim.hpp:23-30)
          if (!first && t != t0)
            PBRL_THROW(PBRL_E_CONFIG, "deserialize_state: Adam step counters differ across tensors");
          first = false;
        }
      }
      if (!is) PBRL_THROW(PBRL_E_CONFIG, "deserialize_state: truncated file");
      CUDA_CHECK(cudaMemcpy2DAsync(m_arena, sh.stride * 4, m.data(), sh.P * 4, sh.P * 4, n,
                                   cudaMemcpyHostToDevice, p->stream));
      CUDA_CHECK(cudaMemcpy2DAsync(v_arena, sh.stride * 4, v.data(), sh.P * 4, sh.P * 4, n,
                                   cudaMemcpyHostToDevice, p->stream));
      CUDA_CHECK(cudaMemcpyAsync(t_dev, t0.data(), 8 * n, cudaMemcpyHostToDevice, p->stream));
      p->sync();
      for (int64_t x : t0) tmax = std::max(tmax, x);
    };
    const int nc = p->ncrit;
    load_adam(p->pol, n, p->pol_m.p, p->pol_v.p, p->t_pol.p);
    load_adam(p->cri, nc, p->cri_m.p, p->cri_v.p, p->t_cri.p);
    load_adam(p->cri, nc, p->cri_m.p + static_cast<size_t>(nc) * p->cri.stride,
              p->cri_v.p + static_cast<size_t>(nc) * p->cri.stride, p->t_cri.p + nc);
    std::vector<double> acc(n);
    std::vector<uint64_t> steps(n);
    is.read(reinterpret_cast<char*>(acc.data()), 8 * n);
    is.read(reinterpret_cast<char*>(steps.data()), 8 * n);
    if (!is) PBRL_THROW(PBRL_E_CONFIG, "deserialize_state: truncated file");
    is.peek();
    if (!is.eof()) PBRL_THROW(PBRL_E_CONFIG, "deserialize_state: trailing bytes (population or shape mismatch)");
    CUDA_CHECK(cudaMemcpyAsync(p->delay_acc.p, acc.data(), 8 * n, cudaMemcpyHostToDevice, p->stream));
    CUDA_CHECK(cudaMemcpyAsync(p->steps.p, steps.data(), 8 * n, cudaMemcpyHostToDevice, p->stream));
    p->delay_host = acc;
    p->t_bound = std::max<uint64_t>(p->t_bound, static_cast<uint64_t>(tmax));
    p->sync();
  });
}

int pbrl_version(int* major, int* minor) {
  if (major) *major = 0;
  if (minor) *minor = 1;
  return PBRL_OK;
}

int pbrl_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return PBRL_E_USAGE;
  std::strncpy(buf, g_last_error.c_str(), len - 1);
  buf[len - 1] = '\0';
  return PBRL_OK;
}

int pbrl_pop_create(const pbrl_pop_desc* desc, pbrl_pop** out) {
  return guarded([&] {
    if (!desc || !out) PBRL_THROW(PBRL_E_USAGE, "null argument");
    *out = reinterpret_cast<pbrl_pop*>(new Pop(*desc));
  });
}

int pbrl_pop_destroy(pbrl_pop* pop) {
  return guarded([&] {
    Pop* p = reinterpret_cast<Pop*>(pop);
    if (!p) return;
    cudaSetDevice(p->device);
    delete p->replay;
    delete p;
  });
}

int pbrl_set_hyper(pbrl_pop* pop, const char* field, const double* v) {
  return guarded([&] {
    Pop* p = P(pop);
    const int f = p->field_index(field ? field : "");
    if (f < 0) PBRL_THROW(PBRL_E_CONFIG, std::string("unknown hyperparameter ") + (field ? field : ""));
    auto saved = p->hyper[f];
    p->hyper[f].assign(v, v + p->n);
    try {
      p->validate_hyper();
    } catch (...) {
      p->hyper[f] = saved;
      throw;
    }
    p->upload_hyper();
  });
}

int pbrl_get_hyper(pbrl_pop* pop, const char* field, double* v) {
  return guarded([&] {
    Pop* p = P(pop);
    const int f = p->field_index(field ? field : "");
    if (f < 0) PBRL_THROW(PBRL_E_CONFIG, std::string("unknown hyperparameter ") + (field ? field : ""));
    std::memcpy(v, p->hyper[f].data(), sizeof(double) * p->n);
  });
}

int pbrl_param_count(pbrl_pop* pop, int net, uint64_t* count) {
  return guarded([&] {
    Pop* p = P(pop);
    p->net_row(net, 0);
    *count = p->net_shape(net).P;
  });
}

int pbrl_get_member(pbrl_pop* pop, int net, uint64_t member, float* flat) {
  return guarded([&] {
    Pop* p = P(pop);
    check_net_member(p, net, member, "flatten_member");
    const float* src = p->net_row(net, member);
    CUDA_CHECK(cudaMemcpyAsync(flat, src, p->net_shape(net).P * 4, cudaMemcpyDeviceToHost,
                               p->stream));
    p->sync();
  });
}

int pbrl_set_member(pbrl_pop* pop, int net, uint64_t member, const float* flat) {
  return guarded([&] {
    Pop* p = P(pop);
    check_net_member(p, net, member, "unflatten_member");
    float* dst = p->net_row(net, member);
    CUDA_CHECK(cudaMemcpyAsync(dst, flat, p->net_shape(net).P * 4, cudaMemcpyHostToDevice,
                               p->stream));
    p->weights_dirty = true;
    p->sync();
  });
}

int pbrl_copy_member(pbrl_pop* pop, int net, uint64_t src, uint64_t dst) {
  return guarded([&] {
    Pop* p = P(pop);
    const uint64_t rows = static_cast<uint64_t>(p->net_members(net));
    if (src >= rows || dst >= rows) PBRL_THROW(PBRL_E_USAGE, "copy_member: index out of range");
    if (src == dst) return;
    CUDA_CHECK(cudaMemcpyAsync(p->net_row(net, dst), p->net_row(net, src),
                               p->net_shape(net).P * 4, cudaMemcpyDeviceToDevice, p->stream));
    p->weights_dirty = true;
    p->sync();
  });
}

int pbrl_get_adam(pbrl_pop* pop, int net, uint64_t member, float* m, float* v, int64_t* t) {
  return guarded([&] {
    Pop* p = P(pop);
    check_net_member(p, net == PBRL_NET_POLICY ? net : PBRL_NET_CRITIC1, member, "get_adam");
    const float *pm, *pv;
    const int64_t* pt;
    size_t P_;
    if (net == PBRL_NET_POLICY) {
      pm = p->pol_m.p + member * p->pol.stride;
      pv = p->pol_v.p + member * p->pol.stride;
      pt = p->t_pol.p + member;
      P_ = p->pol.P;
    } else if (net == PBRL_NET_CRITIC1 || net == PBRL_NET_CRITIC2) {
      const uint64_t row = (net == PBRL_NET_CRITIC1 ? 0 : p->ncrit) + member;
      pm = p->cri_m.p + row * p->cri.stride;
      pv = p->cri_v.p + row * p->cri.stride;
      pt = p->t_cri.p + row;
      P_ = p->cri.P;
    } else {
      PBRL_THROW(PBRL_E_USAGE, "get_adam: network has no optimiser state");
    }
    if (m) CUDA_CHECK(cudaMemcpyAsync(m, pm, P_ * 4, cudaMemcpyDeviceToHost, p->stream));
    if (v) CUDA_CHECK(cudaMemcpyAsync(v, pv, P_ * 4, cudaMemcpyDeviceToHost, p->stream));
    if (t) CUDA_CHECK(cudaMemcpyAsync(t, pt, 8, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
  });
}

int pbrl_get_counters(pbrl_pop* pop, double* delay_acc, uint64_t* steps) {
  return guarded([&] {
    Pop* p = P(pop);
    if (delay_acc)
      CUDA_CHECK(cudaMemcpyAsync(delay_acc, p->delay_acc.p, 8 * p->n, cudaMemcpyDeviceToHost,
                                 p->stream));
    if (steps)
      CUDA_CHECK(cudaMemcpyAsync(steps, p->steps.p, 8 * p->n, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
  });
}

int pbrl_get_alpha(pbrl_pop* pop, float* log_alpha, float* m, float* v, int64_t* t) {
  return guarded([&] {
    Pop* p = P(pop);
    if (p->algo != PBRL_ALGO_SAC) PBRL_THROW(PBRL_E_USAGE, "temperature state is SAC-only");
    const size_t n = p->n;
    if (log_alpha)
      CUDA_CHECK(cudaMemcpyAsync(log_alpha, p->log_alpha.p, 4 * n, cudaMemcpyDeviceToHost, p->stream));
    if (m) CUDA_CHECK(cudaMemcpyAsync(m, p->alpha_m.p, 4 * n, cudaMemcpyDeviceToHost, p->stream));
    if (v) CUDA_CHECK(cudaMemcpyAsync(v, p->alpha_v.p, 4 * n, cudaMemcpyDeviceToHost, p->stream));
    if (t) CUDA_CHECK(cudaMemcpyAsync(t, p->t_alpha.p, 8 * n, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
  });
}

int pbrl_update_batches(pbrl_pop* pop, const pbrl_batch* batches, uint32_t k, uint64_t rows,
                        const uint8_t* policy_mask) {
  return guarded([&] { P(pop)->update_batches(batches, k, rows, policy_mask, false); });
}

int pbrl_update_batches_device(pbrl_pop* pop, const pbrl_batch* batches, uint32_t k,
                               uint64_t rows, const uint8_t* policy_mask) {
  return guarded([&] { P(pop)->update_batches(batches, k, rows, policy_mask, true); });
}

int pbrl_update_batches_losses(pbrl_pop* pop, const pbrl_batch* batches, uint32_t k,
                               uint64_t rows, const uint8_t* policy_mask, double* losses) {
  return guarded([&] {
    if (!losses) PBRL_THROW(PBRL_E_USAGE, "null losses buffer");
    P(pop)->update_batches(batches, k, rows, policy_mask, false, losses);
  });
}

int pbrl_act(pbrl_pop* pop, const float* obs, uint64_t rows, const double* noise_std,
             uint64_t seed, const uint64_t* steps, int deterministic, float* actions) {
  return guarded([&] { P(pop)->act(obs, rows, noise_std, seed, steps, deterministic, actions); });
}

int pbrl_last_losses(pbrl_pop* pop, double* c1, double* c2, double* pl) {
  return guarded([&] {
    Pop* p = P(pop);
    const size_t n = p->n;
    std::vector<double> h(3 * n);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), p->losses.p, 8 * 3 * n, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
    p->shared_losses_layout(h.data());
    if (c1) std::memcpy(c1, h.data(), 8 * n);
    if (c2) std::memcpy(c2, h.data() + n, 8 * n);
    if (pl) std::memcpy(pl, h.data() + 2 * n, 8 * n);
  });
}

// ---------------------------------------------------------------- replay
int pbrl_replay_create(pbrl_pop* pop, uint64_t capacity, int mode) {
  return guarded([&] {
    Pop* p = P(pop);
    if (capacity < 1) PBRL_THROW(PBRL_E_CONFIG, "ReplayBuffer: capacity must be >= 1");
    if (mode != PBRL_REPLAY_PER_AGENT && mode != PBRL_REPLAY_SHARED)
      PBRL_THROW(PBRL_E_CONFIG, "unknown buffer mode");
    auto* r = new Replay();
    r->mode = mode;
    r->cap = capacity;
    r->nbuf = mode == PBRL_REPLAY_PER_AGENT ? p->n : 1;
    r->rw = (2 * p->ds + p->da + 2 + 3) / 4 * 4;
    try {
      r->ring.alloc(static_cast<size_t>(r->nbuf) * capacity * r->rw);
      r->sizes.alloc(r->nbuf);
      r->sizes.zero(p->stream);
      r->ring.zero(p->stream);
    } catch (...) {
      delete r;
      throw;
    }
    r->inserts.assign(r->nbuf, 0);
    r->member.assign(static_cast<size_t>(r->nbuf) * capacity, 0u);
    delete p->replay;
    p->replay = r;
    p->sync();
  });
}

int pbrl_replay_insert(pbrl_pop* pop, const float* s, const float* a, const float* r_,
                       const float* s2, const float* d, const uint32_t* member, uint64_t count) {
  return guarded([&] {
    Pop* p = P(pop);
    Replay* r = p->replay;
    if (!r) PBRL_THROW(PBRL_E_USAGE, "replay buffer not created");
    if (count == 0) return;
    const int ds = p->ds, da = p->da, rw = r->rw;
    // ReplayBuffer::push order (replay.hpp:56-69): slot = inserts % cap, later pushes win
    std::vector<uint64_t> dst(count);
    for (uint64_t i = 0; i < count; ++i) {
      const uint64_t buf = r->mode == PBRL_REPLAY_PER_AGENT ? member[i] : 0;
      if (buf >= static_cast<uint64_t>(r->nbuf))
        PBRL_THROW(PBRL_E_USAGE, "replay insert: member id out of range");
      dst[i] = buf * r->cap + (r->inserts[buf] % r->cap);
      r->member[dst[i]] = member[i];
      r->inserts[buf]++;
    }
    std::unordered_map<uint64_t, uint64_t> last;
    last.reserve(count * 2);
    for (uint64_t i = 0; i < count; ++i) last[dst[i]] = i;
    std::vector<float> rows;
    std::vector<uint64_t> rdst;
    rows.reserve(last.size() * rw);
    for (uint64_t i = 0; i < count; ++i) {
      if (last[dst[i]] != i) continue;
      const size_t o = rows.size();
      rows.resize(o + rw, 0.0f);
      std::memcpy(&rows[o], s + i * ds, 4 * ds);
      std::memcpy(&rows[o + ds], a + i * da, 4 * da);
      std::memcpy(&rows[o + ds + da], s2 + i * ds, 4 * ds);
      rows[o + 2 * ds + da] = r_[i];
      rows[o + 2 * ds + da + 1] = d[i];
      rdst.push_back(dst[i]);
    }
    r->stage_rows.alloc(rows.size());
    r->stage_dst.alloc(rdst.size());
    r->stage_rows.upload(rows.data(), rows.size(), p->stream);
    r->stage_dst.upload(rdst.data(), rdst.size(), p->stream);
    launch_replay_scatter(r->stage_rows.p, r->stage_dst.p, rdst.size(), rw, r->ring.p, p->stream);
    p->count_launch(1);
    std::vector<uint64_t> sz(r->nbuf);
    for (int b = 0; b < r->nbuf; ++b) sz[b] = std::min<uint64_t>(r->inserts[b], r->cap);
    r->sizes.upload(sz.data(), r->nbuf, p->stream);
    p->sync();
  });
}

// ReplayBuffer::save_snapshot (replay.hpp:113-139): "PBRLBUF1", u32 value bytes, u64 capacity,
// obs_dim, act_dim, insert count, then s [cap][ds], a [cap][da], s2 [cap][ds], r [cap],
// done [cap] (every physical slot) and the u32 member ids
int pbrl_replay_save_snapshot(pbrl_pop* pop, uint64_t buffer, const char* path) {
  return guarded([&] {
    Pop* p = P(pop);
    Replay* r = p->replay;
    if (!r) PBRL_THROW(PBRL_E_USAGE, "replay buffer not created");
    if (buffer >= static_cast<uint64_t>(r->nbuf)) PBRL_THROW(PBRL_E_USAGE, "replay: buffer out of range");
    std::ofstream os(path ? path : "", std::ios::binary);
    if (!path || !os) PBRL_THROW(PBRL_E_CONFIG, "save_snapshot: cannot open file");
    const uint64_t cap = r->cap, ds = p->ds, da = p->da;
    std::vector<float> ring(cap * r->rw);
    CUDA_CHECK(cudaMemcpyAsync(ring.data(), r->ring.p + buffer * cap * r->rw, ring.size() * 4,
                               cudaMemcpyDeviceToHost, p->stream));
    p->sync();
    os.write("PBRLBUF1", 8);
    put<uint32_t>(os, 4);
    put<uint64_t>(os, cap);
    put<uint64_t>(os, ds);
    put<uint64_t>(os, da);
    put<uint64_t>(os, r->inserts[buffer]);
    auto cols = [&](uint64_t c0, uint64_t w) {
      std::vector<float> v(cap * w);
      for (uint64_t i = 0; i < cap; ++i)
        std::memcpy(&v[i * w], &ring[i * r->rw + c0], 4 * w);
      os.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 4));
    };
    cols(0, ds);                  // s
    cols(ds, da);                 // a
    cols(ds + da, ds);            // s2
    cols(2 * ds + da, 1);         // r
    cols(2 * ds + da + 1, 1);     // done
    os.write(reinterpret_cast<const char*>(r->member.data() + buffer * cap),
             static_cast<std::streamsize>(cap * 4));
    if (!os) PBRL_THROW(PBRL_E_RESOURCE, "save_snapshot: write failed");
  });
}

// ReplayBuffer::load_snapshot (replay.hpp:141-165) into ring `buffer` of this population's
// replay (the file's capacity / obs_dim / act_dim must match it)
int pbrl_replay_load_snapshot(pbrl_pop* pop, uint64_t buffer, const char* path) {
  return guarded([&] {
    Pop* p = P(pop);
    Replay* r = p->replay;
    if (!r) PBRL_THROW(PBRL_E_USAGE, "replay buffer not created");
    if (buffer >= static_cast<uint64_t>(r->nbuf)) PBRL_THROW(PBRL_E_USAGE, "replay: buffer out of range");
    std::ifstream is(path ? path : "", std::ios::binary);
    if (!path || !is) PBRL_THROW(PBRL_E_CONFIG, "load_snapshot: cannot open file");
    char magic[8];
    is.read(magic, 8);
    if (!is || std::memcmp(magic, "PBRLBUF1", 8) != 0)
      PBRL_THROW(PBRL_E_CONFIG, "ReplayBuffer::load_snapshot: bad magic");
    if (get<uint32_t>(is) != 4) PBRL_THROW(PBRL_E_CONFIG, "ReplayBuffer::load_snapshot: precision mismatch");
    const uint64_t cap = get<uint64_t>(is), ds = get<uint64_t>(is), da = get<uint64_t>(is);
    const uint64_t ins = get<uint64_t>(is);
    if (cap != r->cap || ds != static_cast<uint64_t>(p->ds) || da != static_cast<uint64_t>(p->da))
      PBRL_THROW(PBRL_E_CONFIG, "load_snapshot: capacity / dims differ from this replay buffer");
    std::vector<float> ring(cap * r->rw, 0.0f);
    auto cols = [&](uint64_t c0, uint64_t w) {
      std::vector<float> v(cap * w);
      is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * 4));
      for (uint64_t i = 0; i < cap; ++i) std::memcpy(&ring[i * r->rw + c0], &v[i * w], 4 * w);
    };
    cols(0, ds);
    cols(ds, da);
    cols(ds + da, ds);
    cols(2 * ds + da, 1);
    cols(2 * ds + da + 1, 1);
    std::vector<uint32_t> mem(cap);
    is.read(reinterpret_cast<char*>(mem.data()), static_cast<std::streamsize>(cap * 4));
    if (!is) PBRL_THROW(PBRL_E_CONFIG, "ReplayBuffer::load_snapshot: truncated file");
    CUDA_CHECK(cudaMemcpyAsync(r->ring.p + buffer * cap * r->rw, ring.data(), ring.size() * 4,
                               cudaMemcpyHostToDevice, p->stream));
    std::memcpy(r->member.data() + buffer * cap, mem.data(), cap * 4);
    r->inserts[buffer] = ins;
    std::vector<uint64_t> sz(r->nbuf);
    for (int b = 0; b < r->nbuf; ++b) sz[b] = std::min<uint64_t>(r->inserts[b], r->cap);
    r->sizes.upload(sz.data(), r->nbuf, p->stream);
    p->sync();
  });
}

int pbrl_replay_size(pbrl_pop* pop, uint64_t buffer, uint64_t* size) {
  return guarded([&] {
    Pop* p = P(pop);
    Replay* r = p->replay;
    if (!r) PBRL_THROW(PBRL_E_USAGE, "replay buffer not created");
    if (buffer >= static_cast<uint64_t>(r->nbuf)) PBRL_THROW(PBRL_E_USAGE, "buffer index out of range");
    *size = std::min<uint64_t>(r->inserts[buffer], r->cap);
  });
}

namespace {
bool replay_ready(Pop* p, uint64_t min_size) {
  Replay* r = p->replay;
  if (!r) PBRL_THROW(PBRL_E_USAGE, "replay buffer not created");
  const uint64_t need = std::max<uint64_t>(min_size, 1);
  for (int b = 0; b < r->nbuf; ++b)
    if (std::min<uint64_t>(r->inserts[b], r->cap) < need) return false;
  return true;
}

// act16: the critic-input buffers are bf16 (BF16-mode update); sample_batch reads them back
// as fp32 rows, so it gathers with act16 = 0 (the buffers hold enough bytes for either)
void gather(Pop* p, int B, uint64_t seed, uint64_t draw_id, int act16) {
  Replay* r = p->replay;
  cudaEvent_t a = nullptr;
  p->prof_begin(&a);
  launch_replay_gather(p->n, B, p->ds, p->da, p->lsa, r->rw, r->ring.p, r->cap,
                       r->mode == PBRL_REPLAY_SHARED, r->sizes.p, p->streams.p, seed, draw_id,
                       p->S.in_sa.p, p->S.in_s2a.p, p->S.sa_pi.p, p->S.r.p, p->S.d.p, act16,
                       p->stream, p->S.in_s.p, p->lsp);
  p->count_launch(1);
  p->prof_end(a, PC_GATHER, 0.0, p->pack_bytes(B), 0);
}
}  // namespace

int pbrl_sample_batch(pbrl_pop* pop, uint64_t seed, uint64_t draw_id, uint64_t rows,
                      uint64_t min_size, float* s, float* a, float* r_, float* s2, float* d,
                      int* ready) {
  return guarded([&] {
    Pop* p = P(pop);
    *ready = 0;
    if (!replay_ready(p, min_size)) return;
    const int B = static_cast<int>(rows);
    p->ensure_scratch(B);
    gather(p, B, seed, draw_id, 0);
    p->ones_dirty = true;  // the fp32 rows overwrote the critic-input block
    const size_t nb = static_cast<size_t>(p->n) * B;
    const int dsa = p->lsa;
    std::vector<float> sa(nb * dsa), s2a(nb * dsa);
    CUDA_CHECK(cudaMemcpyAsync(sa.data(), p->S.in_sa.p, 4 * nb * dsa, cudaMemcpyDeviceToHost, p->stream));
    CUDA_CHECK(cudaMemcpyAsync(s2a.data(), p->S.in_s2a.p, 4 * nb * dsa, cudaMemcpyDeviceToHost, p->stream));
    CUDA_CHECK(cudaMemcpyAsync(r_, p->S.r.p, 4 * nb, cudaMemcpyDeviceToHost, p->stream));
    CUDA_CHECK(cudaMemcpyAsync(d, p->S.d.p, 4 * nb, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
    for (size_t i = 0; i < nb; ++i) {
      std::memcpy(s + i * p->ds, &sa[i * dsa], 4 * p->ds);
      std::memcpy(a + i * p->da, &sa[i * dsa + p->ds], 4 * p->da);
      std::memcpy(s2 + i * p->ds, &s2a[i * dsa], 4 * p->ds);
    }
    *ready = 1;
  });
}

int pbrl_update_k_masked(pbrl_pop* pop, uint32_t k, uint64_t seed, uint64_t first_draw_id,
                         uint64_t rows, uint64_t min_size, const uint8_t* policy_mask, int* ready) {
  return guarded([&] {
    Pop* p = P(pop);
    *ready = 0;
    if (k < 1) PBRL_THROW(PBRL_E_CONFIG, "update_k_steps: k must be >= 1");
    if (policy_mask && p->algo != PBRL_ALGO_TD3)
      PBRL_THROW(PBRL_E_USAGE, "policy_member_mask is a TD3 option");
    if (!replay_ready(p, min_size)) return;
    p->validate_hyper();
    const int B = static_cast<int>(rows);
    p->ensure_scratch(B);
    p->ensure_ones();
    p->ensure_corr(p->t_bound + k + 4);
    const uint8_t* d_mask = nullptr;
    p->host_mask = policy_mask;
    if (policy_mask) {
      p->mask_buf.alloc(p->n);
      p->mask_buf.upload(policy_mask, p->n, p->stream);
      d_mask = p->mask_buf.p;
    }
    for (uint32_t i = 0; i < k; ++i) {
      gather(p, B, seed, first_draw_id + i, p->act16() ? 1 : 0);
      p->step(B, d_mask);
    }
    p->host_mask = nullptr;
    CUDA_CHECK(cudaGetLastError());
    *ready = 1;
  });
}

int pbrl_update_k(pbrl_pop* pop, uint32_t k, uint64_t seed, uint64_t first_draw_id,
                  uint64_t rows, uint64_t min_size, int* ready) {
  return pbrl_update_k_masked(pop, k, seed, first_draw_id, rows, min_size, nullptr, ready);
}

// ---------------------------------------------------------------- PBT
int pbrl_pbt_plan(pbrl_pop* pop, const double* fitness, uint64_t n_total, double trunc,
                  uint64_t rng_key, uint64_t* rng_next, uint64_t* replaced, uint64_t* donors,
                  uint32_t* count) {
  return guarded([&] {
    Pop* p = P(pop);
    *count = 0;
    if (n_total < 4) return;  // pbt_plan: populations smaller than 4 are left alone
    const int cut = static_cast<int>(std::ceil(trunc * static_cast<double>(n_total)));
    p->pbt_fit.alloc(n_total);
    p->pbt_order.alloc(n_total);
    p->pbt_rep.alloc(n_total);
    p->pbt_don.alloc(n_total);
    p->pbt_fit.upload(fitness, n_total, p->stream);
    launch_pbt_plan(static_cast<int>(n_total), p->pbt_fit.p, cut, rng_key, *rng_next,
                    p->pbt_order.p, p->pbt_rep.p, p->pbt_don.p, p->stream);
    p->count_launch(1);
    CUDA_CHECK(cudaMemcpyAsync(replaced, p->pbt_rep.p, 8 * cut, cudaMemcpyDeviceToHost, p->stream));
    CUDA_CHECK(cudaMemcpyAsync(donors, p->pbt_don.p, 8 * cut, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
    *rng_next += static_cast<uint64_t>(cut);
    *count = static_cast<uint32_t>(cut);
  });
}

int pbrl_pbt_apply(pbrl_pop* pop, const uint64_t* replaced, const uint64_t* donors,
                   uint32_t count) {
  return guarded([&] {
    Pop* p = P(pop);
    if (count > 0) check_independent(p, "pbt exploit copy");
    const uint64_t lo = p->member_offset, hi = lo + p->n;
    std::vector<uint64_t> src, dst, reset;
    for (uint32_t i = 0; i < count; ++i) {
      const bool dl = replaced[i] >= lo && replaced[i] < hi;
      const bool sl = donors[i] >= lo && donors[i] < hi;
      if (dl) reset.push_back(replaced[i] - lo);
      if (dl && sl) {
        dst.push_back(replaced[i] - lo);
        src.push_back(donors[i] - lo);
      }
    }
    // pairs are applied in plan order (evolve.hpp:174-187); donors and receivers are disjoint
    // strata, so one grouped copy per arena is equivalent to the sequential loop.
    const int np = static_cast<int>(src.size());
    if (np) {
      p->pbt_src.alloc(np);
      p->pbt_dst.alloc(np);
      p->pbt_src.upload(src.data(), np, p->stream);
      p->pbt_dst.upload(dst.data(), np, p->stream);
      p->weights_written_outside();
      launch_member_copy(p->pol_p.p, p->pol.stride, p->pol.P, p->pbt_src.p, p->pbt_dst.p, np, p->stream);
      if (p->algo == PBRL_ALGO_TD3)
        launch_member_copy(p->pol_t.p, p->pol.stride, p->pol.P, p->pbt_src.p, p->pbt_dst.p, np, p->stream);
      for (float* arena : {p->cri_p.p, p->cri_t.p}) {
        for (int c = 0; c < 2; ++c) {
          launch_member_copy(arena + static_cast<size_t>(c) * p->n * p->cri.stride, p->cri.stride,
                             p->cri.P, p->pbt_src.p, p->pbt_dst.p, np, p->stream);
        }
      }
      if (p->algo == PBRL_ALGO_SAC) {
        for (int i = 0; i < np; ++i)
          CUDA_CHECK(cudaMemcpyAsync(p->log_alpha.p + dst[i], p->log_alpha.p + src[i], 4,
                                     cudaMemcpyDeviceToDevice, p->stream));
      }
      p->count_launch(p->algo == PBRL_ALGO_TD3 ? 6 : 5);
      p->weights_dirty = true;
    }
    // MlpAdam::reset_member (optim.hpp:32-35), delay_acc = 0 (evolve.hpp:185)
    const int nr = static_cast<int>(reset.size());
    if (nr) {
      p->pbt_dst.alloc(std::max(np, nr));
      p->pbt_dst.upload(reset.data(), nr, p->stream);
      launch_member_zero(p->pol_m.p, p->pol.stride, p->pbt_dst.p, nr, p->stream);
      launch_member_zero(p->pol_v.p, p->pol.stride, p->pbt_dst.p, nr, p->stream);
      for (float* arena : {p->cri_m.p, p->cri_v.p}) {
        for (int c = 0; c < 2; ++c)
          launch_member_zero(arena + static_cast<size_t>(c) * p->n * p->cri.stride, p->cri.stride,
                             p->pbt_dst.p, nr, p->stream);
      }
      p->count_launch(6);
      for (uint64_t m : reset) {
        const int64_t zero = 0;
        const double dz = 0.0;
        const float fz = 0.0f;
        CUDA_CHECK(cudaMemcpyAsync(p->t_pol.p + m, &zero, 8, cudaMemcpyHostToDevice, p->stream));
        CUDA_CHECK(cudaMemcpyAsync(p->t_cri.p + m, &zero, 8, cudaMemcpyHostToDevice, p->stream));
        CUDA_CHECK(cudaMemcpyAsync(p->t_cri.p + p->n + m, &zero, 8, cudaMemcpyHostToDevice, p->stream));
        if (p->algo == PBRL_ALGO_TD3) {
          CUDA_CHECK(cudaMemcpyAsync(p->delay_acc.p + m, &dz, 8, cudaMemcpyHostToDevice, p->stream));
          if (p->delay_host.size() > m) p->delay_host[m] = 0.0;
        } else {
          CUDA_CHECK(cudaMemcpyAsync(p->t_alpha.p + m, &zero, 8, cudaMemcpyHostToDevice, p->stream));
          CUDA_CHECK(cudaMemcpyAsync(p->alpha_m.p + m, &fz, 4, cudaMemcpyHostToDevice, p->stream));
          CUDA_CHECK(cudaMemcpyAsync(p->alpha_v.p + m, &fz, 4, cudaMemcpyHostToDevice, p->stream));
        }
        p->sync();
      }
    }
    p->sync();
  });
}

int pbrl_pbt_evolve(pbrl_pop* pop, const double* fitness, uint64_t rng_key, uint64_t* rng_next,
                    uint64_t* replaced, uint64_t* donors, uint32_t* count) {
  if (pop && (reinterpret_cast<Pop*>(pop)->member_offset != 0 ||
              reinterpret_cast<Pop*>(pop)->n_global != static_cast<uint64_t>(reinterpret_cast<Pop*>(pop)->n))) {
    g_last_error = "pbt_evolve: single-shard populations only (use plan/apply + export/import)";
    return PBRL_E_USAGE;
  }
  int rc = pbrl_pbt_plan(pop, fitness, reinterpret_cast<Pop*>(pop)->n, 0.3, rng_key, rng_next,
                         replaced, donors, count);
  if (rc != PBRL_OK || *count == 0) return rc;
  rc = pbrl_pbt_apply(pop, replaced, donors, *count);
  if (rc != PBRL_OK) return rc;
  return guarded([&] {
    Pop* p = P(pop);
    Seq rng{rng_key, *rng_next};
    for (uint32_t i = 0; i < *count; ++i) prior_sample(p, rng, replaced[i] - p->member_offset);
    *rng_next = rng.next;
    p->upload_hyper();
  });
}

int pbrl_member_blob_size(pbrl_pop* pop, uint64_t* floats) {
  return guarded([&] {
    Pop* p = P(pop);
    *floats = (p->algo == PBRL_ALGO_TD3) ? 2 * p->pol.P + 4 * p->cri.P : p->pol.P + 4 * p->cri.P + 1;
  });
}

int pbrl_export_member(pbrl_pop* pop, uint64_t member, float* buf) {
  return guarded([&] {
    Pop* p = P(pop);
    check_member(p, member, "export_member");
    check_independent(p, "export_member");
    size_t at = 0;
    for (int net = 0; net < 6; ++net) {
      if (net == PBRL_NET_POLICY_TARGET && p->algo != PBRL_ALGO_TD3) continue;
      const size_t cnt = p->net_shape(net).P;
      CUDA_CHECK(cudaMemcpyAsync(buf + at, p->net_row(net, member), cnt * 4,
                                 cudaMemcpyDeviceToDevice, p->stream));
      at += cnt;
    }
    if (p->algo == PBRL_ALGO_SAC)
      CUDA_CHECK(cudaMemcpyAsync(buf + at, p->log_alpha.p + member, 4, cudaMemcpyDeviceToDevice, p->stream));
    p->sync();
  });
}

int pbrl_import_member(pbrl_pop* pop, uint64_t member, const float* buf) {
  return guarded([&] {
    Pop* p = P(pop);
    check_member(p, member, "import_member");
    check_independent(p, "import_member");
    size_t at = 0;
    for (int net = 0; net < 6; ++net) {
      if (net == PBRL_NET_POLICY_TARGET && p->algo != PBRL_ALGO_TD3) continue;
      const size_t cnt = p->net_shape(net).P;
      CUDA_CHECK(cudaMemcpyAsync(p->net_row(net, member), buf + at, cnt * 4,
                                 cudaMemcpyDeviceToDevice, p->stream));
      at += cnt;
    }
    if (p->algo == PBRL_ALGO_SAC)
      CUDA_CHECK(cudaMemcpyAsync(p->log_alpha.p + member, buf + at, 4, cudaMemcpyDeviceToDevice, p->stream));
    p->weights_dirty = true;
    p->sync();
  });
}

int pbrl_synthetic_batches_device(pbrl_pop* pop, uint64_t count, uint64_t n, uint64_t b,
                                  uint64_t ds, uint64_t da, uint64_t seed, const pbrl_batch* out) {
  return guarded([&] {
    cudaStream_t st = nullptr;
    if (pop) st = P(pop)->stream;
    if (!out) PBRL_THROW(PBRL_E_USAGE, "null output batch");
    launch_synth(count, n, b, ds, da, seed, const_cast<float*>(out->s), const_cast<float*>(out->a),
                 const_cast<float*>(out->r), const_cast<float*>(out->s2),
                 const_cast<float*>(out->done), st);
    g_launches.fetch_add(count);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int pbrl_get_stream(pbrl_pop* pop, void** stream) {
  return guarded([&] { *stream = reinterpret_cast<void*>(P(pop)->stream); });
}

int pbrl_profile_begin(pbrl_pop* pop) {
  return guarded([&] {
    Pop* p = P(pop);
    p->sync();
    p->prof.clear();
    p->prof_fired.clear();
    p->prof_step = 0;
    p->ev_used = 0;
    p->prof_on = true;
  });
}

int pbrl_profile_end(pbrl_pop* pop, char* json, size_t len) {
  return guarded([&] {
    Pop* p = P(pop);
    const std::string r = p->prof_report();
    p->prof_on = false;
    if (!json || len == 0) return;
    std::strncpy(json, r.c_str(), len - 1);
    json[len - 1] = '\0';
  });
}

int pbrl_selftest_libm(int fn, const float* dev_in, float* dev_out, uint64_t count) {
  return guarded([&] {
    if (fn < 0 || fn > 2) PBRL_THROW(PBRL_E_USAGE, "fn: 0 tanhf, 1 expf, 2 log1pf");
    launch_libm_selftest(fn, dev_in, dev_out, count, nullptr);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaDeviceSynchronize());
  });
}

static void selftest_tc(int eb, int a_mn, int b_mn, int M, int N, int K, int groups,
                        const void* A, long long a_ld, long long a_gs, const void* B,
                        long long b_ld, long long b_gs, float* C, long long c_ld, long long c_gs) {
  TcOperand a{A, static_cast<uint64_t>(a_mn ? M : K), static_cast<uint64_t>(a_mn ? K : M),
              static_cast<uint64_t>(groups), static_cast<uint64_t>(a_ld),
              static_cast<uint64_t>(a_gs)};
  TcOperand b{B, static_cast<uint64_t>(b_mn ? N : K), static_cast<uint64_t>(b_mn ? K : N),
              static_cast<uint64_t>(groups), static_cast<uint64_t>(b_ld),
              static_cast<uint64_t>(b_gs)};
  if (!tma_ok(A, a_ld, a_gs, eb) || !tma_ok(B, b_ld, b_gs, eb))
    PBRL_THROW(PBRL_E_SHAPE, "operands are not TMA-aligned");
  TcArgs g;
  g.eb = eb;
  g.M = M;
  g.N = N;
  g.K = K;
  g.groups = groups;
  g.n_members = groups;
  g.epi = EPI_STORE;
  g.C = C;
  g.c_gs = c_gs;
  g.c_rs = c_ld;
  launch_tc_gemm(a, b, a_mn != 0, b_mn != 0, g, nullptr);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaDeviceSynchronize());
}

int pbrl_selftest_tc_gemm(int a_mn, int b_mn, int M, int N, int K, int groups, const float* A,
                          long long a_ld, long long a_gs, const float* B, long long b_ld,
                          long long b_gs, float* C, long long c_ld, long long c_gs) {
  return guarded([&] {
    selftest_tc(4, a_mn, b_mn, M, N, K, groups, A, a_ld, a_gs, B, b_ld, b_gs, C, c_ld, c_gs);
  });
}

int pbrl_selftest_tc_gemm_bf16(int a_mn, int b_mn, int M, int N, int K, int groups,
                               const void* A, long long a_ld, long long a_gs, const void* B,
                               long long b_ld, long long b_gs, float* C, long long c_ld,
                               long long c_gs) {
  return guarded([&] {
    selftest_tc(2, a_mn, b_mn, M, N, K, groups, A, a_ld, a_gs, B, b_ld, b_gs, C, c_ld, c_gs);
  });
}

int pbrl_debug_tc_trace(uint64_t* stamps, int* meta, int max_launches, int* n) {
  return guarded([&] {
    if (!stamps || !meta || !n || max_launches < 0) PBRL_THROW(PBRL_E_USAGE, "null argument");
    std::vector<TcTraceMeta> m(static_cast<size_t>(max_launches));
    *n = tc_trace_dump(reinterpret_cast<unsigned long long*>(stamps), m.data(), max_launches);
    for (int i = 0; i < *n; ++i) std::memcpy(meta + 10 * i, &m[i], sizeof(TcTraceMeta));
  });
}

int pbrl_launch_count(pbrl_pop* pop, uint64_t* launches) {
  (void)pop;
  *launches = g_launches.load();
  return PBRL_OK;
}

int pbrl_synchronize(pbrl_pop* pop) {
  return guarded([&] { P(pop)->sync(); });
}

int pbrl_device_bytes(pbrl_pop* pop, uint64_t* bytes) {
  return guarded([&] {
    Pop* p = P(pop);
    uint64_t b = 0;
    for (auto* d : {&p->pol_p, &p->pol_t, &p->pol_m, &p->pol_v, &p->pol_g, &p->cri_p, &p->cri_t,
                    &p->cri_m, &p->cri_v, &p->cri_g})
      b += d->count * 4;
    if (p->replay) b += p->replay->ring.count * 4;
    *bytes = b;
  });
}


// ---------------------------------------------------------------- sharded PBT
struct pbrl_comm {
  pbrl::Comm* c;
};

int pbrl_nccl_unique_id(void* id, size_t len) {
  return guarded([&] {
    if (!id) PBRL_THROW(PBRL_E_USAGE, "null id buffer");
    nccl_unique_id(id, len);
  });
}

int pbrl_comm_create_nccl(const void* id, int rank, int world, int device, pbrl_comm** out) {
  return guarded([&] {
    if (!id || !out) PBRL_THROW(PBRL_E_USAGE, "null argument");
    *out = nullptr;
    Comm* c = make_nccl_comm(id, rank, world, device);
    *out = new pbrl_comm{c};
  });
}

int pbrl_comm_create_host(const pbrl_comm_ops* ops, int rank, int world, int device,
                          pbrl_comm** out) {
  return guarded([&] {
    if (!out) PBRL_THROW(PBRL_E_USAGE, "null argument");
    *out = nullptr;
    Comm* c = make_host_comm(ops, rank, world, device);
    *out = new pbrl_comm{c};
  });
}

int pbrl_comm_destroy(pbrl_comm* comm) {
  return guarded([&] {
    if (!comm) return;
    delete comm->c;
    delete comm;
  });
}

int pbrl_pbt_evolve_sharded(pbrl_pop* pop, pbrl_comm* comm, const double* local_fitness,
                            int local_ready, double trunc, uint64_t rng_key, uint64_t* rng_next,
                            uint64_t* replaced, uint64_t* donors, uint32_t* count,
                            double* exchange_ms) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  *count = 0;
  int rc = guarded([&] {
    Pop* p = P(pop);
    if (!comm || !comm->c) PBRL_THROW(PBRL_E_USAGE, "pbt_evolve_sharded: null comm");
    check_independent(p, "pbt_evolve_sharded");
    Comm& c = *comm->c;
    const uint64_t n = static_cast<uint64_t>(p->n);
    if (c.device != p->device) PBRL_THROW(PBRL_E_USAGE, "pbt_evolve_sharded: comm on another device");
    if (p->n_global != n * static_cast<uint64_t>(c.world) ||
        p->member_offset != n * static_cast<uint64_t>(c.rank))
      PBRL_THROW(PBRL_E_USAGE, "pbt_evolve_sharded: the population must be split in equal "
                               "contiguous blocks, rank r owning members [r*n, (r+1)*n)");
    const auto t0 = clk::now();
    // 1. readiness + fitness of every member, rank-major
    std::vector<double> send(n + 1), recv((n + 1) * c.world);
    send[0] = local_ready ? 1.0 : 0.0;
    std::memcpy(send.data() + 1, local_fitness, n * 8);
    c.allgather_f64(send.data(), n + 1, recv.data(), p->stream);
    std::vector<double> fit(n * c.world);
    std::string not_ready;
    for (int r = 0; r < c.world; ++r) {
      if (recv[r * (n + 1)] == 0.0) not_ready += (not_ready.empty() ? "" : ",") + std::to_string(r);
      std::memcpy(fit.data() + r * n, recv.data() + r * (n + 1) + 1, n * 8);
    }
    if (!not_ready.empty())
      PBRL_THROW(PBRL_E_NOT_READY, "pbt_rank: every member needs at least one recorded return "
                                   "(ranks not ready: " + not_ready + ")");
    const auto t1 = clk::now();
    // 2. the plan, identical on every rank (pbt_rank + pbt_plan, evolve.hpp:112-145)
    uint32_t cnt = 0;
    const int prc = pbrl_pbt_plan(pop, fit.data(), n * c.world, trunc, rng_key, rng_next,
                                  replaced, donors, &cnt);
    if (prc != PBRL_OK) PBRL_THROW(prc, g_last_error);
    const auto t2 = clk::now();
    if (cnt == 0) {
      if (exchange_ms) exchange_ms[0] = ms(t0, t1), exchange_ms[1] = ms(t1, t2), exchange_ms[2] = 0;
      return;
    }
    // 3. cross-rank exploit copies: one member blob per pair, grouped point-to-point
    uint64_t blob = 0;
    if (pbrl_member_blob_size(pop, &blob) != PBRL_OK) PBRL_THROW(PBRL_E_USAGE, g_last_error);
    std::vector<P2P> ops;
    std::vector<uint64_t> recv_member;
    for (uint32_t i = 0; i < cnt; ++i) {
      const int od = static_cast<int>(replaced[i] / n), os = static_cast<int>(donors[i] / n);
      if (od == os || (od != c.rank && os != c.rank)) continue;
      ops.push_back(P2P{os == c.rank ? od : os, os == c.rank, nullptr, blob});
      recv_member.push_back(os == c.rank ? ~0ull : replaced[i] - p->member_offset);
    }
    if (!ops.empty()) {
      p->pbt_blob.alloc(ops.size() * blob);
      for (size_t i = 0; i < ops.size(); ++i) ops[i].dev = p->pbt_blob.p + i * blob;
      // exports (stream-ordered copies of the donors' rows)
      for (uint32_t i = 0, k = 0; i < cnt; ++i) {
        const int od = static_cast<int>(replaced[i] / n), os = static_cast<int>(donors[i] / n);
        if (od == os || (od != c.rank && os != c.rank)) continue;
        if (os == c.rank) {
          const int erc = pbrl_export_member(pop, donors[i] - p->member_offset, ops[k].dev);
          if (erc != PBRL_OK) PBRL_THROW(erc, g_last_error);
        }
        ++k;
      }
      c.exchange(ops, p->stream);
      for (size_t k = 0; k < ops.size(); ++k) {
        if (ops[k].send) continue;
        const int irc = pbrl_import_member(pop, recv_member[k], ops[k].dev);
        if (irc != PBRL_OK) PBRL_THROW(irc, g_last_error);
      }
    }
    // local pairs + optimiser / delay resets of the local receivers
    const int arc = pbrl_pbt_apply(pop, replaced, donors, cnt);
    if (arc != PBRL_OK) PBRL_THROW(arc, g_last_error);
    // 4. hyper re-draw in lock-step: every rank draws for every replaced member
    Seq rng{rng_key, *rng_next};
    const uint64_t lo = p->member_offset, hi = lo + n;
    for (uint32_t i = 0; i < cnt; ++i) {
      double h[8];
      prior_draw(p->algo, rng, h);
      if (replaced[i] >= lo && replaced[i] < hi) {
        const int nf = p->algo == PBRL_ALGO_TD3 ? 8 : 7;
        for (int f = 0; f < nf; ++f) p->hyper[f][replaced[i] - lo] = h[f];
      }
    }
    *rng_next = rng.next;
    p->upload_hyper();
    p->sync();
    *count = cnt;
    if (exchange_ms) exchange_ms[0] = ms(t0, t1), exchange_ms[1] = ms(t1, t2), exchange_ms[2] = ms(t2, clk::now());
  });
  return rc;
}


// ---------------------------------------------------------------- member state copy (a22)
// slice_member / set_member for whole states (algos.hpp:425-464, :839-886): every network, the
// Adam moments and step counters, steps / streams, delay_acc (TD3) or the temperature and its
// optimiser (SAC), and the member's hypers.  dst and src may be different populations (a
// population and one of its singletons) of the same algorithm and shapes.
int pbrl_copy_member_state(pbrl_pop* dst_pop, uint64_t dm, pbrl_pop* src_pop, uint64_t sm) {
  return guarded([&] {
    Pop* s = P(src_pop);
    Pop* d = P(dst_pop);
    check_independent(s, "slice_member");
    check_independent(d, "set_member");
    check_member(s, sm, "copy_member_state (source)");
    check_member(d, dm, "copy_member_state (destination)");
    if (s->algo != d->algo || s->ds != d->ds || s->da != d->da || s->hidden != d->hidden ||
        s->bound != d->bound)
      PBRL_THROW(PBRL_E_SHAPE, "copy_member_state: populations differ in algorithm or shapes");
    s->sync();
    cudaStream_t st = d->stream;
    auto cp = [&](void* to, const void* from, size_t bytes) {
      CUDA_CHECK(cudaMemcpyAsync(to, from, bytes, cudaMemcpyDefault, st));
    };
    for (int net = 0; net < 6; ++net) {
      if (net == PBRL_NET_POLICY_TARGET && s->algo != PBRL_ALGO_TD3) continue;
      cp(d->net_row(net, dm), s->net_row(net, sm), d->net_shape(net).P * 4);
    }
    for (auto pr : {std::make_pair(&d->pol_m, &s->pol_m), std::make_pair(&d->pol_v, &s->pol_v)})
      cp(pr.first->p + dm * d->pol.stride, pr.second->p + sm * s->pol.stride, d->pol.P * 4);
    for (auto pr : {std::make_pair(&d->cri_m, &s->cri_m), std::make_pair(&d->cri_v, &s->cri_v)})
      for (int c = 0; c < 2; ++c)
        cp(pr.first->p + (c * d->n + dm) * d->cri.stride,
           pr.second->p + (c * s->n + sm) * s->cri.stride, d->cri.P * 4);
    cp(d->t_pol.p + dm, s->t_pol.p + sm, 8);
    cp(d->t_cri.p + dm, s->t_cri.p + sm, 8);
    cp(d->t_cri.p + d->n + dm, s->t_cri.p + s->n + sm, 8);
    cp(d->steps.p + dm, s->steps.p + sm, 8);
    cp(d->streams.p + dm, s->streams.p + sm, 8);
    if (s->algo == PBRL_ALGO_TD3) {
      cp(d->delay_acc.p + dm, s->delay_acc.p + sm, 8);
      if (d->delay_host.size() != static_cast<size_t>(d->n)) d->delay_host.assign(d->n, 0.0);
      d->delay_host[dm] = s->delay_host.size() > sm ? s->delay_host[sm] : 0.0;
    } else {
      cp(d->log_alpha.p + dm, s->log_alpha.p + sm, 4);
      cp(d->alpha_m.p + dm, s->alpha_m.p + sm, 4);
      cp(d->alpha_v.p + dm, s->alpha_v.p + sm, 4);
      cp(d->t_alpha.p + dm, s->t_alpha.p + sm, 8);
    }
    for (size_t f = 0; f < d->hyper.size(); ++f) d->hyper[f][dm] = s->hyper[f][sm];
    d->upload_hyper();
    d->t_bound = std::max(d->t_bound, s->t_bound);
    d->weights_dirty = true;
    d->weights_written_outside();
    d->sync();
  });
}

// ---------------------------------------------------------------- shared critic over shards
int pbrl_attach_comm(pbrl_pop* pop, pbrl_comm* comm) {
  return guarded([&] {
    Pop* p = P(pop);
    if (!comm) {
      p->comm_reduce = nullptr;
      p->use_graphs = p->graphs_allowed;
      p->invalidate_graphs();
      return;
    }
    if (!comm->c) PBRL_THROW(PBRL_E_USAGE, "attach_comm: null comm");
    if (!p->shared)
      PBRL_THROW(PBRL_E_USAGE, "attach_comm: only a shared-critic population exchanges data per step");
    Comm* c = comm->c;
    if (p->n_global != static_cast<uint64_t>(p->n) * c->world ||
        p->member_offset != static_cast<uint64_t>(p->n) * c->rank)
      PBRL_THROW(PBRL_E_CONFIG, "attach_comm: shard layout != (rank * n, world * n)");
    p->comm_reduce = [c](float* buf, size_t count, cudaStream_t s) { c->allreduce_f32(buf, count, s); };
    p->use_graphs = false;  // the host transport cannot sit inside a graph
    p->invalidate_graphs();
  });
}

// ---------------------------------------------------------------- DvD (evolve.hpp:304-525)
int pbrl_set_dvd(pbrl_pop* pop, const double* probe, uint64_t m_states, double length_scale,
                 double jitter, double lambda) {
  return guarded([&] { P(pop)->set_dvd(probe, m_states, length_scale, jitter, lambda); });
}

int pbrl_dvd_embed(pbrl_pop* pop, const double* probe, uint64_t m_states, float* out) {
  return guarded([&] {
    Pop* p = P(pop);
    if (p->algo != PBRL_ALGO_TD3) PBRL_THROW(PBRL_E_USAGE, "dvd_embed: TD3 policies only");
    if (!probe || !out || m_states < 1) PBRL_THROW(PBRL_E_SHAPE, "dvd_embed: probe matrix size != M * observation_dim");
    // dvd_embed_cached (:319-335): probes (double -> T) replicated per member, then the policy
    // forward == deterministic act
    const size_t per = static_cast<size_t>(m_states) * p->ds;
    std::vector<float> obs(per * p->n);
    for (int m = 0; m < p->n; ++m)
      for (size_t i = 0; i < per; ++i) obs[m * per + i] = static_cast<float>(probe[i]);
    std::vector<uint64_t> steps(p->n, 0);
    p->act(obs.data(), m_states, nullptr, 0, steps.data(), 1, out);
  });
}

int pbrl_dvd_loss(const double* emb, uint64_t n, uint64_t dim, double length_scale, double jitter,
                  double lambda, double* loss, double* logdet, double* grad) {
  return guarded([&] {
    if (!emb && n > 0) PBRL_THROW(PBRL_E_USAGE, "dvd_loss: null embeddings");
    dvd_loss_host(emb, n, dim, length_scale, jitter, lambda, loss, logdet, grad);
  });
}

int pbrl_median_pairwise_distance(const double* emb, uint64_t n, uint64_t dim, double* out) {
  return guarded([&] { *out = median_pairwise_distance_host(emb, n, dim); });
}

int pbrl_dvd_lambda(uint64_t step, double start, double end, uint64_t horizon, double* out) {
  return guarded([&] {
    if (horizon == 0 || step >= horizon) {
      *out = end;
    } else {
      const double frac = static_cast<double>(step) / static_cast<double>(horizon);
      *out = start + (end - start) * frac;
    }
  });
}

// ---------------------------------------------------------------- CEM (evolve.hpp:221-297)
struct pbrl_cem {
  std::unique_ptr<Cem> c;
};

int pbrl_cem_create(pbrl_pop* pop, const double* mean, double init_var, pbrl_cem** out) {
  return guarded([&] {
    if (!out) PBRL_THROW(PBRL_E_USAGE, "null output handle");
    auto h = std::make_unique<pbrl_cem>();
    h->c = std::make_unique<Cem>(P(pop), mean, init_var);
    *out = h.release();
  });
}

int pbrl_cem_destroy(pbrl_cem* cem) {
  delete cem;
  return PBRL_OK;
}

static Cem& C_(pbrl_cem* h) {
  if (!h || !h->c) PBRL_THROW(PBRL_E_USAGE, "null CEM handle");
  CUDA_CHECK(cudaSetDevice(h->c->pop->device));
  return *h->c;
}

int pbrl_cem_set_params(pbrl_cem* cem, double noise, double noise_final, double noise_decay,
                        double elite_fraction) {
  return guarded([&] {
    Cem& c = C_(cem);
    c.noise = noise;
    c.noise_final = noise_final;
    c.noise_decay = noise_decay;
    c.elite_fraction = elite_fraction;
  });
}

int pbrl_cem_get(pbrl_cem* cem, double* mean, double* var, double* noise) {
  return guarded([&] {
    Cem& c = C_(cem);
    cudaStream_t s = c.pop->stream;
    if (mean) CUDA_CHECK(cudaMemcpyAsync(mean, c.mean.p, c.dim * 8, cudaMemcpyDeviceToHost, s));
    if (var) CUDA_CHECK(cudaMemcpyAsync(var, c.var.p, c.dim * 8, cudaMemcpyDeviceToHost, s));
    c.pop->sync();
    if (noise) *noise = c.noise;
  });
}

int pbrl_cem_resample(pbrl_cem* cem, uint64_t rng_key, uint64_t* rng_next) {
  return guarded([&] {
    if (!rng_next) PBRL_THROW(PBRL_E_USAGE, "null rng counter");
    C_(cem).resample(rng_key, rng_next);
  });
}

int pbrl_cem_candidates(pbrl_cem* cem, double* out) {
  return guarded([&] {
    Cem& c = C_(cem);
    CUDA_CHECK(cudaMemcpyAsync(out, c.cand.p, c.cand.count * 8, cudaMemcpyDeviceToHost,
                               c.pop->stream));
    c.pop->sync();
  });
}

int pbrl_cem_update(pbrl_cem* cem, const double* scores, uint64_t count) {
  return guarded([&] { C_(cem).update(scores, count); });
}

}  // extern "C"

