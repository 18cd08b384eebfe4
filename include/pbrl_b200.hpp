// pbrl_b200.hpp -- C++ facade over the C ABI (pbrl_b200.h) with the reference's names,
// argument meanings and exception types (proj/core/include/pbrl/{algos,replay,evolve,errors}.hpp),
// so code written against the reference population-trainer API switches by changing
// `namespace pbrl` to `namespace pbrl::b200` and linking libpbrl_b200.so.
//
//   reference                                   here
//   make_td3_state<T>(n, ds, da, hidden, ...)   make_td3_state(n, ds, da, hidden, bound, seed)
//   td3_update_step(st, batch, hyper[, ...])    td3_update_step(st, batch, hyper[, mask])
//   update_k_steps(st, sampler, k, hyper)       update_k_steps(st, sampler, k, hyper)
//   make_sac_state / sac_update_step            same
//   flatten_member(st.policy, i)                st.flatten_member(Net::kPolicy, i)
//   ReplayBuffer + sample_batch                 DeviceReplay + sample_batch / update_k_from_replay
//   pbt_plan / pbt_evolve_trainer               pbt_plan / pbt_evolve_trainer
// State lives in HBM on the population's device; batches are host arrays laid out like
// TransitionBatch (algos.hpp:14-24), row-major [N][B][dim].
#pragma once

#include <algorithm>
#include <cstdint>
#include <deque>
#include <functional>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbrl_b200.h"

namespace pbrl::b200 {

// ---------------------------------------------------------------- errors (errors.hpp:9-48)
class ShapeError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class ConfigError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class UsageError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};
class NotReadyError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ResourceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DataStarvationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DegeneratePopulationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == PBRL_OK) return;
  char buf[1024];
  pbrl_last_error(buf, sizeof(buf));
  const std::string m(buf);
  switch (rc) {
    case PBRL_E_SHAPE: throw ShapeError(m);
    case PBRL_E_CONFIG: throw ConfigError(m);
    case PBRL_E_USAGE: throw UsageError(m);
    case PBRL_E_NOT_READY: throw NotReadyError(m);
    case PBRL_E_RESOURCE: throw ResourceError(m);
    case PBRL_E_STARVATION: throw DataStarvationError(m);
    case PBRL_E_DEGENERATE: throw DegeneratePopulationError(m);
    default: throw DeviceError(m);
  }
}

enum class Net : int {
  kPolicy = PBRL_NET_POLICY,
  kPolicyTarget = PBRL_NET_POLICY_TARGET,
  kCritic1 = PBRL_NET_CRITIC1,
  kCritic2 = PBRL_NET_CRITIC2,
  kCritic1Target = PBRL_NET_CRITIC1_TARGET,
  kCritic2Target = PBRL_NET_CRITIC2_TARGET,
};
enum class Precision : int { kFfma32 = PBRL_PREC_FFMA32, kTf32 = PBRL_PREC_TF32, kBf16 = PBRL_PREC_BF16 };
enum class PopMode : int {  // algos.hpp:26
  kIndependent = PBRL_MODE_INDEPENDENT,
  kSharedCritic = PBRL_MODE_SHARED_CRITIC,
};

// ---------------------------------------------------------------- batches (algos.hpp:14-24)
struct TransitionBatch {
  std::vector<float> s, a, r, s2, done;  // [N][B][ds], [N][B][da], [N][B], [N][B][ds], [N][B]
  std::size_t n = 0, rows = 0;
  std::size_t members() const { return n; }
  pbrl_batch view() const { return pbrl_batch{s.data(), a.data(), r.data(), s2.data(), done.data()}; }
};

// ---------------------------------------------------------------- hyperparameters
struct Td3Hyper {  // algos.hpp:32-109
  std::vector<double> critic_lr, policy_lr, policy_delay_ratio, explore_std, target_std,
      target_clip, gamma, tau;
  static Td3Hyper defaults(std::size_t n) {
    Td3Hyper h;
    h.critic_lr.assign(n, 3e-4);
    h.policy_lr.assign(n, 3e-4);
    h.policy_delay_ratio.assign(n, 0.5);
    h.explore_std.assign(n, 0.1);
    h.target_std.assign(n, 0.2);
    h.target_clip.assign(n, 0.5);
    h.gamma.assign(n, 0.99);
    h.tau.assign(n, 0.005);
    return h;
  }
  std::vector<std::pair<const char*, const std::vector<double>*>> fields() const {
    return {{"critic_lr", &critic_lr},     {"policy_lr", &policy_lr},
            {"policy_delay_ratio", &policy_delay_ratio}, {"explore_std", &explore_std},
            {"target_std", &target_std},   {"target_clip", &target_clip},
            {"gamma", &gamma},             {"tau", &tau}};
  }
};

struct SacHyper {  // algos.hpp:112-156
  std::vector<double> policy_lr, critic_lr, alpha_lr, target_entropy, reward_scale, gamma, tau;
  static SacHyper defaults(std::size_t n, std::size_t action_dim) {
    SacHyper h;
    h.policy_lr.assign(n, 3e-4);
    h.critic_lr.assign(n, 3e-4);
    h.alpha_lr.assign(n, 3e-4);
    h.target_entropy.assign(n, -static_cast<double>(action_dim));
    h.reward_scale.assign(n, 1.0);
    h.gamma.assign(n, 0.99);
    h.tau.assign(n, 0.005);
    return h;
  }
  std::vector<std::pair<const char*, const std::vector<double>*>> fields() const {
    return {{"policy_lr", &policy_lr},       {"critic_lr", &critic_lr},
            {"alpha_lr", &alpha_lr},         {"target_entropy", &target_entropy},
            {"reward_scale", &reward_scale}, {"gamma", &gamma},
            {"tau", &tau}};
  }
};

// ---------------------------------------------------------------- population state
class Population {
 public:
  Population(int algo, std::size_t n, std::size_t obs_dim, std::size_t act_dim,
             const std::vector<std::size_t>& hidden, double action_bound, std::uint64_t seed,
             Precision precision = Precision::kFfma32, int device = 0,
             std::uint64_t member_offset = 0, std::uint64_t n_global = 0,
             PopMode mode = PopMode::kIndependent)
      : n_(n), ds_(obs_dim), da_(act_dim) {
    std::vector<std::uint64_t> h(hidden.begin(), hidden.end());
    pbrl_pop_desc d{};
    d.algo = algo;
    d.n = n;
    d.obs_dim = obs_dim;
    d.act_dim = act_dim;
    d.n_hidden = static_cast<std::uint32_t>(h.size());
    d.hidden = h.data();
    d.action_bound = action_bound;
    d.seed = seed;
    d.precision = static_cast<int>(precision);
    d.device = device;
    d.member_offset = member_offset;
    d.n_global = n_global;
    d.mode = static_cast<int>(mode);
    check(pbrl_pop_create(&d, &h_));
  }
  ~Population() {
    if (h_) pbrl_pop_destroy(h_);
  }
  Population(const Population&) = delete;
  Population& operator=(const Population&) = delete;
  Population(Population&& o) noexcept : h_(o.h_), n_(o.n_), ds_(o.ds_), da_(o.da_) { o.h_ = nullptr; }

  std::size_t members() const { return n_; }
  std::size_t obs_dim() const { return ds_; }
  std::size_t act_dim() const { return da_; }
  pbrl_pop* handle() const { return h_; }

  std::vector<float> flatten_member(Net net, std::size_t i) const {  // net_pop.hpp:163-173
    std::uint64_t c = 0;
    check(pbrl_param_count(h_, static_cast<int>(net), &c));
    std::vector<float> out(c);
    check(pbrl_get_member(h_, static_cast<int>(net), i, out.data()));
    return out;
  }
  void unflatten_member(Net net, std::size_t i, const std::vector<float>& v) {  // :176-189
    check(pbrl_set_member(h_, static_cast<int>(net), i, v.data()));
  }
  void copy_member(Net net, std::size_t src, std::size_t dst) {  // :192-202
    check(pbrl_copy_member(h_, static_cast<int>(net), src, dst));
  }
  std::vector<std::uint64_t> steps() const {
    std::vector<std::uint64_t> s(n_);
    check(pbrl_get_counters(h_, nullptr, s.data()));
    return s;
  }

 protected:
  template <typename H>
  void sync_hyper(const H& hy) {
    for (auto& [name, vec] : hy.fields()) {
      if (vec->size() != n_) throw ConfigError(std::string("hyper: ") + name + " length != N");
      check(pbrl_set_hyper(h_, name, vec->data()));
    }
  }
  friend void td3_update_step(class Td3State&, const TransitionBatch&, const Td3Hyper&,
                              const struct PolicyGradHook*, const std::vector<char>*);
  friend void sac_update_step(class SacState&, const TransitionBatch&, const SacHyper&);
  template <typename S, typename H>
  friend void update_k_steps(S&, const std::function<std::optional<TransitionBatch>()>&,
                             std::size_t, const H&);

  pbrl_pop* h_ = nullptr;
  std::size_t n_, ds_, da_;
};

class Td3State : public Population {  // algos.hpp:165-212
 public:
  using Population::Population;
  std::vector<double> delay_acc() const {
    std::vector<double> d(n_);
    check(pbrl_get_counters(h_, d.data(), nullptr));
    return d;
  }
};

class SacState : public Population {  // algos.hpp:473-521
 public:
  using Population::Population;
};

inline Td3State make_td3_state(std::size_t n, std::size_t obs_dim, std::size_t act_dim,
                               const std::vector<std::size_t>& hidden, double action_bound,
                               std::uint64_t seed, PopMode mode = PopMode::kIndependent,
                               Precision precision = Precision::kFfma32, int device = 0) {
  return Td3State(PBRL_ALGO_TD3, n, obs_dim, act_dim, hidden, action_bound, seed, precision,
                  device, 0, 0, mode);
}

inline SacState make_sac_state(std::size_t n, std::size_t obs_dim, std::size_t act_dim,
                               const std::vector<std::size_t>& hidden, double action_bound,
                               std::uint64_t seed, PopMode mode = PopMode::kIndependent,
                               Precision precision = Precision::kFfma32, int device = 0) {
  return SacState(PBRL_ALGO_SAC, n, obs_dim, act_dim, hidden, action_bound, seed, precision,
                  device, 0, 0, mode);
}

// ---------------------------------------------------------------- DvD (evolve.hpp:304-525)
struct LambdaSchedule {
  double start = 0.0;
  double end = 0.5;
  std::uint64_t horizon = 1;
};

inline double dvd_lambda(std::uint64_t step, const LambdaSchedule& s) {
  double out = 0;
  check(pbrl_dvd_lambda(step, s.start, s.end, s.horizon, &out));
  return out;
}

struct DvDConfig {
  std::vector<double> probe_states;  // row-major M x ds
  std::size_t m_states = 0;
  double length_scale = 1.0;
  double jitter = 1e-6;
  LambdaSchedule schedule;
  void validate(std::size_t population) const {
    if (m_states < population)
      throw ConfigError("DvDConfig: need at least as many probe states as members");
    if (!(length_scale > 0)) throw ConfigError("DvDConfig: length scale must be positive");
    if (jitter < 0) throw ConfigError("DvDConfig: jitter must be >= 0");
  }
};

// dvd_policy_hook(cfg, step): applied on the device inside the update calls it is passed to
struct PolicyGradHook {
  DvDConfig cfg;
  double lambda = 0.0;
};
inline PolicyGradHook dvd_policy_hook(const DvDConfig& cfg, std::uint64_t step) {
  return PolicyGradHook{cfg, dvd_lambda(step, cfg.schedule)};
}

struct DvdLossOut {
  double loss = 0, logdet = 0;
  std::vector<double> grad;  // [N][E]
};
inline DvdLossOut dvd_loss(const std::vector<double>& emb, std::size_t n, double length_scale,
                           double jitter, double lambda) {
  if (n == 0 || emb.size() % n != 0) throw ShapeError("dvd_loss: embeddings not [N, E]");
  DvdLossOut o;
  o.grad.assign(emb.size(), 0.0);
  check(pbrl_dvd_loss(emb.data(), n, emb.size() / n, length_scale, jitter, lambda, &o.loss,
                      &o.logdet, o.grad.data()));
  return o;
}
inline double median_pairwise_distance(const std::vector<double>& emb, std::size_t n) {
  double out = 1.0;
  check(pbrl_median_pairwise_distance(emb.data(), n, n ? emb.size() / n : 0, &out));
  return out;
}
inline std::vector<float> dvd_embed(Population& policies, const std::vector<double>& probe,
                                    std::size_t m_states) {
  std::vector<float> out(policies.members() * m_states * policies.act_dim());
  check(pbrl_dvd_embed(policies.handle(), probe.data(), m_states, out.data()));
  return out;
}

namespace detail {
struct HookScope {  // installs the hook for one update call
  pbrl_pop* h;
  bool on;
  HookScope(pbrl_pop* pop, const PolicyGradHook* hook, std::size_t obs_dim) : h(pop), on(hook) {
    if (!hook) return;
    if (hook->cfg.probe_states.size() != hook->cfg.m_states * obs_dim)
      throw ShapeError("dvd_embed: probe matrix size != M * observation_dim");
    check(pbrl_set_dvd(h, hook->cfg.probe_states.data(), hook->cfg.m_states,
                       hook->cfg.length_scale, hook->cfg.jitter, hook->lambda));
  }
  ~HookScope() {
    if (on) pbrl_set_dvd(h, nullptr, 0, 1.0, 0.0, 0.0);
  }
};
}  // namespace detail

// ---------------------------------------------------------------- CEM (evolve.hpp:221-297)
// The search distribution lives on the population's device; cem_resample draws the candidates
// straight into the policies (pipeline_run.hpp:148-158).
class CEMState {
 public:
  CEMState(Population& policies, const std::vector<double>* mean, double init_var)
      : pop_(&policies) {
    check(pbrl_cem_create(policies.handle(), mean ? mean->data() : nullptr, init_var, &h_));
  }
  ~CEMState() {
    if (h_) pbrl_cem_destroy(h_);
  }
  CEMState(const CEMState&) = delete;
  CEMState& operator=(const CEMState&) = delete;
  double noise = 1e-2, noise_init = 1e-2, noise_final = 1e-3, noise_decay = 0.999;
  double elite_fraction = 0.5;
  pbrl_cem* handle() const { return h_; }
  Population& population() const { return *pop_; }
  void push() const { check(pbrl_cem_set_params(h_, noise, noise_final, noise_decay, elite_fraction)); }

 private:
  Population* pop_;
  pbrl_cem* h_ = nullptr;
};

// cem_resample: RngSequence (key, *next) as the reference's RngSequence(seed, 2, kCemDraw, gen)
inline void cem_resample(CEMState& st, std::uint64_t rng_key, std::uint64_t* rng_next) {
  st.push();
  check(pbrl_cem_resample(st.handle(), rng_key, rng_next));
}
inline void cem_resample_into(CEMState& st, std::uint64_t rng_key, std::uint64_t* rng_next) {
  cem_resample(st, rng_key, rng_next);
}
inline void cem_update(CEMState& st, const std::vector<double>& scores) {
  st.push();
  check(pbrl_cem_update(st.handle(), scores.data(), scores.size()));
  st.noise = std::max(st.noise_final, st.noise * st.noise_decay);
}

// td3_update_step (algos.hpp:351-422); policy_member_mask as in the reference
inline void td3_update_step(Td3State& st, const TransitionBatch& batch, const Td3Hyper& hyper,
                            const PolicyGradHook* hook = nullptr,
                            const std::vector<char>* policy_member_mask = nullptr) {
  if (batch.members() != st.members())
    throw ConfigError("td3_update_step: batch population != state population");
  st.sync_hyper(hyper);
  detail::HookScope hs(st.handle(), hook, st.obs_dim());
  const pbrl_batch b = batch.view();
  std::vector<std::uint8_t> mask;
  if (policy_member_mask) mask.assign(policy_member_mask->begin(), policy_member_mask->end());
  check(pbrl_update_batches(st.h_, &b, 1, batch.rows, mask.empty() ? nullptr : mask.data()));
}

// act (algos.hpp:895-915) / sac_act (:918-942): obs [n][rows][obs_dim] -> actions
// [n][rows][act_dim], exploration noise keyed by (seed, member streams, kExploreNoise, steps[m])
inline std::vector<float> act(Td3State& st, const std::vector<float>& obs, std::size_t rows,
                              const std::vector<double>& noise_std, std::uint64_t seed,
                              const std::vector<std::uint64_t>& steps, bool deterministic) {
  if (obs.size() != st.members() * rows * st.obs_dim() || steps.size() != st.members() ||
      noise_std.size() != st.members())
    throw ShapeError("act: observation / steps / noise_std extents do not match the population");
  std::vector<float> out(st.members() * rows * st.act_dim());
  check(pbrl_act(st.handle(), obs.data(), rows, noise_std.data(), seed, steps.data(),
                 deterministic ? 1 : 0, out.data()));
  return out;
}

inline std::vector<float> sac_act(SacState& st, const std::vector<float>& obs, std::size_t rows,
                                  std::uint64_t seed, const std::vector<std::uint64_t>& steps,
                                  bool deterministic) {
  if (obs.size() != st.members() * rows * st.obs_dim() || steps.size() != st.members())
    throw ShapeError("sac_act: observation / steps extents do not match the population");
  std::vector<float> out(st.members() * rows * st.act_dim());
  check(pbrl_act(st.handle(), obs.data(), rows, nullptr, seed, steps.data(),
                 deterministic ? 1 : 0, out.data()));
  return out;
}

inline void sac_update_step(SacState& st, const TransitionBatch& batch, const SacHyper& hyper) {
  if (batch.members() != st.members())
    throw ConfigError("sac_update_step: batch population != state population");
  st.sync_hyper(hyper);
  const pbrl_batch b = batch.view();
  check(pbrl_update_batches(st.h_, &b, 1, batch.rows, nullptr));
}

// update_k_steps (algos.hpp:953-983): k chained steps, DataStarvationError if the sampler runs dry
template <typename S, typename H>
void update_k_steps(S& st, const std::function<std::optional<TransitionBatch>()>& sampler,
                    std::size_t k, const H& hyper) {
  if (k < 1) throw ConfigError("update_k_steps: k must be >= 1");
  std::vector<TransitionBatch> batches;
  for (std::size_t i = 0; i < k; ++i) {
    auto b = sampler();
    if (!b)
      throw DataStarvationError("update_k_steps: sampler exhausted after " + std::to_string(i) +
                                " of " + std::to_string(k) + " steps");
    batches.push_back(std::move(*b));
  }
  st.sync_hyper(hyper);
  std::vector<pbrl_batch> views;
  for (auto& b : batches) views.push_back(b.view());
  check(pbrl_update_batches(st.h_, views.data(), static_cast<std::uint32_t>(k), batches[0].rows,
                            nullptr));
}

// ---------------------------------------------------------------- replay (replay.hpp)
enum class BufferMode { kPerAgent = PBRL_REPLAY_PER_AGENT, kShared = PBRL_REPLAY_SHARED };

class DeviceReplay {
 public:
  DeviceReplay(Population& pop, std::size_t capacity, BufferMode mode = BufferMode::kPerAgent)
      : pop_(pop) {
    check(pbrl_replay_create(pop.handle(), capacity, static_cast<int>(mode)));
  }
  // batched ReplayBuffer::push (replay.hpp:56-69)
  void insert(const std::vector<float>& s, const std::vector<float>& a,
              const std::vector<float>& r, const std::vector<float>& s2,
              const std::vector<float>& done, const std::vector<std::uint32_t>& member) {
    check(pbrl_replay_insert(pop_.handle(), s.data(), a.data(), r.data(), s2.data(), done.data(),
                             member.data(), member.size()));
  }
  std::size_t size(std::size_t buffer = 0) const {
    std::uint64_t s = 0;
    check(pbrl_replay_size(pop_.handle(), buffer, &s));
    return s;
  }
  Population& pop() { return pop_; }

 private:
  Population& pop_;
};

// sample_batch (replay.hpp:181-204): nullopt when a source buffer holds < max(min_size, 1)
inline std::optional<TransitionBatch> sample_batch(DeviceReplay& rb, std::size_t batch_size,
                                                   std::uint64_t seed, std::uint64_t draw_id,
                                                   std::size_t obs_dim, std::size_t act_dim,
                                                   std::size_t min_size = 1) {
  const std::size_t n = rb.pop().members();
  TransitionBatch b;
  b.n = n;
  b.rows = batch_size;
  b.s.resize(n * batch_size * obs_dim);
  b.a.resize(n * batch_size * act_dim);
  b.r.resize(n * batch_size);
  b.s2.resize(n * batch_size * obs_dim);
  b.done.resize(n * batch_size);
  int ready = 0;
  check(pbrl_sample_batch(rb.pop().handle(), seed, draw_id, batch_size, min_size, b.s.data(),
                          b.a.data(), b.r.data(), b.s2.data(), b.done.data(), &ready));
  if (!ready) return std::nullopt;
  return b;
}

// ---------------------------------------------------------------- PBT (evolve.hpp)
struct PBTState {  // evolve.hpp:80-108
  std::vector<std::deque<double>> returns;
  std::size_t ring_capacity = 10;
  std::uint64_t steps_since_evolve = 0;
  std::uint64_t evolve_interval = 100000;
  double truncation_fraction = 0.3;
  explicit PBTState(std::size_t n = 0) : returns(n) {}
  void record_return(std::size_t m, double v) {
    auto& ring = returns.at(m);
    ring.push_back(v);
    while (ring.size() > ring_capacity) ring.pop_front();
  }
  std::vector<double> fitness() const {
    std::vector<double> f;
    for (const auto& r : returns) {
      if (r.empty()) throw NotReadyError("pbt_rank: every member needs at least one recorded return");
      f.push_back(std::accumulate(r.begin(), r.end(), 0.0) / static_cast<double>(r.size()));
    }
    return f;
  }
};

struct EvolvePlan {
  std::vector<std::size_t> replaced, donors;
};

// pbt_evolve_trainer (evolve.hpp:169-213) with the default priors; rng = (key, next) of the
// RngSequence the caller owns (rng.hpp:74-95)
inline std::optional<EvolvePlan> pbt_evolve_trainer(PBTState& st, Population& trainer,
                                                    std::uint64_t rng_key, std::uint64_t& rng_next) {
  const auto fit = st.fitness();
  std::vector<std::uint64_t> rep(fit.size()), don(fit.size());
  std::uint32_t cnt = 0;
  check(pbrl_pbt_evolve(trainer.handle(), fit.data(), rng_key, &rng_next, rep.data(), don.data(),
                        &cnt));
  if (cnt == 0) return std::nullopt;
  EvolvePlan plan;
  for (std::uint32_t i = 0; i < cnt; ++i) {
    plan.replaced.push_back(rep[i]);
    plan.donors.push_back(don[i]);
    st.returns[rep[i]].clear();
  }
  st.steps_since_evolve = 0;
  return plan;
}

}  // namespace pbrl::b200
