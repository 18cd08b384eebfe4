// pbrl_b200_pipeline.hpp -- the reference's threaded training orchestration (run_training,
// pipeline_run.hpp:77-468, with pipeline.hpp's queues / actor_loop / ingest and replay.hpp's
// RatioController) on top of the B200 population API.  Header-only C++17 over the C ABI
// (include/pbrl_b200.h) and its facade (include/pbrl_b200.hpp).
//
// What changes against the reference:
//   * the replay buffers are the device rings of the learner population: the ingest thread
//     moves transitions from the actor queues into them with batched H2D inserts
//     (pbrl_replay_insert), not one push per transition;
//   * there is no prefetch thread: sampling is part of the device update burst
//     (pbrl_update_k = sample_batch + update_k_steps on the device, draw ids as the reference's
//     prefetcher assigns them);
//   * actors act on the device through their own population handle, refreshed from a device
//     snapshot mailbox (pbrl_mailbox_publish / pbrl_actor_refresh) -- never a host copy of
//     the weights;
//   * every call on the learner handle (update bursts, inserts, publish, PBT) is serialised by
//     one mutex -- the C ABI's threading contract -- and is asynchronous on the device, so the
//     lock is held only while work is enqueued.
// The ratio guard (RatioController) and the bounded queues stay on the host, with the
// reference's semantics.  Environments are outside the B200 path: run_training takes any Env
// (a reset/step interface); PointMassEnv is a small built-in one for tests and demos.
#ifndef PBRL_B200_PIPELINE_HPP
#define PBRL_B200_PIPELINE_HPP

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pbrl_b200.hpp"

namespace pbrl::b200 {

// ---------------------------------------------------------------- RatioController
// replay.hpp:205-298: keeps update steps per environment step near `target` by blocking the
// side that runs ahead; await() bounds the wait; a closed controller always proceeds.
enum class RatioSide { kSample, kInsert };
enum class RatioDecision { kProceed, kBlock };

class RatioController {
 public:
  RatioController(double target, double slack, std::uint64_t warmup_env_steps)
      : target_(target), slack_(slack), warmup_(warmup_env_steps) {
    if (!(target > 0)) throw ConfigError("RatioController: target must be positive");
    if (slack < 0) throw ConfigError("RatioController: slack must be >= 0");
  }
  void on_env_steps(std::uint64_t k) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      env_ += k;
    }
    cv_.notify_all();
  }
  void on_update_steps(std::uint64_t k) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      upd_ += k;
    }
    cv_.notify_all();
  }
  std::uint64_t env_steps() const {
    std::lock_guard<std::mutex> lk(mu_);
    return env_;
  }
  std::uint64_t update_steps() const {
    std::lock_guard<std::mutex> lk(mu_);
    return upd_;
  }
  std::uint64_t warmup_env_steps() const { return warmup_; }
  RatioDecision check(RatioSide side, std::uint64_t pending = 1) const {
    std::lock_guard<std::mutex> lk(mu_);
    return check_locked(side, pending);
  }
  bool await(RatioSide side, std::chrono::milliseconds timeout, std::uint64_t pending = 1) {
    std::unique_lock<std::mutex> lk(mu_);
    return cv_.wait_for(lk, timeout, [&] {
      return closed_ || check_locked(side, pending) == RatioDecision::kProceed;
    });
  }
  void close() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      closed_ = true;
    }
    cv_.notify_all();
  }

 private:
  RatioDecision check_locked(RatioSide side, std::uint64_t pending) const {
    if (side == RatioSide::kSample) {
      if (env_ < std::max<std::uint64_t>(warmup_, 1)) return RatioDecision::kBlock;
      const double lhs = static_cast<double>(upd_ + pending);
      const double rhs = target_ * (1.0 + slack_) * static_cast<double>(std::max<std::uint64_t>(env_, 1));
      return lhs > rhs ? RatioDecision::kBlock : RatioDecision::kProceed;
    }
    const double lhs = static_cast<double>(env_ + pending);
    const double rhs = (static_cast<double>(upd_) / target_) * (1.0 + slack_) +
                       static_cast<double>(warmup_);
    return lhs > rhs ? RatioDecision::kBlock : RatioDecision::kProceed;
  }
  mutable std::mutex mu_;
  std::condition_variable cv_;
  double target_, slack_;
  std::uint64_t warmup_;
  std::uint64_t env_ = 0, upd_ = 0;
  bool closed_ = false;
};

// ---------------------------------------------------------------- BoundedQueue
// pipeline.hpp:89-148: every wait bounded; close() releases both sides.
template <typename Item>
class BoundedQueue {
 public:
  explicit BoundedQueue(std::size_t capacity) : cap_(std::max<std::size_t>(capacity, 1)) {}
  bool push(Item item, std::chrono::milliseconds timeout) {
    std::unique_lock<std::mutex> lk(mu_);
    if (!not_full_.wait_for(lk, timeout, [&] { return closed_ || q_.size() < cap_; })) return false;
    if (closed_) return false;
    q_.push_back(std::move(item));
    not_empty_.notify_one();
    return true;
  }
  bool pop(Item& out, std::chrono::milliseconds timeout) {
    std::unique_lock<std::mutex> lk(mu_);
    if (!not_empty_.wait_for(lk, timeout, [&] { return closed_ || !q_.empty(); })) return false;
    if (q_.empty()) return false;
    out = std::move(q_.front());
    q_.pop_front();
    not_full_.notify_one();
    return true;
  }
  void close() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      closed_ = true;
    }
    not_full_.notify_all();
    not_empty_.notify_all();
  }
  bool closed() const {
    std::lock_guard<std::mutex> lk(mu_);
    return closed_;
  }
  std::size_t size() const {
    std::lock_guard<std::mutex> lk(mu_);
    return q_.size();
  }
  std::size_t capacity() const { return cap_; }

 private:
  mutable std::mutex mu_;
  std::condition_variable not_full_, not_empty_;
  std::deque<Item> q_;
  std::size_t cap_;
  bool closed_ = false;
};

struct Transition {  // replay.hpp:17-29
  std::uint32_t member = 0;
  std::uint64_t seq = 0;
  std::vector<float> s, a, s2;
  float r = 0, done = 0;
};

struct EpisodeReport {  // pipeline.hpp:150-154
  std::size_t member = 0;
  double ep_return = 0;
  bool deterministic_eval = false;
};

class ReportSink {  // pipeline.hpp:156-170
 public:
  void push(EpisodeReport r) {
    std::lock_guard<std::mutex> lk(mu_);
    reports_.push_back(r);
  }
  std::vector<EpisodeReport> drain() {
    std::lock_guard<std::mutex> lk(mu_);
    std::vector<EpisodeReport> out;
    out.swap(reports_);
    return out;
  }

 private:
  std::mutex mu_;
  std::vector<EpisodeReport> reports_;
};

// ---------------------------------------------------------------- device snapshot mailbox
// SnapshotMailbox (pipeline.hpp:53-83) over pbrl_mailbox_*: publish from the learner thread,
// refresh into an actor's own population handle.
class SnapshotMailbox {
 public:
  explicit SnapshotMailbox(Population& learner) { check(pbrl_mailbox_create(learner.handle(), &mb_)); }
  ~SnapshotMailbox() {
    if (mb_) pbrl_mailbox_destroy(mb_);
  }
  SnapshotMailbox(const SnapshotMailbox&) = delete;
  SnapshotMailbox& operator=(const SnapshotMailbox&) = delete;
  std::uint64_t publish(Population& learner, const std::vector<double>& explore_std) {
    std::uint64_t v = 0;
    check(pbrl_mailbox_publish(mb_, learner.handle(),
                               explore_std.empty() ? nullptr : explore_std.data(), &v));
    return v;
  }
  std::uint64_t version() const {
    std::uint64_t v = 0;
    check(pbrl_mailbox_version(mb_, &v));
    return v;
  }
  // actor_loop's refresh(): the version the actor now holds (0 = nothing published yet)
  std::uint64_t refresh(Population& actor, std::vector<double>& explore_std) const {
    std::uint64_t v = 0;
    explore_std.resize(actor.members());
    check(pbrl_actor_refresh(actor.handle(), mb_, &v, explore_std.data()));
    return v;
  }

 private:
  pbrl_mailbox* mb_ = nullptr;
};

// ---------------------------------------------------------------- environments
// The reset / step interface of envs.hpp:41-49 as a class; one instance per member slot.
class Env {
 public:
  virtual ~Env() = default;
  virtual std::size_t observation_dim() const = 0;
  virtual std::size_t action_dim() const = 0;
  virtual double action_bound() const = 0;
  virtual std::size_t horizon() const = 0;
  virtual std::vector<double> reset(std::uint64_t seed) = 0;
  struct Step {
    std::vector<double> obs;
    double reward = 0;
    bool done = false;  // horizon reached (a timeout: bootstrapped by default)
  };
  virtual Step step(const std::vector<double>& action) = 0;
};

// A d-dimensional point mass driven toward the origin: obs = [position, velocity],
// action = acceleration in [-1, 1]^d, reward = -(|p|^2 + 0.1 |a|^2), fixed horizon.
class PointMassEnv final : public Env {
 public:
  explicit PointMassEnv(std::size_t dims = 2, std::size_t horizon = 100, double dt = 0.05)
      : d_(dims), h_(horizon), dt_(dt), p_(dims), v_(dims) {}
  std::size_t observation_dim() const override { return 2 * d_; }
  std::size_t action_dim() const override { return d_; }
  double action_bound() const override { return 1.0; }
  std::size_t horizon() const override { return h_; }
  std::vector<double> reset(std::uint64_t seed) override {
    t_ = 0;
    for (std::size_t i = 0; i < d_; ++i) {
      const std::uint64_t b = mix(mix(seed) ^ mix(i + 1));
      p_[i] = -1.0 + 2.0 * static_cast<double>(b >> 11) * 0x1.0p-53;
      v_[i] = 0.0;
    }
    return obs();
  }
  Step step(const std::vector<double>& a) override {
    Step s;
    double cost = 0;
    for (std::size_t i = 0; i < d_; ++i) {
      const double ai = std::clamp(a[i], -1.0, 1.0);
      v_[i] += ai * dt_;
      p_[i] += v_[i] * dt_;
      cost += p_[i] * p_[i] + 0.1 * ai * ai;
    }
    s.reward = -cost;
    s.done = ++t_ >= h_;
    s.obs = obs();
    return s;
  }

 private:
  static std::uint64_t mix(std::uint64_t x) {  // SplitMix64 finalizer
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  std::vector<double> obs() const {
    std::vector<double> o(p_);
    o.insert(o.end(), v_.begin(), v_.end());
    return o;
  }
  std::size_t d_, h_, t_ = 0;
  double dt_;
  std::vector<double> p_, v_;
};

// ---------------------------------------------------------------- configuration / summary
enum class Algo { kTd3, kSac };
enum class Strategy { kNone, kPbt, kCem, kDvd };

struct RunConfig {  // pipeline.hpp:176-244
  Algo algo = Algo::kTd3;
  PopMode mode = PopMode::kIndependent;
  Strategy strategy = Strategy::kNone;
  std::size_t population = 1;
  std::size_t updates_per_burst = 50;  // K
  std::size_t actor_workers = 1;
  std::function<std::unique_ptr<Env>()> make_env = [] { return std::make_unique<PointMassEnv>(); };
  BufferMode buffer_mode = BufferMode::kPerAgent;
  std::uint64_t seed = 0;
  std::size_t total_updates = 10000;
  std::size_t batch_size = 64;
  std::vector<std::size_t> hidden = {32, 32};
  std::size_t buffer_capacity = 10000;
  std::size_t warmup_per_buffer = 1000;
  double learning_rate = 3e-4;
  double discount = 0.99;
  double explore_std = 0.1;
  double target_noise_std = 0.2;
  double env_steps_per_member_per_update = 1.0;  // the ratio target
  double ratio_slack = 0.05;
  std::size_t eval_every_episodes = 3;  // 0 disables deterministic eval episodes
  bool bootstrap_timeouts = true;
  std::chrono::milliseconds starvation_timeout{30000};
  std::uint64_t pbt_interval = 2000;
  std::size_t cem_generation_updates = 500;  // update steps per generation
  double cem_init_var = 0.0;
  DvDConfig dvd;
  bool dvd_auto_probe = true;  // probe states from environment resets
  std::size_t dvd_probe_count = 16;
  std::size_t insert_block = 256;  // transitions per batched device insert
  Precision precision = Precision::kBf16;
  int device = 0;

  void validate() const {
    if (population < 1) throw ConfigError("RunConfig: population must be >= 1");
    if (updates_per_burst < 1) throw ConfigError("RunConfig: updates_per_burst must be >= 1");
    if (actor_workers < 1) throw ConfigError("RunConfig: actor_workers must be >= 1");
    if (batch_size < 1) throw ConfigError("RunConfig: batch_size must be >= 1");
    if (total_updates < 1) throw ConfigError("RunConfig: total_updates must be >= 1");
    if (!(env_steps_per_member_per_update > 0))
      throw ConfigError("RunConfig: env_steps_per_member_per_update must be positive");
    if (!make_env) throw ConfigError("RunConfig: make_env is required");
    if (strategy == Strategy::kCem || strategy == Strategy::kDvd) {
      if (mode != PopMode::kSharedCritic)
        throw ConfigError("RunConfig: CEM and DvD strategies require shared-critic mode");
      if (buffer_mode != BufferMode::kShared)
        throw ConfigError("RunConfig: CEM and DvD strategies require a shared buffer");
      if (strategy == Strategy::kCem && population % 2 != 0)
        throw ConfigError("RunConfig: CEM needs an even population");
      if (algo != Algo::kTd3)  // pipeline_run.hpp:81-83
        throw ConfigError("RunConfig: CEM and DvD strategies are TD3-only");
    }
    if (strategy == Strategy::kPbt && buffer_mode != BufferMode::kPerAgent)
      throw ConfigError("RunConfig: PBT tunes hyperparameters, so buffers must not be mixed");
  }
};

struct RunSummary {  // pipeline.hpp:246-262
  std::uint64_t env_steps = 0;
  std::uint64_t update_steps = 0;
  std::uint64_t dropped_transitions = 0;
  std::uint64_t evolve_events = 0;
  std::uint64_t published_versions = 0;
  std::uint64_t device_inserts = 0;  // batched pbrl_replay_insert calls
  double wall_seconds = 0;
  double updates_per_member_env_step = 0;
  std::vector<double> final_mean_returns;
  double best_return = 0;
  std::size_t best_member = 0;
  std::uint64_t eval_episodes = 0;
};

namespace detail {

// actor_loop (pipeline.hpp:255-365): act on the device through the actor's own population,
// step the member slots' environments, queue the training transitions, report episodes.
inline void actor_loop(const RunConfig& cfg, const std::vector<std::size_t>& members,
                       Population& actor, const SnapshotMailbox& mailbox,
                       BoundedQueue<Transition>& queue, ReportSink& reports,
                       const std::atomic<bool>& stop) {
  const std::size_t k = members.size(), n = actor.members();
  if (k == 0) return;
  struct Slot {
    std::unique_ptr<Env> env;
    std::vector<double> obs;
    double ep_return = 0;
    std::uint64_t env_steps = 0, episodes = 0, seq = 0;
    bool eval = false;
  };
  std::vector<Slot> slots(k);
  for (std::size_t i = 0; i < k; ++i) {
    slots[i].env = cfg.make_env();
    slots[i].obs = slots[i].env->reset(cfg.seed ^ (members[i] * 2654435761ull));
  }
  const std::size_t ds = slots[0].env->observation_dim(), da = slots[0].env->action_dim();
  std::vector<double> explore;
  while (mailbox.refresh(actor, explore) == 0) {
    if (stop.load() || queue.closed()) return;
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  std::vector<float> obs(n * ds, 0.0f), act(n * da);
  std::vector<std::uint64_t> steps(n, 0);
  std::vector<double> noise(n, 0.0);
  while (!stop.load() && !queue.closed()) {
    mailbox.refresh(actor, explore);  // version-change check every step
    for (std::size_t i = 0; i < k; ++i) {
      const std::size_t m = members[i];
      for (std::size_t d = 0; d < ds; ++d) obs[m * ds + d] = static_cast<float>(slots[i].obs[d]);
      steps[m] = slots[i].env_steps;
      noise[m] = slots[i].eval ? 0.0 : explore[m];
    }
    if (cfg.algo == Algo::kTd3) {
      check(pbrl_act(actor.handle(), obs.data(), 1, noise.data(), cfg.seed, steps.data(), 0,
                     act.data()));
    } else {
      check(pbrl_act(actor.handle(), obs.data(), 1, nullptr, cfg.seed, steps.data(), 0,
                     act.data()));
    }
    for (std::size_t i = 0; i < k; ++i) {
      Slot& sl = slots[i];
      const std::size_t m = members[i];
      std::vector<double> a(da);
      for (std::size_t d = 0; d < da; ++d) a[d] = act[m * da + d];
      Transition tr;
      tr.member = static_cast<std::uint32_t>(m);
      tr.seq = sl.seq++;
      tr.s.assign(sl.obs.begin(), sl.obs.end());
      tr.a.assign(a.begin(), a.end());
      Env::Step res = sl.env->step(a);
      sl.ep_return += res.reward;
      sl.env_steps += 1;
      tr.r = static_cast<float>(res.reward);
      tr.done = (res.done && !cfg.bootstrap_timeouts) ? 1.0f : 0.0f;
      tr.s2.assign(res.obs.begin(), res.obs.end());
      sl.obs = std::move(res.obs);
      if (!sl.eval) {  // eval episodes are score-only
        while (!queue.push(tr, std::chrono::milliseconds(50)))
          if (stop.load() || queue.closed()) return;
      }
      if (res.done) {
        reports.push({m, sl.ep_return, sl.eval});
        sl.episodes += 1;
        sl.ep_return = 0;
        sl.eval = cfg.eval_every_episodes > 0 &&
                  sl.episodes % cfg.eval_every_episodes == cfg.eval_every_episodes - 1;
        sl.obs = sl.env->reset(cfg.seed ^ (m * 2654435761ull) ^ (sl.episodes * 1099511628211ull));
        mailbox.refresh(actor, explore);  // episode-boundary refresh
      }
    }
  }
}

}  // namespace detail

// run_training (pipeline_run.hpp:77-468): TD3 / SAC, independent or shared critic, with PBT,
// CEM (pipeline_run.hpp:143-162, :388-409) or DvD (:164-181, :343-347).
inline RunSummary run_training(const RunConfig& cfg) {
  cfg.validate();
  const std::size_t n = cfg.population;
  auto probe = cfg.make_env();
  const std::size_t ds = probe->observation_dim(), da = probe->action_dim();
  const double bound = probe->action_bound();
  const std::size_t horizon = probe->horizon();
  probe.reset();
  const auto t0 = std::chrono::steady_clock::now();
  auto wall = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  const int algo = cfg.algo == Algo::kTd3 ? PBRL_ALGO_TD3 : PBRL_ALGO_SAC;
  Population learner(algo, n, ds, da, cfg.hidden, bound, cfg.seed, cfg.precision, cfg.device, 0,
                     0, cfg.mode);
  std::mutex learner_mu;  // the C ABI's one-caller-per-handle contract

  // hypers (pipeline_run.hpp:94-125)
  Td3Hyper th = Td3Hyper::defaults(n);
  SacHyper sh = SacHyper::defaults(n, da);
  th.critic_lr.assign(n, cfg.learning_rate);
  th.policy_lr.assign(n, cfg.learning_rate);
  th.gamma.assign(n, cfg.discount);
  th.explore_std.assign(n, cfg.explore_std);
  th.target_std.assign(n, cfg.target_noise_std);
  sh.critic_lr.assign(n, cfg.learning_rate);
  sh.policy_lr.assign(n, cfg.learning_rate);
  sh.alpha_lr.assign(n, cfg.learning_rate);
  sh.gamma.assign(n, cfg.discount);
  auto upload_hyper = [&] {
    auto put = [&](const char* f, const std::vector<double>& v) {
      check(pbrl_set_hyper(learner.handle(), f, v.data()));
    };
    if (algo == PBRL_ALGO_TD3)
      for (auto& [name, vec] : th.fields()) put(name, *vec);
    else
      for (auto& [name, vec] : sh.fields()) put(name, *vec);
  };
  upload_hyper();
  auto explore_vec = [&]() -> std::vector<double> {
    if (algo != PBRL_ALGO_TD3) return std::vector<double>(n, 0.0);
    std::vector<double> v(n);
    check(pbrl_get_hyper(learner.handle(), "explore_std", v.data()));
    return v;
  };

  // device replay rings in the learner population
  const std::size_t nbuf = cfg.buffer_mode == BufferMode::kPerAgent ? n : 1;
  check(pbrl_replay_create(learner.handle(), cfg.buffer_capacity, static_cast<int>(cfg.buffer_mode)));

  const std::size_t workers = std::min(cfg.actor_workers, n);
  const std::size_t queue_cap = (4 * cfg.updates_per_burst * n + workers - 1) / workers;
  std::vector<std::unique_ptr<BoundedQueue<Transition>>> queues;
  for (std::size_t w = 0; w < workers; ++w)
    queues.push_back(std::make_unique<BoundedQueue<Transition>>(queue_cap));
  const double per_member_ratio = cfg.env_steps_per_member_per_update;
  RatioController ctrl(1.0 / (static_cast<double>(n) * per_member_ratio), cfg.ratio_slack,
                       cfg.warmup_per_buffer * nbuf);
  SnapshotMailbox mailbox(learner);
  ReportSink reports;
  std::atomic<bool> stop{false};
  std::atomic<std::uint64_t> dropped{0}, inserts{0}, published{0};
  PBTState pbt(n);
  pbt.evolve_interval = cfg.pbt_interval;
  std::uint64_t pbt_key = 0, pbt_next = 0;
  {  // RngSequence(seed, 0, kDonorChoice, 0) (pipeline_run.hpp:129)
    auto mix = [](std::uint64_t x) {
      x += 0x9E3779B97F4A7C15ull;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
      return x ^ (x >> 31);
    };
    pbt_key = mix(mix(mix(mix(cfg.seed) ^ 0) ^ 8) ^ 0);
  }
  auto mix64 = [](std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  };
  auto stream_key = [&](std::uint64_t seed, std::uint64_t stream, std::uint64_t use,
                        std::uint64_t step) {
    return mix64(mix64(mix64(mix64(seed) ^ stream) ^ use) ^ step);
  };

  // CEM (pipeline_run.hpp:143-162): the distribution around flatten_member(policy, 0), every
  // generation drawn into the policies from RngSequence(seed, 2, kCemDraw, generation)
  std::unique_ptr<CEMState> cem;
  std::vector<std::vector<double>> cem_gen_returns(n);
  std::size_t cem_gen_done = 0;
  std::uint64_t cem_generation = 0;
  std::vector<std::uint8_t> cem_train_mask;
  auto cem_resample = [&] {
    std::uint64_t next = 0;
    cem_resample_into(*cem, stream_key(cfg.seed, 2, 10, cem_generation++), &next);
    for (auto& r : cem_gen_returns) r.clear();
  };
  if (cfg.strategy == Strategy::kCem) cem = std::make_unique<CEMState>(learner, nullptr, cfg.cem_init_var);

  // DvD (pipeline_run.hpp:164-181): probe states from environment resets, the length scale the
  // median pairwise distance of the initial embeddings (frozen for the run)
  DvDConfig dvd = cfg.dvd;
  if (cfg.strategy == Strategy::kDvd) {
    if (cfg.dvd_auto_probe) {
      dvd.m_states = std::max(cfg.dvd_probe_count, n);
      dvd.probe_states.clear();
      auto env = cfg.make_env();
      for (std::size_t i = 0; i < dvd.m_states; ++i) {
        const std::vector<double> obs = env->reset(mix64(cfg.seed ^ 0x9E0B0E5ull) + i);
        dvd.probe_states.insert(dvd.probe_states.end(), obs.begin(), obs.end());
      }
    }
    const std::vector<float> emb = dvd_embed(learner, dvd.probe_states, dvd.m_states);
    dvd.length_scale = median_pairwise_distance(std::vector<double>(emb.begin(), emb.end()), n);
    dvd.validate(n);
  }
  if (cfg.strategy == Strategy::kCem) {  // :322-327
    cem_train_mask.assign(n, 0);
    for (std::size_t m = 0; m < n / 2; ++m) cem_train_mask[m] = 1;
    cem_resample();
  }
  {
    std::lock_guard<std::mutex> lk(learner_mu);
    mailbox.publish(learner, explore_vec());
    published += 1;
  }

  // actors: one device population per worker (the learner's shapes, precision and member ids)
  std::vector<std::unique_ptr<Population>> actor_pops;
  for (std::size_t w = 0; w < workers; ++w)
    actor_pops.push_back(std::make_unique<Population>(algo, n, ds, da, cfg.hidden, bound,
                                                      cfg.seed, cfg.precision, cfg.device));
  std::vector<std::thread> actor_threads;
  for (std::size_t w = 0; w < workers; ++w) {
    std::vector<std::size_t> assigned;
    for (std::size_t m = w; m < n; m += workers) assigned.push_back(m);
    actor_threads.emplace_back([&, w, assigned] {
      detail::actor_loop(cfg, assigned, *actor_pops[w], mailbox, *queues[w], reports, stop);
    });
  }

  // ingest (pipeline.hpp:440-490): validate, ratio gate after warm-up, batched device inserts
  std::thread ingest_thread([&] {
    std::vector<float> s, a, r, s2, d;
    std::vector<std::uint32_t> mem;
    std::vector<std::size_t> fill(nbuf, 0);
    bool warming = cfg.warmup_per_buffer > 0;
    auto flush = [&] {
      if (mem.empty()) return;
      {
        std::lock_guard<std::mutex> lk(learner_mu);
        check(pbrl_replay_insert(learner.handle(), s.data(), a.data(), r.data(), s2.data(),
                                 d.data(), mem.data(), mem.size()));
      }
      inserts += 1;
      if (!stop.load()) ctrl.on_env_steps(mem.size());  // the shutdown drain keeps the data only
      s.clear(), a.clear(), r.clear(), s2.clear(), d.clear(), mem.clear();
    };
    bool all_closed = false;
    while (!all_closed) {
      all_closed = true;
      bool drained = false;
      for (auto& q : queues) {
        Transition tr;
        while (q->pop(tr, std::chrono::milliseconds(0))) {
          drained = true;
          bool ok = tr.s.size() == ds && tr.a.size() == da && tr.s2.size() == ds;
          auto finite = [](const std::vector<float>& v) {
            for (float x : v)
              if (!std::isfinite(x)) return false;
            return true;
          };
          ok = ok && finite(tr.s) && finite(tr.a) && finite(tr.s2) && std::isfinite(tr.r) &&
               (tr.done == 0.0f || tr.done == 1.0f);
          if (!ok) {
            dropped += 1;
            continue;
          }
          if (warming) warming = *std::min_element(fill.begin(), fill.end()) < cfg.warmup_per_buffer;
          if (!warming) {
            // the gate admits the staged block plus this transition; when it blocks, what is
            // staged goes to the device first (it counts as environment steps only then)
            while (!stop.load() && !ctrl.await(RatioSide::kInsert, std::chrono::milliseconds(50),
                                               mem.size() + 1))
              flush();
          }
          s.insert(s.end(), tr.s.begin(), tr.s.end());
          a.insert(a.end(), tr.a.begin(), tr.a.end());
          s2.insert(s2.end(), tr.s2.begin(), tr.s2.end());
          r.push_back(tr.r);
          d.push_back(tr.done);
          mem.push_back(tr.member);
          fill[cfg.buffer_mode == BufferMode::kPerAgent ? tr.member : 0] += 1;
          if (mem.size() >= cfg.insert_block) flush();
        }
        if (!q->closed() || q->size() > 0) all_closed = false;
      }
      if (!drained) flush();
      if (stop.load() && !drained) break;
      if (!drained) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    flush();
  });

  // learner loop (pipeline_run.hpp:330-410): device sample + K updates per burst
  RunSummary summary;
  std::uint64_t done_updates = 0, draw_id = 0;
  std::string abort_reason;
  auto handle_reports = [&] {
    for (const EpisodeReport& r : reports.drain()) {
      if (r.deterministic_eval) {
        summary.eval_episodes += 1;
      } else {
        pbt.record_return(r.member, r.ep_return);
        if (cfg.strategy == Strategy::kCem) cem_gen_returns[r.member].push_back(r.ep_return);
      }
    }
  };
  try {
    while (done_updates < cfg.total_updates && !stop.load()) {
      const std::size_t k_next = std::min(cfg.updates_per_burst, cfg.total_updates - done_updates);
      auto waited = std::chrono::milliseconds(0);
      bool ready = false;
      while (!stop.load()) {
        if (ctrl.await(RatioSide::kSample, std::chrono::milliseconds(100), k_next)) {
          int ok = 0;
          {
            std::lock_guard<std::mutex> lk(learner_mu);
            // DvD: dvd_policy_hook(dvd, done_updates) for this burst (:343-347)
            std::optional<detail::HookScope> hook;
            PolicyGradHook hk;
            if (cfg.strategy == Strategy::kDvd) {
              hk = dvd_policy_hook(dvd, done_updates);
              hook.emplace(learner.handle(), &hk, ds);
            }
            check(pbrl_update_k_masked(learner.handle(), static_cast<std::uint32_t>(k_next),
                                       cfg.seed, draw_id, cfg.batch_size, cfg.warmup_per_buffer,
                                       cem_train_mask.empty() ? nullptr : cem_train_mask.data(),
                                       &ok));
          }
          if (ok) {
            ready = true;
            break;
          }
          std::this_thread::sleep_for(std::chrono::milliseconds(2));  // rings not warm yet
          waited += std::chrono::milliseconds(2);
        } else {
          waited += std::chrono::milliseconds(100);
        }
        if (waited >= cfg.starvation_timeout) {
          abort_reason = "actors starved the learner: ratio guard held past timeout";
          break;
        }
      }
      if (!ready) break;
      draw_id += k_next;
      done_updates += k_next;
      ctrl.on_update_steps(k_next);
      {
        std::lock_guard<std::mutex> lk(learner_mu);
        mailbox.publish(learner, explore_vec());
        published += 1;
      }
      handle_reports();
      if (cfg.strategy == Strategy::kPbt) {
        pbt.steps_since_evolve += k_next;
        bool scored = true;
        for (const auto& q : pbt.returns) scored = scored && !q.empty();
        if (std::getenv("PBRL_PIPELINE_DEBUG"))
          std::fprintf(stderr, "burst done=%llu since=%llu scored=%d\n",
                       (unsigned long long)done_updates,
                       (unsigned long long)pbt.steps_since_evolve, (int)scored);
        if (pbt.steps_since_evolve >= pbt.evolve_interval && scored) {
          std::lock_guard<std::mutex> lk(learner_mu);
          auto plan = pbt_evolve_trainer(pbt, learner, pbt_key, pbt_next);
          if (plan) {
            summary.evolve_events += 1;
            mailbox.publish(learner, explore_vec());
            published += 1;
          }
        }
      }
      if (cfg.strategy == Strategy::kCem) {  // :388-409
        cem_gen_done += k_next;
        if (cem_gen_done >= cfg.cem_generation_updates) {
          bool all_scored = true;
          for (const auto& r : cem_gen_returns) all_scored = all_scored && !r.empty();
          if (all_scored) {  // otherwise the generation extends by another burst
            std::vector<double> scores(n);
            for (std::size_t m = 0; m < n; ++m) {
              double acc = 0;
              for (double v : cem_gen_returns[m]) acc += v;
              scores[m] = acc / static_cast<double>(cem_gen_returns[m].size());
            }
            std::lock_guard<std::mutex> lk(learner_mu);
            cem_update(*cem, scores);
            cem_resample();
            mailbox.publish(learner, explore_vec());
            published += 1;
            summary.evolve_events += 1;
            cem_gen_done = 0;
          }
        }
      }
    }
  } catch (...) {
    stop.store(true);
    ctrl.close();
    for (auto& q : queues) q->close();
    for (auto& t : actor_threads) t.join();
    ingest_thread.join();
    throw;
  }

  // shutdown (pipeline_run.hpp:412-420)
  stop.store(true);
  ctrl.close();
  for (auto& q : queues) q->close();
  for (auto& t : actor_threads) t.join();
  ingest_thread.join();
  check(pbrl_synchronize(learner.handle()));
  handle_reports();
  if (!abort_reason.empty()) throw DataStarvationError("run_training: " + abort_reason);

  summary.env_steps = ctrl.env_steps();
  summary.update_steps = done_updates;
  summary.dropped_transitions = dropped.load();
  summary.device_inserts = inserts.load();
  summary.published_versions = published.load();
  summary.wall_seconds = wall();
  const double warm = static_cast<double>(ctrl.warmup_env_steps());
  if (static_cast<double>(summary.env_steps) > warm) {
    const double per_member = (static_cast<double>(summary.env_steps) - warm) / static_cast<double>(n);
    summary.updates_per_member_env_step =
        per_member > 0 ? static_cast<double>(summary.update_steps) * per_member_ratio / per_member
                       : 0.0;
  }
  summary.final_mean_returns.assign(n, -std::numeric_limits<double>::infinity());
  for (std::size_t m = 0; m < n; ++m) {
    const auto& q = pbt.returns[m];
    if (!q.empty()) {
      double acc = 0;
      for (double v : q) acc += v;
      summary.final_mean_returns[m] = acc / static_cast<double>(q.size());
    }
  }
  summary.best_member = 0;
  summary.best_return = summary.final_mean_returns[0];
  for (std::size_t m = 1; m < n; ++m) {
    if (summary.final_mean_returns[m] > summary.best_return) {
      summary.best_return = summary.final_mean_returns[m];
      summary.best_member = m;
    }
  }
  (void)horizon;
  return summary;
}

}  // namespace pbrl::b200

#endif  // PBRL_B200_PIPELINE_HPP
