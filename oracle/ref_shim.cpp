// Test infrastructure only: a thin extern "C" shim over the UNMODIFIED reference
// library (/root/reference/proj/core), compiled by oracle/Makefile into
// oracle/_ref/libpbrl_ref.so.  Nothing in the product links this file; tests,
// the golden-vector generator and bench.py's CPU-baseline / reference arm load
// it with ctypes to (a) pin the C restatement in oracle/pbrl_oracle.c and
// (b) time the reference CPU path on the host cores.
//
// Every entry point calls reference functions directly:
//   make_td3_state / td3_update_step / td3_critic_target / mse_loss_grads /
//   td3_policy_loss_grads            algos.hpp:181, :351, :241, :288, :318
//   make_sac_state / sac_update_step algos.hpp:490, :781
//   make_synthetic_batches           bench.hpp:69
//   ReplayBuffer / sample_batch      replay.hpp:28, :181
//   pbt_rank / pbt_plan / pbt_evolve_trainer   evolve.hpp:112, :133, :169, :192
//   bench_update                     bench.hpp:137
#include <cstring>
#include <fstream>
#include <memory>
#include <optional>
#include <vector>

#include "pbrl/algos.hpp"
#include "pbrl/bench.hpp"
#include "pbrl/evolve.hpp"
#include "pbrl/replay.hpp"

using namespace pbrl;

namespace {

template <typename T>
PopMLPParams<T>& td3_net(Td3State<T>& st, int net) {
  switch (net) {
    case 0: return st.policy;
    case 1: return st.policy_target;
    case 2: return st.critic1;
    case 3: return st.critic2;
    case 4: return st.critic1_target;
    default: return st.critic2_target;
  }
}

template <typename T>
MlpAdam<T>& td3_opt(Td3State<T>& st, int net) {
  if (net == 0) return st.opt_policy;
  if (net == 2) return st.opt_critic1;
  return st.opt_critic2;
}

template <typename T>
PopMLPParams<T>& sac_net(SacState<T>& st, int net) {
  switch (net) {
    case 0: return st.policy;
    case 2: return st.critic1;
    case 3: return st.critic2;
    case 4: return st.critic1_target;
    default: return st.critic2_target;
  }
}

template <typename T>
MlpAdam<T>& sac_opt(SacState<T>& st, int net) {
  if (net == 0) return st.opt_policy;
  if (net == 2) return st.opt_critic1;
  return st.opt_critic2;
}

std::vector<std::size_t> to_dims(const std::uint64_t* h, std::uint32_t nh) {
  return std::vector<std::size_t>(h, h + nh);
}

template <typename T>
PopTensor<T> tensor_from(const T* p, std::size_t n, std::size_t rows, std::size_t cols) {
  PopTensor<T> t = PopTensor<T>::zeros({n, rows, cols});
  std::memcpy(t.data.data(), p, t.data.size() * sizeof(T));
  return t;
}

template <typename T>
TransitionBatch<T> batch_from(const T* s, const T* a, const T* r, const T* s2, const T* d,
                              std::size_t n, std::size_t b, std::size_t ds, std::size_t da) {
  TransitionBatch<T> out;
  out.s = tensor_from(s, n, b, ds);
  out.a = tensor_from(a, n, b, da);
  out.r = tensor_from(r, n, b, 1);
  out.s2 = tensor_from(s2, n, b, ds);
  out.done = tensor_from(d, n, b, 1);
  return out;
}

Td3Hyper td3_hyper_from(const double* h, std::size_t n) {
  // field order: critic_lr, policy_lr, policy_delay_ratio, explore_std,
  //              target_std, target_clip, gamma, tau
  Td3Hyper hy;
  std::vector<double>* f[8] = {&hy.critic_lr,  &hy.policy_lr,   &hy.policy_delay_ratio,
                               &hy.explore_std, &hy.target_std, &hy.target_clip,
                               &hy.gamma,       &hy.tau};
  for (int i = 0; i < 8; ++i) f[i]->assign(h + i * n, h + (i + 1) * n);
  return hy;
}

void td3_hyper_to(const Td3Hyper& hy, double* h) {
  const std::vector<double>* f[8] = {&hy.critic_lr,  &hy.policy_lr,   &hy.policy_delay_ratio,
                                     &hy.explore_std, &hy.target_std, &hy.target_clip,
                                     &hy.gamma,       &hy.tau};
  const std::size_t n = hy.critic_lr.size();
  for (int i = 0; i < 8; ++i) std::memcpy(h + i * n, f[i]->data(), n * sizeof(double));
}

SacHyper sac_hyper_from(const double* h, std::size_t n) {
  // field order: policy_lr, critic_lr, alpha_lr, target_entropy, reward_scale, gamma, tau
  SacHyper hy;
  std::vector<double>* f[7] = {&hy.policy_lr,      &hy.critic_lr,    &hy.alpha_lr,
                               &hy.target_entropy, &hy.reward_scale, &hy.gamma,
                               &hy.tau};
  for (int i = 0; i < 7; ++i) f[i]->assign(h + i * n, h + (i + 1) * n);
  return hy;
}

void sac_hyper_to(const SacHyper& hy, double* h) {
  const std::vector<double>* f[7] = {&hy.policy_lr,      &hy.critic_lr,    &hy.alpha_lr,
                                     &hy.target_entropy, &hy.reward_scale, &hy.gamma,
                                     &hy.tau};
  const std::size_t n = hy.policy_lr.size();
  for (int i = 0; i < 7; ++i) std::memcpy(h + i * n, f[i]->data(), n * sizeof(double));
}

PBTState pbt_from(const double* rings, const std::uint32_t* counts, std::size_t n,
                  std::size_t ring_cap) {
  PBTState st(n);
  for (std::size_t m = 0; m < n; ++m) {
    for (std::uint32_t j = 0; j < counts[m]; ++j) st.record_return(m, rings[m * ring_cap + j]);
  }
  return st;
}

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return -1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return -2;
  } catch (const UsageError& e) {
    g_err = e.what();
    return -3;
  } catch (const NotReadyError& e) {
    g_err = e.what();
    return -4;
  } catch (const ResourceError& e) {
    g_err = e.what();
    return -5;
  } catch (const DataStarvationError& e) {
    g_err = e.what();
    return -6;
  } catch (const DegeneratePopulationError& e) {
    g_err = e.what();
    return -10;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -9;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_mix64(std::uint64_t x) { return mix64(x); }
std::uint64_t ref_stream_key(std::uint64_t seed, std::uint64_t stream, std::uint64_t use,
                             std::uint64_t step) {
  return RngStream::of(seed, stream, static_cast<RngUse>(use), step).key;
}
double ref_normal_pair(std::uint64_t key, std::uint64_t c) { return RngStream{key}.normal_pair(c); }
double ref_uniform(std::uint64_t key, std::uint64_t c) { return RngStream{key}.uniform(c); }
float ref_tanhf(float x) { return std::tanh(x); }

// ---------------------------------------------------------------- TD3 (float and double)
#define PBRL_REF_TD3(SUFFIX, T)                                                                  \
  void* ref_td3##SUFFIX##_create(std::uint64_t n, std::uint64_t ds, std::uint64_t da,            \
                                 const std::uint64_t* hidden, std::uint32_t nh, double bound,    \
                                 std::uint64_t seed) {                                           \
    return new Td3State<T>(                                                                      \
        make_td3_state<T>(n, ds, da, to_dims(hidden, nh), static_cast<T>(bound), seed));         \
  }                                                                                              \
  void* ref_td3##SUFFIX##_create_mode(std::uint64_t n, std::uint64_t ds, std::uint64_t da,       \
                                      const std::uint64_t* hidden, std::uint32_t nh,             \
                                      double bound, std::uint64_t seed, int shared) {            \
    return new Td3State<T>(make_td3_state<T>(                                                    \
        n, ds, da, to_dims(hidden, nh), static_cast<T>(bound), seed,                             \
        shared ? PopMode::kSharedCritic : PopMode::kIndependent));                               \
  }                                                                                              \
  /* td3_update_step with dvd_policy_hook(cfg, step) (evolve.hpp:507-525) */                     \
  int ref_td3##SUFFIX##_step_dvd(void* h, const T* s, const T* a, const T* r, const T* s2,       \
                                 const T* d, std::uint64_t b, const double* hyper,               \
                                 const char* policy_mask, const double* probe,                   \
                                 std::uint64_t m_states, double length_scale, double jitter,     \
                                 double lam_start, double lam_end, std::uint64_t horizon,        \
                                 std::uint64_t step) {                                           \
    return guarded([&] {                                                                         \
      auto& st = *static_cast<Td3State<T>*>(h);                                                  \
      const std::size_t n = st.members();                                                        \
      auto batch = batch_from(s, a, r, s2, d, n, b, st.obs_dim, st.act_dim);                     \
      auto hy = td3_hyper_from(hyper, n);                                                        \
      DvDConfig cfg;                                                                             \
      cfg.probe_states.assign(probe, probe + m_states * st.obs_dim);                             \
      cfg.m_states = m_states;                                                                   \
      cfg.length_scale = length_scale;                                                           \
      cfg.jitter = jitter;                                                                       \
      cfg.schedule = LambdaSchedule{lam_start, lam_end, horizon};                                \
      PolicyGradHook<T> hook = dvd_policy_hook<T>(cfg, step);                                    \
      std::vector<char> mask;                                                                    \
      if (policy_mask) mask.assign(policy_mask, policy_mask + n);                                \
      td3_update_step<T>(st, batch, hy, &hook, policy_mask ? &mask : nullptr);                   \
    });                                                                                          \
  }                                                                                              \
  void ref_td3##SUFFIX##_dvd_embed(void* h, const double* probe, std::uint64_t m_states,         \
                                   T* out) {                                                     \
    auto& st = *static_cast<Td3State<T>*>(h);                                                    \
    std::vector<T> pr(probe, probe + m_states * st.obs_dim);                                     \
    auto e = dvd_embed(st.policy, pr, m_states);                                                 \
    std::memcpy(out, e.data.data(), e.data.size() * sizeof(T));                                  \
  }                                                                                              \
  void ref_td3##SUFFIX##_destroy(void* h) { delete static_cast<Td3State<T>*>(h); }               \
  void* ref_td3##SUFFIX##_clone(void* h) {                                                       \
    return new Td3State<T>(*static_cast<Td3State<T>*>(h));                                       \
  }                                                                                              \
  std::uint64_t ref_td3##SUFFIX##_param_count(void* h, int net) {                                \
    return td3_net(*static_cast<Td3State<T>*>(h), net).params_per_member();                      \
  }                                                                                              \
  void ref_td3##SUFFIX##_get_net(void* h, int net, std::uint64_t m, T* out) {                    \
    auto v = flatten_member(td3_net(*static_cast<Td3State<T>*>(h), net), m);                     \
    std::memcpy(out, v.data(), v.size() * sizeof(T));                                            \
  }                                                                                              \
  void ref_td3##SUFFIX##_set_net(void* h, int net, std::uint64_t m, const T* in) {               \
    auto& p = td3_net(*static_cast<Td3State<T>*>(h), net);                                       \
    unflatten_member(p, m, std::span<const T>(in, p.params_per_member()));                       \
  }                                                                                              \
  void ref_td3##SUFFIX##_get_adam(void* h, int net, std::uint64_t m, T* mo, T* vo,               \
                                  std::int64_t* t) {                                             \
    auto& opt = td3_opt(*static_cast<Td3State<T>*>(h), net);                                     \
    std::size_t at = 0;                                                                          \
    for (std::size_t l = 0; l < opt.w.size(); ++l) {                                             \
      for (auto* st : {&opt.w[l], &opt.b[l]}) {                                                  \
        const std::size_t s = st->m.member_stride();                                             \
        std::memcpy(mo + at, st->m.member_ptr(m), s * sizeof(T));                                \
        std::memcpy(vo + at, st->v.member_ptr(m), s * sizeof(T));                                \
        at += s;                                                                                 \
      }                                                                                          \
    }                                                                                            \
    *t = opt.w[0].t[m];                                                                          \
  }                                                                                              \
  void ref_td3##SUFFIX##_get_counters(void* h, double* delay_acc, std::uint64_t* steps) {        \
    auto& st = *static_cast<Td3State<T>*>(h);                                                    \
    std::memcpy(delay_acc, st.delay_acc.data(), st.delay_acc.size() * sizeof(double));           \
    std::memcpy(steps, st.steps.data(), st.steps.size() * sizeof(std::uint64_t));                \
  }                                                                                              \
  int ref_td3##SUFFIX##_step(void* h, const T* s, const T* a, const T* r, const T* s2,           \
                             const T* d, std::uint64_t b, const double* hyper,                   \
                             const char* policy_mask) {                                          \
    return guarded([&] {                                                                         \
      auto& st = *static_cast<Td3State<T>*>(h);                                                  \
      const std::size_t n = st.members();                                                        \
      auto batch = batch_from(s, a, r, s2, d, n, b, st.obs_dim, st.act_dim);                     \
      auto hy = td3_hyper_from(hyper, n);                                                        \
      if (policy_mask) {                                                                         \
        std::vector<char> mask(policy_mask, policy_mask + n);                                    \
        td3_update_step<T>(st, batch, hy, nullptr, &mask);                                          \
      } else {                                                                                   \
        td3_update_step(st, batch, hy);                                                          \
      }                                                                                          \
    });                                                                                          \
  }                                                                                              \
  /* losses of the step about to run, from the reference loss functions on the same state */    \
  int ref_td3##SUFFIX##_losses(void* h, const T* s, const T* a, const T* r, const T* s2,         \
                               const T* d, std::uint64_t b, const double* hyper, double* out3) { \
    return guarded([&] {                                                                         \
      Td3State<T> st = *static_cast<Td3State<T>*>(h);                                            \
      const std::size_t n = st.members();                                                        \
      auto batch = batch_from(s, a, r, s2, d, n, b, st.obs_dim, st.act_dim);                     \
      auto hy = td3_hyper_from(hyper, n);                                                        \
      auto y = td3_critic_target(batch, st.policy_target, st.critic1_target, st.critic2_target,  \
                                 hy, st.seed, st.streams, st.steps);                             \
      auto sa = concat_features(batch.s, batch.a);                                               \
      auto [l1, g1] = mse_loss_grads(st.critic1, sa, y);                                         \
      st.opt_critic1.step(st.critic1, g1, hy.critic_lr);                                         \
      auto [l2, g2] = mse_loss_grads(st.critic2, sa, y);                                         \
      auto [lp, gp] = td3_policy_loss_grads(st.policy, st.critic1, batch.s);                     \
      out3[0] = l1;                                                                              \
      out3[1] = l2;                                                                              \
      out3[2] = lp;                                                                              \
    });                                                                                          \
  }                                                                                              \
  int ref_td3##SUFFIX##_target(void* h, const T* s, const T* a, const T* r, const T* s2,         \
                               const T* d, std::uint64_t b, const double* hyper, T* y_out) {     \
    return guarded([&] {                                                                         \
      auto& st = *static_cast<Td3State<T>*>(h);                                                  \
      const std::size_t n = st.members();                                                        \
      auto batch = batch_from(s, a, r, s2, d, n, b, st.obs_dim, st.act_dim);                     \
      auto hy = td3_hyper_from(hyper, n);                                                        \
      auto y = td3_critic_target(batch, st.policy_target, st.critic1_target, st.critic2_target,  \
                                 hy, st.seed, st.streams, st.steps);                             \
      std::memcpy(y_out, y.data.data(), y.data.size() * sizeof(T));                             \
    });                                                                                          \
  }

PBRL_REF_TD3(f, float)
PBRL_REF_TD3(d, double)

// ---------------------------------------------------------------- SAC
#define PBRL_REF_SAC(SUFFIX, T)                                                                  \
  void* ref_sac##SUFFIX##_create(std::uint64_t n, std::uint64_t ds, std::uint64_t da,            \
                                 const std::uint64_t* hidden, std::uint32_t nh, double bound,    \
                                 std::uint64_t seed) {                                           \
    return new SacState<T>(                                                                      \
        make_sac_state<T>(n, ds, da, to_dims(hidden, nh), static_cast<T>(bound), seed));         \
  }                                                                                              \
  void* ref_sac##SUFFIX##_create_mode(std::uint64_t n, std::uint64_t ds, std::uint64_t da,       \
                                      const std::uint64_t* hidden, std::uint32_t nh,             \
                                      double bound, std::uint64_t seed, int shared) {            \
    return new SacState<T>(make_sac_state<T>(                                                    \
        n, ds, da, to_dims(hidden, nh), static_cast<T>(bound), seed,                             \
        shared ? PopMode::kSharedCritic : PopMode::kIndependent));                               \
  }                                                                                              \
  void ref_sac##SUFFIX##_destroy(void* h) { delete static_cast<SacState<T>*>(h); }               \
  std::uint64_t ref_sac##SUFFIX##_param_count(void* h, int net) {                                \
    return sac_net(*static_cast<SacState<T>*>(h), net).params_per_member();                      \
  }                                                                                              \
  void ref_sac##SUFFIX##_get_net(void* h, int net, std::uint64_t m, T* out) {                    \
    auto v = flatten_member(sac_net(*static_cast<SacState<T>*>(h), net), m);                     \
    std::memcpy(out, v.data(), v.size() * sizeof(T));                                            \
  }                                                                                              \
  void ref_sac##SUFFIX##_set_net(void* h, int net, std::uint64_t m, const T* in) {               \
    auto& p = sac_net(*static_cast<SacState<T>*>(h), net);                                       \
    unflatten_member(p, m, std::span<const T>(in, p.params_per_member()));                       \
  }                                                                                              \
  void ref_sac##SUFFIX##_get_adam(void* h, int net, std::uint64_t m, T* mo, T* vo,               \
                                  std::int64_t* t) {                                             \
    auto& opt = sac_opt(*static_cast<SacState<T>*>(h), net);                                     \
    std::size_t at = 0;                                                                          \
    for (std::size_t l = 0; l < opt.w.size(); ++l) {                                             \
      for (auto* st : {&opt.w[l], &opt.b[l]}) {                                                  \
        const std::size_t s = st->m.member_stride();                                             \
        std::memcpy(mo + at, st->m.member_ptr(m), s * sizeof(T));                                \
        std::memcpy(vo + at, st->v.member_ptr(m), s * sizeof(T));                                \
        at += s;                                                                                 \
      }                                                                                          \
    }                                                                                            \
    *t = opt.w[0].t[m];                                                                          \
  }                                                                                              \
  void ref_sac##SUFFIX##_get_alpha(void* h, T* log_alpha, T* am, T* av, std::int64_t* at,        \
                                   std::uint64_t* steps) {                                       \
    auto& st = *static_cast<SacState<T>*>(h);                                                    \
    const std::size_t n = st.members();                                                          \
    for (std::size_t m = 0; m < n; ++m) {                                                        \
      log_alpha[m] = st.log_alpha.data[m];                                                       \
      am[m] = st.opt_alpha.m.data[m];                                                            \
      av[m] = st.opt_alpha.v.data[m];                                                            \
      at[m] = st.opt_alpha.t[m];                                                                 \
      steps[m] = st.steps[m];                                                                    \
    }                                                                                            \
  }                                                                                              \
  int ref_sac##SUFFIX##_step(void* h, const T* s, const T* a, const T* r, const T* s2,           \
                             const T* d, std::uint64_t b, const double* hyper) {                 \
    return guarded([&] {                                                                         \
      auto& st = *static_cast<SacState<T>*>(h);                                                  \
      const std::size_t n = st.members();                                                        \
      auto batch = batch_from(s, a, r, s2, d, n, b, st.obs_dim, st.act_dim);                     \
      sac_update_step(st, batch, sac_hyper_from(hyper, n));                                      \
    });                                                                                          \
  }                                                                                              \
  int ref_sac##SUFFIX##_losses(void* h, const T* s, const T* a, const T* r, const T* s2,         \
                               const T* d, std::uint64_t b, const double* hyper, double* out3) { \
    return guarded([&] {                                                                         \
      SacState<T> st = *static_cast<SacState<T>*>(h);                                            \
      const std::size_t n = st.members();                                                        \
      auto batch = batch_from(s, a, r, s2, d, n, b, st.obs_dim, st.act_dim);                     \
      auto hy = sac_hyper_from(hyper, n);                                                        \
      std::vector<double> alpha(n);                                                              \
      for (std::size_t m = 0; m < n; ++m)                                                        \
        alpha[m] = std::exp(static_cast<double>(st.log_alpha.data[m]));                          \
      auto y = sac_critic_target(st, batch, hy);                                                 \
      auto sa = concat_features(batch.s, batch.a);                                               \
      auto [l1, g1] = mse_loss_grads(st.critic1, sa, y);                                         \
      st.opt_critic1.step(st.critic1, g1, hy.critic_lr);                                         \
      auto [l2, g2] = mse_loss_grads(st.critic2, sa, y);                                         \
      st.opt_critic2.step(st.critic2, g2, hy.critic_lr);                                         \
      auto eps = detail::draw_eps<T>(n, b, st.act_dim, st.seed, st.streams, st.steps,            \
                                     RngUse::kSacEps);                                           \
      auto pol = sac_policy_loss_grads(st.policy, st.critic1, st.critic2, batch.s, alpha, eps,   \
                                       st.action_bound);                                         \
      out3[0] = l1;                                                                              \
      out3[1] = l2;                                                                              \
      out3[2] = pol.loss_sum;                                                                    \
    });                                                                                          \
  }

PBRL_REF_SAC(f, float)
PBRL_REF_SAC(d, double)

// ---------------------------------------------------------------- action selection (float)
int ref_td3f_act(void* h, const float* obs, std::uint64_t rows, const double* noise_std,
                 std::uint64_t seed, const std::uint64_t* steps, int deterministic, float* out) {
  return guarded([&] {
    auto& st = *static_cast<Td3State<float>*>(h);
    const std::size_t n = st.members(), ds = st.policy.in_dim();
    PopTensor<float> o({n, rows, ds}, std::vector<float>(obs, obs + n * rows * ds));
    auto a = act(st.policy, o, std::vector<double>(noise_std, noise_std + n), seed, st.streams,
                 std::vector<std::uint64_t>(steps, steps + n), deterministic != 0);
    std::memcpy(out, a.data.data(), a.data.size() * sizeof(float));
  });
}

int ref_sacf_act(void* h, const float* obs, std::uint64_t rows, std::uint64_t seed,
                 const std::uint64_t* steps, int deterministic, float* out) {
  return guarded([&] {
    auto& st = *static_cast<SacState<float>*>(h);
    const std::size_t n = st.members(), ds = st.policy.in_dim();
    PopTensor<float> o({n, rows, ds}, std::vector<float>(obs, obs + n * rows * ds));
    auto a = sac_act(st.policy, o, st.action_bound, seed, st.streams,
                     std::vector<std::uint64_t>(steps, steps + n), deterministic != 0);
    std::memcpy(out, a.data.data(), a.data.size() * sizeof(float));
  });
}

// ---------------------------------------------------------------- replay snapshots (float)
int ref_replay_save_snapshot(void* h, const char* path) {
  return guarded([&] {
    std::ofstream os(path, std::ios::binary);
    static_cast<ReplayBuffer<float>*>(h)->save_snapshot(os);
  });
}
void* ref_replay_load_snapshot(const char* path) {
  std::ifstream is(path, std::ios::binary);
  return ReplayBuffer<float>::load_snapshot(is).release();
}

// ---------------------------------------------------------------- checkpoints (float)
int ref_td3f_save_checkpoint(void* h, int net, const char* path) {
  return guarded([&] { save_checkpoint(td3_net(*static_cast<Td3State<float>*>(h), net), std::string(path)); });
}
int ref_td3f_load_checkpoint(void* h, int net, const char* path) {
  return guarded([&] {
    td3_net(*static_cast<Td3State<float>*>(h), net) = load_checkpoint<float>(std::string(path));
  });
}
int ref_td3f_serialize_state(void* h, const char* path) {
  return guarded([&] {
    std::ofstream os(path, std::ios::binary);
    serialize_state(*static_cast<Td3State<float>*>(h), os);
  });
}

// ---------------------------------------------------------------- synthetic batches
void ref_synthetic_batches_f(std::uint64_t count, std::uint64_t n, std::uint64_t b,
                             std::uint64_t ds, std::uint64_t da, std::uint64_t seed, float* s,
                             float* a, float* r, float* s2, float* d) {
  auto bs = make_synthetic_batches<float>(count, n, b, ds, da, seed);
  for (std::size_t i = 0; i < count; ++i) {
    std::memcpy(s + i * n * b * ds, bs[i].s.data.data(), n * b * ds * sizeof(float));
    std::memcpy(a + i * n * b * da, bs[i].a.data.data(), n * b * da * sizeof(float));
    std::memcpy(r + i * n * b, bs[i].r.data.data(), n * b * sizeof(float));
    std::memcpy(s2 + i * n * b * ds, bs[i].s2.data.data(), n * b * ds * sizeof(float));
    std::memcpy(d + i * n * b, bs[i].done.data.data(), n * b * sizeof(float));
  }
}

// ---------------------------------------------------------------- replay
void* ref_replay_create(std::uint64_t cap, std::uint64_t ds, std::uint64_t da) {
  return new ReplayBuffer<float>(cap, ds, da);
}
void ref_replay_destroy(void* h) { delete static_cast<ReplayBuffer<float>*>(h); }
void ref_replay_push(void* h, const float* s, const float* a, float r, const float* s2, float d,
                     std::uint32_t member) {
  auto* buf = static_cast<ReplayBuffer<float>*>(h);
  Transition<float> t;
  t.s.assign(s, s + buf->obs_dim());
  t.a.assign(a, a + buf->act_dim());
  t.s2.assign(s2, s2 + buf->obs_dim());
  t.r = r;
  t.done = d;
  t.member = member;
  buf->push(t);
}
std::uint64_t ref_replay_size(void* h) { return static_cast<ReplayBuffer<float>*>(h)->size(); }
// returns 1 when a batch was drawn, 0 when not ready (nullopt), <0 on error
int ref_sample_batch(void** bufs, std::uint64_t nbufs, std::uint64_t batch, int mode,
                     std::uint64_t members, std::uint64_t seed, const std::uint64_t* streams,
                     std::uint64_t draw_id, std::uint64_t min_size, float* s, float* a, float* r,
                     float* s2, float* d) {
  int ready = 0;
  int rc = guarded([&] {
    std::vector<ReplayBuffer<float>*> bv;
    for (std::size_t i = 0; i < nbufs; ++i) bv.push_back(static_cast<ReplayBuffer<float>*>(bufs[i]));
    std::vector<std::uint64_t> sv(streams, streams + members);
    auto out = sample_batch<float>(bv, batch, mode == 0 ? BufferMode::kPerAgent : BufferMode::kShared,
                                   members, seed, sv, draw_id, min_size);
    if (!out) return;
    ready = 1;
    std::memcpy(s, out->s.data.data(), out->s.data.size() * sizeof(float));
    std::memcpy(a, out->a.data.data(), out->a.data.size() * sizeof(float));
    std::memcpy(r, out->r.data.data(), out->r.data.size() * sizeof(float));
    std::memcpy(s2, out->s2.data.data(), out->s2.data.size() * sizeof(float));
    std::memcpy(d, out->done.data.data(), out->done.data.size() * sizeof(float));
  });
  return rc < 0 ? rc : ready;
}

// ---------------------------------------------------------------- PBT
// rings: [n][ring_cap] doubles, counts[n] valid entries (oldest first)
int ref_pbt_rank(const double* rings, const std::uint32_t* counts, std::uint64_t n,
                 std::uint64_t ring_cap, std::uint64_t* order) {
  return guarded([&] {
    auto o = pbt_rank(pbt_from(rings, counts, n, ring_cap));
    for (std::size_t i = 0; i < n; ++i) order[i] = o[i];
  });
}

// rng = (key, next); returns the plan size (0 when n < 4) or <0 on error
int ref_pbt_plan(const double* rings, const std::uint32_t* counts, std::uint64_t n,
                 std::uint64_t ring_cap, double trunc, std::uint64_t rng_key,
                 std::uint64_t* rng_next, std::uint64_t* replaced, std::uint64_t* donors) {
  int cnt = 0;
  int rc = guarded([&] {
    auto st = pbt_from(rings, counts, n, ring_cap);
    st.truncation_fraction = trunc;
    RngSequence rng(RngStream{rng_key});
    rng.next = *rng_next;
    auto plan = pbt_plan(st, rng);
    *rng_next = rng.next;
    if (!plan) return;
    cnt = static_cast<int>(plan->replaced.size());
    for (int i = 0; i < cnt; ++i) {
      replaced[i] = plan->replaced[i];
      donors[i] = plan->donors[i];
    }
  });
  return rc < 0 ? rc : cnt;
}

int ref_td3f_pbt_evolve(void* h, const double* rings, const std::uint32_t* counts,
                        std::uint64_t ring_cap, double* hyper, std::uint64_t rng_key,
                        std::uint64_t* rng_next, std::uint64_t* replaced, std::uint64_t* donors) {
  int cnt = 0;
  int rc = guarded([&] {
    auto& st = *static_cast<Td3State<float>*>(h);
    const std::size_t n = st.members();
    auto pbt = pbt_from(rings, counts, n, ring_cap);
    auto hy = td3_hyper_from(hyper, n);
    RngSequence rng(RngStream{rng_key});
    rng.next = *rng_next;
    auto plan = pbt_evolve_trainer(pbt, st, hy, Td3Prior{}, rng);
    *rng_next = rng.next;
    td3_hyper_to(hy, hyper);
    if (!plan) return;
    cnt = static_cast<int>(plan->replaced.size());
    for (int i = 0; i < cnt; ++i) {
      replaced[i] = plan->replaced[i];
      donors[i] = plan->donors[i];
    }
  });
  return rc < 0 ? rc : cnt;
}

int ref_sacf_pbt_evolve(void* h, const double* rings, const std::uint32_t* counts,
                        std::uint64_t ring_cap, double* hyper, double default_target_entropy,
                        std::uint64_t rng_key, std::uint64_t* rng_next, std::uint64_t* replaced,
                        std::uint64_t* donors) {
  int cnt = 0;
  int rc = guarded([&] {
    auto& st = *static_cast<SacState<float>*>(h);
    const std::size_t n = st.members();
    auto pbt = pbt_from(rings, counts, n, ring_cap);
    auto hy = sac_hyper_from(hyper, n);
    SacPrior prior;
    prior.default_target_entropy = default_target_entropy;
    RngSequence rng(RngStream{rng_key});
    rng.next = *rng_next;
    auto plan = pbt_evolve_trainer(pbt, st, hy, prior, rng);
    *rng_next = rng.next;
    sac_hyper_to(hy, hyper);
    if (!plan) return;
    cnt = static_cast<int>(plan->replaced.size());
    for (int i = 0; i < cnt; ++i) {
      replaced[i] = plan->replaced[i];
      donors[i] = plan->donors[i];
    }
  });
  return rc < 0 ? rc : cnt;
}

// ---------------------------------------------------------------- bench_update
// mode: 0 sequential, 1 vectorized, 2 parallel_threads; algo: 0 td3, 1 sac
int ref_bench_update(int mode, int algo, std::uint64_t n, std::uint64_t k, std::uint64_t reps,
                     std::uint64_t batch, const std::uint64_t* hidden, std::uint32_t nh,
                     std::uint64_t budget_bytes, double* median_ms, double* iqr_ms,
                     double* warmup_ms, std::uint64_t* launches) {
  return guarded([&] {
    BenchConfig cfg;
    cfg.mode = mode == 0 ? BenchMode::kSequential
                         : (mode == 1 ? BenchMode::kVectorized : BenchMode::kParallelThreads);
    cfg.algo = algo == 0 ? BenchAlgo::kTd3 : BenchAlgo::kSac;
    cfg.n = n;
    cfg.k = k;
    cfg.reps = reps;
    cfg.batch = batch;
    cfg.hidden = to_dims(hidden, nh);
    if (budget_bytes) cfg.memory_budget_bytes = budget_bytes;
    auto r = bench_update<float>(cfg);
    *median_ms = r.median_ms;
    *iqr_ms = r.iqr_ms;
    *warmup_ms = r.warmup_ms;
    *launches = r.kernel_launches;
  });
}

std::uint64_t ref_kernel_invocations() { return kernel_invocations().load(); }

// ---------------------------------------------------------------- DvD / CEM (evolve.hpp:221-525)
double ref_dvd_lambda(std::uint64_t step, double start, double end, std::uint64_t horizon) {
  return dvd_lambda(step, LambdaSchedule{start, end, horizon});
}

int ref_dvd_loss(const double* emb, std::uint64_t n, std::uint64_t dim, double length_scale,
                 double jitter, double lambda, double* loss, double* logdet, double* grad) {
  return guarded([&] {
    PopTensor<double> e = PopTensor<double>::zeros({n, dim});
    std::memcpy(e.data.data(), emb, n * dim * sizeof(double));
    DvdLossOut out = dvd_loss(e, length_scale, jitter, lambda);
    *loss = out.loss;
    *logdet = out.logdet;
    std::memcpy(grad, out.grad.data.data(), n * dim * sizeof(double));
  });
}

double ref_median_pairwise_distance(const double* emb, std::uint64_t n, std::uint64_t dim) {
  PopTensor<double> e = PopTensor<double>::zeros({n, dim});
  std::memcpy(e.data.data(), emb, n * dim * sizeof(double));
  return median_pairwise_distance(e);
}

// cem_sample from RngSequence(seed, stream_id, use, step) advanced to *next
void ref_cem_sample(const double* mean, const double* var, double noise, std::uint64_t dim,
                    std::uint64_t count, std::uint64_t key, std::uint64_t* next, double* out) {
  CEMState st;
  st.mean.assign(mean, mean + dim);
  st.var.assign(var, var + dim);
  st.noise = noise;
  RngSequence rng(RngStream{key});
  rng.next = *next;
  auto c = cem_sample(st, count, rng);
  for (std::size_t i = 0; i < count; ++i) std::memcpy(out + i * dim, c[i].data(), dim * 8);
  *next = rng.next;
}

int ref_cem_update(double* mean, double* var, double* noise, double noise_final,
                   double noise_decay, double elite_fraction, std::uint64_t dim,
                   const double* cands, const double* scores, std::uint64_t count) {
  return guarded([&] {
    CEMState st;
    st.mean.assign(mean, mean + dim);
    st.var.assign(var, var + dim);
    st.noise = *noise;
    st.noise_final = noise_final;
    st.noise_decay = noise_decay;
    st.elite_fraction = elite_fraction;
    std::vector<std::vector<double>> c(count);
    for (std::size_t i = 0; i < count; ++i) c[i].assign(cands + i * dim, cands + (i + 1) * dim);
    cem_update(st, c, std::vector<double>(scores, scores + count));
    std::memcpy(mean, st.mean.data(), dim * 8);
    std::memcpy(var, st.var.data(), dim * 8);
    *noise = st.noise;
  });
}

}  // extern "C"
