// Reference-API code ported by changing the namespace (see include/pbrl_b200.hpp):
// make a TD3 population of 4, run 2 update steps on synthetic batches, print a checksum.
#include <cstdio>
#include <random>

#include "pbrl_b200.hpp"

int main() {
  namespace pb = pbrl::b200;
  const std::size_t n = 4, ds = 17, da = 6, B = 64;
  auto st = pb::make_td3_state(n, ds, da, {256, 256}, 1.0, 7, pb::PopMode::kIndependent, pb::Precision::kTf32);
  auto hy = pb::Td3Hyper::defaults(n);
  std::mt19937 gen(1);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  pb::TransitionBatch b;
  b.n = n;
  b.rows = B;
  for (auto* v : {&b.s, &b.s2}) v->resize(n * B * ds);
  b.a.resize(n * B * da);
  b.r.resize(n * B);
  b.done.assign(n * B, 0.f);
  for (auto* v : {&b.s, &b.s2, &b.a, &b.r})
    for (auto& x : *v) x = u(gen);
  for (int k = 0; k < 2; ++k) pb::td3_update_step(st, b, hy);
  double sum = 0;
  for (float x : st.flatten_member(pb::Net::kPolicy, 0)) sum += x;
  std::printf("policy[0] checksum %.6f steps %llu\n", sum,
              static_cast<unsigned long long>(st.steps()[0]));
  // act (algos.hpp:895-915): one observation per member, exploration std 0.1
  std::vector<float> obs(n * ds, 0.5f);
  const auto acts = pb::act(st, obs, 1, std::vector<double>(n, 0.1), 7, st.steps(), false);
  std::printf("act: %zu actions, a[0] = %.4f\n", acts.size(), acts[0]);
  try {
    hy.tau[0] = 2.0;
    pb::td3_update_step(st, b, hy);
  } catch (const pb::ConfigError& e) {
    std::printf("ConfigError as in the reference: %s\n", e.what());
  }
  return 0;
}
