// Host-side pieces of include/pbrl_b200_pipeline.hpp (no device): RatioController semantics
// (replay.hpp:205-298, the reference's test_replay.cpp ratio cases) and BoundedQueue
// (pipeline.hpp:89-148).  Built and run by tests/test_pipeline_host.py.
#include <cassert>
#include <chrono>
#include <cstdio>
#include <thread>

#include "pbrl_b200_pipeline.hpp"

using namespace pbrl::b200;
using namespace std::chrono_literals;

#define EXPECT(c)                                                        \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                          \
    }                                                                    \
  } while (0)

int main() {
  // sample side blocks until warm-up, then keeps updates <= target (1 + slack) env steps
  RatioController c(0.5, 0.0, 10);
  EXPECT(c.check(RatioSide::kSample) == RatioDecision::kBlock);
  c.on_env_steps(10);
  EXPECT(c.check(RatioSide::kSample, 5) == RatioDecision::kProceed);
  EXPECT(c.check(RatioSide::kSample, 6) == RatioDecision::kBlock);
  c.on_update_steps(5);
  EXPECT(c.check(RatioSide::kSample) == RatioDecision::kBlock);
  // insert side: env <= upd / target (1 + slack) + warmup
  EXPECT(c.check(RatioSide::kInsert, 10) == RatioDecision::kProceed);  // 20 <= 10 + 10
  EXPECT(c.check(RatioSide::kInsert, 11) == RatioDecision::kBlock);
  c.on_env_steps(2);
  EXPECT(c.check(RatioSide::kSample) == RatioDecision::kProceed);  // 6 <= 0.5 * 12
  // await: bounded; wakes when the other side moves; closed always proceeds
  EXPECT(!c.await(RatioSide::kSample, 5ms, 2));
  std::thread t([&] {
    std::this_thread::sleep_for(20ms);
    c.on_env_steps(4);
  });
  EXPECT(c.await(RatioSide::kSample, 2000ms, 2));
  t.join();
  c.close();
  EXPECT(c.await(RatioSide::kSample, 1ms, 1000));
  bool threw = false;
  try {
    RatioController bad(0.0, 0.0, 0);
  } catch (const ConfigError&) {
    threw = true;
  }
  EXPECT(threw);

  // bounded queue: capacity, timeouts, FIFO, close releases both sides
  BoundedQueue<int> q(2);
  EXPECT(q.push(1, 1ms) && q.push(2, 1ms));
  EXPECT(!q.push(3, 5ms));
  int v = 0;
  EXPECT(q.pop(v, 1ms) && v == 1);
  EXPECT(q.push(3, 1ms));
  EXPECT(q.pop(v, 1ms) && v == 2 && q.pop(v, 1ms) && v == 3);
  EXPECT(!q.pop(v, 5ms));
  std::thread closer([&] {
    std::this_thread::sleep_for(20ms);
    q.close();
  });
  EXPECT(!q.pop(v, 5000ms));
  closer.join();
  EXPECT(q.closed() && !q.push(4, 1ms));

  // the built-in environment: deterministic resets, horizon, reward sign
  PointMassEnv e(2, 5);
  auto o1 = e.reset(7), o2 = e.reset(7);
  EXPECT(o1 == o2 && o1.size() == 4);
  Env::Step s{};
  for (int i = 0; i < 5; ++i) s = e.step({0.5, -0.5});
  EXPECT(s.done && s.reward <= 0);

  // RunConfig::validate for the shared-critic strategies (pipeline.hpp:229-238,
  // pipeline_run.hpp:81-83): CEM / DvD need shared-critic mode, one shared buffer, TD3, and CEM
  // an even population; PBT needs per-agent buffers
  auto rejects = [](const RunConfig& rc) {
    try {
      rc.validate();
    } catch (const ConfigError&) {
      return true;
    }
    return false;
  };
  RunConfig rc;
  rc.population = 4;
  rc.strategy = Strategy::kCem;
  EXPECT(rejects(rc));  // independent mode
  rc.mode = PopMode::kSharedCritic;
  EXPECT(rejects(rc));  // per-agent buffers
  rc.buffer_mode = BufferMode::kShared;
  EXPECT(!rejects(rc));
  rc.population = 5;
  EXPECT(rejects(rc));  // odd CEM population
  rc.strategy = Strategy::kDvd;
  EXPECT(!rejects(rc));
  rc.algo = Algo::kSac;
  EXPECT(rejects(rc));  // TD3-only strategies
  rc = RunConfig{};
  rc.strategy = Strategy::kPbt;
  rc.buffer_mode = BufferMode::kShared;
  EXPECT(rejects(rc));
  // DvD schedule and configuration checks (evolve.hpp:304-314, :489-503)
  DvDConfig dv;
  dv.m_states = 2;
  bool dthrew = false;
  try {
    dv.validate(3);
  } catch (const ConfigError&) {
    dthrew = true;
  }
  EXPECT(dthrew);
  std::printf("pipeline host: OK\n");
  return 0;
}
