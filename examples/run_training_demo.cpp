// Threaded training on the B200 population API (include/pbrl_b200_pipeline.hpp): W actor
// threads acting on the device from a snapshot mailbox, an ingest thread feeding the device
// replay rings with batched inserts under the ratio guard, and the learner thread running
// device sample + K-update bursts (the reference's run_training, pipeline_run.hpp:77-468).
//
//   run_training_demo [pop] [workers] [total_updates] [K] [none|pbt|cem|dvd (0|1 = none|pbt)]
//                     [bf16|tf32|ffma32]
// cem / dvd run the shared-critic TD3 population on one shared replay ring (pipeline.hpp:229-238).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "pbrl_b200_pipeline.hpp"

using namespace pbrl::b200;

int main(int argc, char** argv) {
  RunConfig cfg;
  cfg.population = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 4;
  cfg.actor_workers = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 2;
  cfg.total_updates = argc > 3 ? std::strtoul(argv[3], nullptr, 10) : 400;
  cfg.updates_per_burst = argc > 4 ? std::strtoul(argv[4], nullptr, 10) : 20;
  const char* strat = argc > 5 ? argv[5] : "none";
  cfg.strategy = (!std::strcmp(strat, "1") || !std::strcmp(strat, "pbt")) ? Strategy::kPbt
                 : !std::strcmp(strat, "cem")                            ? Strategy::kCem
                 : !std::strcmp(strat, "dvd")                            ? Strategy::kDvd
                                                                         : Strategy::kNone;
  if (cfg.strategy == Strategy::kCem || cfg.strategy == Strategy::kDvd) {
    cfg.mode = PopMode::kSharedCritic;
    cfg.buffer_mode = BufferMode::kShared;
    cfg.cem_generation_updates = 100;
    cfg.dvd.schedule = LambdaSchedule{0.0, 0.5, 200};
  }
  const char* prec = argc > 6 ? argv[6] : "bf16";
  cfg.precision = !std::strcmp(prec, "tf32")     ? Precision::kTf32
                  : !std::strcmp(prec, "ffma32") ? Precision::kFfma32
                                                 : Precision::kBf16;
  cfg.hidden = {64, 64};
  cfg.batch_size = 64;
  cfg.buffer_capacity = 5000;
  cfg.warmup_per_buffer = 200;
  cfg.pbt_interval = 100;
  cfg.seed = 11;
  cfg.make_env = [] { return std::make_unique<PointMassEnv>(2, 50); };
  try {
    RunSummary s = run_training(cfg);
    std::printf("summary: update_steps=%llu env_steps=%llu dropped=%llu evolve_events=%llu "
                "published=%llu device_inserts=%llu eval_episodes=%llu ratio=%.3f wall=%.2fs\n",
                (unsigned long long)s.update_steps, (unsigned long long)s.env_steps,
                (unsigned long long)s.dropped_transitions, (unsigned long long)s.evolve_events,
                (unsigned long long)s.published_versions, (unsigned long long)s.device_inserts,
                (unsigned long long)s.eval_episodes, s.updates_per_member_env_step,
                s.wall_seconds);
    std::printf("returns:");
    for (double r : s.final_mean_returns) std::printf(" %.3f", r);
    std::printf("\nbest member %zu: %.3f\n", s.best_member, s.best_return);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "run_training failed: %s\n", e.what());
    return 1;
  }
  return 0;
}
