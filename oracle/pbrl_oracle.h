/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * CPU restatement of the reference population-update path (pbrl, /root/reference/proj/core)
 * in plain C, used only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg
 * as the checker.  The product library (paper_2206_08888_b200/libpbrl_b200.so) never links,
 * loads or calls anything here.
 *
 * Parity pinning: tests/test_oracle_vs_ref.py compares every function here bit-for-bit with
 * the unmodified reference compiled from its own sources (oracle/_ref/libpbrl_ref.so, built by
 * oracle/Makefile), and tests/test_oracle_golden.py against fixtures in tests/golden/ generated
 * from that reference build by oracle/make_golden.py.
 *
 * Layout: every network population is one flat float arena [n][P], member-major, each member
 * in the reference flatten_member order (net_pop.hpp:162-173): W0 (in x out, row-major), b0,
 * W1, b1, ...  — the same layout the device arena uses.
 */
#ifndef PBRL_ORACLE_H
#define PBRL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* counter RNG, rng.hpp:13-70 */
/* derive_tolerances.py only: 0 exact fp32, 1 TF32 operands, 2 BF16 operands */
void ora_set_emulation(int mode);

uint64_t ora_mix64(uint64_t x);
uint64_t ora_stream_key(uint64_t seed, uint64_t stream, uint64_t use, uint64_t step);
uint64_t ora_bits(uint64_t key, uint64_t counter);
double ora_uniform(uint64_t key, uint64_t counter);
double ora_normal_pair(uint64_t key, uint64_t counter);

/* TD3 population state (algos.hpp:165-212).  nets: 0 policy, 1 policy_target, 2 critic1,
 * 3 critic2, 4 critic1_target, 5 critic2_target.  Hyper arrays are [8][n] doubles in the order
 * critic_lr, policy_lr, policy_delay_ratio, explore_std, target_std, target_clip, gamma, tau. */
typedef struct ora_td3 ora_td3;
ora_td3* ora_td3_create(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                        uint32_t nh, double bound, uint64_t seed);
/* shared != 0: PopMode::kSharedCritic -- critic nets (2..5) and their Adam states have ONE
 * member; the critic loss averages over the population folded into the batch */
ora_td3* ora_td3_create_mode(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                             uint32_t nh, double bound, uint64_t seed, int shared);
void ora_td3_destroy(ora_td3* st);
uint64_t ora_td3_param_count(const ora_td3* st, int net);
void ora_td3_get_net(const ora_td3* st, int net, uint64_t m, float* out);
void ora_td3_set_net(ora_td3* st, int net, uint64_t m, const float* in);
void ora_td3_get_adam(const ora_td3* st, int net, uint64_t m, float* mo, float* vo, int64_t* t);
void ora_td3_get_counters(const ora_td3* st, double* delay_acc, uint64_t* steps);
/* y out [n][B]; state untouched */
void ora_td3_target(const ora_td3* st, const float* s2, const float* r, const float* d, uint64_t b,
                    const double* hyper, float* y);
/* one td3_update_step; losses (optional) [3][n]: critic1 MSE, critic2 MSE, policy loss
 * (per member; the policy entry is 0 for members that did not fire).  returns 0 or -2 (config). */
/* act / sac_act (algos.hpp:895-942): actions [n][rows][da] for obs [n][rows][ds] */
void ora_td3_act(const ora_td3* st, const float* obs, uint64_t rows, const double* noise_std,
                 uint64_t seed, const uint64_t* steps, int deterministic, float* out);
int ora_td3_step(ora_td3* st, const float* s, const float* a, const float* r, const float* s2,
                 const float* d, uint64_t b, const double* hyper, const char* policy_mask,
                 double* losses);
/* shared-critic losses: losses[0] = critic1 MSE over all n*b rows, losses[n] = critic2 */

/* DvD (evolve.hpp:304-525).  probe: [m_states][obs] doubles (DvDConfig::probe_states, cast to
 * float as dvd_policy_hook does); lambda = dvd_lambda(step, schedule). */
typedef struct {
  const double* probe;
  uint64_t m_states;
  double length_scale, jitter, lambda;
} ora_dvd;
/* td3_update_step with the dvd_policy_hook (NULL: none).  returns 0, -2, or -10 when the
 * hook's kernel matrix is singular (DegeneratePopulationError; the critic step has run). */
int ora_td3_step_hook(ora_td3* st, const float* s, const float* a, const float* r,
                      const float* s2, const float* d, uint64_t b, const double* hyper,
                      const char* policy_mask, double* losses, const ora_dvd* dvd);
double ora_dvd_lambda(uint64_t step, double start, double end, uint64_t horizon);
/* dvd_loss: emb [n][dim]; grad [n][dim] (optional).  0, -2 (ConfigError), -10 (Degenerate) */
int ora_dvd_loss(const double* emb, uint64_t n, uint64_t dim, double length_scale, double jitter,
                 double lambda, double* loss, double* logdet, double* grad);
double ora_median_pairwise_distance(const double* emb, uint64_t n, uint64_t dim);
/* dvd_embed: out [n][m_states*da] */
void ora_td3_dvd_embed(const ora_td3* st, const double* probe, uint64_t m_states, float* out);

/* CEM (evolve.hpp:221-297): cem_sample draws count x dim normals from the RngSequence
 * (key, *next), candidate-major; cem_update refits mean / var to the elites and decays noise.
 * returns 0 or -2 (ConfigError: fewer than 2, odd count, non-finite score). */
void ora_cem_sample(const double* mean, const double* var, double noise, uint64_t dim,
                    uint64_t count, uint64_t key, uint64_t* next, double* out);
int ora_cem_update(double* mean, double* var, double* noise, double noise_final,
                   double noise_decay, double elite_fraction, uint64_t dim, const double* cands,
                   const double* scores, uint64_t count);

/* SAC population state (algos.hpp:473-521).  nets: 0 policy, 2 critic1, 3 critic2,
 * 4 critic1_target, 5 critic2_target.  Hyper arrays are [7][n]: policy_lr, critic_lr, alpha_lr,
 * target_entropy, reward_scale, gamma, tau. */
typedef struct ora_sac ora_sac;
ora_sac* ora_sac_create(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                        uint32_t nh, double bound, uint64_t seed);
ora_sac* ora_sac_create_mode(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                             uint32_t nh, double bound, uint64_t seed, int shared);
void ora_sac_destroy(ora_sac* st);
uint64_t ora_sac_param_count(const ora_sac* st, int net);
void ora_sac_get_net(const ora_sac* st, int net, uint64_t m, float* out);
void ora_sac_set_net(ora_sac* st, int net, uint64_t m, const float* in);
void ora_sac_get_adam(const ora_sac* st, int net, uint64_t m, float* mo, float* vo, int64_t* t);
void ora_sac_get_alpha(const ora_sac* st, float* log_alpha, float* am, float* av, int64_t* at,
                       uint64_t* steps);
void ora_sac_act(const ora_sac* st, const float* obs, uint64_t rows, uint64_t seed,
                 const uint64_t* steps, int deterministic, float* out);
int ora_sac_step(ora_sac* st, const float* s, const float* a, const float* r, const float* s2,
                 const float* d, uint64_t b, const double* hyper, double* losses);

/* synthetic batches, bench.hpp:69-93; arrays [count][n][b][dim] */
void ora_synthetic_batches(uint64_t count, uint64_t n, uint64_t b, uint64_t ds, uint64_t da,
                           uint64_t seed, float* s, float* a, float* r, float* s2, float* d);

/* replay ring, replay.hpp:28-111, and sample_batch, replay.hpp:181-204 */
typedef struct ora_replay ora_replay;
ora_replay* ora_replay_create(uint64_t cap, uint64_t ds, uint64_t da);
void ora_replay_destroy(ora_replay* rb);
void ora_replay_push(ora_replay* rb, const float* s, const float* a, float r, const float* s2,
                     float d, uint32_t member);
uint64_t ora_replay_size(const ora_replay* rb);
/* mode 0 per-agent, 1 shared; returns 1 ready, 0 not ready; slots (optional) [members][b] */
int ora_sample_batch(ora_replay** bufs, uint64_t nbufs, uint64_t b, int mode, uint64_t members,
                     uint64_t seed, const uint64_t* streams, uint64_t draw_id, uint64_t min_size,
                     float* s, float* a, float* r, float* s2, float* d, uint64_t* slots);

/* PBT, evolve.hpp:80-213.  rings [n][ring_cap] oldest first, counts[n] valid entries.
 * The RngSequence is (key, *next).  Returns the plan size, 0 when n < 4, -4 when a member
 * has no recorded return (NotReadyError). */
int ora_pbt_rank(const double* rings, const uint32_t* counts, uint64_t n, uint64_t ring_cap,
                 uint64_t* order);
int ora_pbt_plan(const double* rings, const uint32_t* counts, uint64_t n, uint64_t ring_cap,
                 double trunc, uint64_t rng_key, uint64_t* rng_next, uint64_t* replaced,
                 uint64_t* donors);
int ora_td3_pbt_evolve(ora_td3* st, const double* rings, const uint32_t* counts,
                       uint64_t ring_cap, double* hyper, uint64_t rng_key, uint64_t* rng_next,
                       uint64_t* replaced, uint64_t* donors);
int ora_sac_pbt_evolve(ora_sac* st, const double* rings, const uint32_t* counts,
                       uint64_t ring_cap, double* hyper, double default_target_entropy,
                       uint64_t rng_key, uint64_t* rng_next, uint64_t* replaced,
                       uint64_t* donors);
/* Td3Prior / SacPrior draws (evolve.hpp:31-73); out [8] / [7] in the hyper field order */
void ora_td3_prior_sample(uint64_t rng_key, uint64_t* rng_next, double* out8);
void ora_sac_prior_sample(uint64_t rng_key, uint64_t* rng_next, double default_te, double* out7);

#ifdef __cplusplus
}
#endif
#endif
