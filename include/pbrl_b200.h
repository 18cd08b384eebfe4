/* pbrl_b200 — C ABI of the B200-native population update path.
 *
 * Drop-in boundary for the reference's proj/core population-trainer API (namespace pbrl,
 * a header-only C++20 template library with no FFI of its own).  Each entry point below names
 * the reference interface it replaces.  A C++ facade with the reference's names and exception
 * types sits on top of this ABI in include/pbrl_b200.hpp; the Python host mirror is
 * paper_2206_08888_b200/pbrl.py.  See INTEGRATION.md for the bindings.
 *
 * Conventions
 *  - Every function returns an int status: PBRL_OK or a negative code that maps 1:1 onto the
 *    reference exception classes in errors.hpp:9-48 (ShapeError, ConfigError, UsageError,
 *    NotReadyError, ResourceError, DataStarvationError) plus CUDA / NCCL failures.
 *    pbrl_last_error() returns the thread-local message of the last failure.
 *  - Host pointers are caller-owned and only read/written during the call.  Device pointers
 *    (the *_device variants) must be valid on the population's device.
 *  - Calls on one handle must be serialised (the reference learner-thread contract,
 *    pipeline_run.hpp:330-355); distinct handles are independent.
 *  - Arrays of per-member values are indexed by LOCAL member (0 .. n-1); a shard created with
 *    member_offset = o keys its RNG streams by global id o + i (algos.hpp:210).
 */
#ifndef PBRL_B200_H
#define PBRL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.hpp:9-48) */
#define PBRL_OK 0
#define PBRL_E_SHAPE (-1)       /* ShapeError */
#define PBRL_E_CONFIG (-2)      /* ConfigError */
#define PBRL_E_USAGE (-3)       /* UsageError */
#define PBRL_E_NOT_READY (-4)   /* NotReadyError */
#define PBRL_E_RESOURCE (-5)    /* ResourceError */
#define PBRL_E_STARVATION (-6)  /* DataStarvationError */
#define PBRL_E_CUDA (-7)
#define PBRL_E_NCCL (-8)
#define PBRL_E_DEGENERATE (-9)  /* DegeneratePopulationError (DvD kernel matrix singular) */

#define PBRL_ALGO_TD3 0
#define PBRL_ALGO_SAC 1

/* arithmetic of the dense contractions; everything else is fp32 in every mode */
#define PBRL_PREC_FFMA32 0 /* CUDA-core fp32, reference k-order, no FMA: bit-exact check mode */
#define PBRL_PREC_BF16 1   /* tcgen05 kind::f16, bf16 operands, fp32 accumulate in TMEM */
#define PBRL_PREC_TF32 2   /* tcgen05 kind::tf32, fp32 operands rounded to tf32 */

/* network ids (Td3State / SacState members, algos.hpp:166-169, :475-477) */
#define PBRL_NET_POLICY 0
#define PBRL_NET_POLICY_TARGET 1 /* TD3 only */
#define PBRL_NET_CRITIC1 2
#define PBRL_NET_CRITIC2 3
#define PBRL_NET_CRITIC1_TARGET 4
#define PBRL_NET_CRITIC2_TARGET 5

/* PopMode (algos.hpp:26): one critic pair per member, or ONE shared critic pair whose batch is
 * the population folded into rows (CEM-RL / DvD; critic_forward, algos.hpp:219-233) */
#define PBRL_MODE_INDEPENDENT 0
#define PBRL_MODE_SHARED_CRITIC 1

#define PBRL_REPLAY_PER_AGENT 0 /* BufferMode::kPerAgent (replay.hpp:175) */
#define PBRL_REPLAY_SHARED 1    /* BufferMode::kShared */

typedef struct pbrl_pop pbrl_pop;

/* Population descriptor: the arguments of make_td3_state / make_sac_state
 * (algos.hpp:181-184, :490-493) plus device placement and sharding. */
typedef struct {
  int algo;                 /* PBRL_ALGO_* */
  uint64_t n;               /* local members on this device */
  uint64_t obs_dim, act_dim;
  uint32_t n_hidden;
  const uint64_t* hidden;   /* hidden widths */
  double action_bound;
  uint64_t seed;            /* make_*_state seed */
  int precision;            /* PBRL_PREC_* */
  int device;               /* CUDA ordinal */
  uint64_t member_offset;   /* global id of local member 0 (0 unless sharded) */
  uint64_t n_global;        /* population size across shards (0 = n) */
  int mode;                 /* PBRL_MODE_* (make_td3_state / make_sac_state `mode`) */
} pbrl_pop_desc;

/* One population batch (TransitionBatch, algos.hpp:14-24): s [n][B][obs], a [n][B][act],
 * r [n][B], s2 [n][B][obs], done [n][B]. */
typedef struct {
  const float* s;
  const float* a;
  const float* r;
  const float* s2;
  const float* done;
} pbrl_batch;

/* ---- lifecycle: make_td3_state / make_sac_state (algos.hpp:181-212, :490-521) */
int pbrl_pop_create(const pbrl_pop_desc* desc, pbrl_pop** out);
int pbrl_pop_destroy(pbrl_pop* pop);
int pbrl_last_error(char* buf, size_t len);
int pbrl_version(int* major, int* minor);

/* ---- hyperparameters: Td3Hyper / SacHyper per-member vectors (algos.hpp:32-156).
 * TD3 fields: critic_lr policy_lr policy_delay_ratio explore_std target_std target_clip gamma tau
 * SAC fields: policy_lr critic_lr alpha_lr target_entropy reward_scale gamma tau
 * pbrl_set_hyper validates like Td3Hyper::validate (algos.hpp:81-108) -> PBRL_E_CONFIG. */
int pbrl_set_hyper(pbrl_pop* pop, const char* field, const double* per_member);
int pbrl_get_hyper(pbrl_pop* pop, const char* field, double* per_member);

/* ---- parameters in flatten_member layout (net_pop.hpp:162-202) */
int pbrl_param_count(pbrl_pop* pop, int net, uint64_t* count);
int pbrl_get_member(pbrl_pop* pop, int net, uint64_t member, float* flat);
int pbrl_set_member(pbrl_pop* pop, int net, uint64_t member, const float* flat);
/* copy_member (net_pop.hpp:192-202) for one network, on device */
int pbrl_copy_member(pbrl_pop* pop, int net, uint64_t src, uint64_t dst);
/* Adam moments of one member in flatten order + its step count (pop_tensor.hpp:299-323);
 * net = PBRL_NET_POLICY / CRITIC1 / CRITIC2 */
int pbrl_get_adam(pbrl_pop* pop, int net, uint64_t member, float* m, float* v, int64_t* t);
/* TD3: delay_acc + steps (algos.hpp:170-171).  SAC: delay_acc unused (may be NULL). */
int pbrl_get_counters(pbrl_pop* pop, double* delay_acc, uint64_t* steps);
/* SAC temperature state: log_alpha, its Adam m, v, t (algos.hpp:478-479) */
int pbrl_get_alpha(pbrl_pop* pop, float* log_alpha, float* m, float* v, int64_t* t);

/* ---- update: td3_update_step / sac_update_step (algos.hpp:351-422, :781-837) chained k
 * times as in update_k_steps (algos.hpp:953-983).  batches: k host batches of B rows;
 * policy_mask (TD3 only, may be NULL): [n] bytes, policy_member_mask of td3_update_step. */
int pbrl_update_batches(pbrl_pop* pop, const pbrl_batch* batches, uint32_t k, uint64_t batch_rows,
                        const uint8_t* policy_mask);
/* Same with device-resident batches (pointers valid on the population's device).  Inside one
 * call (k > 1) the pack of batch i+1 runs beside step i's last Adam on a library stream, so k
 * batches per call are faster than k calls; the batches must stay valid until the call's work
 * has completed on the population's stream. */
int pbrl_update_batches_device(pbrl_pop* pop, const pbrl_batch* batches, uint32_t k,
                               uint64_t batch_rows, const uint8_t* policy_mask);
/* update_k_steps over k HOST batches with every step's losses returned: losses[i][0..2][n] =
 * critic1 / critic2 / policy losses of step i (as pbrl_last_losses).  The H2D copy of batch
 * i+1 overlaps step i (double-buffered staging on a copy stream); returns when all k steps and
 * their loss copies are done.  Pinned host memory recommended. */
int pbrl_update_batches_losses(pbrl_pop* pop, const pbrl_batch* batches, uint32_t k,
                               uint64_t batch_rows, const uint8_t* policy_mask, double* losses);
/* update_k_steps fed by the device replay: per step i, sample_batch(..., draw_id = first+i)
 * (replay.hpp:181-204) then one update.  *ready = 0 (and nothing runs) when a source buffer
 * holds fewer than max(min_size, 1) transitions (sample_batch's nullopt). */
int pbrl_update_k(pbrl_pop* pop, uint32_t k, uint64_t sample_seed, uint64_t first_draw_id,
                  uint64_t batch_rows, uint64_t min_size, int* ready);
/* the same with td3_update_step's policy_member_mask on every step ([n] bytes; TD3) -- the
 * CEM-RL learner trains only the first half of the population (pipeline_run.hpp:322-326) */
int pbrl_update_k_masked(pbrl_pop* pop, uint32_t k, uint64_t sample_seed, uint64_t first_draw_id,
                         uint64_t batch_rows, uint64_t min_size, const uint8_t* policy_mask,
                         int* ready);
/* Per-member losses of the LAST step: critic1 / critic2 MSE (mse_loss_grads, algos.hpp:288-314)
 * and the policy loss (td3_policy_loss_grads :318-338 / sac_policy_loss_grads :643-735);
 * each [n] (TD3 policy entries are 0 for members that did not fire). */
int pbrl_last_losses(pbrl_pop* pop, double* critic1, double* critic2, double* policy);

/* ---- checkpoints: save_checkpoint / load_checkpoint (PBRLNET1, net_pop.hpp:224-304) of one
 * network (PBRL_NET_*) of the population, fp32, byte-compatible with the reference's files;
 * load requires the file's population size / extents / output activation / scale to match
 * (ConfigError otherwise, like a bad magic or truncated file).  serialize_state
 * (algos.hpp:989-1015, TD3): the reference's full-state export byte for byte. */
int pbrl_save_checkpoint(pbrl_pop* pop, int net, const char* path);
int pbrl_load_checkpoint(pbrl_pop* pop, int net, const char* path);
int pbrl_serialize_state(pbrl_pop* pop, const char* path);
/* Inverse of pbrl_serialize_state (TD3): full-trainer resume -- networks, Adam m / v / t,
 * delay_acc, steps -- from that byte layout (the reference writes it, algos.hpp:989-1015, but
 * ships no loader).  ConfigError on a truncated file or a population / shape mismatch. */
int pbrl_deserialize_state(pbrl_pop* pop, const char* path);

/* ---- action selection: act (TD3, algos.hpp:895-915) / sac_act (SAC, :918-942) for every
 * member on rows observations each, keyed by the population's member streams: obs [n][rows][ds]
 * and actions [n][rows][da] are host arrays; steps [n] key the per-member kExploreNoise streams;
 * noise_std [n] (TD3: exploration std in action-bound units, 0 = none; ignored by SAC, may be
 * NULL when deterministic). */
int pbrl_act(pbrl_pop* pop, const float* obs, uint64_t rows, const double* noise_std,
             uint64_t seed, const uint64_t* steps, int deterministic, float* actions);

/* ---- replay: ReplayBuffer (replay.hpp:28-173) held in HBM, one ring per member (per-agent) or
 * one shared ring.  Insert is the batched equivalent of push (:56-69). */
int pbrl_replay_create(pbrl_pop* pop, uint64_t capacity, int mode);
int pbrl_replay_insert(pbrl_pop* pop, const float* s, const float* a, const float* r,
                       const float* s2, const float* done, const uint32_t* member, uint64_t count);
/* ReplayBuffer::save_snapshot / load_snapshot (PBRLBUF1, replay.hpp:113-165) of ring `buffer`,
 * byte-compatible with the reference's files; load requires the same capacity / dims. */
int pbrl_replay_save_snapshot(pbrl_pop* pop, uint64_t buffer, const char* path);
int pbrl_replay_load_snapshot(pbrl_pop* pop, uint64_t buffer, const char* path);
int pbrl_replay_size(pbrl_pop* pop, uint64_t buffer, uint64_t* size);
/* sample_batch (replay.hpp:181-204) into host arrays shaped like pbrl_batch; *ready as above */
int pbrl_sample_batch(pbrl_pop* pop, uint64_t sample_seed, uint64_t draw_id, uint64_t batch_rows,
                      uint64_t min_size, float* s, float* a, float* r, float* s2, float* done,
                      int* ready);

/* ---- PBT exploit/explore (evolve.hpp:112-213).
 * pbrl_pbt_plan: ranks fitness (mean of each member's return ring, evolve.hpp:104-122) and draws
 * donors on device; fitness is [n_total] means over the WHOLE population (all shards).
 * rng_key/rng_next = the RngSequence (rng.hpp:74-95); *rng_next advances by the plan size.
 * replaced/donors receive global ids; *count = ceil(trunc * n_total) (0 when n_total < 4). */
int pbrl_pbt_plan(pbrl_pop* pop, const double* fitness, uint64_t n_total, double trunc,
                  uint64_t rng_key, uint64_t* rng_next, uint64_t* replaced, uint64_t* donors,
                  uint32_t* count);
/* Applies a plan to the local shard: copy every network of donor -> replaced (both local),
 * reset the replaced member's optimiser state (and TD3 delay_acc).  Pairs whose donor or
 * receiver is not local are skipped (the caller moves them with pbrl_export/import_member). */
int pbrl_pbt_apply(pbrl_pop* pop, const uint64_t* replaced, const uint64_t* donors, uint32_t count);
/* Full pbt_evolve_trainer for a single-shard population: plan + apply + hyper re-draw
 * (Td3Prior / SacPrior, evolve.hpp:31-73); returns the plan and updates the hypers. */
int pbrl_pbt_evolve(pbrl_pop* pop, const double* fitness, uint64_t rng_key, uint64_t* rng_next,
                    uint64_t* replaced, uint64_t* donors, uint32_t* count);
/* Member state blob for cross-device exploit copies: every network of one local member,
 * concatenated in net-id order (plus log_alpha for SAC).  dev_buf is a device pointer. */
int pbrl_member_blob_size(pbrl_pop* pop, uint64_t* floats);
int pbrl_export_member(pbrl_pop* pop, uint64_t member, float* dev_buf);
int pbrl_import_member(pbrl_pop* pop, uint64_t member, const float* dev_buf);

/* ---- snapshot publication: SnapshotMailbox / ActorSnapshot (pipeline.hpp:31-83) and the
 * actor refresh of actor_loop (pipeline.hpp:255-285), device-resident.  The learner publishes
 * its policy population (+ per-member exploration scales) into one of three device slots with a
 * stream-ordered copy (never waits for actors); an actor thread owns its own population handle
 * (same shapes, precision and member ids: make it with the learner's descriptor), adopts the
 * newest version with pbrl_actor_refresh and then acts with pbrl_act on its own handle and
 * stream, concurrently with the learner's updates.  Readers never see a half-written slot. */
typedef struct pbrl_mailbox pbrl_mailbox;
int pbrl_mailbox_create(pbrl_pop* learner, pbrl_mailbox** out);
int pbrl_mailbox_destroy(pbrl_mailbox* mb);
/* SnapshotMailbox::publish: *version = the new version (1, 2, ...); explore_std: [n] or NULL */
int pbrl_mailbox_publish(pbrl_mailbox* mb, pbrl_pop* learner, const double* explore_std,
                         uint64_t* version);
int pbrl_mailbox_version(pbrl_mailbox* mb, uint64_t* version);
/* refresh(): copy the newest snapshot into `actor` if its version changed; *version = the
 * version the actor now holds (0 = nothing published yet); explore_std: [n] or NULL */
int pbrl_actor_refresh(pbrl_pop* actor, pbrl_mailbox* mb, uint64_t* version, double* explore_std);
/* ActorSnapshot::compute_checksum of the newest snapshot (FNV-1a, pipeline.hpp:38-47) */
int pbrl_mailbox_checksum(pbrl_mailbox* mb, uint64_t* version, uint64_t* checksum);

/* ---- whole-member state copy: slice_member / set_member for states (algos.hpp:425-464,
 * :839-886).  Copies member sm of src into member dm of dst: every network, Adam m / v / t,
 * steps, streams, delay_acc (TD3) or log_alpha + its Adam state (SAC), and the hypers.  With dst
 * a fresh population of one (make_*_state(1, ...)) it is slice_member(src, sm); with src a
 * singleton it is set_member(dst, dm, single).  Shapes and algorithm must match (ShapeError). */
int pbrl_copy_member_state(pbrl_pop* dst, uint64_t dst_member, pbrl_pop* src, uint64_t src_member);

/* ---- sharded population: the PBT exchange across devices.
 * The reference is single-process; this is pbt_evolve_trainer (evolve.hpp:169-213) for a
 * population split in contiguous member blocks over `world` ranks (rank r owns global members
 * [r*n, (r+1)*n), desc.member_offset = r*n, desc.n_global = world*n).  The update step needs no
 * communication (RNG streams keyed by global id); only PBT exchanges data:
 *   1. all-gather of [ready, fitness of every local member] (doubles);
 *   2. every rank computes the identical plan on device (pbrl_pbt_plan);
 *   3. donor -> replaced copies: same-rank pairs on device, cross-rank pairs as grouped
 *      point-to-point transfers of the member blob (pbrl_export_member layout);
 *   4. optimiser / delay reset of local receivers; the hyper re-draw in lock-step on every rank
 *      (each rank draws the prior sample of every replaced member, applies its own). */
typedef struct pbrl_comm pbrl_comm;

/* host transport: one point-to-point transfer of a HOST buffer */
typedef struct {
  int peer;        /* rank */
  int is_send;     /* 1: send buf to peer, 0: receive into buf from peer */
  float* buf;
  uint64_t floats;
} pbrl_p2p_op;

/* caller-supplied host transport (e.g. gloo through torch.distributed, MPI); both callbacks
 * return 0 on success and are collective over the ranks. */
typedef struct {
  void* ctx;
  /* recv = [world][count] doubles, rank-major */
  int (*allgather_f64)(void* ctx, const double* send, uint64_t count, double* recv);
  /* all ops of this rank as one group (like ncclGroupStart / ncclGroupEnd) */
  int (*exchange)(void* ctx, const pbrl_p2p_op* ops, uint32_t n_ops);
  /* in-place sum over the ranks of buf[count] (shared-critic gradients; may be NULL when no
   * shared-critic population is attached) */
  int (*allreduce_f32)(void* ctx, float* buf, uint64_t count);
} pbrl_comm_ops;

/* NCCL transport over NVLink / NVSwitch: rank 0 calls pbrl_nccl_unique_id, the caller
 * distributes the 128 bytes, every rank calls pbrl_comm_create_nccl with its device. */
int pbrl_nccl_unique_id(void* id, size_t len);
int pbrl_comm_create_nccl(const void* id, int rank, int world, int device, pbrl_comm** out);
int pbrl_comm_create_host(const pbrl_comm_ops* ops, int rank, int world, int device,
                          pbrl_comm** out);
int pbrl_comm_destroy(pbrl_comm* comm);
/* pbt_evolve_trainer for one shard.  local_fitness: [n] means of this rank's members' return
 * rings; local_ready = every local member scored (PBTState::every_member_scored).  If any
 * rank is not ready, EVERY rank returns PBRL_E_NOT_READY (NotReadyError, evolve.hpp:113-115)
 * and nothing changes.  replaced/donors: [ceil(trunc * n_global)] global ids (the plan, same on
 * every rank); *rng_next advances like the single-shard pbrl_pbt_evolve.  The caller clears
 * the return rings of its replaced members (pbt_apply_returns_reset, evolve.hpp:149-152).
 * exchange_ms (may be NULL): [3] host wall times of (fitness all-gather, plan, copies+resets). */
int pbrl_pbt_evolve_sharded(pbrl_pop* pop, pbrl_comm* comm, const double* local_fitness,
                            int local_ready, double trunc, uint64_t rng_key, uint64_t* rng_next,
                            uint64_t* replaced, uint64_t* donors, uint32_t* count,
                            double* exchange_ms);

/* ---- shared critic across shards: the per-step critic-gradient all-reduce.
 * A PBRL_MODE_SHARED_CRITIC population sharded over `world` ranks (member_offset / n_global as
 * above) keeps an identical replica of the one critic pair on every rank; each step sums the
 * critic gradients of the local folded batches over the ranks (NCCL all-reduce, or the host
 * transport's allreduce_f32) before the critic Adam, so every replica takes the same step the
 * unsharded population would (loss scale 2 / (n_global * B), mse_loss_grads algos.hpp:288-314).
 * comm = NULL detaches.  The steps of an attached population run eagerly (no step graph). */
int pbrl_attach_comm(pbrl_pop* pop, pbrl_comm* comm);

/* ---- DvD (evolve.hpp:304-525): log-determinant diversity over behavioural embeddings.
 * pbrl_set_dvd installs dvd_policy_hook(cfg, step) for the following update calls (TD3):
 * probe [m_states][obs] doubles (DvDConfig::probe_states), lambda = dvd_lambda(step, schedule)
 * (lambda 0 or probe NULL: no hook).  On a step where some policy updates, the hook's gradient of
 * -lambda * logdet(K + jitter I) through the policies' embeddings is added to the policy
 * gradients before the policy Adam (add_scaled, optim.hpp:75-85).  A singular kernel matrix
 * fails the update with PBRL_E_DEGENERATE before the step runs. */
int pbrl_set_dvd(pbrl_pop* pop, const double* probe, uint64_t m_states, double length_scale,
                 double jitter, double lambda);
/* dvd_embed (:337-340): out [n][m_states * act] deterministic actions on the probe states */
int pbrl_dvd_embed(pbrl_pop* pop, const double* probe, uint64_t m_states, float* out);
/* dvd_loss (:411-465) on host data: emb [n][dim]; grad [n][dim] (may be NULL) */
int pbrl_dvd_loss(const double* emb, uint64_t n, uint64_t dim, double length_scale, double jitter,
                  double lambda, double* loss, double* logdet, double* grad);
int pbrl_median_pairwise_distance(const double* emb, uint64_t n, uint64_t dim, double* out);
int pbrl_dvd_lambda(uint64_t step, double start, double end, uint64_t horizon, double* out);

/* ---- CEM (evolve.hpp:221-297) over the flat policy vectors of a TD3 population, on device.
 * pbrl_cem_create: cem_init(mean, init_var) with mean [P] doubles, or NULL for
 * flatten_member(policy, 0) as run_training does (pipeline_run.hpp:159-162).
 * pbrl_cem_resample: cem_resample (pipeline_run.hpp:148-158) -- cem_sample(cem, n, rng) with
 * the RngSequence (rng_key, *rng_next), every candidate written into its member's policy, targets
 * set to the policies, policy Adam state reset; the candidates are kept for the refit.
 * pbrl_cem_update: cem_update(cem, candidates, scores[n]) -- elites by stable score order.
 * Single-shard populations only. */
typedef struct pbrl_cem pbrl_cem;
int pbrl_cem_create(pbrl_pop* pop, const double* mean, double init_var, pbrl_cem** out);
int pbrl_cem_destroy(pbrl_cem* cem);
/* CEMState fields (defaults 1e-2 / 1e-3 / 0.999 / 0.5) */
int pbrl_cem_set_params(pbrl_cem* cem, double noise, double noise_final, double noise_decay,
                        double elite_fraction);
int pbrl_cem_get(pbrl_cem* cem, double* mean, double* var, double* noise);
int pbrl_cem_resample(pbrl_cem* cem, uint64_t rng_key, uint64_t* rng_next);
int pbrl_cem_candidates(pbrl_cem* cem, double* out /* [n][P] */);
int pbrl_cem_update(pbrl_cem* cem, const double* scores, uint64_t count);

/* ---- synthetic inputs: make_synthetic_batches (bench.hpp:69-93) generated on the device.
 * out: count device batches; each field is a device pointer to [count][n][b][dim] floats laid out
 * contiguously (out->s holds all count batches).  pop may be NULL (current device). */
int pbrl_synthetic_batches_device(pbrl_pop* pop, uint64_t count, uint64_t n, uint64_t b,
                                  uint64_t obs_dim, uint64_t act_dim, uint64_t seed,
                                  const pbrl_batch* out);

/* ---- diagnostics: the device ports of glibc tanhf (0), expf (1), log1pf (2) over a device
 * array; used by the numerics tests to prove bit-equality with the host libm. */
int pbrl_selftest_libm(int fn, const float* dev_in, float* dev_out, uint64_t count);

/* C[g](i,j) = sum_k A[g](i,k) B[g](k,j) on the tcgen05 path (TF32), fp32 device operands.
 * a_mn: A stored [g][K][M] (else [g][M][K]); b_mn: B stored [g][K][N] (else [g][N][K]). */
int pbrl_selftest_tc_gemm(int a_mn, int b_mn, int M, int N, int K, int groups, const float* A,
                          long long a_ld, long long a_gs, const float* B, long long b_ld,
                          long long b_gs, float* C, long long c_ld, long long c_gs);
/* The same on the BF16 path (tcgen05 kind::f16): A and B are bf16 device arrays (uint16 bit
 * patterns), C is fp32. */
int pbrl_selftest_tc_gemm_bf16(int a_mn, int b_mn, int M, int N, int K, int groups,
                               const void* A, long long a_ld, long long a_gs, const void* B,
                               long long b_ld, long long b_gs, float* C, long long c_ld,
                               long long c_gs);

/* Phase timeline of the tcgen05 GEMM launches recorded since process start when the environment
 * variable PBRL_TC_TRACE is set (diagnostics only; off by default).  Copies up to max_launches
 * launches: stamps[launch][160][64] (globaltimer ns per CTA: entry, setup, per tile producer /
 * MMA start / MMA commit / epilogue start / epilogue end, drain, exit) and meta[launch][10]
 * (BN, A MN-major, B MN-major, fused n_out, M, N, K, groups, epilogue, 0); *n = launches copied. */
int pbrl_debug_tc_trace(uint64_t* stamps, int* meta, int max_launches, int* n);

/* ---- observability */
int pbrl_launch_count(pbrl_pop* pop, uint64_t* launches); /* kernels launched (cf. kernel_invocations, pop_tensor.hpp:21-28) */
int pbrl_synchronize(pbrl_pop* pop);
/* The cudaStream_t every kernel of this population is launched on (for event timing). */
int pbrl_get_stream(pbrl_pop* pop, void** stream);
/* Event-instrumented profiling: between begin and end every launch is bracketed by CUDA events
 * on the population stream; end writes a JSON summary per kernel class
 * {"steps": S, "classes": {"gemm_fwd": {"launches", "ms", "flops", "bytes"}, ...}} where flops /
 * bytes are the algorithmic work (fired members only for gated kernels). */
int pbrl_profile_begin(pbrl_pop* pop);
int pbrl_profile_end(pbrl_pop* pop, char* json, size_t len);
/* Bytes of fp32 state this population keeps in HBM (params, targets, moments, replay). */
int pbrl_device_bytes(pbrl_pop* pop, uint64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif
