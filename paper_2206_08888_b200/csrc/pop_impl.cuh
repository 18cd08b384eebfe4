// Population object (host side of the C ABI).
#pragma once

#include <functional>
#include <unordered_map>

#include <atomic>
#include <string>
#include <vector>

#include "pop.cuh"

namespace pbrl {

extern std::atomic<uint64_t> g_launches;

// Owning device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t count = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), count(o.count) {
    o.p = nullptr;
    o.count = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      count = o.count;
      o.p = nullptr;
      o.count = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    count = 0;
  }
  void alloc(size_t c) {
    if (c <= count && p) return;
    release();
    if (c == 0) return;
    cudaError_t e = cudaMalloc(&p, c * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      throw Error(PBRL_E_RESOURCE, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    }
    count = c;
  }
  void zero(cudaStream_t s) {
    if (p) CUDA_CHECK(cudaMemsetAsync(p, 0, count * sizeof(T), s));
  }
  void upload(const T* h, size_t c, cudaStream_t s) {
    CUDA_CHECK(cudaMemcpyAsync(p, h, c * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// Per-step activations and cotangents for a batch of B rows (grown on demand).
struct Scratch {
  int B = 0;
  DBuf<float> in_sa, in_s2a, sa_pi, r, d, y, tq_out, q, dq, qpi, gq, pt, ga, head, gtop;
  DBuf<float> in_s;  // policy input [s | 1 | pad] (row stride lsp; the ones column as in_sa's)
  DBuf<float> bs[2], ba[2], br[2], bs2[2], bd[2];  // host batches staged (double-buffered)
  std::vector<DBuf<float>> tp_h, ph, pdh, tq_h, ch, dh, qh, qdh;
  DBuf<float> x, th, ls, eps, logp, logp2, lw, tnoise;
  DBuf<uint8_t> clamped;
};

// Action-selection scratch (act / sac_act): rows observations per member.
struct ActScratch {
  int rows = 0;
  DBuf<float> obs, in, out, act;       // obs [n][rows][ds] fp32, in: policy-input block
  std::vector<DBuf<float>> h;          // hidden activations (+ mask bits)
  DBuf<uint64_t> steps;
  DBuf<double> noise;
};

// HBM-resident replay rings (ReplayBuffer, replay.hpp:28-173).
struct Replay {
  int mode = PBRL_REPLAY_PER_AGENT;
  uint64_t cap = 0;
  int nbuf = 0, rw = 0;
  DBuf<float> ring;             // [nbuf][cap][rw]
  DBuf<uint64_t> sizes;         // [nbuf] min(inserts, cap)
  std::vector<uint64_t> inserts;
  std::vector<uint32_t> member;  // [nbuf][cap] Transition::member per slot (host metadata)
  DBuf<float> stage_rows;
  DBuf<uint64_t> stage_dst;
};

// Event-instrumented profiling of one update program (bench.py's roofline numbers): every
// launch is bracketed by events on the population stream and tagged with its algorithmic work.
enum ProfClass { PC_GEMM_FWD = 0, PC_GEMM_DX, PC_GEMM_DW, PC_ADAM, PC_ELEM, PC_GATHER, PC_COUNT };
struct ProfRec {
  int cls;
  double flops, bytes;
  int gated;  // work scales with the number of fired members
  int step;
  cudaEvent_t a, b;
  double gbytes;  // extra bytes that scale with the fired fraction (gated Polyak)
};

// A [groups][rows][ld] activation block; by_member: shared by the critics of one member.
struct Mat {
  const float* p = nullptr;
  long long gs = 0;
  long long ld = 0;
  int by_member = 0;
  // TF32 mode, hidden activations: ReLU mask bits [groups][rows][mld] next to the activations
  uint32_t* mask = nullptr;
  long long mgs = 0, mld = 0;
  // input blocks: column `ones_col` (a padding column) holds 1.0 in every row, so the dW product
  // of the first layer also yields the bias gradient as its extra row (0: no such column)
  int ones_col = 0;
};

inline int pad4(int x) { return (x + 3) / 4 * 4; }

void set_last_error(const std::string& m);  // pbrl_last_error() of the calling thread

struct StepGraph {
  int B = 0;
  bool masked = false;
  bool dvd = false;  // the DvD gradient add sits in the policy half
  bool fire = false;  // TD3: the policy half captured unconditionally (host mirror: some fire)
  cudaGraphExec_t exec = nullptr;
  size_t nodes = 0;       // kernel nodes outside conditional bodies
  size_t cond_nodes = 0;  // kernel nodes inside the policy-half conditional bodies
  bool stage_ev = false;  // records ev_stage_free once the step has read its packed batch
  bool hist = false;      // k_td3_step_begin writes the loss history
};

struct Pop;
// Critic operations of a shared-critic population see it as ONE member whose batch has n*B
// rows (a pure reinterpretation of the [n][B][...] activation blocks); inside the scope the
// population's member count reads 1, so group -> member maps and per-member hyper indices
// (critic_lr[0], tau[0]) follow the reference's shared-mode vectors (algos.hpp:366, :407).
struct CriticFold {
  Pop& p;
  int n0, B;
  CriticFold(Pop& pop, int b);
  ~CriticFold();
};
// the population's own member count back inside a CriticFold scope (policy work between critic
// launches)
struct CriticUnfold {
  Pop& p;
  int n1;
  explicit CriticUnfold(Pop& pop);
  ~CriticUnfold();
};

struct Pop {
  int algo = PBRL_ALGO_TD3, precision = PBRL_PREC_FFMA32, device = 0;
  int n = 0, ds = 0, da = 0;
  uint64_t member_offset = 0, n_global = 0;
  // PopMode::kSharedCritic (algos.hpp:197): ONE critic pair serves every policy; its batch is
  // the population folded into rows (critic_forward, algos.hpp:219-233).  ncrit = critic
  // members (n, or 1); critic2 rows start at ncrit in the critic arenas.
  bool shared = false;
  int ncrit = 0;
  int n_local = 0;  // the population's member count (n reads 1 inside a CriticFold)
  int net_members(int net) const {
    return (net == PBRL_NET_POLICY || net == PBRL_NET_POLICY_TARGET) ? n : ncrit;
  }
  int crows(int B) const { return shared ? n * B : B; }  // rows of one critic group
  // host copy of the [3][n] losses: a folded critic step writes critic2's loss at index 1;
  // report it at n (critic1 / critic2 / policy rows as in independent mode)
  void shared_losses_layout(double* h) const {
    if (shared && n > 1) {
      h[n] = h[1];
      h[1] = 0.0;
    }
  }
  // dq / loss scale rows of the critic MSE (mse_loss_grads): the folded batch of the whole
  // population, across shards when the critic is shared over ranks
  double mse_rows(int B) const {
    return shared ? static_cast<double>(n_global) * B : static_cast<double>(B);
  }
  float bound = 1.0f;
  uint64_t seed = 0;
  std::vector<size_t> hidden;
  NetShape pol, cri;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // capture stream of conditional graph bodies
  size_t cond_body_nodes = 0;

  DBuf<float> pol_p, pol_t, pol_m, pol_v, pol_g;
  DBuf<float> cri_p, cri_t, cri_m, cri_v, cri_g;
  // BF16 mode: bf16 copies of the online / target weights (the tensor-core B operands), kept in
  // step by the fused Adam + Polyak kernel and refreshed after any other weight write
  DBuf<__nv_bfloat16> pol_p16, pol_t16, cri_p16, cri_t16;
  bool weights_dirty = true;
  bool ones_dirty = true;  // the critic-input ones column must be (re)written
  void ensure_ones();
  void refresh_shadows();
  const void* wop(const float* W) const;  // tensor-core operand copy of master weights W
  DBuf<int64_t> t_pol, t_cri, t_alpha;
  DBuf<uint64_t> steps, streams, key_a, key_b;
  DBuf<int> fire;
  DBuf<double> delay_acc, losses;
  // per-step losses of an update_batches call, kept on the device and read back in blocks of
  // kLossHist steps (one D2H per block instead of one per step)
  static constexpr uint32_t kLossHist = 64;
  DBuf<double> loss_hist;
  // TD3: k_td3_step_begin of step i+1 copies step i's losses into the history (no copy launch
  // between the step graphs); hist_base = steps[] at the start of the call
  bool hist_on = false;
  DBuf<uint64_t> hist_base;
  DBuf<float> log_alpha, alpha_m, alpha_v;
  DBuf<uint8_t> mask_buf;

  // hyperparameters: host doubles (reference Td3Hyper / SacHyper) + device casts
  std::vector<std::string> fields;
  std::vector<std::vector<double>> hyper;
  DBuf<float> h_f0, h_f1, h_f2, h_f3, h_f4, h_f5, h_f6, h_f7;
  DBuf<double> h_d0;

  DBuf<float> corr1, corr2;
  size_t corr_len = 0;
  uint64_t t_bound = 0;  // upper bound of every Adam step counter

  Scratch S;
  ActScratch AS;
  void act(const float* obs, uint64_t rows, const double* noise_std, uint64_t seed,
           const uint64_t* steps, int deterministic, float* actions);
  Replay* replay = nullptr;

  bool prof_on = false;
  int prof_step = 0;
  std::vector<ProfRec> prof;
  std::vector<int> prof_fired;  // fired members per profiled step (TD3)
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t prof_event();
  void prof_begin(cudaEvent_t* a);
  void prof_end(cudaEvent_t a, int cls, double flops, double bytes, int gated);
  void prof_step_done();
  std::string prof_report();
  void prof_add_gated_bytes(double bytes);
  // true when the latest kernel on the stream wrote parameters (Adam, PBT copies, init): the
  // next tcgen05 launch must not read its weight operand before the PDL wait
  //
  // PDL window per capture stream: kernels with PDL_ENTRY wait for their predecessor and then
  // trigger; the tcgen05 kernels trigger early (before their wait), so their successor can start
  // while kernels several launches back still run.  A successor may read weights before its
  // wait (b_prefetch) only if no kernel from the last wait-then-trigger launch on (inclusive)
  // wrote weights.  A stream's first kernel after a fork has a full dependency (window empty).
  std::unordered_map<cudaStream_t, bool> wwin;  // true: a weight write may still be in flight
  bool next_early_trigger = false;
  bool tc_prefetch_ok() {
    auto it = wwin.find(stream);
    const bool ok = it != wwin.end() && !it->second;
    next_early_trigger = true;
    return ok;
  }
  void weights_written_outside() {  // PBT copies, set_member, init: every window dirty
    for (auto& kv : wwin) kv.second = true;
    wwin[stream] = true;
  }
  void fork_window(cudaStream_t s) { wwin[s] = false; }

  template <typename F>
  void timed(int cls, double flops, double bytes, int gated, F&& f) {
    cudaEvent_t a = nullptr;
    prof_begin(&a);
    f();
    count_launch(1);
    prof_end(a, cls, flops, bytes, gated);
    const bool writes = cls == PC_ADAM;
    bool& w = wwin.try_emplace(stream, true).first->second;
    w = next_early_trigger ? (w || writes) : writes;
    next_early_trigger = false;
  }

  // algorithmic HBM bytes of one batch pack / replay gather: the transition rows read (s, a, r,
  // s2, done: 2 ds + da + 2 floats) and the operand blocks written (critic input [s|a], target
  // critic input s2, policy-loss critic input s, policy input s, r, done)
  double pack_bytes(int B) const {
    const double rows = static_cast<double>(n) * B;
    return rows * (4.0 * (2 * ds + da + 2) + aeb() * (2.0 * ds + da + ds + ds) + 8.0);
  }

  // actor side of a snapshot mailbox (pbrl_actor_refresh): the version held and its scales
  uint64_t snap_version = 0;
  std::vector<double> snap_explore;

  // PBT scratch
  DBuf<double> pbt_fit;
  DBuf<uint64_t> pbt_order, pbt_rep, pbt_don, pbt_src, pbt_dst;
  DBuf<float> pbt_blob;  // staging of cross-shard exploit copies (pbrl_pbt_evolve_sharded)

  explicit Pop(const pbrl_pop_desc& d);
  ~Pop();

  void sync();
  int field_index(const std::string& f) const;
  void validate_hyper() const;
  void upload_hyper();
  void ensure_corr(size_t need);
  void ensure_scratch(int B);
  void count_launch(uint64_t k) {
    if (!capturing) g_launches.fetch_add(k, std::memory_order_relaxed);
  }
  bool use_tc() const { return precision == PBRL_PREC_TF32 || precision == PBRL_PREC_BF16; }
  // BF16 mode: activations (critic / policy inputs, hidden activations and their cotangents)
  // are stored as bf16; parameters, optimizer state, outputs and losses stay fp32
  bool act16() const { return precision == PBRL_PREC_BF16; }
  int aeb() const { return act16() ? 2 : 4; }
  int padl(int x) const { return act16() ? (x + 7) / 8 * 8 : pad4(x); }
  // element offset into an activation buffer
  float* aoff(const float* p, long long elems) const {
    return reinterpret_cast<float*>(const_cast<char*>(reinterpret_cast<const char*>(p)) +
                                    elems * aeb());
  }
  int lsa = 0;  // padded row stride of the critic-input blocks [s | a]
  int lsp = 0;  // padded row stride of the policy-input block [s | 1]
  Mat policy_input(int B) const {  // the policy's x0: s, with the ones column in TC modes
    Mat m{S.in_s.p, static_cast<long long>(B) * lsp, lsp, 0};
    if (use_tc() && lsp > ds) m.ones_col = ds;
    return m;
  }
  bool use_graphs = true, capturing = false;
  std::vector<StepGraph> graphs;
  void invalidate_graphs();
  void run_program(int B, const uint8_t* d_mask);
  Mat hid(std::vector<DBuf<float>>& v, int l, int B, const NetShape& sh, int by_member);

  void gemm_fwd(const NetShape& sh, const float* W, int l, int groups, int B, Mat X, float* Y,
                long long y_gs, long long y_ld, int epi, const int* active = nullptr,
                float* C2 = nullptr, long long c2_gs = 0, long long c2_ld = 0,
                bool noise = false, const Mat* ymask = nullptr, bool y_act = true);
  void gemm_dx(const NetShape& sh, const float* W, int l, int groups, int B, Mat G, Mat aux,
               float* DX, long long dx_gs, long long dx_ld, int epi, int col0, int ncols,
               const int* active, float scale);
  void gemm_dw(const NetShape& sh, float* Gr, int l, int groups, int B, Mat X, Mat G,
               const int* active, bool bias_done = false, int max_ctas = 0);
  // graph mode, tensor-core modes: the last two weight-gradient products of a 2-hidden-layer
  // backward on two graph branches with split persistent grids (PBRL_NO_DWFORK=1 disables)
  static constexpr int kDwSideCtas = 40;
  // [0]: the step graph, [1]: conditional bodies (a stream that joined one capture stays in it
  // until that capture ends, so each capture graph forks onto its own stream)
  cudaStream_t side3[2] = {nullptr, nullptr};
  cudaEvent_t ev_f3[2] = {nullptr, nullptr}, ev_j3[2] = {nullptr, nullptr};
  bool in_cond_body = false;  // capturing a conditional body (its own capture graph)
  int cta_cap = 0;  // > 0: persistent tcgen05 launches use at most this many CTAs
  // TD3 graph mode: the policy forward on a branch beside the critic Adam (PBRL_POL_FORK = its
  // SMs, 0 disables)
  std::function<void()> pre_adam;
  bool pol_fwd_done = false;
  cudaStream_t side6 = nullptr;
  cudaEvent_t ev_f6 = nullptr, ev_j6 = nullptr;
  int pol_fork_ctas(int B) const {
    static const int v = std::getenv("PBRL_POL_FORK") ? std::atoi(std::getenv("PBRL_POL_FORK")) : 40;
    // only a fused (2-hidden-layer) policy forward of a few tiles fits beside the Adam; a deep /
    // wide one (config E: thousands of tiles) on 40 SMs would outlast it
    const long long tiles = static_cast<long long>(n_local) * ((B + 127) / 128);
    return pol.depth == 3 && tiles <= 2LL * 148 ? v : 0;
  }
  // SMs of the online-critic forward branch while the target chain runs beside it (0: no split;
  // PBRL_FWD_SPLIT overrides).  Only for the fused two-hidden-layer forward with a partial second
  // wave of tiles (config D: 320 on 148 SMs): under one wave (config C: 128) each branch would
  // just get fewer SMs than tiles (measured 112k -> 110k), and with thousands of tiles (config E)
  // every launch fills the machine anyway (28.9k -> 25.5k).
  int fwd_split(int B) const {
    static const int v = std::getenv("PBRL_FWD_SPLIT") ? std::atoi(std::getenv("PBRL_FWD_SPLIT")) : 64;
    const long long tiles = 2LL * (shared ? 1 : n) * ((crows(B) + 127) / 128);
    return cri.depth == 3 && tiles > 148 && tiles <= 3LL * 148 ? v : 0;
  }
  bool dw_fork_ok() const {
    static const bool off = std::getenv("PBRL_NO_DWFORK") != nullptr;
    return capturing && use_tc() && !off;
  }
  void mlp_forward(const NetShape& sh, const float* W, int groups, int B, Mat x,
                   std::vector<DBuf<float>>& hs, float* out, long long out_gs, long long out_ld,
                   int last_epi, const int* active = nullptr, float* C2 = nullptr,
                   long long c2_gs = 0, long long c2_ld = 0, bool noise = false,
                   bool keep_hidden = true, bool out_act = false);
  bool mlp_forward2(const NetShape& sh, const float* W, int groups, int B, Mat x,
                    std::vector<DBuf<float>>& hs, float* out, long long out_gs, long long out_ld,
                    int last_epi, const int* active, float* C2, long long c2_gs, long long c2_ld,
                    bool noise, bool keep_hidden, bool out_act);
  bool fwd2_off = false;  // PBRL_NO_FWD2=1: per-layer launches instead (diagnostics)
  bool gemm_fwd_fused(const NetShape& sh, const float* W, int l, int groups, int B, Mat X, Mat H,
                      bool keep_hidden, float* Y, long long y_gs, long long y_ld, int out_epi,
                      const int* active, float* C2, long long c2_gs, long long c2_ld, bool noise,
                      bool out_act);
  void mlp_backward(const NetShape& sh, const float* W, float* Gr, int groups, int B, Mat G,
                    Mat x0, std::vector<DBuf<float>>& hs, std::vector<DBuf<float>>& dhs,
                    const int* active, const OutBwdArgs* top = nullptr);
  void critic_dx_to_action(int groups, int B, Mat G, std::vector<DBuf<float>>& hs,
                           std::vector<DBuf<float>>& dhs, float* out, long long out_ld, int epi,
                           Mat aux, float scale, const int* active,
                           const OutBwdArgs* top = nullptr);
  void critic_forward(int B);
  bool gemm_dx_to_action(int groups, int B, Mat G, Mat mask, float* out, long long out_ld, int epi,
                         Mat aux, float scale, const int* active);
  void critic_update(int B, const int* polyak_gate, bool forward_done = false);
  bool td_target_fused(int B) const;
  // DvD policy-gradient hook (dvd_policy_hook, evolve.hpp:507-525) for the following update
  // calls: probe block, embeddings, tanh values, cotangents, the hook's gradient arena
  struct Dvd {
    bool on = false;
    int ms = 0, ldx = 0;
    double ls = 1.0, jitter = 1e-6, lambda = 0.0;
    std::vector<double> probe;
    DBuf<float> obs, x, emb, t, gemb, gz, grad;
    std::vector<DBuf<float>> h, dh;
  } dvd;
  void set_dvd(const double* probe, uint64_t m_states, double length_scale, double jitter,
               double lambda);
  void dvd_forward();
  void dvd_prepass();
  // shared critic over shards: in-place sum of the critic gradient arena across ranks before
  // the critic Adam (set by pbrl_attach_comm; the step then runs eagerly)
  std::function<void(float*, size_t, cudaStream_t)> comm_reduce;
  DBuf<float> flag_f;  // the "some member fires" flag as a float for that all-reduce
  bool graphs_allowed = true;  // PBRL_NO_GRAPH unset
  cudaStream_t side2 = nullptr;  // parallel graph branch (critic forward)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void td3_step(int B, const uint8_t* d_mask);
  void td3_policy_half(int B);
  void td3_policy_forward(int B);
  template <typename F>
  void capture_if(cudaGraphConditionalHandle h, cudaStream_t& cap, F&& body);
  size_t cond_nodes = 0;
  // host mirror of the TD3 fire accumulator (k_td3_step_begin's double arithmetic), used only to
  // count the kernels a replayed graph actually runs (the conditional policy half)
  std::vector<double> delay_host;
  const uint8_t* host_mask = nullptr;
  bool host_fires();
  bool eager_fires = true;  // this step's host-mirror fire decision (eager replay)
  // capturing the fire-step graph: the policy half is captured inline (kernels gated per member
  // by the device fire mask) instead of inside the conditional IF node
  bool cap_fire = false;
  bool fire_graphs() const {
    static const bool off = std::getenv("PBRL_NO_FIRE_GRAPH") != nullptr;
    return !off;
  }
  // the non-fire step graph: no policy half at all, and k_td3_step_begin raises a flag in mapped
  // host memory if some member fires after all (the host mirror diverged: the next call fails
  // loudly).  PBRL_COND_GRAPH=1 keeps the device-decided IF node instead (its evaluation after
  // the critic Adam costs ~9 us per non-fire step).
  bool cond_graph() const {
    static const bool on = std::getenv("PBRL_COND_GRAPH") != nullptr;
    return on || !fire_graphs();
  }
  int* guard_h = nullptr;  // mapped pinned host flag
  int* guard_d = nullptr;  // its device alias
  void check_guard();
  void sac_step(int B);
  void step(int B, const uint8_t* d_mask);
  void update_batches(const pbrl_batch* batches, uint32_t k, uint64_t rows,
                      const uint8_t* policy_mask, bool device_ptrs, double* losses_out = nullptr);
  // host-batch staging: H2D copies on their own stream, double-buffered, so the copy of batch
  // i+1 overlaps the update step of batch i
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  bool slot_used[2] = {false, false};
  // TD3 step graphs record ev_stage_free (an external event-record node on a branch) right
  // before the step's last Adam, the point after which nothing in the step reads the packed
  // batch (in_sa / in_s2a / in_s / sa_pi's state part / r / d); inside one update_batches call
  // the next batch's pack then runs on pstream beside that Adam instead of after the graph
  cudaStream_t pstream = nullptr, side_sf = nullptr;
  cudaEvent_t ev_stage_free = nullptr, ev_packed = nullptr, ev_sf_fork = nullptr,
              ev_sf_join = nullptr;
  int stage_mark = 0;  // capture: 1 = mark before the critic Adam, 2 = before the policy Adam
  bool stage_joined = true;  // the marker branch has been joined back
  bool stage_ev_captured = false;  // the graph being captured records ev_stage_free
  bool last_step_stage_ev = false;  // the last step() launched a graph recording ev_stage_free
  bool pack_overlap_ok() const;
  void mark_stage_free();
  void join_stage_free();

  // helpers for member-level access
  float* net_row(int net, uint64_t member);
  const NetShape& net_shape(int net) const;
};

// CEM search distribution over flat policy vectors (CEMState, evolve.hpp:221-297), resident on
// the population's device; the last sampled candidates are kept (double) for the refit
struct Cem {
  Pop* pop;
  size_t dim = 0;
  DBuf<double> mean, var, cand;
  DBuf<uint64_t> order_d;
  double noise = 1e-2, noise_init = 1e-2, noise_final = 1e-3, noise_decay = 0.999;
  double elite_fraction = 0.5;
  bool sampled = false;
  Cem(Pop* p, const double* mean0, double init_var);
  void resample(uint64_t key, uint64_t* next);
  void update(const double* scores, uint64_t count);
};

int dvd_loss_host(const double* emb, uint64_t n, uint64_t dim, double length_scale, double jitter,
                  double lambda, double* loss, double* logdet, double* grad);
double median_pairwise_distance_host(const double* emb, uint64_t n, uint64_t dim);
void launch_add_into(float* acc, const float* other, size_t count, cudaStream_t s);
void launch_flag_convert(int* flag, float* flag_f, int to_float, cudaStream_t s);

}  // namespace pbrl
