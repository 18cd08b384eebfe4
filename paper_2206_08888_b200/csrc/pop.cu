// Population object, device arena and the TD3 / SAC update-step programs.
//
// Device layout (HBM, fp32 master state):
//   policy, policy_target      [n][stride_p]          (TD3; SAC has no policy target)
//   critics, critic targets    [2][n][stride_c]       (critic1 rows 0..n-1, critic2 rows n..2n-1)
//   Adam m / v                 same shapes as the online arenas; t per (network, member)
//   gradients                  same shapes (FFMA32 mode); consumed by the fused Adam kernel
// Each member row holds its parameters in flatten_member order (net_pop.hpp:162-173), so
// get/set_member and PBT copies are single contiguous row copies.
#include "pop_impl.cuh"
#include "tc_gemm.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace pbrl {

float host_logf(float x) { return std::log(x); }

void NetShape::make(const std::vector<size_t>& d, int act, float scale) {
  depth = static_cast<int>(d.size()) - 1;
  if (depth < 1 || depth > kMaxLayers) PBRL_THROW(PBRL_E_CONFIG, "network depth out of range");
  out_act = act;
  out_scale = scale;
  size_t at = 0;
  for (int i = 0; i <= depth; ++i) dims[i] = static_cast<int>(d[i]);
  for (int l = 0; l < depth; ++l) {
    woff[l] = at;
    at += d[l] * d[l + 1];
    boff[l] = at;
    at += d[l + 1];
  }
  P = at;
  stride = (P + 63) / 64 * 64;
}

int NetShape::max_hidden() const {
  int h = 1;
  for (int l = 1; l < depth; ++l) h = std::max(h, dims[l]);
  return h;
}

// ------------------------------------------------------------------ construction
Pop::Pop(const pbrl_pop_desc& d) {
  if (d.algo != PBRL_ALGO_TD3 && d.algo != PBRL_ALGO_SAC) PBRL_THROW(PBRL_E_CONFIG, "unknown algo");
  if (d.n < 1) PBRL_THROW(PBRL_E_CONFIG, "population size must be >= 1");
  if (d.obs_dim < 1 || d.act_dim < 1) PBRL_THROW(PBRL_E_CONFIG, "obs_dim/act_dim must be >= 1");
  if (d.n_hidden > kMaxLayers - 1) PBRL_THROW(PBRL_E_CONFIG, "too many hidden layers");
  if (d.precision != PBRL_PREC_FFMA32 && d.precision != PBRL_PREC_TF32 &&
      d.precision != PBRL_PREC_BF16)
    PBRL_THROW(PBRL_E_CONFIG, "unknown precision mode");
  algo = d.algo;
  precision = d.precision;
  device = d.device;
  n = static_cast<int>(d.n);
  ds = static_cast<int>(d.obs_dim);
  da = static_cast<int>(d.act_dim);
  member_offset = d.member_offset;
  n_global = d.n_global ? d.n_global : d.n;
  if (d.mode != PBRL_MODE_INDEPENDENT && d.mode != PBRL_MODE_SHARED_CRITIC)
    PBRL_THROW(PBRL_E_CONFIG, "unknown population mode");
  shared = d.mode == PBRL_MODE_SHARED_CRITIC;
  ncrit = shared ? 1 : n;
  n_local = n;
  bound = static_cast<float>(d.action_bound);
  seed = d.seed;
  for (uint32_t i = 0; i < d.n_hidden; ++i) {
    if (d.hidden[i] < 1) PBRL_THROW(PBRL_E_CONFIG, "hidden widths must be >= 1");
    hidden.push_back(d.hidden[i]);
  }
  CUDA_CHECK(cudaSetDevice(device));
  CUDA_CHECK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  tc_trace_init();
  use_graphs = graphs_allowed = std::getenv("PBRL_NO_GRAPH") == nullptr;  // eager (ncu profiles)
  fwd2_off = std::getenv("PBRL_NO_FWD2") != nullptr;

  std::vector<size_t> pd{static_cast<size_t>(ds)};
  pd.insert(pd.end(), hidden.begin(), hidden.end());
  pd.push_back(static_cast<size_t>(algo == PBRL_ALGO_TD3 ? da : 2 * da));
  pol.make(pd, algo == PBRL_ALGO_TD3 ? ACT_TANH : ACT_NONE, algo == PBRL_ALGO_TD3 ? bound : 1.0f);
  std::vector<size_t> qd{static_cast<size_t>(ds + da)};
  qd.insert(qd.end(), hidden.begin(), hidden.end());
  qd.push_back(1);
  cri.make(qd, ACT_NONE, 1.0f);

  const size_t np = static_cast<size_t>(n) * pol.stride;
  const size_t nc = 2 * static_cast<size_t>(ncrit) * cri.stride;
  pol_p.alloc(np);
  pol_m.alloc(np);
  pol_v.alloc(np);
  pol_g.alloc(np);
  if (algo == PBRL_ALGO_TD3) pol_t.alloc(np);
  cri_p.alloc(nc);
  cri_t.alloc(nc);
  cri_m.alloc(nc);
  cri_v.alloc(nc);
  cri_g.alloc(nc);
  t_pol.alloc(n);
  t_cri.alloc(2 * ncrit);
  steps.alloc(n);
  streams.alloc(n);
  fire.alloc(n + 1);  // fire[n]: "some member fires" (shared critic's target Polyak gate)
  delay_acc.alloc(n);
  key_a.alloc(n);
  key_b.alloc(n);
  losses.alloc(3 * n);
  if (algo == PBRL_ALGO_SAC) {
    log_alpha.alloc(n);
    alpha_m.alloc(n);
    alpha_v.alloc(n);
    t_alpha.alloc(n);
  }
  for (auto* b : {&pol_p, &pol_m, &pol_v, &pol_g, &pol_t, &cri_p, &cri_t, &cri_m, &cri_v, &cri_g,
                  &log_alpha, &alpha_m, &alpha_v})
    b->zero(stream);
  t_pol.zero(stream);
  t_cri.zero(stream);
  steps.zero(stream);
  fire.zero(stream);
  delay_acc.zero(stream);
  losses.zero(stream);
  t_alpha.zero(stream);
  {
    std::vector<uint64_t> sv(n);
    for (int i = 0; i < n; ++i) sv[i] = member_offset + static_cast<uint64_t>(i);
    streams.upload(sv.data(), n, stream);
  }
  // make_td3_state / make_sac_state seeds (algos.hpp:198-200, :507-509)
  const uint64_t s_pol = mix64(seed ^ (algo == PBRL_ALGO_TD3 ? 0xA1 : 0xD4));
  const uint64_t s_c1 = mix64(seed ^ (algo == PBRL_ALGO_TD3 ? 0xB2 : 0xE5));
  const uint64_t s_c2 = mix64(seed ^ (algo == PBRL_ALGO_TD3 ? 0xC3 : 0xF6));
  launch_init_net(pol, pol_p.p, n, member_offset, s_pol, stream);
  // the shared critic is critic member 0 on every shard (init_pop_mlp(1, ...), algos.hpp:199)
  const uint64_t c_off = shared ? 0 : member_offset;
  launch_init_net(cri, cri_p.p, ncrit, c_off, s_c1, stream);
  launch_init_net(cri, cri_p.p + static_cast<size_t>(ncrit) * cri.stride, ncrit, c_off, s_c2,
                  stream);
  count_launch(3 * pol.depth);
  if (algo == PBRL_ALGO_TD3)
    CUDA_CHECK(cudaMemcpyAsync(pol_t.p, pol_p.p, np * 4, cudaMemcpyDeviceToDevice, stream));
  CUDA_CHECK(cudaMemcpyAsync(cri_t.p, cri_p.p, nc * 4, cudaMemcpyDeviceToDevice, stream));
  if (act16()) {
    pol_p16.alloc(np);
    if (algo == PBRL_ALGO_TD3) pol_t16.alloc(np);
    cri_p16.alloc(nc);
    cri_t16.alloc(nc);
  }
  weights_dirty = true;

  // hyper defaults (Td3Hyper::defaults algos.hpp:42-53, SacHyper::defaults :121-131)
  if (algo == PBRL_ALGO_TD3) {
    fields = {"critic_lr", "policy_lr", "policy_delay_ratio", "explore_std", "target_std",
              "target_clip", "gamma", "tau"};
    const double dv[] = {3e-4, 3e-4, 0.5, 0.1, 0.2, 0.5, 0.99, 0.005};
    for (int f = 0; f < 8; ++f) hyper.push_back(std::vector<double>(n, dv[f]));
  } else {
    fields = {"policy_lr", "critic_lr", "alpha_lr", "target_entropy", "reward_scale", "gamma",
              "tau"};
    const double dv[] = {3e-4, 3e-4, 3e-4, -static_cast<double>(da), 1.0, 0.99, 0.005};
    for (int f = 0; f < 7; ++f) hyper.push_back(std::vector<double>(n, dv[f]));
  }
  for (auto* b : {&h_f0, &h_f1, &h_f2, &h_f3, &h_f4, &h_f5, &h_f6, &h_f7}) b->alloc(n);
  h_d0.alloc(n);
  upload_hyper();
  ensure_corr(1024);
  sync();
}

CriticFold::CriticFold(Pop& pop, int b) : p(pop), n0(pop.n), B(pop.crows(b)) {
  if (p.shared) p.n = 1;
}
CriticFold::~CriticFold() { p.n = n0; }
CriticUnfold::CriticUnfold(Pop& pop) : p(pop), n1(pop.n) {
  if (p.shared) p.n = p.n_local;
}
CriticUnfold::~CriticUnfold() { p.n = n1; }

Pop::~Pop() {
  invalidate_graphs();
  for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
    if (side) cudaStreamDestroy(side);
    if (side2) cudaStreamDestroy(side2);
    if (side6) cudaStreamDestroy(side6);
    if (guard_h) cudaFreeHost(guard_h);
    if (ev_f6) cudaEventDestroy(ev_f6);
    if (ev_j6) cudaEventDestroy(ev_j6);
    for (int i = 0; i < 2; ++i) {
      if (side3[i]) cudaStreamDestroy(side3[i]);
      if (ev_f3[i]) cudaEventDestroy(ev_f3[i]);
      if (ev_j3[i]) cudaEventDestroy(ev_j3[i]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (cstream) cudaStreamDestroy(cstream);
    if (pstream) cudaStreamDestroy(pstream);
    if (side_sf) cudaStreamDestroy(side_sf);
    for (cudaEvent_t e : {ev_stage_free, ev_packed, ev_sf_fork, ev_sf_join})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {ev_copied[0], ev_copied[1], ev_free[0], ev_free[1]})
      if (e) cudaEventDestroy(e);
  }
}

void Pop::sync() {
  CUDA_CHECK(cudaStreamSynchronize(stream));
  check_guard();
}

void Pop::check_guard() {
  if (guard_h && *reinterpret_cast<volatile int*>(guard_h)) {
    *guard_h = 0;
    invalidate_graphs();
    PBRL_THROW(PBRL_E_USAGE,
               "TD3 step graph: a policy fired on a step the host-side policy-delay mirror "
               "predicted to skip (mirror diverged from the device accumulators)");
  }
}

// BF16 mode: re-derive the bf16 tensor-core copies from the fp32 master weights (after init,
// set_member, PBT exploit copies, imports); the update step itself keeps them current
void Pop::refresh_shadows() {
  if (!act16()) return;
  const size_t np = static_cast<size_t>(n) * pol.stride;
  const size_t nc = 2 * static_cast<size_t>(ncrit) * cri.stride;
  launch_to_bf16(pol_p.p, pol_p16.p, np, stream);
  if (pol_t16.p) launch_to_bf16(pol_t.p, pol_t16.p, np, stream);
  launch_to_bf16(cri_p.p, cri_p16.p, nc, stream);
  launch_to_bf16(cri_t.p, cri_t16.p, nc, stream);
  count_launch(pol_t16.p ? 4 : 3);
  weights_written_outside();
  weights_dirty = false;
}

const void* Pop::wop(const float* W) const {
  if (!act16()) return W;
  const std::pair<const DBuf<float>*, const DBuf<__nv_bfloat16>*> arenas[] = {
      {&pol_p, &pol_p16}, {&pol_t, &pol_t16}, {&cri_p, &cri_p16}, {&cri_t, &cri_t16}};
  for (const auto& a : arenas) {
    if (a.first->p && W >= a.first->p && W < a.first->p + a.first->count)
      return a.second->p + (W - a.first->p);
  }
  PBRL_THROW(PBRL_E_USAGE, "bf16 mode: weight operand outside the parameter arenas");
}

int Pop::field_index(const std::string& f) const {
  for (size_t i = 0; i < fields.size(); ++i)
    if (fields[i] == f) return static_cast<int>(i);
  return -1;
}

// Td3Hyper::validate (algos.hpp:81-108); SAC has no validate in the reference beyond lr > 0 in
// adam_step_inplace (pop_tensor.hpp:335-337) and tau in (0,1] in soft_update (:421).
void Pop::validate_hyper() const {
  for (int i = 0; i < n; ++i) {
    if (algo == PBRL_ALGO_TD3) {
      if (!(hyper[0][i] > 0) || !(hyper[1][i] > 0))
        PBRL_THROW(PBRL_E_CONFIG, "Td3Hyper: learning rates must be positive");
      if (!(hyper[2][i] > 0 && hyper[2][i] <= 1.0))
        PBRL_THROW(PBRL_E_CONFIG, "Td3Hyper: policy_delay_ratio must be in (0, 1]");
      if (hyper[3][i] < 0 || hyper[4][i] < 0 || hyper[5][i] < 0)
        PBRL_THROW(PBRL_E_CONFIG, "Td3Hyper: noise parameters must be >= 0");
      if (!(hyper[6][i] >= 0.9 && hyper[6][i] <= 1.0) && hyper[6][i] != 0.0)
        PBRL_THROW(PBRL_E_CONFIG, "Td3Hyper: discount must be in [0.9, 1] (or 0 in tests)");
      if (!(hyper[7][i] > 0 && hyper[7][i] <= 1.0))
        PBRL_THROW(PBRL_E_CONFIG, "Td3Hyper: tau must be in (0, 1]");
    } else {
      if (!(hyper[0][i] > 0) || !(hyper[1][i] > 0) || !(hyper[2][i] > 0))
        PBRL_THROW(PBRL_E_CONFIG, "adam_step: learning rate must be positive");
      if (!(hyper[6][i] > 0 && hyper[6][i] <= 1.0))
        PBRL_THROW(PBRL_E_CONFIG, "soft_update: tau must be in (0, 1]");
    }
  }
}

// Per-member floats exactly as the reference casts them inside the step.
void Pop::upload_hyper() {
  std::vector<float> f[8];
  std::vector<double> dd(n);
  for (auto& v : f) v.resize(n);
  for (int i = 0; i < n; ++i) {
    if (algo == PBRL_ALGO_TD3) {
      f[0][i] = static_cast<float>(hyper[0][i]);                                    // critic lr
      f[1][i] = static_cast<float>(hyper[1][i]);                                    // policy lr
      f[2][i] = static_cast<float>(hyper[4][i] * static_cast<double>(bound));       // noise sd
      f[3][i] = static_cast<float>(hyper[5][i] * static_cast<double>(bound));       // noise clip
      f[4][i] = static_cast<float>(hyper[6][i]);                                    // gamma
      f[5][i] = static_cast<float>(hyper[7][i]);                                    // tau
      f[6][i] = static_cast<float>(1.0 - hyper[7][i]);                              // 1 - tau
      f[7][i] = 0.0f;
      dd[i] = hyper[2][i];                                                          // delay ratio
    } else {
      f[0][i] = static_cast<float>(hyper[0][i]);  // policy lr
      f[1][i] = static_cast<float>(hyper[1][i]);  // critic lr
      f[2][i] = static_cast<float>(hyper[2][i]);  // alpha lr
      f[3][i] = static_cast<float>(hyper[4][i]);  // reward scale
      f[4][i] = static_cast<float>(hyper[5][i]);  // gamma
      f[5][i] = static_cast<float>(hyper[6][i]);  // tau
      f[6][i] = static_cast<float>(1.0 - hyper[6][i]);
      f[7][i] = 0.0f;
      dd[i] = hyper[3][i];  // target entropy
    }
  }
  DBuf<float>* dst[8] = {&h_f0, &h_f1, &h_f2, &h_f3, &h_f4, &h_f5, &h_f6, &h_f7};
  for (int k = 0; k < 8; ++k) dst[k]->upload(f[k].data(), n, stream);
  h_d0.upload(dd.data(), n, stream);
  sync();
}

// Adam bias-correction tables: corr[t] = (T)(1 - pow(beta, t)) computed in double on the host
// with the same libm the reference uses (pop_tensor.hpp:347-350).
void Pop::ensure_corr(size_t need) {
  if (need <= corr_len) return;
  size_t len = std::max<size_t>(need, corr_len * 2);
  std::vector<float> c1(len), c2(len);
  for (size_t t = 0; t < len; ++t) {
    c1[t] = static_cast<float>(1.0 - std::pow(0.9, static_cast<double>(t)));
    c2[t] = static_cast<float>(1.0 - std::pow(0.999, static_cast<double>(t)));
  }
  invalidate_graphs();
  corr1.alloc(len);
  corr2.alloc(len);
  corr1.upload(c1.data(), len, stream);
  corr2.upload(c2.data(), len, stream);
  corr_len = len;
  sync();
}

// ------------------------------------------------------------------ scratch
void Pop::ensure_scratch(int B) {
  if (B <= S.B) return;
  S = Scratch{};
  S.B = B;
  const size_t nb = static_cast<size_t>(n) * B;
  const int L = pol.depth;
  // row strides padded to 4 floats: every activation is a legal TMA source (16 B strides)
  lsa = padl(ds + da);
  lsp = padl(ds + 1);
  S.in_s.alloc(nb * lsp);
  S.in_sa.alloc(nb * lsa);
  S.in_s2a.alloc(nb * lsa);
  S.sa_pi.alloc(nb * lsa);
  S.r.alloc(nb);
  S.d.alloc(nb);
  S.y.alloc(nb);
  S.tq_out.alloc(2 * nb);
  S.q.alloc(2 * nb);
  S.dq.alloc(2 * nb);
  S.qpi.alloc(2 * nb);
  S.gq.alloc(2 * nb);
  S.pt.alloc(nb * da);
  S.ga.alloc(2 * nb * da);
  S.head.alloc(nb * pol.dims[L]);
  S.gtop.alloc(nb * pad4(pol.dims[L]));
  for (int sl = 0; sl < 2; ++sl) {
    S.bs[sl].alloc(nb * ds);
    S.ba[sl].alloc(nb * da);
    S.br[sl].alloc(nb);
    S.bs2[sl].alloc(nb * ds);
    S.bd[sl].alloc(nb);
  }
  slot_used[0] = slot_used[1] = false;
  for (int l = 0; l + 1 < L; ++l) {
    // activations [rows][pad4(H)] + the ReLU mask bits [rows][ceil(H / 32)] (see Pop::hid)
    const size_t h = static_cast<size_t>(padl(pol.dims[l + 1])) + (pol.dims[l + 1] + 31) / 32;
    for (auto* v : {&S.tp_h, &S.ph, &S.pdh}) {
      v->emplace_back();
      v->back().alloc(nb * h);
    }
    for (auto* v : {&S.tq_h, &S.ch, &S.dh, &S.qh, &S.qdh}) {
      v->emplace_back();
      v->back().alloc(2 * nb * h);
    }
  }
  if (algo == PBRL_ALGO_TD3) S.tnoise.alloc(nb * da);
  if (algo == PBRL_ALGO_SAC) {
    S.x.alloc(nb * da);
    S.th.alloc(nb * da);
    S.ls.alloc(nb * da);
    S.eps.alloc(nb * da);
    S.logp.alloc(nb);
    S.logp2.alloc(nb);
    S.lw.alloc(nb);
    S.clamped.alloc(nb * da);
  }
  // fresh buffers: zero so never-written padding columns cannot carry NaN bit patterns
  for (auto* b : {&S.in_sa, &S.in_s2a, &S.sa_pi, &S.gtop, &S.in_s}) b->zero(stream);
  for (auto* v : {&S.tp_h, &S.ph, &S.pdh, &S.tq_h, &S.ch, &S.dh, &S.qh, &S.qdh})
    for (auto& b : *v) b.zero(stream);
  ones_dirty = true;
  invalidate_graphs();
}

// Tensor-core modes: the padding column ds+da of the critic-input block [s | a] holds 1.0 so the
// critics' first-layer dW product (M = ds+da+1 rows) also produces the first-layer bias gradient
// (its extra row lands on b0, which follows W0 in the flat layout).  Forward products never read
// it (their K extent is ds+da).
void Pop::ensure_ones() {
  if (!ones_dirty) return;
  if (use_tc() && lsa > ds + da)
    launch_fill_col(S.in_sa.p, static_cast<long long>(n) * S.B, lsa, ds + da, 1.0f,
                    act16() ? 1 : 0, stream);
  if (use_tc() && lsp > ds)  // the policy input's ones column (its first-layer bias gradient)
    launch_fill_col(S.in_s.p, static_cast<long long>(n) * S.B, lsp, ds, 1.0f, act16() ? 1 : 0,
                    stream);
  ones_dirty = false;
}

// ------------------------------------------------------------------ update entry points
void Pop::update_batches(const pbrl_batch* batches, uint32_t k, uint64_t rows,
                         const uint8_t* policy_mask, bool device_ptrs, double* losses_out) {
  if (k < 1) PBRL_THROW(PBRL_E_CONFIG, "update_k_steps: k must be >= 1");
  if (rows < 1) PBRL_THROW(PBRL_E_SHAPE, "batch rows must be >= 1");
  validate_hyper();
  if (policy_mask && algo != PBRL_ALGO_TD3)
    PBRL_THROW(PBRL_E_USAGE, "policy_member_mask is a TD3 option");
  const int B = static_cast<int>(rows);
  ensure_scratch(B);
  ensure_ones();
  ensure_corr(t_bound + k + 4);
  const uint8_t* d_mask = nullptr;
  host_mask = policy_mask;
  if (policy_mask) {
    mask_buf.alloc(n);
    mask_buf.upload(policy_mask, n, stream);
    d_mask = mask_buf.p;
  }
  const size_t nb = static_cast<size_t>(n) * B;
  for (uint32_t i = 0; i < k; ++i) {
    const pbrl_batch& b = batches[i];
    if (!b.s || !b.a || !b.r || !b.s2 || !b.done) PBRL_THROW(PBRL_E_USAGE, "null batch pointer");
  }
  // every step's losses: a device history of kLossHist slots, read back one block at a time
  const size_t row = static_cast<size_t>(3) * n;
  if (losses_out) loss_hist.alloc(kLossHist * row);
  auto hist_d2h = [&](uint32_t j, bool last) {  // once step j's losses are in the history
    if (j % kLossHist != kLossHist - 1 && !last) return;
    const uint32_t first = j - j % kLossHist;
    CUDA_CHECK(cudaMemcpyAsync(losses_out + first * row, loss_hist.p,
                               (j - first + 1) * row * sizeof(double), cudaMemcpyDeviceToHost,
                               stream));
  };
  // TD3: k_td3_step_begin of step i+1 files step i's losses (keyed by steps[] - hist_base[]),
  // so no copy launch sits between the step graphs
  struct HistScope {
    bool& on;
    ~HistScope() { on = false; }
  } hist_scope{hist_on};
  hist_on = losses_out && algo == PBRL_ALGO_TD3;
  if (hist_on) {
    hist_base.alloc(n);
    CUDA_CHECK(cudaMemcpyAsync(hist_base.p, steps.p, n * sizeof(uint64_t),
                               cudaMemcpyDeviceToDevice, stream));
  }
  if (!device_ptrs && !cstream) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
    for (int sl = 0; sl < 2; ++sl) {
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_copied[sl], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_free[sl], cudaEventDisableTiming));
    }
  }
  // H2D of host batch i into staging slot i % 2 on the copy stream, after the pack that last
  // read that slot (ev_free); the step's pack waits for the copy (ev_copied)
  auto stage = [&](uint32_t i) {
    const pbrl_batch& b = batches[i];
    const int sl = static_cast<int>(i & 1u);
    if (slot_used[sl]) CUDA_CHECK(cudaStreamWaitEvent(cstream, ev_free[sl], 0));
    const cudaMemcpyKind h2d = cudaMemcpyHostToDevice;
    CUDA_CHECK(cudaMemcpyAsync(S.bs[sl].p, b.s, nb * ds * 4, h2d, cstream));
    CUDA_CHECK(cudaMemcpyAsync(S.ba[sl].p, b.a, nb * da * 4, h2d, cstream));
    CUDA_CHECK(cudaMemcpyAsync(S.br[sl].p, b.r, nb * 4, h2d, cstream));
    CUDA_CHECK(cudaMemcpyAsync(S.bs2[sl].p, b.s2, nb * ds * 4, h2d, cstream));
    CUDA_CHECK(cudaMemcpyAsync(S.bd[sl].p, b.done, nb * 4, h2d, cstream));
    CUDA_CHECK(cudaEventRecord(ev_copied[sl], cstream));
    slot_used[sl] = true;
  };
  if (!device_ptrs) stage(0);
  const bool ovl = pack_overlap_ok();
  if (ovl && !pstream) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&pstream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&ev_packed, cudaEventDisableTiming));
  }
  last_step_stage_ev = false;  // across calls the member stream may carry other work
  for (uint32_t i = 0; i < k; ++i) {
    const pbrl_batch& b = batches[i];
    const float *s = b.s, *a = b.a, *r = b.r, *s2 = b.s2, *d = b.done;
    // the pack of batch i overlaps the last Adam of step i-1 (after its ev_stage_free) when
    // step i-1 was a graph that records it; otherwise it runs in member-stream order
    const bool side = ovl && last_step_stage_ev;
    cudaStream_t ps = side ? pstream : stream;
    if (side) CUDA_CHECK(cudaStreamWaitEvent(ps, ev_stage_free, 0));
    if (!device_ptrs) {
      if (i + 1 < k) stage(i + 1);  // overlaps this step
      const int sl = static_cast<int>(i & 1u);
      CUDA_CHECK(cudaStreamWaitEvent(ps, ev_copied[sl], 0));
      s = S.bs[sl].p;
      a = S.ba[sl].p;
      r = S.br[sl].p;
      s2 = S.bs2[sl].p;
      d = S.bd[sl].p;
    }
    timed(PC_GATHER, 0.0, pack_bytes(B), 0, [&] {
      launch_pack_batch(n, B, ds, da, lsa, s, a, r, s2, d, S.in_sa.p, S.in_s2a.p, S.sa_pi.p, S.r.p,
                        S.d.p, act16() ? 1 : 0, ps, S.in_s.p, lsp);
    });
    if (!device_ptrs) CUDA_CHECK(cudaEventRecord(ev_free[i & 1u], ps));
    if (side) {
      CUDA_CHECK(cudaEventRecord(ev_packed, ps));
      CUDA_CHECK(cudaStreamWaitEvent(stream, ev_packed, 0));
    }
    step(B, d_mask);
    if (losses_out && !hist_on) {
      // this step's critic1 / critic2 / policy losses -> a device history slot; the history
      // goes to the host in one copy per kLossHist steps (async, in stream order).  A kernel
      // rather than a copy node, so the programmatic-dependent-launch chain is not broken.
      launch_copy_f64(loss_hist.p + (i % kLossHist) * row, losses.p, row, stream);
      count_launch(1);
      hist_d2h(i, i + 1 == k);
    } else if (hist_on && i >= 1) {
      hist_d2h(i - 1, false);  // step i's begin has filed step i-1's losses
    }
  }
  if (hist_on) {  // the last step's losses (no next begin files them)
    launch_copy_f64(loss_hist.p + ((k - 1) % kLossHist) * row, losses.p, row, stream);
    count_launch(1);
    hist_d2h(k - 1, true);
  }
  host_mask = nullptr;
  host_mask = nullptr;  // the caller's buffer is only valid during the call
  if (losses_out) {
    sync();
    for (uint32_t i = 0; i < k; ++i) shared_losses_layout(losses_out + static_cast<size_t>(i) * 3 * n);
  }
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace pbrl
