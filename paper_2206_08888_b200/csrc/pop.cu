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
  if (d.precision != PBRL_PREC_FFMA32 && d.precision != PBRL_PREC_BF16 &&
      d.precision != PBRL_PREC_TF32)
    PBRL_THROW(PBRL_E_CONFIG, "unknown precision mode");
  algo = d.algo;
  precision = d.precision;
  device = d.device;
  n = static_cast<int>(d.n);
  ds = static_cast<int>(d.obs_dim);
  da = static_cast<int>(d.act_dim);
  member_offset = d.member_offset;
  n_global = d.n_global ? d.n_global : d.n;
  bound = static_cast<float>(d.action_bound);
  seed = d.seed;
  for (uint32_t i = 0; i < d.n_hidden; ++i) {
    if (d.hidden[i] < 1) PBRL_THROW(PBRL_E_CONFIG, "hidden widths must be >= 1");
    hidden.push_back(d.hidden[i]);
  }
  CUDA_CHECK(cudaSetDevice(device));
  CUDA_CHECK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));

  std::vector<size_t> pd{static_cast<size_t>(ds)};
  pd.insert(pd.end(), hidden.begin(), hidden.end());
  pd.push_back(static_cast<size_t>(algo == PBRL_ALGO_TD3 ? da : 2 * da));
  pol.make(pd, algo == PBRL_ALGO_TD3 ? ACT_TANH : ACT_NONE, algo == PBRL_ALGO_TD3 ? bound : 1.0f);
  std::vector<size_t> qd{static_cast<size_t>(ds + da)};
  qd.insert(qd.end(), hidden.begin(), hidden.end());
  qd.push_back(1);
  cri.make(qd, ACT_NONE, 1.0f);

  const size_t np = static_cast<size_t>(n) * pol.stride;
  const size_t nc = 2 * static_cast<size_t>(n) * cri.stride;
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
  t_cri.alloc(2 * n);
  steps.alloc(n);
  streams.alloc(n);
  fire.alloc(n);
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
  launch_init_net(cri, cri_p.p, n, member_offset, s_c1, stream);
  launch_init_net(cri, cri_p.p + static_cast<size_t>(n) * cri.stride, n, member_offset, s_c2,
                  stream);
  count_launch(3 * pol.depth);
  if (algo == PBRL_ALGO_TD3)
    CUDA_CHECK(cudaMemcpyAsync(pol_t.p, pol_p.p, np * 4, cudaMemcpyDeviceToDevice, stream));
  CUDA_CHECK(cudaMemcpyAsync(cri_t.p, cri_p.p, nc * 4, cudaMemcpyDeviceToDevice, stream));

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

Pop::~Pop() {
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

void Pop::sync() { CUDA_CHECK(cudaStreamSynchronize(stream)); }

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
  const int dsa = ds + da;
  const int L = pol.depth;
  S.in_sa.alloc(nb * dsa);
  S.in_s2a.alloc(nb * dsa);
  S.sa_pi.alloc(nb * dsa);
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
  S.gtop.alloc(nb * pol.dims[L]);
  S.bs.alloc(nb * ds);
  S.ba.alloc(nb * da);
  S.br.alloc(nb);
  S.bs2.alloc(nb * ds);
  S.bd.alloc(nb);
  for (int l = 0; l + 1 < L; ++l) {
    const size_t h = static_cast<size_t>(pol.dims[l + 1]);
    S.tp_h.emplace_back();
    S.tp_h.back().alloc(nb * h);
    S.ph.emplace_back();
    S.ph.back().alloc(nb * h);
    S.pdh.emplace_back();
    S.pdh.back().alloc(nb * h);
    S.tq_h.emplace_back();
    S.tq_h.back().alloc(2 * nb * h);
    S.ch.emplace_back();
    S.ch.back().alloc(2 * nb * h);
    S.dh.emplace_back();
    S.dh.back().alloc(2 * nb * h);
    S.qh.emplace_back();
    S.qh.back().alloc(2 * nb * h);
    S.qdh.emplace_back();
    S.qdh.back().alloc(2 * nb * h);
  }
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
}

// ------------------------------------------------------------------ GEMM builders
namespace {
Operand fwd_in(const float* p, long long gs, long long ld, int by_member) {
  Operand o;
  o.p = p;
  o.gs = gs;
  o.rs = ld;
  o.cs = 1;
  o.by_member = by_member;
  return o;
}
Operand as_kmajor_t(const float* p, long long gs, long long ld, int by_member) {
  // X^T for dW: A(i = feature, k = row) = X[k*ld + i]
  Operand o;
  o.p = p;
  o.gs = gs;
  o.rs = 1;
  o.cs = ld;
  o.by_member = by_member;
  return o;
}
}  // namespace

// forward of layer l: Y = act(X W_l + b_l)
void Pop::gemm_fwd(const NetShape& sh, const float* W, int l, int groups, int B, Operand X,
                   float* Y, long long y_gs, long long y_rs, int epi, const int* active,
                   float* C2, long long c2_gs, long long c2_rs, bool noise) {
  GemmArgs g;
  g.M = B;
  g.N = sh.dims[l + 1];
  g.K = sh.dims[l];
  g.groups = groups;
  g.n_members = n;
  g.A = X;
  g.B.p = W + sh.woff[l];
  g.B.gs = static_cast<long long>(sh.stride);
  g.B.rs = sh.dims[l + 1];
  g.B.cs = 1;
  g.bias.p = W + sh.boff[l];
  g.bias.gs = static_cast<long long>(sh.stride);
  g.bias.cs = 1;
  g.C = Y;
  g.c_gs = y_gs;
  g.c_rs = y_rs;
  g.epi = epi;
  g.acc_init = -0.0f;
  g.active = active;
  g.C2 = C2;
  g.c2_gs = c2_gs;
  g.c2_rs = c2_rs;
  g.scale = sh.out_scale;
  if (noise) {
    g.noise_key = key_a.p;
    g.noise_sd = h_f2.p;
    g.noise_clip = h_f3.p;
    g.bound = bound;
  }
  run_gemm(g, PC_GEMM_FWD);
}

// dX of layer l restricted to input columns [col0, col0+ncols): DX = epi(G W_l^T)
void Pop::gemm_dx(const NetShape& sh, const float* W, int l, int groups, int B, Operand G,
                  Operand aux, float* DX, long long dx_gs, long long dx_rs, int epi, int col0,
                  int ncols, const int* active, float scale) {
  GemmArgs g;
  g.M = B;
  g.N = ncols;
  g.K = sh.dims[l + 1];
  g.groups = groups;
  g.n_members = n;
  g.A = G;
  g.B.p = W + sh.woff[l] + static_cast<size_t>(col0) * sh.dims[l + 1];
  g.B.gs = static_cast<long long>(sh.stride);
  g.B.rs = 1;
  g.B.cs = sh.dims[l + 1];
  g.C = DX;
  g.c_gs = dx_gs;
  g.c_rs = dx_rs;
  g.epi = epi;
  g.aux = aux;
  g.acc_init = 0.0f;
  g.active = active;
  g.scale = scale;
  run_gemm(g, PC_GEMM_DX);
}

// dW_l and db_l (as the ones row) into the gradient arena: [X;1]^T G
void Pop::gemm_dw(const NetShape& sh, float* Gr, int l, int groups, int B, Operand XT, Operand G,
                  const int* active) {
  GemmArgs g;
  g.M = sh.dims[l] + 1;
  g.N = sh.dims[l + 1];
  g.K = B;
  g.groups = groups;
  g.n_members = n;
  g.A = XT;
  g.a_ones_row = 1;
  g.B = G;
  g.C = Gr + sh.woff[l];
  g.c_gs = static_cast<long long>(sh.stride);
  g.c_rs = sh.dims[l + 1];
  g.epi = EPI_STORE;
  g.acc_init = 0.0f;
  g.active = active;
  run_gemm(g, PC_GEMM_DW);
}

void Pop::run_gemm(const GemmArgs& g, int cls) {
  // algorithmic FLOPs: the bias ones-row of dW is bookkeeping, not work
  const int M = g.a_ones_row ? g.M - 1 : g.M;
  timed(cls, 2.0 * M * g.N * g.K * g.groups, 0.0, g.active != nullptr,
        [&] { launch_gemm_simt(g, stream); });
}

// ------------------------------------------------------------------ profiling
cudaEvent_t Pop::prof_event() {
  if (ev_used == ev_pool.size()) {
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  return ev_pool[ev_used++];
}

void Pop::prof_begin(cudaEvent_t* a) {
  if (!prof_on) return;
  *a = prof_event();
  CUDA_CHECK(cudaEventRecord(*a, stream));
}

void Pop::prof_end(cudaEvent_t a, int cls, double flops, double bytes, int gated) {
  if (!prof_on) return;
  cudaEvent_t b = prof_event();
  CUDA_CHECK(cudaEventRecord(b, stream));
  prof.push_back(ProfRec{cls, flops, bytes, gated, prof_step, a, b, 0.0});
}

// critic targets are Polyak-updated only for fired members in TD3: extra gated bytes
void Pop::prof_add_gated_bytes(double bytes) {
  if (prof_on && !prof.empty()) prof.back().gbytes += bytes;
}

void Pop::prof_step_done() {
  if (!prof_on) return;
  int nf = n;
  if (algo == PBRL_ALGO_TD3) {
    std::vector<int> f(n);
    CUDA_CHECK(cudaMemcpyAsync(f.data(), fire.p, 4 * n, cudaMemcpyDeviceToHost, stream));
    sync();
    nf = 0;
    for (int v : f) nf += v;
  }
  prof_fired.push_back(nf);
  ++prof_step;
}

std::string Pop::prof_report() {
  sync();
  static const char* names[PC_COUNT] = {"gemm_fwd", "gemm_dx", "gemm_dw", "adam_polyak",
                                        "elementwise", "gather_pack"};
  double ms[PC_COUNT] = {}, fl[PC_COUNT] = {}, by[PC_COUNT] = {};
  long long cnt[PC_COUNT] = {};
  for (const ProfRec& r : prof) {
    float t = 0.0f;
    CUDA_CHECK(cudaEventElapsedTime(&t, r.a, r.b));
    const double frac = (r.gated && r.step < static_cast<int>(prof_fired.size()))
                            ? static_cast<double>(prof_fired[r.step]) / n : 1.0;
    ms[r.cls] += t;
    fl[r.cls] += r.flops * frac;
    by[r.cls] += r.bytes * frac;
    if (r.gbytes > 0.0 && r.step < static_cast<int>(prof_fired.size()))
      by[r.cls] += r.gbytes * static_cast<double>(prof_fired[r.step]) / n;
    cnt[r.cls] += 1;
  }
  std::string out = "{\"steps\": " + std::to_string(prof_step) + ", \"classes\": {";
  for (int c = 0; c < PC_COUNT; ++c) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s\"%s\": {\"launches\": %lld, \"ms\": %.6f, \"flops\": %.6e, "
             "\"bytes\": %.6e}", c ? ", " : "", names[c], cnt[c], ms[c], fl[c], by[c]);
    out += buf;
  }
  out += "}}";
  return out;
}

// ------------------------------------------------------------------ critic update (shared)
// Twin critics as one grouped problem of 2n groups: forward on [s|a], MSE cotangent,
// backward (dW for every layer, dX for layers > 0), fused Adam + target Polyak.
void Pop::critic_update(int B, const int* polyak_gate) {
  const int L = cri.depth, n2 = 2 * n, dsa = ds + da;
  const long long nbB = B;
  Operand x = fwd_in(S.in_sa.p, nbB * dsa, dsa, 1);
  for (int l = 0; l < L; ++l) {
    const bool last = l == L - 1;
    const int h = cri.dims[l + 1];
    float* out = last ? S.q.p : S.ch[l].p;
    gemm_fwd(cri, cri_p.p, l, n2, B, x, out, nbB * h, h, last ? EPI_BIAS : EPI_BIAS_RELU);
    x = fwd_in(out, nbB * h, h, 0);
  }
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_mse(n2, n, B, S.q.p, S.y.p, S.dq.p, losses.p, stream); });
  Operand G = fwd_in(S.dq.p, nbB, 1, 0);
  for (int l = L - 1; l >= 0; --l) {
    Operand xt = (l == 0) ? as_kmajor_t(S.in_sa.p, nbB * dsa, dsa, 1)
                          : as_kmajor_t(S.ch[l - 1].p, nbB * cri.dims[l], cri.dims[l], 0);
    gemm_dw(cri, cri_g.p, l, n2, B, xt, G, nullptr);
    if (l > 0) {
      const int hin = cri.dims[l];
      Operand mask = fwd_in(S.ch[l - 1].p, nbB * hin, hin, 0);
      gemm_dx(cri, cri_p.p, l, n2, B, G, mask, S.dh[l - 1].p, nbB * hin, hin, EPI_RELU_MASK, 0,
              hin, nullptr, 1.0f);
      G = fwd_in(S.dh[l - 1].p, nbB * hin, hin, 0);
    }
  }
  const float* clr = algo == PBRL_ALGO_TD3 ? h_f0.p : h_f1.p;
  timed(PC_ADAM, 0.0, static_cast<double>(cri.P) * (n2) * 28.0, 0,
        [&] { launch_adam(n2, n, cri.P, cri.stride, cri_p.p, cri_m.p, cri_v.p, cri_g.p, t_cri.p, corr1.p,
              corr2.p, clr, nullptr, cri_t.p, h_f5.p, h_f6.p, polyak_gate, stream); });
  // fused target Polyak: +8 B/param (read + write target), every member (SAC) or fired (TD3)
  if (polyak_gate) prof_add_gated_bytes(8.0 * cri.P * n2);
  else if (prof_on && !prof.empty()) prof.back().bytes += 8.0 * cri.P * n2;
}

// forward of `sh` (groups x B rows) from input operand x; hidden activations into hs[l]
void Pop::mlp_forward(const NetShape& sh, const float* W, int groups, int B, Operand x,
                      std::vector<DBuf<float>>& hs, float* out, long long out_gs,
                      long long out_rs, int last_epi, const int* active, float* C2,
                      long long c2_gs, long long c2_rs, bool noise) {
  const int L = sh.depth;
  for (int l = 0; l < L; ++l) {
    const bool last = l == L - 1;
    const int h = sh.dims[l + 1];
    if (last) {
      gemm_fwd(sh, W, l, groups, B, x, out, out_gs, out_rs, last_epi, active, C2, c2_gs, c2_rs,
               noise);
    } else {
      gemm_fwd(sh, W, l, groups, B, x, hs[l].p, static_cast<long long>(B) * h, h, EPI_BIAS_RELU,
               active);
      x = fwd_in(hs[l].p, static_cast<long long>(B) * h, h, 0);
    }
  }
}

// backward of `sh` from the top cotangent G: dW for every layer, dX for layers > 0
void Pop::mlp_backward(const NetShape& sh, const float* W, float* Gr, int groups, int B,
                       Operand G, Operand x0t, std::vector<DBuf<float>>& hs,
                       std::vector<DBuf<float>>& dhs, const int* active) {
  const int L = sh.depth;
  for (int l = L - 1; l >= 0; --l) {
    Operand xt = (l == 0) ? x0t
                          : as_kmajor_t(hs[l - 1].p, static_cast<long long>(B) * sh.dims[l],
                                        sh.dims[l], 0);
    gemm_dw(sh, Gr, l, groups, B, xt, G, active);
    if (l > 0) {
      const int hin = sh.dims[l];
      Operand mask = fwd_in(hs[l - 1].p, static_cast<long long>(B) * hin, hin, 0);
      gemm_dx(sh, W, l, groups, B, G, mask, dhs[l - 1].p, static_cast<long long>(B) * hin, hin,
              EPI_RELU_MASK, 0, hin, active, 1.0f);
      G = fwd_in(dhs[l - 1].p, static_cast<long long>(B) * hin, hin, 0);
    }
  }
}

// critic dX chain from the output cotangent down to the action columns of the input
void Pop::critic_dx_to_action(int groups, int B, Operand G, std::vector<DBuf<float>>& hs,
                              std::vector<DBuf<float>>& dhs, float* out, int epi, Operand aux,
                              float scale, const int* active) {
  const int L = cri.depth;
  for (int l = L - 1; l >= 1; --l) {
    const int hin = cri.dims[l];
    Operand mask = fwd_in(hs[l - 1].p, static_cast<long long>(B) * hin, hin, 0);
    gemm_dx(cri, cri_p.p, l, groups, B, G, mask, dhs[l - 1].p, static_cast<long long>(B) * hin,
            hin, EPI_RELU_MASK, 0, hin, active, 1.0f);
    G = fwd_in(dhs[l - 1].p, static_cast<long long>(B) * hin, hin, 0);
  }
  gemm_dx(cri, cri_p.p, 0, groups, B, G, aux, out, static_cast<long long>(B) * da, da, epi, ds, da,
          active, scale);
}

// ------------------------------------------------------------------ TD3 step (algos.hpp:351-422)
void Pop::td3_step(int B, const uint8_t* d_mask) {
  const int dsa = ds + da;
  const long long nbB = B;
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_td3_step_begin(n, delay_acc.p, h_d0.p, d_mask, fire.p, t_pol.p, t_cri.p, t_cri.p + n,
                        steps.p, streams.p, seed, key_a.p, stream); });
  // td3_critic_target (algos.hpp:241-282): pi'(s2) + clipped noise, twin target critics, y
  mlp_forward(pol, pol_t.p, n, B, fwd_in(S.in_s2a.p, nbB * dsa, dsa, 0), S.tp_h, S.in_s2a.p + ds,
              nbB * dsa, dsa, EPI_BIAS_TANH_NOISE, nullptr, nullptr, 0, 0, true);
  mlp_forward(cri, cri_t.p, 2 * n, B, fwd_in(S.in_s2a.p, nbB * dsa, dsa, 1), S.tq_h, S.tq_out.p,
              nbB, 1, EPI_BIAS);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_td_target(n, B, S.r.p, S.d.p, S.tq_out.p, h_f4.p, S.y.p, stream); });
  // twin critic update; target Polyak fused for members whose policy fires (:401-418)
  critic_update(B, fire.p);
  // td3_policy_loss_grads (:318-338) on the UPDATED critic1, gated by the fire mask
  mlp_forward(pol, pol_p.p, n, B, fwd_in(S.in_sa.p, nbB * dsa, dsa, 0), S.ph, S.sa_pi.p + ds,
              nbB * dsa, dsa, EPI_BIAS_TANH, fire.p, S.pt.p, nbB * da, da);
  mlp_forward(cri, cri_p.p, n, B, fwd_in(S.sa_pi.p, nbB * dsa, dsa, 0), S.qh, S.qpi.p, nbB, 1,
              EPI_BIAS, fire.p);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_td3_policy_loss(n, B, S.qpi.p, fire.p, losses.p + 2 * n, S.gq.p, stream); });
  Operand aux_t = fwd_in(S.pt.p, nbB * da, da, 0);
  critic_dx_to_action(n, B, fwd_in(S.gq.p, nbB, 1, 0), S.qh, S.qdh, S.gtop.p, EPI_TANH_GRAD,
                      aux_t, pol.out_scale, fire.p);
  mlp_backward(pol, pol_p.p, pol_g.p, n, B, fwd_in(S.gtop.p, nbB * da, da, 0),
               as_kmajor_t(S.in_sa.p, nbB * dsa, dsa, 0), S.ph, S.pdh, fire.p);
  timed(PC_ADAM, 0.0, static_cast<double>(pol.P) * (n) * (28.0 + 8.0), 1,
        [&] { launch_adam(n, n, pol.P, pol.stride, pol_p.p, pol_m.p, pol_v.p, pol_g.p, t_pol.p, corr1.p,
              corr2.p, h_f1.p, fire.p, pol_t.p, h_f5.p, h_f6.p, nullptr, stream); });
}

// ------------------------------------------------------------------ SAC step (algos.hpp:781-837)
void Pop::sac_step(int B) {
  const int dsa = ds + da, L = pol.depth;
  const long long nbB = B;
  const int hd = pol.dims[L];
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_sac_step_begin(n, t_pol.p, t_cri.p, t_cri.p + n, t_alpha.p, steps.p, streams.p, seed,
                        key_a.p, key_b.p, stream); });
  // sac_critic_target (algos.hpp:739-776): current policy on s2, eps' draws, twin targets
  mlp_forward(pol, pol_p.p, n, B, fwd_in(S.in_s2a.p, nbB * dsa, dsa, 0), S.tp_h, S.head.p,
              nbB * hd, hd, EPI_BIAS);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_sac_head(n, B, ds, da, S.head.p, key_b.p, bound, S.in_s2a.p, nullptr, nullptr, nullptr,
                  nullptr, nullptr, S.logp2.p, stream); });
  mlp_forward(cri, cri_t.p, 2 * n, B, fwd_in(S.in_s2a.p, nbB * dsa, dsa, 1), S.tq_h, S.tq_out.p,
              nbB, 1, EPI_BIAS);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_sac_y(n, B, S.r.p, S.d.p, S.tq_out.p, S.logp2.p, log_alpha.p, h_f4.p, h_f3.p, S.y.p,
               stream); });
  critic_update(B, nullptr);  // critic targets tracked every step (:827-834)
  // sac_policy_loss_grads (:643-735) through both UPDATED critics
  mlp_forward(pol, pol_p.p, n, B, fwd_in(S.in_sa.p, nbB * dsa, dsa, 0), S.ph, S.head.p, nbB * hd,
              hd, EPI_BIAS);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_sac_head(n, B, ds, da, S.head.p, key_a.p, bound, S.sa_pi.p, S.x.p, S.th.p, S.ls.p,
                  S.clamped.p, S.eps.p, S.logp.p, stream); });
  mlp_forward(cri, cri_p.p, 2 * n, B, fwd_in(S.sa_pi.p, nbB * dsa, dsa, 1), S.qh, S.qpi.p, nbB, 1,
              EPI_BIAS);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_sac_policy_top(n, B, S.qpi.p, S.logp.p, log_alpha.p, losses.p + 2 * n, S.gq.p, S.lw.p,
                        stream); });
  critic_dx_to_action(2 * n, B, fwd_in(S.gq.p, nbB, 1, 0), S.qh, S.qdh, S.ga.p, EPI_STORE,
                      Operand{}, 1.0f, nullptr);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_sac_head_grad(n, B, da, S.ga.p, S.lw.p, S.x.p, S.th.p, S.ls.p, S.clamped.p, S.eps.p,
                       bound, S.gtop.p, stream); });
  mlp_backward(pol, pol_p.p, pol_g.p, n, B, fwd_in(S.gtop.p, nbB * hd, hd, 0),
               as_kmajor_t(S.in_sa.p, nbB * dsa, dsa, 0), S.ph, S.pdh, nullptr);
  timed(PC_ADAM, 0.0, static_cast<double>(pol.P) * (n) * (28.0 + 0.0), 0,
        [&] { launch_adam(n, n, pol.P, pol.stride, pol_p.p, pol_m.p, pol_v.p, pol_g.p, t_pol.p, corr1.p,
              corr2.p, h_f0.p, nullptr, nullptr, nullptr, nullptr, nullptr, stream); });
  timed(PC_ELEM, 0.0, 0.0, 0, [&] { launch_sac_alpha(n, B, S.logp.p, log_alpha.p, h_d0.p, log_alpha.p, alpha_m.p, alpha_v.p,
                   t_alpha.p, corr1.p, corr2.p, h_f2.p, stream); });
}

void Pop::step(int B, const uint8_t* d_mask) {
  ensure_corr(t_bound + 4);
  if (algo == PBRL_ALGO_TD3) td3_step(B, d_mask);
  else sac_step(B);
  t_bound += 1;
  prof_step_done();
}


// ------------------------------------------------------------------ update entry points
void Pop::update_batches(const pbrl_batch* batches, uint32_t k, uint64_t rows,
                         const uint8_t* policy_mask, bool device_ptrs) {
  if (k < 1) PBRL_THROW(PBRL_E_CONFIG, "update_k_steps: k must be >= 1");
  if (rows < 1) PBRL_THROW(PBRL_E_SHAPE, "batch rows must be >= 1");
  validate_hyper();
  if (policy_mask && algo != PBRL_ALGO_TD3)
    PBRL_THROW(PBRL_E_USAGE, "policy_member_mask is a TD3 option");
  const int B = static_cast<int>(rows);
  ensure_scratch(B);
  ensure_corr(t_bound + k + 4);
  const uint8_t* d_mask = nullptr;
  if (policy_mask) {
    mask_buf.alloc(n);
    mask_buf.upload(policy_mask, n, stream);
    d_mask = mask_buf.p;
  }
  const size_t nb = static_cast<size_t>(n) * B;
  const cudaMemcpyKind kind = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  for (uint32_t i = 0; i < k; ++i) {
    const pbrl_batch& b = batches[i];
    if (!b.s || !b.a || !b.r || !b.s2 || !b.done) PBRL_THROW(PBRL_E_USAGE, "null batch pointer");
    const float *s = b.s, *a = b.a, *r = b.r, *s2 = b.s2, *d = b.done;
    if (!device_ptrs) {
      CUDA_CHECK(cudaMemcpyAsync(S.bs.p, b.s, nb * ds * 4, kind, stream));
      CUDA_CHECK(cudaMemcpyAsync(S.ba.p, b.a, nb * da * 4, kind, stream));
      CUDA_CHECK(cudaMemcpyAsync(S.br.p, b.r, nb * 4, kind, stream));
      CUDA_CHECK(cudaMemcpyAsync(S.bs2.p, b.s2, nb * ds * 4, kind, stream));
      CUDA_CHECK(cudaMemcpyAsync(S.bd.p, b.done, nb * 4, kind, stream));
      s = S.bs.p;
      a = S.ba.p;
      r = S.br.p;
      s2 = S.bs2.p;
      d = S.bd.p;
    }
    timed(PC_GATHER, 0.0, 0.0, 0, [&] { launch_pack_batch(n, B, ds, da, s, a, r, s2, d, S.in_sa.p, S.in_s2a.p, S.sa_pi.p, S.r.p,
                      S.d.p, stream); });
    step(B, d_mask);
  }
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace pbrl
