// The TD3 / SAC update-step programs: every dense product of one population update as a
// grouped GEMM launch (tcgen05 in TF32 mode wherever the operands are TMA-legal, the bit-exact
// CUDA-core kernel otherwise and in FFMA32 mode), the fused elementwise steps, and the fused
// Adam + Polyak update; one step is captured once into a CUDA graph and replayed.
#include <cmath>

#include "pop_impl.cuh"
#include "tc_gemm.cuh"

namespace pbrl {

namespace {
Operand simt_op(const float* p, long long gs, long long rs, long long cs, int by_member) {
  Operand o;
  o.p = p;
  o.gs = gs;
  o.rs = rs;
  o.cs = cs;
  o.by_member = by_member;
  return o;
}
}  // namespace

// ------------------------------------------------------------------ GEMM builders
// forward of layer l: Y = act(X W_l + b_l); X is [groups][B][in] (stride X.ld)
void Pop::gemm_fwd(const NetShape& sh, const float* W, int l, int groups, int B, Mat X, float* Y,
                   long long y_gs, long long y_ld, int epi, const int* active, float* C2,
                   long long c2_gs, long long c2_ld, bool noise, const Mat* ymask, bool y_act) {
  const int in = sh.dims[l], out = sh.dims[l + 1];
  const float* Wl = W + sh.woff[l];
  const double flops = 2.0 * B * in * out * groups;
  // algorithmic bytes: X (once per member when shared by the critics), W (the operand copy),
  // b, Y (+ mask bits); activations / operand weights are aeb() bytes wide, Y as stored
  const double ae = aeb(), ye = y_act ? ae : 4.0;
  const double bytes = ae * (static_cast<double>(B) * in * (X.by_member ? n : groups) +
                             static_cast<double>(groups) * in * out) +
                       4.0 * groups * out + ye * groups * B * out +
                       ((ymask && ymask->mask) ? groups * B * ((out + 31) / 32) * 4.0 : 0.0);
  const int eb = aeb();
  const void* Wo = use_tc() ? wop(Wl) : Wl;
  if (use_tc() && out >= 16 && tma_ok(X.p, X.ld, X.gs, eb) && tma_ok(Wo, out, sh.stride, eb)) {
    TcOperand A{X.p, static_cast<uint64_t>(in), static_cast<uint64_t>(B),
                static_cast<uint64_t>(X.by_member ? n : groups), static_cast<uint64_t>(X.ld),
                static_cast<uint64_t>(X.gs)};
    TcOperand Bw{Wo, static_cast<uint64_t>(out), static_cast<uint64_t>(in),
                 static_cast<uint64_t>(groups), static_cast<uint64_t>(out), sh.stride};
    TcArgs a;
    a.eb = eb;
    a.c16 = act16() && y_act ? 1 : 0;
    a.M = B;
    a.N = out;
    a.K = in;
    a.groups = groups;
    a.n_members = n;
    a.a_by_member = X.by_member;
    a.epi = epi;
    a.C = Y;
    a.c_gs = y_gs;
    a.c_rs = y_ld;
    a.bias = W + sh.boff[l];
    a.bias_gs = static_cast<long long>(sh.stride);
    a.C2 = C2;
    a.c2_gs = c2_gs;
    a.c2_rs = c2_ld;
    a.scale = sh.out_scale;
    a.active = active;
    if (noise) {
      a.noise_key = key_a.p;
      a.noise_sd = h_f2.p;
      a.noise_clip = h_f3.p;
      a.bound = bound;
    }
    if (ymask && ymask->mask && epi == EPI_BIAS_RELU) {
      a.mask_out = ymask->mask;
      a.mo_gs = ymask->mgs;
      a.mo_ld = ymask->mld;
    }
    a.b_prefetch = tc_prefetch_ok() ? 1 : 0;
    a.max_ctas = cta_cap;
    timed(PC_GEMM_FWD, flops, bytes, active != nullptr,
          [&] { launch_tc_gemm(A, Bw, false, true, a, stream); });
    return;
  }
  if (act16() && out > 16)
    PBRL_THROW(PBRL_E_CONFIG, "bf16 mode: hidden layers need TMA-legal widths (multiples of 8, >= 16)");
  GemmArgs g;
  g.M = B;
  g.N = out;
  g.K = in;
  g.groups = groups;
  g.n_members = n;
  g.a16 = act16() ? 1 : 0;
  g.c16 = act16() && y_act ? 1 : 0;
  g.rowdot = use_tc() ? 1 : 0;  // no reference summation order to keep outside FFMA32
  g.A = simt_op(X.p, X.gs, X.ld, 1, X.by_member);
  g.B = simt_op(Wl, static_cast<long long>(sh.stride), out, 1, 0);
  g.bias = simt_op(W + sh.boff[l], static_cast<long long>(sh.stride), 0, 1, 0);
  g.C = Y;
  g.c_gs = y_gs;
  g.c_rs = y_ld;
  g.epi = epi;
  g.acc_init = -0.0f;  // "first product assigned" (pop_tensor.hpp:158-160)
  g.active = active;
  g.C2 = C2;
  g.c2_gs = c2_gs;
  g.c2_rs = c2_ld;
  g.scale = sh.out_scale;
  if (noise) {
    g.noise_key = key_a.p;
    g.noise_sd = h_f2.p;
    g.noise_clip = h_f3.p;
    g.bound = bound;
    if (use_tc() && algo == PBRL_ALGO_TD3 && out == da) {  // precomputed by launch_td3_target_noise
      g.noise_eps = S.tnoise.p;
      g.ne_gs = static_cast<long long>(B) * da;
    }
  }
  timed(PC_GEMM_FWD, flops, bytes, active != nullptr, [&] {
    if (out <= 16) launch_fwd_skinny(g, stream);
    else launch_gemm_simt(g, stream);
  });
  if (ymask && ymask->mask && epi == EPI_BIAS_RELU) {
    timed(PC_ELEM, 0.0, 0.0, active != nullptr, [&] {
      launch_mask_bits(groups, B, out, Y, y_gs, y_ld, ymask->mask, ymask->mgs, ymask->mld, active,
                       n, stream);
    });
  }
}

// dX of layer l restricted to input columns [col0, col0+ncols): DX = epi(G W_l^T)
void Pop::gemm_dx(const NetShape& sh, const float* W, int l, int groups, int B, Mat G, Mat aux,
                  float* DX, long long dx_gs, long long dx_ld, int epi, int col0, int ncols,
                  const int* active, float scale) {
  const int out = sh.dims[l + 1];
  const float* Wc = W + sh.woff[l] + static_cast<size_t>(col0) * out;
  const double flops = 2.0 * B * out * ncols * groups;
  // algorithmic bytes: G, the W columns, DX, the ReLU' mask bits (or the tanh values)
  const double ae = aeb(), de = epi == EPI_RELU_MASK ? ae : 4.0;
  const double bytes =
      ae * groups * (static_cast<double>(B) * out + static_cast<double>(out) * ncols) +
      de * groups * static_cast<double>(B) * ncols +
      (epi == EPI_RELU_MASK ? groups * B * ((ncols + 31) / 32) * 4.0
                            : (epi == EPI_TANH_GRAD ? 4.0 * groups * B * ncols : 0.0));
  const int eb = aeb();
  const void* Wco = use_tc() ? wop(Wc) : Wc;
  if (use_tc() && out >= 8 && tma_ok(G.p, G.ld, G.gs, eb) && tma_ok(Wco, out, sh.stride, eb)) {
    TcOperand A{G.p, static_cast<uint64_t>(out), static_cast<uint64_t>(B),
                static_cast<uint64_t>(groups), static_cast<uint64_t>(G.ld),
                static_cast<uint64_t>(G.gs)};
    TcOperand Bw{Wco, static_cast<uint64_t>(out), static_cast<uint64_t>(ncols),
                 static_cast<uint64_t>(groups), static_cast<uint64_t>(out), sh.stride};
    TcArgs a;
    a.eb = eb;
    a.c16 = act16() && epi == EPI_RELU_MASK ? 1 : 0;  // hidden cotangents are activations
    a.M = B;
    a.N = ncols;
    a.K = out;
    a.groups = groups;
    a.n_members = n;
    a.epi = epi;
    a.C = DX;
    a.c_gs = dx_gs;
    a.c_rs = dx_ld;
    a.aux = aux.p;
    a.aux_gs = aux.gs;
    a.aux_rs = aux.ld;
    a.aux_by_member = aux.by_member;
    if (epi == EPI_RELU_MASK && aux.mask) {
      a.mask_in = aux.mask;
      a.mi_gs = aux.mgs;
      a.mi_ld = aux.mld;
      a.mi_by_member = aux.by_member;
    }
    a.scale = scale;
    a.active = active;
    a.b_prefetch = tc_prefetch_ok() ? 1 : 0;
    a.max_ctas = cta_cap;
    timed(PC_GEMM_DX, flops, bytes, active != nullptr,
          [&] { launch_tc_gemm(A, Bw, false, false, a, stream); });
    return;
  }
  if (act16()) PBRL_THROW(PBRL_E_CONFIG, "bf16 mode: dX product without a tensor-core shape");
  GemmArgs g;
  g.M = B;
  g.N = ncols;
  g.K = out;
  g.groups = groups;
  g.n_members = n;
  g.A = simt_op(G.p, G.gs, G.ld, 1, G.by_member);
  g.B = simt_op(Wc, static_cast<long long>(sh.stride), 1, out, 0);
  g.C = DX;
  g.c_gs = dx_gs;
  g.c_rs = dx_ld;
  g.epi = epi;
  g.aux = simt_op(aux.p, aux.gs, aux.ld, 1, aux.by_member);
  g.acc_init = 0.0f;
  g.active = active;
  g.scale = scale;
  timed(PC_GEMM_DX, flops, bytes, active != nullptr, [&] {
    if (out <= 16) launch_dx_skinny(g, stream);
    else launch_gemm_simt(g, stream);
  });
}

// dW_l and db_l into the gradient arena rows: dW = X^T G, db = column sums of G
void Pop::gemm_dw(const NetShape& sh, float* Gr, int l, int groups, int B, Mat X, Mat G,
                  const int* active, bool bias_done, int max_ctas) {
  const int in = sh.dims[l], out = sh.dims[l + 1];
  const double flops = 2.0 * B * in * out * groups;
  // algorithmic bytes: X (once per member when shared), G, dW
  const double ae = aeb();
  const double bytes = ae * (static_cast<double>(B) * in * (X.by_member ? n : groups) +
                             static_cast<double>(groups) * B * out) +
                       4.0 * groups * in * out;
  const int eb = aeb();
  if (use_tc() && out >= 32 && tma_ok(X.p, X.ld, X.gs, eb) && tma_ok(G.p, G.ld, G.gs, eb)) {
    // input block with a ones column at index `in`: one more output row = the bias gradient
    const int mrows = (X.ones_col == in && in + 1 <= X.ld) ? in + 1 : in;
    if (mrows > in) bias_done = true;
    TcOperand A{X.p, static_cast<uint64_t>(mrows), static_cast<uint64_t>(B),
                static_cast<uint64_t>(X.by_member ? n : groups), static_cast<uint64_t>(X.ld),
                static_cast<uint64_t>(X.gs)};
    TcOperand Bg{G.p, static_cast<uint64_t>(out), static_cast<uint64_t>(B),
                 static_cast<uint64_t>(groups), static_cast<uint64_t>(G.ld),
                 static_cast<uint64_t>(G.gs)};
    TcArgs a;
    a.eb = eb;
    a.M = mrows;
    a.N = out;
    a.K = B;
    a.groups = groups;
    a.n_members = n;
    a.a_by_member = X.by_member;
    a.epi = EPI_STORE;
    a.C = Gr + sh.woff[l];
    a.c_gs = static_cast<long long>(sh.stride);
    a.c_rs = out;
    a.active = active;
    a.max_ctas = max_ctas ? max_ctas : cta_cap;
    timed(PC_GEMM_DW, flops, bytes, active != nullptr,
          [&] { launch_tc_gemm(A, Bg, true, true, a, stream); });
    // bias gradient: per-column sums of G in row order (pop_add_bias_backward, :236-250),
    // unless the kernel that produced G already wrote them
    if (!bias_done) timed(PC_ELEM, 0.0, 4.0 * B * out * groups, active != nullptr, [&] {
      launch_colsum(groups, n, B, out, G.p, G.gs, G.ld, Gr + sh.boff[l],
                    static_cast<long long>(sh.stride), active, act16() ? 1 : 0, stream);
    });
    return;
  }
  if (act16()) PBRL_THROW(PBRL_E_CONFIG, "bf16 mode: dW product without a tensor-core shape");
  GemmArgs g;
  g.M = in + 1;  // ones row: C row `in` = column sums of G = the bias gradient (row order)
  g.N = out;
  g.K = B;
  g.groups = groups;
  g.n_members = n;
  g.A = simt_op(X.p, X.gs, 1, X.ld, X.by_member);
  g.a_ones_row = 1;
  g.B = simt_op(G.p, G.gs, G.ld, 1, G.by_member);
  g.C = Gr + sh.woff[l];
  g.c_gs = static_cast<long long>(sh.stride);
  g.c_rs = out;
  g.epi = EPI_STORE;
  g.acc_init = 0.0f;
  g.active = active;
  timed(PC_GEMM_DW, flops, bytes + 4.0 * groups * out, active != nullptr, [&] {
    if (out <= 16) launch_dw_skinny(g, stream);
    else launch_gemm_simt(g, stream);
  });
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
    snprintf(buf, sizeof(buf),
             "%s\"%s\": {\"launches\": %lld, \"ms\": %.6f, \"flops\": %.6e, \"bytes\": %.6e}",
             c ? ", " : "", names[c], cnt[c], ms[c], fl[c], by[c]);
    out += buf;
  }
  out += "}}";
  return out;
}

// ------------------------------------------------------------------ shared building blocks
// hidden-activation buffers hold [rows][ld] floats followed (TF32 mode) by the ReLU mask bits
// [rows][ceil(H / 32)] (ensure_scratch sizes them)
Mat Pop::hid(std::vector<DBuf<float>>& v, int l, int B, const NetShape& sh, int by_member) {
  const int H = sh.dims[l + 1];
  const int ld = padl(H);
  Mat m{v[l].p, static_cast<long long>(B) * ld, ld, by_member};
  if (use_tc()) {
    const long long mw = (H + 31) / 32;
    const long long rows = static_cast<long long>(v[l].count) / (ld + mw);
    m.mask = reinterpret_cast<uint32_t*>(aoff(v[l].p, rows * ld));
    m.mgs = static_cast<long long>(B) * mw;
    m.mld = mw;
  }
  return m;
}

// forward of `sh` (groups x B rows) from input x; hidden activations into hs[l]
void Pop::mlp_forward(const NetShape& sh, const float* W, int groups, int B, Mat x,
                      std::vector<DBuf<float>>& hs, float* out, long long out_gs, long long out_ld,
                      int last_epi, const int* active, float* C2, long long c2_gs,
                      long long c2_ld, bool noise, bool keep_hidden, bool out_act) {
  const int L = sh.depth;
  if (mlp_forward2(sh, W, groups, B, x, hs, out, out_gs, out_ld, last_epi, active, C2, c2_gs,
                   c2_ld, noise, keep_hidden, out_act))
    return;  // both hidden layers and the output layer in one launch (BF16 mode)
  for (int l = 0; l < L; ++l) {
    if (l == L - 1) {
      gemm_fwd(sh, W, l, groups, B, x, out, out_gs, out_ld, last_epi, active, C2, c2_gs, c2_ld,
               noise, nullptr, out_act);
    } else {
      const Mat h = hid(hs, l, B, sh, 0);
      if (l == L - 2 && gemm_fwd_fused(sh, W, l, groups, B, x, h, keep_hidden, out, out_gs, out_ld,
                                       last_epi, active, C2, c2_gs, c2_ld, noise, out_act))
        return;  // the output layer ran in this layer's epilogue
      gemm_fwd(sh, W, l, groups, B, x, const_cast<float*>(h.p), h.gs, h.ld, EPI_BIAS_RELU, active,
               nullptr, 0, 0, false, keep_hidden ? &h : nullptr);
      x = h;
    }
  }
}

// BF16 mode, two hidden layers: the whole forward in one launch (launch_mlp_fwd2); h1 stays in
// shared memory and reaches HBM (with h2 and the mask bits) only when the backward needs it.
bool Pop::mlp_forward2(const NetShape& sh, const float* W, int groups, int B, Mat x,
                       std::vector<DBuf<float>>& hs, float* out, long long out_gs,
                       long long out_ld, int last_epi, const int* active, float* C2,
                       long long c2_gs, long long c2_ld, bool noise, bool keep_hidden,
                       bool out_act) {
  if (!act16() || sh.depth != 3 || fwd2_off) return false;
  Fwd2Args a;
  a.M = B;
  a.in = sh.dims[0];
  a.H1 = sh.dims[1];
  a.H2 = sh.dims[2];
  a.nout = sh.dims[3];
  a.groups = groups;
  a.n_members = n;
  a.X = x.p;
  a.x_ld = x.ld;
  a.x_gs = x.gs;
  a.x_by_member = x.by_member;
  a.W1 = wop(W + sh.woff[0]);
  a.W2 = wop(W + sh.woff[1]);
  a.w_gs = static_cast<long long>(sh.stride);
  a.b1 = W + sh.boff[0];
  a.b2 = W + sh.boff[1];
  a.ow = W + sh.woff[2];
  a.p_gs = static_cast<long long>(sh.stride);
  a.out_epi = last_epi;
  a.out_scale = sh.out_scale;
  a.oC = out;
  a.oc_gs = out_gs;
  a.oc_rs = out_ld;
  a.oc16 = out_act ? 1 : 0;
  a.oC2 = C2;
  a.oc2_gs = c2_gs;
  a.oc2_rs = c2_ld;
  Mat h1{}, h2{};
  if (keep_hidden) {
    h1 = hid(hs, 0, B, sh, 0);
    h2 = hid(hs, 1, B, sh, 0);
    a.H1g = const_cast<float*>(h1.p);
    a.h1_gs = h1.gs;
    a.h1_ld = h1.ld;
    a.m1 = h1.mask;
    a.m1_gs = h1.mgs;
    a.m1_ld = h1.mld;
    a.H2g = const_cast<float*>(h2.p);
    a.h2_gs = h2.gs;
    a.h2_ld = h2.ld;
    // h2's mask bits only when the output layer's backward is a tensor-core dX product (the
    // output-layer backward kernel, mlp_backward's condition, reads ReLU' from the values;
    // the layer-1 dX epilogues read h1's bits)
    const bool out_bwd_kernel =
        sh.dims[3] <= 16 && static_cast<long long>(B) * sh.dims[3] <= 32768;
    a.m2 = out_bwd_kernel ? nullptr : h2.mask;
    a.m2_gs = h2.mgs;
    a.m2_ld = h2.mld;
  }
  a.active = active;
  if (noise) {
    a.noise_key = key_a.p;
    a.noise_sd = h_f2.p;
    a.noise_clip = h_f3.p;
    a.bound = bound;
    if (algo == PBRL_ALGO_TD3 && a.nout == da) {  // precomputed by launch_td3_target_noise
      a.noise_eps = S.tnoise.p;
      a.ne_gs = static_cast<long long>(B) * da;
      a.ne_rs = da;
    }
  }
  if (!mlp_fwd2_ok(a)) return false;
  const int in = a.in, H1 = a.H1, H2 = a.H2, no = a.nout;
  const double flops = 2.0 * B * groups * (static_cast<double>(in) * H1 + H1 * H2 + H2 * no);
  const double bytes =
      2.0 * (static_cast<double>(B) * in * (x.by_member ? n : groups) +
             static_cast<double>(groups) * (in * H1 + H1 * H2)) +
      4.0 * groups * (H1 + H2 + H2 * no + no) + (out_act ? 2.0 : 4.0) * groups * B * no +
      (keep_hidden ? groups * B * (2.0 * (H1 + H2) + 4.0 * ((H1 + 31) / 32 + (H2 + 31) / 32))
                   : 0.0);
  a.max_ctas = cta_cap;
  timed(PC_GEMM_FWD, flops, bytes, active != nullptr, [&] { launch_mlp_fwd2(a, stream); });
  return true;
}

// Last hidden layer + output layer in one tcgen05 launch (TF32 mode): the output layer's few
// columns (1 or 2*act) are evaluated from the hidden row in the epilogue; the hidden activation
// is written only when the backward pass needs it.  Returns false when not applicable.
bool Pop::gemm_fwd_fused(const NetShape& sh, const float* W, int l, int groups, int B, Mat X,
                         Mat H, bool keep_hidden, float* Y, long long y_gs, long long y_ld,
                         int out_epi, const int* active, float* C2, long long c2_gs,
                         long long c2_ld, bool noise, bool out_act) {
  const int in = sh.dims[l], hdim = sh.dims[l + 1], nout = sh.dims[l + 2];
  const int eb = aeb();
  const float* Wl = W + sh.woff[l];
  const void* Wo = use_tc() ? wop(Wl) : Wl;
  if (!use_tc() || hdim < 16 || hdim > 256 || nout > 16 || !tma_ok(X.p, X.ld, X.gs, eb) ||
      !tma_ok(Wo, hdim, sh.stride, eb))
    return false;
  TcOperand A{X.p, static_cast<uint64_t>(in), static_cast<uint64_t>(B),
              static_cast<uint64_t>(X.by_member ? n : groups), static_cast<uint64_t>(X.ld),
              static_cast<uint64_t>(X.gs)};
  TcOperand Bw{Wo, static_cast<uint64_t>(hdim), static_cast<uint64_t>(in),
               static_cast<uint64_t>(groups), static_cast<uint64_t>(hdim), sh.stride};
  TcArgs a;
  a.eb = eb;
  a.c16 = act16() ? 1 : 0;
  a.oc16 = act16() && out_act ? 1 : 0;
  a.M = B;
  a.N = hdim;
  a.K = in;
  a.groups = groups;
  a.n_members = n;
  a.a_by_member = X.by_member;
  a.epi = EPI_BIAS_RELU;
  a.C = const_cast<float*>(H.p);
  a.c_gs = H.gs;
  a.c_rs = H.ld;
  a.bias = W + sh.boff[l];
  a.bias_gs = static_cast<long long>(sh.stride);
  a.active = active;
  a.nout = nout;
  a.ow = W + sh.woff[l + 1];
  a.ow_gs = static_cast<long long>(sh.stride);
  a.out_epi = out_epi;
  a.oC = Y;
  a.oc_gs = y_gs;
  a.oc_rs = y_ld;
  a.oC2 = C2;
  a.oc2_gs = c2_gs;
  a.oc2_rs = c2_ld;
  a.out_scale = sh.out_scale;
  a.store_hidden = keep_hidden ? 1 : 0;
  if (keep_hidden && H.mask) {
    a.mask_out = H.mask;
    a.mo_gs = H.mgs;
    a.mo_ld = H.mld;
  }
  if (noise) {
    a.noise_key = key_a.p;
    a.noise_sd = h_f2.p;
    a.noise_clip = h_f3.p;
    a.bound = bound;
    if (algo == PBRL_ALGO_TD3 && nout == da) {  // precomputed by launch_td3_target_noise
      a.noise_eps = S.tnoise.p;
      a.ne_gs = static_cast<long long>(B) * da;
      a.ne_rs = da;
    }
  }
  const double flops = 2.0 * B * groups * (static_cast<double>(in) * hdim + hdim * nout);
  const double ae = eb, oe = out_act ? ae : 4.0;
  const double bytes =
      ae * (static_cast<double>(B) * in * (X.by_member ? n : groups) +
            static_cast<double>(groups) * in * hdim) +
      4.0 * groups * (hdim + hdim * nout + nout) + oe * groups * B * nout +
      (keep_hidden ? groups * B * (ae * hdim + 4.0 * ((hdim + 31) / 32)) : 0.0);
  a.b_prefetch = tc_prefetch_ok() ? 1 : 0;
  a.max_ctas = cta_cap;
  timed(PC_GEMM_FWD, flops, bytes, active != nullptr,
        [&] { launch_tc_gemm(A, Bw, false, true, a, stream); });
  return true;
}

// backward of `sh` from the top cotangent G: dW for every layer, dX for layers > 0
void Pop::mlp_backward(const NetShape& sh, const float* W, float* Gr, int groups, int B, Mat G,
                       Mat x0, std::vector<DBuf<float>>& hs, std::vector<DBuf<float>>& dhs,
                       const int* active, const OutBwdArgs* top) {
  const int L = sh.depth;
  bool bias_done = false;  // the bias gradient of layer l was produced with its cotangent
  for (int l = L - 1; l >= 0; --l) {
    const Mat x = (l == 0) ? x0 : hid(hs, l - 1, B, sh, 0);
    if (l == L - 1 && sh.dims[L] <= 16 && static_cast<long long>(B) * sh.dims[L] <= 32768) {
      // output layer: dX (masked), dW and db in one pass over the hidden activations
      const int H = sh.dims[l], nout = sh.dims[L];
      OutBwdArgs a;
      a.act16 = act16() ? 1 : 0;
      a.B = B;
      a.H = H;
      a.nout = nout;
      a.groups = groups;
      a.n_members = n;
      a.X = x.p;
      a.x_gs = x.gs;
      a.x_ld = x.ld;
      a.x_by_member = x.by_member;
      a.G = G.p;
      a.g_gs = G.gs;
      a.g_ld = G.ld;
      a.W = W + sh.woff[l];
      a.w_gs = static_cast<long long>(sh.stride);
      a.dW = Gr + sh.woff[l];
      a.dw_gs = static_cast<long long>(sh.stride);
      a.active = active;
      a.exact = use_tc() ? 0 : 1;
      if (top && top->top) {  // top cotangent (TD target / MSE / losses) fused into this launch
        a.top = top->top;
        a.q = top->q;
        a.r = top->r;
        a.d = top->d;
        a.tq = top->tq;
        a.gamma = top->gamma;
        a.y = top->y;
        a.loss = top->loss;
        a.norm_rows = top->norm_rows;
      }
      Mat dh{};
      if (l > 0) {
        dh = hid(dhs, l - 1, B, sh, 0);
        a.dX = const_cast<float*>(dh.p);  // activation buffer (fp32 or bf16)
        a.dx_gs = dh.gs;
        a.dx_ld = dh.ld;
        if (use_tc() && sh.dims[l] >= 32) {  // the tcgen05 dW of layer l-1 skips its colsum
          a.dbx = Gr + sh.boff[l - 1];
          a.dbx_gs = static_cast<long long>(sh.stride);
        }
      }
      // algorithmic bytes: X, G, W, dW + db, dX (+ the fused bias gradient below)
      const double obytes =
          aeb() * (static_cast<double>(B) * H * (x.by_member ? n : groups) +
                   (l > 0 ? static_cast<double>(groups) * B * H : 0.0)) +
          4.0 * groups * (B * nout + 2.0 * (H * nout + nout) + (l > 0 ? H : 0));
      timed(PC_GEMM_DW, 2.0 * B * H * nout * groups * (l > 0 ? 2.0 : 1.0), obytes,
            active != nullptr, [&] { launch_out_backward(a, stream); });
      G = dh;
      bias_done = a.dbx != nullptr;
      continue;
    }
    if (l == 1 && L == 3 && dw_fork_ok()) {
      // graph mode: after the dX product, the two weight-gradient products are independent --
      // dW1 (h1^T dh2) keeps most of the SMs on the main branch while dW0 (x0^T dh1, a few small
      // tiles) runs on a parallel branch on the rest (capped persistent grids co-reside, so
      // dW0 leaves the critical path instead of trailing dW1)
      const Mat dh = hid(dhs, 0, B, sh, 0);
      gemm_dx(sh, W, 1, groups, B, G, x, const_cast<float*>(dh.p), dh.gs, dh.ld, EPI_RELU_MASK,
              0, sh.dims[1], active, 1.0f);
      const int fi = in_cond_body ? 1 : 0;
      cudaStream_t& sd = side3[fi];
      if (!sd) CUDA_CHECK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
      if (!ev_f3[fi]) {
        for (cudaEvent_t* e : {&ev_f3[fi], &ev_j3[fi]})
          CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      }
      static const int side_ctas = std::getenv("PBRL_DW_SIDE") ? std::atoi(std::getenv("PBRL_DW_SIDE"))
                                                               : kDwSideCtas;
      CUDA_CHECK(cudaEventRecord(ev_f3[fi], stream));
      CUDA_CHECK(cudaStreamWaitEvent(sd, ev_f3[fi], 0));
      std::swap(stream, sd);
      fork_window(stream);
      gemm_dw(sh, Gr, 0, groups, B, x0, dh, active, false, side_ctas);
      std::swap(stream, sd);
      CUDA_CHECK(cudaEventRecord(ev_j3[fi], sd));
      gemm_dw(sh, Gr, 1, groups, B, x, G, active, bias_done, num_sms_host() - side_ctas);
      CUDA_CHECK(cudaStreamWaitEvent(stream, ev_j3[fi], 0));
      return;
    }
    if (l > 0) {
      const Mat dh = hid(dhs, l - 1, B, sh, 0);
      gemm_dx(sh, W, l, groups, B, G, x, const_cast<float*>(dh.p), dh.gs, dh.ld, EPI_RELU_MASK,
              0, sh.dims[l], active, 1.0f);
      gemm_dw(sh, Gr, l, groups, B, x, G, active, bias_done);
      G = dh;
    } else {
      gemm_dw(sh, Gr, l, groups, B, x, G, active, bias_done);
    }
    bias_done = false;
  }
}

// critic dX chain from the output cotangent down to the action columns of the input
void Pop::critic_dx_to_action(int groups, int B, Mat G, std::vector<DBuf<float>>& hs,
                              std::vector<DBuf<float>>& dhs, float* out, long long out_ld,
                              int epi, Mat aux, float scale, const int* active, const OutBwdArgs* top) {
  const int L = cri.depth;
  for (int l = L - 1; l >= 1; --l) {
    const Mat mask = hid(hs, l - 1, B, cri, 0);
    const Mat dh = hid(dhs, l - 1, B, cri, 0);
    if (l == 1 && gemm_dx_to_action(groups, B, G, mask, out, out_ld, epi, aux, scale, active))
      return;  // this layer's dX and the action-column dX of the input layer in one launch
    if (l == L - 1 && use_tc() && cri.dims[L] <= 16) {
      // output layer (N_out = 1): dX = relu'(h) * (G W_out^T) by the output-layer backward
      // kernel without its weight gradients (the policy loss discards them, algos.hpp:330-334)
      const int H = cri.dims[l];
      OutBwdArgs a;
      a.act16 = act16() ? 1 : 0;
      a.B = B;
      a.H = H;
      a.nout = cri.dims[L];
      a.groups = groups;
      a.n_members = n;
      a.X = mask.p;
      a.x_gs = mask.gs;
      a.x_ld = mask.ld;
      a.G = G.p;
      a.g_gs = G.gs;
      a.g_ld = G.ld;
      a.W = cri_p.p + cri.woff[l];
      a.w_gs = static_cast<long long>(cri.stride);
      a.dX = const_cast<float*>(dh.p);
      a.dx_gs = dh.gs;
      a.dx_ld = dh.ld;
      a.active = active;
      a.exact = 0;
      if (top && top->top) {
        a.top = top->top;
        a.q = top->q;
        a.loss = top->loss;
      }
      const double obytes = 4.0 * groups *
          (static_cast<double>(B) * a.nout + H * a.nout) + 2.0 * aeb() * groups * B * H;
      timed(PC_GEMM_DX, 2.0 * B * H * a.nout * groups, obytes, active != nullptr,
            [&] { launch_out_backward(a, stream); });
      G = dh;
      continue;
    }
    gemm_dx(cri, cri_p.p, l, groups, B, G, mask, const_cast<float*>(dh.p), dh.gs, dh.ld,
            EPI_RELU_MASK, 0, cri.dims[l], active, 1.0f);
    G = dh;
  }
  gemm_dx(cri, cri_p.p, 0, groups, B, G, aux, out, static_cast<long long>(B) * out_ld, out_ld,
          epi, ds, da, active, scale);
}

// Tensor-core modes: the first hidden layer's dX and the input layer's action-column dX in one
// launch -- dh1 = relu'(h1) (G W1^T) stays in the epilogue registers and is contracted on CUDA
// cores with the action rows of W0 (a_grad[o] = sum_j dh1[j] W0[ds + o][j]) then the tanh
// backward (or a plain store); dh1 never reaches HBM.  Returns false when not applicable.
bool Pop::gemm_dx_to_action(int groups, int B, Mat G, Mat mask, float* out, long long out_ld,
                            int epi, Mat aux, float scale, const int* active) {
  const int H = cri.dims[1], Hn = cri.dims[2];
  const int eb = aeb();
  const float* W1 = cri_p.p + cri.woff[1];
  const void* W1o = wop(W1);
  if (!use_tc() || H > 256 || H < 32 || da > 16 || Hn < 8 || !mask.mask ||
      !tma_ok(G.p, G.ld, G.gs, eb) || !tma_ok(W1o, Hn, cri.stride, eb))
    return false;
  TcOperand A{G.p, static_cast<uint64_t>(Hn), static_cast<uint64_t>(B),
              static_cast<uint64_t>(groups), static_cast<uint64_t>(G.ld),
              static_cast<uint64_t>(G.gs)};
  TcOperand Bw{W1o, static_cast<uint64_t>(Hn), static_cast<uint64_t>(H),
               static_cast<uint64_t>(groups), static_cast<uint64_t>(Hn), cri.stride};
  TcArgs a;
  a.eb = eb;
  a.M = B;
  a.N = H;
  a.K = Hn;
  a.groups = groups;
  a.n_members = n;
  a.epi = EPI_RELU_MASK;
  a.mask_in = mask.mask;
  a.mi_gs = mask.mgs;
  a.mi_ld = mask.mld;
  a.mi_by_member = mask.by_member;
  a.store_hidden = 0;
  a.nout = da;
  a.ow = cri_p.p + cri.woff[0] + static_cast<size_t>(ds) * H;
  a.ow_gs = static_cast<long long>(cri.stride);
  a.ow_tr = 1;
  a.ow_ld = H;
  a.out_epi = epi;
  a.oC = out;
  a.oc_gs = static_cast<long long>(B) * out_ld;
  a.oc_rs = out_ld;
  a.aux = aux.p;
  a.aux_gs = aux.gs;
  a.aux_rs = aux.ld;
  a.aux_by_member = aux.by_member;
  a.scale = scale;
  a.active = active;
  a.b_prefetch = tc_prefetch_ok() ? 1 : 0;
  a.max_ctas = cta_cap;
  const double flops = 2.0 * B * groups * (static_cast<double>(Hn) * H + H * da);
  const double bytes = eb * groups * (static_cast<double>(B) * Hn + static_cast<double>(Hn) * H) +
                       4.0 * groups * (B * ((H + 31) / 32) + H * da + 2.0 * B * da);
  timed(PC_GEMM_DX, flops, bytes, active != nullptr,
        [&] { launch_tc_gemm(A, Bw, false, false, a, stream); });
  return true;
}

// Twin critics as one grouped problem of 2n groups: forward on [s|a], MSE cotangent,
// backward, fused Adam + target Polyak (algos.hpp:369-377, :401-418).
void Pop::critic_forward(int B0) {
  CriticFold f(*this, B0);  // shared critic: 2 groups of n*B rows
  const int B = f.B;
  const Mat x0{S.in_sa.p, static_cast<long long>(B) * lsa, lsa, 1};
  mlp_forward(cri, cri_p.p, 2 * n, B, x0, S.ch, S.q.p, B, 1, EPI_BIAS);
}

void Pop::critic_update(int B0, const int* polyak_gate, bool forward_done) {
  CriticFold f(*this, B0);
  const int B = f.B;
  // shared critic: its target Polyak runs when some member fires (cmask {1}, :407-418)
  if (shared && polyak_gate) polyak_gate = fire.p + f.n0;
  const int nrows = shared ? static_cast<int>(mse_rows(B0)) : 0;
  const int n2 = 2 * n;
  Mat x0{S.in_sa.p, static_cast<long long>(B) * lsa, lsa, 1};
  if (use_tc() && lsa > ds + da) x0.ones_col = ds + da;  // see Pop::ensure_ones
  if (!forward_done) critic_forward(B);
  // tensor-core modes: the TD target (TD3) and mse_loss_grads run inside the output-layer
  // backward; FFMA32 keeps the separate kernels (the reference's operation order).  A shared
  // critic takes y from k_td_target (its gamma is per policy member, not per critic group).
  OutBwdArgs top;
  if (use_tc() && cri.dims[cri.depth] == 1 && B <= 32768) {
    top.top = algo == PBRL_ALGO_TD3 && !shared ? 1 : 2;
    top.q = S.q.p;
    top.r = S.r.p;
    top.d = S.d.p;
    top.tq = S.tq_out.p;
    top.gamma = h_f4.p;
    top.y = S.y.p;
    top.loss = losses.p;
    top.norm_rows = nrows;
  } else {
    timed(PC_ELEM, 0.0, 0.0, 0,
          [&] { launch_mse(n2, n, B, S.q.p, S.y.p, S.dq.p, losses.p, stream, nrows); });
  }
  const float* clr = algo == PBRL_ALGO_TD3 ? h_f0.p : h_f1.p;
  mlp_backward(cri, cri_p.p, cri_g.p, n2, B, Mat{S.dq.p, B, 1, 0}, x0, S.ch, S.dh, nullptr,
               &top);
  if (shared && comm_reduce) {
    // one critic replica per shard: the gradient of the whole folded population is the sum of
    // the shards' (each scaled by 2 / (n_global B)); the target-Polyak gate is "some member of
    // any shard fires"
    comm_reduce(cri_g.p, cri_g.count, stream);
    if (polyak_gate) {
      flag_f.alloc(1);
      int* fl = const_cast<int*>(polyak_gate);
      launch_flag_convert(fl, flag_f.p, 1, stream);
      comm_reduce(flag_f.p, 1, stream);
      launch_flag_convert(fl, flag_f.p, 0, stream);
      count_launch(2);
    }
  }
  if (pre_adam) {  // TD3 graph mode: the policy forward forks off beside the critic Adam
    CriticUnfold u(*this);
    pre_adam();
  }
  if (stage_mark == 1) mark_stage_free();
  // 28 B/param Adam (+2 B/param bf16 operand copy in BF16 mode)
  const double cP = static_cast<double>(cri.P);
  timed(PC_ADAM, 0.0, cP * n2 * (act16() ? 30.0 : 28.0), 0, [&] {
    launch_adam(n2, n, cri.P, cri.stride, cri_p.p, cri_m.p, cri_v.p, cri_g.p, t_cri.p, corr1.p,
                corr2.p, clr, nullptr, cri_t.p, h_f5.p, h_f6.p, polyak_gate, cri_p16.p,
                cri_t16.p, stream);
  });
  // fused target Polyak: +8 B/param (read + write target), every member (SAC) or fired (TD3)
  const double pb = act16() ? 10.0 : 8.0;
  if (polyak_gate) prof_add_gated_bytes(pb * cP * n2);
  else if (prof_on && !prof.empty()) prof.back().bytes += pb * cP * n2;
}

// the tensor-core modes compute the TD target inside the critic's output-layer backward
bool Pop::td_target_fused(int B) const {
  return use_tc() && cri.dims[cri.depth] == 1 && crows(B) <= 32768 && !shared;
}

// ------------------------------------------------------------------ TD3 step (algos.hpp:351-422)
// Graph capture: append an IF node on `h` at the current capture point of `stream` and capture
// body() into its body graph (on cap, a stream of its own).
static size_t kernel_nodes(cudaGraph_t g);

template <typename F>
void Pop::capture_if(cudaGraphConditionalHandle h, cudaStream_t& cap, F&& body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CUDA_CHECK(cudaStreamGetCaptureInfo_v3(stream, &st, nullptr, &g, &deps, nullptr, &nd));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CUDA_CHECK(cudaGraphAddNode(&node, g, deps, nd, &cp));
  CUDA_CHECK(cudaStreamUpdateCaptureDependencies(stream, &node, 1,
                                                 cudaStreamSetCaptureDependencies));
  if (!cap) CUDA_CHECK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t bg = cp.conditional.phGraph_out[0];
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(cap, bg, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
  const cudaStream_t outer = stream, inner = cap;
  std::swap(stream, cap);
  wwin[stream] = true;  // conservative: the body's first kernels do not prefetch weights
  in_cond_body = true;
  try {
    body();
  } catch (...) {
    // a throw may leave a fork unjoined or the member stream swapped with a branch: restore
    // the streams, end the body capture and clear its error before rethrowing
    in_cond_body = false;
    stream = outer;
    cap = inner;
    cudaGraph_t part = nullptr;
    cudaStreamEndCapture(cap, &part);
    (void)cudaGetLastError();
    throw;
  }
  in_cond_body = false;
  std::swap(stream, cap);
  CUDA_CHECK(cudaStreamEndCapture(cap, &bg));
  cond_body_nodes += kernel_nodes(bg);
  ++cond_nodes;
}

// kernel nodes of a captured graph (event-record nodes and the conditional nodes themselves are
// not kernel launches)
static size_t kernel_nodes(cudaGraph_t g) {
  size_t nb = 0;
  CUDA_CHECK(cudaGraphGetNodes(g, nullptr, &nb));
  std::vector<cudaGraphNode_t> nodes(nb);
  if (nb) CUDA_CHECK(cudaGraphGetNodes(g, nodes.data(), &nb));
  size_t k = 0;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    CUDA_CHECK(cudaGraphNodeGetType(nd, &t));
    k += t == cudaGraphNodeTypeKernel ? 1 : 0;
  }
  return k;
}

void Pop::td3_step(int B, const uint8_t* d_mask) {
  const long long nbB = B;
  // graph capture: the policy half of the step sits in conditional IF nodes whose condition
  // k_td3_step_begin sets when any member fires (steps where no policy fires replay only the
  // critic half); eager mode runs it with every launch gated per member instead
  const bool fork = capturing && use_tc();
  // the fire-step graph (cap_fire) has no conditional node: the host mirror predicted that some
  // policy fires, and every policy-half launch is gated per member by the device fire mask
  const bool cond = capturing && !cap_fire && cond_graph();
  const bool guarded = capturing && !cap_fire && !cond;  // non-fire graph, no policy half
  cudaGraphConditionalHandle any_fire = 0;
  if (cond) {
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    CUDA_CHECK(cudaStreamGetCaptureInfo(stream, &st, nullptr, &g, nullptr, nullptr));
    CUDA_CHECK(cudaGraphConditionalHandleCreate(&any_fire, g, 0, cudaGraphCondAssignDefault));
  }
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    launch_td3_step_begin(n, delay_acc.p, h_d0.p, d_mask, fire.p, t_pol.p, t_cri.p,
                          t_cri.p + ncrit, steps.p, streams.p, seed, key_a.p, losses.p + 2 * n,
                          any_fire, cond ? 1 : 0, shared ? 1 : 0, ncrit, stream,
                          guarded ? guard_d : nullptr, hist_on ? loss_hist.p : nullptr,
                          hist_base.p, static_cast<int>(kLossHist));
  });
  // graph mode: the online critics' forward on [s | a] does not depend on the target chain, so
  // it runs on a parallel graph branch (its tiles fill the target chain's partial waves)
  if (fork) {
    if (!side2) CUDA_CHECK(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
    if (!ev_fork) {
      for (cudaEvent_t* e : {&ev_fork, &ev_join})
        CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    CUDA_CHECK(cudaEventRecord(ev_fork, stream));
    CUDA_CHECK(cudaStreamWaitEvent(side2, ev_fork, 0));
    std::swap(stream, side2);
    fork_window(stream);  // full dependency on the fork point: nothing in flight
    // the two branches run side by side on disjoint SM sets (capped persistent grids)
    cta_cap = fwd_split(B);
    critic_forward(B);
    std::swap(stream, side2);
    CUDA_CHECK(cudaEventRecord(ev_join, side2));
    cta_cap = fwd_split(B) ? num_sms_host() - fwd_split(B) : 0;
  }
  // td3_critic_target (algos.hpp:241-282): pi'(s2) + clipped noise, twin target critics, y
  if (use_tc()) {
    timed(PC_ELEM, 0.0, 0.0, 0, [&] {
      launch_td3_target_noise(n, B, da, key_a.p, h_f2.p, h_f3.p, S.tnoise.p, stream);
    });
  }
  const Mat s2{S.in_s2a.p, nbB * lsa, lsa, 0};
  mlp_forward(pol, pol_t.p, n, B, s2, S.tp_h, aoff(S.in_s2a.p, ds), nbB * lsa, lsa,
              EPI_BIAS_TANH_NOISE, nullptr, nullptr, 0, 0, true, false, true);
  {
    CriticFold f(*this, B);
    const long long cB = f.B;
    mlp_forward(cri, cri_t.p, 2 * n, f.B, Mat{S.in_s2a.p, cB * lsa, lsa, 1}, S.tq_h, S.tq_out.p,
                cB, 1, EPI_BIAS, nullptr, nullptr, 0, 0, false, false);
  }
  if (!td_target_fused(B))  // else fused (critic_update)
    timed(PC_ELEM, 0.0, 0.0, 0,
          [&] { launch_td_target(n, B, S.r.p, S.d.p, S.tq_out.p, h_f4.p, S.y.p, stream); });
  cta_cap = 0;
  if (fork) CUDA_CHECK(cudaStreamWaitEvent(stream, ev_join, 0));
  // twin critic update; target Polyak fused for members whose policy fires
  // graph mode, fused forward: the policy forward of the policy half depends only on the
  // policies (unchanged until the policy Adam), so it runs on a branch beside the critic Adam on
  // a few SMs (gated per member by the fire mask: near-empty when no policy fires); the branch
  // rejoins before the policy half
  bool pol_fwd_forked = false;
  static const bool fire_fork = std::getenv("PBRL_FIRE_POL_FORK") == nullptr ||
                                std::atoi(std::getenv("PBRL_FIRE_POL_FORK")) != 0;
  if (fork && pol_fork_ctas(B) > 0 && (cap_fire ? fire_fork : !fire_graphs())) {
    pre_adam = [&] {
      if (!side6) CUDA_CHECK(cudaStreamCreateWithFlags(&side6, cudaStreamNonBlocking));
      if (!ev_f6) {
        for (cudaEvent_t* e : {&ev_f6, &ev_j6})
          CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      }
      CUDA_CHECK(cudaEventRecord(ev_f6, stream));
      CUDA_CHECK(cudaStreamWaitEvent(side6, ev_f6, 0));
      std::swap(stream, side6);
      fork_window(stream);
      cta_cap = pol_fork_ctas(B);
      td3_policy_forward(B);
      cta_cap = 0;
      std::swap(stream, side6);
      CUDA_CHECK(cudaEventRecord(ev_j6, side6));
      pol_fwd_forked = true;
    };
  }
  // the non-fire graph reads its packed batch last in the critic backward, the fire-step graph
  // in the policy backward
  const bool mark = capturing && pack_overlap_ok() && (guarded || cap_fire);
  if (mark && guarded) stage_mark = 1;
  critic_update(B, fire.p, fork);
  pre_adam = nullptr;
  if (pol_fwd_forked) CUDA_CHECK(cudaStreamWaitEvent(stream, ev_j6, 0));
  pol_fwd_done = pol_fwd_forked;
  if (mark && cap_fire) stage_mark = 2;
  if (cond) capture_if(any_fire, side, [&] { td3_policy_half(B); });
  else if (cap_fire || (!capturing && eager_fires)) td3_policy_half(B);  // else: none fires
  stage_mark = 0;
  join_stage_free();
}

// independent-mode step graphs only (TD3: the two step graphs, not the conditional-node one):
// the shared critic and DvD (its pre-pass) keep the pack on the member stream
bool Pop::pack_overlap_ok() const {
  static const bool off = std::getenv("PBRL_NO_PACK_OVERLAP") != nullptr;
  if (off || shared || dvd.on || !use_graphs || prof_on) return false;
  return algo == PBRL_ALGO_SAC || (fire_graphs() && !cond_graph());
}

// capture: an external event-record node for ev_stage_free on a branch forked at the current
// point of the member stream (the next kernel keeps its programmatic edge to its predecessor)
void Pop::mark_stage_free() {
  if (!side_sf) CUDA_CHECK(cudaStreamCreateWithFlags(&side_sf, cudaStreamNonBlocking));
  if (!ev_stage_free) {
    for (cudaEvent_t* e : {&ev_stage_free, &ev_sf_fork, &ev_sf_join})
      CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  CUDA_CHECK(cudaEventRecord(ev_sf_fork, stream));
  CUDA_CHECK(cudaStreamWaitEvent(side_sf, ev_sf_fork, 0));
  CUDA_CHECK(cudaEventRecordWithFlags(ev_stage_free, side_sf, cudaEventRecordExternal));
  CUDA_CHECK(cudaEventRecord(ev_sf_join, side_sf));
  stage_joined = false;
  stage_ev_captured = true;
  stage_mark = 0;
}

void Pop::join_stage_free() {
  if (stage_joined) return;
  CUDA_CHECK(cudaStreamWaitEvent(stream, ev_sf_join, 0));
  stage_joined = true;
}

void Pop::td3_policy_forward(int B) {
  const long long nbB = B;
  const Mat s = policy_input(B);
  mlp_forward(pol, pol_p.p, n, B, s, S.ph, aoff(S.sa_pi.p, ds), nbB * lsa, lsa, EPI_BIAS_TANH,
              fire.p, S.pt.p, nbB * da, da, false, true, true);
}

// td3_policy_loss_grads (:318-338) on the UPDATED critic1, policy Adam and the target Polyak,
// every launch gated by the fire mask
void Pop::td3_policy_half(int B) {
  const long long nbB = B;
  const Mat s = policy_input(B);
  if (!pol_fwd_done) td3_policy_forward(B);
  pol_fwd_done = false;
  // critic1 on [s | pi(s)]; a shared critic runs every member's rows (folded, ungated)
  {
    CriticFold f(*this, B);
    const long long cB = f.B;
    mlp_forward(cri, cri_p.p, n, f.B, Mat{S.sa_pi.p, cB * lsa, lsa, 0}, S.qh, S.qpi.p, cB, 1,
                EPI_BIAS, shared ? nullptr : fire.p);
  }
  OutBwdArgs top;
  if (td_target_fused(B)) {  // fused: critic output-layer dX (the policy loss's -1/B)
    top.top = 3;
    top.q = S.qpi.p;
    top.loss = losses.p + 2 * n;
  } else {
    timed(PC_ELEM, 0.0, 0.0, 0, [&] {
      launch_td3_policy_loss(n, B, S.qpi.p, fire.p, losses.p + 2 * n, S.gq.p, stream);
    });
  }
  const int lt = pad4(da);
  {
    CriticFold f(*this, B);
    const long long cB = f.B;
    critic_dx_to_action(n, f.B, Mat{S.gq.p, cB, 1, 0}, S.qh, S.qdh, S.gtop.p, lt, EPI_TANH_GRAD,
                        Mat{S.pt.p, cB * da, da, 0}, pol.out_scale, shared ? nullptr : fire.p,
                        &top);
  }
  mlp_backward(pol, pol_p.p, pol_g.p, n, B, Mat{S.gtop.p, nbB * lt, lt, 0}, s, S.ph, S.pdh,
               fire.p, nullptr);
  if (dvd.on) {  // the DvD hook's gradient (computed by dvd_prepass before the step)
    const size_t cnt = static_cast<size_t>(n) * pol.stride;
    timed(PC_ELEM, 0.0, 12.0 * cnt, 0, [&] { launch_add_into(pol_g.p, dvd.grad.p, cnt, stream); });
  }
  if (stage_mark == 2) mark_stage_free();
  timed(PC_ADAM, 0.0, static_cast<double>(pol.P) * n * (act16() ? 40.0 : 36.0), 1, [&] {
    launch_adam(n, n, pol.P, pol.stride, pol_p.p, pol_m.p, pol_v.p, pol_g.p, t_pol.p, corr1.p,
                corr2.p, h_f1.p, fire.p, pol_t.p, h_f5.p, h_f6.p, nullptr, pol_p16.p, pol_t16.p,
                stream);
  });
}

// ------------------------------------------------------------------ SAC step (algos.hpp:781-837)
void Pop::sac_step(int B) {
  const int L = pol.depth;
  const long long nbB = B;
  const int hd = pol.dims[L];
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    launch_sac_step_begin(n, t_pol.p, t_cri.p, t_cri.p + n, t_alpha.p, steps.p, streams.p, seed,
                          key_a.p, key_b.p, stream);
  });
  // graph mode: the online critics' forward on [s | a] beside the target chain (split SMs), as in
  // td3_step
  const bool fork = capturing && use_tc();
  const int split = fork ? fwd_split(B) : 0;
  if (fork) {
    if (!side2) CUDA_CHECK(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
    if (!ev_fork) {
      for (cudaEvent_t* e : {&ev_fork, &ev_join})
        CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    CUDA_CHECK(cudaEventRecord(ev_fork, stream));
    CUDA_CHECK(cudaStreamWaitEvent(side2, ev_fork, 0));
    std::swap(stream, side2);
    fork_window(stream);
    cta_cap = split;
    critic_forward(B);
    std::swap(stream, side2);
    CUDA_CHECK(cudaEventRecord(ev_join, side2));
    cta_cap = split ? num_sms_host() - split : 0;
  }
  // sac_critic_target (algos.hpp:739-776): current policy on s2, eps' draws, twin targets
  mlp_forward(pol, pol_p.p, n, B, Mat{S.in_s2a.p, nbB * lsa, lsa, 0}, S.tp_h, S.head.p, nbB * hd,
              hd, EPI_BIAS, nullptr, nullptr, 0, 0, false, false);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    launch_sac_head(n, B, ds, da, lsa, S.head.p, key_b.p, bound, S.in_s2a.p, nullptr, nullptr,
                    nullptr, nullptr, nullptr, S.logp2.p, act16() ? 1 : 0, stream);
  });
  {
    CriticFold f(*this, B);
    const long long cB = f.B;
    mlp_forward(cri, cri_t.p, 2 * n, f.B, Mat{S.in_s2a.p, cB * lsa, lsa, 1}, S.tq_h, S.tq_out.p,
                cB, 1, EPI_BIAS, nullptr, nullptr, 0, 0, false, false);
  }
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    launch_sac_y(n, B, S.r.p, S.d.p, S.tq_out.p, S.logp2.p, log_alpha.p, h_f4.p, h_f3.p, S.y.p,
                 stream);
  });
  cta_cap = 0;
  if (fork) CUDA_CHECK(cudaStreamWaitEvent(stream, ev_join, 0));
  // sac_policy_loss_grads (:643-735): the policy forward + head on s depend only on the policy
  // (updated after this), so in graph mode they run on a branch beside the critic Adam
  const Mat s = policy_input(B);
  auto policy_head = [&] {
    mlp_forward(pol, pol_p.p, n, B, s, S.ph, S.head.p, nbB * hd, hd, EPI_BIAS);
    timed(PC_ELEM, 0.0, 0.0, 0, [&] {
      launch_sac_head(n, B, ds, da, lsa, S.head.p, key_a.p, bound, S.sa_pi.p, S.x.p, S.th.p,
                      S.ls.p, S.clamped.p, S.eps.p, S.logp.p, act16() ? 1 : 0, stream);
    });
  };
  bool pol_forked = false;
  if (fork && pol_fork_ctas(B) > 0) {
    pre_adam = [&] {
      if (!side6) CUDA_CHECK(cudaStreamCreateWithFlags(&side6, cudaStreamNonBlocking));
      if (!ev_f6) {
        for (cudaEvent_t* e : {&ev_f6, &ev_j6})
          CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      }
      CUDA_CHECK(cudaEventRecord(ev_f6, stream));
      CUDA_CHECK(cudaStreamWaitEvent(side6, ev_f6, 0));
      std::swap(stream, side6);
      fork_window(stream);
      cta_cap = pol_fork_ctas(B);
      policy_head();
      cta_cap = 0;
      std::swap(stream, side6);
      CUDA_CHECK(cudaEventRecord(ev_j6, side6));
      pol_forked = true;
    };
  }
  critic_update(B, nullptr, fork);  // critic targets tracked every step (:827-834)
  pre_adam = nullptr;
  if (pol_forked) CUDA_CHECK(cudaStreamWaitEvent(stream, ev_j6, 0));
  else policy_head();
  {
    CriticFold f(*this, B);
    const long long cB = f.B;
    mlp_forward(cri, cri_p.p, 2 * n, f.B, Mat{S.sa_pi.p, cB * lsa, lsa, 1}, S.qh, S.qpi.p, cB, 1,
                EPI_BIAS);
  }
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    launch_sac_policy_top(n, B, S.qpi.p, S.logp.p, log_alpha.p, losses.p + 2 * n, S.gq.p, S.lw.p,
                          stream);
  });
  {
    CriticFold f(*this, B);
    const long long cB = f.B;
    critic_dx_to_action(2 * n, f.B, Mat{S.gq.p, cB, 1, 0}, S.qh, S.qdh, S.ga.p, da, EPI_STORE,
                        Mat{}, 1.0f, nullptr);
  }
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    launch_sac_head_grad(n, B, da, S.ga.p, S.lw.p, S.x.p, S.th.p, S.ls.p, S.clamped.p, S.eps.p,
                         bound, S.gtop.p, stream);
  });
  mlp_backward(pol, pol_p.p, pol_g.p, n, B, Mat{S.gtop.p, nbB * hd, hd, 0}, s, S.ph, S.pdh,
               nullptr);
  // the policy backward is the step's last reader of its packed batch
  if (capturing && pack_overlap_ok()) mark_stage_free();
  timed(PC_ADAM, 0.0, static_cast<double>(pol.P) * n * 28.0, 0, [&] {
    launch_adam(n, n, pol.P, pol.stride, pol_p.p, pol_m.p, pol_v.p, pol_g.p, t_pol.p, corr1.p,
                corr2.p, h_f0.p, nullptr, nullptr, nullptr, nullptr, nullptr, pol_p16.p, nullptr,
                stream);
  });
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    launch_sac_alpha(n, B, S.logp.p, log_alpha.p, h_d0.p, log_alpha.p, alpha_m.p, alpha_v.p,
                     t_alpha.p, corr1.p, corr2.p, h_f2.p, stream);
  });
  join_stage_free();
}

// ------------------------------------------------------------------ action selection
// act / sac_act (algos.hpp:895-942) for the whole population: H2D of obs [n][rows][ds], the
// policy forward in the population's precision mode (bit-exact in FFMA32), exploration noise
// keyed (seed, streams[m], kExploreNoise, steps[m]), D2H of the actions [n][rows][da].
void Pop::act(const float* obs, uint64_t rows_, const double* noise_std, uint64_t seed,
              const uint64_t* steps_h, int deterministic, float* actions) {
  if (rows_ < 1) PBRL_THROW(PBRL_E_SHAPE, "act: observations need at least one row");
  if (!obs || !actions || !steps_h) PBRL_THROW(PBRL_E_USAGE, "act: null argument");
  if (algo == PBRL_ALGO_TD3 && !deterministic && !noise_std)
    PBRL_THROW(PBRL_E_USAGE, "act: noise_std is required unless deterministic");
  const int rows = static_cast<int>(rows_);
  const int L = pol.depth, nout = pol.dims[L];
  const long long nr = static_cast<long long>(n) * rows;
  const int ldi = padl(ds);
  if (rows > AS.rows) {
    AS = ActScratch{};
    AS.rows = rows;
    AS.obs.alloc(nr * ds);
    AS.in.alloc(nr * ldi);
    AS.in.zero(stream);
    AS.out.alloc(nr * nout);
    AS.act.alloc(nr * da);
    for (int l = 0; l + 1 < L; ++l) {
      const size_t h = static_cast<size_t>(padl(pol.dims[l + 1])) + (pol.dims[l + 1] + 31) / 32;
      AS.h.emplace_back();
      AS.h.back().alloc(nr * h);
      AS.h.back().zero(stream);
    }
    AS.steps.alloc(n);
    AS.noise.alloc(n);
  }
  if (act16() && weights_dirty) refresh_shadows();
  AS.steps.upload(steps_h, n, stream);
  if (noise_std) AS.noise.upload(noise_std, n, stream);
  CUDA_CHECK(cudaMemcpyAsync(AS.obs.p, obs, nr * ds * 4, cudaMemcpyHostToDevice, stream));
  launch_pack_obs(nr, ds, ldi, AS.obs.p, AS.in.p, act16() ? 1 : 0, stream);
  count_launch(1);
  const Mat x{AS.in.p, static_cast<long long>(rows) * ldi, ldi, 0};
  if (algo == PBRL_ALGO_TD3) {
    mlp_forward(pol, pol_p.p, n, rows, x, AS.h, AS.act.p, static_cast<long long>(rows) * da, da,
                EPI_BIAS_TANH, nullptr, nullptr, 0, 0, false, false, false);
    if (!deterministic) {
      launch_td3_act_noise(n, static_cast<long long>(rows) * da, AS.act.p, AS.noise.p, streams.p,
                           AS.steps.p, seed, bound, stream);
      count_launch(1);
    }
  } else {
    mlp_forward(pol, pol_p.p, n, rows, x, AS.h, AS.out.p, static_cast<long long>(rows) * nout,
                nout, EPI_BIAS, nullptr, nullptr, 0, 0, false, false, false);
    launch_sac_act(n, rows, da, AS.out.p, streams.p, AS.steps.p, seed, deterministic, bound,
                   AS.act.p, stream);
    count_launch(1);
  }
  CUDA_CHECK(cudaMemcpyAsync(actions, AS.act.p, nr * da * 4, cudaMemcpyDeviceToHost, stream));
  sync();
  CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------------------------ one step (graph replay)
void Pop::run_program(int B, const uint8_t* d_mask) {
  if (algo == PBRL_ALGO_TD3) td3_step(B, d_mask);
  else sac_step(B);
}

bool Pop::host_fires() {
  if (delay_host.size() != static_cast<size_t>(n)) delay_host.assign(n, 0.0);
  bool any = false;
  for (int m = 0; m < n; ++m) {
    bool f = shared;  // shared critic: every policy updates every step
    if (!shared) {
      double acc = delay_host[m] + hyper[2][m];
      if (acc >= 1.0 - 1e-12) {
        acc -= 1.0;
        f = true;
      }
      delay_host[m] = acc;
    }
    if (host_mask && !host_mask[m]) f = false;
    any = any || f;
  }
  return any;
}

void Pop::invalidate_graphs() {
  for (auto& g : graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
  }
  graphs.clear();
}

void Pop::step(int B, const uint8_t* d_mask) {
  check_guard();
  last_step_stage_ev = false;
  if (algo == PBRL_ALGO_TD3 && use_graphs && !guard_h) {  // (not allowed while capturing)
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&guard_h), sizeof(int), cudaHostAllocMapped));
    *guard_h = 0;
    CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&guard_d), guard_h, 0));
  }
  ensure_corr(t_bound + 4);
  const bool fires = algo == PBRL_ALGO_TD3 ? host_fires() : true;  // advances the mirror
  eager_fires = fires;
  // TD3 graph mode: two step graphs, picked by the host mirror's fire decision -- the fire-step
  // graph runs the policy half inline (no conditional-node boundary on its critical path), the
  // other keeps it in the IF node (the device decides: a step the mirror did not predict still
  // updates its policies)
  const bool fg = algo == PBRL_ALGO_TD3 && fires && fire_graphs();
  // the DvD hook runs only when some policy updates (td3_update_step, algos.hpp:394-396)
  if (dvd.on && fires) dvd_prepass();
  if (act16() && weights_dirty) refresh_shadows();
  if (prof_on || !use_graphs) {
    run_program(B, d_mask);
  } else {
    StepGraph* sg = nullptr;
    for (auto& g : graphs)
      if (g.B == B && g.masked == (d_mask != nullptr) && g.dvd == dvd.on && g.fire == fg &&
          g.hist == hist_on)
        sg = &g;
    if (!sg) {
      StepGraph g;
      g.B = B;
      g.masked = d_mask != nullptr;
      g.dvd = dvd.on;
      g.fire = fg;
      g.hist = hist_on;
      cudaGraph_t graph;
      capturing = true;
      cap_fire = fg;
      cond_body_nodes = 0;
      cond_nodes = 0;
      CUDA_CHECK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      const cudaStream_t s0 = stream;
      try {
        run_program(B, d_mask);
      } catch (...) {
        // restore the member stream (a throw inside a fork leaves it swapped with a branch),
        // end the capture (an unjoined branch makes that fail) and clear the error, so the
        // next call does not report it
        stream = s0;
        graph = nullptr;
        if (cudaStreamEndCapture(stream, &graph) == cudaSuccess && graph) cudaGraphDestroy(graph);
        (void)cudaGetLastError();
        capturing = false;
        cap_fire = false;
        stage_mark = 0;
        stage_joined = true;
        stage_ev_captured = false;
        in_cond_body = false;
        cta_cap = 0;
        pre_adam = nullptr;
        throw;
      }
      CUDA_CHECK(cudaStreamEndCapture(stream, &graph));
      capturing = false;
      cap_fire = false;
      g.stage_ev = ev_stage_free && stage_ev_captured;
      stage_ev_captured = false;
      // kernel nodes; the conditional nodes stand for their bodies (the policy half)
      g.nodes = kernel_nodes(graph);
      g.cond_nodes = cond_body_nodes;
      CUDA_CHECK(cudaGraphInstantiate(&g.exec, graph, 0));
      CUDA_CHECK(cudaGraphDestroy(graph));
      graphs.push_back(g);
      sg = &graphs.back();
    }
    CUDA_CHECK(cudaGraphLaunch(sg->exec, stream));
    count_launch(sg->nodes + (fires ? sg->cond_nodes : 0));
    last_step_stage_ev = sg->stage_ev;
  }
  t_bound += 1;
  prof_step_done();
}

}  // namespace pbrl
