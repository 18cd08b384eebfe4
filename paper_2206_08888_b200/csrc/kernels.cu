// CUDA-core kernels of the population update: the FFMA32 check-mode grouped GEMM with fused
// epilogues, and every elementwise / reduction step of TD3 and SAC.  All kernels are grouped
// over population members (grid.z or grid.y = member or member x critic), so the number of
// launches per update step does not depend on the population size (test_bench.cpp:40-53).
#include <math_constants.h>

#include "pop.cuh"

namespace pbrl {

int carveout_pref() {
  // measured on B200 (TD3 pop 80, BF16): round 1 driver default 233.9k, 100% 227.5k, 0% 222.7k,
  // 25-60% ~237k agent-updates/s; end of round 2: 0% 315.9k, 10% 328.2k, 18-25% 333.4k,
  // 33% 332.0k, 50% 330.0k, 75% 321.7k, driver default 312.2k
  static const int c = std::getenv("PBRL_CARVEOUT") ? std::atoi(std::getenv("PBRL_CARVEOUT")) : 25;
  return c;
}

bool pdl_enabled() {
  static const bool on = std::getenv("PBRL_NO_PDL") == nullptr;
  return on;
}

// ================================================================== grouped SIMT GEMM
// Reference order: every output accumulates its products in ascending k in fp32 without FMA
// (pop_tensor.hpp:155-166 forward, :194-206 backward), so results are bit-identical to the CPU.
// Shared fused epilogue of the CUDA-core GEMM family (operation order = the reference's).
__device__ __forceinline__ float simt_epilogue(const GemmArgs& g, float v, int gi, int gj, int grp,
                                               int mem, const float* bias, const float* aux) {
  switch (g.epi) {
    case EPI_BIAS: v = v + bias[gj]; break;
    case EPI_BIAS_RELU: {
      const float z = v + bias[gj];
      v = z > 0.0f ? z : 0.0f;
      break;
    }
    case EPI_BIAS_TANH:
    case EPI_BIAS_TANH_NOISE: {
      const float t = libm_tanhf(v + bias[gj]);
      if (g.C2) g.C2[grp * g.c2_gs + gi * g.c2_rs + gj] = t;
      v = (g.scale != 1.0f) ? t * g.scale : t;
      if (g.epi == EPI_BIAS_TANH_NOISE) {
        // algos.hpp:252-262: eps = clamp((T)normal * sd, +-clip); a = clamp(a + eps, +-bound)
        const uint64_t e = static_cast<uint64_t>(gi) * g.N + gj;
        float eps;
        if (g.noise_eps) {  // the identical draw, precomputed (tensor-core modes)
          eps = g.noise_eps[mem * g.ne_gs + static_cast<long long>(e)];
        } else {
          eps = static_cast<float>(rng_normal_pair(g.noise_key[mem], 2 * e)) * g.noise_sd[mem];
          eps = clampf_ref(eps, -g.noise_clip[mem], g.noise_clip[mem]);
        }
        v = clampf_ref(v + eps, -g.bound, g.bound);
      }
      break;
    }
    case EPI_RELU_MASK:
      if (!(aux[gi * g.aux.rs + gj * g.aux.cs] > 0.0f)) v = 0.0f;
      break;
    case EPI_TANH_GRAD: {
      if (g.scale != 1.0f) v = v * g.scale;
      const float t = aux[gi * g.aux.rs + gj * g.aux.cs];
      v = v * (1.0f - t * t);
      break;
    }
    default: break;
  }
  return v;
}

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    k_gemm_simt(const GemmArgs g) {
  PDL_ENTRY();
  constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY, BK = 16;
  constexpr int A_PER = BK * BM / NT, B_PER = (BK * BN + NT - 1) / NT;
  const int grp = blockIdx.z;
  const int mem = grp % g.n_members;
  if (g.active && !g.active[mem]) return;
  const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
  __shared__ float As[BK][BM + 1];
  __shared__ float Bs[BK][BN + 1];
  const float* A = g.A.p + (g.A.by_member ? mem : grp) * g.A.gs;
  const float* B = g.B.p + (g.B.by_member ? mem : grp) * g.B.gs;
  const int tid = threadIdx.x;
  const int ty = tid / TX, tx = tid % TX;
  const bool a_kc = g.A.cs == 1, b_nc = g.B.cs == 1;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = g.acc_init;

  // register double buffering: the next K-chunk's global loads are in flight while the
  // current chunk is multiplied out of shared memory
  float ra[A_PER], rb[B_PER];
  auto a_pos = [&](int e, int& kk, int& ii) {
    if (a_kc) { kk = e % BK; ii = e / BK; } else { ii = e % BM; kk = e / BM; }
  };
  auto b_pos = [&](int e, int& kk, int& jj) {
    if (b_nc) { jj = e % BN; kk = e / BN; } else { kk = e % BK; jj = e / BK; }
  };
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < A_PER; ++q) {
      int kk, ii;
      a_pos(tid + q * NT, kk, ii);
      const int gi = i0 + ii, gk = k0 + kk;
      float v = 0.0f;
      if (gi < g.M && gk < g.K)
        v = (g.a_ones_row && gi == g.M - 1) ? 1.0f : A[gi * g.A.rs + gk * g.A.cs];
      ra[q] = v;
    }
#pragma unroll
    for (int q = 0; q < B_PER; ++q) {
      const int e = tid + q * NT;
      float v = 0.0f;
      if (e < BK * BN) {
        int kk, jj;
        b_pos(e, kk, jj);
        const int gj = j0 + jj, gk = k0 + kk;
        if (gj < g.N && gk < g.K) v = B[gk * g.B.rs + gj * g.B.cs];
      }
      rb[q] = v;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int q = 0; q < A_PER; ++q) {
      int kk, ii;
      a_pos(tid + q * NT, kk, ii);
      As[kk][ii] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < B_PER; ++q) {
      const int e = tid + q * NT;
      if (e < BK * BN) {
        int kk, jj;
        b_pos(e, kk, jj);
        Bs[kk][jj] = rb[q];
      }
    }
  };

  load(0);
  for (int k0 = 0; k0 < g.K; k0 += BK) {
    stash();
    __syncthreads();
    if (k0 + BK < g.K) load(k0 + BK);
    const int kmax = min(BK, g.K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + i * TY];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = acc[i][j] + a[i] * b[j];
    }
    __syncthreads();
  }

  float* C = g.C + (g.c_by_member ? mem : grp) * g.c_gs;
  const float* bias = g.bias.p ? g.bias.p + (g.bias.by_member ? mem : grp) * g.bias.gs : nullptr;
  const float* aux = g.aux.p ? g.aux.p + (g.aux.by_member ? mem : grp) * g.aux.gs : nullptr;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gi = i0 + ty + i * TY;
    if (gi >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gj = j0 + tx + j * TX;
      if (gj >= g.N) continue;
      C[gi * g.c_rs + gj] = simt_epilogue(g, acc[i][j], gi, gj, grp, mem, bias, aux);
    }
  }
}

void launch_gemm_simt(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.groups <= 0) return;
  if (g.N <= 16) {
    constexpr int BM = 64, BN = 16, TM = 2, TN = 2;
    dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, g.groups);
    launch_k(k_gemm_simt<BM, BN, TM, TN>, grid, (BM / TM) * (BN / TN), 0, s, g);
  } else {
    constexpr int BM = 64, BN = 64, TM = 4, TN = 4;
    dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, g.groups);
    launch_k(k_gemm_simt<BM, BN, TM, TN>, grid, (BM / TM) * (BN / TN), 0, s, g);
  }
}

// ------------------------------------------------------------------ skinny products
// The output layers of the MLPs have N (forward, dW) or K (dX) of 1 (critic) or 6 / 12 (policy).
// These get dedicated CUDA-core kernels with the same ascending-k accumulation (bit-exact in the
// FFMA32 mode) and memory-friendly thread mappings.

// forward, N <= 16: one thread per output row; the X tile is staged through shared memory
// (coalesced), W [K][N] lives in shared memory; acc[o] runs k = 0..K-1.
// AT: element type of A (bf16 activations in BF16 mode); C is bf16 when g.c16
template <int NMAX, typename AT>
__global__ void __launch_bounds__(128) k_fwd_skinny(const GemmArgs g) {
  PDL_ENTRY();
  constexpr int ROWS = 128, KC = 32;
  const int grp = blockIdx.y;
  const int mem = grp % g.n_members;
  if (g.active && !g.active[mem]) return;
  __shared__ float Xs[ROWS][KC + 1];
  __shared__ float Ws[KC][NMAX];
  const AT* A = reinterpret_cast<const AT*>(g.A.p) + (g.A.by_member ? mem : grp) * g.A.gs;
  const float* Bm = g.B.p + (g.B.by_member ? mem : grp) * g.B.gs;
  const int r0 = blockIdx.x * ROWS, tid = threadIdx.x;
  float acc[NMAX];
#pragma unroll
  for (int o = 0; o < NMAX; ++o) acc[o] = g.acc_init;
  for (int k0 = 0; k0 < g.K; k0 += KC) {
    const int kc = min(KC, g.K - k0);
    for (int e = tid; e < ROWS * KC; e += ROWS) {
      const int rr = e / KC, kk = e % KC;
      const int row = r0 + rr;
      Xs[rr][kk] =
          (row < g.M && kk < kc) ? act_ld(A, row * g.A.rs + (k0 + kk) * g.A.cs) : 0.0f;
    }
    for (int e = tid; e < KC * NMAX; e += ROWS) {
      const int kk = e / NMAX, o = e % NMAX;
      Ws[kk][o] = (kk < kc && o < g.N) ? Bm[(k0 + kk) * g.B.rs + o * g.B.cs] : 0.0f;
    }
    __syncthreads();
    for (int kk = 0; kk < kc; ++kk) {
      const float x = Xs[tid][kk];
#pragma unroll
      for (int o = 0; o < NMAX; ++o) acc[o] = acc[o] + x * Ws[kk][o];
    }
    __syncthreads();
  }
  const int row = r0 + tid;
  if (row >= g.M) return;
  const long long cbase = (g.c_by_member ? mem : grp) * g.c_gs;
  const float* bias = g.bias.p ? g.bias.p + (g.bias.by_member ? mem : grp) * g.bias.gs : nullptr;
  const float* aux = g.aux.p ? g.aux.p + (g.aux.by_member ? mem : grp) * g.aux.gs : nullptr;
#pragma unroll
  for (int o = 0; o < NMAX; ++o) {
    if (o >= g.N) continue;
    const float v = simt_epilogue(g, acc[o], row, o, grp, mem, bias, aux);
    if (g.c16) act_st(reinterpret_cast<__nv_bfloat16*>(g.C), cbase + row * g.c_rs + o, v);
    else g.C[cbase + row * g.c_rs + o] = v;
  }
}

// dX with K <= 16 (through the output layer): one thread per (row, column), columns fastest, so
// the relu-mask reads and the stores are coalesced; G rows are warp-broadcast.
template <int KMAX>
__global__ void __launch_bounds__(256) k_dx_skinny(const GemmArgs g) {
  PDL_ENTRY();
  constexpr int RPB = 8;  // rows per block
  const int grp = blockIdx.z;
  const int mem = grp % g.n_members;
  if (g.active && !g.active[mem]) return;
  const float* A = g.A.p + (g.A.by_member ? mem : grp) * g.A.gs;
  const float* Bm = g.B.p + (g.B.by_member ? mem : grp) * g.B.gs;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.N) return;
  float w[KMAX];
#pragma unroll
  for (int o = 0; o < KMAX; ++o) w[o] = (o < g.K) ? Bm[o * g.B.rs + j * g.B.cs] : 0.0f;
  float* C = g.C + (g.c_by_member ? mem : grp) * g.c_gs;
  const float* aux = g.aux.p ? g.aux.p + (g.aux.by_member ? mem : grp) * g.aux.gs : nullptr;
  const int r0 = blockIdx.y * RPB;
  for (int rr = 0; rr < RPB; ++rr) {
    const int row = r0 + rr;
    if (row >= g.M) break;
    float acc = g.acc_init;
#pragma unroll
    for (int o = 0; o < KMAX; ++o)
      if (o < g.K) acc = acc + A[row * g.A.rs + o * g.A.cs] * w[o];
    C[row * g.c_rs + j] = simt_epilogue(g, acc, row, j, grp, mem, nullptr, aux);
  }
}

// dW with N <= 16 (+ bias as the ones row): one thread per input feature i; x = X[b][i] is
// coalesced across threads, G[b][o] is warp-broadcast; acc[o] runs b = 0..B-1.
template <int NMAX>
__global__ void __launch_bounds__(128) k_dw_skinny(const GemmArgs g) {
  PDL_ENTRY();
  const int grp = blockIdx.y;
  const int mem = grp % g.n_members;
  if (g.active && !g.active[mem]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.M) return;
  const float* A = g.A.p + (g.A.by_member ? mem : grp) * g.A.gs;
  const float* Bm = g.B.p + (g.B.by_member ? mem : grp) * g.B.gs;
  const bool ones = g.a_ones_row && i == g.M - 1;
  float acc[NMAX];
#pragma unroll
  for (int o = 0; o < NMAX; ++o) acc[o] = g.acc_init;
  for (int b = 0; b < g.K; ++b) {
    const float x = ones ? 1.0f : A[i * g.A.rs + b * g.A.cs];
#pragma unroll
    for (int o = 0; o < NMAX; ++o)
      if (o < g.N) acc[o] = acc[o] + x * Bm[b * g.B.rs + o * g.B.cs];
  }
  float* C = g.C + (g.c_by_member ? mem : grp) * g.c_gs;
#pragma unroll
  for (int o = 0; o < NMAX; ++o)
    if (o < g.N) C[i * g.c_rs + o] = acc[o];
}

// Output-layer backward in one pass (N_out <= 16): for the layer y = X W + b with cotangent G,
//   dW[i][o] = sum_b X[b][i] G[b][o]      (b ascending, from +0: pop_tensor.hpp:194-206)
//   db[o]    = sum_b G[b][o]              (b ascending: :244-246)
//   dX[b][i] = X[b][i] > 0 ? sum_o G[b][o] W[i][o] : 0   (o ascending; relu' of the layer below)
// One block per (group, 64 input features).  Thread (column i, row slice s) streams its rows of
// X once: dW partials stay in registers, dX is produced and stored on the fly, W[i][:] sits in
// registers and G in shared memory (broadcast reads).  Exact mode uses one slice (b ascending in
// a single accumulator, the reference order); the fast mode splits B into kObSlices slices whose
// partials are combined in slice order through shared memory (deterministic).
constexpr int kObCols = 64, kObSlices = 4;

// AT: activation storage of X / dX (fp32, or bf16 in BF16 mode).  dW == nullptr: dX only (the
// output layer of a critic inside the policy-loss chain, whose weight gradients are discarded).
template <int NO, typename AT>  // fused output width: exact for 1 / 6 / 12, runtime-guarded up to 16
__global__ void __launch_bounds__(kObCols* kObSlices) k_out_backward(OutBwdArgs a) {
  PDL_ENTRY();
  extern __shared__ float sm[];
  constexpr int NA = NO;
  const int nout = NO < 16 ? NO : a.nout, B = a.B;
  float* Gs = sm;                         // [B][nout]
  float* Ps = Gs + B * nout;              // [kObSlices][kObCols][nout] dW partials
  float* Cs = Ps + kObSlices * kObCols * nout;  // [kObSlices][kObCols] dX column sums
  float* Ls = Cs + kObSlices * kObCols;          // [B] loss terms (fused top cotangent)
  const int grp = blockIdx.y;
  const int mem = grp % a.n_members;
  if (a.active && !a.active[mem]) return;
  const int slices = blockDim.x / kObCols;
  const int col = threadIdx.x % kObCols, sl = threadIdx.x / kObCols;
  const int i = blockIdx.x * kObCols + col;
  const AT* X = static_cast<const AT*>(a.X) + (a.x_by_member ? mem : grp) * a.x_gs;
  const float* W = a.W + grp * a.w_gs;
  if (a.top) {  // nout == 1: the top cotangent from the network output (see OutBwdArgs::top)
    const float* qg = a.q + static_cast<long long>(grp) * B;
    const long long mb = static_cast<long long>(mem) * B;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      const float qv = qg[b];
      if (a.top == 3) {
        Gs[b] = -1.0f / static_cast<float>(B);
        Ls[b] = qv;
      } else {
        float yv;
        if (a.top == 1) {
          const float qmin = minf_ref(a.tq[mb + b], a.tq[static_cast<long long>(a.n_members) * B + mb + b]);
          yv = a.r[mb + b] + a.gamma[mem] * (1.0f - a.d[mb + b]) * qmin;
        } else {
          yv = a.y[mb + b];
        }
        const float dl = qv - yv;
        Gs[b] = (2.0f / static_cast<float>(a.norm_rows ? a.norm_rows : B)) * dl;
        Ls[b] = dl;
      }
    }
  } else {
    const float* G = a.G + grp * a.g_gs;
    for (int e = threadIdx.x; e < B * nout; e += blockDim.x) {
      const int b = e / nout, o = e - b * nout;
      Gs[e] = G[static_cast<long long>(b) * a.g_ld + o];
    }
  }
  float w[NA], acc[NA];
#pragma unroll
  for (int o = 0; o < NA; ++o) {
    acc[o] = 0.0f;
    w[o] = (o < nout && i < a.H) ? W[static_cast<long long>(i) * nout + o] : 0.0f;
  }
  __syncthreads();
  const int rows = (B + slices - 1) / slices;
  const int b0 = sl * rows, b1 = min(B, b0 + rows);
  AT* dX = a.dX ? static_cast<AT*>(a.dX) + grp * a.dx_gs : nullptr;
  float csum = 0.0f;  // column sum of this thread's dX rows (bias gradient of the layer below)
  if (i < a.H) {
    constexpr int U = 8;  // independent loads in flight per thread
    int b = b0;
    for (; b + U <= b1; b += U) {
      float xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = act_ld(X, static_cast<long long>(b + u) * a.x_ld + i);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float* g = Gs + (b + u) * nout;
        float d = 0.0f;
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          if (NO == 16 && o >= nout) break;
          acc[o] = acc[o] + xv[u] * g[o];
          d = d + g[o] * w[o];
        }
        const float dv = xv[u] > 0.0f ? d : 0.0f;
        csum = csum + dv;
        if (dX) act_st(dX, static_cast<long long>(b + u) * a.dx_ld + i, dv);
      }
    }
    for (; b < b1; ++b) {
      const float xv = act_ld(X, static_cast<long long>(b) * a.x_ld + i);
      const float* g = Gs + b * nout;
      float d = 0.0f;
#pragma unroll
      for (int o = 0; o < NA; ++o) {
        if (NO == 16 && o >= nout) break;
        acc[o] = acc[o] + xv * g[o];
        d = d + g[o] * w[o];
      }
      const float dv = xv > 0.0f ? d : 0.0f;
      csum = csum + dv;
      if (dX) act_st(dX, static_cast<long long>(b) * a.dx_ld + i, dv);
    }
  }
  if (a.dbx) {  // fused bias gradient of the layer below: slices combined in slice order
    float* db = a.dbx + grp * a.dbx_gs;
    if (slices > 1) {
      Cs[sl * kObCols + col] = csum;
      __syncthreads();
      if (sl == 0 && i < a.H) {
        float t = Cs[col];
        for (int q = 1; q < slices; ++q) t += Cs[q * kObCols + col];
        db[i] = t;
      }
    } else if (i < a.H) {
      db[i] = csum;
    }
  }
  if (a.top && a.loss && blockIdx.x == 0 && threadIdx.x == 0) {  // row order, double
    double acc = 0.0;
    if (a.top == 3) {
      for (int b = 0; b < B; ++b) acc -= static_cast<double>(Ls[b]);
    } else {
      for (int b = 0; b < B; ++b) acc += static_cast<double>(Ls[b]) * static_cast<double>(Ls[b]);
    }
    a.loss[grp] = acc / static_cast<double>(a.top != 3 && a.norm_rows ? a.norm_rows : B);
  }
  if (!a.dW) return;
  float* dW = a.dW + grp * a.dw_gs;
  if (slices > 1) {
#pragma unroll
    for (int o = 0; o < NA; ++o)
      if (o < nout) Ps[(sl * kObCols + col) * nout + o] = acc[o];
    __syncthreads();
    for (int e = threadIdx.x; e < kObCols * nout; e += blockDim.x) {
      const int c = e / nout, o = e - c * nout;
      if (blockIdx.x * kObCols + c >= a.H) continue;
      float t = Ps[c * nout + o];
      for (int q = 1; q < slices; ++q) t += Ps[(q * kObCols + c) * nout + o];
      dW[static_cast<long long>(blockIdx.x * kObCols + c) * nout + o] = t;
    }
  } else if (i < a.H) {
#pragma unroll
    for (int o = 0; o < NA; ++o)
      if (o < nout) dW[static_cast<long long>(i) * nout + o] = acc[o];
  }
  if (blockIdx.x == 0) {  // db: b ascending (exact) / warp tree (fast)
    if (a.exact) {
      for (int o = threadIdx.x; o < nout; o += blockDim.x) {
        float t = 0.0f;
        for (int b = 0; b < B; ++b) t += Gs[b * nout + o];
        dW[static_cast<long long>(a.H) * nout + o] = t;
      }
    } else {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int o = warp; o < nout; o += blockDim.x >> 5) {
        float t = 0.0f;
        for (int b = lane; b < B; b += 32) t += Gs[b * nout + o];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) dW[static_cast<long long>(a.H) * nout + o] = t;
      }
    }
  }
}

// Tensor-core modes: the same pass with 4 adjacent columns per thread (one 8-byte bf16x4 or
// 16-byte fp32x4 load / store per row instead of four scalar ones), 64 columns x 16 row slices
// per block (enough blocks and loads in flight to cover HBM latency); slices combined in slice
// order (deterministic).  Requires H % 4 == 0 and 4-element
// aligned rows (launch_out_backward checks and otherwise uses k_out_backward).
constexpr int kOvQuads = 16;  // CW x 16 columns per block; row slices: ov_slices<NO>()

template <typename AT, int CW> struct VecN;
template <> struct VecN<float, 4> {
  __device__ static void ld(const float* p, float* v) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  }
  __device__ static void st(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct VecN<__nv_bfloat16, 4> {
  __device__ static void ld(const __nv_bfloat16* p, float* v) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  __device__ static void st(__nv_bfloat16* p, const float* v) {
    const __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    const __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&a);
    u.y = *reinterpret_cast<const uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  }
};
template <> struct VecN<float, 2> {
  __device__ static void ld(const float* p, float* v) {
    const float2 u = *reinterpret_cast<const float2*>(p);
    v[0] = u.x; v[1] = u.y;
  }
  __device__ static void st(float* p, const float* v) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
};
template <> struct VecN<__nv_bfloat16, 2> {
  __device__ static void ld(const __nv_bfloat16* p, float* v) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
    v[0] = a.x; v[1] = a.y;
  }
  __device__ static void st(__nv_bfloat16* p, const float* v) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v[0], v[1]);
  }
};

// Resident blocks per SM asked of ptxas and row loads in flight per thread, per output width
// (compile-time PBRL_OBV_{MINB,U}{1,N}).  Measured on B200 (config D BF16, alternating runs):
// single-output (critic) layers 4 blocks / 4 loads (64 registers) against the unconstrained
// 103-register build with 8 loads (2 blocks/SM: 640 blocks in 2.2 waves), 314k -> 322k
// agent-updates/s; 5 blocks (48 registers) 315k.  The 6-output (policy) layer: 3 blocks / 8 loads
// (80 registers) 323k, 4 / 4 322k, 5 / 2 316k; then 8 row slices (128-thread blocks, 4 per SM,
// 94 registers, 8 loads: the 640 blocks resident in one wave) 329.2k -> 330.4k (the critic at 8
// slices: 321k).
#ifndef PBRL_OBV_MINB1
#define PBRL_OBV_MINB1 4
#endif
#ifndef PBRL_OBV_U1
#define PBRL_OBV_U1 4
#endif
#ifndef PBRL_OBV_MINBN
#define PBRL_OBV_MINBN 4
#endif
#ifndef PBRL_OBV_UN
#define PBRL_OBV_UN 8
#endif
#ifndef PBRL_OBV_SL1
#define PBRL_OBV_SL1 16
#endif
#ifndef PBRL_OBV_SLN
#define PBRL_OBV_SLN 8
#endif
template <int NO> __host__ __device__ constexpr int ov_slices() {
  return NO == 1 ? PBRL_OBV_SL1 : PBRL_OBV_SLN;
}
template <int NO, typename AT, int CW>
__global__ void __launch_bounds__(kOvQuads* ov_slices<NO>(),
                                  NO == 1 ? PBRL_OBV_MINB1 : PBRL_OBV_MINBN)
    k_out_backward_v(OutBwdArgs a) {
  PDL_ENTRY();
  extern __shared__ float sm[];
  constexpr int NA = NO, CB = CW * kOvQuads;  // columns per block
  const int nout = NO < 16 ? NO : a.nout, B = a.B;
  float* Gs = sm;                                // [B][nout]
  float* Ls = Gs + B * nout;                     // [B]
  float* Ps = Ls + B;                            // [ov_slices<NO>()][CB][nout]
  float* Cs = Ps + ov_slices<NO>() * CB * nout;        // [ov_slices<NO>()][CB]
  const int grp = blockIdx.y;
  const int mem = grp % a.n_members;
  if (a.active && !a.active[mem]) return;
  const int cq = threadIdx.x % kOvQuads, sl = threadIdx.x / kOvQuads;
  const int c0 = blockIdx.x * CB + CW * cq;  // first of this thread's CW columns
  const bool live = c0 < a.H;
  const AT* X = static_cast<const AT*>(a.X) + (a.x_by_member ? mem : grp) * a.x_gs;
  const float* W = a.W + grp * a.w_gs;
  if (a.top) {
    const float* qg = a.q + static_cast<long long>(grp) * B;
    const long long mb = static_cast<long long>(mem) * B;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      const float qv = qg[b];
      if (a.top == 3) {
        Gs[b] = -1.0f / static_cast<float>(B);
        Ls[b] = qv;
      } else {
        float yv;
        if (a.top == 1) {
          const float qmin =
              minf_ref(a.tq[mb + b], a.tq[static_cast<long long>(a.n_members) * B + mb + b]);
          yv = a.r[mb + b] + a.gamma[mem] * (1.0f - a.d[mb + b]) * qmin;
        } else {
          yv = a.y[mb + b];
        }
        const float dl = qv - yv;
        Gs[b] = (2.0f / static_cast<float>(a.norm_rows ? a.norm_rows : B)) * dl;
        Ls[b] = dl;
      }
    }
  } else {
    // the block's copy of the cotangent: 8 independent loads in flight per thread before any
    // shared store (one global latency instead of one per element)
    const float* G = a.G + grp * a.g_gs;
    constexpr int PF = 8;
    const int tot = B * nout;
    for (int e0 = threadIdx.x; e0 < tot; e0 += PF * blockDim.x) {
      float t[PF];
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int e = e0 + u * blockDim.x;
        const int b = e / nout, o = e - b * nout;
        t[u] = e < tot ? G[static_cast<long long>(b) * a.g_ld + o] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < PF; ++u)
        if (e0 + u * blockDim.x < tot) Gs[e0 + u * blockDim.x] = t[u];
    }
  }
  float w[CW][NA], acc[CW][NA], csum[CW];
#pragma unroll
  for (int c = 0; c < CW; ++c) {
    csum[c] = 0.0f;
#pragma unroll
    for (int o = 0; o < NA; ++o) {
      acc[c][o] = 0.0f;
      w[c][o] = (live && o < nout) ? W[static_cast<long long>(c0 + c) * nout + o] : 0.0f;
    }
  }
  __syncthreads();
  const int rows = (B + ov_slices<NO>() - 1) / ov_slices<NO>();
  const int b0 = sl * rows, b1 = min(B, b0 + rows);
  AT* dX = a.dX ? static_cast<AT*>(a.dX) + grp * a.dx_gs : nullptr;
  if (live) {
    constexpr int U = NO == 1 ? PBRL_OBV_U1 : PBRL_OBV_UN;
    for (int b = b0; b < b1; b += U) {
      float xv[U][CW];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (b + u < b1) VecN<AT, CW>::ld(X + static_cast<long long>(b + u) * a.x_ld + c0, xv[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (b + u >= b1) break;
        const float* g = Gs + (b + u) * nout;
        float dv[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          float d = 0.0f;
#pragma unroll
          for (int o = 0; o < NA; ++o) {
            if (NO == 16 && o >= nout) break;
            acc[c][o] = acc[c][o] + xv[u][c] * g[o];
            d = d + g[o] * w[c][o];
          }
          dv[c] = xv[u][c] > 0.0f ? d : 0.0f;
          csum[c] = csum[c] + dv[c];
        }
        if (dX) VecN<AT, CW>::st(dX + static_cast<long long>(b + u) * a.dx_ld + c0, dv);
      }
    }
  }
  if (a.dbx) {  // fused bias gradient of the layer below
#pragma unroll
    for (int c = 0; c < CW; ++c) Cs[sl * CB + CW * cq + c] = csum[c];
    __syncthreads();
    for (int cc = threadIdx.x; cc < CB; cc += blockDim.x) {
      const int col = blockIdx.x * CB + cc;
      if (col >= a.H) continue;
      float t = Cs[cc];
      for (int q = 1; q < ov_slices<NO>(); ++q) t += Cs[q * CB + cc];
      a.dbx[grp * a.dbx_gs + col] = t;
    }
  }
  if (a.top && a.loss && blockIdx.x == 0 && threadIdx.x < 32) {
    // fast modes only (this kernel never runs in the bit-exact mode): warp tree in double
    // instead of one thread walking the rows
    double s = 0.0;
    for (int b = threadIdx.x; b < B; b += 32) {
      const double l = static_cast<double>(Ls[b]);
      s += a.top == 3 ? -l : l * l;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0)
      a.loss[grp] = s / static_cast<double>(a.top != 3 && a.norm_rows ? a.norm_rows : B);
  }
  if (!a.dW) return;
  float* dW = a.dW + grp * a.dw_gs;
#pragma unroll
  for (int c = 0; c < CW; ++c)
#pragma unroll
    for (int o = 0; o < NA; ++o)
      if (o < nout) Ps[(sl * CB + CW * cq + c) * nout + o] = acc[c][o];
  __syncthreads();
  for (int e = threadIdx.x; e < CB * nout; e += blockDim.x) {
    const int cc = e / nout, o = e - cc * nout;
    const int col = blockIdx.x * CB + cc;
    if (col >= a.H) continue;
    float t = Ps[cc * nout + o];
    for (int q = 1; q < ov_slices<NO>(); ++q) t += Ps[(q * CB + cc) * nout + o];
    dW[static_cast<long long>(col) * nout + o] = t;
  }
  if (blockIdx.x == 0) {  // db of the output layer: warp tree
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int o = warp; o < nout; o += blockDim.x >> 5) {
      float t = 0.0f;
      for (int b = lane; b < B; b += 32) t += Gs[b * nout + o];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
      if (lane == 0) dW[static_cast<long long>(a.H) * nout + o] = t;
    }
  }
}

template <int NO, typename AT>
static bool launch_ob_v(const OutBwdArgs& a, cudaStream_t s) {
  // CW adjacent columns per thread: 4 for single-output layers, 2 for NO <= 8 (the w / acc
  // register tiles are CW x NO floats each); wider outputs keep the scalar kernel
  constexpr int CW = NO == 1 ? 4 : 2;
  if constexpr (NO > 8) {
    return false;
  } else {
    const int eb = sizeof(AT);
    auto al = [&](const void* p) { return reinterpret_cast<uintptr_t>(p) % (CW * eb) == 0; };
    if (a.exact || a.H % CW || a.x_ld % CW || a.x_gs % CW || !al(a.X) ||
        (a.dX && (a.dx_ld % CW || a.dx_gs % CW || !al(a.dX))))
      return false;
    constexpr int CB = CW * kOvQuads;
    const size_t smem = (static_cast<size_t>(a.B) * (a.nout + 1) +
                         static_cast<size_t>(ov_slices<NO>()) * CB * (a.nout + 1)) * 4;
    if (smem > 200 * 1024) return false;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_out_backward_v<NO, AT, CW>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    dim3 grid((a.H + CB - 1) / CB, a.groups);
    launch_k(k_out_backward_v<NO, AT, CW>, grid, kOvQuads * ov_slices<NO>(), smem, s, a);
    return true;
  }
}

template <int NO, typename AT>
static void launch_ob(const OutBwdArgs& a, cudaStream_t s) {
  if (launch_ob_v<NO, AT>(a, s)) return;
  const int slices = a.exact ? 1 : kObSlices;
  const size_t smem =
      (static_cast<size_t>(a.B) * (a.nout + 1) + kObSlices * kObCols * (a.nout + 1)) * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_out_backward<NO, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  dim3 grid((a.H + kObCols - 1) / kObCols, a.groups);
  launch_k(k_out_backward<NO, AT>, grid, kObCols * slices, smem, s, a);
}

template <typename AT>
static void launch_ob_t(const OutBwdArgs& a, cudaStream_t s) {
  switch (a.nout) {
    case 1: launch_ob<1, AT>(a, s); return;
    case 6: launch_ob<6, AT>(a, s); return;
    case 12: launch_ob<12, AT>(a, s); return;
    default: launch_ob<16, AT>(a, s); return;
  }
}

void launch_out_backward(const OutBwdArgs& a, cudaStream_t s) {
  if (a.act16) launch_ob_t<__nv_bfloat16>(a, s);
  else launch_ob_t<float>(a, s);
}

template <typename AT>
static void launch_fwd_skinny_t(const GemmArgs& g, cudaStream_t s) {
  dim3 grid((g.M + 127) / 128, g.groups);
  if (g.N <= 1) launch_k(k_fwd_skinny<1, AT>, grid, 128, 0, s, g);
  else if (g.N <= 8) launch_k(k_fwd_skinny<8, AT>, grid, 128, 0, s, g);
  else launch_k(k_fwd_skinny<16, AT>, grid, 128, 0, s, g);
}

// Tensor-core modes (no reference summation order to keep): an output layer (N <= 16) too wide
// to be fused into the previous layer's epilogue (hidden > 256) as one warp per row -- each lane
// accumulates 8-element slices of K (one 16-byte bf16 / two 16-byte fp32 loads), the N partial
// sums are warp-reduced, lane o applies the epilogue of output o.  W [K][N] of the block's group
// is staged in shared memory.
template <int NMAX, typename AT>
__global__ void __launch_bounds__(256) k_fwd_rowdot(const GemmArgs g) {
  PDL_ENTRY();
  extern __shared__ float Ws[];  // [NMAX][K]: lane slices of 8 consecutive k read as 2 x 16 B
  const int grp = blockIdx.y;
  const int mem = grp % g.n_members;
  if (g.active && !g.active[mem]) return;
  const AT* A = reinterpret_cast<const AT*>(g.A.p) + (g.A.by_member ? mem : grp) * g.A.gs;
  const float* Bm = g.B.p + (g.B.by_member ? mem : grp) * g.B.gs;
  for (int e = threadIdx.x; e < g.K * NMAX; e += blockDim.x) {
    const int o = e / g.K, k = e - o * g.K;
    Ws[e] = o < g.N ? Bm[k * g.B.rs + o * g.B.cs] : 0.0f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long cbase = (g.c_by_member ? mem : grp) * g.c_gs;
  const float* bias = g.bias.p ? g.bias.p + (g.bias.by_member ? mem : grp) * g.bias.gs : nullptr;
  const float* aux = g.aux.p ? g.aux.p + (g.aux.by_member ? mem : grp) * g.aux.gs : nullptr;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  // two rows per warp trip (both rows' loads in flight, each W slice read from shared memory
  // once for both); fast modes only, so the dot runs on FMA
  auto load8 = [&](const AT* xr, int k0, float* x) {
    if (sizeof(AT) == 2) {
      const uint4 u = *reinterpret_cast<const uint4*>(xr + k0);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        x[2 * j] = f.x;
        x[2 * j + 1] = f.y;
      }
    } else {
      const float4 u0 = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(xr) + k0);
      const float4 u1 =
          *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(xr) + k0 + 4);
      x[0] = u0.x; x[1] = u0.y; x[2] = u0.z; x[3] = u0.w;
      x[4] = u1.x; x[5] = u1.y; x[6] = u1.z; x[7] = u1.w;
    }
  };
  for (int r0 = 2 * (blockIdx.x * (blockDim.x >> 5) + warp); r0 < g.M; r0 += 2 * nwarps) {
    const bool two = r0 + 1 < g.M;
    const AT* xa = A + static_cast<long long>(r0) * g.A.rs;
    const AT* xb = two ? xa + g.A.rs : xa;
    float acc[2][NMAX];
#pragma unroll
    for (int o = 0; o < NMAX; ++o) acc[0][o] = acc[1][o] = 0.0f;
    for (int k0 = lane * 8; k0 < g.K; k0 += 256) {
      float x[2][8];
      load8(xa, k0, x[0]);
      load8(xb, k0, x[1]);
#pragma unroll
      for (int o = 0; o < NMAX; ++o) {
        if (NMAX > 1 && o >= g.N) break;
        const float4 w0 = *reinterpret_cast<const float4*>(Ws + o * g.K + k0);
        const float4 w1 = *reinterpret_cast<const float4*>(Ws + o * g.K + k0 + 4);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          float t = acc[r][o];
          t = __fmaf_rn(x[r][0], w0.x, t);
          t = __fmaf_rn(x[r][1], w0.y, t);
          t = __fmaf_rn(x[r][2], w0.z, t);
          t = __fmaf_rn(x[r][3], w0.w, t);
          t = __fmaf_rn(x[r][4], w1.x, t);
          t = __fmaf_rn(x[r][5], w1.y, t);
          t = __fmaf_rn(x[r][6], w1.z, t);
          acc[r][o] = __fmaf_rn(x[r][7], w1.w, t);
        }
      }
    }
#pragma unroll
    for (int o = 0; o < NMAX; ++o) {
      if (NMAX > 1 && o >= g.N) break;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        acc[0][o] += __shfl_xor_sync(0xffffffffu, acc[0][o], off);
        acc[1][o] += __shfl_xor_sync(0xffffffffu, acc[1][o], off);
      }
    }
    // lanes 0..N-1 finish row r0, lanes 16..16+N-1 row r0 + 1 (N <= 16)
    const int r = lane >> 4, o_l = lane & 15;
    if (o_l < g.N && (r == 0 || two)) {
      float v = 0.0f;
#pragma unroll
      for (int o = 0; o < NMAX; ++o)
        if (o == o_l) v = acc[r][o];
      const int row = r0 + r;
      v = simt_epilogue(g, v, row, o_l, grp, mem, bias, aux);
      if (g.c16) act_st(reinterpret_cast<__nv_bfloat16*>(g.C), cbase + row * g.c_rs + o_l, v);
      else g.C[cbase + row * g.c_rs + o_l] = v;
    }
  }
}

template <typename AT>
static bool launch_fwd_rowdot_t(const GemmArgs& g, cudaStream_t s) {
  const int eb = sizeof(AT);
  if (g.K % 8 || g.A.cs != 1 || g.A.rs % 8 || g.A.gs % 8 ||
      reinterpret_cast<uintptr_t>(g.A.p) % (8 * eb) || g.N > 16)
    return false;
  const int nmax = g.N <= 1 ? 1 : (g.N <= 8 ? 8 : 16);
  const size_t smem = static_cast<size_t>(g.K) * nmax * 4;
  if (smem > 96 * 1024) return false;
  // ~16 rows per warp: W is staged once per block, so few blocks per group
  dim3 grid(std::max(1, std::min((g.M + 127) / 128, 16)), g.groups);
  auto go = [&](auto kern) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      attr = true;
    }
    launch_k(kern, grid, 256, smem, s, g);
  };
  if (nmax == 1) go(k_fwd_rowdot<1, AT>);
  else if (nmax == 8) go(k_fwd_rowdot<8, AT>);
  else go(k_fwd_rowdot<16, AT>);
  return true;
}

void launch_fwd_skinny(const GemmArgs& g, cudaStream_t s) {
  if (g.rowdot) {
    if (g.a16 ? launch_fwd_rowdot_t<__nv_bfloat16>(g, s) : launch_fwd_rowdot_t<float>(g, s))
      return;
  }
  if (g.a16) launch_fwd_skinny_t<__nv_bfloat16>(g, s);
  else launch_fwd_skinny_t<float>(g, s);
}

void launch_dx_skinny(const GemmArgs& g, cudaStream_t s) {
  dim3 grid((g.N + 255) / 256, (g.M + 7) / 8, g.groups);
  if (g.K <= 1) launch_k(k_dx_skinny<1>, grid, 256, 0, s, g);
  else if (g.K <= 8) launch_k(k_dx_skinny<8>, grid, 256, 0, s, g);
  else launch_k(k_dx_skinny<16>, grid, 256, 0, s, g);
}

void launch_dw_skinny(const GemmArgs& g, cudaStream_t s) {
  dim3 grid((g.M + 127) / 128, g.groups);
  if (g.N <= 1) launch_k(k_dw_skinny<1>, grid, 128, 0, s, g);
  else if (g.N <= 8) launch_k(k_dw_skinny<8>, grid, 128, 0, s, g);
  else launch_k(k_dw_skinny<16>, grid, 128, 0, s, g);
}

// ================================================================== TD3 step bookkeeping
// Delayed-policy fire mask (algos.hpp:379-393), Adam step counters, target-noise stream keys
// (algos.hpp:253) and steps += 1 (:421).  One thread per member.
__global__ void k_td3_step_begin(int n, double* delay_acc, const double* ratio,
                                 const uint8_t* mask, int* fire, int64_t* t_pol, int64_t* t_c1,
                                 int64_t* t_c2, uint64_t* steps, const uint64_t* streams,
                                 uint64_t seed, uint64_t* noise_key, double* policy_loss,
                                 cudaGraphConditionalHandle any_fire, int set_cond, int shared,
                                 int ncrit, int* guard, double* hist, const uint64_t* hist_base,
                                 int hist_slots) {
  PDL_ENTRY();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  int f = 0;
  if (m < n && hist) {
    // loss history of an update call (pbrl_update_batches_losses): the previous step's
    // critic1 / critic2 / policy losses of this member into its history slot, before this step
    // overwrites them (steps[m] - hist_base[m] = steps of the call already begun)
    const uint64_t s = steps[m] - hist_base[m];
    if (s >= 1) {
      const double* losses = policy_loss - 2 * n;  // [critic1 | critic2 | policy][n]
      double* row = hist + static_cast<size_t>((s - 1) % hist_slots) * 3 * n;
      for (int q = 0; q < 3; ++q) row[q * n + m] = losses[q * n + m];
    }
  }
  if (m < n) {
    if (shared) {
      f = 1;  // shared critic: every policy updates every step (algos.hpp:382-384)
    } else {
      double acc = delay_acc[m] + ratio[m];
      if (acc >= 1.0 - 1e-12) {
        acc -= 1.0;
        f = 1;
      }
      delay_acc[m] = acc;
    }
    if (mask && !mask[m]) f = 0;
    fire[m] = f;
    if (m < ncrit) {
      t_c1[m] += 1;
      t_c2[m] += 1;
    }
    if (f) t_pol[m] += 1;
    // members that do not fire report a zero policy loss (k_td3_policy_loss writes the rest);
    // written here because the policy half may be skipped altogether
    if (!f) policy_loss[m] = 0.0;
    noise_key[m] = stream_key(seed, streams[m], kTargetNoise, steps[m]);
    steps[m] += 1;
  }
  // graph mode: the policy half of the step is an IF node on "some member fires"
  // (default 0 at every graph launch; any block with a firing member sets it)
  const int any = __syncthreads_or(f);
  if (set_cond && any && threadIdx.x == 0) cudaGraphSetConditional(any_fire, 1u);
  // the non-fire step graph (no policy half): a member that fires after all means the host
  // mirror of the accumulators diverged -- flagged in mapped host memory, raised by the host
  if (guard && any && threadIdx.x == 0) {
    *reinterpret_cast<volatile int*>(guard) = 1;
    __threadfence_system();
  }
  if (shared && blockIdx.x == 0) {
    // fire[n]: some member fires -> the shared critic's target Polyak (cmask {1}, :407-418);
    // block 0 scans the whole mask so no cross-block ordering is needed
    int a = 0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) a |= (!mask || mask[j]) ? 1 : 0;
    a = __syncthreads_or(a);
    if (threadIdx.x == 0) fire[n] = a;
  }
}

void launch_td3_step_begin(int n, double* delay_acc, const double* ratio, const uint8_t* mask,
                           int* fire, int64_t* t_pol, int64_t* t_c1, int64_t* t_c2,
                           uint64_t* steps, const uint64_t* streams, uint64_t seed,
                           uint64_t* noise_key, double* policy_loss,
                           cudaGraphConditionalHandle any_fire, int set_cond, int shared,
                           int ncrit, cudaStream_t s, int* guard, double* hist,
                           const uint64_t* hist_base, int hist_slots) {
  launch_k(k_td3_step_begin, (n + 127) / 128, 128, 0, s, n, delay_acc, ratio, mask, fire, t_pol,
           t_c1, t_c2, steps, streams, seed, noise_key, policy_loss, any_fire, set_cond, shared,
           ncrit, guard, hist, hist_base, hist_slots);
}

// concat_features (pop_tensor.hpp:432-456) of the batch into the critic-input layouts
// (IT: 32-bit element indices whenever the batch allows -- the row / column split is then a
// 32-bit division instead of a 64-bit one)
constexpr int kPackU = 2;
template <typename AT, typename IT>
__global__ void k_pack_batch(int n, int B, int ds, int da, int lsa, const float* s,
                             const float* a, const float* r, const float* s2, const float* d,
                             AT* in_sa, AT* in_s2a, AT* sa_pi, float* r_out, float* d_out,
                             AT* in_s, int lsp) {
  PDL_ENTRY();
  const IT dsa = static_cast<IT>(ds + da);
  const IT rows = static_cast<IT>(n) * static_cast<IT>(B);
  const IT total = rows * dsa;
  // kPackU elements per thread, kPackU * gridDim.x * blockDim.x apart: every load of a thread is
  // issued before its stores (the grid covers the batch in one resident wave)
  const IT span = static_cast<IT>(gridDim.x) * blockDim.x;
  for (IT e0 = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; e0 < total;
       e0 += kPackU * span) {
    float v[kPackU], v2[kPackU], rv[kPackU], dv[kPackU];
    IT row[kPackU];
    int col[kPackU];
#pragma unroll
    for (int u = 0; u < kPackU; ++u) {
      const IT e = e0 + u * span;
      row[u] = e / dsa;
      col[u] = static_cast<int>(e - row[u] * dsa);
      if (e >= total) continue;
      const int c = col[u];
      if (c < ds) {
        v[u] = __ldcs(s + static_cast<long long>(row[u]) * ds + c);
        v2[u] = __ldcs(s2 + static_cast<long long>(row[u]) * ds + c);
      } else {
        v[u] = __ldcs(a + static_cast<long long>(row[u]) * da + (c - ds));
      }
      if (c == 0) {
        rv[u] = __ldcs(r + row[u]);
        dv[u] = __ldcs(d + row[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kPackU; ++u) {
      if (e0 + u * span >= total) continue;
      const int c = col[u];
      const long long o = static_cast<long long>(row[u]) * lsa + c;
      act_st(in_sa, o, v[u]);
      if (c < ds) {
        act_st(sa_pi, o, v[u]);
        act_st(in_s2a, o, v2[u]);
        if (in_s) act_st(in_s, static_cast<long long>(row[u]) * lsp + c, v[u]);
      }
      if (c == 0) {
        r_out[row[u]] = rv[u];
        d_out[row[u]] = dv[u];
      }
    }
  }
}

template <typename AT>
static void launch_pack_t(int blocks, bool narrow, cudaStream_t st, int n, int B, int ds, int da,
                          int lsa, const float* s, const float* a, const float* r, const float* s2,
                          const float* d, void* in_sa, void* in_s2a, void* sa_pi, float* r_out,
                          float* d_out, void* in_s, int lsp) {
  if (narrow)
    launch_k(k_pack_batch<AT, unsigned>, blocks, 256, 0, st, n, B, ds, da, lsa, s, a, r, s2, d,
             static_cast<AT*>(in_sa), static_cast<AT*>(in_s2a), static_cast<AT*>(sa_pi), r_out,
             d_out, static_cast<AT*>(in_s), lsp);
  else
    launch_k(k_pack_batch<AT, long long>, blocks, 256, 0, st, n, B, ds, da, lsa, s, a, r, s2, d,
             static_cast<AT*>(in_sa), static_cast<AT*>(in_s2a), static_cast<AT*>(sa_pi), r_out,
             d_out, static_cast<AT*>(in_s), lsp);
}

void launch_pack_batch(int n, int B, int ds, int da, int lsa, const float* s, const float* a,
                       const float* r, const float* s2, const float* d, void* in_sa,
                       void* in_s2a, void* sa_pi, float* r_out, float* d_out, int act16,
                       cudaStream_t st, void* in_s, int lsp) {
  const long long total = static_cast<long long>(n) * B * (ds + da);
  const int blocks =
      static_cast<int>(std::min<long long>((total + 256 * kPackU - 1) / (256 * kPackU), 148 * 8));
  const bool narrow = total + 256LL * kPackU * blocks < (1LL << 32);
  if (act16)
    launch_pack_t<__nv_bfloat16>(blocks, narrow, st, n, B, ds, da, lsa, s, a, r, s2, d, in_sa,
                                 in_s2a, sa_pi, r_out, d_out, in_s, lsp);
  else
    launch_pack_t<float>(blocks, narrow, st, n, B, ds, da, lsa, s, a, r, s2, d, in_sa, in_s2a,
                         sa_pi, r_out, d_out, in_s, lsp);
}

// y = r + gamma*(1-done)*min(Q1', Q2')   (algos.hpp:268-281)
__global__ void k_td_target(int n, int B, const float* r, const float* d, const float* q2n,
                            const float* gamma, float* y) {
  PDL_ENTRY();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * B) return;
  const int m = e / B;
  const float qmin = minf_ref(q2n[e], q2n[n * B + e]);
  y[e] = r[e] + gamma[m] * (1.0f - d[e]) * qmin;
}

void launch_td_target(int n, int B, const float* r, const float* d, const float* q2n,
                      const float* gamma, float* y, cudaStream_t s) {
  launch_k(k_td_target, (n * B + 255) / 256, 256, 0, s, n, B, r, d, q2n, gamma, y);
}

// mse_loss_grads (algos.hpp:288-314): dq = (2/B)(q - y); loss = sum (double) d^2 / B in row order.
// The squares are staged through shared memory by the whole block (coalesced loads, exact
// double products) and summed by one thread in row order (the reference's double rounding).
constexpr int kLossChunk = 1024;

__global__ void k_mse(int n, int B, const float* q, const float* y, float* dq, double* loss,
                      int norm_rows) {
  PDL_ENTRY();
  __shared__ double sq[kLossChunk];
  const int grp = blockIdx.x;
  const int m = grp % n;
  const int nr = norm_rows ? norm_rows : B;  // shared critic: rows of the folded population
  const float scale = 2.0f / static_cast<float>(nr);
  const float* qg = q + static_cast<long long>(grp) * B;
  const float* yg = y + static_cast<long long>(m) * B;
  double acc = 0.0;
  for (int b0 = 0; b0 < B; b0 += kLossChunk) {
    const int nb = min(kLossChunk, B - b0);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      const int b = b0 + i;
      const float dl = qg[b] - yg[b];
      dq[static_cast<long long>(grp) * B + b] = scale * dl;
      sq[i] = static_cast<double>(dl) * static_cast<double>(dl);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < nb; ++i) acc += sq[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[grp] = acc / static_cast<double>(nr);
}

void launch_mse(int groups, int n, int B, const float* q, const float* y, float* dq, double* loss,
                cudaStream_t s, int norm_rows) {
  launch_k(k_mse, groups, 256, 0, s, n, B, q, y, dq, loss, norm_rows);
}

// td3_policy_loss_grads (algos.hpp:318-338): loss = -sum q / B; cotangent -1/B everywhere
__global__ void k_td3_policy_loss(int n, int B, const float* q, const int* fire, double* loss,
                                  float* gq) {
  PDL_ENTRY();
  __shared__ double sq[kLossChunk];
  const int m = blockIdx.x;
  const float gv = -1.0f / static_cast<float>(B);
  for (int b = threadIdx.x; b < B; b += blockDim.x) gq[static_cast<long long>(m) * B + b] = gv;
  if (!fire[m]) {
    if (threadIdx.x == 0) loss[m] = 0.0;
    return;
  }
  double acc = 0.0;
  for (int b0 = 0; b0 < B; b0 += kLossChunk) {
    const int nb = min(kLossChunk, B - b0);
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      sq[i] = static_cast<double>(q[static_cast<long long>(m) * B + b0 + i]);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < nb; ++i) acc -= sq[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[m] = acc / static_cast<double>(B);
}

void launch_td3_policy_loss(int n, int B, const float* q, const int* fire, double* loss,
                            float* gq, cudaStream_t s) {
  launch_k(k_td3_policy_loss, n, 256, 0, s, n, B, q, fire, loss, gq);
}

// ================================================================== fused Adam + Polyak
// adam_step_inplace (pop_tensor.hpp:328-366) with the bias corrections looked up from
// host-computed tables (corr[t] = (float)(1 - pow(beta, t)) in double, exactly :347-350), and
// the target update tgt = (T)tau*on + (T)(1-tau)*tgt (:422-426) fused on the fresh parameter.

// Member rows start 256-byte aligned (stride = P rounded up to 64), so each row is processed as
// float4 vectors (5 x 128-bit loads, 3-4 x 128-bit stores per thread) plus a scalar tail.
// __launch_bounds__(256, 4): at most 64 registers, 4 blocks (32 warps) per SM -- the occupancy
// that keeps enough 128-bit loads in flight for this HBM-bound stream (with 112 registers and 2
// blocks per SM the optimizer launches ran 40% longer on B200).
__global__ void __launch_bounds__(256, 4) k_adam(int n, size_t P, size_t stride,
                                              float* __restrict__ p, float* __restrict__ mo,
                                              float* __restrict__ vo, const float* __restrict__ g,
                                              const int64_t* t, const float* corr1,
                                              const float* corr2, const float* lr,
                                              const int* active, float* __restrict__ tgt,
                                              const float* tau_a, const float* tau_b,
                                              const int* polyak_gate,
                                              __nv_bfloat16* __restrict__ p16,
                                              __nv_bfloat16* __restrict__ t16) {
  PDL_ENTRY();
  const int grp = blockIdx.y;
  const int m = grp % n;
  if (active && !active[m]) return;
  const long long base = static_cast<long long>(grp) * stride;
  AdamScalars a;
  a.b1 = static_cast<float>(0.9);
  a.b2 = static_cast<float>(0.999);
  a.c1 = corr1[t[grp]];
  a.c2 = corr2[t[grp]];
  a.step = lr[m];
  a.epsv = static_cast<float>(1e-8);
  a.polyak = tgt && (!polyak_gate || polyak_gate[m]);
  a.ta = a.polyak ? tau_a[m] : 0.0f;
  a.tb = a.polyak ? tau_b[m] : 0.0f;
  const size_t P4 = P / 4;
  float4* p4 = reinterpret_cast<float4*>(p + base);
  float4* m4 = reinterpret_cast<float4*>(mo + base);
  float4* v4 = reinterpret_cast<float4*>(vo + base);
  const float4* g4 = reinterpret_cast<const float4*>(g + base);
  float4* t4 = a.polyak ? reinterpret_cast<float4*>(tgt + base) : nullptr;
  // two float4 slots per thread per trip, both slots' loads issued before either is updated
  // (more bytes in flight per thread for the HBM-bound stream)
  auto update = [&](size_t k, float4 pv, float4 mv, float4 vv, float4 gv, float4 tv) {
    adam_one(a, pv.x, mv.x, vv.x, gv.x);
    adam_one(a, pv.y, mv.y, vv.y, gv.y);
    adam_one(a, pv.z, mv.z, vv.z, gv.z);
    adam_one(a, pv.w, mv.w, vv.w, gv.w);
    __stcs(&p4[k], pv);  // streaming: the fp32 optimizer state is touched once per step; the
    __stcs(&m4[k], mv);  // bf16 operand copies the next step reads stay in L2 instead
    __stcs(&v4[k], vv);
    if (p16) {  // BF16 mode: the tensor-core copy of the fresh parameters
      __nv_bfloat162* d2 = reinterpret_cast<__nv_bfloat162*>(p16 + base) + 2 * k;
      d2[0] = __floats2bfloat162_rn(pv.x, pv.y);
      d2[1] = __floats2bfloat162_rn(pv.z, pv.w);
    }
    if (a.polyak) {
      tv.x = a.ta * pv.x + a.tb * tv.x;
      tv.y = a.ta * pv.y + a.tb * tv.y;
      tv.z = a.ta * pv.z + a.tb * tv.z;
      tv.w = a.ta * pv.w + a.tb * tv.w;
      __stcs(&t4[k], tv);
      if (t16) {
        __nv_bfloat162* d2 = reinterpret_cast<__nv_bfloat162*>(t16 + base) + 2 * k;
        d2[0] = __floats2bfloat162_rn(tv.x, tv.y);
        d2[1] = __floats2bfloat162_rn(tv.z, tv.w);
      }
    }
  };
  const size_t str = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t k0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k0 < P4;
       k0 += 2 * str) {
    const size_t k1 = k0 + str;
    const bool two = k1 < P4;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 p0 = __ldcs(&p4[k0]), m0 = __ldcs(&m4[k0]), v0 = __ldcs(&v4[k0]),
                 g0 = __ldcs(&g4[k0]);
    const float4 t0 = a.polyak ? __ldcs(&t4[k0]) : z;
    float4 p1 = z, m1 = z, v1 = z, g1 = z, t1 = z;
    if (two) {
      p1 = __ldcs(&p4[k1]);
      m1 = __ldcs(&m4[k1]);
      v1 = __ldcs(&v4[k1]);
      g1 = __ldcs(&g4[k1]);
      if (a.polyak) t1 = __ldcs(&t4[k1]);
    }
    update(k0, p0, m0, v0, g0, t0);
    if (two) update(k1, p1, m1, v1, g1, t1);
  }
  if (blockIdx.x == 0) {
    for (size_t k = P4 * 4 + threadIdx.x; k < P; k += blockDim.x) {
      const long long e = base + static_cast<long long>(k);
      float pk = p[e], mk = mo[e], vk = vo[e];
      adam_one(a, pk, mk, vk, g[e]);
      p[e] = pk;
      mo[e] = mk;
      vo[e] = vk;
      if (p16) p16[e] = __float2bfloat16_rn(pk);
      if (a.polyak) {
        tgt[e] = a.ta * pk + a.tb * tgt[e];
        if (t16) t16[e] = __float2bfloat16_rn(tgt[e]);
      }
    }
  }
}

void launch_adam(int groups, int n, size_t P, size_t stride, float* p, float* m, float* v,
                 const float* g, const int64_t* t, const float* corr1, const float* corr2,
                 const float* lr, const int* active, float* tgt, const float* tau_a,
                 const float* tau_b, const int* polyak_gate, __nv_bfloat16* p16,
                 __nv_bfloat16* t16, cudaStream_t s) {
  const int threads = 256;
  int bx = static_cast<int>((P / 4 + 2 * threads - 1) / (2 * threads));
  bx = bx < 1 ? 1 : bx;
  dim3 grid(bx, groups);
  launch_k(k_adam, grid, threads, 0, s, n, P, stride, p, m, v, g, t, corr1, corr2, lr, active, tgt,
           tau_a, tau_b, polyak_gate, p16, t16);
}

__global__ void k_copy_f64(double* dst, const double* src, size_t count) {
  PDL_ENTRY();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

void launch_copy_f64(double* dst, const double* src, size_t count, cudaStream_t s) {
  launch_k(k_copy_f64, static_cast<int>(std::min<size_t>((count + 255) / 256, 64)), 256, 0, s, dst,
           src, count);
}

__global__ void k_to_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                          size_t count) {
  PDL_ENTRY();
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[e] = __float2bfloat16_rn(src[e]);
}

void launch_to_bf16(const float* src, __nv_bfloat16* dst, size_t count, cudaStream_t s) {
  const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 148 * 8));
  launch_k(k_to_bf16, std::max(blocks, 1), 256, 0, s, src, dst, count);
}

// bias gradient for the tensor-core dW path: column sums of G over the batch, two-level and
// deterministic (32 columns x 8 row segments per block, segments combined in a fixed order).
template <typename AT>
__global__ void __launch_bounds__(256) k_colsum(int n, int B, int N, const AT* G, long long g_gs,
                                                long long g_ld, float* dst, long long dst_gs,
                                                const int* active) {
  PDL_ENTRY();
  const int grp = blockIdx.y;
  if (active && !active[grp % n]) return;
  __shared__ float part[8][33];
  const int c = threadIdx.x & 31, seg = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + c;
  const int rows = (B + 7) / 8;
  const int b0 = seg * rows, b1 = min(B, b0 + rows);
  float acc = 0.0f;
  if (o < N) {
    const AT* g = G + grp * g_gs + o;
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = act_ld(g, static_cast<long long>(b + u) * g_ld);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; b < b1; ++b) acc += act_ld(g, static_cast<long long>(b) * g_ld);
  }
  part[seg][c] = acc;
  __syncthreads();
  if (seg == 0 && o < N) {
    float t = part[0][c];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += part[q][c];
    dst[grp * dst_gs + o] = t;
  }
}

void launch_colsum(int groups, int n, int B, int N, const void* G, long long g_gs, long long g_ld,
                   float* dst, long long dst_gs, const int* active, int act16, cudaStream_t s) {
  dim3 grid((N + 31) / 32, groups);
  if (act16)
    launch_k(k_colsum<__nv_bfloat16>, grid, 256, 0, s, n, B, N,
             static_cast<const __nv_bfloat16*>(G), g_gs, g_ld, dst, dst_gs, active);
  else
    launch_k(k_colsum<float>, grid, 256, 0, s, n, B, N, static_cast<const float*>(G), g_gs, g_ld,
             dst, dst_gs, active);
}

// one thread per (group, row, 32-column word)
__global__ void k_mask_bits(int groups, int B, int H, int mw, const float* h, long long h_gs,
                            long long h_ld, uint32_t* mask, long long m_gs, long long m_ld,
                            const int* active, int n) {
  PDL_ENTRY();
  const long long total = static_cast<long long>(groups) * B * mw;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int w = static_cast<int>(e % mw);
    const long long gr = e / mw;
    const int r = static_cast<int>(gr % B), grp = static_cast<int>(gr / B);
    if (active && !active[grp % n]) continue;
    const float* row = h + grp * h_gs + static_cast<long long>(r) * h_ld;
    uint32_t bits = 0u;
    for (int j = 0; j < 32 && 32 * w + j < H; ++j) bits |= (row[32 * w + j] > 0.0f ? 1u : 0u) << j;
    mask[grp * m_gs + static_cast<long long>(r) * m_ld + w] = bits;
  }
}

void launch_mask_bits(int groups, int B, int H, const float* h, long long h_gs, long long h_ld,
                      uint32_t* mask, long long m_gs, long long m_ld, const int* active, int n,
                      cudaStream_t s) {
  const int mw = (H + 31) / 32;
  const long long total = static_cast<long long>(groups) * B * mw;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 8));
  launch_k(k_mask_bits, blocks, 256, 0, s, groups, B, H, mw, h, h_gs, h_ld, mask, m_gs, m_ld, active,
                                     n);
}

__global__ void k_td3_target_noise(int n, int B, int da, const uint64_t* key, const float* sd,
                                   const float* clip, float* eps) {
  PDL_ENTRY();
  const long long per = static_cast<long long>(B) * da;
  const long long total = per * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(e / per);
    const uint64_t i = static_cast<uint64_t>(e - m * per);  // b * da + o
    const float v = static_cast<float>(rng_normal_pair(key[m], 2 * i)) * sd[m];
    eps[e] = clampf_ref(v, -clip[m], clip[m]);
  }
}

void launch_td3_target_noise(int n, int B, int da, const uint64_t* key, const float* sd,
                             const float* clip, float* eps, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * B * da;
  const int blocks = static_cast<int>(std::min<long long>((total + 127) / 128, 148 * 16));
  launch_k(k_td3_target_noise, blocks, 128, 0, s, n, B, da, key, sd, clip, eps);
}

__global__ void k_fill(float* p, size_t count, float v) {
  PDL_ENTRY();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

void launch_fill(float* p, size_t count, float v, cudaStream_t s) {
  const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 148 * 8));
  launch_k(k_fill, blocks > 0 ? blocks : 1, 256, 0, s, p, count, v);
}

template <typename AT>
__global__ void k_fill_col(AT* p, long long rows, int ld, int col, float v) {
  PDL_ENTRY();
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<long long>(gridDim.x) * blockDim.x)
    act_st(p, r * ld + col, v);
}

void launch_fill_col(void* p, long long rows, int ld, int col, float v, int act16, cudaStream_t s) {
  const int blocks = static_cast<int>(std::min<long long>((rows + 255) / 256, 148 * 4));
  if (act16)
    launch_k(k_fill_col<__nv_bfloat16>, blocks, 256, 0, s, static_cast<__nv_bfloat16*>(p), rows,
             ld, col, v);
  else
    launch_k(k_fill_col<float>, blocks, 256, 0, s, static_cast<float*>(p), rows, ld, col, v);
}

// ================================================================== SAC
__global__ void k_sac_step_begin(int n, int64_t* t_pol, int64_t* t_c1, int64_t* t_c2,
                                 int64_t* t_alpha, uint64_t* steps, const uint64_t* streams,
                                 uint64_t seed, uint64_t* key_eps, uint64_t* key_eps_t) {
  PDL_ENTRY();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  t_pol[m] += 1;
  t_c1[m] += 1;
  t_c2[m] += 1;
  t_alpha[m] += 1;
  key_eps[m] = stream_key(seed, streams[m], kSacEps, steps[m]);
  key_eps_t[m] = stream_key(seed, streams[m], kSacEpsTarget, steps[m]);
  steps[m] += 1;
}

void launch_sac_step_begin(int n, int64_t* t_pol, int64_t* t_c1, int64_t* t_c2, int64_t* t_alpha,
                           uint64_t* steps, const uint64_t* streams, uint64_t seed,
                           uint64_t* key_eps, uint64_t* key_eps_t, cudaStream_t s) {
  launch_k(k_sac_step_begin, (n + 127) / 128, 128, 0, s, n, t_pol, t_c1, t_c2, t_alpha, steps, streams,
                                                   seed, key_eps, key_eps_t);
}

// glibc-exact float transcendentals for SAC (common.cuh)
__device__ __forceinline__ float sac_expf(float x) { return libm_expf(x); }
__device__ __forceinline__ float sac_log1pf(float x) { return libm_log1pf(x); }

// diagnostics: device libm ports over a host array (tests/test_gpu_numerics.py)
__global__ void k_libm_selftest(int fn, const float* in, float* out, uint64_t count) {
  PDL_ENTRY();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float x = in[i];
    out[i] = fn == 0 ? libm_tanhf(x) : (fn == 1 ? libm_expf(x) : libm_log1pf(x));
  }
}

void launch_libm_selftest(int fn, const float* in, float* out, uint64_t count, cudaStream_t s) {
  launch_k(k_libm_selftest, 148 * 8, 256, 0, s, fn, in, out, count);
}

// log_one_minus_tanh_sq (algos.hpp:523-529)
__device__ __forceinline__ float l1mts(float x) {
  const float z = -2.0f * x;
  const float sp = maxf_ref(z, 0.0f) + sac_log1pf(sac_expf(-fabsf(z)));
  return static_cast<float>(1.3862943611198906) - 2.0f * x - 2.0f * sp;
}

// split_policy_head + draw_eps + tanh_gaussian_logprob + tanh squash (algos.hpp:534-629)
template <typename AT>
__global__ void k_sac_head(int n, int B, int ds, int da, int lsa, const float* head, const uint64_t* key,
                           float bound, float log_bound, AT* sa, float* x, float* th,
                           float* ls_out, uint8_t* clamped, float* eps_out, float* logp) {
  PDL_ENTRY();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // (m, b)
  if (e >= n * B) return;
  const int m = e / B, b = e % B;
  const float hl2pi = static_cast<float>(0.9189385332046727);
  const float* h = head + static_cast<long long>(e) * 2 * da;
  float acc = 0.0f;
  for (int j = 0; j < da; ++j) {
    const long long k = static_cast<long long>(e) * da + j;
    const float mu = h[j];
    float ls = h[da + j];
    uint8_t c = 0;
    if (ls < static_cast<float>(-20.0)) { ls = static_cast<float>(-20.0); c = 1; }
    else if (ls > static_cast<float>(2.0)) { ls = static_cast<float>(2.0); c = 1; }
    const float ep = static_cast<float>(
        rng_normal_pair(key[m], 2 * (static_cast<uint64_t>(b) * da + j)));
    const float sig = sac_expf(ls);
    const float xv = mu + sig * ep;
    acc += -0.5f * ep * ep - ls - hl2pi;
    acc -= l1mts(xv);
    acc -= log_bound;
    const float t = libm_tanhf(xv);
    if (x) x[k] = xv;
    if (th) th[k] = t;
    if (ls_out) ls_out[k] = ls;
    if (clamped) clamped[k] = c;
    if (eps_out) eps_out[k] = ep;
    act_st(sa, static_cast<long long>(e) * lsa + ds + j, t * bound);
  }
  logp[e] = acc;
}

void launch_sac_head(int n, int B, int ds, int da, int lsa, const float* head,
                     const uint64_t* key, float bound, void* sa, float* x, float* th, float* ls,
                     uint8_t* clamped, float* eps, float* logp, int act16, cudaStream_t s) {
  extern float host_logf(float);
  if (act16)
    launch_k(k_sac_head<__nv_bfloat16>, (n * B + 127) / 128, 128, 0, s, n, B, ds, da, lsa, head,
             key, bound, host_logf(bound), static_cast<__nv_bfloat16*>(sa), x, th, ls, clamped,
             eps, logp);
  else
    launch_k(k_sac_head<float>, (n * B + 127) / 128, 128, 0, s, n, B, ds, da, lsa, head, key,
             bound, host_logf(bound), static_cast<float*>(sa), x, th, ls, clamped, eps, logp);
}

// ================================================================== action selection
// act (algos.hpp:895-915): a = clamp(a + (T)normal(key_m, 2e) * (T)(std_m * bound), +-bound) for
// members with std_m != 0, key_m = (seed, streams[m], kExploreNoise, steps[m]), e over the
// member's [rows][da] block; a already holds tanh * bound from the forward.
__global__ void k_td3_act_noise(int n, long long per, float* a, const double* noise_std,
                                const uint64_t* streams, const uint64_t* steps, uint64_t seed,
                                float bound) {
  PDL_ENTRY();
  const long long total = static_cast<long long>(n) * per;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / per);
    if (noise_std[m] == 0.0) continue;
    const uint64_t e = static_cast<uint64_t>(i - static_cast<long long>(m) * per);
    const uint64_t key = stream_key(seed, streams[m], kExploreNoise, steps[m]);
    const float sd = static_cast<float>(noise_std[m] * static_cast<double>(bound));
    a[i] = clampf_ref(a[i] + static_cast<float>(rng_normal_pair(key, 2 * e)) * sd, -bound, bound);
  }
}

void launch_td3_act_noise(int n, long long per, float* a, const double* noise_std,
                          const uint64_t* streams, const uint64_t* steps, uint64_t seed,
                          float bound, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * per;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 8));
  launch_k(k_td3_act_noise, std::max(blocks, 1), 256, 0, s, n, per, a, noise_std, streams, steps,
           seed, bound);
}

// sac_act (algos.hpp:918-942): head [n][rows][2 da] -> mu, log_std clamped to [-20, 2]
// (split_policy_head :599-616); mu += exp(log_std) * (T)normal(key_m, 2e) unless deterministic;
// a = tanh(mu) * bound.
__global__ void k_sac_act(int n, int rows, int da, const float* head, const uint64_t* streams,
                          const uint64_t* steps, uint64_t seed, int deterministic, float bound,
                          float* a) {
  PDL_ENTRY();
  const long long per = static_cast<long long>(rows) * da, total = per * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / per);
    const long long e = i - static_cast<long long>(m) * per;
    const long long row = e / da, j = e - row * da;
    const float* h = head + (static_cast<long long>(m) * rows + row) * 2 * da;
    float mu = h[j];
    float ls = h[da + j];
    if (ls < static_cast<float>(-20.0)) ls = static_cast<float>(-20.0);
    else if (ls > static_cast<float>(2.0)) ls = static_cast<float>(2.0);
    if (!deterministic) {
      const uint64_t key = stream_key(seed, streams[m], kExploreNoise, steps[m]);
      mu = mu + sac_expf(ls) * static_cast<float>(rng_normal_pair(key, 2 * static_cast<uint64_t>(e)));
    }
    a[i] = libm_tanhf(mu) * bound;
  }
}

void launch_sac_act(int n, int rows, int da, const float* head, const uint64_t* streams,
                    const uint64_t* steps, uint64_t seed, int deterministic, float bound, float* a,
                    cudaStream_t s) {
  const long long total = static_cast<long long>(n) * rows * da;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 8));
  launch_k(k_sac_act, std::max(blocks, 1), 256, 0, s, n, rows, da, head, streams, steps, seed,
           deterministic, bound, a);
}

// observations [n][rows][ds] (fp32) -> policy-input block [n][rows][ld] (fp32 or bf16)
template <typename AT>
__global__ void k_pack_obs(long long rows_total, int ds, int ld, const float* obs, AT* out) {
  PDL_ENTRY();
  const long long total = rows_total * ds;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / ds;
    act_st(out, r * ld + (i - r * ds), obs[i]);
  }
}

void launch_pack_obs(long long rows_total, int ds, int ld, const float* obs, void* out, int act16,
                     cudaStream_t s) {
  const long long total = rows_total * ds;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 8));
  if (act16)
    launch_k(k_pack_obs<__nv_bfloat16>, std::max(blocks, 1), 256, 0, s, rows_total, ds, ld, obs,
             static_cast<__nv_bfloat16*>(out));
  else
    launch_k(k_pack_obs<float>, std::max(blocks, 1), 256, 0, s, rows_total, ds, ld, obs,
             static_cast<float*>(out));
}

// y = rs*r + gamma*(1-d)*(min(Q1',Q2') - alpha*logp')  (algos.hpp:759-774)
__global__ void k_sac_y(int n, int B, const float* r, const float* d, const float* q2n,
                        const float* logp2, const float* log_alpha, const float* gamma,
                        const float* rscale, float* y) {
  PDL_ENTRY();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * B) return;
  const int m = e / B;
  const float alpha = sac_expf(log_alpha[m]);
  const float qmin = minf_ref(q2n[e], q2n[n * B + e]);
  y[e] = rscale[m] * r[e] + gamma[m] * (1.0f - d[e]) * (qmin - alpha * logp2[e]);
}

void launch_sac_y(int n, int B, const float* r, const float* d, const float* q2n,
                  const float* logp2, const float* log_alpha, const float* gamma,
                  const float* rscale, float* y, cudaStream_t s) {
  launch_k(k_sac_y, (n * B + 255) / 256, 256, 0, s, n, B, r, d, q2n, logp2, log_alpha, gamma, rscale,
                                              y);
}

// policy-loss cotangents (algos.hpp:665-692): -1/B routed to the smaller critic, logp weight
// alpha/B, loss accumulated per member in row order (double).
__global__ void k_sac_policy_top(int n, int B, const float* q2n, const float* logp,
                                 const float* log_alpha, double* loss, float* gq2n, float* lw) {
  PDL_ENTRY();
  const int m = blockIdx.x;
  const float am = static_cast<float>(exp(static_cast<double>(log_alpha[m])));
  const float inv_rows = 1.0f / static_cast<float>(B);
  const long long o = static_cast<long long>(m) * B;
  const long long o2 = static_cast<long long>(n) * B + o;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const float q1 = q2n[o + b], q2 = q2n[o2 + b];
    lw[o + b] = am * inv_rows;
    gq2n[o + b] = (q1 <= q2) ? -inv_rows : 0.0f;
    gq2n[o2 + b] = (q1 <= q2) ? 0.0f : -inv_rows;
  }
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int b = 0; b < B; ++b) {
      const float qmin = minf_ref(q2n[o + b], q2n[o2 + b]);
      acc += static_cast<double>(am * logp[o + b] - qmin) / static_cast<double>(B);
    }
    loss[m] = acc;
  }
}

void launch_sac_policy_top(int n, int B, const float* q2n, const float* logp,
                           const float* log_alpha, double* loss, float* gq2n, float* lw,
                           cudaStream_t s) {
  launch_k(k_sac_policy_top, n, 256, 0, s, n, B, q2n, logp, log_alpha, loss, gq2n, lw);
}

// tanh_gaussian_logprob_backward + the action path (algos.hpp:571-595, :705-724) -> head grad
__global__ void k_sac_head_grad(int n, int B, int da, const float* ga2n, const float* lw,
                                const float* x, const float* th, const float* ls,
                                const uint8_t* clamped, const float* eps, float bound,
                                float* gh) {
  PDL_ENTRY();
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;  // (m,b,j)
  const long long total = static_cast<long long>(n) * B * da;
  if (e >= total) return;
  const long long row = e / da;
  const int j = static_cast<int>(e % da);
  const float w = lw[row];
  const float dlogp_dx = 2.0f * libm_tanhf(x[e]);
  const float el = sac_expf(ls[e]);
  float gmu = w * dlogp_dx;
  float gls = w * (dlogp_dx * el * eps[e] - 1.0f);
  const float ga = ga2n[e] + ga2n[total + e];
  const float t = th[e];
  const float dadx = bound * (1.0f - t * t);
  const float gx = ga * dadx;
  gmu += gx;
  gls += gx * el * eps[e];
  if (clamped[e]) gls = 0.0f;
  gh[row * 2 * da + j] = gmu;
  gh[row * 2 * da + da + j] = gls;
}

void launch_sac_head_grad(int n, int B, int da, const float* ga2n, const float* lw,
                          const float* x, const float* th, const float* ls,
                          const uint8_t* clamped, const float* eps, float bound, float* gh,
                          cudaStream_t s) {
  const long long total = static_cast<long long>(n) * B * da;
  launch_k(k_sac_head_grad, static_cast<int>((total + 255) / 256), 256, 0, s, 
      n, B, da, ga2n, lw, x, th, ls, clamped, eps, bound, gh);
}

// temperature step (algos.hpp:814-825): g = -alpha * mean_b(logp + target_entropy) in double,
// then a one-parameter Adam on log_alpha.
__global__ void k_sac_alpha(int n, int B, const float* logp, const double* te,
                            float* log_alpha, float* am, float* av, const int64_t* t,
                            const float* corr1, const float* corr2, const float* lr) {
  PDL_ENTRY();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const double alpha = exp(static_cast<double>(log_alpha[m]));
  double mt = 0.0;
  for (int b = 0; b < B; ++b) mt += static_cast<double>(logp[static_cast<long long>(m) * B + b]) + te[m];
  mt /= static_cast<double>(B);
  const float g = static_cast<float>(-alpha * mt);
  const float b1 = static_cast<float>(0.9), b2 = static_cast<float>(0.999);
  const float mk = b1 * am[m] + (1.0f - b1) * g;
  const float vk = b2 * av[m] + (1.0f - b2) * g * g;
  am[m] = mk;
  av[m] = vk;
  const float mhat = mk / corr1[t[m]];
  const float vhat = vk / corr2[t[m]];
  log_alpha[m] = log_alpha[m] - lr[m] * mhat / (sqrtf(vhat) + static_cast<float>(1e-8));
}

void launch_sac_alpha(int n, int B, const float* logp, const float* log_alpha_in,
                      const double* target_entropy, float* log_alpha, float* am, float* av,
                      const int64_t* t, const float* corr1, const float* corr2, const float* lr,
                      cudaStream_t s) {
  (void)log_alpha_in;
  launch_k(k_sac_alpha, (n + 127) / 128, 128, 0, s, n, B, logp, target_entropy, log_alpha, am, av, t,
                                              corr1, corr2, lr);
}

// ================================================================== replay
// ReplayBuffer rows live in HBM as [buffer][cap][rw] floats: s | a | s2 | r | done | pad.
__global__ void k_replay_scatter(const float* rows, const uint64_t* dst_row, uint64_t count,
                                 int rw, float* ring) {
  PDL_ENTRY();
  const long long total = static_cast<long long>(count) * rw;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / rw;
    const int c = static_cast<int>(e % rw);
    ring[dst_row[i] * rw + c] = rows[e];
  }
}

void launch_replay_scatter(const float* rows, const uint64_t* dst_row, uint64_t count, int rw,
                           float* ring, cudaStream_t s) {
  const long long total = static_cast<long long>(count) * rw;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  launch_k(k_replay_scatter, blocks > 0 ? blocks : 1, 256, 0, s, rows, dst_row, count, rw, ring);
}

// sample_batch (replay.hpp:181-204): slot = bits(key, b) % size with key =
// RngStream::of(seed, streams[m], kSample, draw_id), rows gathered into the critic-input layouts.
// Warp w gathers rows [8w, 8w + 8): lanes 0-7 each derive one row's slot (stream key, counter
// hash, modulo), the slots are broadcast, and the 8 rows' words are loaded together (up to 11
// independent loads per lane in flight, one memory round trip for 8 random rows) before they are
// routed into the critic-input layouts.
constexpr int kGatherRows = 8;

template <typename AT>
__global__ void __launch_bounds__(256) k_replay_gather(
    int n, int B, int ds, int da, int lsa, int rw, const float* ring, uint64_t cap, int shared,
    const uint64_t* sizes, const uint64_t* streams, uint64_t seed, uint64_t draw_id, AT* in_sa,
    AT* in_s2a, AT* sa_pi, float* r_out, float* d_out, AT* in_s, int lsp) {
  PDL_ENTRY();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int rows = n * B;
  const int g0 = warp * kGatherRows;
  if (g0 >= rows) return;
  const int width = 2 * ds + da + 2;  // s | a | s2 | r | done
  uint64_t base = 0;
  if (lane < kGatherRows && g0 + lane < rows) {
    const int g = g0 + lane, m = g / B, b = g - m * B;
    const int buf = shared ? 0 : m;
    const uint64_t key = stream_key(seed, streams[m], kSample, draw_id);
    const uint64_t slot = rng_bits(key, static_cast<uint64_t>(b)) % sizes[buf];
    base = (static_cast<uint64_t>(buf) * cap + slot) * rw;
  }
  constexpr int kMaxPer = 16;  // words per lane: 8 rows x width <= 32 x 16 (width <= 64)
  const int total = kGatherRows * width;
  float v[kMaxPer];
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int e = lane + 32 * u;
    const int r = e / width;
    const uint64_t rb = __shfl_sync(0xffffffffu, base, r < kGatherRows ? r : 0);
    v[u] = (e < total && g0 + r < rows) ? __ldcs(ring + rb + (e - r * width)) : 0.0f;
  }
  const int dsa = ds + da;
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int e = lane + 32 * u;
    if (e >= total) break;
    const int r = e / width, c = e - r * width;
    const int g = g0 + r;
    if (g >= rows) continue;
    const long long o = static_cast<long long>(g) * lsa;
    const float x = v[u];
    if (c < ds) {
      act_st(in_sa, o + c, x);
      if (sa_pi) act_st(sa_pi, o + c, x);
      if (in_s) act_st(in_s, static_cast<long long>(g) * lsp + c, x);
    } else if (c < dsa) {
      act_st(in_sa, o + c, x);
    } else if (c < dsa + ds) {
      act_st(in_s2a, o + (c - dsa), x);
    } else if (c == dsa + ds) {
      r_out[g] = x;
    } else {
      d_out[g] = x;
    }
  }
}

void launch_replay_gather(int n, int B, int ds, int da, int lsa, int rw, const float* ring,
                          uint64_t cap, int shared, const uint64_t* sizes,
                          const uint64_t* streams, uint64_t seed, uint64_t draw_id,
                          void* in_sa, void* in_s2a, void* sa_pi, float* r_out, float* d_out,
                          int act16, cudaStream_t s, void* in_s, int lsp) {
  if (2 * ds + da + 2 > 64)
    PBRL_THROW(PBRL_E_CONFIG, "replay gather: transitions wider than 64 words");
  const long long warps = (static_cast<long long>(n) * B + kGatherRows - 1) / kGatherRows;
  const int blocks = static_cast<int>((warps * 32 + 255) / 256);
  if (act16)
    launch_k(k_replay_gather<__nv_bfloat16>, blocks, 256, 0, s, n, B, ds, da, lsa, rw, ring, cap,
             shared, sizes, streams, seed, draw_id, static_cast<__nv_bfloat16*>(in_sa),
             static_cast<__nv_bfloat16*>(in_s2a), static_cast<__nv_bfloat16*>(sa_pi), r_out,
             d_out, static_cast<__nv_bfloat16*>(in_s), lsp);
  else
    launch_k(k_replay_gather<float>, blocks, 256, 0, s, n, B, ds, da, lsa, rw, ring, cap, shared,
             sizes, streams, seed, draw_id, static_cast<float*>(in_sa),
             static_cast<float*>(in_s2a), static_cast<float*>(sa_pi), r_out, d_out,
             static_cast<float*>(in_s), lsp);
}

// ================================================================== PBT
// pbt_rank (evolve.hpp:112-122) as a stable rank: position of i = #{j : f_j > f_i} +
// #{j < i : f_j == f_i}; then pbt_plan (:133-145): replaced[i] = order[n-1-i],
// donors[i] = order[bits(key, next + i) % cut].  One block.
__global__ void k_pbt_plan(int n, const double* fitness, int cut, uint64_t key, uint64_t next,
                           uint64_t* order, uint64_t* replaced, uint64_t* donors) {
  PDL_ENTRY();
  // stable descending rank = #(better) + #(equal with a lower index).  NaN fitness (a diverged
  // member) ranks as -inf, so the comparison is a total order and `order` a permutation.
  auto rank_key = [](double f) { return f != f ? -CUDART_INF : f; };
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double fi = rank_key(fitness[i]);
    int pos = 0;
    for (int j = 0; j < n; ++j) {
      const double fj = rank_key(fitness[j]);
      pos += (fj > fi) || (j < i && fj == fi);
    }
    order[pos] = static_cast<uint64_t>(i);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cut; i += blockDim.x) {
    replaced[i] = order[n - 1 - i];
    donors[i] = order[rng_bits(key, next + static_cast<uint64_t>(i)) % static_cast<uint64_t>(cut)];
  }
}

void launch_pbt_plan(int n, const double* fitness, int cut, uint64_t key, uint64_t next,
                     uint64_t* order, uint64_t* replaced, uint64_t* donors, cudaStream_t s) {
  launch_k(k_pbt_plan, 1, 256, 0, s, n, fitness, cut, key, next, order, replaced, donors);
}

// copy_member (net_pop.hpp:192-202) for many (src, dst) pairs of one arena
__global__ void k_member_copy(float* arena, size_t stride, size_t P, const uint64_t* src,
                              const uint64_t* dst) {
  PDL_ENTRY();
  const int pr = blockIdx.y;
  const uint64_t s = src[pr], d = dst[pr];
  if (s == d) return;
  const float* a = arena + s * stride;
  float* b = arena + d * stride;
  for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < P;
       k += static_cast<size_t>(gridDim.x) * blockDim.x)
    b[k] = a[k];
}

void launch_member_copy(float* arena, size_t stride, size_t P, const uint64_t* src,
                        const uint64_t* dst, int pairs, cudaStream_t s) {
  if (pairs <= 0) return;
  dim3 grid(static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((P + 1023) / 1024, 64))),
            pairs);
  launch_k(k_member_copy, grid, 256, 0, s, arena, stride, P, src, dst);
}

__global__ void k_member_zero(float* arena, size_t stride, const uint64_t* dst) {
  PDL_ENTRY();
  float* b = arena + dst[blockIdx.y] * stride;
  for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < stride;
       k += static_cast<size_t>(gridDim.x) * blockDim.x)
    b[k] = 0.0f;
}

void launch_member_zero(float* arena, size_t stride, const uint64_t* dst, int pairs,
                        cudaStream_t s) {
  if (pairs <= 0) return;
  dim3 grid(static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((stride + 1023) / 1024, 64))),
            pairs);
  launch_k(k_member_zero, grid, 256, 0, s, arena, stride, dst);
}

// ================================================================== init
// init_pop_mlp (net_pop.hpp:69-100): w = (T)(lo + (hi-lo)*u) in double per (member, layer)
// stream; exact on the device (IEEE double ops, no contraction).
__global__ void k_init_layer(float* arena, size_t stride, size_t woff, size_t boff, int fi,
                             int fo, uint64_t member_offset, uint64_t seed, int layer) {
  PDL_ENTRY();
  const int m = blockIdx.y;
  const uint64_t gm = member_offset + static_cast<uint64_t>(m);
  const double wb = sqrt(1.0 / static_cast<double>(fi));
  const double bb = 1.0 / sqrt(static_cast<double>(fi));
  const uint64_t ws = stream_key(seed, gm, kInitWeight, static_cast<uint64_t>(layer));
  const uint64_t bs = stream_key(seed, gm, kInitBias, static_cast<uint64_t>(layer));
  float* w = arena + static_cast<size_t>(m) * stride + woff;
  float* bv = arena + static_cast<size_t>(m) * stride + boff;
  const size_t nw = static_cast<size_t>(fi) * fo;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < nw + fo;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (e < nw) {
      w[e] = static_cast<float>(-wb + (wb - (-wb)) * rng_uniform(ws, e));
    } else {
      const size_t k = e - nw;
      bv[k] = static_cast<float>(-bb + (bb - (-bb)) * rng_uniform(bs, k));
    }
  }
}

void launch_init_net(const NetShape& sh, float* arena, int n, uint64_t member_offset,
                     uint64_t seed, cudaStream_t s) {
  for (int l = 0; l < sh.depth; ++l) {
    const size_t cnt = static_cast<size_t>(sh.dims[l]) * sh.dims[l + 1] + sh.dims[l + 1];
    dim3 grid(static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((cnt + 255) / 256, 64))),
              n);
    launch_k(k_init_layer, grid, 256, 0, s, arena, sh.stride, sh.woff[l], sh.boff[l], sh.dims[l],
                                      sh.dims[l + 1], member_offset, seed, l);
  }
}

// make_synthetic_batches (bench.hpp:69-93): per batch i, s/a/r/s2 ~ U[-1,1) from
// RngStream::of(seed, i, kGeneric, 1..4) and done = U < 0.02 from step 5; element e counters.
__global__ void k_synth(uint64_t n_elems_s, uint64_t n_elems_a, uint64_t n_elems_r, uint64_t seed,
                        uint64_t batch, float* s, float* a, float* r, float* s2, float* d) {
  PDL_ENTRY();
  const uint64_t ks = stream_key(seed, batch, kGeneric, 1), ka = stream_key(seed, batch, kGeneric, 2),
                 kr = stream_key(seed, batch, kGeneric, 3), k2 = stream_key(seed, batch, kGeneric, 4),
                 kd = stream_key(seed, batch, kGeneric, 5);
  const uint64_t total = 2 * n_elems_s + n_elems_a + 2 * n_elems_r;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t k = e;
    if (k < n_elems_s) { s[k] = static_cast<float>(-1.0 + (1.0 - (-1.0)) * rng_uniform(ks, k)); continue; }
    k -= n_elems_s;
    if (k < n_elems_a) { a[k] = static_cast<float>(-1.0 + (1.0 - (-1.0)) * rng_uniform(ka, k)); continue; }
    k -= n_elems_a;
    if (k < n_elems_r) { r[k] = static_cast<float>(-1.0 + (1.0 - (-1.0)) * rng_uniform(kr, k)); continue; }
    k -= n_elems_r;
    if (k < n_elems_s) { s2[k] = static_cast<float>(-1.0 + (1.0 - (-1.0)) * rng_uniform(k2, k)); continue; }
    k -= n_elems_s;
    d[k] = rng_uniform(kd, k) < 0.02 ? 1.0f : 0.0f;
  }
}

void launch_synth(uint64_t count, uint64_t n, uint64_t b, uint64_t ds, uint64_t da, uint64_t seed,
                  float* s, float* a, float* r, float* s2, float* d, cudaStream_t st) {
  const uint64_t es = n * b * ds, ea = n * b * da, er = n * b;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t total = 2 * es + ea + 2 * er;
    const int blocks = static_cast<int>(std::min<uint64_t>((total + 255) / 256, 148 * 16));
    launch_k(k_synth, blocks, 256, 0, st, es, ea, er, seed, i, s + i * es, a + i * ea, r + i * er,
                                    s2 + i * es, d + i * er);
  }
}

}  // namespace pbrl
