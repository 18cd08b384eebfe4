// Host interface of the tcgen05 grouped GEMM (tc_gemm.cu).
#pragma once

#include <cstdint>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace pbrl {

// A 3-D operand in global memory: [groups][rows][cols] with element (r, c) of group g at
// p + g*gs + r*ld + c (elements of TcArgs::eb bytes: fp32 in TF32 mode, bf16 in BF16 mode).
// rows / cols are the LOGICAL extents (TMA zero-fills past them).
struct TcOperand {
  const void* p = nullptr;
  uint64_t cols = 0, rows = 0, groups = 0, ld = 0, gs = 0;
};

struct TcArgs {
  int M = 0, N = 0, K = 0, groups = 0, n_members = 1;
  int eb = 4;   // operand element bytes: 4 = fp32 (kind::tf32), 2 = bf16 (kind::f16)
  int c16 = 0;  // C (incl. the fused hidden store) is bf16 (activations in BF16 mode)
  int oc16 = 0; // the fused output layer's oC is bf16 (actions written into critic inputs)
  int stages = 4;  // smem pipeline depth (set by the launcher)
  int a_by_member = 0, b_by_member = 0;
  int epi = 0;
  void* C = nullptr;
  long long c_gs = 0, c_rs = 0;
  int c_by_member = 0;
  const float* bias = nullptr;
  long long bias_gs = 0;
  const float* aux = nullptr;
  long long aux_gs = 0, aux_rs = 0;
  int aux_by_member = 0;
  float* C2 = nullptr;
  long long c2_gs = 0, c2_rs = 0;
  float scale = 1.0f;
  const int* active = nullptr;
  const uint64_t* noise_key = nullptr;
  const float* noise_sd = nullptr;
  const float* noise_clip = nullptr;
  float bound = 1.0f;
  // Fused output layer (requires the whole hidden width in one tile, N <= BN): the epilogue
  // applies bias + ReLU to its hidden row h and evaluates y[o] = sum_j h[j] * ow[j][o] + ob[o]
  // (j ascending) followed by out_epi; the hidden row is stored only if store_hidden.
  int nout = 0;
  const float* ow = nullptr;  // W_out [N][nout] of group g at ow + g * ow_gs; b_out follows it
  long long ow_gs = 0;
  int out_epi = 0;
  void* oC = nullptr;
  long long oc_gs = 0, oc_rs = 0;
  float* oC2 = nullptr;
  long long oc2_gs = 0, oc2_rs = 0;
  float out_scale = 1.0f;
  int store_hidden = 1;
  // dX variant of the fused output layer (the policy-loss chain's last critic dX straight into
  // the action columns): hidden = ReLU'-masked accumulator (mask bits, no bias), output-layer
  // weights read transposed, w(j, o) = ow[g * ow_gs + o * ow_ld + j], no output bias; out_epi
  // EPI_TANH_GRAD (aux = tanh values, scale) or EPI_STORE
  int ow_tr = 0;
  long long ow_ld = 0;
  // ReLU masks as bits: a storing BIAS_RELU / fused epilogue writes bit (c % 32) of word c / 32
  // of row r = (h[r][c] > 0) to mask_out; EPI_RELU_MASK reads mask_in (when set) instead of aux
  uint32_t* mask_out = nullptr;
  long long mo_gs = 0, mo_ld = 0;
  const uint32_t* mask_in = nullptr;
  long long mi_gs = 0, mi_ld = 0;
  int mi_by_member = 0;
  // precomputed clipped target-policy noise [group][row][nout] for out_epi BIAS_TANH_NOISE
  const float* noise_eps = nullptr;
  long long ne_gs = 0, ne_rs = 0;
  int c_tma = 0, aux_tma = 0;  // set by launch_tc_gemm
  unsigned long long* trace = nullptr;  // diagnostics timeline (PBRL_TC_TRACE), see tc_gemm.cu
  int b_prefetch = 0;  // B (weights) may be read before the PDL wait (predecessor wrote none)
  int max_ctas = 0;    // > 0: cap the persistent grid (a concurrent launch takes the other SMs)
};

struct TcTraceMeta {
  int bn, a_mn, b_mn, nout, M, N, K, groups, epi, pad;
};
// copies the recorded launch timelines ([launch][160 CTAs][64 stamps], ns) and their metadata
void tc_trace_init();  // allocates the trace buffer when PBRL_TC_TRACE is set
int tc_trace_dump(unsigned long long* host, TcTraceMeta* meta, int max_launches);

// TMA requirements: 16-byte aligned base and strides (elements of eb bytes).
bool tma_ok(const void* base, uint64_t row_stride_elems, uint64_t group_stride_elems, int eb = 4);

// a_mn / b_mn: operand is MN-major (the M / N index is the contiguous one in memory).
//   A K-major : A(m, k) = A.p[g][m][k]  (rows = M extent, cols = K extent)
//   A MN-major: A(m, k) = A.p[g][k][m]  (rows = K extent, cols = M extent)
//   B K-major : B(n, k) = B.p[g][n][k]  (rows = N extent, cols = K extent)
//   B MN-major: B(n, k) = B.p[g][k][n]  (rows = K extent, cols = N extent)
void launch_tc_gemm(const TcOperand& A, const TcOperand& B, bool a_mn, bool b_mn,
                    const TcArgs& g, cudaStream_t s);

// Two hidden layers and the output layer of one MLP forward in ONE persistent launch (BF16
// mode): per 128-row tile of a group, h1 = relu(X W1 + b1) is written by the epilogue straight
// into shared memory as the K-major tcgen05 operand of h2 = relu(h1 W2 + b2), whose epilogue
// evaluates the output layer (out_epi as in TcArgs).  h1 / h2 and their ReLU mask bits reach HBM
// only when kept for the backward pass (H1g / H2g non-null).  Requirements: in <= 64, H1 a
// multiple of 64 and <= 256, H2 a multiple of 32 and <= 256, nout <= 16.
struct Fwd2Args {
  int M = 0, in = 0, H1 = 0, H2 = 0, groups = 0, n_members = 1;
  int max_ctas = 0;  // > 0: cap the persistent grid (a concurrent branch takes the other SMs)
  const void* X = nullptr;  // bf16 [groups or members][M][x_ld]
  long long x_ld = 0, x_gs = 0;
  int x_by_member = 0;
  const void* W1 = nullptr;  // bf16 operand copies, W1 [in][H1], W2 [H1][H2], group stride w_gs
  const void* W2 = nullptr;
  long long w_gs = 0;
  const float* b1 = nullptr;  // fp32 master rows (group stride p_gs): b1, b2, W_out [H2][nout]
  const float* b2 = nullptr;  // followed by b_out
  const float* ow = nullptr;
  long long p_gs = 0;
  int nout = 0, out_epi = 0;
  float out_scale = 1.0f;
  void* oC = nullptr;
  long long oc_gs = 0, oc_rs = 0;
  int oc16 = 0;
  float* oC2 = nullptr;
  long long oc2_gs = 0, oc2_rs = 0;
  void* H1g = nullptr;  // bf16 [groups][M][h1_ld] + mask bits m1 (nullptr: not kept)
  long long h1_gs = 0, h1_ld = 0;
  uint32_t* m1 = nullptr;
  long long m1_gs = 0, m1_ld = 0;
  void* H2g = nullptr;
  long long h2_gs = 0, h2_ld = 0;
  uint32_t* m2 = nullptr;
  long long m2_gs = 0, m2_ld = 0;
  const int* active = nullptr;
  const uint64_t* noise_key = nullptr;
  const float* noise_sd = nullptr;
  const float* noise_clip = nullptr;
  float bound = 1.0f;
  const float* noise_eps = nullptr;
  long long ne_gs = 0, ne_rs = 0;
  unsigned long long* trace = nullptr;  // diagnostics (PBRL_TC_TRACE)
};
bool mlp_fwd2_ok(const Fwd2Args& a);
void launch_mlp_fwd2(const Fwd2Args& a, cudaStream_t s);

int num_sms_host();  // multiprocessors of the current device

}  // namespace pbrl
