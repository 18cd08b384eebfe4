// Internal declarations of the B200 population-update library.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pbrl_b200.h"
#include "common.cuh"

namespace pbrl {

constexpr int kMaxLayers = 8;
enum Act { ACT_NONE = 0, ACT_RELU = 1, ACT_TANH = 2 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PBRL_THROW(code, msg) throw ::pbrl::Error((code), (msg))
#define CUDA_CHECK(x)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw ::pbrl::Error(PBRL_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

// ---- programmatic dependent launch (PDL).  Every kernel is launched with
// programmaticStreamSerialization, so it may start while its stream predecessor is still
// draining; PDL_ENTRY() (the first statement of every kernel) waits for the predecessor grid to
// complete and be visible (griddepcontrol.wait) and then lets this grid's own successor start
// launching (griddepcontrol.launch_dependents).  Kernel launch latency and the prologue of the
// next kernel overlap the tail of the previous one; CUDA-graph capture keeps the edges.
#define PDL_ENTRY()                                                   \
  do {                                                                \
    asm volatile("griddepcontrol.wait;" ::: "memory");                \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   \
  } while (0)

bool pdl_enabled();  // PBRL_NO_PDL=1 disables the attribute (diagnostics)

// Activation storage: fp32 (FFMA32 / TF32 modes) or bf16 (BF16 mode); arithmetic is fp32.
__device__ __forceinline__ float act_ld(const float* p, long long i) { return p[i]; }
__device__ __forceinline__ float act_ld(const __nv_bfloat16* p, long long i) {
  return __bfloat162float(p[i]);
}
__device__ __forceinline__ void act_st(float* p, long long i, float v) { p[i] = v; }
__device__ __forceinline__ void act_st(__nv_bfloat16* p, long long i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

// Every kernel states the same preferred shared-memory carveout (a kernel that needs more gets
// more), so the small kernels between the big tensor-core ones do not flip the SMs' L1 /
// shared-memory split back and forth; the value was picked by measurement (kernels.cu).
// PBRL_CARVEOUT=<percent> overrides (diagnostics; -1 = driver default).
int carveout_pref();

template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
              Args&&... args) {
  static bool carve_set = false;
  if (!carve_set) {
    const int c = carveout_pref();
    if (c >= 0)
      CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c));
    carve_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// A population of identically shaped MLPs (PopMLPParams, net_pop.hpp:17-43).  On device every
// member occupies `stride` floats (P rounded up to 64 so member rows are 256 B aligned); the
// first P floats are the member in flatten_member order: W0 [in][out], b0, W1, b1, ...
struct NetShape {
  int depth = 0;
  int dims[kMaxLayers + 1] = {};
  int out_act = ACT_NONE;
  float out_scale = 1.0f;
  size_t P = 0, stride = 0;
  size_t woff[kMaxLayers] = {}, boff[kMaxLayers] = {};
  void make(const std::vector<size_t>& d, int act, float scale);
  int max_hidden() const;
};

// ------------------------------------------------------------------ GEMM launch descriptor
// C[g](i,j) = epi( sum_k A[g](i,k) * B[g](k,j) ), k ascending (the reference order).
// Operand element (r,c) of group g lives at base + grp*gs + r*rs + c*cs, where grp = g, or
// the member id m = g % n_members when the operand is shared by the critics of one member.
enum Epi {
  EPI_STORE = 0,        // C = acc
  EPI_BIAS = 1,         // C = acc + bias[j]
  EPI_BIAS_RELU = 2,    // C = relu(acc + bias[j])
  EPI_BIAS_TANH = 3,    // t = tanh(acc + bias[j]); C2 = t; C = t * scale
  EPI_BIAS_TANH_NOISE = 4,  // as EPI_BIAS_TANH, then TD3 target smoothing noise on C
  EPI_RELU_MASK = 5,    // C = aux(i,j) > 0 ? acc : 0       (activation_backward, relu)
  EPI_TANH_GRAD = 6,    // g = acc * scale; C = g * (1 - aux^2)   (tanh backward, aux = t)
};

struct Operand {
  const float* p = nullptr;
  long long gs = 0, rs = 0, cs = 0;
  int by_member = 0;
};

struct GemmArgs {
  int M = 0, N = 0, K = 0, groups = 0, n_members = 1;
  Operand A, B;
  int a_ones_row = 0;  // row M-1 of A is all ones: C row M-1 = column sums of B (bias grad)
  int a16 = 0, c16 = 0;  // BF16 mode (k_fwd_skinny only): A / C are bf16 activations
  int rowdot = 0;        // tensor-core modes: k_fwd_skinny may use the warp-per-row kernel
  float* C = nullptr;
  long long c_gs = 0, c_rs = 0;
  int c_by_member = 0;
  int epi = EPI_STORE;
  Operand bias;        // bias row vector (cs = 1)
  Operand aux;         // relu mask source / tanh values
  float* C2 = nullptr; // tanh values out
  long long c2_gs = 0, c2_rs = 0;
  float scale = 1.0f;
  float acc_init = 0.0f;     // -0.0f reproduces "first product assigned" (pop_tensor.hpp:158-160)
  const int* active = nullptr;  // per-member gate (policy fire mask)
  // target smoothing noise (algos.hpp:252-262)
  const uint64_t* noise_key = nullptr;
  const float* noise_sd = nullptr;
  const float* noise_clip = nullptr;
  // tensor-core modes: the same draws precomputed by k_td3_target_noise, [member][M][N]
  const float* noise_eps = nullptr;
  long long ne_gs = 0;
  float bound = 1.0f;
};

void launch_gemm_simt(const GemmArgs& g, cudaStream_t s);

// adam_step_inplace per element (pop_tensor.hpp:345-363)
struct AdamScalars {
  float b1, b2, c1, c2, step, epsv, ta, tb;
  bool polyak;
};

__device__ __forceinline__ float adam_one(const AdamScalars& a, float& p, float& mo, float& vo,
                                          float gk) {
  const float mk = a.b1 * mo + (1.0f - a.b1) * gk;
  const float vk = a.b2 * vo + (1.0f - a.b2) * gk * gk;
  mo = mk;
  vo = vk;
  const float mhat = mk / a.c1;
  const float vhat = vk / a.c2;
  p = p - a.step * mhat / (sqrtf(vhat) + a.epsv);
  return p;
}
// Output-layer backward in one pass (dX with relu mask, dW, db), N_out <= 16.
struct OutBwdArgs {
  int B = 0, H = 0, nout = 0, groups = 0, n_members = 1;
  int act16 = 0;             // X and dX are bf16 activations (BF16 mode)
  const void* X = nullptr;   // [groups][B][x_ld]  input of the output layer (post-ReLU)
  long long x_gs = 0, x_ld = 0;
  int x_by_member = 0;
  const float* G = nullptr;  // [groups][B][g_ld]  cotangent of the output
  long long g_gs = 0, g_ld = 0;
  const float* W = nullptr;  // [groups] weight rows, W [H][nout] at each group's base
  long long w_gs = 0;
  float* dW = nullptr;       // gradient rows: dW [H][nout] then db [nout] (nullptr: dX only)
  long long dw_gs = 0;
  void* dX = nullptr;        // [groups][B][dx_ld] (nullptr: input layer, no dX)
  long long dx_gs = 0, dx_ld = 0;
  float* dbx = nullptr;      // optional: column sums of dX = the bias gradient of the layer below
  long long dbx_gs = 0;
  // nout == 1 only: the cotangent G computed in the kernel from the network output q [groups][B]
  //   top 1: TD3 critic, dq = (2/B)(q - y), y = r + gamma (1 - d) min(tq1, tq2) (td3_critic_target
  //          + mse_loss_grads, algos.hpp:268-307); loss[grp] = sum_b (q - y)^2 / B (double)
  //   top 2: critic with a given TD target y [members][B] (SAC)
  //   top 3: TD3 policy loss through critic 1, dq = -1/B; loss[grp] = -sum_b q / B
  int top = 0;
  const float* q = nullptr;
  const float *r = nullptr, *d = nullptr, *tq = nullptr, *gamma = nullptr, *y = nullptr;
  double* loss = nullptr;
  const int* active = nullptr;
  int exact = 1;  // 1: reference summation order (FFMA32); 0: warp-parallel tree (TF32)
  int norm_rows = 0;  // top 1/2: rows of the MSE mean (0 = B; shared critic: n_global * B)
};
void launch_out_backward(const OutBwdArgs& a, cudaStream_t s);

// skinny shapes (output layers): forward N <= 16, dX K <= 16, dW N <= 16
void launch_fwd_skinny(const GemmArgs& g, cudaStream_t s);
void launch_dx_skinny(const GemmArgs& g, cudaStream_t s);
void launch_dw_skinny(const GemmArgs& g, cudaStream_t s);

// ------------------------------------------------------------------ elementwise launchers
struct Hyper;  // device per-member hyper floats

void launch_td3_step_begin(int n, double* delay_acc, const double* ratio, const uint8_t* mask,
                           int* fire, int64_t* t_pol, int64_t* t_c1, int64_t* t_c2,
                           uint64_t* steps, const uint64_t* streams, uint64_t seed,
                           uint64_t* noise_key, double* policy_loss,
                           cudaGraphConditionalHandle any_fire, int set_cond, int shared,
                           int ncrit, cudaStream_t s, int* guard = nullptr, double* hist = nullptr,
                           const uint64_t* hist_base = nullptr, int hist_slots = 0);
// in_sa / in_s2a / sa_pi are activation buffers: fp32, or bf16 when act16
void launch_pack_batch(int n, int B, int ds, int da, int lsa, const float* s, const float* a,
                       const float* r, const float* s2, const float* d, void* in_sa,
                       void* in_s2a, void* sa_pi, float* r_out, float* d_out, int act16,
                       cudaStream_t st, void* in_s = nullptr, int lsp = 0);
void launch_td_target(int n, int B, const float* r, const float* d, const float* q2n,
                      const float* gamma, float* y, cudaStream_t s);
// norm_rows: rows of the MSE mean (0 = B; the folded population when the critic is shared)
void launch_mse(int groups, int n, int B, const float* q, const float* y, float* dq, double* loss,
                cudaStream_t s, int norm_rows = 0);
void launch_td3_policy_loss(int n, int B, const float* q, const int* fire, double* loss,
                            float* gq, cudaStream_t s);
// Adam (pop_tensor.hpp:328-366) over a [groups][stride] arena, first P floats per group, with
// per-member lr, optional fire gate, and an optional fused Polyak update of a target arena
// (soft_update_members_inplace, :412-428) gated per member by polyak_gate (NULL = always).
void launch_adam(int groups, int n, size_t P, size_t stride, float* p, float* m, float* v,
                 const float* g, const int64_t* t, const float* corr1, const float* corr2,
                 const float* lr, const int* active, float* tgt, const float* tau_a,
                 const float* tau_b, const int* polyak_gate, __nv_bfloat16* p16,
                 __nv_bfloat16* t16, cudaStream_t s);
// bf16 copy of an fp32 arena (the BF16 mode's tensor-core weight operands)
void launch_to_bf16(const float* src, __nv_bfloat16* dst, size_t count, cudaStream_t s);
void launch_fill(float* p, size_t count, float v, cudaStream_t s);
void launch_copy_f64(double* dst, const double* src, size_t count, cudaStream_t s);
// column `col` of a [rows][ld] activation block := v (fp32, or bf16 when act16)
void launch_fill_col(void* p, long long rows, int ld, int col, float v, int act16, cudaStream_t s);
// bias gradient of a layer: dst[g][o] = sum_b G[g][b][o] in row order (groups gated by active)
void launch_colsum(int groups, int n, int B, int N, const void* G, long long g_gs, long long g_ld,
                   float* dst, long long dst_gs, const int* active, int act16, cudaStream_t s);

// ReLU mask bits of a hidden activation (TF32 mode, CUDA-core fallback layers):
// mask[g][r][w] bit j = (h[g][r][32w + j] > 0)
void launch_mask_bits(int groups, int B, int H, const float* h, long long h_gs, long long h_ld,
                      uint32_t* mask, long long m_gs, long long m_ld, const int* active, int n,
                      cudaStream_t s);
// TD3 target-policy smoothing noise for the fused tcgen05 epilogue (algos.hpp:252-262):
// eps[m][b][o] = clamp((T)normal(key_m, 2 (b da + o)) * sd_m, -clip_m, clip_m)
void launch_td3_target_noise(int n, int B, int da, const uint64_t* key, const float* sd,
                             const float* clip, float* eps, cudaStream_t s);

// SAC
void launch_sac_step_begin(int n, int64_t* t_pol, int64_t* t_c1, int64_t* t_c2, int64_t* t_alpha,
                           uint64_t* steps, const uint64_t* streams, uint64_t seed,
                           uint64_t* key_eps, uint64_t* key_eps_t, cudaStream_t s);
// split_policy_head + tanh_gaussian_logprob + squash (algos.hpp:534-616): head [n][B][2da] ->
// act into sa (cols ds..), x, th, ls (clamped), clamped flag, logp.
void launch_sac_head(int n, int B, int ds, int da, int lsa, const float* head, const uint64_t* key,
                     float bound, void* sa, float* x, float* th, float* ls, uint8_t* clamped,
                     float* eps, float* logp, int act16, cudaStream_t s);
void launch_sac_y(int n, int B, const float* r, const float* d, const float* q2n,
                  const float* logp2, const float* log_alpha, const float* gamma,
                  const float* rscale, float* y, cudaStream_t s);
void launch_sac_policy_top(int n, int B, const float* q2n, const float* logp,
                           const float* log_alpha, double* loss, float* gq2n, float* lw,
                           cudaStream_t s);
void launch_sac_head_grad(int n, int B, int da, const float* ga2n, const float* lw,
                          const float* x, const float* th, const float* ls,
                          const uint8_t* clamped, const float* eps, float bound, float* gh,
                          cudaStream_t s);
void launch_sac_alpha(int n, int B, const float* logp, const float* log_alpha_in,
                      const double* target_entropy, float* log_alpha, float* am, float* av,
                      const int64_t* t, const float* corr1, const float* corr2, const float* lr,
                      cudaStream_t s);

// action selection (act / sac_act, algos.hpp:895-942)
void launch_td3_act_noise(int n, long long per, float* a, const double* noise_std,
                          const uint64_t* streams, const uint64_t* steps, uint64_t seed,
                          float bound, cudaStream_t s);
void launch_sac_act(int n, int rows, int da, const float* head, const uint64_t* streams,
                    const uint64_t* steps, uint64_t seed, int deterministic, float bound, float* a,
                    cudaStream_t s);
void launch_pack_obs(long long rows_total, int ds, int ld, const float* obs, void* out, int act16,
                     cudaStream_t s);

// replay
void launch_replay_scatter(const float* rows, const uint64_t* dst_row, uint64_t count, int rw,
                           float* ring, cudaStream_t s);
void launch_replay_gather(int n, int B, int ds, int da, int lsa, int rw, const float* ring,
                          uint64_t cap, int shared, const uint64_t* sizes,
                          const uint64_t* streams, uint64_t seed, uint64_t draw_id,
                          void* in_sa, void* in_s2a, void* sa_pi, float* r_out, float* d_out,
                          int act16, cudaStream_t s, void* in_s = nullptr, int lsp = 0);

// PBT
void launch_pbt_plan(int n, const double* fitness, int cut, uint64_t key, uint64_t next,
                     uint64_t* order, uint64_t* replaced, uint64_t* donors, cudaStream_t s);
void launch_member_copy(float* arena, size_t stride, size_t P, const uint64_t* src,
                        const uint64_t* dst, int pairs, cudaStream_t s);
void launch_member_zero(float* arena, size_t stride, const uint64_t* dst, int pairs,
                        cudaStream_t s);

void launch_synth(uint64_t count, uint64_t n, uint64_t b, uint64_t ds, uint64_t da, uint64_t seed,
                  float* s, float* a, float* r, float* s2, float* d, cudaStream_t st);

void launch_libm_selftest(int fn, const float* in, float* out, uint64_t count, cudaStream_t s);

// init (init_pop_mlp, net_pop.hpp:69-100)
void launch_init_net(const NetShape& sh, float* arena, int n, uint64_t member_offset,
                     uint64_t seed, cudaStream_t s);

}  // namespace pbrl
