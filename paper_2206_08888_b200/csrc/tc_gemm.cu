// tcgen05 grouped GEMM for sm_100a (TF32 operands in shared memory, fp32 accumulators in TMEM).
//
// One CTA computes one 128 x BN output tile of one group (member, or member x critic):
//   warp 0 / lane 0  : TMA producer -- 3-D tensor maps [group][rows][cols], 128B swizzle,
//                      hardware zero-fill past the logical extents (ragged K = 17 / 23 etc.)
//   warp 1           : TMEM allocation; lane 0 issues tcgen05.mma.cta_group::1.kind::tf32
//   warps 0-3        : epilogue -- tcgen05.ld 32x32b (one accumulator row per thread) and the
//                      same fused epilogues as the FFMA32 check mode (bias, ReLU, tanh*bound,
//                      TD3 target noise, ReLU-mask and tanh backward)
// Operand majorness is a template parameter: K-major (row-major [rows][K]) or MN-major
// ([K][rows], e.g. the weights W[in][out] as the B operand of a forward layer, or X^T / G for dW),
// so every product of the MLP forward and backward reads the tensors in their natural layout.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "pop_impl.cuh"
#include "tc_gemm.cuh"

namespace pbrl {

namespace {

constexpr int kBM = 128;        // UMMA M (cta_group::1)
constexpr int kBK = 32;         // fp32 K per stage = one 128-byte swizzle row
constexpr int kMaxStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Bounded wait: a phase that never completes (a pipeline bug) traps after ~20 s instead of
// hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t tries = 0;; ++tries) {
    uint32_t done;
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t"
        "}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (tries > (1u << 26)) asm volatile("trap;");
  }
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Shared-memory matrix descriptor (tcgen05 "version 1").  layout: 2 = SWIZZLE_128B (K-major
// operands: 8-row x 128 B atoms), 1 = SWIZZLE_128B_BASE32B (MN-major TF32 operands: 4-row x 128 B
// atoms with a 32-byte swizzle granule -- the only MN-major smem layout tf32 supports).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                          uint64_t layout) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
__host__ __device__ constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
}

}  // namespace

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(128, 2)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const TcArgs g) {
  constexpr uint32_t A_BYTES = kBM * kBK * 4;  // 16 KB
  constexpr uint32_t B_BYTES = BN * kBK * 4;
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment for the 128B swizzle atoms, by offsetting within the shared array so the
  // compiler keeps the shared address space (LDS/STS, not generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int kStages = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * STAGE);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tmem_full = empty + kMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  // fused output layer: bias [BN] and W_out [BN][nout] staged after the barriers
  float* fz_bias = reinterpret_cast<float*>(smem + kStages * STAGE + 256);
  float* fz_w = fz_bias + BN;

  const int grp = blockIdx.z;
  const int mem = grp % g.n_members;
  if (g.active && !g.active[mem]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
  const int nout = g.nout;
  if (nout > 0) {
    const float* bsrc = g.bias + grp * g.bias_gs;
    const float* wsrc = g.ow + grp * g.ow_gs;
    for (int e = threadIdx.x; e < BN; e += blockDim.x) fz_bias[e] = e < g.N ? bsrc[e] : 0.0f;
    for (int e = threadIdx.x; e < BN * nout; e += blockDim.x)
      fz_w[e] = e < g.N * nout ? wsrc[e] : 0.0f;
  }
  const int ga = g.a_by_member ? mem : grp;
  const int gb = g.b_by_member ? mem : grp;
  const int nk = (g.K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols<BN>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      if (kb >= kStages) mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      uint8_t* sb = sa + A_BYTES;
      mbar_expect_tx(&full[s], STAGE);
      const int k0 = kb * kBK;
      if (A_MN) {
#pragma unroll
        for (int j = 0; j < kBM / 32; ++j) tma_load_3d(&tmA, &full[s], sa + j * 4096, m0 + 32 * j, k0, ga);
      } else {
        tma_load_3d(&tmA, &full[s], sa, k0, m0, ga);
      }
      if (B_MN) {
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) tma_load_3d(&tmB, &full[s], sb + j * 4096, n0 + 32 * j, k0, gb);
      } else {
        tma_load_3d(&tmB, &full[s], sb, k0, n0, gb);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    // instruction descriptor: D f32, A/B tf32, majorness, N >> 3, M >> 4
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) |
                               ((B_MN ? 1u : 0u) << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
                               (static_cast<uint32_t>(kBM >> 4) << 24);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      mbar_wait(&full[s], (kb / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_base = smem_u32(smem + s * STAGE);
      const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < kBK / 8; ++kk) {
        // K-major: +32 B inside the 128 B swizzle row (SBO = 8 rows = 1 KB);
        // MN-major: +1 KB = the next 8 K-rows (SBO = 4 rows = 512 B, LBO = next 32-wide MN box)
        const uint64_t da = A_MN ? sdesc(a_base + kk * 1024, 4096, 512, 1)
                                 : sdesc(a_base + kk * 32, 16, 1024, 2);
        const uint64_t db = B_MN ? sdesc(b_base + kk * 1024, 4096, 512, 1)
                                 : sdesc(b_base + kk * 32, 16, 1024, 2);
        mma_tf32(tmem, da, db, idesc, (kb | kk) ? 1u : 0u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(tmem_full);
  }

  // ---------------- epilogue: all four warps.  tcgen05.ld gives thread `lane` of warp w the
  // accumulator row 32w + lane; each 32-column chunk is transposed through shared memory (the
  // pipeline stages are idle once every MMA has completed) so that lanes map to columns: bias /
  // aux loads and the C stores are then 128-byte coalesced and all issued before they are used.
  __syncwarp();
  mbar_wait(tmem_full, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float* T = reinterpret_cast<float*>(smem) + warp * (32 * 33);
  const int row0 = m0 + warp * 32;
  float* C = g.C + (g.c_by_member ? mem : grp) * g.c_gs;
  const float* bias = g.bias ? g.bias + grp * g.bias_gs : nullptr;
  const float* aux = g.aux ? g.aux + (g.aux_by_member ? mem : grp) * g.aux_gs : nullptr;
  const int epi = g.epi;
  constexpr int CW = BN < 32 ? BN : 32;  // chunk width
  if (nout > 0) {
    // hidden layer + output layer: thread = accumulator row; h = relu(acc + b) chunk by chunk,
    // y[o] += h[j] * W_out[j][o] in ascending j; h optionally stored (transposed, coalesced)
    float oacc[16];
#pragma unroll
    for (int o = 0; o < 16; ++o) oacc[o] = 0.0f;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += CW) {
      if (c0 >= g.N) break;
      float v[32];
      const uint32_t taddr =
          tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0);
      tmem_ld16(taddr, v);
      if (CW == 32) tmem_ld16(taddr + 16, v + 16);
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const float z = v[j] + fz_bias[c0 + j];
        const float h = (c0 + j < g.N && z > 0.0f) ? z : 0.0f;
        v[j] = h;
        const float* wr = fz_w + (c0 + j) * nout;
#pragma unroll
        for (int o = 0; o < 16; ++o)
          if (o < nout) oacc[o] = oacc[o] + h * wr[o];
      }
      if (g.store_hidden) {
#pragma unroll
        for (int j = 0; j < CW; ++j) T[lane * 33 + j] = v[j];
        __syncwarp();
        const int col = n0 + c0 + lane;
        if (lane < CW && col < g.N) {
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) {
            const int row = row0 + rr;
            if (row < g.M) C[static_cast<long long>(row) * g.c_rs + col] = T[rr * 33 + lane];
          }
        }
        __syncwarp();
      }
    }
    const int row = row0 + lane;
    if (row < g.M) {
      const float* ob = fz_w + g.N * nout;  // b_out follows W_out in the arena row
      const float* obg = g.ow + grp * g.ow_gs + static_cast<long long>(g.N) * nout;
      (void)ob;
      float* oC = g.oC + grp * g.oc_gs + static_cast<long long>(row) * g.oc_rs;
      const bool tanh_out = g.out_epi == EPI_BIAS_TANH || g.out_epi == EPI_BIAS_TANH_NOISE;
#pragma unroll
      for (int o = 0; o < 16; ++o) {
        if (o >= nout) break;
        const float y = oacc[o] + obg[o];
        float r = y;
        if (tanh_out) {
          const float t = libm_tanhf(y);
          if (g.oC2) g.oC2[grp * g.oc2_gs + static_cast<long long>(row) * g.oc2_rs + o] = t;
          r = (g.out_scale != 1.0f) ? t * g.out_scale : t;
          if (g.out_epi == EPI_BIAS_TANH_NOISE) {
            const uint64_t e = static_cast<uint64_t>(row) * nout + o;
            float eps = static_cast<float>(rng_normal_pair(g.noise_key[mem], 2 * e)) *
                        g.noise_sd[mem];
            eps = clampf_ref(eps, -g.noise_clip[mem], g.noise_clip[mem]);
            r = clampf_ref(r + eps, -g.bound, g.bound);
          }
        }
        oC[o] = r;
      }
    }
  } else
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += CW) {
    if (n0 + c0 >= g.N) break;
    {
      float v[32];
      const uint32_t taddr =
          tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0);
      tmem_ld16(taddr, v);
      if (CW == 32) tmem_ld16(taddr + 16, v + 16);
#pragma unroll
      for (int j = 0; j < CW; ++j) T[lane * 33 + j] = v[j];
    }
    __syncwarp();
    const int col = n0 + c0 + lane;
    const bool col_ok = lane < CW && col < g.N;
    if (epi == EPI_BIAS_TANH || epi == EPI_BIAS_TANH_NOISE) {
      // transcendental epilogue (policy output layer): row loop straight out of shared memory
      if (col_ok) {
        const float bv = bias ? bias[col] : 0.0f;
#pragma unroll 1
        for (int rr = 0; rr < 32; ++rr) {
          const int row = row0 + rr;
          if (row >= g.M) break;
          const float t = libm_tanhf(T[rr * 33 + lane] + bv);
          if (g.C2) g.C2[grp * g.c2_gs + static_cast<long long>(row) * g.c2_rs + col] = t;
          float y = (g.scale != 1.0f) ? t * g.scale : t;
          if (epi == EPI_BIAS_TANH_NOISE) {
            const uint64_t e = static_cast<uint64_t>(row) * g.N + col;
            float eps = static_cast<float>(rng_normal_pair(g.noise_key[mem], 2 * e)) *
                        g.noise_sd[mem];
            eps = clampf_ref(eps, -g.noise_clip[mem], g.noise_clip[mem]);
            y = clampf_ref(y + eps, -g.bound, g.bound);
          }
          C[static_cast<long long>(row) * g.c_rs + col] = y;
        }
      }
      __syncwarp();
      continue;
    }
    float x[32];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) x[rr] = T[rr * 33 + lane];
    __syncwarp();
    if (col_ok) {
      const float bv = bias ? bias[col] : 0.0f;
      if (epi == EPI_RELU_MASK || epi == EPI_TANH_GRAD) {
        float av[32];
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const int row = min(row0 + rr, g.M - 1);  // clamped: rows >= M are not stored
          av[rr] = aux[static_cast<long long>(row) * g.aux_rs + col];
        }
        if (epi == EPI_RELU_MASK) {
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) x[rr] = (av[rr] > 0.0f) ? x[rr] : 0.0f;
        } else {
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) {
            float y = x[rr];
            if (g.scale != 1.0f) y = y * g.scale;
            x[rr] = y * (1.0f - av[rr] * av[rr]);
          }
        }
      } else if (epi == EPI_BIAS) {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) x[rr] = x[rr] + bv;
      } else if (epi == EPI_BIAS_RELU) {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const float z = x[rr] + bv;
          x[rr] = z > 0.0f ? z : 0.0f;
        }
      }
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) {
        const int row = row0 + rr;
        if (row < g.M) C[static_cast<long long>(row) * g.c_rs + col] = x[rr];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_cols<BN>()));
  }
}

// ------------------------------------------------------------------ host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

void load_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) PBRL_THROW(PBRL_E_CUDA, "cuTensorMapEncodeTiled unavailable");
}

template <int BN>
size_t smem_bytes(int stages, int nout) {
  // stages (>= the 4 x 32 x 33 float epilogue transpose tiles), barriers, fused-output staging
  const size_t st = static_cast<size_t>(stages) * (kBM * kBK * 4 + BN * kBK * 4);
  return std::max<size_t>(st, 4 * 32 * 33 * 4) + 1024 + 256 +
         (nout > 0 ? static_cast<size_t>(BN) * (1 + nout) * 4 : 0);
}

template <int BN, bool A_MN, bool B_MN>
void launch_tpl(const CUtensorMap& a, const CUtensorMap& b, TcArgs g, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    CUDA_CHECK(cudaFuncSetAttribute(k_tc_gemm<BN, A_MN, B_MN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem_bytes<BN>(kMaxStages, 16))));
    attr_set = true;
  }
  // pipeline depth: enough to cover K, capped so two CTAs share an SM (TMEM 2 x 256 columns)
  const int nk = (g.K + kBK - 1) / kBK;
  g.stages = std::max(1, std::min(nk, BN >= 256 ? 2 : 3));
  dim3 grid((g.N + BN - 1) / BN, (g.M + kBM - 1) / kBM, g.groups);
  if (g.nout > 0 && (g.N > BN || g.nout > 16)) PBRL_THROW(PBRL_E_USAGE, "tc_gemm: bad fused output");
  k_tc_gemm<BN, A_MN, B_MN><<<grid, 128, smem_bytes<BN>(g.stages, g.nout), s>>>(a, b, g);
}

template <bool A_MN, bool B_MN>
void launch_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, const TcArgs& g,
               cudaStream_t s) {
  switch (bn) {
    case 16: if constexpr (!B_MN) { launch_tpl<16, A_MN, B_MN>(a, b, g, s); return; } break;
    case 64: launch_tpl<64, A_MN, B_MN>(a, b, g, s); return;
    case 128: launch_tpl<128, A_MN, B_MN>(a, b, g, s); return;
    case 256: launch_tpl<256, A_MN, B_MN>(a, b, g, s); return;
    default: break;
  }
  PBRL_THROW(PBRL_E_USAGE, "tc_gemm: unsupported tile width");
}
}  // namespace

CUtensorMap make_tmap(const float* base, uint64_t cols, uint64_t rows, uint64_t groups,
                      uint64_t row_stride_elems, uint64_t group_stride_elems, uint32_t box_cols,
                      uint32_t box_rows, bool mn_major) {
  load_encode();
  CUtensorMap m;
  cuuint64_t dims[3] = {cols, rows, groups};
  cuuint64_t strides[2] = {row_stride_elems * 4, group_stride_elems * 4};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) PBRL_THROW(PBRL_E_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

bool tma_ok(const float* base, uint64_t row_stride_elems, uint64_t group_stride_elems) {
  return (reinterpret_cast<uintptr_t>(base) % 16 == 0) && (row_stride_elems % 4 == 0) &&
         (group_stride_elems % 4 == 0);
}

int pick_bn(int N, bool b_mn) {
  if (N <= 16 && !b_mn) return 16;
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  return 256;
}

void launch_tc_gemm(const TcOperand& A, const TcOperand& B, bool a_mn, bool b_mn,
                    const TcArgs& g, cudaStream_t s) {
  const int bn = pick_bn(g.N, b_mn);
  // A: K-major tile = 32 (K) x 128 (M) box; MN-major = 32 (M) x 32 (K) boxes
  const CUtensorMap ta = a_mn ? make_tmap(A.p, A.cols, A.rows, A.groups, A.ld, A.gs, 32, 32, true)
                              : make_tmap(A.p, A.cols, A.rows, A.groups, A.ld, A.gs, 32, kBM, false);
  const CUtensorMap tb = b_mn ? make_tmap(B.p, B.cols, B.rows, B.groups, B.ld, B.gs, 32, 32, true)
                              : make_tmap(B.p, B.cols, B.rows, B.groups, B.ld, B.gs, 32, bn, false);
  if (a_mn && b_mn) launch_bn<true, true>(bn, ta, tb, g, s);
  else if (a_mn) launch_bn<true, false>(bn, ta, tb, g, s);
  else if (b_mn) launch_bn<false, true>(bn, ta, tb, g, s);
  else launch_bn<false, false>(bn, ta, tb, g, s);
}

}  // namespace pbrl
