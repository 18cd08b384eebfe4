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
#include <cstdlib>
#include <mutex>

#include "pop_impl.cuh"
#include "tc_gemm.cuh"

namespace pbrl {

namespace {

constexpr int kBM = 128;        // UMMA M (cta_group::1)
constexpr int kRowBytes = 128;  // K per stage = one 128-byte swizzle row (32 fp32 / 64 bf16)
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

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 consecutive accumulator columns of this thread's TMEM lane; asynchronous until
// tmem_ld_wait(v), which also orders every later use of v after the wait
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
        "=f"(v[14]), "=f"(v[15]), "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]),
        "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]),
        "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait(float* v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  asm volatile(""
               : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]),
                 "+f"(v[6]), "+f"(v[7]), "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]),
                 "+f"(v[12]), "+f"(v[13]), "+f"(v[14]), "+f"(v[15]));
  asm volatile(""
               : "+f"(v[16]), "+f"(v[17]), "+f"(v[18]), "+f"(v[19]), "+f"(v[20]), "+f"(v[21]),
                 "+f"(v[22]), "+f"(v[23]), "+f"(v[24]), "+f"(v[25]), "+f"(v[26]), "+f"(v[27]),
                 "+f"(v[28]), "+f"(v[29]), "+f"(v[30]), "+f"(v[31]));
}

// 16-column variants (half the registers per in-flight buffer)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
        "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait16(float* v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  asm volatile(""
               : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]),
                 "+f"(v[6]), "+f"(v[7]), "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]),
                 "+f"(v[12]), "+f"(v[13]), "+f"(v[14]), "+f"(v[15]));
}

template <int BN>
__host__ __device__ constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
}

}  // namespace

// Out-of-line transcendentals for the epilogues: every inlined copy of these long code paths
// is cold instruction memory the first time a launch reaches it (one L2 round trip per 128-byte
// line); a single shared copy is fetched once per SM and then stays in the instruction cache.
__device__ __noinline__ float epi_tanhf(float x) { return libm_tanhf(x); }
__device__ __noinline__ float epi_normal(uint64_t key, uint64_t c) {
  return static_cast<float>(rng_normal_pair(key, c));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant (column halves)
constexpr int kEpiThreads = kEpiWarps * 32;

__device__ __forceinline__ void epi_bar_sync() {  // the epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

__device__ __forceinline__ void quad_bar_sync(int q) {  // the two warps of lane quadrant q
  asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// 1-D bulk copy global -> shared, completion on an mbarrier (size and addresses 16 B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 32 rows x 128 B box with the 128-byte swizzle: 16-byte chunk j of row r lives at
// r * 128 + ((j ^ (r & 7)) << 4)
__device__ __forceinline__ uint32_t sw128(int r, int j) {
  return static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4));
}
// 32 rows x 64 B box (32 bf16) with the 64-byte swizzle: chunk j (0..3) of row r at
// r * 64 + ((j ^ ((r >> 1) & 3)) << 4)
__device__ __forceinline__ uint32_t sw64(int r, int j) {
  return static_cast<uint32_t>(r * 64 + ((j ^ ((r >> 1) & 3)) << 4));
}
// one cvt.rn.bf16x2.f32 (F2FP.BF16.F32.PACK_AB); lo in the low half, round-to-nearest-even
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// Optional phase timeline (TcArgs::trace, diagnostics only): per CTA kTraceSlots globaltimer
// stamps -- [0] entry, [1] after setup, per tile it < kTraceTiles: [2+6it+0] producer issues the
// first TMA, [+1] MMA sees the first stage, [+2] MMA commits the tile, [+3] epilogue sees the
// accumulator, [+4] epilogue done; [62] epilogue drained its TMA stores, [63] exit.
constexpr int kTraceSlots = 64, kTraceTiles = 10;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TC_TRACE(slot)                                                    \
  do {                                                                    \
    if (g.trace) g.trace[blockIdx.x * kTraceSlots + (slot)] = gtimer();   \
  } while (0)
#define TC_TRACE_TILE(it, k)                                              \
  do {                                                                    \
    if (g.trace && (it) < kTraceTiles) TC_TRACE(2 + 6 * (it) + (k));      \
  } while (0)

constexpr uint32_t kEpiBufBytes = 4096;                  // one 32 x 32 fp32 box
constexpr uint32_t kEpiWarpBytes = 2 * kEpiBufBytes;     // per warp: 2 boxes
constexpr uint32_t kEpiBytes = kEpiWarps * kEpiWarpBytes;

// Persistent, warp-specialised grouped GEMM.  Grid <= #SMs; CTA b walks tiles b, b+grid, ...
// (tile = group x M-tile x N-tile).  warp 0: TMA producer over a `stages`-deep smem ring;
// warp 1: TMEM allocation + single-thread tcgen05.mma issue into one of TWO accumulator buffers;
// warps 2-9: epilogue, two warps per TMEM lane quadrant (warp % 4) splitting the tile's columns
// -- each thread keeps its accumulator row (32-column tcgen05.ld, next chunk in flight while
// the current one is processed), adds the bias / applies ReLU / the ReLU' mask (bit masks),
// writes 128B-swizzled 32 x 32 boxes with 128-bit stores and TMA-stores them.  The
// double-buffered accumulator lets the epilogue of tile i run while tile i+1's MMAs run.
//
// EB = operand element bytes: 4 -> fp32 operands, kind::tf32 (8 K per MMA; MN-major operands as
// 32 x 32 boxes in the 128B_BASE32B layout); 2 -> bf16 operands, kind::f16 (16 K per MMA;
// MN-major operands as 64 x 64 boxes in the plain 128B swizzle).  A stage is one 128-byte K row
// of every operand row either way (32 fp32 or 64 bf16 K values).
template <int BN, bool A_MN, bool B_MN, int NO, int EB>
__global__ void __launch_bounds__(64 + kEpiThreads, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX,
              const TcArgs g) {
  constexpr int kBK = kRowBytes / EB;          // K elements per stage
  constexpr int MNBOX = EB == 4 ? 32 : 64;     // MN extent of one MN-major TMA box
  constexpr uint32_t MNBOX_BYTES = MNBOX * kBK * EB;  // 4 KB (fp32) / 8 KB (bf16)
  constexpr int KMMA = EB == 4 ? 8 : 16;       // K per tcgen05.mma
  constexpr uint32_t A_BYTES = kBM * kRowBytes;  // 16 KB
  constexpr uint32_t B_BYTES = BN * kRowBytes;
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t ACC_COLS = tmem_cols<BN>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment for the swizzle atoms, by offsetting within the shared array so the
  // compiler keeps the shared address space (LDS/STS, not generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = g.stages;
  uint8_t* epi_smem = smem + S * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint64_t* abar = tempty + 2;           // [epilogue warp] mask-box barriers
  uint64_t* sbar = abar + kEpiWarps;      // bias / output-layer staging
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sbar + 1);
  float* fz_bias = reinterpret_cast<float*>(epi_smem + kEpiBytes + 256);
  float* fz_w = fz_bias + BN;
  float* osum = fz_w + BN * (NO > 0 ? NO : 0);  // [2][4][32][NO] fused-output partial sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (g.M + kBM - 1) / kBM, n_tiles = (g.N + BN - 1) / BN;
  const int num_tiles = g.groups * m_tiles * n_tiles;
  const int nk = (g.K + kBK - 1) / kBK;
  // fused output width: compile-time for the common 1 / 6 / 12, runtime-guarded up to 16
  const int nout = (NO > 0 && NO < 16) ? NO : (NO == 0 ? 0 : g.nout);
  if (threadIdx.x == 0) TC_TRACE(0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    for (int a = 0; a < kEpiWarps; ++a) mbar_init(&abar[a], 1);
    mbar_init(sbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * ACC_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) {
    TC_TRACE(1);
    // early PDL trigger: the successor's launch and prologue overlap this whole grid.  The host
    // lets a successor prefetch weights before its own wait only if no kernel since the last
    // wait-then-trigger launch wrote weights (Pop::tc_prefetch_ok), because with early triggers
    // the successor can start while kernels several launches back are still running.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }

  auto decode = [&](int t, int& grp, int& m0, int& n0) {
    const int nt = t % n_tiles;
    const int r = t / n_tiles;
    m0 = (r % m_tiles) * kBM;
    grp = r / m_tiles;
    n0 = nt * BN;
  };
  auto active = [&](int grp) { return !g.active || g.active[grp % g.n_members]; };

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      // PDL: the weight operand B of the first tile's first stages is independent of the
      // predecessor kernel (b_prefetch: the host knows the predecessor wrote no weights), so it
      // is requested before griddepcontrol.wait; everything else waits for the predecessor.
      int npre = 0;
      if (g.b_prefetch && !g.active && static_cast<int>(blockIdx.x) < num_tiles) {
        int grp, m0, n0;
        decode(blockIdx.x, grp, m0, n0);
        const int gb = g.b_by_member ? grp % g.n_members : grp;
        npre = min(S, nk);
        for (int kb = 0; kb < npre; ++kb) {
          uint8_t* sb = smem + kb * STAGE + A_BYTES;
          mbar_expect_tx(&full[kb], STAGE);
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / MNBOX; ++j)
              tma_load_3d(&tmB, &full[kb], sb + j * MNBOX_BYTES, n0 + MNBOX * j, kb * kBK, gb);
          } else {
            tma_load_3d(&tmB, &full[kb], sb, kb * kBK, n0, gb);
          }
        }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int cnt = 0, pit = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int grp, m0, n0;
        decode(t, grp, m0, n0);
        if (!active(grp)) continue;
        TC_TRACE_TILE(pit, 0);
        ++pit;
        const int mem = grp % g.n_members;
        const int ga = g.a_by_member ? mem : grp;
        const int gb = g.b_by_member ? mem : grp;
        for (int kb = 0; kb < nk; ++kb, ++cnt) {
          const int s = cnt % S;
          if (cnt >= S) mbar_wait(&empty[s], ((cnt / S) - 1) & 1);
          uint8_t* sa = smem + s * STAGE;
          uint8_t* sb = sa + A_BYTES;
          const bool pre = cnt < npre;  // B already requested before the PDL wait
          if (!pre) mbar_expect_tx(&full[s], STAGE);
          const int k0 = kb * kBK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < kBM / MNBOX; ++j)
              tma_load_3d(&tmA, &full[s], sa + j * MNBOX_BYTES, m0 + MNBOX * j, k0, ga);
          } else {
            tma_load_3d(&tmA, &full[s], sa, k0, m0, ga);
          }
          if (pre) {
          } else if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / MNBOX; ++j)
              tma_load_3d(&tmB, &full[s], sb + j * MNBOX_BYTES, n0 + MNBOX * j, k0, gb);
          } else {
            tma_load_3d(&tmB, &full[s], sb, k0, n0, gb);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (instruction descriptor: D f32, A/B tf32, majorness, N, M)
    if (lane == 0) {
      constexpr uint32_t fmt = EB == 4 ? 2u : 1u;  // TF32 / BF16
      constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((A_MN ? 1u : 0u) << 15) |
                                 ((B_MN ? 1u : 0u) << 16) |
                                 (static_cast<uint32_t>(BN >> 3) << 17) |
                                 (static_cast<uint32_t>(kBM >> 4) << 24);
      int cnt = 0, it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int grp, m0, n0;
        decode(t, grp, m0, n0);
        if (!active(grp)) continue;
        const int acc = it & 1;
        if (it >= 2) mbar_wait(&tempty[acc], ((it >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dtmem = tmem + static_cast<uint32_t>(acc) * ACC_COLS;
        for (int kb = 0; kb < nk; ++kb, ++cnt) {
          const int s = cnt % S;
          mbar_wait(&full[s], (cnt / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (kb == 0) TC_TRACE_TILE(it, 1);
          const uint32_t a_base = smem_u32(smem + s * STAGE);
          const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < kBK / KMMA; ++kk) {
            // K-major: +32 B inside the 128 B swizzle row (SBO = 8 rows = 1 KB);
            // MN-major fp32: +1 KB = the next 8 K-rows (128B_BASE32B: SBO = 4 rows = 512 B,
            // LBO = next 32-wide MN box); MN-major bf16: +2 KB = the next 16 K-rows (128B
            // swizzle: SBO = 8 rows = 1 KB, LBO = next 64-wide MN box)
            const uint32_t mn_step = KMMA * kRowBytes;
            const uint64_t da =
                A_MN ? (EB == 4 ? sdesc(a_base + kk * mn_step, MNBOX_BYTES, 512, 1)
                                : sdesc(a_base + kk * mn_step, MNBOX_BYTES, 1024, 2))
                     : sdesc(a_base + kk * 32, 16, 1024, 2);
            const uint64_t db =
                B_MN ? (EB == 4 ? sdesc(b_base + kk * mn_step, MNBOX_BYTES, 512, 1)
                                : sdesc(b_base + kk * mn_step, MNBOX_BYTES, 1024, 2))
                     : sdesc(b_base + kk * 32, 16, 1024, 2);
            if (EB == 4) mma_tf32(dtmem, da, db, idesc, (kb | kk) ? 1u : 0u);
            else mma_bf16(dtmem, da, db, idesc, (kb | kk) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[acc]);
        TC_TRACE_TILE(it, 2);
        ++it;
      }
    }
  } else {
    // ---------------- epilogue warps: warp w reads TMEM lane quadrant q = w % 4 (tile rows
    // 32q..32q+31, one row per thread) and processes column half hf = (w - 2) / 4 of the tile
    const int ew = warp - 2;
    const int q = warp & 3;
    const int hf = ew >> 2;
    uint8_t* wbuf = epi_smem + ew * kEpiWarpBytes;  // this warp's two 4 KB boxes
    float* T = reinterpret_cast<float*>(wbuf);        // general path: 32 x 33 transpose tile
    uint64_t* wbar = abar + ew;
    const int epi = g.epi;
    const bool mask_bits = epi == EPI_RELU_MASK && g.mask_in != nullptr;
    const bool aux_boxes = epi == EPI_RELU_MASK && !mask_bits;
    const bool fast = g.c_tma &&
                      (epi == EPI_STORE || epi == EPI_BIAS || epi == EPI_BIAS_RELU ||
                       (epi == EPI_RELU_MASK && (g.aux_tma || mask_bits))) && BN >= 32;
    const int nbox = aux_boxes ? 1 : 2;  // C boxes in flight per warp (the other one: mask box)
    constexpr int MW = BN >= 32 ? BN / 32 : 1;  // mask words per row of a tile
    constexpr int CW = BN < 32 ? BN : 32;       // chunk width
    constexpr int NCH = BN / CW;                // chunks per tile
    constexpr int HCH = NCH >= 2 ? NCH / 2 : 1;  // chunks per column half
    const int cbeg = hf * HCH;
    const bool half_active = NCH >= 2 || hf == 0;
    const bool need_bias = g.bias && (epi == EPI_BIAS || epi == EPI_BIAS_RELU || nout > 0);
    constexpr int NA = NO > 0 ? NO : 1;
    int it = 0, nchunk = 0, nstage = 0;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // predecessor's outputs are visible
    // zero the staging area once: columns past N (never bulk-written) must read as 0
    for (int e = threadIdx.x - 64; e < BN * (1 + (nout > 0 ? nout : 0)); e += kEpiThreads)
      fz_bias[e] = 0.0f;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int grp, m0, n0;
      decode(t, grp, m0, n0);
      if (!active(grp)) continue;
      const int mem = grp % g.n_members;
      const int acc = it & 1;
      const int row0 = m0 + q * 32;
      const int row = row0 + lane;
      const int cg = g.c_by_member ? mem : grp;
      const int xg = g.aux_by_member ? mem : grp;
      // C element (r, c) of this group: fp32, or bf16 when c16
      char* Cb = static_cast<char*>(g.C) + cg * g.c_gs * (g.c16 ? 2 : 4);
      auto cstore = [&](long long idx, float x) {
        if (g.c16) reinterpret_cast<__nv_bfloat16*>(Cb)[idx] = __float2bfloat16_rn(x);
        else reinterpret_cast<float*>(Cb)[idx] = x;
      };
      const float* bias = g.bias ? g.bias + grp * g.bias_gs : nullptr;
      const float* aux = g.aux ? g.aux + xg * g.aux_gs : nullptr;
      if (nout > 0 && g.ow_tr) {
        // dX variant: gather the transposed output-layer weights (a few KB) into fz_w
        epi_bar_sync();
        const float* wsrc = g.ow + grp * g.ow_gs;
        const int nd = nout > 0 ? nout : 1;  // (NO = 0 instantiations: dead code)
        for (int e = threadIdx.x - 64; e < BN * nout; e += kEpiThreads) {
          const int j = e / nd, o = e - j * nd;
          fz_w[e] = j < g.N ? __ldg(wsrc + o * g.ow_ld + j) : 0.0f;
        }
        epi_bar_sync();
      } else if (need_bias) {
        // stage this tile's bias (and output-layer weights) once the previous tile is consumed:
        // one bulk copy issued before waiting for the accumulator, so it overlaps the MMAs
        epi_bar_sync();
        const float* bsrc = bias + n0;
        const float* wsrc = nout > 0 ? g.ow + grp * g.ow_gs : nullptr;
        const uint32_t bbytes = static_cast<uint32_t>(min(BN, g.N - n0)) * 4;
        const uint32_t wbytes = static_cast<uint32_t>(g.N * nout) * 4;
        const bool bulk = (reinterpret_cast<uintptr_t>(bsrc) % 16 == 0) && bbytes % 16 == 0 &&
                          (nout == 0 || ((reinterpret_cast<uintptr_t>(wsrc) % 16 == 0) &&
                                         wbytes % 16 == 0));
        if (bulk) {
          if (threadIdx.x == 64) {
            mbar_expect_tx(sbar, bbytes + (nout > 0 ? wbytes : 0));
            bulk_g2s(fz_bias, bsrc, bbytes, sbar);
            if (nout > 0) bulk_g2s(fz_w, wsrc, wbytes, sbar);
          }
          mbar_wait(sbar, nstage & 1);
          ++nstage;
        } else {
          for (int e = threadIdx.x - 64; e < BN; e += kEpiThreads)
            fz_bias[e] = (n0 + e < g.N) ? bias[n0 + e] : 0.0f;
          if (nout > 0)
            for (int e = threadIdx.x - 64; e < BN * nout; e += kEpiThreads)
              fz_w[e] = e < g.N * nout ? wsrc[e] : 0.0f;
          epi_bar_sync();
        }
      }
      // per-row operands of the epilogue, loaded before the accumulator wait (overlaps the MMAs)
      uint32_t mw[MW];
#pragma unroll
      for (int k = 0; k < MW; ++k) mw[k] = 0u;
      if (mask_bits && row < g.M) {
        const uint32_t* mp = g.mask_in + (g.mi_by_member ? mem : grp) * g.mi_gs +
                             static_cast<long long>(row) * g.mi_ld + (n0 >> 5);
        const int nw = min(MW, (g.N - n0 + 31) >> 5);
        if (MW % 4 == 0 && nw == MW && (g.mi_ld & 3) == 0 && ((n0 >> 5) & 3) == 0) {
#pragma unroll
          for (int k = 0; k < MW; k += 4) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(mp + k));
            mw[k] = u.x;
            mw[k + 1] = u.y;
            mw[k + 2] = u.z;
            mw[k + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int k = 0; k < MW; ++k) mw[k] = k < nw ? __ldg(mp + k) : 0u;
        }
      }
      float ob[NA], ep[NA];
      if (nout > 0 && hf == 0) {
        const float* obg = g.ow + grp * g.ow_gs + static_cast<long long>(g.N) * nout;
        const bool noisy = g.out_epi == EPI_BIAS_TANH_NOISE && g.noise_eps && row < g.M;
        const float* eg =
            noisy ? g.noise_eps + grp * g.ne_gs + static_cast<long long>(row) * g.ne_rs : nullptr;
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          ob[o] = (o < nout && !g.ow_tr) ? __ldg(obg + o) : 0.0f;
          ep[o] = (noisy && o < nout) ? __ldg(eg + o) : 0.0f;
        }
      }
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (threadIdx.x == 64) TC_TRACE_TILE(it, 3);
      const uint32_t tacc =
          tmem + static_cast<uint32_t>(acc) * ACC_COLS + (static_cast<uint32_t>(q * 32) << 16);

      // one 32-column chunk of this thread's row -> swizzled box -> TMA store
      auto store_box = [&](const float* v, int c0) {
        uint8_t* box = wbuf + (nbox == 2 ? (nchunk & 1) : 0) * kEpiBufBytes;
        if (lane == 0 && nchunk >= nbox) {  // box reused nbox chunks later
          if (nbox == 2) tma_store_wait_read<1>();
          else tma_store_wait_read<0>();
        }
        __syncwarp();
        if (g.c16) {  // 32 rows x 64 B bf16 box, 64-byte swizzle
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 w4 = make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]),
                                  pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                                  pack_bf16x2(v[8 * j + 4], v[8 * j + 5]),
                                  pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
            *reinterpret_cast<uint4*>(box + sw64(lane, j)) = w4;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 w4 = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            *reinterpret_cast<float4*>(box + sw128(lane, j)) = w4;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) tma_store_3d(&tmC, box, n0 + c0, row0, cg);
        ++nchunk;
      };
      // bit j of the returned word = (v[j] > 0): the ReLU mask of one 32-column chunk
      auto mask_word = [&](const float* v) {
        uint32_t bits = 0u;
#pragma unroll
        for (int j = 0; j < 32; ++j) bits |= (v[j] > 0.0f ? 1u : 0u) << j;
        return bits;
      };
      uint32_t* mrow = (g.mask_out && row < g.M)
                           ? g.mask_out + grp * g.mo_gs + static_cast<long long>(row) * g.mo_ld
                           : nullptr;

      if (nout > 0) {
        // hidden layer + fused output layer: y[o] += relu(acc + b)[j] * W_out[j][o], j ascending
        // within each column half; the halves are added in order (deterministic)
        float oacc[NA];
#pragma unroll
        for (int o = 0; o < NA; ++o) oacc[o] = 0.0f;
        float v[2][32];
        if (half_active) tmem_ld32(tacc + static_cast<uint32_t>(cbeg * CW), v[0]);
#pragma unroll 2
        for (int ci = 0; ci < HCH; ++ci) {
          const int c0 = (cbeg + ci) * CW;
          float* cur = v[ci & 1];
          if (half_active) {
            tmem_ld_wait(cur);
            if (ci + 1 < HCH && c0 + CW < g.N)
              tmem_ld32(tacc + static_cast<uint32_t>(c0 + CW), v[(ci + 1) & 1]);
          }
          if (!half_active || c0 >= g.N) continue;
          if (mask_bits) {  // dX variant: relu'(h_below) from the mask bits
            uint32_t bits = 0u;
#pragma unroll
            for (int k = 0; k < MW; ++k)
              if (k == cbeg + ci) bits = mw[k];
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              const float h = ((bits >> j) & 1u) ? cur[j] : 0.0f;
              cur[j] = h;
              const float* wr = fz_w + (c0 + j) * nout;
#pragma unroll
              for (int o = 0; o < NA; ++o) {
                if (NO == 16 && o >= nout) break;
                oacc[o] = oacc[o] + h * wr[o];
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              const float z = cur[j] + fz_bias[c0 + j];
              const float h = (c0 + j < g.N && z > 0.0f) ? z : 0.0f;
              cur[j] = h;
              const float* wr = fz_w + (c0 + j) * nout;
#pragma unroll
              for (int o = 0; o < NA; ++o) {
                if (NO == 16 && o >= nout) break;
                oacc[o] = oacc[o] + h * wr[o];
              }
            }
          }
          if (g.store_hidden) {
            store_box(cur, c0);
            if (mrow && CW == 32) mrow[c0 >> 5] = mask_word(cur);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (threadIdx.x == 64) TC_TRACE_TILE(it, 4);
        // half 1 hands its partial sums to half 0 (double-buffered by tile parity)
        float* os = osum + ((acc * 4 + q) * 32 + lane) * NA;
        if (hf == 1) {
#pragma unroll
          for (int o = 0; o < NA; ++o) os[o] = oacc[o];
        }
        quad_bar_sync(q);
        if (threadIdx.x == 64) TC_TRACE_TILE(it, 5);
        if (hf == 0 && row < g.M) {
          const long long obase = grp * g.oc_gs + static_cast<long long>(row) * g.oc_rs;
          const bool tanh_out = g.out_epi == EPI_BIAS_TANH || g.out_epi == EPI_BIAS_TANH_NOISE;
          const float* arow = (g.out_epi == EPI_TANH_GRAD && aux)
                                  ? aux + static_cast<long long>(row) * g.aux_rs : nullptr;
#pragma unroll
          for (int o = 0; o < NA; ++o) {
            if (o >= nout) break;
            const float y = (oacc[o] + os[o]) + ob[o];
            float r = y;
            if (arow) {  // tanh backward of the policy head (activation_backward, tanh)
              const float gy = (g.scale != 1.0f) ? y * g.scale : y;
              const float th = arow[o];
              r = gy * (1.0f - th * th);
            } else if (tanh_out) {
              const float th = epi_tanhf(y);
              if (g.oC2) g.oC2[grp * g.oc2_gs + static_cast<long long>(row) * g.oc2_rs + o] = th;
              r = (g.out_scale != 1.0f) ? th * g.out_scale : th;
              if (g.out_epi == EPI_BIAS_TANH_NOISE) {
                float eps;
                if (g.noise_eps) {
                  eps = ep[o];
                } else {
                  const uint64_t e = static_cast<uint64_t>(row) * nout + o;
                  eps = epi_normal(g.noise_key[mem], 2 * e) * g.noise_sd[mem];
                  eps = clampf_ref(eps, -g.noise_clip[mem], g.noise_clip[mem]);
                }
                r = clampf_ref(r + eps, -g.bound, g.bound);
              }
            }
            if (g.oc16) static_cast<__nv_bfloat16*>(g.oC)[obase + o] = __float2bfloat16_rn(r);
            else static_cast<float*>(g.oC)[obase + o] = r;
          }
        }
        ++it;
        continue;
      }

      if (fast) {
        float v[2][32];
        if (half_active) tmem_ld32(tacc + static_cast<uint32_t>(cbeg * 32), v[0]);
#pragma unroll 2
        for (int ci = 0; ci < HCH; ++ci) {
          const int c0 = (cbeg + ci) * 32;
          float* cur = v[ci & 1];
          if (half_active) {
            tmem_ld_wait(cur);
            if (ci + 1 < HCH && n0 + c0 + 32 < g.N)
              tmem_ld32(tacc + static_cast<uint32_t>(c0 + 32), v[(ci + 1) & 1]);
          }
          if (!half_active || n0 + c0 >= g.N) continue;
          if (aux_boxes && lane == 0) {
            mbar_expect_tx(wbar, kEpiBufBytes);
            tma_load_3d(&tmX, wbar, wbuf + kEpiBufBytes, n0 + c0, row0, xg);
          }
          if (epi == EPI_BIAS) {
#pragma unroll
            for (int j = 0; j < 32; ++j) cur[j] = cur[j] + fz_bias[c0 + j];
          } else if (epi == EPI_BIAS_RELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float z = cur[j] + fz_bias[c0 + j];
              cur[j] = z > 0.0f ? z : 0.0f;
            }
          } else if (mask_bits) {
            uint32_t bits = 0u;
#pragma unroll
            for (int k = 0; k < MW; ++k)  // register select (no local-memory indexing)
              if (k == cbeg + ci) bits = mw[k];
#pragma unroll
            for (int j = 0; j < 32; ++j) cur[j] = ((bits >> j) & 1u) ? cur[j] : 0.0f;
          } else if (aux_boxes) {
            // the k-th use of this warp's mask box completes phase k
            mbar_wait(wbar, nchunk & 1);
            const uint8_t* xbox = wbuf + kEpiBufBytes;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 m4 = *reinterpret_cast<const float4*>(xbox + sw128(lane, j));
              cur[4 * j] = m4.x > 0.0f ? cur[4 * j] : 0.0f;
              cur[4 * j + 1] = m4.y > 0.0f ? cur[4 * j + 1] : 0.0f;
              cur[4 * j + 2] = m4.z > 0.0f ? cur[4 * j + 2] : 0.0f;
              cur[4 * j + 3] = m4.w > 0.0f ? cur[4 * j + 3] : 0.0f;
            }
            __syncwarp();  // box consumed before the next chunk's load overwrites it
          }
          store_box(cur, c0);
          if (mrow && epi == EPI_BIAS_RELU) mrow[(n0 + c0) >> 5] = mask_word(cur);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (threadIdx.x == 64) TC_TRACE_TILE(it, 4);
        ++it;
        continue;
      }

      // ---- general path (tanh / noise / tanh-grad epilogues, narrow tiles): transpose the
      // chunk through shared memory so lanes map to columns, coalesced loads and stores
      if (half_active) {
#pragma unroll 1
        for (int ci = 0; ci < HCH; ++ci) {
          const int c0 = (cbeg + ci) * CW;
          if (n0 + c0 >= g.N) break;
          {
            float v[32];
            tmem_ld32(tacc + static_cast<uint32_t>(c0), v);
            tmem_ld_wait(v);
#pragma unroll
            for (int j = 0; j < CW; ++j) T[lane * 33 + j] = v[j];
          }
          __syncwarp();
          const int col = n0 + c0 + lane;
          const bool col_ok = lane < CW && col < g.N;
          const bool need_aux = epi == EPI_RELU_MASK || epi == EPI_TANH_GRAD;
          if (col_ok) {
            const float bv = bias ? bias[col] : 0.0f;
#pragma unroll 1
            for (int r8 = 0; r8 < 32; r8 += 8) {
              // the 8 aux loads of this row group are issued together (independent round trips)
              float av[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int rw = row0 + r8 + u;
                av[u] = (need_aux && rw < g.M)
                            ? __ldg(aux + static_cast<long long>(rw) * g.aux_rs + col)
                            : 0.0f;
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int rr = r8 + u;
                const int rw = row0 + rr;
                if (rw >= g.M) break;
                float x = T[rr * 33 + lane];
                switch (epi) {
                  case EPI_BIAS: x = x + bv; break;
                  case EPI_BIAS_RELU: {
                    const float z = x + bv;
                    x = z > 0.0f ? z : 0.0f;
                    break;
                  }
                  case EPI_BIAS_TANH:
                  case EPI_BIAS_TANH_NOISE: {
                    const float th = epi_tanhf(x + bv);
                    if (g.C2) g.C2[grp * g.c2_gs + static_cast<long long>(rw) * g.c2_rs + col] = th;
                    x = (g.scale != 1.0f) ? th * g.scale : th;
                    if (epi == EPI_BIAS_TANH_NOISE) {
                      const uint64_t e = static_cast<uint64_t>(rw) * g.N + col;
                      float eps = epi_normal(g.noise_key[mem], 2 * e) * g.noise_sd[mem];
                      eps = clampf_ref(eps, -g.noise_clip[mem], g.noise_clip[mem]);
                      x = clampf_ref(x + eps, -g.bound, g.bound);
                    }
                    break;
                  }
                  case EPI_RELU_MASK:
                    if (!(av[u] > 0.0f)) x = 0.0f;
                    break;
                  case EPI_TANH_GRAD: {
                    if (g.scale != 1.0f) x = x * g.scale;
                    const float th = av[u];
                    x = x * (1.0f - th * th);
                    break;
                  }
                  default: break;
                }
                cstore(static_cast<long long>(rw) * g.c_rs + col, x);
              }
            }
          }
          __syncwarp();
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (threadIdx.x == 64) TC_TRACE_TILE(it, 4);
      ++it;
    }
    if (lane == 0) tma_store_wait_all();
    if (threadIdx.x == 64) TC_TRACE(62);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(2 * ACC_COLS));
  }
  if (threadIdx.x == 0) TC_TRACE(63);
}

// ------------------------------------------------------------------ fused two-layer forward
// k_mlp_fwd2 (BF16 mode): one persistent launch evaluates hidden layer 1, hidden layer 2 and the
// output layer of an MLP population.  Per 128-row tile of a group:
//   producer : X tile (one 64-wide K chunk: in <= 64) and W1 into the layer-1 buffers, then W2
//              through a ring of 64-row K chunks (3 deep: most of the next tile's W2 lands
//              while the current tile's layer-2 epilogue runs)
//   MMA      : acc1 (TMEM cols 0..255) = X W1; after the E1 warps have turned acc1 into h1 in
//              shared memory, acc2 (cols 256..511) = h1 W2 with A read from that shared-memory
//              copy (K-major, 128B swizzle) -- h1 never round-trips through HBM
//   E1 warps : relu(acc1 + b1) -> bf16 K-major operand tile (+ HBM copy and mask bits when kept)
//   E2 warps : relu(acc2 + b2) -> output layer on CUDA cores (+ h2 to HBM when kept, stored
//              straight from registers: the W2 ring holds the shared memory a staging box would)
// E1 and E2 are separate warp groups: E1 of tile i+1 runs while E2 drains tile i (acc1 and acc2
// are disjoint TMEM columns; E1 only waits until the layer-2 MMA of tile i has read sH1), so
// the per-tile period is E1 + the layer-2 MMA tail instead of E1 + MMA + E2.
constexpr uint32_t kF2H1 = 65536;  // h1 operand: 4 K chunks x (128 rows x 128 B)
constexpr uint32_t kF2X = kBM * kRowBytes;   // 16 KB
constexpr uint32_t kF2W = 256 * kRowBytes;   // 32 KB: 64 K rows x 256 N, as 4 boxes of 64 x 64
constexpr int kF2Threads = 64 + 2 * kEpiThreads;  // TMA, MMA, 8 E1 warps, 8 E2 warps
// W2 ring depth (2 when the output layer's shared memory is large)
template <int NO>
__host__ __device__ constexpr int f2_ring() { return NO <= 6 ? 3 : 2; }

template <int NO>
__host__ __device__ constexpr size_t fwd2_smem() {
  return kF2H1 + kF2X + kF2W + f2_ring<NO>() * kF2W + 256 + 3 * 256 * 4 + 256 * NO * 4 +
         2 * kBM * NO * 4 + 1024;
}

__device__ __forceinline__ void e2_bar_sync() {  // the E2 warps only
  asm volatile("bar.sync 6, %0;" ::"n"(kEpiThreads) : "memory");
}

// NO = 1, 6, 12: exact output width; NO = 16: any width <= 16 (runtime g.nout)
template <int NO>
__global__ void __launch_bounds__(kF2Threads, 1)
    k_mlp_fwd2(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
               const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmH1,
               const Fwd2Args g) {
  constexpr bool kRt = NO == 16;
  constexpr bool kEarly = NO <= 6;  // output bias / noise loaded before E2 (register budget)
  constexpr int R = f2_ring<NO>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sH1 = smem;
  uint8_t* sX = sH1 + kF2H1;
  uint8_t* sW1 = sX + kF2X;
  uint8_t* sW2 = sW1 + kF2W;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW2 + R * kF2W);
  uint64_t* l1full = bars;
  uint64_t* l1empty = bars + 1;
  uint64_t* w2full = bars + 2;   // [R <= 3]
  uint64_t* w2empty = bars + 5;  // [R <= 3]
  uint64_t* acc1full = bars + 8;
  uint64_t* acc2full = bars + 9;
  uint64_t* acc2empty = bars + 10;
  uint64_t* sbar1 = bars + 11;   // [2] b1 staging (E1, double-buffered: the next tile's b1 is
                                 // fetched while this tile's E1 runs)
  uint64_t* h1kc = bars + 13;    // [4]: K chunk kc of h1 written (4 warps of its column half)
  uint64_t* sbar2 = bars + 17;   // b2 / W_out staging (E2)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);
  float* fz_b1 = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [2][256]
  float* fz_b2 = fz_b1 + 512;
  float* fz_w = fz_b2 + 256;
  float* osum = fz_w + 256 * NO;  // [2][4][32][NO]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (g.M + kBM - 1) / kBM;
  const int num_tiles = g.groups * m_tiles;
  const int nk2 = g.H1 / 64;
  // layer-2 K chunk order: the two column halves of E1 are written concurrently, so the MMAs
  // alternate halves (0, 2, 1, 3 for H1 = 256) and start after the first chunk of each half
  auto korder = [&](int j) { return (j & 1) * (nk2 / 2) + (j >> 1); };
  const int nout = kRt ? g.nout : NO;
  if (threadIdx.x == 0) TC_TRACE(0);

  if (threadIdx.x == 0) {
    mbar_init(l1full, 1);
    mbar_init(l1empty, 1);
    for (int s = 0; s < R; ++s) {
      mbar_init(&w2full[s], 1);
      mbar_init(&w2empty[s], 1);
    }
    mbar_init(acc1full, 1);
    for (int k = 0; k < 4; ++k) mbar_init(&h1kc[k], kEpiWarps / 2);
    mbar_init(acc2full, 1);
    mbar_init(acc2empty, kEpiWarps);
    mbar_init(&sbar1[0], 1);
    mbar_init(&sbar1[1], 1);
    mbar_init(sbar2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW2)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) {
    TC_TRACE(1);
    // early PDL trigger: the successor's launch and prologue overlap this whole grid.  The host
    // lets a successor prefetch weights before its own wait only if no kernel since the last
    // wait-then-trigger launch wrote weights (Pop::tc_prefetch_ok), because with early triggers
    // the successor can start while kernels several launches back are still running.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  auto active = [&](int grp) { return !g.active || g.active[grp % g.n_members]; };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int it = 0, cnt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int grp = t / m_tiles, m0 = (t % m_tiles) * kBM;
        if (!active(grp)) continue;
        const int mem = grp % g.n_members;
        if (it > 0) mbar_wait(l1empty, (it - 1) & 1);
        mbar_expect_tx(l1full, kF2X + kF2W);
        tma_load_3d(&tmX, l1full, sX, 0, m0, g.x_by_member ? mem : grp);
#pragma unroll
        for (int j = 0; j < 4; ++j) tma_load_3d(&tmW1, l1full, sW1 + j * 8192, 64 * j, 0, grp);
        for (int kc = 0; kc < nk2; ++kc, ++cnt) {
          const int s = cnt % R;
          if (cnt >= R) mbar_wait(&w2empty[s], (cnt / R - 1) & 1);
          mbar_expect_tx(&w2full[s], kF2W);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            tma_load_3d(&tmW2, &w2full[s], sW2 + s * kF2W + j * 8192, 64 * j, 64 * korder(kc),
                        grp);
        }
        ++it;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer (bf16 x bf16 -> f32, A K-major, B MN-major)
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                 (static_cast<uint32_t>(256 >> 3) << 17) |
                                 (static_cast<uint32_t>(kBM >> 4) << 24);
      int it = 0, cnt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        if (!active(t / m_tiles)) continue;
        // acc1 is free: every h1 chunk of the previous tile was waited on below, i.e. E1 has
        // read acc1 out
        mbar_wait(l1full, it & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(tmem, sdesc(smem_u32(sX) + kk * 32, 16, 1024, 2),
                   sdesc(smem_u32(sW1) + kk * 2048, 8192, 1024, 2), idesc, kk ? 1u : 0u);
        mma_commit(l1empty);
        mma_commit(acc1full);
        if (it > 0) mbar_wait(acc2empty, (it - 1) & 1);
        for (int j = 0; j < nk2; ++j, ++cnt) {
          const int kc = korder(j), s = cnt % R;
          mbar_wait(&h1kc[kc], it & 1);  // this K chunk of h1 is in shared memory
          mbar_wait(&w2full[s], (cnt / R) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16(tmem + 256, sdesc(smem_u32(sH1) + kc * 16384 + kk * 32, 16, 1024, 2),
                     sdesc(smem_u32(sW2) + s * kF2W + kk * 2048, 8192, 1024, 2), idesc,
                     (j | kk) ? 1u : 0u);
          mma_commit(&w2empty[s]);
        }
        mma_commit(acc2full);  // also: the layer-2 MMAs have read sH1
        TC_TRACE_TILE(it, 5);  // every h1 chunk of this tile was waited on and issued
        ++it;
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ---------------- E1: warp w reads TMEM lane quadrant q = w % 4, column half hf of acc1
    const int ew = warp - 2, q = warp & 3, hf = ew >> 2;
    const int hc1 = g.H1 / 64;  // 32-column chunks of h1 per half
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int grp = t / m_tiles, m0 = (t % m_tiles) * kBM;
      if (!active(grp)) continue;
      const int row0 = m0 + q * 32, row = row0 + lane;
      const int r = q * 32 + lane;  // row inside the tile
      if (threadIdx.x == 64) TC_TRACE_TILE(it, 0);
      // every E1 warp is done with the previous tile (its b1 buffer is free, its h1 stores have
      // read sH1 out); prefetch the next active tile's b1 into that buffer
      if (lane == 0) tma_store_wait_read<0>();
      __syncwarp();
      epi_bar_sync();
      if (threadIdx.x == 64) {
        auto stage_b1 = [&](int tt, int buf) {
          mbar_expect_tx(&sbar1[buf], g.H1 * 4);
          bulk_g2s(fz_b1 + buf * 256, g.b1 + (tt / m_tiles) * g.p_gs, g.H1 * 4, &sbar1[buf]);
        };
        if (it == 0) stage_b1(t, 0);
        for (int tn = t + gridDim.x; tn < num_tiles; tn += gridDim.x) {
          if (active(tn / m_tiles)) {
            stage_b1(tn, (it + 1) & 1);
            break;
          }
        }
      }
      const float* b1s = fz_b1 + (it & 1) * 256;
      mbar_wait(&sbar1[it & 1], (it >> 1) & 1);
      mbar_wait(acc1full, it & 1);
      if (it > 0) mbar_wait(acc2full, (it - 1) & 1);  // the layer-2 MMAs have read sH1
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (threadIdx.x == 64) TC_TRACE_TILE(it, 1);
      const uint32_t tacc = tmem + (static_cast<uint32_t>(q * 32) << 16);
      uint32_t* mrow = (g.m1 && row < g.M)
                           ? g.m1 + grp * g.m1_gs + static_cast<long long>(row) * g.m1_ld
                           : nullptr;
      // 16-column sub-chunks in register pairs (va, vb): the next sub-chunk's tcgen05.ld is in
      // flight while the current one is processed (static register names, 96-register budget)
      // (mask bits only when a mask is kept: two instantiations of the sub-chunk body)
      uint32_t bits = 0u;
      auto e1_body = [&](float* cur, int c0, auto keep_mask) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float z = cur[j] + b1s[c0 + j];
          cur[j] = z > 0.0f ? z : 0.0f;
          if constexpr (decltype(keep_mask)::value) bits |= (z > 0.0f ? 1u : 0u) << ((c0 & 16) + j);
        }
        uint8_t* rowp = sH1 + (c0 >> 6) * 16384 + r * 128;
        const int j0 = (c0 & 63) >> 3;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint4 w4 = make_uint4(pack_bf16x2(cur[8 * u], cur[8 * u + 1]),
                                      pack_bf16x2(cur[8 * u + 2], cur[8 * u + 3]),
                                      pack_bf16x2(cur[8 * u + 4], cur[8 * u + 5]),
                                      pack_bf16x2(cur[8 * u + 6], cur[8 * u + 7]));
          *reinterpret_cast<uint4*>(rowp + (((j0 + u) ^ (r & 7)) << 4)) = w4;
        }
        if constexpr (decltype(keep_mask)::value) {
          if (c0 & 16) {
            mrow[c0 >> 5] = bits;
            bits = 0u;
          }
        }
      };
      auto e1_sub = [&](float* cur, int c0) {
        if (mrow) e1_body(cur, c0, std::true_type{});
        else e1_body(cur, c0, std::false_type{});
      };
      float va[16], vb[16];
      const int cb = hf * hc1 * 32;  // a multiple of 64: every 4 sub-chunks are one K chunk
      const int ns = hc1 * 2;
      tmem_ld16(tacc + static_cast<uint32_t>(cb), va);
#pragma unroll 1
      for (int si = 0; si < ns; si += 2) {
        tmem_ld_wait16(va);
        tmem_ld16(tacc + static_cast<uint32_t>(cb + (si + 1) * 16), vb);
        e1_sub(va, cb + si * 16);
        tmem_ld_wait16(vb);
        if (si + 2 < ns) tmem_ld16(tacc + static_cast<uint32_t>(cb + (si + 2) * 16), va);
        e1_sub(vb, cb + (si + 1) * 16);
        if ((si & 3) == 2) {
          // K chunk kc complete in this warp's rows: visible to the MMA (async proxy), to HBM
          const int kc = (cb + si * 16) >> 6;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (g.H1g) tma_store_3d(&tmH1, sH1 + kc * 16384 + q * 4096, kc * 64, row0, grp);
            mbar_arrive(&h1kc[kc]);
          }
        }
      }
      if (threadIdx.x == 64) TC_TRACE_TILE(it, 2);
      ++it;
    }
    if (lane == 0) tma_store_wait_all();
  } else {
    // ---------------- E2: warp w reads TMEM lane quadrant q = w % 4, column half hf of acc2
    const int ew = warp - 2 - kEpiWarps, q = warp & 3, hf = ew >> 2;
    constexpr int NA = NO;
    const int hc2 = (g.H2 + 63) / 64;  // 32-column chunks of h2 per half
    const int tid2 = threadIdx.x - 64 - kEpiThreads;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int grp = t / m_tiles, m0 = (t % m_tiles) * kBM;
      if (!active(grp)) continue;
      const int mem = grp % g.n_members;
      const int row0 = m0 + q * 32, row = row0 + lane;
      // ---- stage b2, W_out of this group once every E2 warp is done with the previous tile's
      e2_bar_sync();
      if (tid2 == 0) {
        const uint32_t by2 = g.H2 * 4, byw = g.H2 * nout * 4;
        mbar_expect_tx(sbar2, by2 + byw);
        bulk_g2s(fz_b2, g.b2 + grp * g.p_gs, by2, sbar2);
        bulk_g2s(fz_w, g.ow + grp * g.p_gs, byw, sbar2);
      }
      const float* obg = g.ow + grp * g.p_gs + static_cast<long long>(g.H2) * nout;
      const bool noisy = g.out_epi == EPI_BIAS_TANH_NOISE && g.noise_eps && row < g.M;
      const float* eg =
          noisy ? g.noise_eps + grp * g.ne_gs + static_cast<long long>(row) * g.ne_rs : nullptr;
      float ob[NA], ep[NA];
      if (kEarly && hf == 0) {  // narrow outputs: output bias and noise in flight during E2
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          ob[o] = __ldg(obg + o);
          ep[o] = noisy ? __ldg(eg + o) : 0.0f;
        }
      }
      mbar_wait(sbar2, it & 1);
      mbar_wait(acc2full, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (tid2 == 0) TC_TRACE_TILE(it, 3);
      const uint32_t tacc = tmem + 256u + (static_cast<uint32_t>(q * 32) << 16);
      uint32_t* mrow = (g.m2 && row < g.M)
                           ? g.m2 + grp * g.m2_gs + static_cast<long long>(row) * g.m2_ld
                           : nullptr;
      // output-layer partial dot products (fused multiply-add: BF16 mode only); a single output
      // keeps 4 interleaved partial sums so the FMA chain is not one dependent sequence
      float oacc[NA], o1p[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int o = 0; o < NA; ++o) oacc[o] = 0.0f;
      // 16-column sub-chunks, double-buffered like E1; kept h2 rows go to HBM as 2 x 16 B
      __nv_bfloat16* h2row = (g.H2g && row < g.M)
                                 ? static_cast<__nv_bfloat16*>(g.H2g) + grp * g.h2_gs +
                                       static_cast<long long>(row) * g.h2_ld
                                 : nullptr;
      uint32_t bits = 0u;
      auto e2_body = [&](float* cur, int c0, auto keep_mask) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float z = cur[j] + fz_b2[c0 + j];
          const float h = z > 0.0f ? z : 0.0f;
          cur[j] = h;
          if constexpr (decltype(keep_mask)::value) bits |= (z > 0.0f ? 1u : 0u) << ((c0 & 16) + j);
          const float* wr = fz_w + (c0 + j) * nout;
          if constexpr (NO == 1) {
            if (j & 3) o1p[(j & 3) - 1] = __fmaf_rn(h, wr[0], o1p[(j & 3) - 1]);
            else oacc[0] = __fmaf_rn(h, wr[0], oacc[0]);
          } else {
#pragma unroll
            for (int o = 0; o < NA; ++o) {
              if (kRt && o >= nout) break;
              oacc[o] = __fmaf_rn(h, wr[o], oacc[o]);
            }
          }
        }
        if (h2row) {
#pragma unroll
          for (int u = 0; u < 2; ++u)
            *reinterpret_cast<uint4*>(h2row + c0 + 8 * u) =
                make_uint4(pack_bf16x2(cur[8 * u], cur[8 * u + 1]),
                           pack_bf16x2(cur[8 * u + 2], cur[8 * u + 3]),
                           pack_bf16x2(cur[8 * u + 4], cur[8 * u + 5]),
                           pack_bf16x2(cur[8 * u + 6], cur[8 * u + 7]));
        }
        if constexpr (decltype(keep_mask)::value) {
          if (c0 & 16) {
            mrow[c0 >> 5] = bits;
            bits = 0u;
          }
        }
      };
      auto e2_sub = [&](float* cur, int c0) {
        if (mrow) e2_body(cur, c0, std::true_type{});
        else e2_body(cur, c0, std::false_type{});
      };
      const int cb = hf * hc2 * 32;
      const int nc = max(0, min(hc2, (g.H2 - cb + 31) / 32));  // this half's chunks < H2
      const int ns = 2 * nc;                                   // 16-column sub-chunks
      float va[16], vb[16];
      if (ns > 0) tmem_ld16(tacc + static_cast<uint32_t>(cb), va);
#pragma unroll 1
      for (int si = 0; si < ns; si += 2) {
        tmem_ld_wait16(va);
        tmem_ld16(tacc + static_cast<uint32_t>(cb + (si + 1) * 16), vb);
        e2_sub(va, cb + si * 16);
        tmem_ld_wait16(vb);
        if (si + 2 < ns) tmem_ld16(tacc + static_cast<uint32_t>(cb + (si + 2) * 16), va);
        e2_sub(vb, cb + (si + 1) * 16);
      }
      if constexpr (NO == 1) oacc[0] = (oacc[0] + o1p[0]) + (o1p[1] + o1p[2]);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc2empty);
      if (tid2 == 0) TC_TRACE_TILE(it, 4);
      // half 1 hands its partial sums to half 0 (double-buffered by tile parity)
      float* os = osum + (((it & 1) * 4 + q) * 32 + lane) * NA;
      if (hf == 1) {
#pragma unroll
        for (int o = 0; o < NA; ++o) os[o] = oacc[o];
      }
      quad_bar_sync(q);
      if (hf == 0 && row < g.M) {
        if (!kEarly) {
#pragma unroll
          for (int o = 0; o < NA; ++o) {
            if (o >= nout) break;
            ob[o] = __ldg(obg + o);
            ep[o] = noisy ? __ldg(eg + o) : 0.0f;
          }
        }
        const long long obase = grp * g.oc_gs + static_cast<long long>(row) * g.oc_rs;
        const bool tanh_out = g.out_epi == EPI_BIAS_TANH || g.out_epi == EPI_BIAS_TANH_NOISE;
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          if (o >= nout) break;
          const float y = (oacc[o] + os[o]) + ob[o];
          float rr = y;
          if (tanh_out) {
            const float th = epi_tanhf(y);
            if (g.oC2) g.oC2[grp * g.oc2_gs + static_cast<long long>(row) * g.oc2_rs + o] = th;
            rr = (g.out_scale != 1.0f) ? th * g.out_scale : th;
            if (g.out_epi == EPI_BIAS_TANH_NOISE) {
              float eps;
              if (g.noise_eps) {
                eps = ep[o];
              } else {
                const uint64_t e = static_cast<uint64_t>(row) * nout + o;
                eps = epi_normal(g.noise_key[mem], 2 * e) * g.noise_sd[mem];
                eps = clampf_ref(eps, -g.noise_clip[mem], g.noise_clip[mem]);
              }
              rr = clampf_ref(rr + eps, -g.bound, g.bound);
            }
          }
          if (g.oc16) static_cast<__nv_bfloat16*>(g.oC)[obase + o] = __float2bfloat16_rn(rr);
          else static_cast<float*>(g.oC)[obase + o] = rr;
        }
      }
      ++it;
    }
    if (tid2 == 0) TC_TRACE(62);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
  if (threadIdx.x == 0) TC_TRACE(63);
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

template <int BN, int NO>
constexpr size_t smem_bytes(int stages) {
  // stage ring, epilogue boxes, barriers, bias / output-layer staging, fused-output partial
  // sums, 1 KB alignment slack
  return static_cast<size_t>(stages) * (kBM + BN) * kRowBytes + kEpiBytes + 256 + 1024 +
         static_cast<size_t>(BN) * (1 + NO) * 4 + static_cast<size_t>(2 * kBM) * NO * 4;
}
constexpr size_t kMaxSmem = 232448;  // 227 KB opt-in per block (sm_100)

template <int BN, int NO>
constexpr int max_stages() {
  int s = BN >= 256 ? 3 : kMaxStages;
  while (s > 1 && smem_bytes<BN, NO>(s) > kMaxSmem) --s;
  return s;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <int BN, bool A_MN, bool B_MN, int NO, int EB>
void launch_tpl(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                const CUtensorMap& x, TcArgs g, cudaStream_t s) {
  constexpr int smax = max_stages<BN, NO>();
  static_assert(smem_bytes<BN, NO>(smax) <= kMaxSmem, "tc_gemm: shared memory budget");
  static bool attr_set = false;
  if (!attr_set) {
    CUDA_CHECK(cudaFuncSetAttribute(k_tc_gemm<BN, A_MN, B_MN, NO, EB>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem_bytes<BN, NO>(smax))));
    attr_set = true;
  }
  // persistent: one CTA per SM (TMEM holds two BN-column accumulators)
  const int kbk = kRowBytes / EB;
  const int nk = (g.K + kbk - 1) / kbk;
  g.stages = std::max(1, std::min(nk, smax));
  const int tiles = g.groups * ((g.M + kBM - 1) / kBM) * ((g.N + BN - 1) / BN);
  if (g.nout > 0 && (g.N > BN || g.nout > 16)) PBRL_THROW(PBRL_E_USAGE, "tc_gemm: bad fused output");
  const int ctas = std::min(tiles, g.max_ctas > 0 ? std::min(g.max_ctas, num_sms()) : num_sms());
  launch_k(k_tc_gemm<BN, A_MN, B_MN, NO, EB>, ctas, 64 + kEpiThreads,
           smem_bytes<BN, NO>(g.stages), s, a, b, c, x, g);
}

template <bool A_MN, bool B_MN, int EB>
void launch_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
               const CUtensorMap& x, const TcArgs& g, cudaStream_t s) {
  if (g.nout > 0) {  // fused output layer: forward (K-major A, MN-major B) or dX (K / K)
    if constexpr (!A_MN && B_MN) {
      if (bn == 256) {
        switch (g.nout) {
          case 1: launch_tpl<256, false, true, 1, EB>(a, b, c, x, g, s); return;
          case 6: launch_tpl<256, false, true, 6, EB>(a, b, c, x, g, s); return;
          case 12: launch_tpl<256, false, true, 12, EB>(a, b, c, x, g, s); return;
          default: launch_tpl<256, false, true, 16, EB>(a, b, c, x, g, s); return;
        }
      }
    }
    if constexpr (!A_MN && !B_MN) {
      if (bn == 256) {
        if (g.nout == 6) launch_tpl<256, false, false, 6, EB>(a, b, c, x, g, s);
        else launch_tpl<256, false, false, 16, EB>(a, b, c, x, g, s);
        return;
      }
    }
    PBRL_THROW(PBRL_E_USAGE, "tc_gemm: fused output layer needs the 256-wide forward tile");
  }
  switch (bn) {
    case 16: if constexpr (!B_MN) { launch_tpl<16, A_MN, B_MN, 0, EB>(a, b, c, x, g, s); return; } break;
    case 64: launch_tpl<64, A_MN, B_MN, 0, EB>(a, b, c, x, g, s); return;
    case 128: launch_tpl<128, A_MN, B_MN, 0, EB>(a, b, c, x, g, s); return;
    case 256: launch_tpl<256, A_MN, B_MN, 0, EB>(a, b, c, x, g, s); return;
    default: break;
  }
  PBRL_THROW(PBRL_E_USAGE, "tc_gemm: unsupported tile width");
}
}  // namespace

int num_sms_host() { return num_sms(); }

// 3-D tensor map over [groups][rows][cols] elements of eb bytes (fp32 or bf16); swizzle: 128B
// for K-major operand tiles (and 32 x 32 fp32 epilogue boxes), 128B_ATOM_32B for MN-major fp32
// operand boxes, 64B for 32 x 32 bf16 epilogue boxes
enum TmapSwz { SWZ_128 = 0, SWZ_128_ATOM32 = 1, SWZ_64 = 2 };
CUtensorMap make_tmap(const void* base, int eb, uint64_t cols, uint64_t rows, uint64_t groups,
                      uint64_t row_stride_elems, uint64_t group_stride_elems, uint32_t box_cols,
                      uint32_t box_rows, int swz) {
  load_encode();
  CUtensorMap m;
  cuuint64_t dims[3] = {cols, rows, groups};
  cuuint64_t strides[2] = {row_stride_elems * eb, group_stride_elems * eb};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = swz == SWZ_128_ATOM32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                : swz == SWZ_64      ? CU_TENSOR_MAP_SWIZZLE_64B
                                                     : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = g_encode(&m, eb == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                        3, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) PBRL_THROW(PBRL_E_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

bool tma_ok(const void* base, uint64_t row_stride_elems, uint64_t group_stride_elems, int eb) {
  return (reinterpret_cast<uintptr_t>(base) % 16 == 0) && ((row_stride_elems * eb) % 16 == 0) &&
         ((group_stride_elems * eb) % 16 == 0);
}

// Tile width: the persistent grid walks `tiles` tiles on #SM CTAs, so a launch lasts
// ceil(tiles / #SM) tile-times -- with a few hundred tiles the last partial wave is a large share
// (80 members x 2 row tiles = 160 tiles on 148 SMs: 2 waves for 1.08 waves of work).  Narrower
// tiles make the waves finer at the cost of re-reading A per N tile and a per-tile epilogue
// start-up; the model below (cost ~ waves x (BN + 48)) picks the cheapest legal width.
// PBRL_TC_BN=<64|128|256> pins it (diagnostics).
int pick_bn(const TcArgs& g, bool b_mn) {
  const int N = g.N;
  if (N <= 16 && !b_mn) return 16;
  if (g.nout > 0) return 256;  // the fused output layer needs the whole hidden row
  static const int pin = std::getenv("PBRL_TC_BN") ? std::atoi(std::getenv("PBRL_TC_BN")) : 0;
  if (pin == 64 || pin == 128 || pin == 256) return pin;
  const int m_tiles = (g.M + kBM - 1) / kBM;
  const int sms = g.max_ctas > 0 ? std::min(g.max_ctas, num_sms()) : num_sms();
  int best = 256;
  double best_cost = 1e30;
  for (int bn : {64, 128, 256}) {
    const long long tiles = static_cast<long long>(g.groups) * m_tiles * ((N + bn - 1) / bn);
    const double waves = static_cast<double>((tiles + sms - 1) / sms);
    // per-tile cost: its columns plus a fixed ~160-column equivalent (pipeline fill, epilogue
    // setup; measured: every config-D product is faster at 256 than at 128 with 1.7x the waves)
    const double cost = waves * (std::min(bn, ((N + 31) / 32) * 32) + 160);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = bn;
    }
    if (bn >= N) break;  // wider tiles only add padding
  }
  return best;
}

// Diagnostics: with PBRL_TC_TRACE set, every launch (in issue / capture order) gets its own
// slice of a device trace buffer; pbrl_debug_tc_trace copies it out with per-launch metadata.
namespace {
constexpr int kTraceLaunches = 96, kTraceCtas = 160;
unsigned long long* g_trace = nullptr;
int g_trace_n = 0;
TcTraceMeta g_trace_meta[kTraceLaunches];
}  // namespace

void tc_trace_init() {  // outside stream capture (population construction)
  if (g_trace || std::getenv("PBRL_TC_TRACE") == nullptr) return;
  const size_t bytes = static_cast<size_t>(kTraceLaunches) * kTraceCtas * kTraceSlots * 8;
  CUDA_CHECK(cudaMalloc(&g_trace, bytes));
  CUDA_CHECK(cudaMemset(g_trace, 0, bytes));
}

int tc_trace_dump(unsigned long long* host, TcTraceMeta* meta, int max_launches) {
  if (!g_trace) return 0;
  const int n = std::min(std::min(g_trace_n, kTraceLaunches), max_launches);
  CUDA_CHECK(cudaDeviceSynchronize());
  CUDA_CHECK(cudaMemcpy(host, g_trace, static_cast<size_t>(n) * kTraceCtas * kTraceSlots * 8,
                        cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) meta[i] = g_trace_meta[i];
  return n;
}

void launch_tc_gemm(const TcOperand& A, const TcOperand& B, bool a_mn, bool b_mn,
                    const TcArgs& g0, cudaStream_t s) {
  TcArgs g = g0;
  const int bn = pick_bn(g, b_mn);
  if (g_trace && g_trace_n < kTraceLaunches) {
    g.trace = g_trace + static_cast<size_t>(g_trace_n) * kTraceCtas * kTraceSlots;
    g_trace_meta[g_trace_n] = TcTraceMeta{bn, a_mn ? 1 : 0, b_mn ? 1 : 0, g.nout, g.M, g.N, g.K,
                                          g.groups, g.epi, 0};
    ++g_trace_n;
  }
  // operand boxes: K-major = one 128-byte K row x (128 | BN) rows; MN-major = 32 x 32 fp32
  // (128B_ATOM_32B) or 64 x 64 bf16 (128B) boxes
  const int eb = g.eb;
  const uint32_t kbk = 128 / eb, mnb = eb == 4 ? 32 : 64;
  const int mn_swz = eb == 4 ? SWZ_128_ATOM32 : SWZ_128;
  const CUtensorMap ta =
      a_mn ? make_tmap(A.p, eb, A.cols, A.rows, A.groups, A.ld, A.gs, mnb, kbk, mn_swz)
           : make_tmap(A.p, eb, A.cols, A.rows, A.groups, A.ld, A.gs, kbk, kBM, SWZ_128);
  const CUtensorMap tb =
      b_mn ? make_tmap(B.p, eb, B.cols, B.rows, B.groups, B.ld, B.gs, mnb, kbk, mn_swz)
           : make_tmap(B.p, eb, B.cols, B.rows, B.groups, B.ld, B.gs, kbk, bn, SWZ_128);
  // epilogue boxes: C stores as 32 x 32 boxes (fp32: 128B swizzle, bf16: 64B swizzle) and
  // fp32 ReLU'-mask loads
  CUtensorMap tc{}, tx{};
  const int ceb = g.c16 ? 2 : 4;
  g.c_tma = bn >= 32 && !g.c_by_member && g.C && tma_ok(g.C, g.c_rs, g.c_gs, ceb) ? 1 : 0;
  if (g.c_tma)
    tc = make_tmap(g.C, ceb, g.N, g.M, g.groups, g.c_rs, g.c_gs, 32, 32, g.c16 ? SWZ_64 : SWZ_128);
  g.aux_tma = bn >= 32 && g.aux && tma_ok(g.aux, g.aux_rs, g.aux_gs) ? 1 : 0;
  if (g.aux_tma)
    tx = make_tmap(g.aux, 4, g.N, g.M, g.aux_by_member ? g.n_members : g.groups, g.aux_rs,
                   g.aux_gs, 32, 32, SWZ_128);
  if (g.nout > 0 && g.store_hidden && !g.c_tma)
    PBRL_THROW(PBRL_E_USAGE, "tc_gemm: fused output layer needs a TMA-legal hidden buffer");
  if (g.nout > 0 && g.ow_tr && !g.mask_in)
    PBRL_THROW(PBRL_E_USAGE, "tc_gemm: fused dX output needs the ReLU mask bits");
  if (eb == 2 && g.epi == EPI_RELU_MASK && !g.mask_in)
    PBRL_THROW(PBRL_E_USAGE, "tc_gemm: bf16 ReLU' epilogues need the mask bits");
  if (eb == 4) {
    if (a_mn && b_mn) launch_bn<true, true, 4>(bn, ta, tb, tc, tx, g, s);
    else if (a_mn) launch_bn<true, false, 4>(bn, ta, tb, tc, tx, g, s);
    else if (b_mn) launch_bn<false, true, 4>(bn, ta, tb, tc, tx, g, s);
    else launch_bn<false, false, 4>(bn, ta, tb, tc, tx, g, s);
  } else {
    if (a_mn && b_mn) launch_bn<true, true, 2>(bn, ta, tb, tc, tx, g, s);
    else if (a_mn) launch_bn<true, false, 2>(bn, ta, tb, tc, tx, g, s);
    else if (b_mn) launch_bn<false, true, 2>(bn, ta, tb, tc, tx, g, s);
    else launch_bn<false, false, 2>(bn, ta, tb, tc, tx, g, s);
  }
}

bool mlp_fwd2_ok(const Fwd2Args& a) {
  auto al16 = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  return a.in >= 1 && a.in <= 64 && a.H1 % 128 == 0 && a.H1 <= 256 && a.H2 % 32 == 0 &&
         a.H2 >= 32 && a.H2 <= 256 && a.nout >= 1 && a.nout <= 16 && a.x_ld % 8 == 0 &&
         a.x_gs % 8 == 0 && a.w_gs % 8 == 0 && a.p_gs % 4 == 0 && al16(a.X) && al16(a.W1) &&
         al16(a.W2) && al16(a.b1) && al16(a.b2) && al16(a.ow) &&
         (!a.H1g || (al16(a.H1g) && a.h1_ld % 8 == 0 && a.h1_gs % 8 == 0)) &&
         (!a.H2g || (al16(a.H2g) && a.h2_ld % 8 == 0 && a.h2_gs % 8 == 0));
}

namespace {
template <int NO>
void launch_fwd2_tpl(const Fwd2Args& a, cudaStream_t s) {
  constexpr size_t smem = fwd2_smem<NO>();
  static_assert(smem <= kMaxSmem, "fwd2: shared memory budget");
  static bool attr_set = false;
  if (!attr_set) {
    CUDA_CHECK(cudaFuncSetAttribute(k_mlp_fwd2<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    attr_set = true;
  }
  const CUtensorMap tx = make_tmap(a.X, 2, a.in, a.M, a.x_by_member ? a.n_members : a.groups,
                                   a.x_ld, a.x_gs, 64, kBM, SWZ_128);
  const CUtensorMap tw1 = make_tmap(a.W1, 2, a.H1, a.in, a.groups, a.H1, a.w_gs, 64, 64, SWZ_128);
  const CUtensorMap tw2 = make_tmap(a.W2, 2, a.H2, a.H1, a.groups, a.H2, a.w_gs, 64, 64, SWZ_128);
  CUtensorMap th1{};
  if (a.H1g) th1 = make_tmap(a.H1g, 2, a.H1, a.M, a.groups, a.h1_ld, a.h1_gs, 64, 32, SWZ_128);
  const int tiles = a.groups * ((a.M + kBM - 1) / kBM);
  const int ctas = std::min(tiles, a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms());
  launch_k(k_mlp_fwd2<NO>, ctas, kF2Threads, smem, s, tx, tw1, tw2, th1, a);
}
}  // namespace

void launch_mlp_fwd2(const Fwd2Args& a0, cudaStream_t s) {
  Fwd2Args a = a0;
  if (!mlp_fwd2_ok(a)) PBRL_THROW(PBRL_E_USAGE, "fused forward: unsupported shape / alignment");
  if (g_trace && g_trace_n < kTraceLaunches) {
    a.trace = g_trace + static_cast<size_t>(g_trace_n) * kTraceCtas * kTraceSlots;
    // epi 99 marks the fused two-layer forward in the trace metadata (tools/tc_trace.py)
    g_trace_meta[g_trace_n] = TcTraceMeta{256, 0, 1, a.nout, a.M, a.H2, a.H1, a.groups, 99, 0};
    ++g_trace_n;
  }
  switch (a.nout) {
    case 1: launch_fwd2_tpl<1>(a, s); return;
    case 6: launch_fwd2_tpl<6>(a, s); return;
    case 12: launch_fwd2_tpl<12>(a, s); return;
    default: launch_fwd2_tpl<16>(a, s); return;  // any width <= 16
  }
}

}  // namespace pbrl
