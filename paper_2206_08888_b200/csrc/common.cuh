// Shared device helpers for the population-update kernels (sm_100a).
//
// The whole library is compiled with --fmad=false: every float expression below rounds after
// each operation exactly like the reference CPU build (x86-64 SSE, no FMA contraction), which is
// what makes the FFMA32 check mode bit-exact.  Tensor-core kernels are unaffected by the flag.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pbrl {

// ------------------------------------------------------------------ counter RNG (rng.hpp:13-70)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// RngStream::of (rng.hpp:39-46)
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream,
                                                        uint64_t use, uint64_t step) {
  uint64_t k = mix64(seed);
  k = mix64(k ^ stream);
  k = mix64(k ^ use);
  return mix64(k ^ step);
}

__host__ __device__ __forceinline__ uint64_t rng_bits(uint64_t key, uint64_t c) {
  return mix64(key ^ mix64(c));
}

__device__ __forceinline__ double rng_uniform(uint64_t key, uint64_t c) {
  return static_cast<double>(rng_bits(key, c) >> 11) * 0x1.0p-53;
}

// Box-Muller in double (rng.hpp:66-70).  CUDA's double log/cos are within 1-2 ulp of glibc's;
// the draw is cast to float by every caller, so a difference survives only when the double lies
// within a few ulp of a float rounding boundary (~1e-8 per draw).
__device__ __forceinline__ double rng_normal_pair(uint64_t key, uint64_t c) {
  const double u1 = (static_cast<double>(rng_bits(key, c) >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = rng_uniform(key, c + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.28318530717958647692 * u2);
}

enum RngUse : uint64_t {
  kInitWeight = 1, kInitBias = 2, kExploreNoise = 3, kTargetNoise = 4, kSacEps = 5,
  kSacEpsTarget = 6, kSample = 7, kDonorChoice = 8, kHyperDraw = 9, kGeneric = 12
};

// ------------------------------------------------------------------ libm-exact tanhf
// The reference calls std::tanh(float) = glibc tanhf, the fdlibm algorithm (tanh via expm1f).
// This is an independent implementation of that published algorithm; it agrees with the host
// libm on all 2^32 inputs (checked exhaustively on the CPU, and on the device by
// tests/test_gpu_numerics.py).
__device__ __forceinline__ uint32_t fbits(float x) { return __float_as_uint(x); }
__device__ __forceinline__ float bitsf(uint32_t u) { return __uint_as_float(u); }

__device__ inline float fdlibm_expm1f(float x) {
  const float one = 1.0f, huge = 1.0e+30f, tiny = 1.0e-30f;
  const float o_threshold = 8.8721679688e+01f, ln2_hi = 6.9313812256e-01f,
              ln2_lo = 9.0580006145e-06f, invln2 = 1.4426950216e+00f;
  const float Q1 = -3.3333335072e-02f, Q2 = 1.5873016091e-03f, Q3 = -7.9365076090e-05f,
              Q4 = 4.0082177293e-06f, Q5 = -2.0109921195e-07f;
  float y, hi, lo, c = 0.0f, t, e, hxs, hfx, r1;
  int32_t k;
  uint32_t hx = fbits(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  if (hx >= 0x4195b844u) {
    if (hx >= 0x42b17218u) {
      if (hx > 0x7f800000u) return x + x;
      if (hx == 0x7f800000u) return xsb == 0 ? x : -1.0f;
      if (x > o_threshold) return huge * huge;
    }
    if (xsb) return tiny - one;
  }
  if (hx > 0x3eb17218u) {
    if (hx < 0x3F851592u) {
      if (!xsb) { hi = x - ln2_hi; lo = ln2_lo; k = 1; }
      else { hi = x + ln2_hi; lo = -ln2_lo; k = -1; }
    } else {
      k = static_cast<int32_t>(invln2 * x + (xsb == 0 ? 0.5f : -0.5f));
      t = static_cast<float>(k);
      hi = x - t * ln2_hi;
      lo = t * ln2_lo;
    }
    x = hi - lo;
    c = (hi - x) - lo;
  } else if (hx < 0x33000000u) {
    t = huge + x;
    return x - (t - (huge + x));
  } else {
    k = 0;
  }
  hfx = 0.5f * x;
  hxs = x * hfx;
  r1 = one + hxs * (Q1 + hxs * (Q2 + hxs * (Q3 + hxs * (Q4 + hxs * Q5))));
  t = 3.0f - r1 * hfx;
  e = hxs * ((r1 - t) / (6.0f - x * t));
  if (k == 0) return x - (x * e - hxs);
  e = (x * (e - c) - c);
  e -= hxs;
  if (k == -1) return 0.5f * (x - e) - 0.5f;
  if (k == 1) {
    if (x < -0.25f) return -2.0f * (e - (x + 0.5f));
    return one + 2.0f * (x - e);
  }
  if (k <= -2 || k > 56) {
    y = one - (e - x);
    y = bitsf(fbits(y) + (static_cast<uint32_t>(k) << 23));
    return y - one;
  }
  if (k < 23) {
    t = bitsf(0x3f800000u - (0x1000000u >> k));
    y = t - (e - x);
    y = bitsf(fbits(y) + (static_cast<uint32_t>(k) << 23));
  } else {
    t = bitsf(static_cast<uint32_t>(0x7f - k) << 23);
    y = x - (e + t);
    y += one;
    y = bitsf(fbits(y) + (static_cast<uint32_t>(k) << 23));
  }
  return y;
}

__device__ inline float libm_tanhf(float x) {
  const float one = 1.0f, two = 2.0f, tiny = 1.0e-30f;
  float t, z;
  const int32_t jx = static_cast<int32_t>(fbits(x));
  const int32_t ix = jx & 0x7fffffff;
  if (ix >= 0x7f800000) return (jx >= 0) ? one / x + one : one / x - one;
  if (ix < 0x41b00000) {
    if (ix == 0) return x;
    if (ix < 0x24000000) return x * (one + x);
    if (ix >= 0x3f800000) {
      t = fdlibm_expm1f(two * fabsf(x));
      z = one - two / (t + two);
    } else {
      t = fdlibm_expm1f(-two * fabsf(x));
      z = -t / (t + two);
    }
  } else {
    z = one - tiny;
  }
  return jx >= 0 ? z : -z;
}

// std::clamp / std::min / std::max comparison order (libstdc++)
__device__ __forceinline__ float clampf_ref(float v, float lo, float hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}
__device__ __forceinline__ float minf_ref(float a, float b) { return b < a ? b : a; }
__device__ __forceinline__ float maxf_ref(float a, float b) { return a < b ? b : a; }

}  // namespace pbrl
