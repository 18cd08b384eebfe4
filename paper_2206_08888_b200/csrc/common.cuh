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
//
// Attribution: the expm1f / tanhf / expf / log1pf algorithms and their polynomial constants
// below follow fdlibm as distributed in glibc (sysdeps/ieee754/flt-32), which carries this
// notice:
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this software is freely granted,
//   provided that this notice is preserved.
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

// ------------------------------------------------------------------ libm-exact expf / log1pf
// SAC calls std::exp / std::log1p on floats (algos.hpp:527, :555, :590, :763).  glibc's expf is
// the table-driven 2^(k/32) * poly(r) algorithm evaluated in double (x86-64 dispatches its FMA
// build); log1pf is the fdlibm algorithm.  Both implementations below agree with the host libm on
// all 2^32 inputs (exhaustive CPU check; device check in tests/test_gpu_numerics.py).
__constant__ uint64_t kExp2Tab32[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

// tab[i] = bits(2^(i/32)) - (i << 47), i.e. correctly rounded 2^(i/32) with the exponent
// contribution removed; generated with 60-digit decimal arithmetic.
__device__ inline float libm_expf(float x) {
  const double InvLn2N = 0x1.71547652b82fep+0 * 32, Shift = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32, C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32,
               C2 = 0x1.62e42ff0c52d6p-1 / 32;
  const double xd = static_cast<double>(x);
  const uint32_t abstop = (fbits(x) >> 20) & 0x7ff;
  if (abstop >= (fbits(88.0f) >> 20)) {
    if (fbits(x) == 0xff800000u) return 0.0f;
    if (abstop >= (0x7f800000u >> 20)) return x + x;
    if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
    if (x < -0x1.9fe368p6f) return 0.0f;
  }
  double kd = fma(InvLn2N, xd, Shift);
  const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
  kd -= Shift;
  const double r = fma(InvLn2N, xd, -kd);
  uint64_t t = kExp2Tab32[ki % 32];
  t += ki << (52 - 5);
  const double s = __longlong_as_double(static_cast<long long>(t));
  const double z = fma(C0, r, C1);
  const double r2 = r * r;
  double y = fma(C2, r, 1.0);
  y = fma(z, r2, y);
  y = y * s;
  return static_cast<float>(y);
}

__device__ inline float libm_log1pf(float x) {
  const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f, two25 = 3.355443200e+07f,
              Lp1 = 6.6666668653e-01f, Lp2 = 4.0000000596e-01f, Lp3 = 2.8571429849e-01f,
              Lp4 = 2.2222198546e-01f, Lp5 = 1.8183572590e-01f, Lp6 = 1.5313838422e-01f,
              Lp7 = 1.4798198640e-01f, zero = 0.0f;
  float hfsq, f = 0.0f, c = 0.0f, s, z, R, u;
  int32_t k, hu = 0;
  const int32_t hx = static_cast<int32_t>(fbits(x));
  const int32_t ax = hx & 0x7fffffff;
  k = 1;
  if (hx < 0x3ed413d7) {
    if (ax >= 0x3f800000) {
      if (x == -1.0f) return -two25 / zero;
      return (x - x) / (x - x);
    }
    if (ax < 0x31000000) {
      if (ax < 0x24800000) return x;
      return x - x * x * 0.5f;
    }
    if (hx > 0 || hx <= static_cast<int32_t>(0xbe95f61f)) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7f800000) return x + x;
  if (k != 0) {
    if (hx < 0x5a000000) {
      u = 1.0f + x;
      hu = static_cast<int32_t>(fbits(u));
      k = (hu >> 23) - 127;
      c = (k > 0) ? 1.0f - (u - x) : x - (u - 1.0f);
      c /= u;
    } else {
      u = x;
      hu = static_cast<int32_t>(fbits(u));
      k = (hu >> 23) - 127;
      c = 0;
    }
    hu &= 0x007fffff;
    if (hu < 0x3504f7) {
      u = bitsf(static_cast<uint32_t>(hu) | 0x3f800000u);
    } else {
      k += 1;
      u = bitsf(static_cast<uint32_t>(hu) | 0x3f000000u);
      hu = (0x00800000 - hu) >> 2;
    }
    f = u - 1.0f;
  }
  hfsq = 0.5f * f * f;
  if (hu == 0) {
    if (f == zero) {
      if (k == 0) return zero;
      c += k * ln2_lo;
      return k * ln2_hi + c;
    }
    R = hfsq * (1.0f - 0.66666666666666666f * f);
    if (k == 0) return f - R;
    return k * ln2_hi - ((R - (k * ln2_lo + c)) - f);
  }
  s = f / (2.0f + f);
  z = s * s;
  R = z * (Lp1 + z * (Lp2 + z * (Lp3 + z * (Lp4 + z * (Lp5 + z * (Lp6 + z * Lp7))))));
  if (k == 0) return f - (hfsq - s * (hfsq + R));
  return k * ln2_hi - ((hfsq - (s * (hfsq + R) + (k * ln2_lo + c))) - f);
}

// std::clamp / std::min / std::max comparison order (libstdc++)
__device__ __forceinline__ float clampf_ref(float v, float lo, float hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}
__device__ __forceinline__ float minf_ref(float a, float b) { return b < a ? b : a; }
__device__ __forceinline__ float maxf_ref(float a, float b) { return a < b ? b : a; }

}  // namespace pbrl
