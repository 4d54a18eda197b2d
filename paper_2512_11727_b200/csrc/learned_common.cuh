// Shared device helpers of the learned backend: counter-based RNG, bf16
// conversion and the deterministic expf.  Each one mirrors the function of
// the same name in oracle/ecco_oracle.c so the FFMA path is bit-exact.
#pragma once
#include <stdint.h>

__device__ __forceinline__ void philox4x32(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                           uint32_t k0, uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

__device__ __forceinline__ uint16_t f32_to_bf16(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

__device__ __forceinline__ float usym(uint32_t w) {
  return __fsub_rn(__fmul_rn((float)(w >> 8), 0x1p-23f), 1.0f);
}

// orc_expf: ln2 range reduction + degree-6 Horner, all explicitly rounded.
__device__ __forceinline__ float ecco_expf(float x) {
  if (x < -87.0f) return 0.0f;
  if (x > 88.0f) x = 88.0f;
  const float k = rintf(__fmul_rn(x, 0x1.715476p+0f));
  float r = __fmaf_rn(k, -0x1.62e400p-1f, x);
  r = __fmaf_rn(k, -0x1.7f7d1cp-20f, r);
  float q = 0x1.6c16c2p-10f;
  q = __fmaf_rn(q, r, 0x1.111112p-7f);
  q = __fmaf_rn(q, r, 0x1.555556p-5f);
  q = __fmaf_rn(q, r, 0x1.555556p-3f);
  q = __fmaf_rn(q, r, 0.5f);
  q = __fmaf_rn(q, r, 1.0f);
  q = __fmaf_rn(q, r, 1.0f);
  const int ki = (int)k;
  return __fmul_rn(q, __uint_as_float((uint32_t)(ki + 127) << 23));
}
