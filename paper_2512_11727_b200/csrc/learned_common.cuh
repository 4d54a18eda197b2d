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

// Shapes of the learned backend (ecco_config).
struct LDims {
  int F, H, C, D, B, R, S;
  float lr, noise;
};


__device__ __forceinline__ void seed_key(uint64_t seed, uint32_t salt, uint32_t& k0,
                                         uint32_t& k1) {
  k0 = (uint32_t)seed ^ salt;
  k1 = (uint32_t)(seed >> 32);
}


// Rows of one (job, step) minibatch: source by the cumulative source_mix in
// map order, frame uniform in the ring.  Writes the element offset of the
// row in the frame table and its label.
__device__ __forceinline__ void sample_one(const LDims& g, uint64_t seed, int job_id, int n_src,
                                           const int* src_cam, const double* src_frac,
                                           int window, int micro, int step, int s, int* cam_out,
                                           int* frame_out) {
  uint32_t k0, k1, out[4];
  seed_key(seed, (uint32_t)job_id * 0x9E3779B9u + 0x632BE5ABu, k0, k1);
  const uint32_t wt = ((uint32_t)window & 0xFFFFFFu) | (2u << 24);
  philox4x32((uint32_t)s, (uint32_t)step, (uint32_t)micro, wt, k0, k1, out);
  const double u = __dmul_rn((double)(((uint64_t)out[0] << 21) | (out[1] >> 11)), 0x1p-53);
  double cum = 0.0;
  int pick = n_src - 1;
  for (int i = 0; i < n_src; ++i) {
    cum = __dadd_rn(cum, src_frac[i]);
    if (u < cum) {
      pick = i;
      break;
    }
  }
  *cam_out = src_cam[pick];
  *frame_out = (int)(out[2] % (uint32_t)g.R);
}

