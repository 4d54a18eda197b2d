// Learned backend (backend L): synthetic camera streams resident in HBM,
// counter-based frame sampler, grouped MLP forward/backward/SGD for every
// job in one launch per phase, and the camera x group evaluation matrix.
//
// Specification: oracle/ecco_oracle.c (orc_gen_frames, orc_sample,
// orc_sgd_step, orc_count_correct).  The kernels in this file are the
// ECCO_MATH_FFMA_EXACT path: every output element is produced by one thread
// that accumulates in the oracle's sequential order with explicit fmaf, so
// results are bit-identical to the oracle.  The tensor-core path
// (tc_kernels.cu) replaces the two dense contractions.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "ctx.cuh"
#include "learned_common.cuh"
#include "tc_kernels.cuh"

namespace {

LDims dims(const ecco_ctx* c) {
  return {c->cfg.feat_dim,  c->cfg.hidden_dim,  c->cfg.num_classes, c->cfg.scene_dims,
          c->cfg.minibatch, c->cfg.ring_frames, c->cfg.eval_samples, c->cfg.sgd_lr,
          c->cfg.feature_noise};
}

// ---------------------------------------------------------------- streams --

__global__ void k_l_prototypes(LDims g, uint64_t seed, float* P, float* Q) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.C * g.F) return;
  const int k = idx / g.F, f = idx % g.F;
  uint32_t k0, k1, out[4];
  seed_key(seed, 0u, k0, k1);
  philox4x32((uint32_t)f, (uint32_t)k, 0u, 0xFE000000u, k0, k1, out);
  P[idx] = usym(out[0]);
  for (int d = 0; d < g.D; ++d) {
    philox4x32((uint32_t)f, (uint32_t)k, 1u + d, 0xFE000000u, k0, k1, out);
    Q[((size_t)k * g.D + d) * g.F + f] = __fmul_rn(usym(out[0]), 4.0f);
  }
}

// One thread per (camera, frame, 4 features); labels by the f4 == 0 thread.
// tag 0: training ring (R frames), tag 1: labelled eval set (S frames).
__global__ void __launch_bounds__(256) k_l_gen_frames(LDims g, uint64_t seed, int n_cams,
                                                      int window, int tag, int n_frames,
                                                      const double* scenes, const float* P,
                                                      const float* Q, uint16_t* x, int32_t* y) {
  const int f4n = g.F / 4;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t total = (size_t)n_cams * n_frames * f4n;
  if (idx >= total) return;
  const int f4 = (int)(idx % f4n);
  const size_t rf = idx / f4n;
  const int r = (int)(rf % n_frames);
  const int cam = (int)(rf / n_frames);
  uint32_t k0, k1, out[4];
  seed_key(seed, 0u, k0, k1);
  const uint32_t wt = ((uint32_t)window & 0xFFFFFFu) | ((uint32_t)tag << 24);
  philox4x32(0xFFFFFFFFu, (uint32_t)r, (uint32_t)cam, wt, k0, k1, out);
  const int lab = (int)(out[0] % (uint32_t)g.C);
  if (f4 == 0) y[rf] = lab;
  philox4x32((uint32_t)f4, (uint32_t)r, (uint32_t)cam, wt, k0, k1, out);
  float sd[8];
  for (int d = 0; d < g.D; ++d) sd[d] = (float)scenes[(size_t)cam * g.D + d];
  uint16_t v4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = f4 * 4 + i;
    const float nz = __fsub_rn(__fmul_rn((float)((out[i] & 0xFFFFu) + (out[i] >> 16)), 0x1p-16f), 1.0f);
    float v = P[(size_t)lab * g.F + f];
    for (int d = 0; d < g.D; ++d) v = __fmaf_rn(sd[d], Q[((size_t)lab * g.D + d) * g.F + f], v);
    v = __fmaf_rn(g.noise, nz, v);
    v4[i] = f32_to_bf16(v);
  }
  uint2 packed;
  packed.x = (uint32_t)v4[0] | ((uint32_t)v4[1] << 16);
  packed.y = (uint32_t)v4[2] | ((uint32_t)v4[3] << 16);
  *reinterpret_cast<uint2*>(x + rf * g.F + (size_t)f4 * 4) = packed;
}

// --------------------------------------------------------------- weights --

// Base model (orc_init_weights): every new job starts from it.
__global__ void k_l_init_weights(LDims g, uint64_t seed, int n, const int* slots, float* w,
                                 size_t n_params, bool w1_t) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * n_params) return;
  const int j = (int)(idx / n_params);
  const size_t q = idx % n_params;
  uint32_t k0, k1, out[4];
  seed_key(seed, 0x27D4EB2Fu, k0, k1);
  float v = 0.0f;
  const size_t fh = (size_t)g.F * g.H;
  const size_t w2o = fh + g.H;
  if (q < fh) {
    const int f = (int)(q / g.H), h = (int)(q % g.H);
    philox4x32((uint32_t)h, (uint32_t)f, 1u, 3u << 24, k0, k1, out);
    v = __fmul_rn(usym(out[0]), __fsqrt_rn(__fdiv_rn(6.0f, (float)g.F)));
  } else if (q >= w2o && q < w2o + (size_t)g.H * g.C) {
    const size_t r = q - w2o;
    const int k = (int)(r / g.C), c = (int)(r % g.C);
    philox4x32((uint32_t)c, (uint32_t)k, 2u, 3u << 24, k0, k1, out);
    v = __fmul_rn(usym(out[0]), __fsqrt_rn(__fdiv_rn(6.0f, (float)g.H)));
  }
  size_t dst = q;
  if (w1_t && q < fh) dst = (q % g.H) * (size_t)g.F + q / g.H;  // W1 stored [H][F]
  w[(size_t)slots[j] * n_params + dst] = v;
}

// ------------------------------------------------------------- sampler --

__global__ void k_l_sample(LDims g, uint64_t seed, int n_jobs, const int* job_ids,
                           const int* steps, const int* src_off, const int* src_cam,
                           const double* src_frac, const int* micro_base, int window, int t,
                           int step, const int32_t* labels, int64_t* row_off, int32_t* row_lab) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_jobs * g.B) return;
  const int j = idx / g.B, s = idx % g.B;
  if (step >= steps[j]) return;
  int cam, frame;
  const int s0 = src_off[j];
  sample_one(g, seed, job_ids[j], src_off[j + 1] - s0, src_cam + s0, src_frac + s0, window,
             micro_base[j] + t, step, s, &cam, &frame);
  const int64_t row = (int64_t)cam * g.R + frame;
  row_off[idx] = row * g.F;
  row_lab[idx] = labels[row];
}

__global__ void k_l_sample_debug(LDims g, uint64_t seed, int job_id, int n_src,
                                 const int* src_cam, const double* src_frac, int window,
                                 int micro, int step, int* out_cam, int* out_frame) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= g.B) return;
  sample_one(g, seed, job_id, n_src, src_cam, src_frac, window, micro, step, s, out_cam + s,
             out_frame + s);
}

// ------------------------------------------------------ FFMA contractions --
//
// Row blocks of 64 rows share one model slot.  Z[row, h] = sum_f x[row,f] *
// W1[f,h] (sequential f) + b1[h].  256 threads, 64 x 128 output tile, each
// thread owns 4 rows x 8 columns.

constexpr int kRB = 64;   // rows per block

// Which training rows are live in this SGD step: rows of job j are
// [j*rows_per_job, (j+1)*rows_per_job); a job whose step budget is spent
// (step >= steps[j]) is skipped.  steps == nullptr means always live.
struct Gate {
  const int* steps;
  int step;
  int rows_per_job;
  __device__ __forceinline__ bool live_row(size_t r) const {
    return steps == nullptr || step < steps[r / rows_per_job];
  }
};
constexpr int kHB = 128;  // hidden columns per block
constexpr int kKT = 32;   // k tile

// HB hidden units per block (128, or 32 when the grid would not fill the
// GPU); a thread owns 4 rows x HB/16 columns; k sequential per output.
template <int HB>
__global__ void __launch_bounds__(256) k_l_hidden_ffma(LDims g, const uint16_t* xbase,
                                                       const int64_t* row_off,
                                                       const int* blk_slot, Gate gate,
                                                       const float* wbase, size_t n_params,
                                                       float* Z) {
  constexpr int NC = HB / 16;
  const int blk = blockIdx.x;
  if (!gate.live_row((size_t)blk * kRB)) return;
  const int h0 = blockIdx.y * HB;
  const float* W1 = wbase + (size_t)blk_slot[blk] * n_params;
  const float* b1 = W1 + (size_t)g.F * g.H;
  __shared__ float As[kKT][kRB + 4];
  __shared__ __align__(16) float Bs[kKT][HB];
  __shared__ int64_t rows[kRB];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  if (tid < kRB) rows[tid] = row_off[(size_t)blk * kRB + tid];
  __syncthreads();
  float acc[4][NC];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[i][j] = 0.0f;
  for (int k0 = 0; k0 < g.F; k0 += kKT) {
    // X tile: 64 rows x 32 k (bf16 pairs), transposed into As[k][row]
    for (int e = tid; e < kRB * kKT / 2; e += 256) {
      const int r = e / (kKT / 2), kk = (e % (kKT / 2)) * 2;
      const uint32_t two = *reinterpret_cast<const uint32_t*>(xbase + rows[r] + k0 + kk);
      As[kk][r] = __uint_as_float(two << 16);
      As[kk + 1][r] = __uint_as_float(two & 0xFFFF0000u);
    }
    for (int e = tid; e < kKT * HB / 4; e += 256) {
      const int kk = e / (HB / 4), c4 = (e % (HB / 4)) * 4;
      *reinterpret_cast<float4*>(&Bs[kk][c4]) =
          *reinterpret_cast<const float4*>(W1 + (size_t)(k0 + kk) * g.H + h0 + c4);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kKT; ++kk) {
      float a[4], b[NC];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < NC; ++j) b[j] = Bs[kk][tx * NC + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const size_t r = (size_t)blk * kRB + ty * 4 + i;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int h = h0 + tx * NC + j;
      Z[r * g.H + h] = __fadd_rn(acc[i][j], b1[h]);
    }
  }
}

// One 64-row x 128-unit tile (row block blk, unit block hb) on 128 threads
// (tid 0..127), with its own shared-memory tile and a barrier over those
// threads only (sync).
struct H8Smem {
  float As[2][kKT][kRB];  // [buffer][k][row]
  float Bs[2][kKT][128];  // [buffer][k][unit]
  int64_t rows[kRB];
};

__device__ __forceinline__ void h8_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

template <typename Sync>
__device__ __forceinline__ void hidden8_tile(const LDims& g, const uint16_t* xbase,
                                             const int64_t* row_off, const int* blk_slot,
                                             const float* wbase, size_t n_params, float* Z,
                                             int blk, int hb, int tid, H8Smem& sm, Sync sync) {
  constexpr int HB = 128;
  const int h0 = hb * HB;
  const float* W1 = wbase + (size_t)blk_slot[blk] * n_params;
  const float* b1 = W1 + (size_t)g.F * g.H;
  const int tx = tid & 15, ty = tid >> 4;  // units 4 tx.. and 64 + 4 tx.., rows 8 ty..
  if (tid < kRB) sm.rows[tid] = row_off[(size_t)blk * kRB + tid];
  sync();
  // per K tile: X 64 rows x 32 k (bf16 pairs, 8 words per thread) through
  // registers (fp32 conversion and transpose), W1 32 k x 128 units by
  // cp.async straight into the other buffer; one barrier per K tile
  uint32_t xr[8];
  auto fetch_x = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // a thread keeps one row (L1 hits), lanes cover rows
      const int e = tid + u * 128, r = e & 63, kk = (e >> 6) * 2;
      xr[u] = *reinterpret_cast<const uint32_t*>(xbase + sm.rows[r] + k0 + kk);
    }
  };
  auto store_x = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * 128, r = e & 63, kk = (e >> 6) * 2;  // (conflict-free stores)
      sm.As[buf][kk][r] = __uint_as_float(xr[u] << 16);
      sm.As[buf][kk + 1][r] = __uint_as_float(xr[u] & 0xFFFF0000u);
    }
  };
  auto fetch_w = [&](int k0, int buf) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * 128, kk = e >> 5, c4 = (e & 31) * 4;
      h8_cp16(&sm.Bs[buf][kk][c4], W1 + (size_t)(k0 + kk) * g.H + h0 + c4);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = make_float2(0.0f, 0.0f);
  fetch_w(0, 0);
  fetch_x(0);
  store_x(0);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  sync();
  const int nkt = g.F / kKT;
  for (int t = 0; t < nkt; ++t) {
    const int cur = t & 1, nxt = cur ^ 1;
    const bool more = t + 1 < nkt;
    if (more) {
      fetch_w((t + 1) * kKT, nxt);
      fetch_x((t + 1) * kKT);
    }
    const float(*As)[kRB] = sm.As[cur];
    const float(*Bs)[128] = sm.Bs[cur];
#pragma unroll 4
    for (int kk = 0; kk < kKT; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      // units 4 tx..4 tx+3 and 64 + 4 tx..: lanes at a 16-byte stride (no
      // bank conflict; a 32-byte stride would conflict 2-way)
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float4 b1v = *reinterpret_cast<const float4*>(&Bs[kk][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w),
                            make_float2(b1v.x, b1v.y), make_float2(b1v.z, b1v.w)};
#pragma unroll
      for (int q = 0; q < 4; ++q)  // b pair in the operand reuse cache across rows
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][q] = __ffma2_rn(make_float2(av[i], av[i]), bv[q], acc[i][q]);
    }
    if (more) {
      store_x(nxt);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    sync();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const size_t r = (size_t)blk * kRB + ty * 8 + i;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int h = h0 + (q < 2 ? tx * 4 + 2 * q : 64 + tx * 4 + 2 * (q - 2));
      *reinterpret_cast<float2*>(Z + r * g.H + h) =
          make_float2(__fadd_rn(acc[i][q].x, b1[h]), __fadd_rn(acc[i][q].y, b1[h + 1]));
    }
  }
}

// Wide-grid form: 64 rows x 128 hidden units per block of 128 threads, 8
// rows x 8 units (two groups of 4) per thread (8 + 8 operands from shared
// memory per 64 FMAs: the 1 B/FMA the FFMA pipe sustains, where the 4 x 8
// tile above needs 1.5), packed fma.rn.f32x2 pairs along the units (each
// lane an fmaf chain, f ascending from 0, b1 added last: the oracle's
// order), the next K tile loaded into registers while this one computes.
__global__ void __launch_bounds__(128, 4) k_l_hidden_ffma8(LDims g, const uint16_t* xbase,
                                                        const int64_t* row_off,
                                                        const int* blk_slot, Gate gate,
                                                        const float* wbase, size_t n_params,
                                                        float* Z) {
  extern __shared__ __align__(16) uint8_t dsm8[];
  H8Smem& sm = *reinterpret_cast<H8Smem*>(dsm8);
  if (!gate.live_row((size_t)blockIdx.x * kRB)) return;
  hidden8_tile(g, xbase, row_off, blk_slot, wbase, n_params, Z, blockIdx.x, blockIdx.y,
               threadIdx.x, sm, [] { __syncthreads(); });
}

// 64-thread form: 8 rows x 16 units per thread (64 packed accumulator pairs:
// 0.75 B of shared memory per FMA, the FFMA pipe the bound), same tiles,
// buffers and per-output order as hidden8_tile.
__global__ void __launch_bounds__(64, 4) k_l_hidden_ffma16(LDims g, const uint16_t* xbase,
                                                        const int64_t* row_off,
                                                        const int* blk_slot, Gate gate,
                                                        const float* wbase, size_t n_params,
                                                        float* Z) {
  extern __shared__ __align__(16) uint8_t dsm16[];
  H8Smem& sm = *reinterpret_cast<H8Smem*>(dsm16);
  const int blk = blockIdx.x;
  if (!gate.live_row((size_t)blk * kRB)) return;
  constexpr int HB = 128;
  const int h0 = blockIdx.y * HB;
  const float* W1 = wbase + (size_t)blk_slot[blk] * n_params;
  const float* b1 = W1 + (size_t)g.F * g.H;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;  // units 4 tx + 32 j.., rows 8 ty..
  sm.rows[tid] = row_off[(size_t)blk * kRB + tid];
  __syncthreads();
  uint32_t xr[16];
  auto fetch_x = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {  // a thread keeps one row (L1 hits), lanes cover rows
      const int e = tid + u * 64, r = e & 63, kk = (e >> 6) * 2;
      xr[u] = *reinterpret_cast<const uint32_t*>(xbase + sm.rows[r] + k0 + kk);
    }
  };
  auto store_x = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + u * 64, r = e & 63, kk = (e >> 6) * 2;
      sm.As[buf][kk][r] = __uint_as_float(xr[u] << 16);
      sm.As[buf][kk + 1][r] = __uint_as_float(xr[u] & 0xFFFF0000u);
    }
  };
  auto fetch_w = [&](int k0, int buf) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + u * 64, kk = e >> 5, c4 = (e & 31) * 4;
      h8_cp16(&sm.Bs[buf][kk][c4], W1 + (size_t)(k0 + kk) * g.H + h0 + c4);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float2 acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[i][q] = make_float2(0.0f, 0.0f);
  fetch_w(0, 0);
  fetch_x(0);
  store_x(0);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int nkt = g.F / kKT;
  for (int t = 0; t < nkt; ++t) {
    const int cur = t & 1, nxt = cur ^ 1;
    const bool more = t + 1 < nkt;
    if (more) {
      fetch_w((t + 1) * kKT, nxt);
      fetch_x((t + 1) * kKT);
    }
    const float(*As)[kRB] = sm.As[cur];
    const float(*Bs)[128] = sm.Bs[cur];
#pragma unroll 2
    for (int kk = 0; kk < kKT; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float2 bv[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // units 32 j + 4 tx..: lanes at a 16-byte stride
        const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][32 * j + tx * 4]);
        bv[2 * j] = make_float2(b.x, b.y);
        bv[2 * j + 1] = make_float2(b.z, b.w);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)  // b pair in the operand reuse cache across rows
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][q] = __ffma2_rn(make_float2(av[i], av[i]), bv[q], acc[i][q]);
    }
    if (more) {
      store_x(nxt);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const size_t r = (size_t)blk * kRB + ty * 8 + i;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int h = h0 + 32 * (q >> 1) + tx * 4 + 2 * (q & 1);
      *reinterpret_cast<float2*>(Z + r * g.H + h) =
          make_float2(__fadd_rn(acc[i][q].x, b1[h]), __fadd_rn(acc[i][q].y, b1[h + 1]));
    }
  }
}

// Persistent form for a matrix that runs BESIDE other work (the
// oracle-exact window's regroup matrix next to the serial chains): one
// 512-thread block per SM (4 independent 128-thread tile workers, a named
// barrier each; the padded shared memory keeps a second block off the SM),
// at most (SMs - reserve) blocks, so the reserved SMs stay whole for the
// chains' clusters.  Same tiles, same arithmetic.
constexpr uint32_t kH8PersistentSmem = 4u * (uint32_t)sizeof(H8Smem);  // 4 workers: one block per SM
__global__ void __launch_bounds__(512, 1) k_l_hidden_ffma8_persistent(
    LDims g, const uint16_t* xbase, const int64_t* row_off, const int* blk_slot, Gate gate,
    const float* wbase, size_t n_params, float* Z, int nb, int nhb) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int grp = threadIdx.x >> 7, tid = threadIdx.x & 127;
  H8Smem& sm = reinterpret_cast<H8Smem*>(dsm)[grp];
  auto sync = [grp] { asm volatile("bar.sync %0, 128;" ::"r"(grp + 1) : "memory"); };
  for (long w = (long)blockIdx.x * 4 + grp; w < (long)nb * nhb; w += (long)gridDim.x * 4) {
    const int blk = (int)(w / nhb), hb = (int)(w % nhb);
    if (!gate.live_row((size_t)blk * kRB)) continue;
    hidden8_tile(g, xbase, row_off, blk_slot, wbase, n_params, Z, blk, hb, tid, sm, sync);
    sync();  // (the next tile's row table overwrites this one's)
  }
}

// Launches the hidden layer with the widest tile that still fills the GPU.
static void launch_hidden_ffma(ecco_ctx* ctx, int nb, const LDims& g, const uint16_t* xbase,
                               const int64_t* row_off, const int* blk_slot, Gate gate,
                               const float* wbase, size_t n_params, float* Z) {
  // ECCO_FFMA_HIDDEN8: 0 never, 1 always (tests), unset: wide grids only
  const char* e = getenv("ECCO_FFMA_HIDDEN8");
  const bool h8 = e ? e[0] == '1' : (long)nb * (g.H / kHB) >= 8 * 148;
  if (h8 && g.H % 128 == 0 && g.F % kKT == 0 && ctx->reserve_sms > 0) {
    // beside the context stream's chains: persistent, the reserved SMs left whole
    static DeviceFlags attr;
    if (!attr.done(ctx->cfg.device)) {
      ECCO_CUDA(cudaFuncSetAttribute(k_l_hidden_ffma8_persistent,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kH8PersistentSmem));
      attr.mark(ctx->cfg.device);
    }
    int sms = 0;
    ECCO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->cfg.device));
    const long items = (long)nb * (g.H / 128);
    const int grid = (int)std::max(1L, std::min<long>((items + 3) / 4, sms - ctx->reserve_sms));
    k_l_hidden_ffma8_persistent<<<grid, 512, kH8PersistentSmem, ctx->stream>>>(
        g, xbase, row_off, blk_slot, gate, wbase, n_params, Z, nb, g.H / 128);
  } else if (h8 && g.H % 128 == 0 && g.F % kKT == 0 &&
             !(getenv("ECCO_FFMA_HIDDEN16") && getenv("ECCO_FFMA_HIDDEN16")[0] == '0')) {
    // (8 x 16 per thread: +2.6% over the 8 x 8 tile at C3; ECCO_FFMA_HIDDEN16=0 keeps that one)
    static DeviceFlags attr16;
    if (!attr16.done(ctx->cfg.device)) {
      ECCO_CUDA(cudaFuncSetAttribute(k_l_hidden_ffma16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(H8Smem)));
      attr16.mark(ctx->cfg.device);
    }
    k_l_hidden_ffma16<<<dim3(nb, g.H / 128), 64, sizeof(H8Smem), ctx->stream>>>(
        g, xbase, row_off, blk_slot, gate, wbase, n_params, Z);
  } else if (h8 && g.H % 128 == 0 && g.F % kKT == 0) {
    static DeviceFlags attr8;
    if (!attr8.done(ctx->cfg.device)) {
      ECCO_CUDA(cudaFuncSetAttribute(k_l_hidden_ffma8, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(H8Smem)));
      attr8.mark(ctx->cfg.device);
    }
    k_l_hidden_ffma8<<<dim3(nb, g.H / 128), 128, sizeof(H8Smem), ctx->stream>>>(
        g, xbase, row_off, blk_slot, gate, wbase, n_params, Z);
  }
  else if ((long)nb * (g.H / kHB) >= 2 * 148)
    k_l_hidden_ffma<kHB><<<dim3(nb, g.H / kHB), 256, 0, ctx->stream>>>(g, xbase, row_off, blk_slot,
                                                                       gate, wbase, n_params, Z);
  else
    k_l_hidden_ffma<32><<<dim3(nb, g.H / 32), 256, 0, ctx->stream>>>(g, xbase, row_off, blk_slot,
                                                                     gate, wbase, n_params, Z);
}

// The head contractions of the general path, shared-memory tiled:
//   logits[row, c] = sum_k relu(Z[row, k]) * W2[k, c] (k ascending) + b2[c]
//   dH[row, k]     = Z[row, k] > 0 ? sum_c DL[row, c] * W2[k, c] (c ascending) : 0
//   W2[k, c]      -= lr * sum_s relu(Z[s, k]) * DL[s, c] (s ascending); b2 likewise
// Every output keeps that sequential accumulation order (one __fmaf_rn per
// term, orc_sgd_step's order), so the FFMA math stays bit-exact with the
// oracle; the tiles only stop W2 / Z / DL being re-read per output.
constexpr int kHT = 32;  // reduction chunk of the tiled head kernels

// logits: 64 rows x 32 classes per block, 4 rows x 4 classes per thread.
// (split-K form, tensor-core math only -- the sum order is not the
// oracle's: block z covers hidden units [z*kspan, (z+1)*kspan) and writes
// its partial (no b2) to L + z*n_rows*C; k_l_logits_sum adds the partials in
// z order and b2.  kspan = H is the exact form.)
// NT threads: a block covers 64 rows x NT / 4 classes (NT = 128: 32 classes;
// NT = 64: the 16 of the classifier, no idle class lanes), 4 rows x 4
// classes per thread, k ascending from 0 per output.
template <int NT>
__global__ void __launch_bounds__(NT) k_l_logits_t(LDims g, int n_rows, const int* blk_slot,
                                                   Gate gate, const float* wbase,
                                                   size_t n_params, const float* Z, float* L,
                                                   int kspan = 0) {
  constexpr int CW = NT / 4;  // classes per block
  const int blk = blockIdx.x, c0 = blockIdx.y * CW;
  const int kb = kspan > 0 ? blockIdx.z * kspan : 0;
  const int ke = kspan > 0 ? kb + kspan : g.H;
  const bool part = kspan > 0;
  if (part) L += (size_t)blockIdx.z * n_rows * g.C;
  if (!gate.live_row((size_t)blk * kRB)) return;
  const float* W2 = wbase + (size_t)blk_slot[blk] * n_params + (size_t)g.F * g.H + g.H;
  const float* b2 = W2 + (size_t)g.H * g.C;
  __shared__ __align__(16) float Zs[kHT][kRB + 4];
  __shared__ __align__(16) float Ws[kHT][CW + 4];
  const int tid = threadIdx.x, tx = tid % (CW / 4), ty = tid / (CW / 4);
  float acc[4][4] = {};
  const size_t r0 = (size_t)blk * kRB;
  // next chunk's Z / W2 values prefetched into registers (load-latency bound)
  constexpr int kZ = kRB * kHT / NT, kW = kHT * CW / NT;
  float zr[kZ], wr[kW];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < kZ; ++u) {
      const int e = tid + u * NT, r = e / kHT, k = e % kHT;
      zr[u] = Z[(r0 + r) * g.H + k0 + k];
    }
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const int e = tid + u * NT, k = e / CW, c = e % CW;
      wr[u] = c0 + c < g.C ? W2[(size_t)(k0 + k) * g.C + c0 + c] : 0.0f;
    }
  };
  fetch(kb);
  for (int k0 = kb; k0 < ke; k0 += kHT) {
#pragma unroll
    for (int u = 0; u < kZ; ++u) {
      const int e = tid + u * NT;
      Zs[e % kHT][e / kHT] = zr[u] > 0.0f ? zr[u] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const int e = tid + u * NT;
      Ws[e / CW][e % CW] = wr[u];
    }
    __syncthreads();
    if (k0 + kHT < ke) fetch(k0 + kHT);
#pragma unroll 8
    for (int k = 0; k < kHT; ++k) {
      const float4 z = *reinterpret_cast<const float4*>(&Zs[k][ty * 4]);
      const float4 w = *reinterpret_cast<const float4*>(&Ws[k][tx * 4]);
      const float zv[4] = {z.x, z.y, z.z, z.w}, wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = __fmaf_rn(zv[i], wv[q], acc[i][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + tx * 4 + q;
      if (c < g.C) L[(r0 + ty * 4 + i) * g.C + c] = part ? acc[i][q] : __fadd_rn(acc[i][q], b2[c]);
    }
}

// logits = sum of the ks split-K partials (z ascending) + b2 of the row's model.
__global__ void k_l_logits_sum(LDims g, int n_rows, int ks, const int* blk_slot, Gate gate,
                               const float* wbase, size_t n_params, const float* Lp, float* L) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)n_rows * g.C) return;
  const size_t r = e / g.C;
  if (!gate.live_row(r)) return;
  const int c = (int)(e % g.C);
  const float* b2 = wbase + (size_t)blk_slot[r / kRB] * n_params + (size_t)g.F * g.H + g.H +
                    (size_t)g.H * g.C;
  float v = Lp[e];
  for (int z = 1; z < ks; ++z) v = __fadd_rn(v, Lp[(size_t)z * n_rows * g.C + e]);
  L[e] = __fadd_rn(v, b2[c]);
}

// dH: 64 rows x 64 hidden units per block, 8 rows x 4 units per thread; c ascending.
__global__ void __launch_bounds__(128) k_l_dh_t(LDims g, int n_rows, const int* blk_slot,
                                                Gate gate, const float* wbase, size_t n_params,
                                                const float* Z, const float* DL, float* DH) {
  const int blk = blockIdx.x, h0 = blockIdx.y * 64;
  if (!gate.live_row((size_t)blk * kRB)) return;
  const float* W2 = wbase + (size_t)blk_slot[blk] * n_params + (size_t)g.F * g.H + g.H;
  __shared__ __align__(16) float Ds[kHT][kRB + 4];
  __shared__ __align__(16) float Ws[kHT][64 + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[8][4] = {};
  const size_t r0 = (size_t)blk * kRB;
  constexpr int kDv = kRB * kHT / 128, kWv = 64 * kHT / 128;
  float dr[kDv], wr[kWv];
  auto fetch = [&](int c0) {  // next chunk into registers (load-latency bound)
    const int nc = min(kHT, g.C - c0);
#pragma unroll
    for (int u = 0; u < kDv; ++u) {
      const int e = tid + u * 128, r = e / kHT, c = e % kHT;
      dr[u] = c < nc ? DL[(r0 + r) * g.C + c0 + c] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kWv; ++u) {
      const int e = tid + u * 128, h = e / kHT, c = e % kHT;
      wr[u] = c < nc ? W2[(size_t)(h0 + h) * g.C + c0 + c] : 0.0f;
    }
  };
  fetch(0);
  for (int c0 = 0; c0 < g.C; c0 += kHT) {
    const int nc = min(kHT, g.C - c0);
#pragma unroll
    for (int u = 0; u < kDv; ++u) {
      const int e = tid + u * 128;
      Ds[e % kHT][e / kHT] = dr[u];
    }
#pragma unroll
    for (int u = 0; u < kWv; ++u) {
      const int e = tid + u * 128;
      Ws[e % kHT][e / kHT] = wr[u];
    }
    __syncthreads();
    if (c0 + kHT < g.C) fetch(c0 + kHT);
    for (int c = 0; c < nc; ++c) {
      const float4 w = *reinterpret_cast<const float4*>(&Ws[c][tx * 4]);
      const float4 d0 = *reinterpret_cast<const float4*>(&Ds[c][ty * 8]);
      const float4 d1 = *reinterpret_cast<const float4*>(&Ds[c][ty * 8 + 4]);
      const float wv[4] = {w.x, w.y, w.z, w.w};
      const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = __fmaf_rn(dv[i], wv[q], acc[i][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const size_t o = (r0 + ty * 8 + i) * g.H + h0 + tx * 4 + q;
      DH[o] = Z[o] > 0.0f ? acc[i][q] : 0.0f;
    }
}

// W2 / b2 update of one job: 64 hidden units x 32 classes per block, 4 x 4
// per thread; rows s ascending.  Blocks of the first hidden tile also sum
// the b2 gradient of their classes.
__global__ void __launch_bounds__(128) k_l_update2_t(LDims g, int n_jobs, const int* slots,
                                                     const int* steps, int step, float* wbase,
                                                     size_t n_params, const float* Z,
                                                     const float* DL) {
  const int j = blockIdx.x, h0 = blockIdx.y * 64, c0 = blockIdx.z * 32;
  if (step >= steps[j]) return;
  float* W2 = wbase + (size_t)slots[j] * n_params + (size_t)g.F * g.H + g.H;
  float* b2 = W2 + (size_t)g.H * g.C;
  __shared__ __align__(16) float Zs[kHT][64 + 4];
  __shared__ __align__(16) float Ds[kHT][32 + 4];
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  float acc[4][4] = {};
  float bacc = 0.0f;
  const size_t r0 = (size_t)j * g.B;
  // the next chunk's Z / DL values are loaded into registers while this
  // chunk's products run (the kernel is bound by global-load latency)
  constexpr int kZ = kHT * 64 / 128, kD = kHT * 32 / 128;
  float zr[kZ], dr[kD];
  auto fetch = [&](int s0) {
    const int ns = min(kHT, g.B - s0);
#pragma unroll
    for (int u = 0; u < kZ; ++u) {
      const int e = tid + u * 128, s = e / 64, h = e % 64;
      zr[u] = s < ns ? Z[(r0 + s0 + s) * g.H + h0 + h] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kD; ++u) {
      const int e = tid + u * 128, s = e / 32, c = e % 32;
      dr[u] = s < ns && c0 + c < g.C ? DL[(r0 + s0 + s) * g.C + c0 + c] : 0.0f;
    }
  };
  fetch(0);
  for (int s0 = 0; s0 < g.B; s0 += kHT) {
    const int ns = min(kHT, g.B - s0);
#pragma unroll
    for (int u = 0; u < kZ; ++u) {
      const int e = tid + u * 128;
      Zs[e / 64][e % 64] = zr[u] > 0.0f ? zr[u] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kD; ++u) {
      const int e = tid + u * 128;
      Ds[e / 32][e % 32] = dr[u];
    }
    __syncthreads();
    if (s0 + kHT < g.B) fetch(s0 + kHT);
    for (int s = 0; s < ns; ++s) {
      const float4 z = *reinterpret_cast<const float4*>(&Zs[s][ty * 4]);
      const float4 d = *reinterpret_cast<const float4*>(&Ds[s][tx * 4]);
      const float zv[4] = {z.x, z.y, z.z, z.w}, dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = __fmaf_rn(zv[i], dv[q], acc[i][q]);
    }
    if (blockIdx.y == 0 && tid < 32)
      for (int s = 0; s < ns; ++s) bacc = __fadd_rn(bacc, Ds[s][tid]);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + tx * 4 + q;
      if (c < g.C) {
        float* w = W2 + (size_t)(h0 + ty * 4 + i) * g.C + c;
        *w = __fmaf_rn(-g.lr, acc[i][q], *w);
      }
    }
  if (blockIdx.y == 0 && tid < 32 && c0 + tid < g.C)
    b2[c0 + tid] = __fmaf_rn(-g.lr, bacc, b2[c0 + tid]);
}

// Softmax cross-entropy gradient of one training row.
__global__ void k_l_softmax_grad(LDims g, int n_rows, Gate gate, const float* L,
                                 const int32_t* lab, float* DL, float* loss_rows) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  if (!gate.live_row(r)) return;
  const float* l = L + (size_t)r * g.C;
  float m = l[0];
  for (int c = 1; c < g.C; ++c) m = l[c] > m ? l[c] : m;
  float sum = 0.0f;
  for (int c = 0; c < g.C; ++c) sum = __fadd_rn(sum, ecco_expf(__fsub_rn(l[c], m)));
  const float invB = __fdiv_rn(1.0f, (float)g.B);
  const int y = lab[r];
  for (int c = 0; c < g.C; ++c) {
    const float p = __fdiv_rn(ecco_expf(__fsub_rn(l[c], m)), sum);
    DL[(size_t)r * g.C + c] = __fmul_rn(__fsub_rn(p, c == y ? 1.0f : 0.0f), invB);
  }
  loss_rows[r] = logf(sum) - (l[y] - m);
}

// W1[f,h] -= lr * sum_s x[s,f] * dh[s,h] (sequential s).  Tile 64 f x 128 h.
__global__ void __launch_bounds__(256) k_l_update1_ffma(LDims g, const int* slots,
                                                        const int* steps, int step,
                                                        const uint16_t* xbase,
                                                        const int64_t* row_off, float* wbase,
                                                        size_t n_params, const float* DH) {
  const int j = blockIdx.z;
  if (step >= steps[j]) return;
  const int f0 = blockIdx.x * 64, h0 = blockIdx.y * kHB;
  float* W1 = wbase + (size_t)slots[j] * n_params;
  __shared__ float As[kKT][64 + 4];
  __shared__ __align__(16) float Bs[kKT][kHB];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[i][q] = 0.0f;
  const size_t r0 = (size_t)j * g.B;
  for (int s0 = 0; s0 < g.B; s0 += kKT) {
    for (int e = tid; e < kKT * 32; e += 256) {  // 32 samples x 64 f (bf16 pairs)
      const int s = e / 32, ff = (e % 32) * 2;
      const uint32_t two = *reinterpret_cast<const uint32_t*>(xbase + row_off[r0 + s0 + s] + f0 + ff);
      As[s][ff] = __uint_as_float(two << 16);
      As[s][ff + 1] = __uint_as_float(two & 0xFFFF0000u);
    }
    for (int e = tid; e < kKT * kHB / 4; e += 256) {
      const int s = e / (kHB / 4), c4 = (e % (kHB / 4)) * 4;
      *reinterpret_cast<float4*>(&Bs[s][c4]) =
          *reinterpret_cast<const float4*>(DH + (r0 + s0 + s) * g.H + h0 + c4);
    }
    __syncthreads();
#pragma unroll 8
    for (int s = 0; s < kKT; ++s) {
      float a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[s][ty * 4 + i];
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[s][tx * 8]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[s][tx * 8 + 4]);
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b4.x; b[5] = b4.y; b[6] = b4.z; b[7] = b4.w;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[i][q] = __fmaf_rn(a[i], b[q], acc[i][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = f0 + ty * 4 + i;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const size_t o = (size_t)f * g.H + h0 + tx * 8 + q;
      W1[o] = __fmaf_rn(-g.lr, acc[i][q], W1[o]);
    }
  }
}

__global__ void k_l_update_b1(LDims g, int n_jobs, const int* slots, const int* steps, int step,
                              float* wbase, size_t n_params, const float* DH) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_jobs * g.H) return;
  const int j = idx / g.H, h = idx % g.H;
  if (step >= steps[j]) return;
  float* b1 = wbase + (size_t)slots[j] * n_params + (size_t)g.F * g.H;
  const size_t r0 = (size_t)j * g.B;
  float a = 0.0f;
  for (int s = 0; s < g.B; ++s) a = __fadd_rn(a, DH[(r0 + s) * g.H + h]);
  b1[h] = __fmaf_rn(-g.lr, a, b1[h]);
}

// Mean minibatch loss per job for this step (diagnostics).
__global__ void k_l_loss_mean(LDims g, int n_jobs, const int* slots, const int* steps, int step,
                              const float* loss_rows, float* out, int T, int t) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_jobs) return;
  if (step == 0 && steps[j] == 0) out[(size_t)slots[j] * T + t] = __int_as_float(0x7fc00000);
  if (step >= steps[j]) return;
  double a = 0.0;
  for (int s = 0; s < g.B; ++s) a += loss_rows[(size_t)j * g.B + s];
  out[(size_t)slots[j] * T + t] = (float)(a / g.B);
}

// ------------------------------------------------------------- eval ------

// Correct-prediction count of each (slot, camera) pair over the camera's S
// eval frames; one warp per (pair, row), first-max argmax like the oracle.
__global__ void k_l_count(LDims g, int n_pairs, const float* L,
                          const int32_t* eval_labels, const int* pair_cam, int* counts) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_pairs * g.S) return;
  const int p = r / g.S, s = r % g.S;
  const float* l = L + (size_t)r * g.C;
  int best = 0;
  for (int c = 1; c < g.C; ++c)
    if (l[c] > l[best]) best = c;
  if (best == eval_labels[(size_t)pair_cam[p] * g.S + s]) atomicAdd(&counts[p], 1);
}

__global__ void k_l_pair_rows(LDims g, int n_pairs, const int* pair_slot, const int* pair_cam,
                              int64_t* row_off, int* blk_slot) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_pairs * g.S) return;
  const int p = r / g.S, s = r % g.S;
  row_off[r] = ((int64_t)pair_cam[p] * g.S + s) * g.F;
  if (r % kRB == 0) blk_slot[r / kRB] = pair_slot[p];
}

// acc = count / S; masked pairs become NaN.
__global__ void k_l_matrix_out(LDims g, int n, const int* counts, const int* pair_out,
                               double* out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  out[pair_out[p]] = __ddiv_rn((double)counts[p], (double)g.S);
}

__global__ void k_l_fill_nan(size_t n, double* out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __longlong_as_double(0x7ff8000000000000LL);
}

// Per-job mean over members (sequential in member order).
__global__ void k_l_job_mean(LDims g, int n_jobs, const int* mem_off, const int* counts,
                             double floor_acc, double* out, int stride, int col) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_jobs) return;
  const int m0 = mem_off[j], nm = mem_off[j + 1] - m0;
  double sum = 0.0;
  for (int m = 0; m < nm; ++m) sum = __dadd_rn(sum, __ddiv_rn((double)counts[m0 + m], (double)g.S));
  out[(size_t)j * stride + col] = nm == 0 ? floor_acc : __ddiv_rn(sum, (double)nm);
}

// Serial chains (one job, `depth` snapshots evaluated in one pass): the
// (snapshot, member) pair list -- pair u * n_mem + m is member m under
// snapshot u (virtual slot u of the snapshot pool) -- and each snapshot's
// member mean, in k_l_job_mean's order.
__global__ void k_l_serial_pairs(int n_mem, int depth, const int* mem_cam, int* pair_slot,
                                 int* pair_cam) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_mem * depth) return;
  pair_slot[i] = i / n_mem;
  pair_cam[i] = mem_cam[i % n_mem];
}
__global__ void k_l_serial_mean(LDims g, int n_mem, int depth, const int* counts, double* out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= depth) return;
  double sum = 0.0;
  for (int m = 0; m < n_mem; ++m)
    sum = __dadd_rn(sum, __ddiv_rn((double)counts[(size_t)u * n_mem + m], (double)g.S));
  out[1 + u] = __ddiv_rn(sum, (double)n_mem);
}

// Warp-reduced argmax / threshold of group_request (grouping.cpp:30-39) per
// probe row.  The matrix is n_blocks column blocks of gb columns, block b
// stored row-major at M + b*n*gb (n_blocks = 1: plain n x gb row-major; the
// all-gathered column blocks of every rank otherwise).
// group_request's join rule (grouping.cpp:30-39) per camera row, one warp
// per row: among unmasked columns with acc >= req the highest accuracy, ties
// to the lowest group id (strict '>' over jobs in ascending id order).  The
// id of column j is ids[j] when a column -> group map is given (cost-balanced
// placement: a rank's block holds any groups), else j; ids[j] < 0 marks a
// padding column.
__global__ void k_l_route(int n, int gb, int n_blocks, const double* M, const double* req,
                          const int* ids, int* best_col, double* best_acc) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (i >= n) return;
  int bc = -1;
  double ba = 0.0;
  const double r = req ? req[i] : 0.0;
  const int g = gb * n_blocks;
  for (int j = lane; j < g; j += 32) {
    const int id = ids ? ids[j] : j;
    if (id < 0) continue;
    const int b = j / gb;
    const double a = M[((size_t)b * n + i) * gb + (j - b * gb)];
    if (a != a || a < r) continue;  // masked (NaN) or below the device accuracy
    if (bc < 0 || a > ba || (a == ba && id < bc)) {
      bc = id;
      ba = a;
    }
  }
  for (int off = 16; off; off >>= 1) {
    const int oc = __shfl_down_sync(0xffffffffu, bc, off);
    const double oa = __shfl_down_sync(0xffffffffu, ba, off);
    if (oc >= 0 && (bc < 0 || oa > ba || (oa == ba && oc < bc))) {
      bc = oc;
      ba = oa;
    }
  }
  if (lane == 0) {
    best_col[i] = bc;
    best_acc[i] = bc >= 0 ? ba : 0.0;
  }
}

__global__ void k_l_copy_weights(int n_jobs, const int* slots, const float* src_base,
                                 size_t src_slot_stride, size_t src_off, float* dst_base,
                                 size_t dst_slot_stride, size_t dst_off, size_t n_params,
                                 const int* sel) {
  const int j = blockIdx.y;
  if (sel && sel[j] <= 0) return;
  const int slot = slots[j];
  const float4* s = reinterpret_cast<const float4*>(src_base + (size_t)slot * src_slot_stride +
                                                    src_off + (sel ? (size_t)(sel[j] - 1) * n_params : 0));
  float4* d = reinterpret_cast<float4*>(dst_base + (size_t)slot * dst_slot_stride + dst_off);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_params / 4;
       i += (size_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

}  // namespace

// ====================================================================
namespace lbackend {

static inline unsigned nblk(size_t n, int b) { return (unsigned)((n + b - 1) / b); }

void init(ecco_ctx* ctx) {
  const LDims g = dims(ctx);
  k_l_prototypes<<<nblk((size_t)g.C * g.F, 256), 256, 0, ctx->stream>>>(g, ctx->cfg.seed,
                                                                         ctx->d_proto_p, ctx->d_proto_q);
  ECCO_LAUNCHED(ctx);
  // the tensor-core math evaluates through the fused kernel (eval_kernels.cu)
  // (wide models -- the detection head -- through k_eval_wide, trained by
  // the wide fused chain)
  if (ctx->cfg.math == ECCO_MATH_TC_BF16 && fused::supported(ctx)) {
    const bool chain = fused::train_supported(ctx) || fused::wide_supported(ctx);
    fused::init_shadow(ctx, ctx->sh_commit);
    fused::init_shadow(ctx, ctx->sh_spec);
    if (chain) {  // chains evaluate on a side stream, alternating shadows
      fused::init_shadow(ctx, ctx->sh_spec2);
      fused::init_shadow(ctx, ctx->sh_pool, (size_t)ctx->cfg.max_depth);
      ECCO_CUDA(cudaStreamCreateWithFlags(&ctx->eval_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        ECCO_CUDA(cudaEventCreateWithFlags(&ctx->ev_chain[i], cudaEventDisableTiming));
        ECCO_CUDA(cudaEventCreateWithFlags(&ctx->ev_eval[i], cudaEventDisableTiming));
      }
    }
    ctx->sh_dirty.assign(ctx->cfg.max_jobs, 1);
    ctx->fused_eval = true;
    ctx->fused_train = chain;
    ctx->w1_t = chain;
  } else if (ctx->cfg.math == ECCO_MATH_TC_BF16 && fused::wide_supported(ctx)) {
    // wide models (detection head): fused chains, members evaluated on the
    // general path on a side stream beside the next micro-window's chain
    ctx->fused_train = true;
    ctx->w1_t = true;  // [H][F]: a CTA's master slice is contiguous
    ECCO_CUDA(cudaStreamCreateWithFlags(&ctx->eval_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      ECCO_CUDA(cudaEventCreateWithFlags(&ctx->ev_chain[i], cudaEventDisableTiming));
      ECCO_CUDA(cudaEventCreateWithFlags(&ctx->ev_eval[i], cudaEventDisableTiming));
    }
  }
}

// Refreshes the committed-model shadow for the dirty slots among `slots`.
static void refresh_committed(ecco_ctx* ctx, const int* slots, int n) {
  std::vector<int> todo;
  for (int i = 0; i < n; ++i)
    if (ctx->sh_dirty[slots[i]]) {
      ctx->sh_dirty[slots[i]] = 0;
      todo.push_back(slots[i]);
    }
  fused::refresh_shadow(ctx, ctx->sh_commit, ctx->d_w, ctx->n_params, todo);
}

// The tile plan of a pairs-mode evaluation (which slots each 128/256-row
// tile walks), uploaded once: a chain of micro-windows evaluates the same
// (member, slot) pairs after every micro-window, so it reuses the plan and
// the host never waits for the stream inside the chain (a pageable upload
// would drain it first).
struct PairsPlan {
  int n_pairs = 0, n_tiles = 0, n_ent = 0;
  bool pair = false;
  const int* d_ent = nullptr;
  const int* d_ebeg = nullptr;
};

static PairsPlan plan_pairs(ecco_ctx* ctx, int n_pairs, const int* h_slot, int ent_buf,
                            int ebeg_buf) {
  const int S = ctx->cfg.eval_samples;
  PairsPlan pl;
  pl.n_pairs = n_pairs;
  pl.pair = fused::pair_supported(ctx);
  const int TR = pl.pair ? 256 : 128;
  pl.n_tiles = (int)(((size_t)n_pairs * S + TR - 1) / TR);
  std::vector<int> ebeg(pl.n_tiles + 1), ent;
  for (int m = 0; m < pl.n_tiles; ++m) {
    ebeg[m] = (int)ent.size();
    const int p_lo = (int)((size_t)m * TR / S);
    const int p_hi = std::min(n_pairs, (int)(((size_t)m * TR + TR - 1) / S) + 1);
    for (int p = p_lo; p < p_hi; ++p)
      if (std::find(ent.begin() + ebeg[m], ent.end(), h_slot[p]) == ent.end()) ent.push_back(h_slot[p]);
  }
  ebeg[pl.n_tiles] = (int)ent.size();
  pl.n_ent = (int)ent.size();
  pl.d_ent = ctx->upload(ent_buf, ent.data(), ent.size());
  pl.d_ebeg = ctx->upload(ebeg_buf, ebeg.data(), ebeg.size());
  return pl;
}

static void pair_counts_planned(ecco_ctx* ctx, const Shadow& sh, const float* wbase,
                                size_t wstride, const PairsPlan& pl, const int* d_slot,
                                const int* d_cam, int* d_counts) {
  ECCO_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(int) * std::max(pl.n_pairs, 1), ctx->stream));
  fused::eval_counts(ctx, sh, wbase, wstride, pl.n_pairs, d_cam, pl.n_ent, pl.d_ent, pl.d_ent,
                     pl.n_tiles, pl.d_ebeg, d_slot, 0, d_counts, nullptr, (double)pl.n_pairs,
                     pl.pair);
}

void refresh_models(ecco_ctx* ctx, const int* h_slots, int n) {
  if (ctx->fused_eval && n > 0) refresh_committed(ctx, h_slots, n);
}

// Fused pairs-mode counts: probe p = camera h_cam/d_cam[p] under slot
// h_slot[p]; consecutive probes of one slot share 128-row tiles.
static void pair_counts_fused(ecco_ctx* ctx, const Shadow& sh, const float* wbase, size_t wstride,
                              int n_pairs, const int* h_slot, const int* d_slot, const int* d_cam,
                              int* d_counts) {
  const int S = ctx->cfg.eval_samples;
  // 128-row tiles, or 256-row super tiles for the CTA-pair kernel (half the
  // W1^T stream per FLOP): each tile walks the distinct slots of its pairs
  const bool pair = fused::pair_supported(ctx);
  const int TR = pair ? 256 : 128;
  const int n_tiles = (int)(((size_t)n_pairs * S + TR - 1) / TR);
  std::vector<int> ebeg(n_tiles + 1), ent;
  for (int m = 0; m < n_tiles; ++m) {
    ebeg[m] = (int)ent.size();
    const int p_lo = (int)((size_t)m * TR / S);
    const int p_hi = std::min(n_pairs, (int)(((size_t)m * TR + TR - 1) / S) + 1);
    for (int p = p_lo; p < p_hi; ++p)
      if (std::find(ent.begin() + ebeg[m], ent.end(), h_slot[p]) == ent.end()) ent.push_back(h_slot[p]);
  }
  ebeg[n_tiles] = (int)ent.size();
  int* d_ent = ctx->upload(12, ent.data(), ent.size());
  int* d_ebeg = ctx->upload(13, ebeg.data(), ebeg.size());
  ECCO_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(int) * std::max(n_pairs, 1), ctx->stream));
  fused::eval_counts(ctx, sh, wbase, wstride, n_pairs, d_cam, (int)ent.size(), d_ent, d_ent,
                     n_tiles, d_ebeg, d_slot, 0, d_counts, nullptr, (double)n_pairs, pair);
}

// The general (unfused) tensor-core evaluation of a fixed list of (slot,
// camera) pairs, planned once: the wide fused chain (detection-head shapes)
// evaluates the same member pairs after every micro-window, so the 128-row
// tile list and the evaluated slots are built on the host from the host's
// pair slots and uploaded ONCE per call -- no device->host read or pageable
// upload (which would drain the stream) inside the chain.
struct GeneralPlan {
  bool ok = false;
  int n_pairs = 0, n_tiles = 0, n_us = 0;
  const TcTile* d_tiles = nullptr;
  const int* d_us = nullptr;
};

static GeneralPlan plan_general(ecco_ctx* ctx, int n_pairs, const int* h_slot, int tiles_buf = 19,
                                int us_buf = 20) {
  const LDims g = dims(ctx);
  GeneralPlan pl;
  const int chunk = std::max(1, (int)std::min<size_t>(n_pairs, (size_t)(256u << 20) / ((size_t)g.S * g.H * 4)));
  if (n_pairs == 0 || n_pairs > chunk || g.S % kRB || g.H % 256 || ctx->cfg.math != ECCO_MATH_TC_BF16)
    return pl;  // pair_counts (chunked, per-call plan) serves the rest
  const int nb = n_pairs * g.S / kRB;
  std::vector<int> hslot(nb);
  for (int b = 0; b < nb; ++b) hslot[b] = h_slot[(size_t)b * kRB / g.S];
  std::vector<TcTile> tiles;  // same cut as pair_counts: never straddle two models
  for (int b = 0; b < nb;) {
    const int take = (b + 1 < nb && hslot[b + 1] == hslot[b]) ? 2 : 1;
    tiles.push_back({hslot[b], b * kRB, take * kRB, 0});
    b += take;
  }
  std::vector<int> us(hslot);
  std::sort(us.begin(), us.end());
  us.erase(std::unique(us.begin(), us.end()), us.end());
  pl.d_tiles = ctx->upload(tiles_buf, tiles.data(), tiles.size());
  pl.d_us = ctx->upload(us_buf, us.data(), us.size());
  pl.n_tiles = (int)tiles.size();
  pl.n_us = (int)us.size();
  pl.n_pairs = n_pairs;
  pl.ok = true;
  return pl;
}

static void pair_counts_general_planned(ecco_ctx* ctx, const GeneralPlan& pl, const float* wbase,
                                        size_t wstride, const int* d_pair_slot,
                                        const int* d_pair_cam, int* d_counts) {
  const LDims g = dims(ctx);
  const int np = pl.n_pairs, rows = np * g.S, nb = rows / kRB;
  ECCO_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(int) * np, ctx->stream));
  int64_t* row_off = (int64_t*)ctx->scratch[4].get(sizeof(int64_t) * rows);
  int* blk_slot = (int*)ctx->scratch[5].get(sizeof(int) * nb);
  float* Z = (float*)ctx->scratch[6].get(sizeof(float) * (size_t)rows * g.H);
  float* L = (float*)ctx->scratch[7].get(sizeof(float) * (size_t)rows * g.C);
  k_l_pair_rows<<<nblk(rows, 256), 256, 0, ctx->stream>>>(g, np, d_pair_slot, d_pair_cam, row_off,
                                                           blk_slot);
  ECCO_LAUNCHED(ctx);
  // (slots index job models, or the snapshots of a serial chain)
  const size_t n_img = (size_t)std::max(ctx->cfg.max_jobs, ctx->cfg.max_depth);
  uint16_t* w1t = (uint16_t*)ctx->train_scratch[9].get(n_img * g.H * g.F * 2);
  fused::shadow_w1t(ctx, pl.d_us, pl.n_us, wbase, wstride, w1t);
  tc::fwd_hidden_bf16(ctx, ctx->d_eval, row_off, pl.d_tiles, pl.n_tiles, nullptr, 0, w1t, n_img,
                      wbase, wstride, Z, (double)rows);
  ECCO_TIMED(ctx, ECCO_KSTAT_EVAL_PAIRS, 2.0 * rows * g.H * g.C, (double)rows * g.H * 4,
             (k_l_logits_t<128><<<dim3(rows / kRB, (g.C + 31) / 32), 128, 0, ctx->stream>>>(
                 g, rows, blk_slot, Gate{nullptr, 0, 1}, wbase, wstride, Z, L)));
  ECCO_LAUNCHED(ctx);
  k_l_count<<<nblk(rows, 256), 256, 0, ctx->stream>>>(g, np, L, ctx->d_eval_labels, d_pair_cam,
                                                       d_counts);
  ECCO_LAUNCHED(ctx);
}

void generate_frames(ecco_ctx* ctx, int window) {
  const LDims g = dims(ctx);
  if (ctx->n_cams == 0) return;
  size_t total = (size_t)ctx->n_cams * g.R * (g.F / 4);
  k_l_gen_frames<<<nblk(total, 256), 256, 0, ctx->stream>>>(
      g, ctx->cfg.seed, ctx->n_cams, window, 0, g.R, ctx->d_scenes, ctx->d_proto_p,
      ctx->d_proto_q, ctx->d_frames, ctx->d_labels);
  ECCO_LAUNCHED(ctx);
  total = (size_t)ctx->n_cams * g.S * (g.F / 4);
  k_l_gen_frames<<<nblk(total, 256), 256, 0, ctx->stream>>>(
      g, ctx->cfg.seed, ctx->n_cams, window, 1, g.S, ctx->d_scenes, ctx->d_proto_p,
      ctx->d_proto_q, ctx->d_eval, ctx->d_eval_labels);
  ECCO_LAUNCHED(ctx);
  ctx->frames_window = window;
}

void seed(ecco_ctx* ctx, int n, const int* h_job_ids, const int* d_slots, const int* d_job_ids) {
  (void)h_job_ids;
  (void)d_job_ids;
  if (n == 0) return;
  const LDims g = dims(ctx);
  k_l_init_weights<<<nblk((size_t)n * ctx->n_params, 256), 256, 0, ctx->stream>>>(
      g, ctx->cfg.seed, n, d_slots, ctx->d_w, ctx->n_params, ctx->w1_t);
  ECCO_LAUNCHED(ctx);
}

// The whole oracle-exact evaluation of one (slot, camera) pair in one block
// (FFMA math, S = 64 rows, H = 256, C = 16): Z = X.W1 + b1 for all 256 units
// (8 rows x 16 units per thread, W1 tiles of 16 k by cp.async into double
// buffers), relu rows into shared memory in two 32-row halves, logits =
// relu(Z).W2 + b2 (one fmaf chain per output, k ascending), the first-max
// argmax per row, the correct count -- no hidden activations or logits in
// HBM, one launch for any number of pairs.  168 registers and 56 KB of
// shared memory: three blocks (12 warps) per SM hide the FFMA2 and shared
// load latencies that two blocks left exposed.  Every output keeps the
// oracle's order (orc count_correct).
constexpr int kFE_H = 256, kFE_C = 16, kFE_KT = 16, kFE_HALF = kRB / 2;
struct FESmem {
  union {
    struct {
      float As[2][kFE_KT][kRB];      // [buffer][k][row]
      float Bs[2][kFE_KT][kFE_H];    // [buffer][k][unit]
    } g;
    float Rs[kFE_HALF][kFE_H + 4];   // relu(Z + b1), one half of the rows
  } u;
  float W2s[kFE_H][kFE_C];
};
// Dense matrix mode (cams != nullptr): block p is the p-th pair of the
// n x gj matrix in group tiles of `tile` groups, cameras outer (eval_matrix's
// order), its count written at i * gj + j -- no pair lists.
struct FEMatrix {
  const int* cams = nullptr;
  const int* slots = nullptr;
  int n = 0, gj = 0, tile = 1;
};
__global__ void __launch_bounds__(128, 3) k_l_eval_ffma_fused(LDims g, int n_pairs,
                                                             const int* pair_slot,
                                                             const int* pair_cam, FEMatrix mx,
                                                             const uint16_t* eval,
                                                             const int32_t* eval_labels,
                                                             const float* wbase, size_t n_params,
                                                             int* counts) {
  extern __shared__ __align__(16) uint8_t dsmf[];
  FESmem& sm = *reinterpret_cast<FESmem*>(dsmf);
  int p = blockIdx.x, slot, cam;
  if (mx.cams) {
    const int per_tile = mx.n * mx.tile, t = p / per_tile, rr = p - t * per_tile;
    const int w = min(mx.tile, mx.gj - t * mx.tile), i = rr / w, j = t * mx.tile + rr % w;
    slot = mx.slots[j];
    cam = mx.cams[i];
    p = i * mx.gj + j;  // the count's place in the matrix
  } else {
    slot = pair_slot[p];
    cam = pair_cam[p];
  }
  const float* W1 = wbase + (size_t)slot * n_params;
  const float* b1 = W1 + (size_t)g.F * kFE_H;
  const float* W2 = b1 + kFE_H;
  const float* b2 = W2 + (size_t)kFE_H * kFE_C;
  const uint16_t* X = eval + (size_t)cam * kRB * g.F;  // the camera's 64 eval rows
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // units 4 tx + 64 j.., rows 8 ty..
  // W2 (16 KB) beside the first K tile
  for (int e = tid; e < kFE_H * kFE_C / 4; e += 128) h8_cp16(&sm.W2s[0][0] + 4 * e, W2 + 4 * e);
  constexpr int kXU = kRB * kFE_KT / 2 / 128;  // bf16 pairs per thread per tile
  uint32_t xr[kXU];
  auto fetch_x = [&](int k0) {
#pragma unroll
    for (int u = 0; u < kXU; ++u) {  // lanes cover rows, a thread keeps one row
      const int e = tid + u * 128, r = e & 63, kk = (e >> 6) * 2;
      xr[u] = *reinterpret_cast<const uint32_t*>(X + (size_t)r * g.F + k0 + kk);
    }
  };
  auto store_x = [&](int buf) {
#pragma unroll
    for (int u = 0; u < kXU; ++u) {
      const int e = tid + u * 128, r = e & 63, kk = (e >> 6) * 2;
      sm.u.g.As[buf][kk][r] = __uint_as_float(xr[u] << 16);
      sm.u.g.As[buf][kk + 1][r] = __uint_as_float(xr[u] & 0xFFFF0000u);
    }
  };
  auto fetch_w = [&](int k0, int buf) {
#pragma unroll
    for (int u = 0; u < kFE_KT * kFE_H / 4 / 128; ++u) {
      const int e = tid + u * 128, kk = e >> 6, c4 = (e & 63) * 4;
      h8_cp16(&sm.u.g.Bs[buf][kk][c4], W1 + (size_t)(k0 + kk) * kFE_H + c4);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float2 acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[i][q] = make_float2(0.0f, 0.0f);
  fetch_w(0, 0);
  fetch_x(0);
  store_x(0);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int nkt = g.F / kFE_KT;
  for (int t = 0; t < nkt; ++t) {
    const int cur = t & 1, nxt = cur ^ 1;
    const bool more = t + 1 < nkt;
    if (more) {
      fetch_w((t + 1) * kFE_KT, nxt);
      fetch_x((t + 1) * kFE_KT);
    }
    const float(*As)[kRB] = sm.u.g.As[cur];
    const float(*Bs)[kFE_H] = sm.u.g.Bs[cur];
#pragma unroll 2
    for (int kk = 0; kk < kFE_KT; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float2 bv[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // units 64 j + 4 tx..: lanes at a 16-byte stride
        const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][64 * j + tx * 4]);
        bv[2 * j] = make_float2(b.x, b.y);
        bv[2 * j + 1] = make_float2(b.z, b.w);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)  // b pair in the operand reuse cache across rows
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][q] = __ffma2_rn(make_float2(av[i], av[i]), bv[q], acc[i][q]);
    }
    if (more) {
      store_x(nxt);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
  }
  // per half: relu(Z + b1) rows into shared memory (the GEMM buffers are
  // dead), then logits: thread t -> row t / 4 of the half, classes
  // 4 (t & 3)..+4, k ascending; the row's 16 logits meet in lane t & ~3,
  // which scans them in class order (first max).
  const int lr = tid >> 2, cb = (tid & 3) * 4;
  int n_ok = 0;
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    if ((ty >> 2) == half) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (ty & 3) * 8 + i;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int h = 64 * (q >> 1) + tx * 4 + 2 * (q & 1);
          const float z0 = __fadd_rn(acc[i][q].x, __ldg(b1 + h));
          const float z1 = __fadd_rn(acc[i][q].y, __ldg(b1 + h + 1));
          *reinterpret_cast<float2*>(&sm.u.Rs[r][h]) =
              make_float2(z0 > 0.0f ? z0 : 0.0f, z1 > 0.0f ? z1 : 0.0f);
        }
      }
    }
    __syncthreads();
    float l[4] = {};
#pragma unroll 8
    for (int k = 0; k < kFE_H; ++k) {
      const float z = sm.u.Rs[lr][k];
      const float4 w = *reinterpret_cast<const float4*>(&sm.W2s[k][cb]);
      l[0] = __fmaf_rn(z, w.x, l[0]);
      l[1] = __fmaf_rn(z, w.y, l[1]);
      l[2] = __fmaf_rn(z, w.z, l[2]);
      l[3] = __fmaf_rn(z, w.w, l[3]);
    }
    float v[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float lc = __fadd_rn(l[c], __ldg(b2 + cb + c));
#pragma unroll
      for (int s = 0; s < 4; ++s) v[4 * s + c] = __shfl_sync(0xffffffffu, lc, (tid & ~3) + s);
    }
    if ((tid & 3) == 0) {
      int best = 0;
      float bv = v[0];
#pragma unroll
      for (int c = 1; c < 16; ++c)
        if (v[c] > bv) {
          bv = v[c];
          best = c;
        }
      n_ok += best == eval_labels[(size_t)cam * kRB + half * kFE_HALF + lr];
    }
    __syncthreads();  // Rs is rewritten by the next half
  }
  const int n0 = __syncthreads_count(n_ok & 1), n1 = __syncthreads_count(n_ok >> 1);
  if (tid == 0) counts[p] = n0 + 2 * n1;
}

// The exact pair evaluation in one block applies: FFMA math at S = 64,
// H = 256, C = 16, F % 16 = 0, not beside the chains (there the persistent
// GEMM leaves whole SMs to the chain's cluster); ECCO_FFMA_FUSED_EVAL=0
// keeps the chunked kernels.
static bool fe_ok(ecco_ctx* ctx, const LDims& g) {
  const char* ef = getenv("ECCO_FFMA_FUSED_EVAL");
  return ctx->cfg.math == ECCO_MATH_FFMA_EXACT && g.S == kRB && g.H == kFE_H && g.C == kFE_C &&
         g.F % kFE_KT == 0 && ctx->reserve_sms == 0 && !(ef && ef[0] == '0');
}
static void fe_launch(ecco_ctx* ctx, const LDims& g, int n_pairs, const int* d_pair_slot,
                      const int* d_pair_cam, FEMatrix mx, int* d_counts) {
  if (n_pairs <= 0) return;
  static DeviceFlags attr;
  if (!attr.done(ctx->cfg.device)) {
    ECCO_CUDA(cudaFuncSetAttribute(k_l_eval_ffma_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sizeof(FESmem)));
    attr.mark(ctx->cfg.device);
  }
  const double rows = (double)n_pairs * g.S;
  ECCO_TIMED(ctx, ECCO_KSTAT_EVAL_MATRIX, 2.0 * rows * g.F * g.H + 2.0 * rows * g.H * g.C,
             rows * g.F * 2 + (double)n_pairs * 4,
             (k_l_eval_ffma_fused<<<n_pairs, 128, sizeof(FESmem), ctx->stream>>>(
                 g, n_pairs, d_pair_slot, d_pair_cam, mx, ctx->d_eval, ctx->d_eval_labels,
                 ctx->d_w, ctx->n_params, d_counts)));
  ECCO_LAUNCHED(ctx);
}

// Counts for a list of (slot, camera) pairs, chunked to bound scratch (1 GiB
// of hidden activations per chunk: few, large launches -- a full C4 matrix
// in ~300 chunks, each a wide grid).
static void pair_counts(ecco_ctx* ctx, int n_pairs, const int* d_pair_slot, const int* d_pair_cam,
                        int* d_counts) {
  const LDims g = dims(ctx);
  if (fe_ok(ctx, g)) {  // one block per pair: hidden layer, head, argmax and count on chip
    fe_launch(ctx, g, n_pairs, d_pair_slot, d_pair_cam, FEMatrix{}, d_counts);
    return;
  }
  ECCO_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(int) * std::max(n_pairs, 1), ctx->stream));
  const int chunk = std::max(1, (int)std::min<size_t>(n_pairs, (size_t)(1u << 30) / ((size_t)g.S * g.H * 4)));
  for (int p0 = 0; p0 < n_pairs; p0 += chunk) {
    const int np = std::min(chunk, n_pairs - p0);
    const int rows = np * g.S;
    const int nb = rows / kRB;
    int64_t* row_off = (int64_t*)ctx->scratch[4].get(sizeof(int64_t) * rows);
    int* blk_slot = (int*)ctx->scratch[5].get(sizeof(int) * nb);
    float* Z = (float*)ctx->scratch[6].get(sizeof(float) * (size_t)rows * g.H);
    float* L = (float*)ctx->scratch[7].get(sizeof(float) * (size_t)rows * g.C);
    k_l_pair_rows<<<nblk(rows, 256), 256, 0, ctx->stream>>>(g, np, d_pair_slot + p0,
                                                             d_pair_cam + p0, row_off, blk_slot);
    ECCO_LAUNCHED(ctx);
    if (ctx->cfg.math == ECCO_MATH_TC_BF16) {
      // tensor-core hidden layer: 128-row tiles that never straddle two
      // models (tiles are cut at slot changes of the 64-row pair blocks)
      std::vector<int> hslot(nb);
      ECCO_CUDA(ctx_memcpy(ctx, hslot.data(), blk_slot, sizeof(int) * nb, cudaMemcpyDeviceToHost, ctx->stream));
      ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
      std::vector<TcTile> tiles;
      for (int b = 0; b < nb;) {
        const int take = (b + 1 < nb && hslot[b + 1] == hslot[b]) ? 2 : 1;
        tiles.push_back({hslot[b], b * kRB, take * kRB, 0});
        b += take;
      }
      TcTile* d_tiles = (TcTile*)ctx->scratch[8].get(sizeof(TcTile) * tiles.size());
      ECCO_CUDA(ctx_memcpy(ctx, d_tiles, tiles.data(), sizeof(TcTile) * tiles.size(), cudaMemcpyHostToDevice, ctx->stream));
      if (g.H % 256 == 0) {  // bf16 against a W1^T shadow of the evaluated models
        std::vector<int> us(hslot);
        std::sort(us.begin(), us.end());
        us.erase(std::unique(us.begin(), us.end()), us.end());
        int* d_us = ctx->upload(14, us.data(), us.size());  // scratch 14: this use only
        uint16_t* w1t =
            (uint16_t*)ctx->train_scratch[9].get((size_t)ctx->cfg.max_jobs * g.H * g.F * 2);
        fused::shadow_w1t(ctx, d_us, (int)us.size(), ctx->d_w, ctx->n_params, w1t);
        tc::fwd_hidden_bf16(ctx, ctx->d_eval, row_off, d_tiles, (int)tiles.size(), nullptr, 0,
                            w1t, (size_t)ctx->cfg.max_jobs, ctx->d_w, ctx->n_params, Z,
                            (double)rows);
      } else {
        tc::fwd_hidden(ctx, ctx->d_eval, row_off, d_tiles, (int)tiles.size(), nullptr, 0, ctx->d_w,
                       ctx->n_params, Z, (double)rows);
      }
    } else {
      ECCO_TIMED(ctx, ECCO_KSTAT_EVAL_MATRIX, 2.0 * rows * g.F * g.H,
                 (double)rows * g.F * 2 + (double)g.F * g.H * 4,
                 launch_hidden_ffma(ctx, nb, g, ctx->d_eval, row_off, blk_slot,
                                    Gate{nullptr, 0, 1}, ctx->d_w, ctx->n_params, Z));
      ECCO_LAUNCHED(ctx);
    }
    // (C <= 16: 64-thread blocks of 16 classes, no idle class lanes)
    if (g.C <= 16)
      ECCO_TIMED(ctx, ECCO_KSTAT_EVAL_PAIRS, 2.0 * rows * g.H * g.C, (double)rows * g.H * 4,
                 (k_l_logits_t<64><<<dim3(rows / kRB, 1), 64, 0, ctx->stream>>>(
                     g, rows, blk_slot, Gate{nullptr, 0, 1}, ctx->d_w, ctx->n_params, Z, L)));
    else
      ECCO_TIMED(ctx, ECCO_KSTAT_EVAL_PAIRS, 2.0 * rows * g.H * g.C, (double)rows * g.H * 4,
                 (k_l_logits_t<128><<<dim3(rows / kRB, (g.C + 31) / 32), 128, 0, ctx->stream>>>(
                     g, rows, blk_slot, Gate{nullptr, 0, 1}, ctx->d_w, ctx->n_params, Z, L)));
    ECCO_LAUNCHED(ctx);
    k_l_count<<<nblk(rows, 256), 256, 0, ctx->stream>>>(g, np, L, ctx->d_eval_labels,
                                                         d_pair_cam + p0, d_counts + p0);
    ECCO_LAUNCHED(ctx);
  }
}

void eval_matrix(ecco_ctx* ctx, int n, const int* d_cams, int gj, const int* d_slots,
                 const uint8_t* d_mask, double* d_out, const int* h_slots) {
  if (n == 0 || gj == 0) return;
  if (ctx->fused_eval && h_slots) {
    // dense camera x group counts in one fused launch, then acc = count / S
    refresh_committed(ctx, h_slots, gj);
    std::vector<int> col(gj);
    for (int j = 0; j < gj; ++j) col[j] = j;
    int* d_col = ctx->upload(12, col.data(), gj);
    int* d_cnt = (int*)ctx->scratch[3].get(sizeof(int) * (size_t)n * gj);
    ECCO_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int) * (size_t)n * gj, ctx->stream));
    fused::eval_counts(ctx, ctx->sh_commit, ctx->d_w, ctx->n_params, n, d_cams, gj, d_slots, d_col,
                       0, nullptr, nullptr, gj, d_cnt, nullptr, (double)n * gj);
    fused::counts_to_acc(ctx, (size_t)n * gj, d_cnt, d_mask, d_out);
    return;
  }
  const size_t total = (size_t)n * gj;
  const char* et = getenv("ECCO_PAIR_TILE");
  const int tile_g = std::max(1, et ? atoi(et) : 64);
  if (!d_mask && fe_ok(ctx, dims(ctx)) && total <= (size_t)INT32_MAX) {
    // dense exact matrix: the pairs' order from the block index, no lists
    int* d_cnt = (int*)ctx->scratch[3].get(sizeof(int) * total);
    FEMatrix mx;
    mx.cams = d_cams;
    mx.slots = d_slots;
    mx.n = n;
    mx.gj = gj;
    mx.tile = tile_g;
    fe_launch(ctx, dims(ctx), (int)total, nullptr, nullptr, mx, d_cnt);
    fused::counts_to_acc(ctx, total, d_cnt, nullptr, d_out);
    return;
  }
  // host-side pair list (mask applied on the host copy when given)
  std::vector<int> slots(gj), cams(n);
  ECCO_CUDA(ctx_memcpy(ctx, slots.data(), d_slots, sizeof(int) * gj, cudaMemcpyDeviceToHost, ctx->stream));
  ECCO_CUDA(ctx_memcpy(ctx, cams.data(), d_cams, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<uint8_t> mask;
  if (d_mask) {
    mask.resize(total);
    ECCO_CUDA(ctx_memcpy(ctx, mask.data(), d_mask, total, cudaMemcpyDeviceToHost, ctx->stream));
  }
  ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  // Pairs in group tiles: tile_g groups (their W1 stays in L2: 64 x 512 KB
  // at the bench shape), cameras outer and the tile's groups inner, so each
  // camera's eval rows are read once per tile and each W1 once per window
  // rather than once per pair (camera-major order re-read the 500 groups'
  // 256 MB of W1 from HBM for every camera).  Counts are per pair and land
  // through po, so the order is invisible to the result.
  std::vector<int> ps, pc, po;
  ps.reserve(total);
  for (int j0 = 0; j0 < gj; j0 += tile_g)
    for (int i = 0; i < n; ++i)
      for (int j = j0; j < std::min(gj, j0 + tile_g); ++j) {
        const size_t o = (size_t)i * gj + j;
        if (d_mask && !mask[o]) continue;
        ps.push_back(slots[j]);
        pc.push_back(cams[i]);
        po.push_back((int)o);
      }
  if (d_mask) {
    k_l_fill_nan<<<nblk(total, 256), 256, 0, ctx->stream>>>(total, d_out);
    ECCO_LAUNCHED(ctx);
  }
  const int np = (int)ps.size();
  if (np == 0) return;
  int* d_ps = ctx->upload(0, ps.data(), np);
  int* d_pc = ctx->upload(1, pc.data(), np);
  int* d_po = ctx->upload(2, po.data(), np);
  int* d_cnt = (int*)ctx->scratch[3].get(sizeof(int) * np);
  pair_counts(ctx, np, d_ps, d_pc, d_cnt);
  k_l_matrix_out<<<nblk(np, 256), 256, 0, ctx->stream>>>(dims(ctx), np, d_cnt, d_po, d_out);
  ECCO_LAUNCHED(ctx);
}

void debug_logits(ecco_ctx* ctx, int n, const int* h_cams, int gj, const int* h_slots,
                  float* out) {
  const LDims g = dims(ctx);
  refresh_committed(ctx, h_slots, gj);
  std::vector<int> col(gj);
  for (int j = 0; j < gj; ++j) col[j] = j;
  int* d_cams = ctx->upload(11, h_cams, n);
  int* d_sl = ctx->upload(12, h_slots, gj);
  int* d_col = ctx->upload(13, col.data(), gj);
  const size_t nl = (size_t)n * g.S * gj * g.C;
  DevBuf cnt, lg;
  int* d_cnt = (int*)cnt.get(sizeof(int) * (size_t)n * gj);
  float* d_lg = (float*)lg.get(sizeof(float) * nl);
  ECCO_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int) * (size_t)n * gj, ctx->stream));
  fused::eval_counts(ctx, ctx->sh_commit, ctx->d_w, ctx->n_params, n, d_cams, gj, d_sl, d_col, 0,
                     nullptr, nullptr, gj, d_cnt, d_lg, (double)n * gj);
  ECCO_CUDA(ctx_memcpy(ctx, out, d_lg, sizeof(float) * nl, cudaMemcpyDeviceToHost, ctx->stream));
  ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
}

void eval_pairs(ecco_ctx* ctx, int n, const int* d_cams, const int* d_slots, double* d_out,
                const int* h_slots) {
  if (n == 0) return;
  if (ctx->fused_eval && h_slots) {
    refresh_committed(ctx, h_slots, n);
    int* d_cnt = (int*)ctx->scratch[3].get(sizeof(int) * n);
    pair_counts_fused(ctx, ctx->sh_commit, ctx->d_w, ctx->n_params, n, h_slots, d_slots, d_cams,
                      d_cnt);
    fused::counts_to_acc(ctx, (size_t)n, d_cnt, nullptr, d_out);
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  DevBuf cnt, idx;
  int* d_cnt = (int*)cnt.get(sizeof(int) * n);
  std::vector<int> po(n);
  for (int i = 0; i < n; ++i) po[i] = i;
  int* d_po = (int*)idx.get(sizeof(int) * n);
  ECCO_CUDA(ctx_memcpy(ctx, d_po, po.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
  pair_counts(ctx, n, d_slots, d_cams, d_cnt);
  k_l_matrix_out<<<nblk(n, 256), 256, 0, ctx->stream>>>(dims(ctx), n, d_cnt, d_po, d_out);
  ECCO_LAUNCHED(ctx);
  ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  cnt.release();
  idx.release();
}

void route_propose(ecco_ctx* ctx, int n, const int* d_cams, const double* d_req, int gj,
                   const int* d_slots, const uint8_t* d_mask, int* d_best, double* d_best_acc) {
  if (n == 0) return;
  double* M = nullptr;
  DevBuf tmp;
  if (gj > 0) {
    M = (double*)tmp.get(sizeof(double) * (size_t)n * gj);
    eval_matrix(ctx, n, d_cams, gj, d_slots, d_mask, M);
  }
  k_l_route<<<nblk((size_t)n * 32, 256), 256, 0, ctx->stream>>>(n, gj, 1, M, d_req, nullptr, d_best,
                                                                 d_best_acc);
  ECCO_LAUNCHED(ctx);
  ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  tmp.release();
}

static void member_pairs(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_mem_off,
                         const int* d_mem_cam, std::vector<int>& h_off, int** d_ps,
                         std::vector<int>* h_ps = nullptr) {
  h_off.resize(n_jobs + 1);
  std::vector<int> slots(n_jobs);
  ECCO_CUDA(ctx_memcpy(ctx, h_off.data(), d_mem_off, sizeof(int) * (n_jobs + 1), cudaMemcpyDeviceToHost, ctx->stream));
  ECCO_CUDA(ctx_memcpy(ctx, slots.data(), d_slots, sizeof(int) * n_jobs, cudaMemcpyDeviceToHost, ctx->stream));
  ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<int> ps(h_off[n_jobs]);
  for (int j = 0; j < n_jobs; ++j)
    for (int m = h_off[j]; m < h_off[j + 1]; ++m) ps[m] = slots[j];
  *d_ps = ctx->upload(0, ps.data(), ps.size());
  if (h_ps) *h_ps = std::move(ps);
  (void)d_mem_cam;
}

void eval_jobs(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_mem_off,
               const int* d_mem_cam, double* d_out) {
  if (n_jobs == 0) return;
  std::vector<int> off, hps;
  int* d_ps = nullptr;
  member_pairs(ctx, n_jobs, d_slots, d_mem_off, d_mem_cam, off, &d_ps, &hps);
  const int np = off[n_jobs];
  int* d_cnt = (int*)ctx->scratch[3].get(sizeof(int) * std::max(np, 1));
  if (np && ctx->fused_eval) {
    refresh_committed(ctx, hps.data(), np);
    pair_counts_fused(ctx, ctx->sh_commit, ctx->d_w, ctx->n_params, np, hps.data(), d_ps, d_mem_cam,
                      d_cnt);
  } else if (np) {
    pair_counts(ctx, np, d_ps, d_mem_cam, d_cnt);
  }
  k_l_job_mean<<<nblk(n_jobs, 128), 128, 0, ctx->stream>>>(dims(ctx), n_jobs, d_mem_off, d_cnt,
                                                            ctx->cfg.params.acc_floor, d_out, 1, 0);
  ECCO_LAUNCHED(ctx);
}

void trajectories(ecco_ctx* ctx, int n_jobs, const int* h_job_ids, const int* d_slots,
                  const int* d_job_ids, const int* h_steps, const int* d_src_off,
                  const int* d_src_cam, const double* d_src_frac, const int* d_mem_off,
                  const int* d_mem_cam, const int* d_micro_base, int window, int depth,
                  double* d_out) {
  (void)h_job_ids;
  if (n_jobs == 0) return;
  const LDims g = dims(ctx);
  const size_t np = ctx->n_params;
  const int T = ctx->cfg.max_depth;
  ECCO_REQUIRE(depth <= T, "depth exceeds max_depth");
  int max_steps = 0;
  for (int j = 0; j < n_jobs; ++j) max_steps = std::max(max_steps, h_steps[j]);
  int* d_steps = ctx->upload(1, h_steps, n_jobs);
  // member pairs for evaluate
  std::vector<int> off, hps;
  int* d_ps = nullptr;
  member_pairs(ctx, n_jobs, d_slots, d_mem_off, d_mem_cam, off, &d_ps, &hps);
  const int n_mem = off[n_jobs];
  int* d_cnt = (int*)ctx->scratch[3].get(sizeof(int) * std::max(n_mem, 1));
  // training scratch: rows = n_jobs * B
  // (the fused step keeps everything on chip: no row scratch)
  const int rows = ctx->fused_train ? 0 : n_jobs * g.B;
  const int nb = rows / kRB;
  DevBuf* ts = ctx->train_scratch;  // persistent across calls (no cudaMalloc per window)
  int64_t* row_off = rows ? (int64_t*)ts[0].get(sizeof(int64_t) * rows) : nullptr;
  int32_t* row_lab = rows ? (int32_t*)ts[1].get(sizeof(int32_t) * rows) : nullptr;
  int* blk_slot = rows ? (int*)ts[2].get(sizeof(int) * nb) : nullptr;
  float* Z = rows ? (float*)ts[3].get(sizeof(float) * (size_t)rows * g.H) : nullptr;
  float* L = rows ? (float*)ts[4].get(sizeof(float) * (size_t)rows * g.C) : nullptr;
  float* DL = rows ? (float*)ts[5].get(sizeof(float) * (size_t)rows * g.C) : nullptr;
  float* DH = rows ? (float*)ts[6].get(sizeof(float) * (size_t)rows * g.H) : nullptr;
  float* loss_rows = rows ? (float*)ts[7].get(sizeof(float) * rows) : nullptr;
  // tensor-core math with few head blocks (one group's chain: the K = H
  // logits loop is latency bound on a handful of SMs): split-K logits
  int head_ks = 1;
  if (rows && ctx->cfg.math == ECCO_MATH_TC_BF16 && !ctx->fused_train) {
    const int blocks = (rows / kRB) * ((g.C + 31) / 32);
    while (head_ks < 16 && blocks * head_ks * 2 <= 128 && (g.H / (head_ks * 2)) % kHT == 0)
      head_ks *= 2;
  }
  float* Lp = head_ks > 1 ? (float*)ts[10].get(sizeof(float) * (size_t)head_ks * rows * g.C)
                          : nullptr;
  // spec chain buffer per slot: T snapshots; train in place in snapshot t-1
  std::vector<int> slots(n_jobs);
  ECCO_CUDA(ctx_memcpy(ctx, slots.data(), d_slots, sizeof(int) * n_jobs, cudaMemcpyDeviceToHost, ctx->stream));
  ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<int> hb_slot(nb);
  const int rb_per_job = g.B / kRB;
  for (int j = 0; nb && j < n_jobs; ++j)
    for (int q = 0; q < rb_per_job; ++q) hb_slot[j * rb_per_job + q] = slots[j];
  if (nb)
    ECCO_CUDA(ctx_memcpy(ctx, blk_slot, hb_slot.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, ctx->stream));
  // the spec snapshots use a virtual "slot" base: wspec + slot * T * np + (t-1) * np
  const size_t spec_stride = (size_t)T * np;
  // tensor-core path: one 128-row tile (or the whole minibatch when B < 128)
  // per job and 128 rows
  const bool tc_math = ctx->cfg.math == ECCO_MATH_TC_BF16 && !ctx->fused_train;
  // 128-row minibatches with H a multiple of 256 run the forward in bf16
  // against a W1^T shadow the dW1 update keeps current (tc_kernels.cu)
  const bool tc_bf16 = tc_math && g.B % 128 == 0 && g.H % 256 == 0;
  uint16_t* w1t_train =
      tc_bf16 ? (uint16_t*)ts[8].get((size_t)ctx->cfg.max_jobs * g.H * g.F * 2) : nullptr;
  std::vector<TcTile> tiles;
  TcTile* d_tiles = nullptr;
  if (tc_math) {
    ECCO_REQUIRE(g.F % 128 == 0 && g.B % 32 == 0, "tensor-core path needs F % 128 == 0, B % 32 == 0");
    for (int j = 0; j < n_jobs; ++j)
      for (int r = 0; r < g.B; r += 128) tiles.push_back({slots[j], j * g.B + r, std::min(128, g.B - r), j});
    d_tiles = (TcTile*)ctx->scratch[9].get(sizeof(TcTile) * tiles.size());
    ECCO_CUDA(ctx_memcpy(ctx, d_tiles, tiles.data(), sizeof(TcTile) * tiles.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  // the per-micro-window evaluation plan and idle-job list, uploaded once
  PairsPlan spec_plan;
  const int* d_idle = nullptr;
  int n_idle = 0;
  if (n_mem && ctx->fused_eval) {
    spec_plan = plan_pairs(ctx, n_mem, hps.data(), 16, 17);
    std::vector<int> idle;
    for (int j = 0; j < n_jobs; ++j)
      if (h_steps[j] <= 0) idle.push_back(slots[j]);
    n_idle = (int)idle.size();
    d_idle = ctx->upload(18, idle.data(), idle.size());
  }
  // the wide chain's member evaluations: the general path, planned once
  GeneralPlan gen_plan;
  if (n_mem && !ctx->fused_eval && ctx->fused_train) gen_plan = plan_general(ctx, n_mem, hps.data());
  // acc[:, 0] from the committed models
  if (gen_plan.ok) {
    pair_counts_general_planned(ctx, gen_plan, ctx->d_w, ctx->n_params, d_ps, d_mem_cam, d_cnt);
  } else if (n_mem && ctx->fused_eval) {
    refresh_committed(ctx, hps.data(), n_mem);
    pair_counts_planned(ctx, ctx->sh_commit, ctx->d_w, ctx->n_params, spec_plan, d_ps, d_mem_cam,
                        d_cnt);
  } else if (n_mem) {
    pair_counts(ctx, n_mem, d_ps, d_mem_cam, d_cnt);
  }
  k_l_job_mean<<<nblk(n_jobs, 128), 128, 0, ctx->stream>>>(g, n_jobs, d_mem_off, d_cnt,
                                                            ctx->cfg.params.acc_floor, d_out, depth + 1, 0);
  ECCO_LAUNCHED(ctx);
  // Fused chains: the sampled rows of all `depth` micro-windows are drawn in
  // one launch, each micro-window's chain reads state t-1 and leaves state t
  // (no copy), and -- with a side stream -- the member evaluation of state t
  // runs beside the chain of state t+1 (the two alternate between the two
  // speculative shadows: chain t+2 rewrites the shadow eval t reads, so it
  // waits for it).
  // Serial mode -- one job on the fused chain with >= 2 micro-windows (the
  // exact replay's extension chains): every micro-window in ONE launch from
  // on-chip state (no per-micro-window setup, write-back of the starting
  // model or launch gap), then the member evaluations of all `depth`
  // snapshots as one batched pass over the snapshot pool's images.
  // Bit-identical to the per-micro-window launches (same arithmetic; the
  // masters round-trip exactly), tests/test_gpu_learned.py.
  // (wide chains: the planned general evaluation of all snapshots)
  const bool wide = ctx->fused_train && !fused::train_supported(ctx);
  // The oracle-exact math on its fused FFMA chain (ffma_chain.cu): one launch
  // per micro-window (or one per call in serial mode), the same arithmetic
  // as the per-step FFMA kernels below bit for bit
  const bool ffma_chain = !ctx->fused_train && ctx->cfg.math == ECCO_MATH_FFMA_EXACT &&
                          fused::ffma_chain_supported(ctx);
  if (ffma_chain) {
    fused::chain_rows(ctx, n_jobs, d_job_ids, d_steps, h_steps, d_src_off, d_src_cam, d_src_frac,
                      d_micro_base, depth, window, false);
    if (n_jobs == 1 && depth >= 2 && n_mem > 0 && h_steps[0] > 0 && !getenv("ECCO_NO_SERIAL_CHAIN")) {
      // serial: every micro-window in one launch, then the member
      // evaluations of all snapshots in one batched pass
      float* sbase = ctx->d_wspec + (size_t)slots[0] * spec_stride;
      fused::train_ffma(ctx, 1, d_slots, d_steps, h_steps, 0, depth, ctx->d_w, np, ctx->d_wspec,
                        spec_stride, 0, depth, np);
      const int n_pairs = n_mem * depth;
      int* d_vslot = (int*)ctx->scratch[21].get(sizeof(int) * n_pairs);
      int* d_vcam = (int*)ctx->scratch[22].get(sizeof(int) * n_pairs);
      int* d_vcnt = (int*)ctx->scratch[23].get(sizeof(int) * n_pairs);
      k_l_serial_pairs<<<nblk(n_pairs, 256), 256, 0, ctx->stream>>>(n_mem, depth, d_mem_cam, d_vslot,
                                                                    d_vcam);
      ECCO_LAUNCHED(ctx);
      float* saved = ctx->d_w;
      const size_t saved_np = ctx->n_params;
      ctx->d_w = sbase;  // snapshot u = "slot" u of the pair evaluation
      ctx->n_params = np;
      try {
        pair_counts(ctx, n_pairs, d_vslot, d_vcam, d_vcnt);
      } catch (...) {
        ctx->d_w = saved;
        ctx->n_params = saved_np;
        throw;
      }
      ctx->d_w = saved;
      ctx->n_params = saved_np;
      k_l_serial_mean<<<nblk(depth, 64), 64, 0, ctx->stream>>>(g, n_mem, depth, d_vcnt, d_out);
      ECCO_LAUNCHED(ctx);
      ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
      return;
    }
  }
  const bool serial = ctx->fused_train && n_jobs == 1 && depth >= 2 && n_mem > 0 &&
                      h_steps[0] > 0 && !getenv("ECCO_NO_SERIAL_CHAIN") &&
                      (ctx->fused_eval ? ctx->sh_pool.w1t != nullptr
                                       : gen_plan.ok && (size_t)n_mem * depth * g.S * g.H * 4 <= (256u << 20));
  if (serial) {
    fused::chain_rows(ctx, n_jobs, d_job_ids, d_steps, h_steps, d_src_off, d_src_cam, d_src_frac,
                      d_micro_base, depth, window);
    float* sbase = ctx->d_wspec + (size_t)slots[0] * spec_stride;  // snapshot t at sbase + (t-1) np
    fused::train_chain(ctx, nullptr, 1, d_slots, d_steps, h_steps, 0, depth, ctx->d_w, np,
                       ctx->d_wspec, spec_stride, 0, depth, np);
    const int n_pairs = n_mem * depth;
    int* d_vslot = (int*)ctx->scratch[21].get(sizeof(int) * n_pairs);
    int* d_vcam = (int*)ctx->scratch[22].get(sizeof(int) * n_pairs);
    int* d_vcnt = (int*)ctx->scratch[23].get(sizeof(int) * n_pairs);
    k_l_serial_pairs<<<nblk(n_pairs, 256), 256, 0, ctx->stream>>>(n_mem, depth, d_mem_cam, d_vslot,
                                                                  d_vcam);
    ECCO_LAUNCHED(ctx);
    std::vector<int> hv(n_pairs), us(depth);
    for (int i = 0; i < n_pairs; ++i) hv[i] = i / n_mem;
    for (int u = 0; u < depth; ++u) us[u] = u;
    if (!ctx->fused_eval) {
      const GeneralPlan vplan = plan_general(ctx, n_pairs, hv.data(), 24, 25);
      ECCO_REQUIRE(vplan.ok, "serial wide chain: evaluation plan");
      pair_counts_general_planned(ctx, vplan, sbase, np, d_vslot, d_vcam, d_vcnt);
    } else {
      const int* d_us = ctx->upload(24, us.data(), us.size());
      fused::refresh_shadow_dev(ctx, ctx->sh_pool, sbase, np, d_us, depth, d_us, depth);
      const PairsPlan vplan = plan_pairs(ctx, n_pairs, hv.data(), 25, 20);
      pair_counts_planned(ctx, ctx->sh_pool, sbase, np, vplan, d_vslot, d_vcam, d_vcnt);
    }
    k_l_serial_mean<<<nblk(depth, 64), 64, 0, ctx->stream>>>(g, n_mem, depth, d_vcnt, d_out);
    ECCO_LAUNCHED(ctx);
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  const bool side = ctx->fused_train && ctx->eval_stream && n_mem > 0 && (ctx->fused_eval || gen_plan.ok);
  if (ctx->fused_train)
    fused::chain_rows(ctx, n_jobs, d_job_ids, d_steps, h_steps, d_src_off, d_src_cam, d_src_frac,
                      d_micro_base, depth, window);
  if (side) {  // the side stream sees everything enqueued so far (acc[:, 0], plans, rows)
    ECCO_CUDA(cudaEventRecord(ctx->ev_chain[0], ctx->stream));
    ECCO_CUDA(cudaStreamWaitEvent(ctx->eval_stream, ctx->ev_chain[0], 0));
  }
  for (int t = 1; t <= depth; ++t) {
    // weights of state t are addressed as wbase + slot * spec_stride
    float* wt = ctx->d_wspec + (size_t)(t - 1) * np;
    if (ctx->fused_train) {  // one launch: every job's whole micro-window on chip
      const float* src = t == 1 ? ctx->d_w : ctx->d_wspec + (size_t)(t - 2) * np;
      Shadow* sh = (t & 1) ? &ctx->sh_spec : &ctx->sh_spec2;
      if (side && t >= 3) ECCO_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_eval[t & 1], 0));
      fused::train_chain(ctx, sh, n_jobs, d_slots, d_steps, h_steps, t - 1, depth, src,
                         t == 1 ? np : spec_stride, wt, spec_stride, t - 1);
      if (side) {
        ECCO_CUDA(cudaEventRecord(ctx->ev_chain[t & 1], ctx->stream));
        ECCO_CUDA(cudaStreamWaitEvent(ctx->eval_stream, ctx->ev_chain[t & 1], 0));
        cudaStream_t main_stream = ctx->stream;
        ctx->stream = ctx->eval_stream;  // the evaluation of state t, on the side stream
        try {
          if (gen_plan.ok) {  // wide chains: the planned general evaluation of snapshot t
            pair_counts_general_planned(ctx, gen_plan, wt, spec_stride, d_ps, d_mem_cam, d_cnt);
          } else {
            // (the narrow chain wrote its trained jobs' W1^T images itself)
            if (wide)
              fused::refresh_shadow_dev(ctx, *sh, wt, spec_stride, d_slots, n_jobs, d_slots, n_jobs);
            else
              fused::refresh_shadow_dev(ctx, *sh, wt, spec_stride, d_slots, n_jobs, d_idle, n_idle);
            pair_counts_planned(ctx, *sh, wt, spec_stride, spec_plan, d_ps, d_mem_cam, d_cnt);
          }
          k_l_job_mean<<<nblk(n_jobs, 128), 128, 0, ctx->stream>>>(
              g, n_jobs, d_mem_off, d_cnt, ctx->cfg.params.acc_floor, d_out, depth + 1, t);
          ECCO_LAUNCHED(ctx);
        } catch (...) {
          ctx->stream = main_stream;
          throw;
        }
        ctx->stream = main_stream;
        ECCO_CUDA(cudaEventRecord(ctx->ev_eval[t & 1], ctx->eval_stream));
        continue;
      }
    } else if (ffma_chain) {  // state t-1 -> state t in one launch
      const float* src = t == 1 ? ctx->d_w : ctx->d_wspec + (size_t)(t - 2) * np;
      fused::train_ffma(ctx, n_jobs, d_slots, d_steps, h_steps, t - 1, depth, src,
                        t == 1 ? np : spec_stride, wt, spec_stride, t - 1);
    } else {
      // state t starts as a copy of state t-1
      if (t == 1)
        k_l_copy_weights<<<dim3(64, n_jobs), 256, 0, ctx->stream>>>(n_jobs, d_slots, ctx->d_w, np,
                                                                    0, ctx->d_wspec, spec_stride, 0,
                                                                    np, nullptr);
      else
        k_l_copy_weights<<<dim3(64, n_jobs), 256, 0, ctx->stream>>>(
            n_jobs, d_slots, ctx->d_wspec, spec_stride, (size_t)(t - 2) * np, ctx->d_wspec,
            spec_stride, (size_t)(t - 1) * np, np, nullptr);
      ECCO_LAUNCHED(ctx);
    }
    if (tc_bf16 && !ctx->fused_train) fused::shadow_w1t(ctx, d_slots, n_jobs, wt, spec_stride, w1t_train);
    for (int step = 0; step < (ctx->fused_train || ffma_chain ? 0 : max_steps); ++step) {
      const Gate gate{d_steps, step, g.B};
      int live = 0;
      for (int j = 0; j < n_jobs; ++j) live += step < h_steps[j];
      const double lrows = (double)live * g.B;
      k_l_sample<<<nblk(rows, 256), 256, 0, ctx->stream>>>(
          g, ctx->cfg.seed, n_jobs, d_job_ids, d_steps, d_src_off, d_src_cam, d_src_frac,
          d_micro_base, window, t - 1, step, ctx->d_labels, row_off, row_lab);
      ECCO_LAUNCHED(ctx);
      if (tc_bf16) {
        tc::fwd_hidden_bf16(ctx, ctx->d_frames, row_off, d_tiles, (int)tiles.size(), d_steps, step,
                            w1t_train, (size_t)ctx->cfg.max_jobs, wt, spec_stride, Z, lrows);
      } else if (tc_math) {
        tc::fwd_hidden(ctx, ctx->d_frames, row_off, d_tiles, (int)tiles.size(), d_steps, step, wt,
                       spec_stride, Z, lrows);
      } else {
        ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_STEP, 2.0 * lrows * g.F * g.H,
                   lrows * g.F * 2 + (double)live * g.F * g.H * 4,
                   launch_hidden_ffma(ctx, nb, g, ctx->d_frames, row_off, blk_slot, gate, wt,
                                      spec_stride, Z));
        ECCO_LAUNCHED(ctx);
      }
      ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_HEAD, 8.0 * lrows * g.H * g.C, lrows * g.H * 12,
                 ((head_ks > 1
                       ? (k_l_logits_t<128><<<dim3(rows / kRB, (g.C + 31) / 32, head_ks), 128, 0,
                                         ctx->stream>>>(g, rows, blk_slot, gate, wt, spec_stride,
                                                        Z, Lp, g.H / head_ks),
                          k_l_logits_sum<<<nblk((size_t)rows * g.C, 256), 256, 0, ctx->stream>>>(
                              g, rows, head_ks, blk_slot, gate, wt, spec_stride, Lp, L))
                       : k_l_logits_t<128><<<dim3(rows / kRB, (g.C + 31) / 32), 128, 0, ctx->stream>>>(
                             g, rows, blk_slot, gate, wt, spec_stride, Z, L)),
                  (k_l_softmax_grad<<<nblk(rows, 128), 128, 0, ctx->stream>>>(
                      g, rows, gate, L, row_lab, DL, loss_rows)),
                  (k_l_dh_t<<<dim3(rows / kRB, g.H / 64), 128, 0, ctx->stream>>>(
                      g, rows, blk_slot, gate, wt, spec_stride, Z, DL, DH)),
                  (k_l_update2_t<<<dim3(n_jobs, g.H / 64, (g.C + 31) / 32), 128, 0,
                                   ctx->stream>>>(g, n_jobs, d_slots, d_steps, step, wt,
                                                  spec_stride, Z, DL))));
      ctx->launches += 3;
      ECCO_LAUNCHED(ctx);
      if (tc_math) {
        tc::dw1_update(ctx, ctx->d_frames, row_off, d_slots, d_steps, step, n_jobs, wt, spec_stride,
                       DH, live, w1t_train);
      } else {
        ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_DW1, 2.0 * lrows * g.F * g.H,
                   (double)live * (g.B * g.F * 2.0 + g.B * g.H * 4.0 + 2.0 * g.F * g.H * 4),
                   (k_l_update1_ffma<<<dim3(g.F / 64, g.H / kHB, n_jobs), 256, 0, ctx->stream>>>(
                       g, d_slots, d_steps, step, ctx->d_frames, row_off, wt, spec_stride, DH)));
        ECCO_LAUNCHED(ctx);
      }
      k_l_update_b1<<<nblk((size_t)n_jobs * g.H, 256), 256, 0, ctx->stream>>>(
          g, n_jobs, d_slots, d_steps, step, wt, spec_stride, DH);
      ECCO_LAUNCHED(ctx);
      k_l_loss_mean<<<nblk(n_jobs, 128), 128, 0, ctx->stream>>>(
          g, n_jobs, d_slots, d_steps, step, loss_rows, ctx->d_losses, T, t - 1);
      ECCO_LAUNCHED(ctx);
    }
    // evaluate state t
    if (n_mem && ctx->fused_eval) {
      // the chain wrote the W1^T image of every job it trained: only idle
      // jobs' images are rebuilt (all of them on the unfused path)
      fused::refresh_shadow_dev(ctx, ctx->sh_spec, wt, spec_stride, d_slots, n_jobs,
                                ctx->fused_train && !wide ? d_idle : d_slots,
                                ctx->fused_train && !wide ? n_idle : n_jobs);
      pair_counts_planned(ctx, ctx->sh_spec, wt, spec_stride, spec_plan, d_ps, d_mem_cam, d_cnt);
      k_l_job_mean<<<nblk(n_jobs, 128), 128, 0, ctx->stream>>>(g, n_jobs, d_mem_off, d_cnt,
                                                                ctx->cfg.params.acc_floor, d_out, depth + 1, t);
      ECCO_LAUNCHED(ctx);
      continue;
    }
    if (gen_plan.ok) {  // wide chains: no host round trip between micro-windows
      pair_counts_general_planned(ctx, gen_plan, wt, spec_stride, d_ps, d_mem_cam, d_cnt);
      k_l_job_mean<<<nblk(n_jobs, 128), 128, 0, ctx->stream>>>(g, n_jobs, d_mem_off, d_cnt,
                                                                ctx->cfg.params.acc_floor, d_out, depth + 1, t);
      ECCO_LAUNCHED(ctx);
      continue;
    }
    // (exact path) temporarily point the pair evaluation at the snapshot
    float* saved = ctx->d_w;
    const size_t saved_np = ctx->n_params;
    ctx->d_w = wt;
    ctx->n_params = spec_stride;
    try {
      if (n_mem) pair_counts(ctx, n_mem, d_ps, d_mem_cam, d_cnt);
    } catch (...) {
      ctx->d_w = saved;
      ctx->n_params = saved_np;
      throw;
    }
    ctx->d_w = saved;
    ctx->n_params = saved_np;
    k_l_job_mean<<<nblk(n_jobs, 128), 128, 0, ctx->stream>>>(g, n_jobs, d_mem_off, d_cnt,
                                                              ctx->cfg.params.acc_floor, d_out, depth + 1, t);
    ECCO_LAUNCHED(ctx);
  }
  if (side) {  // the context stream (the caller's copy of d_out) waits for the last evaluation
    ECCO_CUDA(cudaEventRecord(ctx->ev_eval[0], ctx->eval_stream));
    ECCO_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_eval[0], 0));
  }
  ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
}

void commit(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_granted) {
  if (n_jobs == 0) return;
  const size_t np = ctx->n_params;
  const size_t spec_stride = (size_t)ctx->cfg.max_depth * np;
  k_l_copy_weights<<<dim3(64, n_jobs), 256, 0, ctx->stream>>>(n_jobs, d_slots, ctx->d_wspec,
                                                              spec_stride, 0, ctx->d_w, np, 0, np,
                                                              d_granted);
  ECCO_LAUNCHED(ctx);
}

void route_matrix(ecco_ctx* ctx, int n, int gb, int n_blocks, const double* d_M,
                  const double* d_req, const int* d_ids, int* d_best, double* d_best_acc) {
  if (n == 0) return;
  k_l_route<<<nblk((size_t)n * 32, 256), 256, 0, ctx->stream>>>(n, gb, n_blocks, d_M, d_req,
                                                                 d_ids, d_best, d_best_acc);
  ECCO_LAUNCHED(ctx);
}

void sample_indices(ecco_ctx* ctx, int job_id, int n_src, const int* d_src_cam,
                    const double* d_src_frac, int window, int micro, int step, int* d_cam,
                    int* d_frame) {
  const LDims g = dims(ctx);
  k_l_sample_debug<<<nblk(g.B, 128), 128, 0, ctx->stream>>>(g, ctx->cfg.seed, job_id, n_src,
                                                             d_src_cam, d_src_frac, window, micro,
                                                             step, d_cam, d_frame);
  ECCO_LAUNCHED(ctx);
}

}  // namespace lbackend
