// Fused FP32 (FFMA) SGD chain of the learned backend: the ORACLE-EXACT math
// (ECCO_MATH_FFMA_EXACT) in one launch per micro-window -- every job's
// steps[j] SGD steps of gather, forward, softmax cross-entropy, backward and
// update -- on one thread-block cluster per job, instead of nine kernels per
// SGD step on a handful of SMs (learned_kernels.cu's general FFMA path,
// ~115 us per step of a single job's serial chain).
//
// Bit-exact with oracle/ecco_oracle.c orc_sgd_step (and so with the general
// FFMA path): every output is ONE thread's fmaf chain in the oracle's order --
//   Z[s][h]     = (fmaf over f ascending of x[s][f] W1[f][h], from 0) + b1[h]
//   L[s][c]     = (fmaf over k ascending of relu(Z[s][k]) W2[k][c]) + b2[c]
//   softmax     = k_l_softmax_grad's sequence (max, ascending sum of ecco_expf,
//                 IEEE divide, (p - onehot) * (1/B))
//   dH[s][k]    = Z[s][k] > 0 ? fmaf over c ascending of dL[s][c] W2[k][c] : 0
//                 (pre-update W2)
//   W2[k][c]   <- fmaf(-lr, fmaf over s ascending of relu(Z[s][k]) dL[s][c], W2)
//   b2[c]      <- fmaf(-lr, sum over s ascending of dL[s][c], b2)
//   W1[f][h]   <- fmaf(-lr, fmaf over s ascending of x[s][f] dH[s][h], W1)
//   b1[h]      <- fmaf(-lr, sum over s ascending of dH[s][h], b1)
// -- so the tiling below changes where each chain runs, never its order.
//
// Cluster of H/16 CTAs (16 for H = 256: a non-portable cluster); CTA r owns
// hidden units [16r, 16r+16) and rows [r RP, r RP + RP) (RP = 128 / cluster):
//   smem    X (the step's 128 sampled rows, bf16, 16-byte chunks XOR-swizzled
//           by row quad), the fp32 W1 master slice [F][16] (resident for the
//           whole micro-window), a full copy of W2 (rows padded to C + 1:
//           conflict-free both along k and along c), b1 slice, b2, the own
//           pre-activations Z[128][16], and the exchange buffers below
//   step    gather X (cp.async) -> Z of own units (FFMA, 2 rows x 4 units per
//           thread, all warps) -> relu rows to the row owners (DSMEM) -> cluster barrier
//           -> owner: logits of its rows over all H, softmax, dL (to every
//           CTA), dH of its rows for all units (to each unit's CTA), row
//           losses (to CTA 0) -> cluster barrier -> own W2 rows (to every
//           CTA's copy), b2, b1 (warps 4-7) beside W1 (FFMA, 8 features x 8
//           units per thread, warps 0-3)
// Two cluster barriers per step; everything else is CTA-local.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "ctx.cuh"
#include "learned_common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

constexpr int kB = 128;        // minibatch rows
constexpr int kHS = 16;        // hidden units per CTA
constexpr int kC = 16;         // classes
constexpr int kThreads = 256;  // 8 warps
constexpr int kMaxNC = 16;

struct FfmaArgs {
  LDims g;
  const int* slots;
  const int* steps;
  const int32_t* rows;  // [job][row steps][kB] frame-table row of every sampled frame (chain_rows)
  const int32_t* labs;  // ... and its label
  int row_step0, rows_T;
  const uint16_t* frames;
  const float* wsrc;  // fp32 models the micro-window starts from (W1 [F][H])
  size_t wsrc_stride;
  float* wbase;  // ... and where it leaves them (a snapshot; may equal wsrc)
  size_t wstride;
  float* losses;
  int loss_T, loss_t;
  // serial mode (n_micro_launch > 1, one job): micro-window u's model is
  // written to wbase + u * wmicro and its loss to loss_t + u
  int n_micro_launch;
  size_t wmicro;
  int trace;
};

struct FLayout {
  uint32_t x, w1, w2, b1, b2, z, rrecv, dl, dh, lown, loss, rows, total;
};

__host__ __device__ inline FLayout flayout(int F, int H, int nc) {
  FLayout L{};
  const int rp = kB / nc;
  uint32_t o = 0;
  L.x = o;  // [128][F] bf16, 16-byte chunk j of row s at j ^ ((s >> 2) & 7)
  o += (uint32_t)kB * F * 2u;
  L.w1 = o;  // [F][16] fp32
  o += (uint32_t)F * kHS * 4u;
  L.w2 = o;  // [H][C + 1] fp32 (full copy)
  o += (uint32_t)H * (kC + 1) * 4u;
  o = (o + 15u) & ~15u;
  L.b1 = o;
  o += kHS * 4u;
  L.b2 = o;
  o += kC * 4u;
  L.z = o;  // [128][16] fp32 own pre-activations
  o += kB * kHS * 4u;
  L.rrecv = o;  // [rp][H] fp32 relu rows of the owned rows, all units
  o += (uint32_t)rp * H * 4u;
  L.dl = o;  // [128][C] fp32 dL of every row
  o += kB * kC * 4u;
  L.dh = o;  // [128][16] fp32 dH of own units, every row
  o += kB * kHS * 4u;
  L.lown = o;  // [rp][C] logits / dL of the owned rows
  o += (uint32_t)rp * kC * 4u;
  L.loss = o;  // [128] row losses (CTA 0)
  o += kB * 4u;
  L.rows = o;  // [2][128] frame-table rows of this step and the next
  o += 2u * kB * 4u;
  L.total = o;
  return L;
}

__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

// Byte offset of bf16 element (s, f) in the swizzled X tile (row = F * 2 bytes).
__device__ __forceinline__ uint32_t xoff(int F, int s, int f) {
  const uint32_t chunk = (uint32_t)(f >> 3) ^ (uint32_t)((s >> 2) & 7);
  return (uint32_t)s * (uint32_t)F * 2u + (chunk << 4) + (uint32_t)(f & 7) * 2u;
}

// 4 consecutive bf16 features (f % 4 == 0) of row s as fp32 (exact).
__device__ __forceinline__ void ld_x4(const uint8_t* xs, int F, int s, int f, float (&x)[4]) {
  const uint2 v = *reinterpret_cast<const uint2*>(xs + xoff(F, s, f));
  x[0] = __uint_as_float(v.x << 16);
  x[1] = __uint_as_float(v.x & 0xFFFF0000u);
  x[2] = __uint_as_float(v.y << 16);
  x[3] = __uint_as_float(v.y & 0xFFFF0000u);
}

// [step][point] clock64 of CTA 0, steps 0-3 (ECCO_FFMA_TRACE)
__device__ long long g_ffma_trace[4 * 16];
// (compiled in only with -DECCO_FFMA_TRACE_BUILD: the clock reads stall the
// warp that takes them, measurably, even when the stamp is not stored)
#ifdef ECCO_FFMA_TRACE_BUILD
#define FTS(k)                                                                              \
  do {                                                                                      \
    if (a.trace && blockIdx.x == 0 && tid == 0 && t < 4) g_ffma_trace[t * 16 + (k)] = clock64(); \
  } while (0)
#else
#define FTS(k) \
  do {         \
  } while (0)
#endif

// Packed FP32 FMA (fma.rn.f32x2, sm_100): two IEEE fmaf in one instruction.
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

template <int NC, int F>
__global__ void __launch_bounds__(kThreads, 1) k_train_ffma(FfmaArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int RP = kB / NC;
  const int H = a.g.H;
  constexpr int C = kC;
  constexpr int CP = kC + 1;  // padded W2 row
  const FLayout L = flayout(F, H, NC);
  uint8_t* xs = smem + L.x;
  float* w1s = reinterpret_cast<float*>(smem + L.w1);
  float* w2s = reinterpret_cast<float*>(smem + L.w2);
  float* b1s = reinterpret_cast<float*>(smem + L.b1);
  float* b2s = reinterpret_cast<float*>(smem + L.b2);
  float* zs = reinterpret_cast<float*>(smem + L.z);
  float* rrecv = reinterpret_cast<float*>(smem + L.rrecv);
  float* dls = reinterpret_cast<float*>(smem + L.dl);
  float* dhs = reinterpret_cast<float*>(smem + L.dh);
  float* lown = reinterpret_cast<float*>(smem + L.lown);
  float* lossv = reinterpret_cast<float*>(smem + L.loss);
  int32_t* rowbuf = reinterpret_cast<int32_t*>(smem + L.rows);

  const uint32_t r = cluster_ctarank();
  const int j = blockIdx.x / NC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int slot = a.slots[j];
  const int nsteps = a.steps[j];
  const int h0 = (int)r * kHS;
  const float lr = a.g.lr;

  // ---------------------------------------------------------- setup --
  {
    const float* src = a.wsrc + (size_t)slot * a.wsrc_stride;
    for (int e = tid; e < F * kHS; e += kThreads) w1s[e] = src[(size_t)(e / kHS) * H + h0 + e % kHS];
    const float* b1 = src + (size_t)F * H;
    const float* W2 = b1 + H;
    const float* b2 = W2 + (size_t)H * C;
    for (int e = tid; e < H * C; e += kThreads) w2s[(e / C) * CP + e % C] = W2[e];
    if (tid < kHS) b1s[tid] = b1[h0 + tid];
    if (tid < C) b2s[tid] = b2[tid];
  }
  __syncthreads();

  // every CTA of the cluster is running before any DSMEM store reaches it
  cluster_sync();
  const uint32_t rrecv_a = smem_u32(rrecv), dl_a = smem_u32(dls), dh_a = smem_u32(dhs);
  const uint32_t loss_a = smem_u32(lossv), w2_a = smem_u32(w2s);
  const int total = nsteps * a.n_micro_launch;
  for (int t = 0; t < total; ++t) {
    const int u = t / (nsteps > 0 ? nsteps : 1);
    const size_t rstep = (size_t)j * a.rows_T + a.row_step0 + t;
    // this step's frame-table rows were staged in shared memory during the
    // previous step (the first step's here); the next step's are staged now
    // and used after the end-of-step barrier
    const int32_t* rows = rowbuf + (t & 1) * kB;
    if (t == 0) {
      if (tid < kB) rowbuf[tid] = a.rows[rstep * kB + tid];
      __syncthreads();
    }

    // ------------------------------------------------------ gather X --
    FTS(0);
    // the next step's frame-table rows: loaded now, stored after the forward
    const int32_t next_row =
        warp >= 4 && t + 1 < total ? __ldg(a.rows + (rstep + 1) * kB + tid - 128) : 0;
    {
      const int cpr = F / 8;  // 16-byte chunks per row
      for (int e = tid; e < kB * cpr; e += kThreads) {
        const int s = e / cpr, ch = e % cpr;
        cp_async16(xs + xoff(F, s, ch * 8), a.frames + (size_t)rows[s] * F + ch * 8);
      }
      cp_async_wait_all();
    }
    __syncthreads();
    // ------------------------------ Z = X.W1 + b1 of the own 16 units --
    FTS(1);
    // all 8 warps: warp w owns units [4 (w & 3), +4) (warp-uniform: the W1
    // loads broadcast), lane l rows 4l + 2 (w >> 2) + {0, 1}; 8 features per
    // iteration, X by one 16-byte load per row (the (s >> 2) & 7 chunk
    // swizzle keeps each quarter-warp's 8 rows on distinct banks).  2 x 4
    // outputs per thread, two warps per scheduler to hide the shared-load
    // latency (one warp per scheduler left it exposed).
    {
      const int hq = (warp & 3) * 4, s0 = 4 * lane + 2 * (warp >> 2);
      float2 ac[2][2] = {};  // (row, unit pair): fma.rn.f32x2, each lane an fmaf chain
#pragma unroll 2
      for (int f = 0; f < F; f += 8) {
        uint32_t px[2][4];
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2) {
          const uint4 v = *reinterpret_cast<const uint4*>(xs + xoff(F, s0 + r2, f));
          px[r2][0] = v.x;
          px[r2][1] = v.y;
          px[r2][2] = v.z;
          px[r2][3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 w = *reinterpret_cast<const float4*>(w1s + (f + i) * kHS + hq);
          const float2 wa = make_float2(w.x, w.y), wb = make_float2(w.z, w.w);
          float xs2[2];
#pragma unroll
          for (int r2 = 0; r2 < 2; ++r2) {
            const uint32_t pw = px[r2][i >> 1];
            xs2[r2] = __uint_as_float(i & 1 ? pw & 0xFFFF0000u : pw << 16);
          }
#pragma unroll
          for (int r2 = 0; r2 < 2; ++r2)  // wa, then wb, in the operand reuse cache
            ac[r2][0] = fma2(make_float2(xs2[r2], xs2[r2]), wa, ac[r2][0]);
#pragma unroll
          for (int r2 = 0; r2 < 2; ++r2)
            ac[r2][1] = fma2(make_float2(xs2[r2], xs2[r2]), wb, ac[r2][1]);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int s = s0 + i;
        float z[4], rl[4];
        const float av[4] = {ac[i][0].x, ac[i][0].y, ac[i][1].x, ac[i][1].y};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          z[q] = __fadd_rn(av[q], b1s[hq + q]);
          rl[q] = z[q] > 0.0f ? z[q] : 0.0f;
        }
        *reinterpret_cast<float4*>(zs + s * kHS + hq) = make_float4(z[0], z[1], z[2], z[3]);
        // relu row piece -> the row's owner, at its units' columns
        const uint32_t dst = rrecv_a + (uint32_t)(((s % RP) * H + h0 + hq) * 4);
        st_cluster_v4(mapa_shared(dst, (uint32_t)(s / RP)), rl[0], rl[1], rl[2], rl[3]);
      }
    }
    if (warp >= 4 && t + 1 < total)  // the next step's rows (loaded before the gather)
      rowbuf[((t + 1) & 1) * kB + tid - 128] = next_row;
    FTS(2);
    cluster_sync();  // every owned row's relu values are in
    FTS(3);
    // ------------------------------------------- owner: logits, dL, dH --
    {
      const int rb = (int)r * RP;  // first owned row
      for (int o = tid; o < RP * C; o += kThreads) {
        const int sl = o / C, c = o % C;
        const float* rr = rrecv + sl * H;
        float acc = 0.0f;
#pragma unroll 8
        for (int k = 0; k < H; ++k) acc = __fmaf_rn(rr[k], w2s[k * CP + c], acc);
        lown[sl * C + c] = __fadd_rn(acc, b2s[c]);
      }
      __syncthreads();
      // softmax cross-entropy of the owned rows (k_l_softmax_grad's
      // sequence): one half-warp per row, lane c holds class c; the max and
      // the ascending sum are formed in the same order by every lane
      for (int o = tid; o < RP * C; o += kThreads) {
        const int sl = o / C, c = o % C;
        const unsigned hm = 0xFFFFu << (lane & 16);
        const float* l = lown + sl * C;
        float m = l[0];
#pragma unroll
        for (int cc = 1; cc < C; ++cc) m = l[cc] > m ? l[cc] : m;
        const float lc = l[c];
        const float e = ecco_expf(__fsub_rn(lc, m));
        float sum = 0.0f;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) sum = __fadd_rn(sum, __shfl_sync(hm, e, cc, 16));
        const float invB = __fdiv_rn(1.0f, (float)kB);
        const int y = a.labs[rstep * kB + rb + sl];
        const float p = __fdiv_rn(e, sum);
        const float dl = __fmul_rn(__fsub_rn(p, c == y ? 1.0f : 0.0f), invB);
        const float ly = l[y];
        __syncwarp(hm);
        lown[sl * C + c] = dl;
        const uint32_t dst = dl_a + (uint32_t)(((rb + sl) * C + c) * 4);
        for (uint32_t d = 0; d < (uint32_t)NC; ++d) st_cluster_f32(mapa_shared(dst, d), dl);
        if (c == 0)
          st_cluster_f32(mapa_shared(loss_a + (uint32_t)((rb + sl) * 4), 0u),
                         logf(sum) - (ly - m));
      }
      __syncthreads();
      // dH of the owned rows for every unit (pre-update W2), to the unit's CTA
      for (int sl = warp; sl < RP; sl += kThreads / 32) {
        float dlr[C];  // (registers: the DSMEM stores below clobber memory)
#pragma unroll
        for (int c = 0; c < C; ++c) dlr[c] = lown[sl * C + c];
        const float* rr = rrecv + sl * H;
        for (int k = lane; k < H; k += 32) {
          float acc = 0.0f;
#pragma unroll
          for (int c = 0; c < C; ++c) acc = __fmaf_rn(dlr[c], w2s[k * CP + c], acc);
          const float dh = rr[k] > 0.0f ? acc : 0.0f;
          st_cluster_f32(mapa_shared(dh_a + (uint32_t)(((rb + sl) * kHS + k % kHS) * 4),
                                     (uint32_t)(k / kHS)),
                         dh);
        }
      }
    }
    FTS(4);
    cluster_sync();  // every row's dL and every own unit's dH are in
    FTS(5);
    // ------------------------------------------------------- updates --
    {
      // warps 0-3: W1 += -lr X^T dH, 8 features x 8 units per thread (rows
      // ascending); warps 4-7 meanwhile: the own W2 rows (two elements per
      // thread, to every CTA's copy), b2 and the own b1 (rows ascending)
      if (warp < 4) {
        const int hq = (tid & 1) * 8;
        for (int fb = tid >> 1; fb < F / 8; fb += 64) {
          const int f0 = fb * 8;
          float2 acc[8][4] = {};  // (feature, unit pair)
#pragma unroll 2
          for (int s = 0; s < kB; ++s) {
            const uint4 v = *reinterpret_cast<const uint4*>(xs + xoff(F, s, f0));
            const uint32_t pv[4] = {v.x, v.y, v.z, v.w};
            const float4 d0 = *reinterpret_cast<const float4*>(dhs + s * kHS + hq);
            const float4 d1 = *reinterpret_cast<const float4*>(dhs + s * kHS + hq + 4);
            const float2 d[4] = {make_float2(d0.x, d0.y), make_float2(d0.z, d0.w),
                                 make_float2(d1.x, d1.y), make_float2(d1.z, d1.w)};
            float xv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              xv[i] = __uint_as_float(i & 1 ? pv[i >> 1] & 0xFFFF0000u : pv[i >> 1] << 16);
#pragma unroll
            for (int q = 0; q < 4; ++q)  // d pair in the operand reuse cache across features
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i][q] = fma2(make_float2(xv[i], xv[i]), d[q], acc[i][q]);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float* w = w1s + (f0 + i) * kHS + hq + 2 * q;
              w[0] = __fmaf_rn(-lr, acc[i][q].x, w[0]);
              w[1] = __fmaf_rn(-lr, acc[i][q].y, w[1]);
            }
        }
      } else {
        const int u2 = tid - 128;  // 0..127: W2 elements u2 and u2 + 128
        float aw[2] = {0.0f, 0.0f}, ab = 0.0f;
        const int kl0 = u2 / C, kl1 = (u2 + 128) / C, cw = u2 % C;
#pragma unroll 8
        for (int s = 0; s < kB; ++s) {
          const float z0 = zs[s * kHS + kl0], z1 = zs[s * kHS + kl1], g = dls[s * C + cw];
          aw[0] = __fmaf_rn(z0 > 0.0f ? z0 : 0.0f, g, aw[0]);
          aw[1] = __fmaf_rn(z1 > 0.0f ? z1 : 0.0f, g, aw[1]);
          if (u2 < C) ab = __fadd_rn(ab, g);
          else if (u2 >= 32 && u2 < 32 + kHS) ab = __fadd_rn(ab, dhs[s * kHS + u2 - 32]);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = h0 + (e ? kl1 : kl0);
          const float w = __fmaf_rn(-lr, aw[e], w2s[k * CP + cw]);
          const uint32_t wa = w2_a + (uint32_t)((k * CP + cw) * 4);
          for (uint32_t d = 0; d < (uint32_t)NC; ++d) st_cluster_f32(mapa_shared(wa, d), w);
        }
        if (u2 < C) b2s[u2] = __fmaf_rn(-lr, ab, b2s[u2]);
        else if (u2 >= 32 && u2 < 32 + kHS) b1s[u2 - 32] = __fmaf_rn(-lr, ab, b1s[u2 - 32]);
      }
      if (r == 0 && tid == 64 && ((t + 1) % nsteps == 0)) {  // the micro-window's last step loss
        double s = 0.0;
        for (int i = 0; i < kB; ++i) s += lossv[i];
        a.losses[(size_t)slot * a.loss_T + a.loss_t + u] = (float)(s / kB);
      }
    }
    __syncthreads();
    FTS(6);
    // ----------------------------------------- snapshot at micro-window end --
    if ((t + 1) % nsteps == 0 && (t + 1) < total) {
      float* dst = a.wbase + (size_t)slot * a.wstride + (size_t)u * a.wmicro;
      for (int e = tid; e < F * kHS; e += kThreads) dst[(size_t)(e / kHS) * H + h0 + e % kHS] = w1s[e];
      float* b1 = dst + (size_t)F * H;
      float* W2 = b1 + H;
      if (tid < kHS) b1[h0 + tid] = b1s[tid];
      for (int e = tid; e < kHS * C; e += kThreads) W2[(size_t)h0 * C + e] = w2s[(h0 + e / C) * CP + e % C];
      if (r == 0 && tid < C) W2[(size_t)H * C + tid] = b2s[tid];
    }
  }
  // ---------------------------------------------------- write-back --
  // (the other CTAs' W2 rows of the last step arrive by DSMEM; none is read here)
  const int ulast = a.n_micro_launch - 1;
  float* dst = a.wbase + (size_t)slot * a.wstride + (size_t)ulast * a.wmicro;
  for (int e = tid; e < F * kHS; e += kThreads) dst[(size_t)(e / kHS) * H + h0 + e % kHS] = w1s[e];
  float* b1 = dst + (size_t)F * H;
  float* W2 = b1 + H;
  if (tid < kHS) b1[h0 + tid] = b1s[tid];
  for (int e = tid; e < kHS * C; e += kThreads) W2[(size_t)h0 * C + e] = w2s[(h0 + e / C) * CP + e % C];
  if (r == 0 && tid < C) W2[(size_t)H * C + tid] = b2s[tid];
  if (nsteps == 0 && r == 0 && tid == 0)
    for (int u = 0; u < a.n_micro_launch; ++u)
      a.losses[(size_t)slot * a.loss_T + a.loss_t + u] = __int_as_float(0x7fc00000);
  cluster_sync();  // no CTA exits while a peer may still store into its shared memory
}

template <int NC, int F>
void launch_nc(const cudaLaunchConfig_t& lc0, const FfmaArgs& a, int device) {
  static DeviceFlags attr;
  if (!attr.done(device)) {
    ECCO_CUDA(cudaFuncSetAttribute(k_train_ffma<NC, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   232448));
    if (NC > 8)
      ECCO_CUDA(cudaFuncSetAttribute(k_train_ffma<NC, F>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr.mark(device);
  }
  cudaLaunchConfig_t lc = lc0;
  ECCO_CUDA(cudaLaunchKernelEx(&lc, k_train_ffma<NC, F>, a));
}

template <int F>
void launch_f(int nc, const cudaLaunchConfig_t& lc, const FfmaArgs& a, int device) {
  switch (nc) {
    case 16: launch_nc<16, F>(lc, a, device); break;
    case 8: launch_nc<8, F>(lc, a, device); break;
    case 4: launch_nc<4, F>(lc, a, device); break;
    default: launch_nc<2, F>(lc, a, device); break;
  }
}

}  // namespace

namespace fused {

// B = 128, C = 16, H = 16 x (2, 4, 8, 16), F = 128 / 256 / 512 and
// the shared-memory layout within the opt-in limit.  ECCO_FFMA_CHAIN=0 keeps
// the general per-step FFMA kernels (the A/B reference of the tests).
bool ffma_chain_supported(const ecco_ctx* ctx) {
  const ecco_config& g = ctx->cfg;
  const char* e = getenv("ECCO_FFMA_CHAIN");
  if (e && e[0] == '0') return false;
  const int nc = g.hidden_dim / kHS;
  return g.minibatch == kB && g.num_classes == kC && g.hidden_dim % kHS == 0 && nc >= 2 &&
         nc <= kMaxNC && (nc & (nc - 1)) == 0 &&
         (g.feat_dim == 128 || g.feat_dim == 256 || g.feat_dim == 512) &&
         flayout(g.feat_dim, g.hidden_dim, nc).total <= 232448;
}

void train_ffma(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_steps,
                const int* h_steps, int micro, int n_micro, const float* wsrc, size_t wsrc_stride,
                float* wbase, size_t wstride, int loss_t, int n_launch, size_t wmicro) {
  if (n_jobs == 0) return;
  ECCO_REQUIRE(n_launch == 1 || n_jobs == 1, "serial FFMA chain: one job");
  const ecco_config& c = ctx->cfg;
  int max_steps = 0;
  for (int j = 0; j < n_jobs; ++j) max_steps = std::max(max_steps, h_steps[j]);
  FfmaArgs a{};
  a.g = LDims{c.feat_dim, c.hidden_dim, c.num_classes, c.scene_dims, c.minibatch,
              c.ring_frames, c.eval_samples, c.sgd_lr, c.feature_noise};
  a.slots = d_slots;
  a.steps = d_steps;
  a.rows = (const int32_t*)ctx->train_scratch[0].p;  // chain_rows() of this call
  a.labs = (const int32_t*)ctx->train_scratch[1].p;
  a.row_step0 = micro * max_steps;
  a.rows_T = n_micro * max_steps;
  a.frames = ctx->d_frames;
  a.wsrc = wsrc;
  a.wsrc_stride = wsrc_stride;
  a.wbase = wbase;
  a.wstride = wstride;
  a.losses = ctx->d_losses;
  a.loss_T = c.max_depth;
  a.loss_t = loss_t;
  a.n_micro_launch = n_launch;
  a.wmicro = wmicro;
  const int nc = c.hidden_dim / kHS;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(nc * n_jobs));
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = flayout(c.feat_dim, c.hidden_dim, nc).total;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const double F = c.feat_dim, H = c.hidden_dim, C = c.num_classes;
  double steps = 0, live = 0;
  for (int j = 0; j < n_jobs; ++j) {
    steps += (double)h_steps[j] * n_launch;
    live += h_steps[j] > 0;
  }
  const double flops = steps * kB * (4.0 * F * H + 6.0 * H * C);
  const double bytes = steps * kB * F * 2.0 + live * (F * H + H + H * C + C) * 8.0;
  a.trace = getenv("ECCO_FFMA_TRACE") ? 1 : 0;
  ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_STEP, flops, bytes,
             (c.feat_dim == 512   ? launch_f<512>(nc, lc, a, c.device)
              : c.feat_dim == 256 ? launch_f<256>(nc, lc, a, c.device)
                                  : launch_f<128>(nc, lc, a, c.device)));
  ECCO_LAUNCHED(ctx);
  if (a.trace) {  // points: 0 gather, 1 forward, 2 relu sent, 3 barrier 1, 4 head done, 5 barrier 2, 6 updates done
    long long tr[4 * 16];
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    ECCO_CUDA(cudaMemcpyFromSymbol(tr, g_ffma_trace, sizeof(tr)));
    for (int t = 0; t < 4; ++t) {
      fprintf(stderr, "ffma step %d:", t);
      for (int k = 1; k < 7; ++k) fprintf(stderr, " %d:%lld", k, tr[t * 16 + k] - tr[t * 16]);
      fprintf(stderr, "\n");
    }
  }
}

}  // namespace fused
