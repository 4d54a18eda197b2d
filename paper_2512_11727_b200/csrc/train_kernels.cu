// Fused SGD step of the learned backend (tensor-core math): ONE launch
// trains every group's model by one minibatch step -- sampling, gather,
// forward, softmax cross-entropy, backward and the SGD update -- one CTA
// per group (job), nothing staged through HBM but the updated weights.
//
//   sample   B = 128 frame indices per job from the counter RNG
//            (sample_one, identical to the exact path and the oracle), rows
//            gathered by cp.async into a 128B-swizzled K-major X tile
//            (bf16, exact) that stays in shared memory for the whole step
//   fwd      Z = X . W1                 tcgen05 kind::f16, N = H, TMEM
//            (W1^T bf16 shadow streamed by TMA, 2 stages)
//   head     logits = relu(Z+b1) . W2 + b2 (two threads per row, half the
//            hidden columns each), softmax, dL, dH = (dL . W2^T) * (Z+b1 > 0)
//            -- CUDA cores, W2 in smem; no block-wide syncs per column
//   dW2/db1  dW2 = R^T . dL and db1 = dH^T . 1 as tcgen05 MMAs (M = 128
//            hidden units per tile, N = 16): R = bf16(relu(Z+b1)) is written
//            MN-major over the X tile once dW1 no longer needs it, dL and a
//            ones tile as 32B-swizzled MN-major B operands
//   dW1      G = X^T . dH               tcgen05 kind::f16 with BOTH operands
//            MN-major (X^T is the same smem tile read transposed; dH is
//            written MN-major by the head), M = 128 features per tile
//   update   W1 -= lr * G (fp32 masters, stored transposed [H][F] in this
//            mode so the read-modify-write is coalesced) and the bf16 W1^T
//            shadow rewritten for the next step's forward
//
// Numerics: X exact (bf16 frames); W1, dH, R and dL rounded to bf16 at the
// tensor-core contractions, fp32 accumulation, fp32 masters; logits / softmax
// / dH fp32 on CUDA cores.  Tolerance in tests/test_gpu_learned.py.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "learned_common.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

constexpr int kB = 128;        // minibatch rows = UMMA M
constexpr int kThreads = 256;  // 8 warps
constexpr int kC = 16;         // classes held in registers by the head
constexpr int kHC = 8;         // hidden columns per head-backward chunk

struct TrainArgs {
  LDims g;
  uint64_t seed;
  const int* slots;
  const int* job_ids;
  const int* steps;
  const int* src_off;
  const int* src_cam;
  const double* src_frac;
  const int* micro_base;
  int micro_add;  // micro index = micro_base[j] + micro_add
  int window;
  int step;
  const uint16_t* frames;
  const int32_t* labels;
  float* wbase;  // fp32 masters being trained
  size_t wstride;
  uint16_t* w1t;  // bf16 W1^T shadow [slot][H][F]
  float* losses;  // losses[slot * loss_T + loss_t]
  int loss_T, loss_t;
};

struct Layout {
  uint32_t x, wb, w2, dl, pl, rows, labs, b2, loss, bars, tmem, total;
};

__host__ __device__ inline Layout layout(int F, int H, int C) {
  Layout L{};
  uint32_t o = 0;
  L.x = o;
  o += (uint32_t)(F / 64) * 16384u;  // X (later R): F/64 swizzle chunks of 128 rows x 128 B
  L.wb = o;
  o += (uint32_t)H * 256u;  // 2 W1^T stages (H x 64 bf16) == dH (128 x H bf16)
  L.w2 = o;
  o += (uint32_t)H * C * 4u;
  L.dl = o;
  o += (uint32_t)kB * C * 4u;  // dL fp32 [row][class]
  L.pl = o;
  o += (uint32_t)kB * C * 4u;  // partial logits of the second half; later dL / ones B tiles
  L.rows = o;
  o += kB * 8u;
  L.labs = o;
  o += kB * 4u;
  L.b2 = o;
  o += (uint32_t)C * 4u;
  L.loss = o;
  o += kB * 4u;
  o = (o + 7u) & ~7u;
  L.bars = o;
  o += 8u * 8u;  // full[2] empty[2] zfull gfull gempty dfull
  L.tmem = o;
  o += 16u;
  L.total = o;
  return L;
}

// MN-major operand with 32-byte swizzle (16 two-byte elements per row of an
// atom, 8 K rows = 256 B): element (n, k) of a [K][16] tile.
__device__ __forceinline__ uint32_t sw32_off(int n, int k) {
  return (uint32_t)k * 32u + ((((uint32_t)n >> 3) ^ (((uint32_t)k >> 2) & 1u)) << 4) +
         ((uint32_t)n & 7u) * 2u;
}

__global__ void __launch_bounds__(kThreads, 1)
    k_train_step(const __grid_constant__ CUtensorMap map_w1t, TrainArgs a) {
  const int j = blockIdx.x;
  if (a.step >= a.steps[j]) return;
  extern __shared__ __align__(1024) uint8_t smem[];
  const LDims g = a.g;
  const int F = g.F, H = g.H;
  const Layout L = layout(F, H, kC);
  uint8_t* sX = smem + L.x;
  uint8_t* sWB = smem + L.wb;
  float* sW2 = (float*)(smem + L.w2);
  float* sDL = (float*)(smem + L.dl);
  float* sPL = (float*)(smem + L.pl);
  int64_t* sRow = (int64_t*)(smem + L.rows);
  int* sLab = (int*)(smem + L.labs);
  float* sB2 = (float*)(smem + L.b2);
  float* sLoss = (float*)(smem + L.loss);
  uint64_t* full = (uint64_t*)(smem + L.bars);  // [2]
  uint64_t* empty = full + 2;                   // [2]
  uint64_t* zfull = full + 4;
  uint64_t* gfull = full + 5;
  uint64_t* gempty = full + 6;
  uint64_t* dfull = full + 7;
  uint32_t* sTmem = (uint32_t*)(smem + L.tmem);
  const uint32_t stage_bytes = (uint32_t)H * 128u;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int slot = a.slots[j];
  float* W1 = a.wbase + (size_t)slot * a.wstride;
  float* b1 = W1 + (size_t)F * H;
  float* W2 = b1 + H;
  float* b2 = W2 + (size_t)H * kC;
  uint16_t* W1T = a.w1t + (size_t)slot * H * F;
  const float lr = g.lr;

  // ---------------------------------------------------------------- setup --
  if (tid == 0) {
    if (smem_u32(smem) & 1023u) __trap();  // 128B-swizzle atoms need 1 KB alignment
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(zfull, 1);
    mbar_init(gfull, 1);
    mbar_init(gempty, 8);
    mbar_init(dfull, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(sTmem, 512);
  if (tid < kB) {  // the minibatch: identical draws to the exact path (k_l_sample)
    const int s0 = a.src_off[j];
    int cam, frame;
    sample_one(g, a.seed, a.job_ids[j], a.src_off[j + 1] - s0, a.src_cam + s0, a.src_frac + s0,
               a.window, a.micro_base[j] + a.micro_add, a.step, tid, &cam, &frame);
    const int64_t row = (int64_t)cam * g.R + frame;
    sRow[tid] = row * F;
    sLab[tid] = a.labels[row];
  }
  for (int i = tid; i < H * kC / 4; i += kThreads)
    reinterpret_cast<float4*>(sW2)[i] = reinterpret_cast<const float4*>(W2)[i];
  if (tid < kC) sB2[tid] = b2[tid];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sTmem;

  // first two W1^T K-chunks in flight while the rows are gathered
  const int nkc = F / 64;
  if (warp == 0) {
    if (elect_one()) {
      for (int s = 0; s < 2 && s < nkc; ++s) {
        mbar_expect_tx(&full[s], stage_bytes);
        tma_load_2d(sWB + s * stage_bytes, &map_w1t, s * 64, slot * H, &full[s]);
      }
    }
    __syncwarp();
  }
  // gather: row s, 16-byte piece c16 -> chunk c16/8, swizzled column
  const int per_row = F / 8;
  for (int p = tid; p < kB * per_row; p += kThreads) {
    const int s = p / per_row, c16 = p % per_row;
    const int kc = c16 >> 3, c = c16 & 7;
    cp_async16(sX + kc * 16384 + s * 128 + ((c ^ (s & 7)) << 4), a.frames + sRow[s] + c16 * 8);
  }
  cp_async_wait_all();
  fence_async_smem();
  __syncthreads();

  // ----------------------------------------------------------- forward MMA --
  if (warp == 0) {
    tc_fence_after();
    const uint32_t idf = idesc(kB, H, kFmtBF16);
    const uint64_t dX = desc_kmajor_sw128(smem_u32(sX));
    const uint64_t dW = desc_kmajor_sw128(smem_u32(sWB));
    for (int kc = 0; kc < nkc; ++kc) {
      const int s = kc & 1;
      const uint32_t ph = (kc >> 1) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ss(tmem, dX + ((kc * 16384 + kk * 32) >> 4),
                      dW + ((s * stage_bytes + kk * 32) >> 4), idf, (kc | kk) != 0);
        mma_commit(&empty[s]);
        if (kc == nkc - 1) mma_commit(zfull);
      }
      __syncwarp();
      if (kc + 2 < nkc) {
        mbar_wait(&empty[s], ph);
        if (elect_one()) {
          mbar_expect_tx(&full[s], stage_bytes);
          tma_load_2d(sWB + s * stage_bytes, &map_w1t, (kc + 2) * 64, slot * H, &full[s]);
        }
        __syncwarp();
      }
    }
  }

  // ------------------------------------------------------- head: logits --
  // Two threads per minibatch row: warps w and w+4 share TMEM lane quadrant
  // w%4 and take hidden columns [part*H/2, (part+1)*H/2).
  const int q = warp & 3, part = warp >> 2;
  const int s = q * 32 + lane;  // minibatch row (TMEM lane)
  const uint32_t lane_base = (uint32_t)(q * 32) << 16;
  const int hh = H / 2, h_lo = part * hh;
  mbar_wait(zfull, 0);
  tc_fence_after();
  float lg[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) lg[c] = 0.0f;
  for (int c0 = h_lo; c0 < h_lo + hh; c0 += 32) {
    uint32_t r[32];
    tmem_ld32_nowait(tmem + lane_base + c0, r);
    tmem_ld_wait();
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      const float z = __fadd_rn(__uint_as_float(r[i]), b1[c0 + i]);
      const float rz = z > 0.0f ? z : 0.0f;
      const float4* w = reinterpret_cast<const float4*>(sW2 + (c0 + i) * kC);
#pragma unroll
      for (int c4 = 0; c4 < kC / 4; ++c4) {
        const float4 v = w[c4];
        lg[4 * c4 + 0] = __fmaf_rn(rz, v.x, lg[4 * c4 + 0]);
        lg[4 * c4 + 1] = __fmaf_rn(rz, v.y, lg[4 * c4 + 1]);
        lg[4 * c4 + 2] = __fmaf_rn(rz, v.z, lg[4 * c4 + 2]);
        lg[4 * c4 + 3] = __fmaf_rn(rz, v.w, lg[4 * c4 + 3]);
      }
    }
  }
  if (part == 1) {
#pragma unroll
    for (int c = 0; c < kC; ++c) sPL[s * kC + c] = lg[c];
  }
  __syncthreads();
  if (part == 0) {  // softmax cross-entropy (orc_sgd_step's order after the sum)
#pragma unroll
    for (int c = 0; c < kC; ++c) lg[c] = __fadd_rn(__fadd_rn(lg[c], sPL[s * kC + c]), sB2[c]);
    float m = lg[0];
#pragma unroll
    for (int c = 1; c < kC; ++c) m = lg[c] > m ? lg[c] : m;
    float e[kC], sum = 0.0f;
#pragma unroll
    for (int c = 0; c < kC; ++c) {
      e[c] = ecco_expf(__fsub_rn(lg[c], m));
      sum = __fadd_rn(sum, e[c]);
    }
    const float invB = __fdiv_rn(1.0f, (float)kB);
    const int y = sLab[s];
    float ly = lg[0];
#pragma unroll
    for (int c = 0; c < kC; ++c) {
      sDL[s * kC + c] = __fmul_rn(__fsub_rn(__fdiv_rn(e[c], sum), c == y ? 1.0f : 0.0f), invB);
      ly = c == y ? lg[c] : ly;
    }
    sLoss[s] = logf(sum) - (ly - m);
  }
  __syncthreads();

  // ---------------------------------------------- head: dH (no block syncs) --
  {
    float dl[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) dl[c] = sDL[s * kC + c];
    for (int c0 = h_lo; c0 < h_lo + hh; c0 += 32) {
      uint32_t r[32];
      tmem_ld32_nowait(tmem + lane_base + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int g8 = 0; g8 < 4; ++g8) {
        float dh[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int h = c0 + g8 * 8 + i;
          const float z = __fadd_rn(__uint_as_float(r[g8 * 8 + i]), b1[h]);
          float acc = 0.0f;
          const float4* w = reinterpret_cast<const float4*>(sW2 + h * kC);
#pragma unroll
          for (int c4 = 0; c4 < kC / 4; ++c4) {
            const float4 v = w[c4];
            acc = __fmaf_rn(dl[4 * c4 + 0], v.x, acc);
            acc = __fmaf_rn(dl[4 * c4 + 1], v.y, acc);
            acc = __fmaf_rn(dl[4 * c4 + 2], v.z, acc);
            acc = __fmaf_rn(dl[4 * c4 + 3], v.w, acc);
          }
          dh[i] = z > 0.0f ? acc : 0.0f;
        }
        // dH as the MN-major operand (row s, 64-column atoms): dW1's B, db1's A
        const int h0 = c0 + g8 * 8;
        uint4 pk;
        pk.x = pack_bf16x2(dh[0], dh[1]);
        pk.y = pack_bf16x2(dh[2], dh[3]);
        pk.z = pack_bf16x2(dh[4], dh[5]);
        pk.w = pack_bf16x2(dh[6], dh[7]);
        *reinterpret_cast<uint4*>(sWB + (h0 >> 6) * 16384 + s * 128 +
                                  ((((h0 & 63) >> 3) ^ (s & 7)) << 4)) = pk;
      }
    }
  }
  // dL and a ones tile as 32B-swizzled MN-major B operands (N = 16, K = rows)
  {
    uint8_t* sDLb = reinterpret_cast<uint8_t*>(sPL);  // partial logits are consumed
    uint8_t* sOnes = sDLb + kB * 32;
    if (part == 0) {
#pragma unroll
      for (int c = 0; c < kC; c += 2) {
        const uint32_t pk = pack_bf16x2(sDL[s * kC + c], sDL[s * kC + c + 1]);
        *reinterpret_cast<uint32_t*>(sDLb + sw32_off(c, s)) = pk;
      }
    } else {
#pragma unroll
      for (int c = 0; c < kC; c += 2)
        *reinterpret_cast<uint32_t*>(sOnes + sw32_off(c, s)) = 0x3F803F80u;  // bf16 1.0 x 2
    }
  }
  fence_async_smem();  // dH / dL / ones (generic stores) -> tensor-core reads
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ------------------------------------------------- dW1 = X^T . dH, update --
  // One 256-column accumulator at TMEM [256, 512) (Z stays in [0, 256) for R).
  const int nmt = F / 128;
  const uint32_t idg = idesc_major(128, H, kFmtBF16, 1, 1);
  auto issue = [&](int mt) {
    if (elect_one()) {
#pragma unroll
      for (int k16 = 0; k16 < kB / 16; ++k16) {
        const uint64_t da =
            desc_mnmajor_sw128(smem_u32(sX) + (2 * mt) * 16384 + k16 * 2048, 16384, 1024);
        const uint64_t db = desc_mnmajor_sw128(smem_u32(sWB) + k16 * 2048, 16384, 1024);
        mma_bf16_ss(tmem + 256, da, db, idg, k16 != 0);
      }
      mma_commit(gfull);
    }
    __syncwarp();
  };
  if (warp == 0) issue(0);
  const int cp = part;
  const int hw = H / 2;
  for (int mt = 0; mt < nmt; ++mt) {
    mbar_wait(gfull, mt & 1);
    tc_fence_after();
    const int f = mt * 128 + q * 32 + lane;
    for (int c0 = cp * hw; c0 < (cp + 1) * hw; c0 += 32) {
      uint32_t r[32];
      tmem_ld32_nowait(tmem + lane_base + 256 + c0, r);
      // masters are [H][F]: for each h the warp's 32 lanes (32 consecutive
      // f) touch one 128-byte line -- coalesced, 32 independent loads
      float w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) w[i] = W1[(size_t)(c0 + i) * F + f];
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float nw = __fmaf_rn(-lr, __uint_as_float(r[i]), w[i]);
        W1[(size_t)(c0 + i) * F + f] = nw;
        W1T[(size_t)(c0 + i) * F + f] = (uint16_t)(pack_bf16x2(nw, 0.0f) & 0xFFFF);
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(gempty);
    if (warp == 0 && mt + 1 < nmt) {
      mbar_wait(gempty, mt & 1);
      tc_fence_after();
      issue(mt + 1);
    }
  }

  // ------------------------------ dW2 = R^T . dL, db1 = dH^T . 1 (tensor) --
  // The last dW1 MMA has completed (every thread waited on it), so the X tile
  // is free: R = bf16(relu(Z + b1)) goes there, MN-major like dH.
  for (int c0 = h_lo; c0 < h_lo + hh; c0 += 32) {
    uint32_t r[32];
    tmem_ld32_nowait(tmem + lane_base + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int g8 = 0; g8 < 4; ++g8) {
      const int h0 = c0 + g8 * 8;
      float rz[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float z = __fadd_rn(__uint_as_float(r[g8 * 8 + i]), b1[h0 + i]);
        rz[i] = z > 0.0f ? z : 0.0f;
      }
      uint4 pk;
      pk.x = pack_bf16x2(rz[0], rz[1]);
      pk.y = pack_bf16x2(rz[2], rz[3]);
      pk.z = pack_bf16x2(rz[4], rz[5]);
      pk.w = pack_bf16x2(rz[6], rz[7]);
      *reinterpret_cast<uint4*>(sX + (h0 >> 6) * 16384 + s * 128 +
                                ((((h0 & 63) >> 3) ^ (s & 7)) << 4)) = pk;
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idw = idesc_major(128, kC, kFmtBF16, 1, 1);
      const uint32_t dlb = smem_u32(sPL), onesb = dlb + kB * 32;
      for (int t2 = 0; t2 < H / 128; ++t2) {
#pragma unroll
        for (int k16 = 0; k16 < kB / 16; ++k16) {
          const uint64_t bdl = smem_desc(dlb + k16 * 512, 256, 256, kSwizzle32B);
          const uint64_t bon = smem_desc(onesb + k16 * 512, 256, 256, kSwizzle32B);
          const uint64_t ar =
              desc_mnmajor_sw128(smem_u32(sX) + (2 * t2) * 16384 + k16 * 2048, 16384, 1024);
          const uint64_t ad =
              desc_mnmajor_sw128(smem_u32(sWB) + (2 * t2) * 16384 + k16 * 2048, 16384, 1024);
          mma_bf16_ss(tmem + t2 * kC, ar, bdl, idw, k16 != 0);          // dW2 tile
          mma_bf16_ss(tmem + 64 + t2 * kC, ad, bon, idw, k16 != 0);     // db1 tile
        }
      }
      mma_commit(dfull);
    }
    __syncwarp();
  }
  mbar_wait(dfull, 0);
  tc_fence_after();
  if (part < H / 128) {  // thread owns hidden unit h = part*128 + lane quadrant row
    const int h = part * 128 + q * 32 + lane;
    uint32_t r[16], rb[16];
    tmem_ld16_nowait(tmem + lane_base + part * kC, r);
    tmem_ld16_nowait(tmem + lane_base + 64 + part * kC, rb);
    tmem_ld_wait();
    float4* w2row = reinterpret_cast<float4*>(W2 + (size_t)h * kC);
#pragma unroll
    for (int c4 = 0; c4 < kC / 4; ++c4) {
      const float4 o = reinterpret_cast<const float4*>(sW2 + h * kC)[c4];
      float4 n;
      n.x = __fmaf_rn(-lr, __uint_as_float(r[4 * c4 + 0]), o.x);
      n.y = __fmaf_rn(-lr, __uint_as_float(r[4 * c4 + 1]), o.y);
      n.z = __fmaf_rn(-lr, __uint_as_float(r[4 * c4 + 2]), o.z);
      n.w = __fmaf_rn(-lr, __uint_as_float(r[4 * c4 + 3]), o.w);
      w2row[c4] = n;
    }
    b1[h] = __fmaf_rn(-lr, __uint_as_float(rb[0]), b1[h]);
  }
  if (tid < kC) {
    float acc = 0.0f;
    for (int q2 = 0; q2 < kB; ++q2) acc = __fadd_rn(acc, sDL[q2 * kC + tid]);
    b2[tid] = __fmaf_rn(-lr, acc, sB2[tid]);
  }

  // ------------------------------------------------------------- loss, end --
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    double acc = 0.0;
    for (int q2 = 0; q2 < kB; ++q2) acc += sLoss[q2];
    a.losses[(size_t)slot * a.loss_T + a.loss_t] = (float)(acc / kB);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace

namespace fused {

bool train_supported(const ecco_ctx* ctx) {
  const ecco_config& g = ctx->cfg;
  if (g.minibatch != kB || g.num_classes != kC || g.feat_dim % 128 || g.feat_dim > 512 ||
      g.hidden_dim != 256)
    return false;
  return layout(g.feat_dim, g.hidden_dim, kC).total <= 232448;
}

void train_step(ecco_ctx* ctx, const Shadow& sh, int n_jobs, const int* d_slots,
                const int* d_job_ids, const int* d_steps, const int* d_src_off,
                const int* d_src_cam, const double* d_src_frac, const int* d_micro_base,
                int micro_add, int window, int step, float* wbase, size_t wstride, int loss_t,
                double live_rows) {
  if (n_jobs == 0) return;
  const ecco_config& c = ctx->cfg;
  TrainArgs a{};
  a.g = {c.feat_dim, c.hidden_dim, c.num_classes, c.scene_dims, c.minibatch, c.ring_frames,
         c.eval_samples, c.sgd_lr, c.feature_noise};
  a.seed = c.seed;
  a.slots = d_slots;
  a.job_ids = d_job_ids;
  a.steps = d_steps;
  a.src_off = d_src_off;
  a.src_cam = d_src_cam;
  a.src_frac = d_src_frac;
  a.micro_base = d_micro_base;
  a.micro_add = micro_add;
  a.window = window;
  a.step = step;
  a.frames = ctx->d_frames;
  a.labels = ctx->d_labels;
  a.wbase = wbase;
  a.wstride = wstride;
  a.w1t = sh.w1t;
  a.losses = ctx->d_losses;
  a.loss_T = c.max_depth;
  a.loss_t = loss_t;
  const uint32_t smem = layout(c.feat_dim, c.hidden_dim, kC).total;
  static bool attr = false;
  if (!attr) {
    ECCO_CUDA(cudaFuncSetAttribute(k_train_step, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    attr = true;
  }
  const double F = c.feat_dim, H = c.hidden_dim, C = c.num_classes;
  const double flops = live_rows * (4.0 * F * H + 6.0 * H * C);
  const double bytes = live_rows * F * 2.0 + live_rows / kB * (F * H * (4.0 + 4.0 + 2.0 + 2.0));
  ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_STEP, flops, bytes,
             (k_train_step<<<n_jobs, kThreads, smem, ctx->stream>>>(
                 *(const CUtensorMap*)sh.map_w_train, a)));
  ECCO_LAUNCHED(ctx);
}

}  // namespace fused
