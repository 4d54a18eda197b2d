// Fused camera x group evaluation (K6 of SURVEY.md 2): for every (probe
// camera, group model) pair, the number of the camera's S labelled eval frames
// that the group's MLP classifies correctly -- hidden layer, ReLU, logits,
// argmax and the correct-count in ONE persistent kernel, nothing but the
// counts written to HBM.
//
//   Z      = X[128 rows, F] . W1[F, H]        tcgen05 kind::f16 (bf16 in, fp32
//                                             accumulate in TMEM), H in halves
//                                             of N = 128
//   R      = bf16(relu(Z + b1))               epilogue warps: TMEM -> regs ->
//                                             TMEM (A operand of the next MMA)
//   logits = R[128, H] . W2[H, C]             tcgen05 kind::f16, A from TMEM
//   count += (argmax(logits + b2) == label)   warp ballot + popc, one atomic
//                                             per (warp, pair)
//
// Rows of a 128-row tile are 2 x 64 eval frames (S % 64 == 0): each 64-row
// block is one TMA box at the probe camera's eval-set row, so any camera list
// can be probed.  The tile's X stays resident in shared memory (F <= 512:
// <= 128 KB, loaded once per tile by TMA with 128-byte swizzle) while the
// group models stream through a 5-6 stage TMA pipeline of 128-row W1^T boxes
// (bf16 shadow of the fp32 masters, refreshed when a model changes), so the
// tensor cores read only W1 from L2 per group: 256 FLOP per L2 byte.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer, warps
// 2-5 epilogue (TMEM lane quadrant = warp % 4).  TMEM (512 columns):
//   [0,256)   Z, two 128-column buffers      (MMA <-> epilogue double buffer)
//   [256,384) R, two 64-column bf16 buffers  (epilogue <-> MMA double buffer)
//   [384,..)  logits, 1-2 buffers of C columns
// Numerics: X is exact in bf16, W1 and R are rounded to bf16; accumulation is
// fp32.  DESIGN.md states the tolerance against the fp32 oracle.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "sm100.cuh"

using namespace sm100;

namespace {

constexpr int kTileRows = 128;
constexpr int kKC = 64;               // K per TMA box / pipeline stage (one 128-B swizzle atom)
constexpr int kHalf = 128;            // N of the hidden-layer MMA
constexpr int kThreads = 320;  // 2 control warps + 8 epilogue warps
constexpr uint32_t kBoxBytes = kHalf * 128;   // one W1^T stage: 128 rows x 64 bf16
constexpr uint32_t kAChunk = kTileRows * 128; // one X K-chunk: 128 rows x 64 bf16
constexpr int kMaxStages = 8;
constexpr uint32_t kTmemZ = 0, kTmemR = 256, kTmemL = 384;

struct EvalBars {
  uint64_t a_full, a_empty;
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t w2_full[2], w2_empty[2];
  uint64_t z_full[2], z_empty[2], r_full[2], r_empty[2];
  uint64_t l_full[2], l_empty[2];
  uint32_t tmem_base;
};

struct EvalArgs {
  int n_rows;            // n_probes * S
  int S;
  int F, H, C;
  int n_tiles;
  const int* cams;       // probe -> camera table index
  const int32_t* labels; // camera table eval labels [cam * S + s]
  // entries: (slot, output column); dense mode: every tile walks all n_ent;
  // pairs mode (tile_ebeg != null): tile m walks [tile_ebeg[m], tile_ebeg[m+1])
  const int* ent_slot;
  const int* ent_col;
  int n_ent;
  const int* tile_ebeg;
  const int* probe_slot; // pairs mode: a row counts only under its probe's own slot
  int ld;                // dense: counts[p * ld + col]; pairs: counts[p]
  int* counts;
  const float* wbase;    // fp32 masters: b1 at +F*H, b2 at +F*H+H+H*C
  size_t wstride;
  const uint8_t* w2t;    // per slot: W2^T bf16 K-major 128B-swizzled image
  uint32_t w2t_bytes;    // W2^T part of the per-slot image
  uint32_t img_bytes;    // whole image: W2^T | b1 (H fp32) | b2 (C fp32)
  uint32_t w2t_stride;   // smem stride of the two W2^T buffers (1024-aligned)
  uint32_t bias_bytes;   // b1 | b2 part of the image (smem stride of its buffers)
  int stages;
  int nl;                // logits buffers (1 or 2)
  float* dbg_logits;     // optional: [n_rows][n_ent][C] logits + b2 (dense mode tests)
  int* tile_ctr;         // pair kernel: next super tile (zeroed before the launch)
};

__device__ __forceinline__ int tile_ent_begin(const EvalArgs& a, int m) {
  return a.tile_ebeg ? a.tile_ebeg[m] : 0;
}
__device__ __forceinline__ int tile_ent_end(const EvalArgs& a, int m) {
  return a.tile_ebeg ? a.tile_ebeg[m + 1] : a.n_ent;
}

__global__ void __launch_bounds__(kThreads, 1)
    k_eval_fused(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                 EvalArgs a) {
  // everything lives in dynamic shared memory (no static smem), so the base
  // is 1 KB aligned as the 128B-swizzle atoms require (checked below)
  extern __shared__ __align__(1024) uint8_t smem[];
  const int nkc = a.F / kKC;
  const int nh = a.H / kHalf;
  uint8_t* sA = smem;                                   // nkc x 16 KB
  uint8_t* sB = sA + nkc * kAChunk;                     // stages x 16 KB
  uint8_t* sW2 = sB + a.stages * kBoxBytes;             // 2 x w2t_stride (W2^T images)
  uint8_t* sBias = sW2 + 2 * a.w2t_stride;              // 2 x bias_bytes (b1 | b2)
  EvalBars* bars = reinterpret_cast<EvalBars*>(sBias + 2 * a.bias_bytes);
  uint64_t& a_full = bars->a_full;
  uint64_t& a_empty = bars->a_empty;
  uint64_t* full = bars->full;
  uint64_t* empty = bars->empty;
  uint64_t* w2_full = bars->w2_full;
  uint64_t* w2_empty = bars->w2_empty;
  uint64_t* z_full = bars->z_full;
  uint64_t* z_empty = bars->z_empty;
  uint64_t* r_full = bars->r_full;
  uint64_t* r_empty = bars->r_empty;
  uint64_t* l_full = bars->l_full;
  uint64_t* l_empty = bars->l_empty;
  uint32_t& tmem_base = bars->tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    if (smem_u32(smem) & 1023u) __trap();
    tma_prefetch(&map_x);
    tma_prefetch(&map_w);
    mbar_init(&a_full, 1);
    mbar_init(&a_empty, 1);
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&w2_full[b], 1);
      mbar_init(&w2_empty[b], 1 + 4);  // MMA commit + the 4 logits warps
      mbar_init(&z_full[b], 1);
      mbar_init(&z_empty[b], 8);
      mbar_init(&r_full[b], 8);
      mbar_init(&r_empty[b], 1);
      mbar_init(&l_full[b], 1);
      mbar_init(&l_empty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    // (whole warp walks the schedule; one elected lane issues)
    int stage = 0;
    uint32_t sph = 0;
    uint32_t u = 0, t = 0;
    for (int m = blockIdx.x; m < a.n_tiles; m += gridDim.x, ++t) {
      if (t > 0) mbar_wait(&a_empty, (t - 1) & 1);
      if (elect_one()) {
        mbar_expect_tx(&a_full, (uint32_t)nkc * kAChunk);
        for (int h2 = 0; h2 < 2; ++h2) {
          int b = m * 2 + h2;
          if (b * 64 >= a.n_rows) b = 0;  // padding rows: any valid box, masked later
          const int p = (b * 64) / a.S, soff = (b * 64) % a.S;
          const int row = a.cams[p] * a.S + soff;
          for (int kc = 0; kc < nkc; ++kc)
            tma_load_2d(sA + kc * kAChunk + h2 * (kAChunk / 2), &map_x, kc * kKC, row, &a_full);
        }
      }
      __syncwarp();
      const int e1 = tile_ent_end(a, m);
      for (int e = tile_ent_begin(a, m); e < e1; ++e, ++u) {
        const int slot = a.ent_slot[e];
        const int wb = u & 1;
        mbar_wait(&w2_empty[wb], ((u >> 1) & 1) ^ 1);
        if (elect_one()) {
          const uint8_t* img = a.w2t + (size_t)slot * a.img_bytes;
          mbar_expect_tx(&w2_full[wb], a.img_bytes);
          bulk_load(sW2 + wb * a.w2t_stride, img, a.w2t_bytes, &w2_full[wb]);
          bulk_load(sBias + wb * a.bias_bytes, img + a.w2t_bytes, a.bias_bytes, &w2_full[wb]);
        }
        __syncwarp();
        for (int hf = 0; hf < nh; ++hf) {
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&empty[stage], sph ^ 1);
            if (elect_one()) {
              mbar_expect_tx(&full[stage], kBoxBytes);
              tma_load_2d(sB + stage * kBoxBytes, &map_w, kc * kKC, slot * a.H + hf * kHalf,
                          &full[stage]);
            }
            __syncwarp();
            if (++stage == a.stages) {
              stage = 0;
              sph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    // Descriptors are built once; K steps and pipeline stages only add their
    // byte offset (>> 4) to the start-address field.
    const uint32_t id1 = idesc(kTileRows, kHalf, kFmtBF16);
    const uint32_t id2 = idesc(kTileRows, a.C, kFmtBF16);
    const uint64_t dA0 = desc_kmajor_sw128(smem_u32(sA));
    const uint64_t dB0 = desc_kmajor_sw128(smem_u32(sB));
    const uint64_t dW0 = desc_kmajor_sw128(smem_u32(sW2));
    int stage = 0;
    uint32_t sph = 0;
    uint32_t u = 0, t = 0;
    long prev = -1;  // pending layer-2 for sequence index prev (v = u * nh + hf)
    auto layer2 = [&](uint32_t w) {
      const uint32_t uw = w / nh, hw = w % nh;
      const uint32_t rb = w & 1, lb = uw % a.nl, wb = uw & 1;
      if (hw == 0) {
        mbar_wait(&w2_full[wb], (uw >> 1) & 1);
        mbar_wait(&l_empty[lb], ((uw / a.nl) & 1) ^ 1);
      }
      mbar_wait(&r_full[rb], (w >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dW = dW0 + ((wb * a.w2t_stride) >> 4);
#pragma unroll
        for (int k16 = 0; k16 < kHalf / 16; ++k16) {
          const int kg = hw * kHalf + k16 * 16;  // K index into H
          mma_bf16_ts(tmem + kTmemL + lb * a.C, tmem + kTmemR + rb * 64 + k16 * 8,
                      dW + (((kg / 64) * (a.C * 128) + (kg % 64) * 2) >> 4), id2,
                      (hw | k16) != 0);
        }
        mma_commit(&r_empty[rb]);
        if (hw == (uint32_t)nh - 1) {
          mma_commit(&l_full[lb]);
          mma_commit(&w2_empty[wb]);
        }
      }
      __syncwarp();
    };
    for (int m = blockIdx.x; m < a.n_tiles; m += gridDim.x, ++t) {
      mbar_wait(&a_full, t & 1);
      tc_fence_after();
      const int e1 = tile_ent_end(a, m);
      for (int e = tile_ent_begin(a, m); e < e1; ++e, ++u) {
        for (int hf = 0; hf < nh; ++hf) {
          const uint32_t v = u * nh + hf, zb = v & 1;
          mbar_wait(&z_empty[zb], ((v >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dz = tmem + kTmemZ + zb * kHalf;
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&full[stage], sph);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t da = dA0 + ((kc * kAChunk) >> 4);
              const uint64_t db = dB0 + ((stage * kBoxBytes) >> 4);
#pragma unroll
              for (int kk = 0; kk < kKC / 16; ++kk)
                mma_bf16_ss(dz, da + kk * 2, db + kk * 2, id1, (kc | kk) != 0);
              mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == a.stages) {
              stage = 0;
              sph ^= 1;
            }
          }
          if (elect_one()) mma_commit(&z_full[zb]);
          __syncwarp();
          if (prev >= 0) layer2((uint32_t)prev);
          prev = v;
        }
      }
      if (elect_one()) mma_commit(&a_empty);
      __syncwarp();
    }
    if (prev >= 0) layer2((uint32_t)prev);
  } else {
    // ----------------------------------------------------------- epilogue --
    // 8 warps: two per TMEM lane quadrant, each converting 64 of a half's
    // 128 Z columns; the cp == 0 warp of each quadrant also reads the logits.
    const int q = warp & 3;
    const int cp = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t u = 0;
    for (int m = blockIdx.x; m < a.n_tiles; m += gridDim.x) {
      const int R = m * kTileRows + row;
      const bool valid = R < a.n_rows;
      const int p = valid ? R / a.S : 0;
      const int label = valid ? a.labels[(size_t)a.cams[p] * a.S + (R % a.S)] : -1;
      const int pslot = (valid && a.probe_slot) ? a.probe_slot[p] : -1;
      const int e1 = tile_ent_end(a, m);
      for (int e = tile_ent_begin(a, m); e < e1; ++e, ++u) {
        const uint32_t wb = u & 1;
        const float* b1 = reinterpret_cast<const float*>(sBias + wb * a.bias_bytes);
        const float* b2 = b1 + a.H;
        mbar_wait(&w2_full[wb], (u >> 1) & 1);  // b1 / b2 of this model are in smem
        for (int hf = 0; hf < nh; ++hf) {
          const uint32_t v = u * nh + hf, zb = v & 1;
          const int c0 = cp * 64;
          mbar_wait(&z_full[zb], (v >> 1) & 1);
          mbar_wait(&r_empty[zb], ((v >> 1) & 1) ^ 1);
          tc_fence_after();
          uint32_t r[64];
          tmem_ld32_nowait(tmem + lane_base + kTmemZ + zb * kHalf + c0, r);
          tmem_ld32_nowait(tmem + lane_base + kTmemZ + zb * kHalf + c0 + 32, r + 32);
          tmem_ld_wait();
          const float4* bb = reinterpret_cast<const float4*>(b1 + hf * kHalf + c0);
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float4 b = bb[i];
            const float z0 = fmaxf(__uint_as_float(r[4 * i + 0]) + b.x, 0.0f);
            const float z1 = fmaxf(__uint_as_float(r[4 * i + 1]) + b.y, 0.0f);
            const float z2 = fmaxf(__uint_as_float(r[4 * i + 2]) + b.z, 0.0f);
            const float z3 = fmaxf(__uint_as_float(r[4 * i + 3]) + b.w, 0.0f);
            pk[2 * i] = pack_bf16x2(z0, z1);
            pk[2 * i + 1] = pack_bf16x2(z2, z3);
          }
          tmem_st16(tmem + lane_base + kTmemR + zb * 64 + c0 / 2, pk);
          tmem_st16(tmem + lane_base + kTmemR + zb * 64 + c0 / 2 + 16, pk + 16);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&z_empty[zb]);
            mbar_arrive(&r_full[zb]);
          }
        }
        if (cp != 0) continue;
        // logits of pair (tile row, entry e)
        const int slot = a.ent_slot[e];
        const uint32_t lb = u % a.nl;
        mbar_wait(&l_full[lb], (u / a.nl) & 1);
        tc_fence_after();
        int best = 0;
        float bestv = 0.0f;
        for (int c0 = 0; c0 < a.C; c0 += 16) {
          uint32_t r[16];
          tmem_ld16_nowait(tmem + lane_base + kTmemL + lb * a.C + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float l = __uint_as_float(r[i]) + b2[c0 + i];
            if ((c0 | i) == 0 || l > bestv) {
              bestv = l;
              best = c0 + i;
            }
            if (a.dbg_logits && valid)
              a.dbg_logits[((size_t)R * a.n_ent + e) * a.C + c0 + i] = l;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&l_empty[lb]);
          mbar_arrive(&w2_empty[wb]);  // b2 (and b1) of this buffer no longer read
        }
        const bool ok = valid && best == label && (pslot < 0 || pslot == slot);
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0 && bal) {
          const size_t idx = a.probe_slot ? (size_t)p : (size_t)p * a.ld + a.ent_col[e];
          atomicAdd(a.counts + idx, __popc(bal));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}


// ---------------------------------------------------------------------------
// CTA-pair variant (dense matrices): two SMs of a cluster run the hidden
// layer as M = 256 tcgen05 MMAs (cta_group::2).  Each CTA keeps its own 128
// eval rows resident and streams only HALF of every W1^T box (64 of the 128
// hidden columns): the W1^T bytes per FLOP per SM halve, which doubles the
// work buffered by the same 5 shared-memory stages -- the v4 kernel was bound
// by exactly that (TMA latency x bytes in flight, profiles/r01_summary.md).
// The pair leader issues every MMA; the follower's TMA loads complete on the
// leader's barriers (cp.async.bulk.tensor .cta_group::2); MMA commits are
// multicast to both CTAs; epilogue warps of both CTAs arrive on the leader's
// barriers.  The second layer (logits, N = C = 16) is also a pair MMA with A
// (bf16 relu(Z + b1)) from each CTA's TMEM and W2^T split 8 + 8 rows.
constexpr uint32_t kPairBox = 64 * 128;  // W1^T half box: 64 rows x 64 bf16
constexpr int kMaxPairStages = 12;

struct PairBars {
  uint64_t a_full, a_empty;
  uint64_t full[kMaxPairStages], empty[kMaxPairStages];
  uint64_t w2_full[2], w2_empty[2];
  uint64_t bias_full[2], bias_empty[2];
  uint64_t z_full[2], z_empty[2], r_full[2], r_empty[2];
  uint64_t l_full[2], l_empty[2];
  // dynamic super-tile queue: the leader's producer takes the next tile from
  // a global counter and publishes it to both CTAs (the follower's copy by
  // st.async); every role walks the queue in order; the leader's tq_empty
  // collects the releases of both CTAs' consumers
  uint64_t tq_full[4], tq_empty[4];
  int tq[4];
  uint32_t tmem_base;
};

__device__ __forceinline__ void st_async_s32(uint32_t addr, int v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.s32 [%0], %1, [%2];" ::"r"(addr),
               "r"(v), "r"(mbar)
               : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_eval_pair(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                const __grid_constant__ CUtensorMap map_w2, EvalArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int nkc = a.F / kKC;
  const int nh = a.H / kHalf;
  const uint32_t w2h = (uint32_t)(a.H / 64) * 1024u;  // this CTA's W2^T half: 8 rows per atom
  uint8_t* sA = smem;
  uint8_t* sB = sA + nkc * kAChunk;
  uint8_t* sW2 = sB + a.stages * kPairBox;
  uint8_t* sBias = sW2 + 2 * w2h;
  PairBars* bars = reinterpret_cast<PairBars*>(sBias + 2 * a.bias_bytes);
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  auto lead = [&](uint64_t* bar) { return mapa_shared(smem_u32(bar), 0); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int n_super = (a.n_rows + 2 * kTileRows - 1) / (2 * kTileRows);

  if (warp == 0 && lane == 0) {
    if (smem_u32(smem) & 1023u) __trap();
    tma_prefetch(&map_x);
    tma_prefetch(&map_w);
    tma_prefetch(&map_w2);
    mbar_init(&bars->a_full, 1);
    mbar_init(&bars->a_empty, 1);
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->w2_full[b], 1);
      mbar_init(&bars->w2_empty[b], 1);
      mbar_init(&bars->bias_full[b], 1);
      mbar_init(&bars->bias_empty[b], 4);
      mbar_init(&bars->z_full[b], 1);
      mbar_init(&bars->z_empty[b], 16);
      mbar_init(&bars->r_full[b], 16);
      mbar_init(&bars->r_empty[b], 1);
      mbar_init(&bars->l_full[b], 1);
      mbar_init(&bars->l_empty[b], 8);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bars->tq_full[i], 1);
      mbar_init(&bars->tq_empty[i], 1 + 8 + 8 + 1);  // MMA, 2 x 8 epilogue warps, follower producer
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(&bars->tmem_base, 512);
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers and TMEM are live before any cross-CTA use
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    int stage = 0;
    uint32_t sph = 0, u = 0;
    for (uint32_t t = 0;; ++t) {
      const int qs = t & 3;
      int m;
      if (leader) {
        if (t >= 4) mbar_wait(&bars->tq_empty[qs], ((t >> 2) - 1) & 1);
        if (lane == 0) {
          const int g = atomicAdd(a.tile_ctr, 1);
          m = g < n_super ? g : -1;
          bars->tq[qs] = m;
          st_async_s32(mapa_shared(smem_u32(&bars->tq[qs]), 1), m,
                       mapa_shared(smem_u32(&bars->tq_full[qs]), 1));
          mbar_arrive(&bars->tq_full[qs]);
        }
        m = __shfl_sync(0xffffffffu, m, 0);
      } else {
        if (lane == 0) mbar_expect_tx(&bars->tq_full[qs], 4);
        mbar_wait(&bars->tq_full[qs], (t >> 2) & 1);
        m = bars->tq[qs];
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(lead(&bars->tq_empty[qs]));
      }
      if (m < 0) break;
      if (t > 0) mbar_wait(&bars->a_empty, (t - 1) & 1);
      if (elect_one()) {
        if (leader) mbar_expect_tx(&bars->a_full, 2u * nkc * kAChunk);
        for (int h2 = 0; h2 < 2; ++h2) {
          int b = m * 4 + (int)rank * 2 + h2;
          if (b * 64 >= a.n_rows) b = 0;  // padding rows: any valid box, masked later
          const int p = (b * 64) / a.S, soff = (b * 64) % a.S;
          const int row = a.cams[p] * a.S + soff;
          for (int kc = 0; kc < nkc; ++kc)
            tma_load_2d_pair(sA + kc * kAChunk + h2 * (kAChunk / 2), &map_x, kc * kKC, row,
                             lead(&bars->a_full));
        }
      }
      __syncwarp();
      for (int e = tile_ent_begin(a, m), e1 = tile_ent_end(a, m); e < e1; ++e, ++u) {
        const int slot = a.ent_slot[e];
        const int wb = u & 1;
        mbar_wait(&bars->w2_empty[wb], ((u >> 1) & 1) ^ 1);
        mbar_wait(&bars->bias_empty[wb], ((u >> 1) & 1) ^ 1);
        if (elect_one()) {
          if (leader) mbar_expect_tx(&bars->w2_full[wb], 2u * w2h);
          tma_load_5d_pair(sW2 + wb * w2h, &map_w2, 0, 0, (int)rank, 0, slot,
                           lead(&bars->w2_full[wb]));
          mbar_expect_tx(&bars->bias_full[wb], a.bias_bytes);
          bulk_load(sBias + wb * a.bias_bytes, a.w2t + (size_t)slot * a.img_bytes + a.w2t_bytes,
                    a.bias_bytes, &bars->bias_full[wb]);
        }
        __syncwarp();
        for (int hf = 0; hf < nh; ++hf) {
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&bars->empty[stage], sph ^ 1);
            if (elect_one()) {
              if (leader) mbar_expect_tx(&bars->full[stage], 2u * kPairBox);
              tma_load_2d_pair(sB + stage * kPairBox, &map_w, kc * kKC,
                               slot * a.H + hf * kHalf + (int)rank * 64, lead(&bars->full[stage]));
            }
            __syncwarp();
            if (++stage == a.stages) {
              stage = 0;
              sph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------- MMA issuer (leader) ----
    if (leader) {
      const uint32_t id1 = idesc(2 * kTileRows, kHalf, kFmtBF16);
      const uint32_t id2 = idesc(2 * kTileRows, a.C, kFmtBF16);
      const uint64_t dA0 = desc_kmajor_sw128(smem_u32(sA));
      const uint64_t dB0 = desc_kmajor_sw128(smem_u32(sB));
      const uint64_t dW0 = desc_kmajor_sw128(smem_u32(sW2));
      int stage = 0;
      uint32_t sph = 0, u = 0, t = 0;
      long prev = -1;
      auto layer2 = [&](uint32_t w) {
        const uint32_t uw = w / nh, hw = w % nh;
        const uint32_t rb = w & 1, lb = uw % a.nl, wb = uw & 1;
        if (hw == 0) {
          mbar_wait(&bars->w2_full[wb], (uw >> 1) & 1);
          mbar_wait(&bars->l_empty[lb], ((uw / a.nl) & 1) ^ 1);
        }
        mbar_wait(&bars->r_full[rb], (w >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dW = dW0 + ((wb * w2h) >> 4);
#pragma unroll
          for (int k16 = 0; k16 < kHalf / 16; ++k16) {
            const int kg = hw * kHalf + k16 * 16;
            mma2_bf16_ts(tmem + kTmemL + lb * a.C, tmem + kTmemR + rb * 64 + k16 * 8,
                         dW + (((kg / 64) * 1024 + (kg % 64) * 2) >> 4), id2, (hw | k16) != 0);
          }
          mma2_commit_mc(&bars->r_empty[rb], 3);
          if (hw == (uint32_t)nh - 1) {
            mma2_commit_mc(&bars->l_full[lb], 3);
            mma2_commit_mc(&bars->w2_empty[wb], 3);
          }
        }
        __syncwarp();
      };
      for (;; ++t) {
        const int qs = t & 3;
        mbar_wait(&bars->tq_full[qs], (t >> 2) & 1);
        const int m = bars->tq[qs];
        if (m < 0) break;
        mbar_wait(&bars->a_full, t & 1);
        tc_fence_after();
        for (int e = tile_ent_begin(a, m), e1 = tile_ent_end(a, m); e < e1; ++e, ++u) {
          for (int hf = 0; hf < nh; ++hf) {
            const uint32_t v = u * nh + hf, zb = v & 1;
            mbar_wait(&bars->z_empty[zb], ((v >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t dz = tmem + kTmemZ + zb * kHalf;
            for (int kc = 0; kc < nkc; ++kc) {
              mbar_wait(&bars->full[stage], sph);
              tc_fence_after();
              if (elect_one()) {
                const uint64_t da = dA0 + ((kc * kAChunk) >> 4);
                const uint64_t db = dB0 + ((stage * kPairBox) >> 4);
#pragma unroll
                for (int kk = 0; kk < kKC / 16; ++kk)
                  mma2_bf16_ss(dz, da + kk * 2, db + kk * 2, id1, (kc | kk) != 0);
                mma2_commit_mc(&bars->empty[stage], 3);
              }
              __syncwarp();
              if (++stage == a.stages) {
                stage = 0;
                sph ^= 1;
              }
            }
            if (elect_one()) mma2_commit_mc(&bars->z_full[zb], 3);
            __syncwarp();
            if (prev >= 0) layer2((uint32_t)prev);
            prev = v;
          }
        }
        if (elect_one()) mma2_commit_mc(&bars->a_empty, 3);
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->tq_empty[qs]);
      }
      if (prev >= 0) layer2((uint32_t)prev);
    }
  } else {
    // ---------------------------------------------- epilogue (both CTAs) --
    const int q = warp & 3;
    const int cp = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t u = 0;
    for (uint32_t t = 0;; ++t) {
      const int qs = t & 3;
      mbar_wait(&bars->tq_full[qs], (t >> 2) & 1);
      const int m = bars->tq[qs];
      if (m < 0) break;
      const int R = m * 2 * kTileRows + (int)rank * kTileRows + row;
      const bool valid = R < a.n_rows;
      const int p = valid ? R / a.S : 0;
      const int label = valid ? a.labels[(size_t)a.cams[p] * a.S + (R % a.S)] : -1;
      for (int e = tile_ent_begin(a, m), e1 = tile_ent_end(a, m); e < e1; ++e, ++u) {
        const uint32_t wb = u & 1;
        const int slot = a.ent_slot[e];
        const float* b1 = reinterpret_cast<const float*>(sBias + wb * a.bias_bytes);
        const float* b2 = b1 + a.H;
        mbar_wait(&bars->bias_full[wb], (u >> 1) & 1);
        for (int hf = 0; hf < nh; ++hf) {
          const uint32_t v = u * nh + hf, zb = v & 1;
          const int c0 = cp * 64;
          mbar_wait(&bars->z_full[zb], (v >> 1) & 1);
          mbar_wait(&bars->r_empty[zb], ((v >> 1) & 1) ^ 1);
          tc_fence_after();
          uint32_t r[64];
          tmem_ld32_nowait(tmem + lane_base + kTmemZ + zb * kHalf + c0, r);
          tmem_ld32_nowait(tmem + lane_base + kTmemZ + zb * kHalf + c0 + 32, r + 32);
          tmem_ld_wait();
          const float4* bb = reinterpret_cast<const float4*>(b1 + hf * kHalf + c0);
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float4 b = bb[i];
            const float z0 = fmaxf(__uint_as_float(r[4 * i + 0]) + b.x, 0.0f);
            const float z1 = fmaxf(__uint_as_float(r[4 * i + 1]) + b.y, 0.0f);
            const float z2 = fmaxf(__uint_as_float(r[4 * i + 2]) + b.z, 0.0f);
            const float z3 = fmaxf(__uint_as_float(r[4 * i + 3]) + b.w, 0.0f);
            pk[2 * i] = pack_bf16x2(z0, z1);
            pk[2 * i + 1] = pack_bf16x2(z2, z3);
          }
          tmem_st16(tmem + lane_base + kTmemR + zb * 64 + c0 / 2, pk);
          tmem_st16(tmem + lane_base + kTmemR + zb * 64 + c0 / 2 + 16, pk + 16);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_cluster(lead(&bars->z_empty[zb]));
            mbar_arrive_cluster(lead(&bars->r_full[zb]));
          }
        }
        if (cp != 0) continue;
        const uint32_t lb = u % a.nl;
        mbar_wait(&bars->l_full[lb], (u / a.nl) & 1);
        tc_fence_after();
        int best = 0;
        float bestv = 0.0f;
        for (int c0 = 0; c0 < a.C; c0 += 16) {
          uint32_t r[16];
          tmem_ld16_nowait(tmem + lane_base + kTmemL + lb * a.C + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float l = __uint_as_float(r[i]) + b2[c0 + i];
            if ((c0 | i) == 0 || l > bestv) {
              bestv = l;
              best = c0 + i;
            }
            if (a.dbg_logits && valid)
              a.dbg_logits[((size_t)R * a.n_ent + e) * a.C + c0 + i] = l;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(lead(&bars->l_empty[lb]));
          mbar_arrive(&bars->bias_empty[wb]);
        }
        // pairs mode: a row counts only under its probe's own slot
        const bool ok = valid && best == label && (!a.probe_slot || a.probe_slot[p] == slot);
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0 && bal) {
          const size_t idx = a.probe_slot ? (size_t)p : (size_t)p * a.ld + a.ent_col[e];
          atomicAdd(a.counts + idx, __popc(bal));
        }
      }
      __syncwarp();
      if (lane == 0) {  // this warp is done with the tile's queue slot
        if (leader)
          mbar_arrive(&bars->tq_empty[qs]);
        else
          mbar_arrive_cluster(lead(&bars->tq_empty[qs]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs into the follower's TMEM are all complete
  if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

// ---------------------------------------------------------------------------
// Wide variant (F > 512 -- the detection head of BASELINE configs[4], F = 1024,
// H = 1024, C = 96): a 128-row X tile of F = 1024 bf16 (256 KB) does not fit
// in shared memory, so X streams WITH the model: every pipeline stage carries
// the tile's X chunk (128 rows x 64 features: the two 64-row camera boxes)
// and the W1^T box of the same K chunk (128 hidden x 64 features), both
// 128B-swizzled K-major, and one MMA step consumes both.  The X chunk is
// re-read from L2 once per hidden half, the W1^T box once per tile.  W2^T
// streams per hidden half (C rows x 128 K = two swizzle atoms: one
// contiguous bulk copy of the slot's image) through two buffers, b1 | b2 per
// entry through two more.  TMEM, warp roles, epilogue and numerics are those
// of k_eval_fused (the logits single-buffered when 2 C > 128), so a row's
// count does not depend on which kernel evaluated it.
constexpr uint32_t kWideStage = kAChunk + kBoxBytes;  // 32 KB: X chunk | W1^T box

struct WideBars {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t w2_full[2], w2_empty[2];
  uint64_t bias_full[2], bias_empty[2];
  uint64_t z_full[2], z_empty[2], r_full[2], r_empty[2];
  uint64_t l_full[2], l_empty[2];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads, 1)
    k_eval_wide(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                EvalArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int nkc = a.F / kKC;
  const int nh = a.H / kHalf;
  const uint32_t w2c = (uint32_t)a.C * 256u;  // W2^T of one hidden half: 2 atoms x C rows x 128 B
  uint8_t* sS = smem;                         // stages x (X chunk | W1^T box)
  uint8_t* sW2 = sS + a.stages * kWideStage;  // 2 x w2t_stride (W2^T hidden halves)
  uint8_t* sBias = sW2 + 2 * a.w2t_stride;    // 2 x bias_bytes (b1 | b2)
  WideBars* bars = reinterpret_cast<WideBars*>(sBias + 2 * a.bias_bytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    if (smem_u32(smem) & 1023u) __trap();
    tma_prefetch(&map_x);
    tma_prefetch(&map_w);
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->w2_full[b], 1);
      mbar_init(&bars->w2_empty[b], 1);    // the layer-2 MMA commit
      mbar_init(&bars->bias_full[b], 32);  // the producer warp's lanes
      mbar_init(&bars->bias_empty[b], 256);  // every epilogue thread: b1 read, and b2 by the logits warps
      mbar_init(&bars->z_full[b], 1);
      mbar_init(&bars->z_empty[b], 8);
      mbar_init(&bars->r_full[b], 8);
      mbar_init(&bars->r_empty[b], 1);
      mbar_init(&bars->l_full[b], 1);
      mbar_init(&bars->l_empty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    int stage = 0;
    uint32_t sph = 0, u = 0;
    for (int m = blockIdx.x; m < a.n_tiles; m += gridDim.x) {
      int xrow[2];
      for (int h2 = 0; h2 < 2; ++h2) {
        int b = m * 2 + h2;
        if (b * 64 >= a.n_rows) b = 0;  // padding rows: any valid box, masked later
        xrow[h2] = a.cams[(b * 64) / a.S] * a.S + (b * 64) % a.S;
      }
      for (int e = tile_ent_begin(a, m), e1 = tile_ent_end(a, m); e < e1; ++e, ++u) {
        const int slot = a.ent_slot[e];
        const uint8_t* img = a.w2t + (size_t)slot * a.img_bytes;
        for (int hf = 0; hf < nh; ++hf) {
          const uint32_t v = u * nh + hf;
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&bars->empty[stage], sph ^ 1);
            if (elect_one()) {
              uint8_t* st = sS + stage * kWideStage;
              mbar_expect_tx(&bars->full[stage], kWideStage);
              tma_load_2d(st, &map_x, kc * kKC, xrow[0], &bars->full[stage]);
              tma_load_2d(st + kAChunk / 2, &map_x, kc * kKC, xrow[1], &bars->full[stage]);
              tma_load_2d(st + kAChunk, &map_w, kc * kKC, slot * a.H + hf * kHalf,
                          &bars->full[stage]);
            }
            __syncwarp();
            if (++stage == a.stages) {
              stage = 0;
              sph ^= 1;
            }
          }
          // after the half's stages (they pace the tensor cores): the entry's
          // biases once, then this half's W2^T (read by its layer-2 MMAs,
          // which the MMA warp issues after the NEXT half's K loop)
          if (hf == 0) {  // (4.5 KB: plain warp copies, every lane arrives)
            const uint32_t bb = u & 1;
            mbar_wait(&bars->bias_empty[bb], ((u >> 1) & 1) ^ 1);
            const uint4* src = reinterpret_cast<const uint4*>(img + a.w2t_bytes);
            uint4* dst = reinterpret_cast<uint4*>(sBias + bb * a.bias_bytes);
            for (uint32_t i = lane; i < a.bias_bytes / 16; i += 32) dst[i] = __ldg(src + i);
            mbar_arrive(&bars->bias_full[bb]);
          }
          const uint32_t wb = v & 1;
          mbar_wait(&bars->w2_empty[wb], ((v >> 1) & 1) ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&bars->w2_full[wb], w2c);
            bulk_load(sW2 + wb * a.w2t_stride, img + (size_t)hf * w2c, w2c, &bars->w2_full[wb]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    const uint32_t id1 = idesc(kTileRows, kHalf, kFmtBF16);
    const uint32_t id2 = idesc(kTileRows, a.C, kFmtBF16);
    const uint64_t dS0 = desc_kmajor_sw128(smem_u32(sS));
    const uint64_t dW0 = desc_kmajor_sw128(smem_u32(sW2));
    int stage = 0;
    uint32_t sph = 0, u = 0;
    long prev = -1;  // pending layer-2 for sequence index prev (v = u * nh + hf)
    auto layer2 = [&](uint32_t w) {
      const uint32_t uw = w / nh, hw = w % nh;
      const uint32_t rb = w & 1, wb = w & 1, lb = uw % a.nl;
      if (hw == 0) mbar_wait(&bars->l_empty[lb], ((uw / a.nl) & 1) ^ 1);
      mbar_wait(&bars->w2_full[wb], (w >> 1) & 1);
      mbar_wait(&bars->r_full[rb], (w >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dW = dW0 + ((wb * a.w2t_stride) >> 4);
#pragma unroll
        for (int k16 = 0; k16 < kHalf / 16; ++k16) {
          const int kg = k16 * 16;  // K index within the hidden half
          mma_bf16_ts(tmem + kTmemL + lb * a.C, tmem + kTmemR + rb * 64 + k16 * 8,
                      dW + (((kg / 64) * (a.C * 128) + (kg % 64) * 2) >> 4), id2,
                      (hw | k16) != 0);
        }
        mma_commit(&bars->r_empty[rb]);
        mma_commit(&bars->w2_empty[wb]);
        if (hw == (uint32_t)nh - 1) mma_commit(&bars->l_full[lb]);
      }
      __syncwarp();
    };
    for (int m = blockIdx.x; m < a.n_tiles; m += gridDim.x) {
      for (int e = tile_ent_begin(a, m), e1 = tile_ent_end(a, m); e < e1; ++e, ++u) {
        for (int hf = 0; hf < nh; ++hf) {
          const uint32_t v = u * nh + hf, zb = v & 1;
          mbar_wait(&bars->z_empty[zb], ((v >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dz = tmem + kTmemZ + zb * kHalf;
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&bars->full[stage], sph);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t da = dS0 + ((stage * kWideStage) >> 4);
              const uint64_t db = da + (kAChunk >> 4);
#pragma unroll
              for (int kk = 0; kk < kKC / 16; ++kk)
                mma_bf16_ss(dz, da + kk * 2, db + kk * 2, id1, (kc | kk) != 0);
              mma_commit(&bars->empty[stage]);
            }
            __syncwarp();
            if (++stage == a.stages) {
              stage = 0;
              sph ^= 1;
            }
          }
          if (elect_one()) mma_commit(&bars->z_full[zb]);
          __syncwarp();
          if (prev >= 0) layer2((uint32_t)prev);
          prev = v;
        }
      }
    }
    if (prev >= 0) layer2((uint32_t)prev);
  } else {
    // ----------------------------------------------------------- epilogue --
    // as k_eval_fused: 8 warps, two per TMEM lane quadrant, each converting
    // 64 of a half's 128 Z columns; the cp == 0 warps also read the logits
    const int q = warp & 3;
    const int cp = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t u = 0;
    for (int m = blockIdx.x; m < a.n_tiles; m += gridDim.x) {
      const int R = m * kTileRows + row;
      const bool valid = R < a.n_rows;
      const int p = valid ? R / a.S : 0;
      const int label = valid ? a.labels[(size_t)a.cams[p] * a.S + (R % a.S)] : -1;
      const int pslot = (valid && a.probe_slot) ? a.probe_slot[p] : -1;
      for (int e = tile_ent_begin(a, m), e1 = tile_ent_end(a, m); e < e1; ++e, ++u) {
        const uint32_t bb = u & 1;
        const float* b1 = reinterpret_cast<const float*>(sBias + bb * a.bias_bytes);
        const float* b2 = b1 + a.H;
        mbar_wait(&bars->bias_full[bb], (u >> 1) & 1);
        for (int hf = 0; hf < nh; ++hf) {
          const uint32_t v = u * nh + hf, zb = v & 1;
          const int c0 = cp * 64;
          mbar_wait(&bars->z_full[zb], (v >> 1) & 1);
          mbar_wait(&bars->r_empty[zb], ((v >> 1) & 1) ^ 1);
          tc_fence_after();
          uint32_t r[64];
          tmem_ld32_nowait(tmem + lane_base + kTmemZ + zb * kHalf + c0, r);
          tmem_ld32_nowait(tmem + lane_base + kTmemZ + zb * kHalf + c0 + 32, r + 32);
          tmem_ld_wait();
          const float4* bv = reinterpret_cast<const float4*>(b1 + hf * kHalf + c0);
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float4 b = bv[i];
            const float z0 = fmaxf(__uint_as_float(r[4 * i + 0]) + b.x, 0.0f);
            const float z1 = fmaxf(__uint_as_float(r[4 * i + 1]) + b.y, 0.0f);
            const float z2 = fmaxf(__uint_as_float(r[4 * i + 2]) + b.z, 0.0f);
            const float z3 = fmaxf(__uint_as_float(r[4 * i + 3]) + b.w, 0.0f);
            pk[2 * i] = pack_bf16x2(z0, z1);
            pk[2 * i + 1] = pack_bf16x2(z2, z3);
          }
          tmem_st16(tmem + lane_base + kTmemR + zb * 64 + c0 / 2, pk);
          tmem_st16(tmem + lane_base + kTmemR + zb * 64 + c0 / 2 + 16, pk + 16);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&bars->z_empty[zb]);
            mbar_arrive(&bars->r_full[zb]);
          }
        }
        if (cp != 0) {  // this thread's last b1 read of the entry is done
          mbar_arrive(&bars->bias_empty[bb]);
          continue;
        }
        const int slot = a.ent_slot[e];
        const uint32_t lb = u % a.nl;
        mbar_wait(&bars->l_full[lb], (u / a.nl) & 1);
        tc_fence_after();
        int best = 0;
        float bestv = 0.0f;
        for (int c0 = 0; c0 < a.C; c0 += 16) {
          uint32_t r[16];
          tmem_ld16_nowait(tmem + lane_base + kTmemL + lb * a.C + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float l = __uint_as_float(r[i]) + b2[c0 + i];
            if ((c0 | i) == 0 || l > bestv) {
              bestv = l;
              best = c0 + i;
            }
            if (a.dbg_logits && valid)
              a.dbg_logits[((size_t)R * a.n_ent + e) * a.C + c0 + i] = l;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->l_empty[lb]);
        mbar_arrive(&bars->bias_empty[bb]);  // b1 (all halves done) and b2 no longer read
        const bool ok = valid && best == label && (pslot < 0 || pslot == slot);
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0 && bal) {
          const size_t idx = a.probe_slot ? (size_t)p : (size_t)p * a.ld + a.ent_col[e];
          atomicAdd(a.counts + idx, __popc(bal));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------ shadows ------
// W1^T (bf16, [slot][H][F]) from the fp32 masters W1 [F][H]: 32x32 transpose.
__global__ void k_shadow_w1t(int F, int H, const int* slots, const float* wbase, size_t wstride,
                             uint16_t* w1t, bool w1_t) {
  __shared__ float t[32][33];
  const int slot = slots[blockIdx.z];
  const float* W1 = wbase + (size_t)slot * wstride;
  const int f0 = blockIdx.x * 32, h0 = blockIdx.y * 32;
  if (w1_t) {  // masters already [H][F]: convert in place order
    uint16_t* dst = w1t + (size_t)slot * H * F;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const size_t o = (size_t)(h0 + i) * F + f0 + threadIdx.x;
      dst[o] = (uint16_t)(pack_bf16x2(W1[o], 0.0f) & 0xFFFF);
    }
    return;
  }
  for (int i = threadIdx.y; i < 32; i += blockDim.y)
    t[i][threadIdx.x] = W1[(size_t)(f0 + i) * H + h0 + threadIdx.x];
  __syncthreads();
  uint16_t* dst = w1t + (size_t)slot * H * F;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const float x = t[threadIdx.x][i];  // W1[f0 + tx][h0 + i]
    const uint32_t pk = pack_bf16x2(x, 0.0f);
    dst[(size_t)(h0 + i) * F + f0 + threadIdx.x] = (uint16_t)(pk & 0xFFFF);
  }
}

// W2^T image: C rows x H (K) bf16, K-major, 128-byte swizzle atoms of 64 K
// elements; atom kb of row n at kb*(C*128) + n*128, 16-byte chunk j of the
// row stored at chunk j ^ (n % 8).
// One block per (slot, 64-wide K atom): the detection head's 96 x 1024 image
// is 16 blocks' work, not one block's (a serial chain's snapshot images
// are rebuilt per call, on the evaluation's critical path).
__global__ void k_shadow_w2t(int F, int H, int C, const int* slots, const float* wbase,
                             size_t wstride, uint8_t* w2t, uint32_t img_bytes) {
  const int slot = slots[blockIdx.x];
  const float* b1 = wbase + (size_t)slot * wstride + (size_t)F * H;
  const float* W2 = b1 + H;
  const float* b2 = W2 + (size_t)H * C;
  uint8_t* img = w2t + (size_t)slot * img_bytes;
  if (blockIdx.y == 0) {
    float* ib = reinterpret_cast<float*>(img + (size_t)C * H * 2);
    for (int i = threadIdx.x; i < H; i += blockDim.x) ib[i] = b1[i];
    for (int i = threadIdx.x; i < C; i += blockDim.x) ib[H + i] = b2[i];
  }
  const int k0 = blockIdx.y * 64, k1 = min(H, k0 + 64);
  for (int idx = k0 * C + threadIdx.x; idx < k1 * C; idx += blockDim.x) {
    const int n = idx % C, k = idx / C;  // W2[k][n]
    const int kb = k / 64, kw = k % 64;
    const int chunk = (kw * 2) / 16, within = (kw * 2) % 16;
    const size_t off = (size_t)kb * (C * 128) + n * 128 + ((chunk ^ (n & 7)) * 16) + within;
    const uint32_t pk = pack_bf16x2(W2[(size_t)k * C + n], 0.0f);
    *reinterpret_cast<uint16_t*>(img + off) = (uint16_t)(pk & 0xFFFF);
  }
}

__global__ void k_counts_to_acc(size_t n, const int* counts, int S, const uint8_t* mask,
                                double* out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = (mask && !mask[i]) ? __longlong_as_double(0x7ff8000000000000LL)
                              : __ddiv_rn((double)counts[i], (double)S);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ECCO_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      ecco_throw(ECCO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 2-D bf16 row-major [rows][cols] map with a {64, box_rows} box, 128-B swizzle.
CUtensorMap make_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) ecco_throw(ECCO_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

// 5-D view of the per-slot W2^T images for the CTA-pair kernel: (64 bf16 of
// a 128-byte row, 8 rows, 2 halves, H/64 atoms, slots); one box = one CTA's
// half (8 rows of every atom), copied as-is (the image is pre-swizzled).
CUtensorMap make_w2_pair_map(const void* base, uint64_t slots, int H, int C, uint32_t img_bytes) {
  CUtensorMap m;
  const cuuint64_t dims[5] = {64, 8, 2, (cuuint64_t)(H / 64), slots};
  const cuuint64_t strides[4] = {128, 1024, (cuuint64_t)C * 128, img_bytes};
  const cuuint32_t box[5] = {64, 8, 1, (cuuint32_t)(H / 64), 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base),
                                 dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) ecco_throw(ECCO_ERR_CUDA, "cuTensorMapEncodeTiled (W2^T pair view) failed");
  return m;
}

// The CTA-pair kernel serves dense matrices with C == 16; ECCO_EVAL_PAIR=0
// forces the single-CTA kernel (tests run both).
bool pair_enabled(const ecco_config& g) {
  const char* e = getenv("ECCO_EVAL_PAIR");
  return g.num_classes == 16 && g.feat_dim <= 512 && !(e && e[0] == '0');
}

// Test knob: caps the persistent grid (CTA pairs / CTAs) so a handful of
// cameras exercise the multi-tile regime of the production grid (C4: ~34
// super tiles per pair) -- queue wrap, per-tile barrier phases, TMEM buffer
// parity across tiles.  Unset or <= 0: no cap.
int grid_cap(const char* name) {
  const char* e = getenv(name);
  const int v = e ? atoi(e) : 0;
  return v > 0 ? v : (1 << 30);
}

int sm_count(int device) {
  int n = 0;
  ECCO_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
  return n;
}

}  // namespace

namespace fused {

uint32_t w2t_bytes(const ecco_config& g) { return (uint32_t)g.num_classes * g.hidden_dim * 2; }
uint32_t img_bytes(const ecco_config& g) {
  return (w2t_bytes(g) + 4u * (g.hidden_dim + g.num_classes) + 15u) & ~15u;
}

CUtensorMap tensor_map_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return make_map(base, rows, cols, box_rows);
}

bool pair_supported(const ecco_ctx* ctx) {
  return pair_enabled(ctx->cfg);
}

// k_eval_fused: the 128-row X tile resident in shared memory (F <= 512)
static bool resident_supported(const ecco_config& g) {
  return g.feat_dim % 64 == 0 && g.feat_dim <= 512 && g.hidden_dim % kHalf == 0 &&
         g.num_classes % 16 == 0 && g.num_classes <= 64 &&
         (size_t)g.num_classes * g.hidden_dim * 2 <= 16384 && g.eval_samples % 64 == 0 &&
         g.feat_dim / 64 * 16384 + 2 * ((w2t_bytes(g) + 1023) / 1024 * 1024) +
                 2 * (img_bytes(g) - w2t_bytes(g)) + sizeof(EvalBars) + 2 * 16384 <= 232448;
}

// k_eval_wide: X streamed with the model (any F % 64 == 0; logits C <= 128
// columns of TMEM beside Z and R), at least 3 pipeline stages.  ECCO_EVAL_WIDE=0
// leaves wide shapes on the general (unfused) path.
static uint32_t wide_w2_stride(const ecco_config& g) {
  return ((uint32_t)g.num_classes * 256u + 1023u) & ~1023u;
}
static size_t wide_fixed_smem(const ecco_config& g) {
  return 2 * (size_t)wide_w2_stride(g) + 2 * (size_t)(img_bytes(g) - w2t_bytes(g)) +
         sizeof(WideBars);
}
static bool wide_eval_supported(const ecco_config& g) {
  const char* e = getenv("ECCO_EVAL_WIDE");
  return !(e && e[0] == '0') && g.feat_dim % 64 == 0 && g.hidden_dim % kHalf == 0 &&
         g.num_classes % 16 == 0 && g.num_classes <= 128 && g.eval_samples % 64 == 0 &&
         wide_fixed_smem(g) + 3 * (size_t)kWideStage <= 232448;
}

bool supported(const ecco_ctx* ctx) {
  return resident_supported(ctx->cfg) || wide_eval_supported(ctx->cfg);
}


void refresh_shadow(ecco_ctx* ctx, Shadow& sh, const float* wbase, size_t wstride,
                    const std::vector<int>& slots, const std::vector<int>* w1t_slots) {
  if (slots.empty()) return;
  const ecco_config& g = ctx->cfg;
  int* d_sl = ctx->upload(10, slots.data(), slots.size());
  const int n = (int)slots.size();
  const std::vector<int>& s1 = w1t_slots ? *w1t_slots : slots;
  if (!s1.empty()) {
    const int* d_s1 = w1t_slots ? ctx->upload(15, s1.data(), s1.size()) : d_sl;
    k_shadow_w1t<<<dim3(g.feat_dim / 32, g.hidden_dim / 32, (unsigned)s1.size()), dim3(32, 8), 0,
                   ctx->stream>>>(g.feat_dim, g.hidden_dim, d_s1, wbase, wstride, sh.w1t, ctx->w1_t);
    ECCO_LAUNCHED(ctx);
  }
  k_shadow_w2t<<<dim3(n, (g.hidden_dim + 63) / 64), 256, 0, ctx->stream>>>(
      g.feat_dim, g.hidden_dim, g.num_classes, d_sl, wbase, wstride, sh.w2t, img_bytes(g));
  ECCO_LAUNCHED(ctx);
}

void refresh_shadow_dev(ecco_ctx* ctx, Shadow& sh, const float* wbase, size_t wstride,
                        const int* d_slots, int n, const int* d_w1t_slots, int n1) {
  if (n == 0) return;
  const ecco_config& g = ctx->cfg;
  if (n1 > 0) {
    k_shadow_w1t<<<dim3(g.feat_dim / 32, g.hidden_dim / 32, (unsigned)n1), dim3(32, 8), 0,
                   ctx->stream>>>(g.feat_dim, g.hidden_dim, d_w1t_slots, wbase, wstride, sh.w1t,
                                  ctx->w1_t);
    ECCO_LAUNCHED(ctx);
  }
  k_shadow_w2t<<<dim3(n, (g.hidden_dim + 63) / 64), 256, 0, ctx->stream>>>(
      g.feat_dim, g.hidden_dim, g.num_classes, d_slots, wbase, wstride, sh.w2t, img_bytes(g));
  ECCO_LAUNCHED(ctx);
}

void shadow_w1t(ecco_ctx* ctx, const int* d_slots, int n, const float* wbase, size_t wstride,
                uint16_t* w1t) {
  if (n == 0) return;
  const ecco_config& g = ctx->cfg;
  k_shadow_w1t<<<dim3(g.feat_dim / 32, g.hidden_dim / 32, n), dim3(32, 8), 0, ctx->stream>>>(
      g.feat_dim, g.hidden_dim, d_slots, wbase, wstride, w1t, ctx->w1_t);
  ECCO_LAUNCHED(ctx);
}

void init_shadow(ecco_ctx* ctx, Shadow& sh, size_t images) {
  const ecco_config& g = ctx->cfg;
  const size_t slots = images ? images : (size_t)g.max_jobs;
  ECCO_CUDA(cudaMalloc((void**)&sh.w1t, slots * g.hidden_dim * g.feat_dim * 2));
  ECCO_CUDA(cudaMalloc((void**)&sh.w2t, slots * img_bytes(g)));
  sh.map_w = new CUtensorMap(make_map(sh.w1t, slots * g.hidden_dim, g.feat_dim, kHalf));
  sh.map_w_pair = new CUtensorMap(make_map(sh.w1t, slots * g.hidden_dim, g.feat_dim, 64));
  if (g.num_classes == 16)
    sh.map_w2_pair = new CUtensorMap(make_w2_pair_map(sh.w2t, slots, g.hidden_dim, g.num_classes,
                                                      img_bytes(g)));
}

void free_shadow(Shadow& sh) {
  if (sh.w1t) cudaFree(sh.w1t);
  if (sh.w2t) cudaFree(sh.w2t);
  delete (CUtensorMap*)sh.map_w;
  delete (CUtensorMap*)sh.map_w_pair;
  delete (CUtensorMap*)sh.map_w2_pair;
  sh = Shadow{};
}

void eval_counts(ecco_ctx* ctx, const Shadow& sh, const float* wbase, size_t wstride,
                 int n_probes, const int* d_cams, int n_ent, const int* d_ent_slot,
                 const int* d_ent_col, int n_tiles_override, const int* d_tile_ebeg,
                 const int* d_probe_slot, int ld, int* d_counts, float* dbg_logits,
                 double live_pairs, bool pair_tiles) {
  const ecco_config& g = ctx->cfg;
  if (!ctx->map_x) ctx->map_x = new CUtensorMap(make_map(ctx->d_eval, (uint64_t)g.max_cameras * g.eval_samples,
                                                         g.feat_dim, 64));
  EvalArgs a{};
  a.n_rows = n_probes * g.eval_samples;
  a.S = g.eval_samples;
  a.F = g.feat_dim;
  a.H = g.hidden_dim;
  a.C = g.num_classes;
  a.n_tiles = n_tiles_override > 0 ? n_tiles_override : (a.n_rows + kTileRows - 1) / kTileRows;
  a.cams = d_cams;
  a.labels = ctx->d_eval_labels;
  a.ent_slot = d_ent_slot;
  a.ent_col = d_ent_col;
  a.n_ent = n_ent;
  a.tile_ebeg = d_tile_ebeg;
  a.probe_slot = d_probe_slot;
  a.ld = ld;
  a.counts = d_counts;
  a.wbase = wbase;
  a.wstride = wstride;
  a.w2t = sh.w2t;
  a.w2t_bytes = w2t_bytes(g);
  a.img_bytes = img_bytes(g);
  a.w2t_stride = (a.w2t_bytes + 1023u) & ~1023u;
  a.bias_bytes = a.img_bytes - a.w2t_bytes;
  a.nl = 2 * g.num_classes <= 128 ? 2 : 1;
  a.dbg_logits = dbg_logits;
  const size_t fixed = (size_t)(a.F / kKC) * kAChunk + 2 * (size_t)a.w2t_stride +
                       2 * (size_t)a.bias_bytes + sizeof(EvalBars);
  const size_t max_smem = 232448;  // opt-in per-block limit (no static smem)
  const bool resident = resident_supported(g);  // else k_eval_wide (X streamed)
  a.stages = resident ? (int)std::min<size_t>(kMaxStages, (max_smem - fixed) / kBoxBytes) : 0;
  ECCO_REQUIRE(!resident || a.stages >= 2, "fused eval: shared memory too small for the pipeline");
  const size_t smem = fixed + (size_t)a.stages * kBoxBytes;
  static DeviceFlags attr;  // per device: the attribute applies to the current device
  if (!attr.done(g.device)) {
    ECCO_CUDA(cudaFuncSetAttribute(k_eval_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)max_smem));
    attr.mark(g.device);
  }
  if (a.n_tiles == 0 || n_ent == 0) return;
  const double flops = 2.0 * live_pairs * g.eval_samples *
                       ((double)g.feat_dim * g.hidden_dim + (double)g.hidden_dim * g.num_classes);
  const double bytes = (double)a.n_rows * g.feat_dim * 2 +
                       (double)n_ent * (g.feat_dim * g.hidden_dim * 2.0 + a.img_bytes) +
                       4.0 * live_pairs;
  const int kind = d_tile_ebeg ? ECCO_KSTAT_EVAL_PAIRS : ECCO_KSTAT_EVAL_MATRIX;
  if ((pair_tiles || (!d_tile_ebeg && !d_probe_slot)) && sh.map_w2_pair && pair_enabled(g)) {
    // CTA-pair kernel: 256-row super tiles, half a W1^T box per CTA per stage
    const size_t pfixed = (size_t)(a.F / kKC) * kAChunk + 2 * (size_t)(a.H / 64) * 1024 +
                          2 * (size_t)a.bias_bytes + sizeof(PairBars);
    a.stages = (int)std::min<size_t>(kMaxPairStages, (max_smem - pfixed) / kPairBox);
    ECCO_REQUIRE(a.stages >= 2, "fused eval (pair): shared memory too small for the pipeline");
    const size_t psmem = pfixed + (size_t)a.stages * kPairBox;
    static DeviceFlags pattr;
    if (!pattr.done(g.device)) {
      ECCO_CUDA(cudaFuncSetAttribute(k_eval_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)max_smem));
      pattr.mark(g.device);
    }
    const int n_super = (a.n_rows + 2 * kTileRows - 1) / (2 * kTileRows);
    const int pairs = std::max(1, std::min({n_super, (sm_count(g.device) - ctx->reserve_sms) / 2,
                                            grid_cap("ECCO_EVAL_MAX_PAIRS")}));
    a.tile_ctr = (int*)ctx->tile_ctr.get(sizeof(int));
    ECCO_CUDA(cudaMemsetAsync(a.tile_ctr, 0, sizeof(int), ctx->stream));
    ECCO_TIMED(ctx, kind, flops, bytes,
               (k_eval_pair<<<2 * pairs, kThreads, psmem, ctx->stream>>>(
                   *(const CUtensorMap*)ctx->map_x, *(const CUtensorMap*)sh.map_w_pair,
                   *(const CUtensorMap*)sh.map_w2_pair, a)));
    ECCO_LAUNCHED(ctx);
    return;
  }
  const int grid = std::max(1, std::min({a.n_tiles, sm_count(g.device) - ctx->reserve_sms,
                                         grid_cap("ECCO_EVAL_MAX_CTAS")}));
  if (!resident) {
    // wide shapes: X streams with the model (k_eval_wide)
    ECCO_REQUIRE(wide_eval_supported(g), "fused eval: unsupported shape");
    a.w2t_stride = wide_w2_stride(g);
    const size_t wfixed = wide_fixed_smem(g);
    a.stages = (int)std::min<size_t>(kMaxStages, (max_smem - wfixed) / kWideStage);
    const size_t wsmem = wfixed + (size_t)a.stages * kWideStage;
    static DeviceFlags wattr;
    if (!wattr.done(g.device)) {
      ECCO_CUDA(cudaFuncSetAttribute(k_eval_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)max_smem));
      wattr.mark(g.device);
    }
    ECCO_TIMED(ctx, kind, flops, bytes,
               (k_eval_wide<<<grid, kThreads, wsmem, ctx->stream>>>(
                   *(const CUtensorMap*)ctx->map_x, *(const CUtensorMap*)sh.map_w, a)));
    ECCO_LAUNCHED(ctx);
    return;
  }
  ECCO_TIMED(ctx, kind, flops, bytes,
             (k_eval_fused<<<grid, kThreads, smem, ctx->stream>>>(*(const CUtensorMap*)ctx->map_x,
                                                                  *(const CUtensorMap*)sh.map_w, a)));
  ECCO_LAUNCHED(ctx);
}

void counts_to_acc(ecco_ctx* ctx, size_t n, const int* d_counts, const uint8_t* d_mask,
                   double* d_out) {
  if (!n) return;
  k_counts_to_acc<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
      n, d_counts, ctx->cfg.eval_samples, d_mask, d_out);
  ECCO_LAUNCHED(ctx);
}

}  // namespace fused
