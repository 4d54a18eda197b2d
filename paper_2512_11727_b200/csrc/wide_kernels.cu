// Fused SGD chain for the wide (detection-head) models of the learned
// backend, BASELINE configs[4]: F = 1024 -> H = 512/1024 -> C <= 128
// (default 96), minibatch 128.  ONE launch runs every group's whole
// micro-window -- steps[j] SGD steps, each gather, forward, softmax
// cross-entropy, backward and update -- on one thread-block cluster of H/64
// CTAs per group (16 for the 1024-wide hidden layer: a non-portable cluster).
// All five contractions run on tcgen05 (kind::f16, bf16 operands, fp32
// accumulation); the numerics are those of the F <= 512 chain
// (train_kernels.cu, tests/test_gpu_learned.py::_step_emulated).
//
// What differs from the F <= 512 chain, and why:
//   * a group's fp32 masters (4.4 MB at 1024-1024-96) do not fit on chip
//     (TMEM 256 KB + smem 227 KB per SM, 16 SMs): CTA r keeps the bf16 W1
//     operand of its 64 hidden units resident in shared memory (F x 128 B)
//     and read-modify-writes its contiguous fp32 master slice W1[64r:64r+64, :]
//     (stored [H][F], 256 KB) in place in the snapshot every step -- an L2
//     round trip (the slice stays L2-resident across the chain); each warp
//     access is 128 contiguous bytes (32 features of one hidden unit: TMEM
//     lane = feature).  ([F][H] with 16-byte accesses measured 4x slower: 32
//     lines per warp instruction.)  dW1 = X^T.bf16(-lr dH) is computed tile by tile
//     (128 features x 64 hidden) into two TMEM buffers; the epilogue warps add
//     it to the master and rebuild that tile's bf16 operand rows.
//   * the 128 sampled rows (256 KB of bf16 at F = 1024) do not fit either:
//     they stream twice per step (forward: K = F; dW1: M = F) through a
//     2-slot ring of 32 KB (two 64-feature chunks of all 128 rows), gathered
//     straight from the frame table by TMA tile::gather4 (4 rows x 128 B per
//     copy, 128B-swizzled where the MMAs read them), one producer warp.
//   * the softmax over C = 96 classes: each CTA's partial logits (128 x 96
//     fp32, 48 KB) go to the CTA owning the row block (128/cs rows) by
//     st.async over DSMEM; one warp per owned row sums the partials in fixed
//     source order, softmax, dL; bf16 dL rows are broadcast into every CTA's
//     operand tile, the owned rows' fp32 db2 partial to every CTA.
//   * the receive buffers (partial logits, dL, db2 partials) and the R / dH
//     operands live inside the W1 operand region, which is dead between the
//     forward's completion and the rebuild of its tile; a CTA therefore
//     announces "forward done" to every CTA of the cluster (fwd_done) before
//     any of them may write its receive buffer.
//
// Roles: warps 0-7 epilogue (TMEM lane quadrant q = warp % 4, column half
// p = warp / 4; also the owner softmax, one warp per owned row), warp 8 the
// row gather (TMA), warp 9 the MMA issuer (one elected lane).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "chain_common.cuh"
#include "ctx.cuh"
#include "learned_common.cuh"
#include "sm100.cuh"

using namespace sm100;
using namespace chain;

namespace {

constexpr int kB = 128;                   // minibatch rows = UMMA M
constexpr int kHS = 64;                   // hidden units per CTA
constexpr int kEpi = 256;                 // epilogue threads (warps 0-7)
constexpr int kThreads = kEpi + 64;       // + warp 8 (gather), warp 9 (MMA)
constexpr int kMaxNM = 8;                 // 128-feature tiles (F <= 1024)
constexpr uint32_t kSlot = 32768;         // ring slot: two 64-feature chunks of 128 rows
constexpr uint32_t kColZ = 0;             // Z, then dL.W2^T (64 columns)
constexpr uint32_t kColL = 64;            // partial logits (C <= 96)
constexpr uint32_t kColW2 = 160;          // dW2 (rows 0-63 = hidden units)
constexpr uint32_t kColW2M = 256;         // the fp32 W2 master slice (rows 0-63)
constexpr uint32_t kColB1 = 352;          // -lr db1 (16 columns)
constexpr uint32_t kColD = 384;           // two dW1 tile buffers of 64 columns

struct WideArgs {
  LDims g;
  const int* slots;
  const int* steps;
  const int32_t* rows;  // [job][row steps][kB] frame-table row of every sampled frame
  const int32_t* labs;  // ... and its label
  int row_step0, rows_T;
  const uint16_t* frames;
  const float* wsrc;  // fp32 models the micro-window starts from (W1 stored [H][F])
  size_t wsrc_stride;
  float* wbase;  // ... and the snapshot it trains in place (may equal wsrc)
  size_t wstride;
  float* losses;
  int loss_T, loss_t;
  int trace;  // ECCO_WIDE_TRACE: clock64 stamps of CTA 0, steps 0-3 (g_wide_trace)
  // Serial mode (n_micro_launch > 1, one job): the launch trains that many
  // consecutive micro-windows, micro-window u's model at wbase + u * wmicro
  int n_micro_launch;
  size_t wmicro;
  int st_exchange;  // ECCO_WIDE_ST_ASYNC: partial logits by per-thread st.async
                    // instead of bulk copies (compute-sanitizer memcheck does
                    // not model shared::cta -> shared::cluster bulk copies)
};

// [step][point] cycles since the step start of CTA 0 (tools/wide_trace.md)
__device__ unsigned long long g_wide_trace[4 * 32];
#define WTS(k)                                                                            \
  do {                                                                                    \
    if (a.trace && blockIdx.x == 0 && t < 4) g_wide_trace[t * 32 + (k)] = clock64(); \
  } while (0)

struct WBars {
  uint64_t full[2], empty[2];  // ring
  uint64_t zfull, r_ready, plfull, recv_full, dl_full, dhfull, w2full, dh_ready, b1full;
  uint64_t dfull[2], dempty[2];  // dW1 tile buffers
  uint64_t fwd_done[2];          // every CTA's forward of step t done (by step parity)
  uint64_t stage_free;           // the partial logits staged in the ring have been sent
  uint64_t xready[kMaxNM];       // W1 operand tile rebuilt
};

struct WLayout {
  uint32_t ring, w1op, w2img, ones, rowbuf, b1, b2, loss, bars, tmem, total;
  uint32_t recv, r, dl, db2, dh, alias_end;  // inside w1op
};

__host__ __device__ inline WLayout wlayout(int F, int C, int cs) {
  WLayout L{};
  uint32_t o = 0;
  L.ring = o;
  o += 2 * kSlot;
  L.w1op = o;  // MN-major [f][64 hidden] bf16, 128B-swizzled
  o += (uint32_t)F * 128u;
  L.w2img = o;  // [class][64 hidden] bf16, K-major 128B-swizzled (C % 8 == 0)
  o += (uint32_t)C * 128u;
  L.ones = o;  // bf16 1.0 [row][16], 32B-swizzled: db1 = dH^T . 1
  o += kB * 32u;
  L.rowbuf = o;  // fp32 dL of the owned rows [row][class]
  o += (uint32_t)(kB / cs) * C * 4u;
  L.b1 = o;
  o += kHS * 4u;
  L.b2 = o;
  o += (uint32_t)C * 4u;
  L.loss = o;
  o += kB * 4u;
  o = (o + 7u) & ~7u;
  L.bars = o;
  o += (uint32_t)sizeof(WBars);
  L.tmem = o;
  o += 16u;
  L.total = o;
  uint32_t a = L.w1op;
  L.recv = a;  // [src rank][row of the owner block][class] fp32
  a += (uint32_t)kB * C * 4u;
  a = (a + 1023u) & ~1023u;
  L.r = a;  // bf16 R [row][64], K-major / MN-major
  a += 16384u;
  L.dl = a;  // bf16 dL [class atom][row][64 classes]
  a += 32768u;
  L.db2 = a;  // [owner rank][class] fp32
  a += (uint32_t)cs * C * 4u;
  L.alias_end = a;
  L.dh = L.w1op + (uint32_t)F * 128u - 16384u;  // bf16 -lr dH: the last tile, rebuilt last
  return L;
}

__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(kEpi) : "memory"); }

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"((uint64_t)map),
               "r"(c0), "r"(c1)
               : "memory");
}

// The sampled rows of every (job, micro-window, step) of the call, gathered
// from the frame table into one contiguous minibatch [128][F] each (same
// indexing as the rows k_chain_rows drew): the chain then streams each
// 64-feature chunk of a step with ONE 2-D TMA box instead of 32 gather4
// copies.  One block per (job, row step); warp w copies rows w, w + 8, ...
__global__ void k_wide_gather(const int* steps, int max_steps, int n_row_steps,
                              const int32_t* rows, const uint16_t* frames, int F, uint16_t* xall) {
  const int j = blockIdx.x, y = blockIdx.y;
  if (y % max_steps >= steps[j]) return;
  const size_t o = ((size_t)j * n_row_steps + y) * kB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v = F / 8;  // 16-byte pieces per row
  for (int i = warp; i < kB; i += 8) {
    const uint4* src = reinterpret_cast<const uint4*>(frames + (size_t)rows[o + i] * F);
    uint4* dst = reinterpret_cast<uint4*>(xall + (o + i) * F);
    for (int c = lane; c < v; c += 32) dst[c] = __ldg(src + c);
  }
}

// bf16 dL of classes [c, c+4) of `row` in the [atom][row][64 classes] tile.
__device__ __forceinline__ uint32_t dl_off(int row, int c) {
  const int cc = c & 63;
  return (uint32_t)(c >> 6) * 16384u + (uint32_t)row * 128u +
         ((uint32_t)((cc >> 3) ^ (row & 7)) << 4) + (uint32_t)(cc & 7) * 2u;
}
// The 32 fp32 master values W1[h0 + 32p + i][f], i < 32 ([H][F]: stride F;
// a warp's lanes read 32 consecutive features, 128 contiguous bytes).
template <int F>
__device__ __forceinline__ void ld_master(const float* p, float (&m)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) m[i] = p[(size_t)i * F];
}

// bf16 element (class c, hidden h) of the W2 image.
__device__ __forceinline__ uint32_t w2img_off(int c, int h) {
  return (uint32_t)c * 128u + ((uint32_t)((h >> 3) ^ (c & 7)) << 4) + (uint32_t)(h & 7) * 2u;
}

// F and C are compile-time: the 32 master rows of a thread's tile sit at
// immediate offsets from one base register (runtime strides spilled).
template <int F, int C>
__global__ void __launch_bounds__(kThreads, 1)
    k_train_wide(const __grid_constant__ CUtensorMap map_x, WideArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const LDims g = a.g;
  const int H = g.H;
  const int cs = H / kHS;
  const int j = blockIdx.x / cs;
  const int r = (int)cluster_ctarank();
  const int nsteps = a.steps[j];  // per micro-window
  const int total = nsteps * a.n_micro_launch;
  const int slot = a.slots[j];
  const float* src = a.wsrc + (size_t)slot * a.wsrc_stride;
  float* dst = a.wbase + (size_t)slot * a.wstride;
  if (nsteps <= 0) {  // no step: the snapshot is the starting model (the cluster copies it)
    if (src != dst) {
      const size_t np = (size_t)F * H + H + (size_t)H * C + C;
      for (size_t i = (size_t)r * blockDim.x + threadIdx.x; i < np; i += (size_t)cs * blockDim.x)
        dst[i] = src[i];
    }
    return;  // the whole cluster (same job) leaves
  }
  const WLayout L = wlayout(F, C, cs);
  uint8_t* ring = smem + L.ring;
  uint8_t* sW1 = smem + L.w1op;
  uint8_t* sW2i = smem + L.w2img;
  uint8_t* sOnes = smem + L.ones;
  float* sRowbuf = (float*)(smem + L.rowbuf);
  float* sB1 = (float*)(smem + L.b1);
  float* sB2 = (float*)(smem + L.b2);
  float* sLoss = (float*)(smem + L.loss);
  float* sRecv = (float*)(smem + L.recv);
  uint8_t* sR = smem + L.r;
  uint8_t* sDL = smem + L.dl;
  float* sDb2 = (float*)(smem + L.db2);
  uint8_t* sDH = smem + L.dh;
  WBars* bars = (WBars*)(smem + L.bars);
  uint32_t* sTmem = (uint32_t*)(smem + L.tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int RP = kB / cs;  // rows owned per CTA
  const int NM = F / 128;  // 128-feature tiles
  const int h0 = r * kHS;
  const float lr = g.lr;
  float* W1 = dst;  // [H][F]: this CTA's slice is rows h0 .. h0+63, contiguous
  float* b1 = W1 + (size_t)F * H;
  float* W2 = b1 + H;  // [H][C]
  float* b2 = W2 + (size_t)H * C;
  const float* sb1 = src + (size_t)F * H;
  const float* sW2s = sb1 + H;
  const float* sb2 = sW2s + (size_t)H * C;
  const int32_t* jrows = a.rows + ((size_t)j * a.rows_T + a.row_step0) * kB;
  const int32_t* jlabs = a.labs + ((size_t)j * a.rows_T + a.row_step0) * kB;

  // ---------------------------------------------------------------- setup --
  if (tid == 0) {
    if (smem_u32(smem) & 1023u) __trap();  // 128B-swizzle atoms need 1 KB alignment
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->full[i], 1);
      mbar_init(&bars->empty[i], 1);
      mbar_init(&bars->dfull[i], 1);
      mbar_init(&bars->dempty[i], kEpi / 2);
      mbar_init(&bars->fwd_done[i], cs);
    }
    mbar_init(&bars->zfull, 1);
    mbar_init(&bars->r_ready, kEpi);
    mbar_init(&bars->plfull, 1);
    mbar_init(&bars->recv_full, 1);
    mbar_init(&bars->dl_full, 1);
    mbar_init(&bars->dhfull, 1);
    mbar_init(&bars->w2full, 1);
    mbar_init(&bars->dh_ready, kEpi);
    mbar_init(&bars->b1full, 1);
    mbar_init(&bars->stage_free, 1);
    for (int mt = 0; mt < kMaxNM; ++mt) mbar_init(&bars->xready[mt], kEpi / 2);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(sTmem, 512);
  if (tid < kHS) sB1[tid] = sb1[h0 + tid];
  if (tid < C) sB2[tid] = sb2[tid];
  for (int i = tid; i < kB * 32 / 16; i += kThreads)
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  __syncthreads();  // the copied slices are visible to the whole CTA
  const int q = warp & 3, p = (warp >> 2) & 1;
  const int s = q * 32 + lane;  // epilogue: minibatch row / feature of the tile (TMEM lane)
  const uint32_t lane_base = (uint32_t)(q * 32) << 16;
  if (tid < kEpi) {
    for (int mt = 0; mt < NM; ++mt) {  // bf16 W1 operand from the master slice
      float m[32];
      ld_master<F>(src + (size_t)(h0 + p * 32) * F + mt * 128 + s, m);
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(m[i]);
      put_row32(sW1, mt * 128 + s, p, w);
    }
    for (int e = tid; e < C * kHS / 8; e += kEpi) {  // W2 image
      const int c = e >> 3, hc = e & 7;
      const float* w = sW2s + (size_t)(h0 + hc * 8) * C + c;
      uint4 pk;
      pk.x = pack_bf16x2(w[0 * C], w[1 * C]);
      pk.y = pack_bf16x2(w[2 * C], w[3 * C]);
      pk.z = pack_bf16x2(w[4 * C], w[5 * C]);
      pk.w = pack_bf16x2(w[6 * C], w[7 * C]);
      *reinterpret_cast<uint4*>(sW2i + c * 128 + ((hc ^ (c & 7)) << 4)) = pk;
    }
  }
  tc_fence_before();
  __syncthreads();  // (the TMEM allocation is visible)
  tc_fence_after();
  const uint32_t tmem = *sTmem;
  if (tid < kEpi && q < 2) {  // the W2 master slice -> TMEM lane s (hidden unit h0 + s)
    const float* w = sW2s + (size_t)(h0 + s) * C + p * (C / 2);
    for (int c16 = 0; c16 < C / 32; ++c16) {
      uint32_t v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(w[c16 * 16 + i]);
      tmem_st16(tmem + lane_base + kColW2M + p * (C / 2) + c16 * 16, v);
    }
    tmem_st_wait();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA of the cluster is running before any DSMEM traffic
  tc_fence_after();
  // the rest of micro-window u's model (the W2 master slice from TMEM, b1,
  // b2) and its loss -> snapshot u (epilogue threads, after the step)
  auto write_rest = [&](int u) {
    const size_t o = (size_t)u * a.wmicro;
    if (q < 2) {
      float* w = W2 + o + (size_t)(h0 + s) * C + p * (C / 2);
      for (int c16 = 0; c16 < C / 32; ++c16) {
        uint32_t v[16];
        tmem_ld16_nowait(tmem + lane_base + kColW2M + p * (C / 2) + c16 * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) w[c16 * 16 + i] = __uint_as_float(v[i]);
      }
    }
    if (tid < kHS) b1[o + h0 + tid] = sB1[tid];
    if (r == 0 && tid < C) b2[o + tid] = sB2[tid];
    if (r == 0 && tid == 0) {
      double acc = 0.0;
      for (int i = 0; i < kB; ++i) acc += sLoss[i];
      a.losses[(size_t)slot * a.loss_T + a.loss_t + u] = (float)(acc / kB);
    }
  };
  const uint32_t ring_a = smem_u32(ring), w1_a = smem_u32(sW1), w2i_a = smem_u32(sW2i);
  const uint32_t r_a = smem_u32(sR), dl_a = smem_u32(sDL), dh_a = smem_u32(sDH);

  if (warp == 8) {
    // ------------------------------------------------ row loads (TMA) --
    // per step: the forward's 128-feature slot pairs, then dW1's; each slot
    // is two 64-feature boxes of the step's 128 gathered rows (k_wide_gather)
    uint32_t k = 0;
    for (int t = 0; t < total; ++t) {
      const int row0 = (int)(((size_t)j * a.rows_T + a.row_step0 + t) * kB);
      if (lane == 0 && t + 1 < total && r < F / 64)  // this CTA's box of the next step -> L2
        tma_prefetch_2d(&map_x, r * 64, row0 + kB);
      for (int pass = 0; pass < 2; ++pass)
        for (int mt = 0; mt < NM; ++mt, ++k) {
          const int sl = (int)(k & 1u);
          const uint32_t u = k >> 1;
          if (u) mbar_wait(&bars->empty[sl], (u - 1) & 1u);
          // the head stages this step's partial logits in the ring after the
          // forward: dW1's rows load once they have been sent
          if (pass == 1 && mt == 0) mbar_wait(&bars->stage_free, (uint32_t)t & 1u);
          if (lane == 0) {
            mbar_expect_tx(&bars->full[sl], kSlot);
            tma_load_2d(ring + sl * kSlot, &map_x, (2 * mt) * 64, row0, &bars->full[sl]);
            tma_load_2d(ring + sl * kSlot + 16384, &map_x, (2 * mt + 1) * 64, row0, &bars->full[sl]);
            if (mt == 0) WTS(26 + pass);
          }
          __syncwarp();
        }
      if (lane == 0) WTS(28);
    }
  } else if (warp == 9) {
    // ------------------------------------------------------- MMA issuer --
    const uint32_t idf = idesc_major(kB, kHS, kFmtBF16, 0, 1);   // X . W1
    const uint32_t idl = idesc(kB, C, kFmtBF16);                 // R . W2
    const uint32_t idh = idesc_major(kB, kHS, kFmtBF16, 0, 1);   // dL . W2^T
    const uint32_t idw2 = idesc_major(128, C, kFmtBF16, 1, 1);   // R^T . dL (rows 64+ alias)
    const uint32_t idg = idesc_major(128, kHS, kFmtBF16, 1, 1);  // X^T . dH
    const uint32_t idb = idesc_major(128, 16, kFmtBF16, 1, 1);   // dH^T . 1 (rows 64+ alias)
    uint32_t k = 0, nd = 0;
    for (int t = 0; t < total; ++t) {
      const uint32_t ph = (uint32_t)t & 1u;
      for (int mt = 0; mt < NM; ++mt, ++k) {  // Z = X . W1
        const int sl = (int)(k & 1u);
        if (t > 0) mbar_wait(&bars->xready[mt], (uint32_t)(t - 1) & 1u);
        mbar_wait(&bars->full[sl], (k >> 1) & 1u);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ss(tmem + kColZ, desc_kmajor_sw128(ring_a + sl * kSlot + cc * 16384 + kk * 32),
                          desc_mnmajor_sw128(w1_a + ((2 * mt + cc) * 4 + kk) * 2048, 16384, 1024), idf,
                          (mt | cc | kk) != 0);
          mma_commit(&bars->empty[sl]);
          if (mt == NM - 1) mma_commit(&bars->zfull);
        }
        __syncwarp();
        if (lane == 0 && (mt == 0 || mt == NM - 1)) WTS(mt == 0 ? 20 : 21);
      }
      mbar_wait(&bars->r_ready, ph);  // partial logits = R . W2 slice
      tc_fence_after();
      if (lane == 0) WTS(22);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ss(tmem + kColL, desc_kmajor_sw128(r_a + kk * 32), desc_kmajor_sw128(w2i_a + kk * 32),
                      idl, kk != 0);
        mma_commit(&bars->plfull);
      }
      __syncwarp();
      mbar_wait(&bars->dl_full, ph);  // dL.W2^T and dW2 = R^T.dL
      fence_async_smem();
      tc_fence_after();
      if (lane == 0) WTS(23);
      if (elect_one()) {
        for (int kq = 0; kq < C / 16; ++kq)
          mma_bf16_ss(tmem + kColZ, desc_kmajor_sw128(dl_a + (kq >> 2) * 16384 + (kq & 3) * 32),
                      desc_mnmajor_sw128(w2i_a + kq * 2048, 16384, 1024), idh, kq != 0);
        mma_commit(&bars->dhfull);
#pragma unroll
        for (int k16 = 0; k16 < kB / 16; ++k16)
          mma_bf16_ss(tmem + kColW2, desc_mnmajor_sw128(r_a + k16 * 2048, 0, 1024),
                      desc_mnmajor_sw128(dl_a + k16 * 2048, 16384, 1024), idw2, k16 != 0);
        mma_commit(&bars->w2full);
      }
      __syncwarp();
      mbar_wait(&bars->dh_ready, ph);  // -lr db1, then dW1 tile by tile
      tc_fence_after();
      if (lane == 0) WTS(24);
      for (int mt = 0; mt < NM; ++mt, ++k, ++nd) {
        const int sl = (int)(k & 1u), b = (int)(nd & 1u);
        mbar_wait(&bars->full[sl], (k >> 1) & 1u);
        if (nd >= 2) mbar_wait(&bars->dempty[b], ((nd >> 1) - 1) & 1u);
        tc_fence_after();
        if (elect_one()) {
          if (mt == 0) {
#pragma unroll
            for (int k16 = 0; k16 < kB / 16; ++k16)
              mma_bf16_ss(tmem + kColB1, desc_mnmajor_sw128(dh_a + k16 * 2048, 0, 1024),
                          smem_desc(smem_u32(sOnes) + k16 * 512, 256, 256, kSwizzle32B), idb, k16 != 0);
            mma_commit(&bars->b1full);
          }
#pragma unroll
          for (int k16 = 0; k16 < kB / 16; ++k16)
            mma_bf16_ss(tmem + kColD + b * 64,
                        desc_mnmajor_sw128(ring_a + sl * kSlot + k16 * 2048, 16384, 1024),
                        desc_mnmajor_sw128(dh_a + k16 * 2048, 16384, 1024), idg, k16 != 0);
          mma_commit(&bars->empty[sl]);
          mma_commit(&bars->dfull[b]);
        }
        __syncwarp();
        if (lane == 0 && mt == NM - 1) WTS(25);
      }
    }
  } else {
    // --------------------------------------------------------- epilogue --
    const int half = C / 2;  // partial-logit / dW2 columns per column half
    uint32_t nd = 0;
    for (int t = 0; t < total; ++t) {
      const uint32_t ph = (uint32_t)t & 1u;
      if (a.trace && blockIdx.x == 0 && t < 4 && tid == 0) g_wide_trace[t * 32 + 31] = clock64();
      if (tid == 0) {  // this step's incoming DSMEM bytes
        mbar_expect_tx(&bars->recv_full, (uint32_t)kB * C * 4u);
        mbar_expect_tx(&bars->dl_full, (uint32_t)kB * C * 2u + (uint32_t)cs * C * 4u + (r == 0 ? kB * 4u : 0u));
      }
      // labels of the owned rows this warp handles (rows warp, warp + 8 of the block)
      const int lab0 = jlabs[(size_t)t * kB + r * RP + warp];
      const int lab1 = RP > 8 ? jlabs[(size_t)t * kB + r * RP + warp + 8] : 0;

      // ------------------------------------------ R = relu(Z + b1) --
      mbar_wait(&bars->zfull, ph);
      tc_fence_after();
      if (tid == 0) WTS(1);
      uint32_t mask;
      {
        uint32_t zr[32];
        tmem_ld32_nowait(tmem + lane_base + kColZ + p * 32, zr);
        tmem_ld_wait();
        mask = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float z = __fadd_rn(__uint_as_float(zr[i]), sB1[p * 32 + i]);
          mask |= (z > 0.0f ? 1u : 0u) << i;
          zr[i] = __float_as_uint(z > 0.0f ? z : 0.0f);
        }
        put_row32(sR, s, p, zr);
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->r_ready);
      // the forward has read this CTA's W1 operand region: every CTA may now
      // write its receive buffers there (one lane per destination CTA)
      if (warp == 7 && lane < cs)
        mbar_arrive_cluster(mapa_shared(smem_u32(&bars->fwd_done[t & 1]), (uint32_t)lane));

      // ------------------------------ partial logits -> the row owner --
      // staged in the ring (free between the forward and dW1's row loads)
      // as [owner][row of its block][class] fp32, 16-byte chunks swizzled
      // within groups of 8 by the row (conflict-free stores), then one bulk
      // DSMEM copy per owner into its receive buffer (source block r)
      mbar_wait(&bars->plfull, ph);
      tc_fence_after();
      if (tid == 0) WTS(2);
      {
        uint32_t pl[64];
#pragma unroll
        for (int c16 = 0; c16 < 4; ++c16)
          if (c16 * 16 < half) tmem_ld16_nowait(tmem + lane_base + kColL + p * half + c16 * 16, pl + c16 * 16);
        tmem_ld_wait();
        tc_fence_before();
        const int tr = s % RP;
        if (a.st_exchange) {  // straight into the owner's receive buffer, same layout
          mbar_wait(&bars->fwd_done[t & 1], (uint32_t)(t >> 1) & 1u);
          const uint32_t o = (uint32_t)(s / RP);
          const uint32_t row_a = mapa_shared(smem_u32(sRecv + ((size_t)r * RP + tr) * C), o);
          const uint32_t bar = mapa_shared(smem_u32(&bars->recv_full), o);
#pragma unroll
          for (int c4 = 0; c4 < 16; ++c4)
            if (c4 * 4 < half) {
              const int ch = p * (half / 4) + c4;
              st_async_v4(row_a + ((ch & ~7) | ((ch & 7) ^ (tr & 7))) * 16, __uint_as_float(pl[4 * c4]),
                          __uint_as_float(pl[4 * c4 + 1]), __uint_as_float(pl[4 * c4 + 2]),
                          __uint_as_float(pl[4 * c4 + 3]), bar);
            }
        } else {
          uint8_t* st = ring + (size_t)(s / RP) * RP * C * 4 + (size_t)tr * C * 4;
#pragma unroll
          for (int c4 = 0; c4 < 16; ++c4)
            if (c4 * 4 < half) {
              const int ch = p * (half / 4) + c4;
              *reinterpret_cast<uint4*>(st + ((ch & ~7) | ((ch & 7) ^ (tr & 7))) * 16) =
                  make_uint4(pl[4 * c4], pl[4 * c4 + 1], pl[4 * c4 + 2], pl[4 * c4 + 3]);
            }
          fence_async_smem();  // generic stores -> the bulk copies' reads
        }
      }
      if (a.st_exchange) {
        if (tid == 0) mbar_arrive(&bars->stage_free);
      } else {
        bar_epi();
        if (warp == 0) {
          if (lane < cs) {
            mbar_wait(&bars->fwd_done[t & 1], (uint32_t)(t >> 1) & 1u);
            if (lane == 0) WTS(3);
            const uint32_t blk = (uint32_t)RP * C * 4u;
            bulk_s2c(mapa_shared(smem_u32(sRecv) + (uint32_t)r * blk, (uint32_t)lane),
                     smem_u32(ring) + (uint32_t)lane * blk, blk,
                     mapa_shared(smem_u32(&bars->recv_full), (uint32_t)lane));
            bulk_commit();
            bulk_wait_read_all();
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->stage_free);
        }
      }

      // --------------- owned rows: logits, softmax, dL -> every CTA --
      for (int tt = warp; tt < RP; tt += 8) {
        mbar_wait(&bars->recv_full, ph);
        if (tid == 0) WTS(4);
        const int row = r * RP + tt;
        const bool act = 4 * lane < C;
        const int c0 = act ? 4 * lane : 0;
        const int pc = ((lane & ~7) | ((lane & 7) ^ (tt & 7))) * 4;  // the staged swizzle
        float4 lg = *reinterpret_cast<const float4*>(sRecv + (size_t)tt * C + (act ? pc : 0));
        for (int sr = 1; sr < cs; ++sr) {
          const float4 v = *reinterpret_cast<const float4*>(sRecv + ((size_t)sr * RP + tt) * C + (act ? pc : 0));
          lg = make_float4(__fadd_rn(lg.x, v.x), __fadd_rn(lg.y, v.y), __fadd_rn(lg.z, v.z),
                           __fadd_rn(lg.w, v.w));
        }
        const float4 bb = *reinterpret_cast<const float4*>(sB2 + c0);
        lg = make_float4(__fadd_rn(lg.x, bb.x), __fadd_rn(lg.y, bb.y), __fadd_rn(lg.z, bb.z),
                         __fadd_rn(lg.w, bb.w));
        float m = act ? fmaxf(fmaxf(lg.x, lg.y), fmaxf(lg.z, lg.w)) : -INFINITY;
#pragma unroll
        for (int x = 1; x < 32; x <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, x));
        const float4 e = act ? make_float4(expf_nb(__fsub_rn(lg.x, m)), expf_nb(__fsub_rn(lg.y, m)),
                                           expf_nb(__fsub_rn(lg.z, m)), expf_nb(__fsub_rn(lg.w, m)))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        float sum = __fadd_rn(__fadd_rn(e.x, e.y), __fadd_rn(e.z, e.w));
#pragma unroll
        for (int x = 1; x < 32; x <<= 1) sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, x));
        constexpr float invB = 1.0f / kB;  // exact (power of two)
        const float inv = __frcp_rn(sum);
        const int y = (tt == warp ? lab0 : lab1) - c0;  // class within this lane's quad (0..3 if mine)
        const float4 dl = make_float4(__fmul_rn(__fsub_rn(__fmul_rn(e.x, inv), y == 0 ? 1.0f : 0.0f), invB),
                                      __fmul_rn(__fsub_rn(__fmul_rn(e.y, inv), y == 1 ? 1.0f : 0.0f), invB),
                                      __fmul_rn(__fsub_rn(__fmul_rn(e.z, inv), y == 2 ? 1.0f : 0.0f), invB),
                                      __fmul_rn(__fsub_rn(__fmul_rn(e.w, inv), y == 3 ? 1.0f : 0.0f), invB));
        if (act) {
          const uint32_t lo = pack_bf16x2(dl.x, dl.y), hi = pack_bf16x2(dl.z, dl.w);
          const uint32_t off = dl_off(row, c0);
          for (int d = 0; d < cs; ++d)
            st_async_v2b32(mapa_shared(dl_a + off, (uint32_t)d), lo, hi,
                           mapa_shared(smem_u32(&bars->dl_full), (uint32_t)d));
          *reinterpret_cast<float4*>(sRowbuf + (size_t)tt * C + c0) = dl;
          if (y >= 0 && y < 4) {
            const float ly = y == 0 ? lg.x : y == 1 ? lg.y : y == 2 ? lg.z : lg.w;
            st_async_f32(mapa_shared(smem_u32(sLoss + row), 0u), __logf(sum) - (ly - m),
                         mapa_shared(smem_u32(&bars->dl_full), 0u));
          }
        }
      }
      if (tid == 0) WTS(5);
      bar_epi();  // every owned row's fp32 dL in sRowbuf
      if (tid < C / 4) {  // db2 partial of the owned rows (fixed row order) -> every CTA
        float4 acc = reinterpret_cast<const float4*>(sRowbuf)[tid];
        for (int tt = 1; tt < RP; ++tt) {
          const float4 v = reinterpret_cast<const float4*>(sRowbuf + (size_t)tt * C)[tid];
          acc = make_float4(__fadd_rn(acc.x, v.x), __fadd_rn(acc.y, v.y), __fadd_rn(acc.z, v.z),
                            __fadd_rn(acc.w, v.w));
        }
        for (int d = 0; d < cs; ++d)
          st_async_v4(mapa_shared(smem_u32(sDb2 + r * C + 4 * tid), (uint32_t)d), acc.x, acc.y, acc.z,
                      acc.w, mapa_shared(smem_u32(&bars->dl_full), (uint32_t)d));
      }
      mbar_wait(&bars->dl_full, ph);
      if (tid == 0) WTS(6);
      if (tid < C) {  // b2 (identical in every CTA: same partials, same order)
        float acc = sDb2[tid];
        for (int o = 1; o < cs; ++o) acc = __fadd_rn(acc, sDb2[o * C + tid]);
        sB2[tid] = __fmaf_rn(-lr, acc, sB2[tid]);
      }

      // ------------------------------------ dH = (dL.W2^T) * (Z > 0) --
      mbar_wait(&bars->dhfull, ph);
      tc_fence_after();
      if (tid == 0) WTS(7);
      {
        uint32_t dh[32];
        tmem_ld32_nowait(tmem + lane_base + kColZ + p * 32, dh);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i)
          dh[i] = (mask >> i) & 1u ? __float_as_uint(__fmul_rn(-lr, __uint_as_float(dh[i]))) : 0u;
        put_row32(sDH, s, p, dh);  // -lr dH, MN-major over rows: dW1's B operand
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->dh_ready);

      if (tid == 0) WTS(9);
      // -------------- W1 += X^T.(-lr dH): master tiles and operand rows --
      // two tile streams: warps 0-3 (p = 0) take the even tiles (TMEM buffer
      // 0), warps 4-7 the odd ones (buffer 1), each thread both 32-column
      // halves of its feature -- one group's TMEM reads overlap the other's
      // master round trip
      // the master is read-modify-written in the snapshot: micro-window u's
      // first step reads the model it starts from (the source model, or
      // snapshot u-1 in serial mode) and writes snapshot u -- the copy
      // rides on the update
      const int u = t / nsteps;
      float* W1w = W1 + (size_t)u * a.wmicro;
      const float* W1r = t % nsteps ? W1w : u == 0 ? src : W1w - a.wmicro;
      for (int mt = p; mt < NM; mt += 2, ++nd) {
        const int f = mt * 128 + s;
        float m0[32], m1[32];
        ld_master<F>(W1r + (size_t)h0 * F + f, m0);
        mbar_wait(&bars->dfull[p], nd & 1u);
        tc_fence_after();
        if (tid == 0) WTS(10 + mt);
        uint32_t d0[32], d1[32];
        tmem_ld32_nowait(tmem + lane_base + kColD + p * 64, d0);
        tmem_ld32_nowait(tmem + lane_base + kColD + p * 64 + 32, d1);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars->dempty[p]);
        ld_master<F>(W1r + (size_t)(h0 + 32) * F + f, m1);
        float* wm = W1w + (size_t)h0 * F + f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float w = __fadd_rn(m0[i], __uint_as_float(d0[i]));
          wm[(size_t)i * F] = w;
          d0[i] = __float_as_uint(w);
        }
        put_row32(sW1, f, 0, d0);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float w = __fadd_rn(m1[i], __uint_as_float(d1[i]));
          wm[(size_t)(32 + i) * F] = w;
          d1[i] = __float_as_uint(w);
        }
        put_row32(sW1, f, 1, d1);
        fence_async_smem();  // the rebuilt rows (generic stores) -> the next forward
        mbar_arrive(&bars->xready[mt]);
      }
      // ---------- W2 -= lr dW2, the master in TMEM (off the critical path:
      // the next step's logits read the image only after the end-of-step
      // barrier) --
      if (q < 2) {  // TMEM lanes 0-63 = hidden unit s of this CTA
        mbar_wait(&bars->w2full, ph);
        tc_fence_after();
        uint32_t w[64];
#pragma unroll
        for (int c16 = 0; c16 < 4; ++c16)
          if (c16 * 16 < half) tmem_ld16_nowait(tmem + lane_base + kColW2 + p * half + c16 * 16, w + c16 * 16);
        tmem_ld_wait();
        uint32_t m[64];
#pragma unroll
        for (int c16 = 0; c16 < 4; ++c16)
          if (c16 * 16 < half) tmem_ld16_nowait(tmem + lane_base + kColW2M + p * half + c16 * 16, m + c16 * 16);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          if (c >= half) break;
          const float nw = __fmaf_rn(-lr, __uint_as_float(w[c]), __uint_as_float(m[c]));
          m[c] = __float_as_uint(nw);
          *reinterpret_cast<uint16_t*>(sW2i + w2img_off(p * half + c, s)) =
              (uint16_t)(pack_bf16x2(nw, 0.0f) & 0xFFFFu);
        }
#pragma unroll
        for (int c16 = 0; c16 < 4; ++c16)
          if (c16 * 16 < half) tmem_st16(tmem + lane_base + kColW2M + p * half + c16 * 16, m + c16 * 16);
        tmem_st_wait();
      }

      if (q < 2 && p == 0) {  // b1 row s, already scaled by -lr
        mbar_wait(&bars->b1full, ph);
        tc_fence_after();
        uint32_t v[8];
        tmem_ld8_nowait(tmem + lane_base + kColB1, v);
        tmem_ld_wait();
        sB1[s] = __fadd_rn(sB1[s], __uint_as_float(v[0]));
      }
      fence_async_smem();  // the W2 image -> the next step's MMAs
      tc_fence_before();
      if (tid == 0) WTS(18);
      bar_epi();
      if ((t + 1) % nsteps == 0 && t + 1 < total)  // serial mode: micro-window u is done
        write_rest(u);
    }
  }

  // ------------------------------------------------------------ write back --
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < kEpi) write_rest(a.n_micro_launch - 1);
  cluster_sync();  // no CTA leaves while the cluster may still address its shared memory
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace

namespace fused {

// The instantiated shape: the detection head of BASELINE configs[4]
// (F = 1024, C = 96) with a 512- or 1024-wide hidden layer.
constexpr int kWF = 1024, kWC = 96;
#define K_WIDE k_train_wide<kWF, kWC>

static bool wide_shape(const ecco_config& g) {
  if (g.minibatch != kB || g.feat_dim != kWF || g.num_classes != kWC ||
      (g.hidden_dim != 8 * kHS && g.hidden_dim != 16 * kHS))
    return false;
  const WLayout L = wlayout(g.feat_dim, g.num_classes, g.hidden_dim / kHS);
  return L.alias_end <= L.dh && L.total <= 232448;
}

static cudaLaunchConfig_t wide_config(const ecco_config& c, int n_jobs, cudaStream_t st,
                                      cudaLaunchAttribute* at) {
  const int cs = c.hidden_dim / kHS;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(cs * std::max(n_jobs, 1)));
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = wlayout(c.feat_dim, c.num_classes, cs).total;
  lc.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return lc;
}

static void wide_attrs(int device) {
  static DeviceFlags attr;  // per device: the attributes apply to the current device
  if (attr.done(device)) return;
  ECCO_CUDA(cudaFuncSetAttribute(K_WIDE, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
  ECCO_CUDA(cudaFuncSetAttribute(K_WIDE, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  attr.mark(device);
}

void wide_gather(ecco_ctx* ctx, int n_jobs, const int* d_steps, int max_steps, int n_micro) {
  const ecco_config& c = ctx->cfg;
  const int n_row_steps = n_micro * max_steps;
  uint16_t* xall = (uint16_t*)ctx->train_scratch[11].get((size_t)n_jobs * n_row_steps * kB *
                                                          c.feat_dim * 2);
  k_wide_gather<<<dim3(n_jobs, n_row_steps), 256, 0, ctx->stream>>>(
      d_steps, max_steps, n_row_steps, (const int32_t*)ctx->train_scratch[0].p, ctx->d_frames,
      c.feat_dim, xall);
  ECCO_LAUNCHED(ctx);
}

bool wide_supported(const ecco_ctx* ctx) {
  const ecco_config& g = ctx->cfg;
  if (!wide_shape(g)) return false;
  // a cluster of H/64 CTAs at one CTA per SM must fit on the device (16 is
  // beyond the portable cluster size)
  wide_attrs(g.device);
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t lc = wide_config(g, 1, ctx->stream, at);
  int n = 0;
  const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)K_WIDE, &lc);
  if (getenv("ECCO_DEBUG")) {
    int nb = -1;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, (const void*)K_WIDE);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)K_WIDE, kThreads, lc.dynamicSmemBytes);
    fprintf(stderr, "ecco: wide chain: cluster %d x %u B smem, %d resident clusters (%s); %d blocks/SM, %d regs, %zu static smem\n",
            g.hidden_dim / kHS, (unsigned)lc.dynamicSmemBytes, n, cudaGetErrorString(e), nb, fa.numRegs, fa.sharedSizeBytes);
  }
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return n > 0;
}

void train_wide(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_steps,
                const int* h_steps, int micro, int n_micro, const float* wsrc, size_t wsrc_stride,
                float* wbase, size_t wstride, int loss_t, int n_launch, size_t wmicro) {
  ECCO_REQUIRE(n_launch == 1 || n_jobs == 1, "serial wide chain: one job");
  if (n_jobs == 0) return;
  const ecco_config& c = ctx->cfg;
  const LDims g{c.feat_dim, c.hidden_dim, c.num_classes, c.scene_dims, c.minibatch,
                c.ring_frames, c.eval_samples, c.sgd_lr, c.feature_noise};
  int max_steps = 0;
  for (int j = 0; j < n_jobs; ++j) max_steps = std::max(max_steps, h_steps[j]);
  WideArgs a{};
  a.g = g;
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
  a.trace = getenv("ECCO_WIDE_TRACE") ? 1 : 0;
  a.st_exchange = getenv("ECCO_WIDE_ST_ASYNC") ? 1 : 0;
  wide_attrs(c.device);
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t lc = wide_config(c, n_jobs, ctx->stream, at);
  const double F = c.feat_dim, H = c.hidden_dim, C = c.num_classes;
  double steps = 0, live = 0;
  for (int j = 0; j < n_jobs; ++j) {
    steps += (double)h_steps[j] * n_launch;
    live += h_steps[j] > 0;
  }
  // algorithmic work: every live step's forward + backward; bytes: the
  // sampled rows once per step, the masters in and out once per chain (the
  // per-step master round trips stay in L2)
  const double flops = steps * kB * (4.0 * F * H + 6.0 * H * C);
  const double params = F * H + H + H * C + C;
  const double bytes = steps * kB * F * 2.0 + live * params * 8.0;
  const uint16_t* xall = (const uint16_t*)ctx->train_scratch[11].p;  // wide_gather() of this call
  const CUtensorMap map_x =
      tensor_map_bf16(xall, (uint64_t)n_jobs * a.rows_T * kB, c.feat_dim, kB);
  ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_STEP, flops, bytes,
             ECCO_CUDA(cudaLaunchKernelEx(&lc, K_WIDE, map_x, a)));
  ECCO_LAUNCHED(ctx);
  if (a.trace) {
    unsigned long long tr[4 * 32];
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    // (points: 1 zfull, 2 plfull, 3 fwd_done, 4 recv_full, 5 dL sent, 6 dl_full,
    //  7 dhfull, 9 dW2 done, 10+mt dW1 tile mt, 18 step end; MMA 20/21 forward
    //  first/last, 22 r_ready, 23 dl_full, 24 dh_ready, 25 dW1 issued;
    //  gather 26/27 pass start, 28 step issued)
    ECCO_CUDA(cudaMemcpyFromSymbol(tr, g_wide_trace, sizeof(tr)));
    for (int t = 0; t < 4; ++t) {
      fprintf(stderr, "wide step %d:", t);
      for (int k = 0; k < 31; ++k)
        if (tr[t * 32 + k]) fprintf(stderr, " %d:%lld", k, (long long)(tr[t * 32 + k] - tr[t * 32 + 31]));
      fprintf(stderr, "\n");
    }
  }
}

}  // namespace fused
