// Fused SGD chain of the learned backend (tensor-core math): ONE launch runs
// every group's whole micro-window -- steps[j] SGD steps, each sampling,
// gather, forward, softmax cross-entropy, backward and update -- on one
// thread-block cluster per group (job).  The group's model never leaves the
// chip between steps: HBM sees the fp32 masters once in and once out per
// micro-window, plus the sampled frame rows.
//
// Cluster of H/64 CTAs; CTA r owns hidden units [64r, 64r+64):
//   TMEM     fp32 master slice W1[:, 64r:64r+64] (F/128 tiles of 128 lanes x
//            64 columns) and the dW1 accumulator of the same shape; the
//            forward accumulator Z (128 rows x 64) aliases dW1's first tile
//   smem     X tile (128 sampled rows, bf16, 128B-swizzled K-major; also read
//            MN-major as X^T), the bf16 W1^T operand built from the master,
//            W2/b1 slices, b2, dL
//   step     sample + gather X (cp.async, overlapped with the previous
//            step's update) -> Z = X.W1 (tcgen05 kind::f16, N = 64) ->
//            partial logits relu(Z+b1).W2 of the CTA's 64 hidden units, sent
//            to the CTA owning the row block over DSMEM -> owner sums the
//            partials in fixed order, softmax, dL, broadcasts dL rows to the
//            cluster -> dH = (dL.W2^T)*(Z>0) -> dW1 = X^T.dH (tcgen05, both
//            operands MN-major) while dW2 = R^T.dL, db1, db2 run on the CUDA
//            cores -> master update in TMEM, bf16 operand rewritten
//
// Numerics: X exact (bf16 frames); W1 rounded to bf16 for the forward and dH
// rounded to bf16 for dW1 and db1; fp32 accumulation, fp32 masters; the head
// (logits, softmax, dL, dH) and dW2 = R^T.dL are fp32 on CUDA cores.
// Tolerance in tests/test_gpu_learned.py.
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
constexpr int kThreads = 256;  // 8 warps: lane quadrant q = warp % 4, half p = warp / 4
constexpr int kC = 16;         // classes (logits held in registers)
constexpr int kHS = 64;        // hidden units per CTA of the cluster
constexpr int kMaxCluster = 8;

struct ChainArgs {
  LDims g;
  const int* slots;
  const int* steps;
  const int32_t* rows;  // [job][max_steps][kB] frame-table row of every sampled frame
  const int32_t* labs;  // [job][max_steps][kB] its label
  int max_steps;
  const uint16_t* frames;
  float* wbase;  // fp32 masters being trained (W1 stored [H][F])
  size_t wstride;
  uint16_t* w1t;  // bf16 W1^T evaluation shadow [slot][H][F], written at the end
  float* losses;  // losses[slot * loss_T + loss_t] = mean loss of the last step
  int loss_T, loss_t;
};

// Every (job, step, row) draw of the micro-window, ahead of the chain
// (sample_one: the same draws as k_l_sample and the oracle's orc_sample).
__global__ void k_chain_rows(LDims g, uint64_t seed, const int* job_ids, const int* steps,
                             const int* src_off, const int* src_cam, const double* src_frac,
                             const int* micro_base, int micro_add, int window, int max_steps,
                             const int32_t* labels, int32_t* rows, int32_t* labs) {
  const int j = blockIdx.x, step = blockIdx.y, s = threadIdx.x;
  if (step >= steps[j]) return;
  int cam, frame;
  const int s0 = src_off[j];
  sample_one(g, seed, job_ids[j], src_off[j + 1] - s0, src_cam + s0, src_frac + s0, window,
             micro_base[j] + micro_add, step, s, &cam, &frame);
  const int32_t row = cam * g.R + frame;
  const size_t o = ((size_t)j * max_steps + step) * kB + s;
  rows[o] = row;
  labs[o] = labels[row];
}

struct Layout {
  uint32_t x, sc, recv, dl, w2, b1, b2, rows, labs, loss, bars, tmem, total;
};

// sc: the bf16 W1 operand (MN-major: F rows of 64 hidden units, 128 B); between
// the forward MMA and the update it holds dH (MN-major, 16 KB) and R (fp32,
// 32 KB) instead.
__host__ __device__ inline Layout layout(int F) {
  Layout L{};
  uint32_t o = 0;
  L.x = o;
  o += (uint32_t)(F / 64) * 16384u;
  L.sc = o;
  o += std::max((uint32_t)F * 128u, 49152u);
  L.recv = o;
  o += 2u * kB * kC * 4u;  // [src rank][half][row of the owner block][class]
  L.dl = o;
  o += kB * kC * 4u;
  L.w2 = o;
  o += kHS * kC * 4u;
  L.b1 = o;
  o += kHS * 4u;
  L.b2 = o;
  o += kC * 4u;
  L.rows = o;
  o += 2u * kB * 8u;
  L.labs = o;
  o += 2u * kB * 4u;
  L.loss = o;
  o += kB * 4u;
  o = (o + 7u) & ~7u;
  L.bars = o;
  o += 4u * 8u;
  L.tmem = o;
  o += 16u;
  L.total = o;
  return L;
}

__host__ __device__ inline uint32_t tmem_cols(int F) {
  uint32_t n = (uint32_t)(F / 128) * 128u;  // master + dW1
  uint32_t a = 32;
  while (a < n) a <<= 1;
  return a;
}

// Remote (or own) shared-memory store whose bytes complete_tx on the
// destination CTA's mbarrier.
__device__ __forceinline__ void st_async_v4(uint32_t addr, float a, float b, float c, float d,
                                            uint32_t mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
          addr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t addr, float a, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(addr),
               "f"(a), "r"(mbar)
               : "memory");
}

// R[s][h] (fp32, 64 per row) with the 16-byte chunk index XORed by the row:
// the head's row-per-lane float4 stores spread over all banks.
__device__ __forceinline__ int r_idx(int s, int h) {
  return s * kHS + ((((h >> 2) ^ s) & 15) << 2) + (h & 3);
}

// 32 fp32 -> bf16 into row `row` (128 B) of an MN-major 128B-swizzled operand
// of 64 columns, columns [32p, 32p+32).
__device__ __forceinline__ void put_row32(uint8_t* base, int row, int p, const uint32_t (&w)[32]) {
#pragma unroll
  for (int g8 = 0; g8 < 4; ++g8) {
    uint4 pk;
    pk.x = pack_bf16x2(__uint_as_float(w[g8 * 8 + 0]), __uint_as_float(w[g8 * 8 + 1]));
    pk.y = pack_bf16x2(__uint_as_float(w[g8 * 8 + 2]), __uint_as_float(w[g8 * 8 + 3]));
    pk.z = pack_bf16x2(__uint_as_float(w[g8 * 8 + 4]), __uint_as_float(w[g8 * 8 + 5]));
    pk.w = pack_bf16x2(__uint_as_float(w[g8 * 8 + 6]), __uint_as_float(w[g8 * 8 + 7]));
    const int hc = p * 4 + g8;
    *reinterpret_cast<uint4*>(base + row * 128 + ((hc ^ (row & 7)) << 4)) = pk;
  }
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&w)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
      "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]),
      "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]),
      "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]),
      "r"(w[30]), "r"(w[31])
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) k_train_chain(ChainArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const LDims g = a.g;
  const int F = g.F, H = g.H;
  const int cs = H / kHS;
  const int j = blockIdx.x / cs;
  const int r = (int)cluster_ctarank();
  const int nsteps = a.steps[j];
  if (nsteps <= 0) return;  // the whole cluster (same job) leaves
  const Layout L = layout(F);
  uint8_t* sX = smem + L.x;
  uint8_t* sSC = smem + L.sc;                   // W1 operand, MN-major [f][64 hidden]
  uint8_t* sDH = sSC;                           // MN-major dH, 128 rows x 128 B
  float* sR = (float*)(sSC + 16384);            // relu(Z + b1), fp32 [128][64] swizzled
  float* sRecv = (float*)(smem + L.recv);
  float* sDL = (float*)(smem + L.dl);
  float* sW2 = (float*)(smem + L.w2);
  float* sB1 = (float*)(smem + L.b1);
  float* sB2 = (float*)(smem + L.b2);
  int64_t* sRow = (int64_t*)(smem + L.rows);    // [2][kB] element offsets
  int* sLab = (int*)(smem + L.labs);            // [2][kB]
  float* sLoss = (float*)(smem + L.loss);
  uint64_t* zfull = (uint64_t*)(smem + L.bars);
  uint64_t* gfull = zfull + 1;
  uint64_t* recv_full = zfull + 2;  // owner rows' partial logits arrived (st.async)
  uint64_t* dl_full = zfull + 3;    // every dL row (and, on rank 0, every loss) arrived
  uint32_t* sTmem = (uint32_t*)(smem + L.tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, p = warp >> 2;
  const int s = q * 32 + lane;  // minibatch row of this thread (TMEM lane)
  const uint32_t lane_base = (uint32_t)(q * 32) << 16;
  const int RP = kB / cs;       // rows owned per CTA for the softmax
  const int NM = F / 128;       // master / dW1 tiles
  const uint32_t gcol = (uint32_t)NM * 64u;  // dW1 accumulator (and Z) column base
  const int slot = a.slots[j];
  float* W1 = a.wbase + (size_t)slot * a.wstride;
  float* b1 = W1 + (size_t)F * H;
  float* W2 = b1 + H;
  float* b2 = W2 + (size_t)H * kC;
  const float lr = g.lr;
  const int h0 = r * kHS;  // first hidden unit of this CTA
  const int32_t* jrows = a.rows + (size_t)j * a.max_steps * kB;
  const int32_t* jlabs = a.labs + (size_t)j * a.max_steps * kB;
  const uint32_t recv_bytes = 2u * kB * kC * 4u;
  const uint32_t dl_bytes = kB * kC * 4u + (r == 0 ? kB * 4u : 0u);

  // rows of buffer `buf` -> X tile: row i, 16-byte piece c16 -> chunk c16/8
  auto gather = [&](int buf) {
    const int per_row = F / 8;
    for (int i = warp; i < kB; i += kThreads / 32) {
      const uint16_t* src = a.frames + sRow[buf * kB + i];
      for (int c16 = lane; c16 < per_row; c16 += 32)
        cp_async16(sX + (c16 >> 3) * 16384 + i * 128 + (((c16 & 7) ^ (i & 7)) << 4), src + c16 * 8);
    }
  };

  // ---------------------------------------------------------------- setup --
  if (tid == 0) {
    if (smem_u32(smem) & 1023u) __trap();  // 128B-swizzle atoms need 1 KB alignment
    mbar_init(zfull, 1);
    mbar_init(gfull, 1);
    mbar_init(recv_full, 1);
    mbar_init(dl_full, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(sTmem, tmem_cols(F));
  if (tid < kB) {
    sRow[tid] = (int64_t)jrows[tid] * F;
  } else {
    sLab[tid - kB] = jlabs[tid - kB];
  }
  for (int i = tid; i < kHS * kC / 4; i += kThreads)
    reinterpret_cast<float4*>(sW2)[i] = reinterpret_cast<const float4*>(W2 + (size_t)h0 * kC)[i];
  if (tid < kHS) sB1[tid] = b1[h0 + tid];
  if (tid < kC) sB2[tid] = b2[tid];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sTmem;
  gather(0);
  // master slice -> TMEM; its bf16 image -> the W1 operand
  for (int mt = 0; mt < NM; ++mt) {
    const int f = mt * 128 + s;
    uint32_t w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(W1[(size_t)(h0 + p * 32 + i) * F + f]);
    tmem_st32(tmem + lane_base + mt * 64 + p * 32, w);
    put_row32(sSC, f, p, w);
  }
  tmem_st_wait();
  cp_async_wait_all();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA of the cluster is running before any DSMEM store
  tc_fence_after();

  const uint32_t idf = idesc_major(kB, kHS, kFmtBF16, 0, 1);
  const uint32_t idg = idesc_major(128, kHS, kFmtBF16, 1, 1);
  const uint64_t dX = desc_kmajor_sw128(smem_u32(sX));
  const int nkc = F / 64;

  for (int step = 0; step < nsteps; ++step) {
    const int cur = step & 1;
    const uint32_t ph = (uint32_t)step & 1u;
    if (tid == 0) {  // this step's incoming DSMEM bytes
      mbar_expect_tx(recv_full, recv_bytes);
      mbar_expect_tx(dl_full, dl_bytes);
    }
    // ------------------------------------------------------ forward MMA --
    if (warp == 0) {
      if (elect_one()) {
        for (int kc = 0; kc < nkc; ++kc)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16_ss(tmem + gcol, dX + ((kc * 16384 + kk * 32) >> 4),
                        desc_mnmajor_sw128(smem_u32(sSC) + (kc * 4 + kk) * 2048, 16384, 1024), idf,
                        (kc | kk) != 0);
        mma_commit(zfull);
      }
      __syncwarp();
    }
    // next step's rows: loads in flight across the forward and the head
    int32_t nxt = 0;
    const bool more = step + 1 < nsteps;
    if (more) nxt = tid < kB ? jrows[(step + 1) * kB + tid] : jlabs[(step + 1) * kB + tid - kB];
    mbar_wait(zfull, ph);
    tc_fence_after();

    // ------------------------------- head: partial logits of 64 hidden --
    float rz[32];
    {
      uint32_t zr[32];
      tmem_ld32_nowait(tmem + lane_base + gcol + p * 32, zr);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float z = __fadd_rn(__uint_as_float(zr[i]), sB1[p * 32 + i]);
        rz[i] = z > 0.0f ? z : 0.0f;
      }
    }
    {
      float pl[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) pl[c] = 0.0f;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float4* w = reinterpret_cast<const float4*>(sW2 + (p * 32 + i) * kC);
#pragma unroll
        for (int c4 = 0; c4 < kC / 4; ++c4) {
          const float4 v = w[c4];
          pl[4 * c4 + 0] = __fmaf_rn(rz[i], v.x, pl[4 * c4 + 0]);
          pl[4 * c4 + 1] = __fmaf_rn(rz[i], v.y, pl[4 * c4 + 1]);
          pl[4 * c4 + 2] = __fmaf_rn(rz[i], v.z, pl[4 * c4 + 2]);
          pl[4 * c4 + 3] = __fmaf_rn(rz[i], v.w, pl[4 * c4 + 3]);
        }
      }
      // partials -> the CTA owning row s
      const uint32_t o = (uint32_t)(s / RP);
      const uint32_t dst = mapa_shared(smem_u32(sRecv + ((r * 2 + p) * RP + (s % RP)) * kC), o);
      const uint32_t bar = mapa_shared(smem_u32(recv_full), o);
#pragma unroll
      for (int c4 = 0; c4 < kC / 4; ++c4)
        st_async_v4(dst + c4 * 16, pl[4 * c4], pl[4 * c4 + 1], pl[4 * c4 + 2], pl[4 * c4 + 3], bar);
      // R for dW2 (the W1 operand is dead once the forward completed)
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(sR + r_idx(s, p * 32 + i)) =
            make_float4(rz[i], rz[i + 1], rz[i + 2], rz[i + 3]);
    }

    // ----------------------- owner rows: logits, softmax, dL broadcast --
    if (tid < RP) {
      mbar_wait(recv_full, ph);
      const int row = r * RP + tid;
      float lg[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) lg[c] = sRecv[tid * kC + c];
      for (int sh = 1; sh < 2 * cs; ++sh) {
        const float* pr = sRecv + (sh * RP + tid) * kC;
#pragma unroll
        for (int c = 0; c < kC; ++c) lg[c] = __fadd_rn(lg[c], pr[c]);
      }
#pragma unroll
      for (int c = 0; c < kC; ++c) lg[c] = __fadd_rn(lg[c], sB2[c]);
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
      const int y = sLab[cur * kB + row];
      float ly = lg[0], dl[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        dl[c] = __fmul_rn(__fsub_rn(__fdiv_rn(e[c], sum), c == y ? 1.0f : 0.0f), invB);
        ly = c == y ? lg[c] : ly;
      }
      for (int d = 0; d < cs; ++d) {
        const uint32_t dst = mapa_shared(smem_u32(sDL + row * kC), (uint32_t)d);
        const uint32_t bar = mapa_shared(smem_u32(dl_full), (uint32_t)d);
#pragma unroll
        for (int c4 = 0; c4 < kC / 4; ++c4)
          st_async_v4(dst + c4 * 16, dl[4 * c4], dl[4 * c4 + 1], dl[4 * c4 + 2], dl[4 * c4 + 3], bar);
      }
      st_async_f32(mapa_shared(smem_u32(sLoss + row), 0u), logf(sum) - (ly - m),
                   mapa_shared(smem_u32(dl_full), 0u));
    }
    if (more) {  // next step's rows into the other buffer
      if (tid < kB)
        sRow[(cur ^ 1) * kB + tid] = (int64_t)nxt * F;
      else
        sLab[(cur ^ 1) * kB + tid - kB] = nxt;
    }
    mbar_wait(dl_full, ph);

    // --------------------------------------------- dH = (dL.W2^T)*(Z>0) --
    {
      float dl[kC];
#pragma unroll
      for (int c4 = 0; c4 < kC / 4; ++c4) {
        const float4 v = reinterpret_cast<const float4*>(sDL + s * kC)[c4];
        dl[4 * c4] = v.x;
        dl[4 * c4 + 1] = v.y;
        dl[4 * c4 + 2] = v.z;
        dl[4 * c4 + 3] = v.w;
      }
      uint32_t dh[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float4* w = reinterpret_cast<const float4*>(sW2 + (p * 32 + i) * kC);
        float acc = 0.0f;
#pragma unroll
        for (int c4 = 0; c4 < kC / 4; ++c4) {
          const float4 v = w[c4];
          acc = __fmaf_rn(dl[4 * c4 + 0], v.x, acc);
          acc = __fmaf_rn(dl[4 * c4 + 1], v.y, acc);
          acc = __fmaf_rn(dl[4 * c4 + 2], v.z, acc);
          acc = __fmaf_rn(dl[4 * c4 + 3], v.w, acc);
        }
        dh[i] = __float_as_uint(rz[i] > 0.0f ? acc : 0.0f);
      }
      put_row32(sDH, s, p, dh);  // MN-major over rows: dW1's B operand
    }
    fence_async_smem();  // dH (generic stores) -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    // ------------------------------------------- dW1 = X^T . dH (tensor) --
    if (warp == 0) {
      if (elect_one()) {
        for (int mt = 0; mt < NM; ++mt)
#pragma unroll
          for (int k16 = 0; k16 < kB / 16; ++k16)
            mma_bf16_ss(tmem + gcol + mt * 64,
                        desc_mnmajor_sw128(smem_u32(sX) + (2 * mt) * 16384 + k16 * 2048, 16384, 1024),
                        desc_mnmajor_sw128(smem_u32(sDH) + k16 * 2048, 16384, 1024), idg, k16 != 0);
        mma_commit(gfull);
      }
      __syncwarp();
    }

    // -------------------- dW2 = R^T.dL, db1 = dH^T.1, db2 = dL^T.1 (fp32) --
    {
      const int h = tid >> 2, cq = tid & 3;  // hidden unit, class quad
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 16
      for (int i = 0; i < kB; ++i) {
        const float rv = sR[r_idx(i, h)];
        const float4 d = reinterpret_cast<const float4*>(sDL + i * kC)[cq];
        acc.x = __fmaf_rn(rv, d.x, acc.x);
        acc.y = __fmaf_rn(rv, d.y, acc.y);
        acc.z = __fmaf_rn(rv, d.z, acc.z);
        acc.w = __fmaf_rn(rv, d.w, acc.w);
      }
      float4* w = reinterpret_cast<float4*>(sW2 + h * kC) + cq;
      const float4 o = *w;
      *w = make_float4(__fmaf_rn(-lr, acc.x, o.x), __fmaf_rn(-lr, acc.y, o.y),
                       __fmaf_rn(-lr, acc.z, o.z), __fmaf_rn(-lr, acc.w, o.w));
    }
    if (tid < kHS) {  // db1 from the bf16 dH operand (as the dW1 contraction sees it)
      const int hc = tid >> 3, hw = tid & 7;
      float acc = 0.0f;
#pragma unroll 16
      for (int i = 0; i < kB; ++i)
        acc = __fadd_rn(acc, bf16_to_f32(*reinterpret_cast<const uint16_t*>(
                                 sDH + i * 128 + ((hc ^ (i & 7)) << 4) + hw * 2)));
      sB1[tid] = __fmaf_rn(-lr, acc, sB1[tid]);
    } else if (tid >= 2 * kHS && tid < 2 * kHS + kC) {
      const int c = tid - 2 * kHS;
      float acc = 0.0f;
#pragma unroll 16
      for (int i = 0; i < kB; ++i) acc = __fadd_rn(acc, sDL[i * kC + c]);
      sB2[c] = __fmaf_rn(-lr, acc, sB2[c]);
    }

    // ------------------ next rows in flight, then the master update (TMEM) --
    mbar_wait(gfull, ph);
    tc_fence_after();
    __syncthreads();  // R / dH reads done: the W1 operand may be rewritten
    if (more) gather(cur ^ 1);  // X is free once dW1 completed
    for (int mt = 0; mt < NM; ++mt) {
      uint32_t wr[32], gr[32];
      tmem_ld32_nowait(tmem + lane_base + mt * 64 + p * 32, wr);
      tmem_ld32_nowait(tmem + lane_base + gcol + mt * 64 + p * 32, gr);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        wr[i] = __float_as_uint(__fmaf_rn(-lr, __uint_as_float(gr[i]), __uint_as_float(wr[i])));
      tmem_st32(tmem + lane_base + mt * 64 + p * 32, wr);
      put_row32(sSC, mt * 128 + s, p, wr);
    }
    tmem_st_wait();
    cp_async_wait_all();
    fence_async_smem();  // X rows + W1 operand -> next forward
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  // ------------------------------------------------------------ write back --
  for (int mt = 0; mt < NM; ++mt) {
    const int f = mt * 128 + s;
    uint32_t wr[32];
    tmem_ld32_nowait(tmem + lane_base + mt * 64 + p * 32, wr);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const size_t o = (size_t)(h0 + p * 32 + i) * F + f;
      const float w = __uint_as_float(wr[i]);
      W1[o] = w;
      if (a.w1t) a.w1t[(size_t)slot * H * F + o] = (uint16_t)(pack_bf16x2(w, 0.0f) & 0xFFFF);
    }
  }
  for (int i = tid; i < kHS * kC / 4; i += kThreads)
    reinterpret_cast<float4*>(W2 + (size_t)h0 * kC)[i] = reinterpret_cast<const float4*>(sW2)[i];
  if (tid < kHS) b1[h0 + tid] = sB1[tid];
  if (r == 0 && tid < kC) b2[tid] = sB2[tid];
  if (r == 0 && tid == 0) {
    double acc = 0.0;
    for (int i = 0; i < kB; ++i) acc += sLoss[i];
    a.losses[(size_t)slot * a.loss_T + a.loss_t] = (float)(acc / kB);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, tmem_cols(F));
}

}  // namespace

namespace fused {

bool train_supported(const ecco_ctx* ctx) {
  const ecco_config& g = ctx->cfg;
  if (g.minibatch != kB || g.num_classes != kC || g.feat_dim % 128 || g.feat_dim > 512 ||
      g.hidden_dim % kHS || g.hidden_dim / kHS > kMaxCluster || g.hidden_dim / kHS < 1)
    return false;
  return layout(g.feat_dim).total <= 232448;
}

void train_chain(ecco_ctx* ctx, const Shadow* sh, int n_jobs, const int* d_slots,
                 const int* d_job_ids, const int* d_steps, const int* h_steps,
                 const int* d_src_off, const int* d_src_cam, const double* d_src_frac,
                 const int* d_micro_base, int micro_add, int window, float* wbase, size_t wstride,
                 int loss_t) {
  if (n_jobs == 0) return;
  const ecco_config& c = ctx->cfg;
  const LDims g{c.feat_dim, c.hidden_dim, c.num_classes, c.scene_dims, c.minibatch,
                c.ring_frames, c.eval_samples, c.sgd_lr, c.feature_noise};
  int max_steps = 0;
  for (int j = 0; j < n_jobs; ++j) max_steps = std::max(max_steps, h_steps[j]);
  if (max_steps == 0) return;
  ECCO_REQUIRE((double)c.max_cameras * c.ring_frames < 2147483647.0,
               "fused SGD chain: frame-table rows must fit int32");
  const size_t nrows = (size_t)n_jobs * max_steps * kB;
  int32_t* rows = (int32_t*)ctx->train_scratch[0].get(nrows * 4);
  int32_t* labs = (int32_t*)ctx->train_scratch[1].get(nrows * 4);
  k_chain_rows<<<dim3(n_jobs, max_steps), kB, 0, ctx->stream>>>(
      g, c.seed, d_job_ids, d_steps, d_src_off, d_src_cam, d_src_frac, d_micro_base, micro_add,
      window, max_steps, ctx->d_labels, rows, labs);
  ECCO_LAUNCHED(ctx);
  ChainArgs a{};
  a.g = g;
  a.slots = d_slots;
  a.steps = d_steps;
  a.rows = rows;
  a.labs = labs;
  a.max_steps = max_steps;
  a.frames = ctx->d_frames;
  a.wbase = wbase;
  a.wstride = wstride;
  a.w1t = sh ? sh->w1t : nullptr;
  a.losses = ctx->d_losses;
  a.loss_T = c.max_depth;
  a.loss_t = loss_t;
  const uint32_t smem = layout(c.feat_dim).total;
  static bool attr = false;
  if (!attr) {
    ECCO_CUDA(cudaFuncSetAttribute(k_train_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    attr = true;
  }
  const int cs = c.hidden_dim / kHS;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(cs * n_jobs));
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  // algorithmic work: every live step's fwd + bwd; bytes: fp32 masters in and
  // out once per chain plus the gathered rows
  const double F = c.feat_dim, H = c.hidden_dim, C = c.num_classes;
  double steps = 0, live = 0;
  for (int j = 0; j < n_jobs; ++j) {
    steps += h_steps[j];
    live += h_steps[j] > 0;
  }
  const double flops = steps * kB * (4.0 * F * H + 6.0 * H * C);
  const double params = F * H + H + H * C + C;
  const double bytes = steps * kB * F * 2.0 + live * params * 8.0;
  ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_STEP, flops, bytes,
             ECCO_CUDA(cudaLaunchKernelEx(&lc, k_train_chain, a)));
  ECCO_LAUNCHED(ctx);
}

}  // namespace fused
