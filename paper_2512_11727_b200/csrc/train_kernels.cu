// Fused SGD chain of the learned backend (tensor-core math): ONE launch runs
// every group's whole micro-window -- steps[j] SGD steps, each sampling,
// gather, forward, softmax cross-entropy, backward and update -- on one
// thread-block cluster per group (job).  The group's model never leaves the
// chip between steps: HBM sees the fp32 masters once in and once out per
// micro-window, plus the sampled frame rows.
//
// Cluster of H/64 CTAs; CTA r owns hidden units [64r, 64r+64):
//   TMEM     fp32 master slice W1[:, 64r:64r+64] (F/128 tiles of 128 lanes x
//            64 columns), the forward / dH accumulators (128 x 64), the
//            partial logits (128 x 16) and dW2 (64 x 16)
//   smem     X tile (128 sampled rows, bf16, 128B-swizzled K-major; also read
//            MN-major as X^T), the bf16 W1 operand built from the master, the
//            bf16 W2 slice image, R / dH / dL operands, fp32 W2/b1 slices, b2
//   step     Z = X.W1 (tcgen05 kind::f16, N = 64) -> R = relu(Z+b1) ->
//            partial logits R.W2 (tcgen05, N = 16) sent to the CTA owning the
//            row block by st.async over DSMEM -> owner (4 threads per row)
//            sums the partials in fixed order, softmax, dL, broadcasts dL
//            rows -> dL.W2^T and dW2 = R^T.dL (tcgen05) -> dH =
//            (dL.W2^T)*(Z>0) -> the master ACCUMULATES X^T.(-lr dH) on the
//            tensor core (D += A.B into the TMEM master, one commit per
//            128-feature tile) and -lr db1 = (-lr dH)^T.1 -> bf16 W1 operand
//            rows rebuilt from each finished tile; the next step's rows are
//            prefetched to L2 while dL is in flight and gathered (cp.async)
//            into each X chunk as soon as the tile reading it completes
//
// Numerics: X exact (bf16 frames); every tensor-core operand bf16 (W1, R,
// W2, dL, -lr dH), fp32 accumulation, fp32 masters (W1 += X^T.bf16(-lr dH)
// in the accumulator); bias adds, softmax, dL and db2 fp32 on CUDA cores.  Tolerance in tests/test_gpu_learned.py.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "learned_common.cuh"
#include "sm100.cuh"
#include "chain_common.cuh"

using namespace sm100;
using namespace chain;

namespace {

constexpr int kB = 128;        // minibatch rows = UMMA M
constexpr int kThreads = 256;  // 8 warps: lane quadrant q = warp % 4, half p = warp / 4
constexpr int kC = 16;         // classes (logits held in registers)
constexpr int kHS = 64;        // hidden units per CTA of the cluster
constexpr int kMaxCluster = 8;
constexpr int kGatherWarps = 4;  // warps 1-4 each issue a quarter of a tile's gather4 copies

struct ChainArgs {
  LDims g;
  const int* slots;
  const int* steps;
  const int32_t* rows;  // [job][max_steps][kB] frame-table row of every sampled frame
  const int32_t* labs;  // [job][max_steps][kB] its label
  int max_steps;
  int row_step0;        // first row step of this micro-window in rows / labs
  int rows_T;           // row steps per job in rows / labs (micro-windows x max_steps)
  const uint16_t* frames;
  const float* wsrc;    // fp32 masters the micro-window starts from (W1 stored [H][F])
  size_t wsrc_stride;
  float* wbase;         // ... and where it leaves them (a snapshot; may equal wsrc)
  size_t wstride;
  uint16_t* w1t;  // bf16 W1^T evaluation shadow [slot][H][F], written at the end
  float* losses;  // losses[slot * loss_T + loss_t] = mean loss of the last step
  int loss_T, loss_t;
  // Serial mode (n_micro_launch > 1, one job): the launch trains that many
  // consecutive micro-windows from on-chip state, leaving micro-window u's
  // model at wbase + u * wmicro (and its loss at loss_t + u)
  int n_micro_launch;
  size_t wmicro;
};

// Every (job, step, row) draw of the micro-window, ahead of the chain
// (sample_one: the same draws as k_l_sample and the oracle's orc_sample).
// (grid.y covers n_micro x max_steps row steps: micro-window micro_add + y /
// max_steps, step y % max_steps; rows laid out [job][micro][step][kB])
__global__ void k_chain_rows(LDims g, uint64_t seed, const int* job_ids, const int* steps,
                             const int* src_off, const int* src_cam, const double* src_frac,
                             const int* micro_base, int micro_add, int window, int max_steps,
                             const int32_t* labels, int32_t* rows, int32_t* labs) {
  const int j = blockIdx.x, step = blockIdx.y % max_steps, mi = blockIdx.y / max_steps;
  const int s = threadIdx.x;
  if (step >= steps[j]) return;
  int cam, frame;
  const int s0 = src_off[j];
  sample_one(g, seed, job_ids[j], src_off[j + 1] - s0, src_cam + s0, src_frac + s0, window,
             micro_base[j] + micro_add + mi, step, s, &cam, &frame);
  const int32_t row = cam * g.R + frame;
  const size_t o = ((size_t)j * gridDim.y + blockIdx.y) * kB + s;
  rows[o] = row;
  labs[o] = labels[row];
}

struct Layout {
  uint32_t x, sc, dlb, ones, w2i, dl, recv, w2, b1, b2, rows, labs, loss, bars, tmem, total;
};

// sc: the bf16 W1 operand (MN-major: F rows of 64 hidden units, 128 B); R
// (bf16, 128 x 64) and dH (bf16, MN-major over rows) occupy its last 32 KB
// between the forward MMA and the update of the last dW1 pass.
__host__ __device__ inline Layout layout(int F) {
  Layout L{};
  uint32_t o = 0;
  L.x = o;
  o += (uint32_t)(F / 64) * 16384u;
  L.sc = o;
  o += std::max((uint32_t)F * 128u, 32768u);
  L.dlb = o;
  o += kB * 32u;  // bf16 dL [row][16], 32B-swizzled
  L.ones = o;
  o += kB * 32u;  // bf16 1.0 [row][16]: db1 = dH^T . 1 on the tensor core
  L.w2i = o;
  o += kC * 128u;  // bf16 W2 slice image [class][64 hidden], 128B-swizzled
  L.dl = o;
  o += kB * kC * 4u;
  L.recv = o;
  o += kB * kC * 4u;  // [src rank][row of the owner block][class]
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
  o += 20u * 8u;
  L.tmem = o;
  o += 16u;
  L.total = o;
  return L;
}

// TMEM columns: master [0, 64*NM) (the dW1 MMAs accumulate into it), Z /
// dL.W2^T [A, A+64), partial logits / -lr db1 [A+64, A+80), dW2 [A+80, A+96)
// with A = 64*NM.
__host__ __device__ inline uint32_t tmem_cols(int) { return 512; }

// bf16 dL row (16 classes, 32 B) of the 32B-swizzled tile: K-major A of
// dL.W2^T and MN-major B of dW2 = R^T.dL share it.
__device__ __forceinline__ uint32_t dlb_off(int row, int chunk) {
  return (uint32_t)row * 32u + ((uint32_t)(chunk ^ ((row >> 2) & 1)) << 4);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_train_chain(const __grid_constant__ CUtensorMap map_rows, ChainArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const LDims g = a.g;
  const int F = g.F, H = g.H;
  const int cs = H / kHS;
  const int j = blockIdx.x / cs;
  const int r = (int)cluster_ctarank();
  const int nsteps = a.steps[j];
  if (nsteps <= 0) {  // no step: the snapshot is the starting model (the cluster copies it)
    const int slot0 = a.slots[j];
    const float* src = a.wsrc + (size_t)slot0 * a.wsrc_stride;
    float* dst = a.wbase + (size_t)slot0 * a.wstride;
    if (src != dst) {
      const size_t np = (size_t)g.F * g.H + g.H + (size_t)g.H * g.C + g.C;
      for (size_t i = (size_t)r * blockDim.x + threadIdx.x; i < np; i += (size_t)cs * blockDim.x)
        dst[i] = src[i];
    }
    return;  // the whole cluster (same job) leaves
  }
  const Layout L = layout(F);
  const uint32_t SC = std::max((uint32_t)F * 128u, 32768u);
  uint8_t* sX = smem + L.x;
  uint8_t* sSC = smem + L.sc;                 // W1 operand, MN-major [f][64 hidden]
  uint8_t* sR = sSC + SC - 32768u;            // bf16 R [row][64], K-major / MN-major
  uint8_t* sDH = sSC + SC - 16384u;           // bf16 dH [row][64], MN-major over rows
  uint8_t* sDLb = smem + L.dlb;
  uint8_t* sW2i = smem + L.w2i;
  uint8_t* sOnes = smem + L.ones;
  float* sB2r = (float*)(smem + L.dl);  // [kB / 8][kC] db2 partial sums of 8-row blocks
  float* sRecv = (float*)(smem + L.recv);
  float* sW2 = (float*)(smem + L.w2);
  float* sB1 = (float*)(smem + L.b1);
  float* sB2 = (float*)(smem + L.b2);
  int* sRow = (int*)(smem + L.rows);          // [2][kB] frame-table rows
  int* sLab = (int*)(smem + L.labs);          // [2][kB]
  float* sLoss = (float*)(smem + L.loss);
  uint64_t* zfull = (uint64_t*)(smem + L.bars);
  uint64_t* plfull = zfull + 1;
  uint64_t* dhfull = zfull + 2;  // dL.W2^T and dW2 accumulated
  uint64_t* recv_full = zfull + 5;  // owner rows' partial logits arrived (st.async)
  uint64_t* dl_full = zfull + 6;    // every dL row (and, on rank 0, every loss) arrived
  uint64_t* w2full = zfull + 7;     // dW2 accumulated
  uint64_t* gt = zfull + 8;         // [NM] dW1 tile mt accumulated into the master
  uint64_t* xready = zfull + 12;    // [NM] tile mt's W1 operand rows rebuilt in smem
  uint64_t* xfull = zfull + 16;     // [NM] tile mt's next-step X chunks landed (TMA gather4)
  uint32_t* sTmem = (uint32_t*)(smem + L.tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, p = warp >> 2;
  const int s = q * 32 + lane;  // minibatch row of this thread (TMEM lane)
  const uint32_t lane_base = (uint32_t)(q * 32) << 16;
  const int RP = kB / cs;       // rows owned per CTA for the softmax
  const int NM = F / 128;       // master / dW1 tiles
  const int nkc = F / 64;
  const uint32_t acol = (uint32_t)NM * 64u;  // Z / dL.W2^T
  const uint32_t plcol = acol + 64u, w2col = acol + 80u;
  const int slot = a.slots[j];
  float* W1 = a.wbase + (size_t)slot * a.wstride;
  float* b1 = W1 + (size_t)F * H;
  float* W2 = b1 + H;
  float* b2 = W2 + (size_t)H * kC;
  const float* sW1 = a.wsrc + (size_t)slot * a.wsrc_stride;  // the starting model
  const float* sb1 = sW1 + (size_t)F * H;
  const float* sW2g = sb1 + H;
  const float* sb2 = sW2g + (size_t)H * kC;
  const float lr = g.lr;
  const int h0 = r * kHS;  // first hidden unit of this CTA
  const int32_t* jrows = a.rows + ((size_t)j * a.rows_T + a.row_step0) * kB;
  const int32_t* jlabs = a.labs + ((size_t)j * a.rows_T + a.row_step0) * kB;
  const uint32_t recv_bytes = kB * kC * 4u;
  // bf16 dL rows + the 8-row db2 partials (+ every row's loss on rank 0)
  const uint32_t dl_bytes = kB * 32u + (kB / 8) * kC * 4u + (r == 0 ? kB * 4u : 0u);

  // rows of buffer `buf`, 16-byte pieces [c0, c0 + n) of each row (n a power
  // of two) -> X tile, by threads [t0, kThreads); a warp covers consecutive
  // pieces of one row, piece c16 lands in chunk c16/8
  const uint32_t xsm = smem_u32(sX);
  auto gather = [&](int buf, int c0, int n, int t0) {
    const int* rows = sRow + buf * kB;
    const int lsh = 31 - __clz(n);
#pragma unroll 4
    for (int pc = tid - t0; pc < kB * n; pc += kThreads - t0) {
      const int i = pc >> lsh, c16 = c0 + (pc & (n - 1));
      cp_async16_s(xsm + (c16 >> 3) * 16384 + i * 128 + (((c16 & 7) ^ (i & 7)) << 4),
                   a.frames + (int64_t)rows[i] * F + c16 * 8);
    }
  };
  auto build_w2i = [&]() {
    for (int e = tid; e < kC * kHS / 8; e += kThreads) {
      const int c = e >> 3, hc = e & 7;
      const float* w = sW2 + hc * 8 * kC + c;
      uint4 pk;
      pk.x = pack_bf16x2(w[0 * kC], w[1 * kC]);
      pk.y = pack_bf16x2(w[2 * kC], w[3 * kC]);
      pk.z = pack_bf16x2(w[4 * kC], w[5 * kC]);
      pk.w = pack_bf16x2(w[6 * kC], w[7 * kC]);
      *reinterpret_cast<uint4*>(sW2i + c * 128 + ((hc ^ (c & 7)) << 4)) = pk;
    }
  };

  // ---------------------------------------------------------------- setup --
  if (tid == 0) {
    if (smem_u32(smem) & 1023u) __trap();  // 128B-swizzle atoms need 1 KB alignment
    mbar_init(zfull, 1);
    mbar_init(plfull, 1);
    mbar_init(dhfull, 1);
    for (int mt = 0; mt < NM; ++mt) {
      mbar_init(gt + mt, 1);
      mbar_init(xready + mt, kThreads - 32);
      mbar_init(xfull + mt, kGatherWarps);
    }
    mbar_init(recv_full, 1);
    mbar_init(dl_full, 1);
    mbar_init(w2full, 1);
    fence_barrier_init();
  }
  // this CTA's master slice (64 rows x F fp32) -> L2 at once: the tile-by-tile
  // loads below then wait on L2, not on four HBM round trips
  for (int li = tid; li < kHS * (F / 32); li += kThreads)
    prefetch_l2(sW1 + (size_t)(h0 + li / (F / 32)) * F + (li % (F / 32)) * 32);
  if (warp == 0) tmem_alloc(sTmem, tmem_cols(F));
  if (tid < kB) {
    sRow[tid] = jrows[tid];
  } else {
    sLab[tid - kB] = jlabs[tid - kB];
  }
  for (int i = tid; i < kHS * kC / 4; i += kThreads)
    reinterpret_cast<float4*>(sW2)[i] = reinterpret_cast<const float4*>(sW2g + (size_t)h0 * kC)[i];
  if (tid < kHS) sB1[tid] = sb1[h0 + tid];
  if (tid < kC) sB2[tid] = sb2[tid];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sTmem;
  gather(0, 0, F / 8, 0);
  build_w2i();
  for (int i = tid; i < kB * 32 / 16; i += kThreads)
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  // master slice -> TMEM; its bf16 image -> the W1 operand
  for (int mt = 0; mt < NM; ++mt) {
    const int f = mt * 128 + s;
    uint32_t w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(sW1[(size_t)(h0 + p * 32 + i) * F + f]);
    tmem_st32(tmem + lane_base + mt * 64 + p * 32, w);
    put_row32(sSC, f, p, w);
  }
  tmem_st_wait();
  cp_async_wait_all();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA of the cluster is running before any DSMEM traffic
  tc_fence_after();

  const uint32_t idf = idesc_major(kB, kHS, kFmtBF16, 0, 1);     // X . W1
  const uint32_t idl = idesc(kB, kC, kFmtBF16);                  // R . W2
  const uint32_t idh = idesc_major(kB, kHS, kFmtBF16, 0, 1);     // dL . W2^T
  const uint32_t idw2 = idesc_major(128, kC, kFmtBF16, 1, 1);    // R^T . dL (rows 64+ alias)
  const uint32_t idg = idesc_major(128, kHS, kFmtBF16, 1, 1);    // X^T . dH
  const uint32_t idb = idesc_major(128, kC, kFmtBF16, 1, 1);     // dH^T . 1 (rows 64+ alias)
  const uint64_t dX = desc_kmajor_sw128(smem_u32(sX));
  auto issue_fwd = [&](int kc0, int kc1) {  // Z (+)= X[:, chunks kc0..kc1) . W1
    for (int kc = kc0; kc < kc1; ++kc)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16_ss(tmem + acol, dX + ((kc * 16384 + kk * 32) >> 4),
                    desc_mnmajor_sw128(smem_u32(sSC) + (kc * 4 + kk) * 2048, 16384, 1024), idf,
                    (kc | kk) != 0);
  };

  // global step index over the launch's micro-windows (serial mode: the
  // rows of one job's consecutive micro-windows are consecutive row steps)
  const int total = nsteps * a.n_micro_launch;
  for (int step = 0; step < total; ++step) {
    const int cur = step & 1;
    const uint32_t ph = (uint32_t)step & 1u;
    const bool more = step + 1 < total;
    // the last step of a micro-window that is not the launch's last: its
    // model is written out as the rebuild reads it (serial mode)
    const bool boundary = more && (step + 1) % nsteps == 0;
    const size_t snap = (size_t)(step / nsteps) * a.wmicro;
    if (tid == 0) {  // this step's incoming DSMEM bytes
      mbar_expect_tx(recv_full, recv_bytes);
      mbar_expect_tx(dl_full, dl_bytes);
    }
    // ------------------------------------------------------ forward MMA --
    // (steps after the first: issued tile by tile at the end of the
    // previous step, as the W1 operand rows and the gathered rows land)
    if (step == 0 && warp == 0) {
      if (elect_one()) {
        issue_fwd(0, nkc);
        mma_commit(zfull);
      }
      __syncwarp();
    }
    // next step's rows: loads in flight across the forward and the head
    int32_t nxt = 0;
    if (more) nxt = tid < kB ? jrows[(step + 1) * kB + tid] : jlabs[(step + 1) * kB + tid - kB];
    mbar_wait(zfull, ph);
    tc_fence_after();

    // ---------------------------- R = relu(Z + b1) -> partial logits MMA --
    uint32_t mask;  // bit i: Z + b1 > 0 for hidden unit p*32 + i
    {
      uint32_t zr[32];
      tmem_ld32_nowait(tmem + lane_base + acol + p * 32, zr);
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
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ss(tmem + plcol, desc_kmajor_sw128(smem_u32(sR) + kk * 32),
                      desc_kmajor_sw128(smem_u32(sW2i) + kk * 32), idl, kk != 0);
        mma_commit(plfull);
      }
      __syncwarp();
    }
    mbar_wait(plfull, ph);
    tc_fence_after();
    if (p == 0) {  // partials -> the CTA owning row s
      uint32_t pl[kC];
      tmem_ld16_nowait(tmem + lane_base + plcol, pl);
      tmem_ld_wait();
      const uint32_t o = (uint32_t)(s / RP);
      const uint32_t dst = mapa_shared(smem_u32(sRecv + (r * RP + (s % RP)) * kC), o);
      const uint32_t bar = mapa_shared(smem_u32(recv_full), o);
#pragma unroll
      for (int c4 = 0; c4 < kC / 4; ++c4)
        st_async_v4(dst + c4 * 16, __uint_as_float(pl[4 * c4]), __uint_as_float(pl[4 * c4 + 1]),
                    __uint_as_float(pl[4 * c4 + 2]), __uint_as_float(pl[4 * c4 + 3]), bar);
    }

    // ----------------------- owner rows: logits, softmax, dL broadcast --
    // four threads per owned row (warps 4..), one class quad each
    if (tid >= kB && tid < kB + 4 * RP) {
      mbar_wait(recv_full, ph);
      const int t = (tid - kB) >> 2, cq = tid & 3, row = r * RP + t;
      const float4* rv = reinterpret_cast<const float4*>(sRecv);
      float4 lg = rv[t * 4 + cq];
      for (int src = 1; src < cs; ++src) {
        const float4 v = rv[(src * RP + t) * 4 + cq];
        lg = make_float4(__fadd_rn(lg.x, v.x), __fadd_rn(lg.y, v.y), __fadd_rn(lg.z, v.z),
                         __fadd_rn(lg.w, v.w));
      }
      const float4 bb = reinterpret_cast<const float4*>(sB2)[cq];
      lg = make_float4(__fadd_rn(lg.x, bb.x), __fadd_rn(lg.y, bb.y), __fadd_rn(lg.z, bb.z),
                       __fadd_rn(lg.w, bb.w));
      float m = fmaxf(fmaxf(lg.x, lg.y), fmaxf(lg.z, lg.w));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
      const float4 e = make_float4(expf_nb(__fsub_rn(lg.x, m)), expf_nb(__fsub_rn(lg.y, m)),
                                   expf_nb(__fsub_rn(lg.z, m)), expf_nb(__fsub_rn(lg.w, m)));
      float sum = __fadd_rn(__fadd_rn(e.x, e.y), __fadd_rn(e.z, e.w));
      sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, 1));
      sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, 2));
      constexpr float invB = 1.0f / kB;  // exact (power of two)
      const float inv = __frcp_rn(sum);
      const int y = sLab[cur * kB + row] - cq * 4;  // class within this quad (0..3 if mine)
      const float4 dl = make_float4(__fmul_rn(__fsub_rn(__fmul_rn(e.x, inv), y == 0 ? 1.0f : 0.0f), invB),
                                    __fmul_rn(__fsub_rn(__fmul_rn(e.y, inv), y == 1 ? 1.0f : 0.0f), invB),
                                    __fmul_rn(__fsub_rn(__fmul_rn(e.z, inv), y == 2 ? 1.0f : 0.0f), invB),
                                    __fmul_rn(__fsub_rn(__fmul_rn(e.w, inv), y == 3 ? 1.0f : 0.0f), invB));
      // bf16 dL straight into every CTA's MMA operand tile, and the fp32 db2
      // partial of this warp's 8 rows (fixed butterfly over the row lanes)
      const uint32_t lo = pack_bf16x2(dl.x, dl.y), hi = pack_bf16x2(dl.z, dl.w);
      float4 b2s = dl;
#pragma unroll
      for (int x = 4; x < 32; x <<= 1)
        b2s = make_float4(__fadd_rn(b2s.x, __shfl_xor_sync(0xffffffffu, b2s.x, x)),
                          __fadd_rn(b2s.y, __shfl_xor_sync(0xffffffffu, b2s.y, x)),
                          __fadd_rn(b2s.z, __shfl_xor_sync(0xffffffffu, b2s.z, x)),
                          __fadd_rn(b2s.w, __shfl_xor_sync(0xffffffffu, b2s.w, x)));
      const uint32_t dlo = dlb_off(row, cq >> 1) + (cq & 1) * 8u;
      for (int d = 0; d < cs; ++d) {
        const uint32_t bar = mapa_shared(smem_u32(dl_full), (uint32_t)d);
        st_async_v2b32(mapa_shared(smem_u32(sDLb) + dlo, (uint32_t)d), lo, hi, bar);
        if ((lane >> 2) == 0)
          st_async_v4(mapa_shared(smem_u32(sB2r + (row >> 3) * kC + cq * 4), (uint32_t)d), b2s.x,
                      b2s.y, b2s.z, b2s.w, bar);
      }
      if (y >= 0 && y < 4) {
        const float ly = y == 0 ? lg.x : y == 1 ? lg.y : y == 2 ? lg.z : lg.w;
        st_async_f32(mapa_shared(smem_u32(sLoss + row), 0u), __logf(sum) - (ly - m),
                     mapa_shared(smem_u32(dl_full), 0u));
      }
    }
    if (more) {  // next step's rows into the other buffer
      if (tid < kB)
        sRow[(cur ^ 1) * kB + tid] = nxt;
      else
        sLab[(cur ^ 1) * kB + tid - kB] = nxt;
    }
    if (more && tid < kB) {  // next rows -> L2 (this CTA's block of them), while dL is in flight
      const int lpr = F / 64;  // 128-byte lines per row
      for (int li = tid; li < RP * lpr; li += kB) {
        const int row = r * RP + li / lpr;
        prefetch_l2(a.frames + (int64_t)jrows[(step + 1) * kB + row] * F + (li % lpr) * 64);
      }
    }
    mbar_wait(dl_full, ph);

    // ------------------------------------- dL.W2^T and dW2 = R^T.dL --
    // (the owners wrote the bf16 dL tile with st.async: no local pass)
    if (warp == 0) {
      fence_async_smem();
      tc_fence_after();
      if (elect_one()) {
        mma_bf16_ss(tmem + acol, smem_desc(smem_u32(sDLb), 16, 256, kSwizzle32B),
                    desc_mnmajor_sw128(smem_u32(sW2i), 16384, 1024), idh, 0);
        mma_commit(dhfull);
#pragma unroll
        for (int k16 = 0; k16 < kB / 16; ++k16)
          mma_bf16_ss(tmem + w2col, desc_mnmajor_sw128(smem_u32(sR) + k16 * 2048, 0, 1024),
                      smem_desc(smem_u32(sDLb) + k16 * 512, 256, 256, kSwizzle32B), idw2, k16 != 0);
        mma_commit(w2full);
      }
      __syncwarp();
    }
    mbar_wait(dhfull, ph);
    tc_fence_after();

    // ------------------------------------------------ dH = (dL.W2^T)*(Z>0) --
    {
      uint32_t dh[32];
      tmem_ld32_nowait(tmem + lane_base + acol + p * 32, dh);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        dh[i] = (mask >> i) & 1u ? __float_as_uint(__fmul_rn(-lr, __uint_as_float(dh[i]))) : 0u;
      put_row32(sDH, s, p, dh);  // -lr dH, MN-major over rows: dW1's B operand
    }
    fence_async_smem();  // dH (generic stores) -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    // ---------- dW1: the master accumulates X^T . (-lr dH) on the tensor core --
    // one commit per 128-feature tile: its bf16 operand rows are rebuilt and
    // the next rows' X chunks gathered while the later tiles' MMAs run
    if (warp == 0) {
      if (elect_one()) {
        for (int mt = 0; mt < NM; ++mt) {
#pragma unroll
          for (int k16 = 0; k16 < kB / 16; ++k16)
            mma_bf16_ss(tmem + mt * 64,
                        desc_mnmajor_sw128(smem_u32(sX) + (2 * mt) * 16384 + k16 * 2048, 16384, 1024),
                        desc_mnmajor_sw128(smem_u32(sDH) + k16 * 2048, 16384, 1024), idg, 1);
          if (mt == NM - 1)  // -lr db1 into the (consumed) partial-logit columns
#pragma unroll
            for (int k16 = 0; k16 < kB / 16; ++k16)
              mma_bf16_ss(tmem + plcol, desc_mnmajor_sw128(smem_u32(sDH) + k16 * 2048, 0, 1024),
                          smem_desc(smem_u32(sOnes) + k16 * 512, 256, 256, kSwizzle32B), idb,
                          k16 != 0);
          mma_commit(gt + mt);
        }
      }
      __syncwarp();
    }
    // warp 0 is held by the MMA queue until the dW1 MMAs drain: the other
    // warps take its share (warp 4 both column halves of lane quadrant 0)
    if (p == 1 && q < 2) {  // dW2 row h = s (TMEM lanes 0-63)
      mbar_wait(w2full, ph);
      tc_fence_after();
      uint32_t w2r[kC];
      tmem_ld16_nowait(tmem + lane_base + w2col, w2r);
      tmem_ld_wait();
      float4* w = reinterpret_cast<float4*>(sW2 + s * kC);
#pragma unroll
      for (int c4 = 0; c4 < kC / 4; ++c4) {
        const float4 o = w[c4];
        w[c4] = make_float4(__fmaf_rn(-lr, __uint_as_float(w2r[4 * c4]), o.x),
                            __fmaf_rn(-lr, __uint_as_float(w2r[4 * c4 + 1]), o.y),
                            __fmaf_rn(-lr, __uint_as_float(w2r[4 * c4 + 2]), o.z),
                            __fmaf_rn(-lr, __uint_as_float(w2r[4 * c4 + 3]), o.w));
      }
    }
    // (tile 2's rows overwrite R, tile 3's dH: both read by MMAs its commit covers)
    // As soon as tile mt's dW1 MMAs have read its X chunks (gt[mt]), warps
    // 1-4 each issue a quarter of the next step's rows for those two chunks
    // as TMA gather4 copies (4 rows x 128 B each, landing 128B-swizzled where
    // the forward MMA reads them; completion on xfull[mt]), and warps 1-7
    // rebuild the tile's bf16 W1 operand rows from the TMEM master and publish
    // them on xready[mt]; warp 0 issues the next step's forward chunks 2mt,
    // 2mt+1 once both have landed.  The row gather no longer occupies the
    // warps or the LSU (it was a cp.async loop of 2,048 16-byte pieces per tile).
    if (warp > 0) {
      const int* nrows = sRow + (cur ^ 1) * kB;
      for (int mt = 0; mt < NM; ++mt) {
        mbar_wait(gt + mt, ph);
        tc_fence_after();
        if (more && warp <= kGatherWarps) {
          if (elect_one()) {
            constexpr int kGroups = kB / 4 / kGatherWarps;  // row groups of 4 per issuing warp
            mbar_expect_tx(xfull + mt, 2u * kGroups * 512u);
            const int g0 = (warp - 1) * kGroups;
            for (int cc = 0; cc < 2; ++cc) {
              const int kc = 2 * mt + cc;
              for (int gi = g0; gi < g0 + kGroups; ++gi) {
                const int i0 = gi * 4;
                tma_gather4(sX + kc * 16384 + i0 * 128, &map_rows, kc * 64, nrows[i0],
                            nrows[i0 + 1], nrows[i0 + 2], nrows[i0 + 3], xfull + mt);
              }
            }
          }
          __syncwarp();
        }
        uint32_t wr[32];
        tmem_ld32_nowait(tmem + lane_base + mt * 64 + p * 32, wr);
        if (warp == 4) {
          uint32_t w0[32];
          tmem_ld32_nowait(tmem + lane_base + mt * 64, w0);
          tmem_ld_wait();
          put_row32(sSC, mt * 128 + s, 0, w0);
          if (boundary) {
            float* wo = W1 + snap + (size_t)h0 * F + mt * 128 + s;
#pragma unroll
            for (int i = 0; i < 32; ++i) wo[(size_t)i * F] = __uint_as_float(w0[i]);
          }
        } else {
          tmem_ld_wait();
        }
        put_row32(sSC, mt * 128 + s, p, wr);
        if (boundary) {
          float* wo = W1 + snap + (size_t)(h0 + p * 32) * F + mt * 128 + s;
#pragma unroll
          for (int i = 0; i < 32; ++i) wo[(size_t)i * F] = __uint_as_float(wr[i]);
        }
        if (more) {
          fence_async_smem();  // the rebuilt rows (generic stores) -> the forward MMA
          mbar_arrive(xready + mt);
        }
      }
    } else if (more) {
      for (int mt = 0; mt < NM; ++mt) {
        mbar_wait(xready + mt, ph);
        mbar_wait(xfull + mt, ph);
        tc_fence_after();
        if (elect_one()) {
          issue_fwd(2 * mt, 2 * mt + 2);
          if (mt == NM - 1) mma_commit(zfull);
        }
        __syncwarp();
      }
    }
    if (p == 1 && q < 2) {  // db1 row h = s (TMEM lanes 0-63), already scaled by -lr
      uint32_t v[8];
      tmem_ld8_nowait(tmem + lane_base + plcol, v);
      tmem_ld_wait();
      sB1[s] = __fadd_rn(sB1[s], __uint_as_float(v[0]));
    }
    __syncthreads();  // sW2 updated
    build_w2i();
    if (tid >= 32 && tid < 32 + kC) {
      const int c = tid - 32;
      float acc = sB2r[c];
#pragma unroll
      for (int b = 1; b < kB / 8; ++b) acc = __fadd_rn(acc, sB2r[b * kC + c]);
      sB2[c] = __fmaf_rn(-lr, acc, sB2[c]);
    }
    fence_async_smem();  // the W2 operand -> next step's MMAs
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (boundary) {  // the rest of micro-window step / nsteps's model and its loss
      for (int i = tid; i < kHS * kC / 4; i += kThreads)
        reinterpret_cast<float4*>(W2 + snap + (size_t)h0 * kC)[i] = reinterpret_cast<const float4*>(sW2)[i];
      if (tid < kHS) b1[snap + h0 + tid] = sB1[tid];
      if (r == 0 && tid < kC) b2[snap + tid] = sB2[tid];
      if (r == 0 && tid == 0) {
        double acc = 0.0;
        for (int i = 0; i < kB; ++i) acc += sLoss[i];
        a.losses[(size_t)slot * a.loss_T + a.loss_t + step / nsteps] = (float)(acc / kB);
      }
    }
  }

  // ------------------------------------------------------------ write back --
  // (the launch's last micro-window: snapshot n_micro_launch - 1)
  const size_t last = (size_t)(a.n_micro_launch - 1) * a.wmicro;
  W1 += last;
  b1 += last;
  W2 += last;
  b2 += last;
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
    a.losses[(size_t)slot * a.loss_T + a.loss_t + a.n_micro_launch - 1] = (float)(acc / kB);
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
      (g.feat_dim & (g.feat_dim - 1)) ||
      (g.hidden_dim != 4 * kHS && g.hidden_dim != 8 * kHS))
    return false;
  return layout(g.feat_dim).total <= 232448;
}

void chain_rows(ecco_ctx* ctx, int n_jobs, const int* d_job_ids, const int* d_steps,
                const int* h_steps, const int* d_src_off, const int* d_src_cam,
                const double* d_src_frac, const int* d_micro_base, int n_micro, int window,
                bool wide_rows) {
  if (n_jobs == 0 || n_micro == 0) return;
  const ecco_config& c = ctx->cfg;
  const LDims g{c.feat_dim, c.hidden_dim, c.num_classes, c.scene_dims, c.minibatch,
                c.ring_frames, c.eval_samples, c.sgd_lr, c.feature_noise};
  int max_steps = 0;
  for (int j = 0; j < n_jobs; ++j) max_steps = std::max(max_steps, h_steps[j]);
  if (max_steps == 0) return;
  ECCO_REQUIRE((double)c.max_cameras * c.ring_frames < 2147483647.0,
               "fused SGD chain: frame-table rows must fit int32");
  const size_t nrows = (size_t)n_jobs * n_micro * max_steps * kB;
  int32_t* rows = (int32_t*)ctx->train_scratch[0].get(nrows * 4);
  int32_t* labs = (int32_t*)ctx->train_scratch[1].get(nrows * 4);
  k_chain_rows<<<dim3(n_jobs, n_micro * max_steps), kB, 0, ctx->stream>>>(
      g, c.seed, d_job_ids, d_steps, d_src_off, d_src_cam, d_src_frac, d_micro_base, 0, window,
      max_steps, ctx->d_labels, rows, labs);
  ECCO_LAUNCHED(ctx);
  if (wide_rows && !train_supported(ctx)) wide_gather(ctx, n_jobs, d_steps, max_steps, n_micro);
}

void train_chain(ecco_ctx* ctx, const Shadow* sh, int n_jobs, const int* d_slots,
                 const int* d_steps, const int* h_steps, int micro, int n_micro,
                 const float* wsrc, size_t wsrc_stride, float* wbase, size_t wstride,
                 int loss_t, int n_launch, size_t wmicro) {
  if (n_jobs == 0) return;
  ECCO_REQUIRE(n_launch == 1 || (n_jobs == 1 && !sh), "serial chain: one job, no shadow");
  if (!train_supported(ctx)) {  // the detection-head shape: wide_kernels.cu
    train_wide(ctx, n_jobs, d_slots, d_steps, h_steps, micro, n_micro, wsrc, wsrc_stride, wbase,
               wstride, loss_t, n_launch, wmicro);
    return;
  }
  const ecco_config& c = ctx->cfg;
  const LDims g{c.feat_dim, c.hidden_dim, c.num_classes, c.scene_dims, c.minibatch,
                c.ring_frames, c.eval_samples, c.sgd_lr, c.feature_noise};
  int max_steps = 0;
  for (int j = 0; j < n_jobs; ++j) max_steps = std::max(max_steps, h_steps[j]);
  ChainArgs a{};
  a.g = g;
  a.slots = d_slots;
  a.steps = d_steps;
  a.rows = (const int32_t*)ctx->train_scratch[0].p;  // chain_rows() of this call
  a.labs = (const int32_t*)ctx->train_scratch[1].p;
  a.max_steps = max_steps;
  a.row_step0 = micro * max_steps;
  a.rows_T = n_micro * max_steps;
  a.frames = ctx->d_frames;
  a.wsrc = wsrc;
  a.wsrc_stride = wsrc_stride;
  a.wbase = wbase;
  a.wstride = wstride;
  a.w1t = sh ? sh->w1t : nullptr;
  a.losses = ctx->d_losses;
  a.loss_T = c.max_depth;
  a.loss_t = loss_t;
  a.n_micro_launch = n_launch;
  a.wmicro = wmicro;
  const uint32_t smem = layout(c.feat_dim).total;
  static DeviceFlags attr;  // per device: the attribute applies to the current device
  if (!attr.done(c.device)) {  // the opt-in maximum: every supported shape fits
    ECCO_CUDA(cudaFuncSetAttribute(k_train_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   232448));
    attr.mark(c.device);
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
    steps += (double)h_steps[j] * n_launch;
    live += h_steps[j] > 0;
  }
  const double flops = steps * kB * (4.0 * F * H + 6.0 * H * C);
  const double params = F * H + H + H * C + C;
  const double bytes = steps * kB * F * 2.0 + live * params * 4.0 * (1 + n_launch);
  // the frame table as a 2-D bf16 tensor [camera*R + frame][F]: TMA gather4
  // rows of 64 columns, 128B swizzle (the forward's X operand layout)
  const CUtensorMap map_rows =
      tensor_map_bf16(ctx->d_frames, (uint64_t)ctx->cfg.max_cameras * c.ring_frames, c.feat_dim, 1);
  ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_STEP, flops, bytes,
             ECCO_CUDA(cudaLaunchKernelEx(&lc, k_train_chain, map_rows, a)));
  ECCO_LAUNCHED(ctx);
}

}  // namespace fused
