// Sampled-row ingest: instead of uploading every camera's ring, the window's
// SGD draws are marked in a bitmap on the device and only the marked rows
// are read straight out of pinned host memory (zero-copy over PCIe) into the
// back frame buffer, on the copy stream, while the previous window computes.
// The rows the kernels later read are exactly the marked ones (same draws),
// so the result is identical to a full upload (tests/test_gpu_learned.py).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "ctx.cuh"
#include "learned_common.cuh"

namespace {

// Marks every ring row the trajectories' SGD steps draw (the same
// counter-RNG draws as the chain, sample_one) in `flags`; in check mode
// (have != null) counts the draws whose row is NOT in `have` instead.
__global__ void k_mark_sampled(LDims g, uint64_t seed, const int* job_ids, const int* steps,
                               const int* src_off, const int* src_cam, const double* src_frac,
                               const int* micro_base, int window, uint32_t* flags,
                               const uint32_t* have, unsigned* missing) {
  const int j = blockIdx.x, step = blockIdx.y, t = blockIdx.z;
  if (step >= steps[j]) return;
  const int s0 = src_off[j];
  for (int s = threadIdx.x; s < g.B; s += blockDim.x) {
    int cam, frame;
    sample_one(g, seed, job_ids[j], src_off[j + 1] - s0, src_cam + s0, src_frac + s0, window,
               micro_base[j] + t, step, s, &cam, &frame);
    const uint32_t row = (uint32_t)cam * (uint32_t)g.R + (uint32_t)frame;
    if (have) {
      if (!((have[row >> 5] >> (row & 31)) & 1u)) atomicAdd(missing, 1u);
    } else {
      atomicOr(flags + (row >> 5), 1u << (row & 31));
    }
  }
}

// One warp per 32-row bitmap word (grid-stride); the warp copies the word's
// marked rows G at a time, every lane holding up to kPieces 16-byte pieces
// in flight (PCIe reads are latency-bound: ILP, not bandwidth, per warp).
constexpr int kPieces = 6;
__global__ void __launch_bounds__(1024, 1) k_fetch_rows(const uint4* __restrict__ src, uint4* dst,
                                                     const uint32_t* flags, size_t n_words,
                                                     int row_u4, unsigned long long* count,
                                                     uint32_t* have) {
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t n_warps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const int G = max(1, min(4, 32 * kPieces / row_u4));  // rows per batch
  unsigned long long rows = 0;
  for (size_t w = warp; w < n_words; w += n_warps) {
    // top-up mode (have != null): rows already present are skipped, and the
    // word's rows are present afterwards
    const uint32_t want = flags[w], had = have ? have[w] : 0u;
    uint32_t bits = want & ~had;
    rows += __popc(bits);
    while (bits) {
      uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;  // registers, not a local array
      int nr = 0;
      while (bits && nr < G) {
        const uint32_t row = (uint32_t)w * 32u + (uint32_t)(__ffs(bits) - 1);
        bits &= bits - 1;
        r0 = nr == 0 ? row : r0;
        r1 = nr == 1 ? row : r1;
        r2 = nr == 2 ? row : r2;
        r3 = nr == 3 ? row : r3;
        ++nr;
      }
      const int pieces = nr * row_u4;
      for (int base = 0; base < pieces; base += 32 * kPieces) {  // (one pass unless F > 1536)
        uint4 v[kPieces];
        uint32_t o[kPieces];  // 16-byte piece index (< 2^32: checked by the host)
#pragma unroll
        for (int i = 0; i < kPieces; ++i) {
          const int pc = base + lane + 32 * i, q = pc / row_u4;
          o[i] = (q == 0 ? r0 : q == 1 ? r1 : q == 2 ? r2 : r3) * (uint32_t)row_u4 + pc % row_u4;
          if (pc < pieces) v[i] = src[o[i]];
        }
#pragma unroll
        for (int i = 0; i < kPieces; ++i)
          if (base + lane + 32 * i < pieces) dst[o[i]] = v[i];
      }
    }
    __syncwarp();
    if (have && lane == 0 && (want & ~had)) have[w] = had | want;
  }
  if (lane == 0 && rows) atomicAdd(count, rows);
}

}  // namespace

namespace stage {

void mark_sampled(ecco_ctx* ctx, cudaStream_t st, int n_jobs, const int* d_job_ids,
                  const int* d_steps, int max_steps, const int* d_src_off, const int* d_src_cam,
                  const double* d_src_frac, const int* d_micro_base, int depth, int window,
                  uint32_t* d_flags, const uint32_t* d_have, unsigned* d_missing) {
  if (n_jobs == 0 || max_steps == 0 || depth == 0) return;
  const ecco_config& c = ctx->cfg;
  const LDims g{c.feat_dim, c.hidden_dim, c.num_classes, c.scene_dims, c.minibatch,
                c.ring_frames, c.eval_samples, c.sgd_lr, c.feature_noise};
  k_mark_sampled<<<dim3(n_jobs, max_steps, depth), std::min(c.minibatch, 256), 0, st>>>(
      g, c.seed, d_job_ids, d_steps, d_src_off, d_src_cam, d_src_frac, d_micro_base, window,
      d_flags, d_have, d_missing);
  ECCO_LAUNCHED(ctx);
}

void fetch_rows(ecco_ctx* ctx, cudaStream_t st, const uint16_t* host_dev, uint16_t* dst,
                const uint32_t* d_flags, size_t n_words, unsigned long long* d_count,
                uint32_t* d_have) {
  if (n_words == 0) return;
  ECCO_REQUIRE(n_words * 32 * (ctx->cfg.feat_dim / 8) < (1ull << 32),
               "sampled-row fetch: ring table too large for 32-bit piece offsets");
  // four CTAs (128 warps, 6 pieces in flight per lane; ECCO_FETCH_CTAS) beside whatever runs;
  // the CTA-pair evaluation kernel takes its super tiles from a counter, so
  // a pair that starts late (its TPC hosts a fetch CTA) just takes fewer
  static const int fetch_ctas = [] {
    const char* e = getenv("ECCO_FETCH_CTAS");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : 4;
  }();
  k_fetch_rows<<<fetch_ctas, 1024, 0, st>>>(reinterpret_cast<const uint4*>(host_dev),
                                   reinterpret_cast<uint4*>(dst), d_flags, n_words,
                                   ctx->cfg.feat_dim / 8, d_count, d_have);
  ECCO_LAUNCHED(ctx);
}

}  // namespace stage
