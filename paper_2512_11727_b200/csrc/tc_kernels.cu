// Tensor-core path of the learned backend (ECCO_MATH_TC_BF16): the two dense
// contractions of every SGD step and of the evaluation matrix run on the 5th
// generation tensor cores (tcgen05.mma kind::tf32, fp32 accumulators in TMEM).
//
//   fwd   Z[rows, H]  = X[rows, F] . W1[F, H] + b1      (K = F)
//   dW1   W1[F, H]   -= lr * X[B, F]^T . dH[B, H]       (K = B samples)
//
// One CTA owns a 128 x N_tile output tile (N_tile in {64, 128, 256}).  Four
// warps stream 32-wide K chunks of both operands from HBM/L2 into shared
// memory in the canonical no-swizzle UMMA layouts (X rows are a gather over
// the sampled frames, so the loads are per-thread 16-byte vectors rather than
// TMA boxes), double-buffered against the asynchronous MMAs; one thread issues
// tcgen05.mma and commits to an mbarrier per stage; the epilogue drains TMEM
// with tcgen05.ld (32 lanes x 32 columns per warp instruction) and fuses the
// bias add (fwd) or the SGD update (dW1).
//
// Shared-memory layout (fp32 elements, "core matrix" = 8 rows x 16 bytes):
// kind::tf32 takes both operands K-major, so every operand tile -- X rows,
// W1 columns, X^T and dH^T -- is staged K-major through registers:
//   off(r,k) = (r/8)*1024 + (k/4)*128 + (r%8)*16 + (k%4)*4
//   LBO = 128 (next 4 k), SBO = 1024 (next 8 rows); one K=8 MMA step = +256 B.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "sm100.cuh"
#include "tc_kernels.cuh"

namespace {

constexpr int kM = 128;   // UMMA M (rows of a tile)
constexpr int kKC = 32;   // K elements per pipeline chunk (4 MMAs of K = 8)
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, majors, N, M.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int a_mn_major, int b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn_major << 15) |
         ((uint32_t)b_mn_major << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// 32 lanes x 32 columns: thread t of warp w gets TMEM lane 32w+t, columns c..c+31.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Stores v = (element (r..r+3, k)) into a K-major tile: 4 rows, one column.
__device__ __forceinline__ void kmajor_put4(float* tile, int r, int k, float4 v) {
  uint8_t* base = (uint8_t*)tile + (k >> 2) * 128 + (k & 3) * 4;
  const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ri = r + i;
    *reinterpret_cast<float*>(base + (ri >> 3) * 1024 + (ri & 7) * 16) = e[i];
  }
}

// Element e of a K-major staging pass (kKC = 32 K indices x groups of 4
// MN rows) -> (K index, MN group): within a warp the lanes cover 4
// consecutive K x 8 consecutive groups (lane bits 0-1: K, 2-4: group), so
// every scalar store of kmajor_put4 hits 8 banks (4-way) instead of 2
// (16-way), and the global loads stay contiguous 64- / 128-byte runs.
__device__ __forceinline__ int stage_k(int e) { return 4 * ((e >> 5) & 7) + (e & 3); }
__device__ __forceinline__ int stage_g(int e) {
  return 8 * (e >> 8) + 2 * ((e >> 3) & 3) + ((e >> 2) & 1);
}

__device__ __forceinline__ float4 bf16x4_to_f32(uint2 p) {
  return make_float4(__uint_as_float(p.x << 16), __uint_as_float(p.x & 0xFFFF0000u),
                     __uint_as_float(p.y << 16), __uint_as_float(p.y & 0xFFFF0000u));
}

// --------------------------------------------------------------------------
// fwd: one CTA per (row tile, N tile).  A = X rows (gathered bf16 -> fp32),
// B = W1 columns n0..n0+NT; both K-major.
struct FwdArgs {
  const uint16_t* xbase;
  const int64_t* row_off;  // element offset of each row's features
  const TcTile* tiles;     // per row tile: slot, first row, valid rows, job
  const int* steps;        // nullable gate: tile live iff step < steps[job]
  int step;
  const float* wbase;
  size_t wstride;
  float* Z;
  int F, H, NT;
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) k_tc_fwd(FwdArgs a) {
  const TcTile tile = a.tiles[blockIdx.x];
  if (a.steps && a.step >= a.steps[tile.job]) return;
  const int n0 = blockIdx.y * NT;
  extern __shared__ __align__(1024) uint8_t smem[];
  float* sA[2] = {(float*)smem, (float*)(smem + 16384)};
  float* sB[2] = {(float*)(smem + 32768), (float*)(smem + 32768 + NT * kKC * 4)};
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base;
  __shared__ int64_t rows[kM];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid < kM) rows[tid] = tid < tile.nrows ? a.row_off[tile.row0 + tid] : -1;
  if (warp == 0) tmem_alloc(&tmem_base, (uint32_t)NT);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const float* W1 = a.wbase + (size_t)tile.slot * a.wstride;
  const int nk = a.F / kKC;
  const uint32_t idesc = idesc_tf32(kM, NT, 0, 0);
  // per thread and chunk: kA groups of 4 X features, kB 16-byte W1 vectors;
  // the next chunk's loads are in flight while this chunk's MMAs run
  constexpr int kA = kM * (kKC / 4) / kThreads, kBv = kKC * (NT / 4) / kThreads;
  uint2 ra[kA];
  float4 rb[kBv];
  auto load = [&](int kc) {
    const int k0 = kc * kKC;
#pragma unroll
    for (int u = 0; u < kA; ++u) {
      const int e = tid + u * kThreads, r = e >> 3, c = e & 7;
      ra[u] = rows[r] >= 0 ? *reinterpret_cast<const uint2*>(a.xbase + rows[r] + k0 + c * 4)
                           : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kBv; ++u) {
      const int e = tid + u * kThreads, k = stage_k(e), n4 = stage_g(e);
      rb[u] = *reinterpret_cast<const float4*>(W1 + (size_t)(k0 + k) * a.H + n0 + n4 * 4);
    }
  };
  load(0);
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    if (kc >= 2) mbar_wait(&bar[s], ((kc - 2) >> 1) & 1);
#pragma unroll
    for (int u = 0; u < kA; ++u) {
      const int e = tid + u * kThreads, r = e >> 3, c = e & 7;
      *reinterpret_cast<float4*>((uint8_t*)sA[s] + (r >> 3) * 1024 + c * 128 + (r & 7) * 16) =
          bf16x4_to_f32(ra[u]);
    }
#pragma unroll
    for (int u = 0; u < kBv; ++u) {
      const int e = tid + u * kThreads;
      kmajor_put4(sB[s], stage_g(e) * 4, stage_k(e), rb[u]);
    }
    if (kc + 1 < nk) load(kc + 1);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aaddr = smem_u32(sA[s]), baddr = smem_u32(sB[s]);
#pragma unroll
      for (int kk = 0; kk < kKC / 8; ++kk) {
        const uint64_t da = smem_desc(aaddr + kk * 256, 128, 1024);
        const uint64_t db = smem_desc(baddr + kk * 256, 128, 1024);
        mma_tf32(tmem, da, db, idesc, (kc | kk) ? 1u : 0u);
      }
      mma_commit(&bar[s]);
    }
  }
  mbar_wait(&bar[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
  tc_fence_after();
  // epilogue: row = 32*warp + lane; z = acc + b1
  const int r = warp * 32 + (tid & 31);
  const float* b1 = W1 + (size_t)a.F * a.H;
  for (int c0 = 0; c0 < NT; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    if (r < tile.nrows) {
      float* zr = a.Z + (size_t)(tile.row0 + r) * a.H + n0 + c0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 o;
        o.x = v[i] + b1[n0 + c0 + i];
        o.y = v[i + 1] + b1[n0 + c0 + i + 1];
        o.z = v[i + 2] + b1[n0 + c0 + i + 2];
        o.w = v[i + 3] + b1[n0 + c0 + i + 3];
        *reinterpret_cast<float4*>(zr + i) = o;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, (uint32_t)NT);
}

// --------------------------------------------------------------------------
// dW1: one CTA per (job, F tile of 128, H tile of NT).  A = X^T (element
// (f, s) = x[s][f]), B = dH^T (element (h, s)), both K-major; K = B rows.
struct Dw1Args {
  const uint16_t* xbase;
  const int64_t* row_off;  // rows of job j: [j*B, (j+1)*B)
  const int* slots;
  const int* steps;
  int step;
  float* wbase;
  size_t wstride;
  const float* DH;
  int F, H, B, NT;
  float lr;
  uint16_t* w1t;  // nullable: bf16 W1^T shadow [slot][H][F]
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) k_tc_dw1(Dw1Args a) {
  const int j = blockIdx.z;
  if (a.step >= a.steps[j]) return;
  const int f0 = blockIdx.x * kM, n0 = blockIdx.y * NT;
  extern __shared__ __align__(1024) uint8_t smem[];
  float* sA[2] = {(float*)smem, (float*)(smem + 16384)};
  float* sB[2] = {(float*)(smem + 32768), (float*)(smem + 32768 + NT * kKC * 4)};
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc(&tmem_base, (uint32_t)NT);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const size_t r0 = (size_t)j * a.B;
  const int nk = a.B / kKC;
  const uint32_t idesc = idesc_tf32(kM, NT, 0, 0);
  {  // the W1 tile the epilogue read-modify-writes -> L2 while the MMAs run
    const float* wt = a.wbase + (size_t)a.slots[j] * a.wstride + (size_t)f0 * a.H + n0;
    constexpr int kLines = kM * NT / 32;  // 128-byte lines of the tile
    for (int li = tid; li < kLines; li += kThreads)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(wt + (size_t)(li / (NT / 32)) * a.H +
                                                     (li % (NT / 32)) * 32));
  }
  constexpr int kA = kKC * (kM / 4) / kThreads, kBv = kKC * (NT / 4) / kThreads;
  uint2 ra[kA];
  float4 rb[kBv];
  auto load = [&](int kc) {
    const int k0 = kc * kKC;
#pragma unroll
    for (int u = 0; u < kA; ++u) {
      const int e = tid + u * kThreads, k = stage_k(e), m4 = stage_g(e);
      ra[u] = *reinterpret_cast<const uint2*>(a.xbase + a.row_off[r0 + k0 + k] + f0 + m4 * 4);
    }
#pragma unroll
    for (int u = 0; u < kBv; ++u) {
      const int e = tid + u * kThreads, k = stage_k(e), n4 = stage_g(e);
      rb[u] = *reinterpret_cast<const float4*>(a.DH + (r0 + k0 + k) * a.H + n0 + n4 * 4);
    }
  };
  load(0);
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    if (kc >= 2) mbar_wait(&bar[s], ((kc - 2) >> 1) & 1);
    // A = X^T (element (f, s)), B = dH^T (element (h, s)), both K-major
#pragma unroll
    for (int u = 0; u < kA; ++u) {
      const int e = tid + u * kThreads;
      kmajor_put4(sA[s], stage_g(e) * 4, stage_k(e), bf16x4_to_f32(ra[u]));
    }
#pragma unroll
    for (int u = 0; u < kBv; ++u) {
      const int e = tid + u * kThreads;
      kmajor_put4(sB[s], stage_g(e) * 4, stage_k(e), rb[u]);
    }
    if (kc + 1 < nk) load(kc + 1);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aaddr = smem_u32(sA[s]), baddr = smem_u32(sB[s]);
#pragma unroll
      for (int kk = 0; kk < kKC / 8; ++kk) {
        const uint64_t da = smem_desc(aaddr + kk * 256, 128, 1024);
        const uint64_t db = smem_desc(baddr + kk * 256, 128, 1024);
        mma_tf32(tmem, da, db, idesc, (kc | kk) ? 1u : 0u);
      }
      mma_commit(&bar[s]);
    }
  }
  mbar_wait(&bar[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
  tc_fence_after();
  // epilogue: each warp's 32 feature rows x 32 gradient columns go through a
  // shared-memory transpose so the W1 read-modify-write runs along rows
  // (128-byte coalesced) instead of one 16-byte piece per feature row
  float* W1 = a.wbase + (size_t)a.slots[j] * a.wstride;
  const int lane = tid & 31;
  float* tr = reinterpret_cast<float*>(smem) + warp * 32 * 33;  // operand stages are free
  // 16-byte accesses: lane = (row group rr = lane / 8, column quad cq =
  // lane % 8) covers 4 rows x 32 columns per instruction; the shadow lane =
  // (column group, feature quad) writes 8 bytes; tr reads conflict-free
  const int rr = lane >> 3, cq = lane & 7;
  for (int c0 = 0; c0 < NT; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) tr[i * 33 + lane] = v[i];  // tr[col][row]
    __syncwarp();
    float* wrow = W1 + (size_t)(f0 + warp * 32 + rr) * a.H + n0 + c0 + 4 * cq;
    float4 wv[8];
#pragma unroll
    for (int it = 0; it < 8; ++it)  // rows 4 * it + rr: 8 x 16 bytes in flight
      wv[it] = *reinterpret_cast<const float4*>(wrow + (size_t)(4 * it) * a.H);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int r = 4 * it + rr;
      float* t = tr + (4 * cq) * 33 + r;
      const float4 nw = make_float4(fmaf(-a.lr, t[0], wv[it].x), fmaf(-a.lr, t[33], wv[it].y),
                                    fmaf(-a.lr, t[66], wv[it].z), fmaf(-a.lr, t[99], wv[it].w));
      *reinterpret_cast<float4*>(wrow + (size_t)(4 * it) * a.H) = nw;
      t[0] = nw.x;  // (col, row) -> the updated value, for the shadow below
      t[33] = nw.y;
      t[66] = nw.z;
      t[99] = nw.w;
    }
    __syncwarp();
    if (a.w1t) {  // shadow [h][f]: lane = (h group, 4 consecutive features), 8-byte stores
      uint16_t* sh = a.w1t + (size_t)a.slots[j] * a.H * a.F + (size_t)(n0 + c0 + rr) * a.F + f0 +
                     warp * 32 + 4 * cq;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const float* t = tr + (4 * it + rr) * 33 + 4 * cq;
        *reinterpret_cast<uint2*>(sh + (size_t)(4 * it) * a.F) =
            make_uint2(sm100::pack_bf16x2(t[0], t[1]), sm100::pack_bf16x2(t[2], t[3]));
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, (uint32_t)NT);
}

// --------------------------------------------------------------------------
// fwd, bf16: one CTA per (128-row training tile, 256 hidden columns).  A = X
// rows gathered by cp.async into a 128B-swizzled K-major stage (bf16, exact),
// B = the bf16 W1^T shadow by TMA ({64, 256} boxes), kind::f16 MMAs (M 128,
// N 256, K 16) into TMEM, 2 stages of K = 64 (two CTAs per SM hide the
// gather latency better than four stages in one).
constexpr int kBfNT = 256;
constexpr uint32_t kBfA = 128 * 128, kBfB = kBfNT * 128;  // bytes per stage

struct FwdBfArgs {
  const uint16_t* xbase;
  const int64_t* row_off;
  const TcTile* tiles;
  const int* steps;
  int step;
  const float* wbase;  // b1 at + F*H
  size_t wstride;
  float* Z;
  int F, H;
};

// STG pipeline stages: 2 (96 KB, two CTAs per SM) for full grids, 4 (192 KB)
// when the grid is small (a single group's chain: the K loop is latency bound)
template <int STG>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_fwd_bf16(const __grid_constant__ CUtensorMap map_w, FwdBfArgs a) {
  const TcTile tile = a.tiles[blockIdx.x];
  if (a.steps && a.step >= a.steps[tile.job]) return;
  const int n0 = blockIdx.y * kBfNT;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STG * kBfA;
  __shared__ uint64_t full[STG], empty[STG], done;
  __shared__ uint32_t tmem_base;
  __shared__ int64_t rows[kM];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  rows[tid] = tile.nrows > tid ? a.row_off[tile.row0 + tid] : a.row_off[tile.row0];
  if (warp == 0) tmem_alloc(&tmem_base, (uint32_t)kBfNT);
  if (tid == 0) {
    if (sm100::smem_u32(smem) & 1023u) __trap();
    for (int s = 0; s < STG; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int nk = a.F / 64;
  const int brow = tile.slot * a.H + n0;  // first W1^T row of this CTA
  // A gather: thread tid owns row tid, its 8 16-byte pieces of the chunk
  auto load = [&](int kc) {
    const int s = kc % STG;
    const uint32_t dst = sm100::smem_u32(sA + s * kBfA) + tid * 128;
    const uint16_t* src = a.xbase + rows[tid] + kc * 64;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + ((c ^ (tid & 7)) << 4)),
                   "l"(src + c * 8)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (tid == 0) {
      sm100::mbar_expect_tx(&full[s], kBfB);
      sm100::tma_load_2d(sB + s * kBfB, &map_w, kc * 64, brow, &full[s]);
    }
  };
  for (int kc = 0; kc < STG - 1 && kc < nk; ++kc) load(kc);
  const uint32_t idf = sm100::idesc(kM, kBfNT, sm100::kFmtBF16);
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % STG;
    const int nx = kc + STG - 1;
    if (nx < nk) {
      if (nx >= STG) mbar_wait(&empty[nx % STG], ((nx / STG) - 1) & 1);
      load(nx);
      asm volatile("cp.async.wait_group %0;" ::"n"(STG - 1) : "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      mbar_wait(&full[s], (kc / STG) & 1);
      tc_fence_after();
      const uint64_t da = sm100::desc_kmajor_sw128(sm100::smem_u32(sA + s * kBfA));
      const uint64_t db = sm100::desc_kmajor_sw128(sm100::smem_u32(sB + s * kBfB));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        sm100::mma_bf16_ss(tmem, da + kk * 2, db + kk * 2, idf, (kc | kk) != 0);
      sm100::mma_commit(&empty[s]);
      if (kc == nk - 1) sm100::mma_commit(&done);
    }
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  const int r = warp * 32 + lane;
  const float* b1 = a.wbase + (size_t)tile.slot * a.wstride + (size_t)a.F * a.H;
  for (int c0 = 0; c0 < kBfNT; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    if (r < tile.nrows) {
      float* zr = a.Z + (size_t)(tile.row0 + r) * a.H + n0 + c0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 o;
        o.x = v[i] + b1[n0 + c0 + i];
        o.y = v[i + 1] + b1[n0 + c0 + i + 1];
        o.z = v[i + 2] + b1[n0 + c0 + i + 2];
        o.w = v[i + 3] + b1[n0 + c0 + i + 3];
        *reinterpret_cast<float4*>(zr + i) = o;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, (uint32_t)kBfNT);
}

int pick_nt(int H, int ctas_per_nt1) {
  // widest tile that still gives >= 148 CTAs, never below 64
  int nt = std::min(H, 256);
  while (nt > 64 && (long)ctas_per_nt1 * (H / nt) < 148) nt /= 2;
  while (H % nt) nt /= 2;
  return nt;
}

size_t smem_bytes(int NT) { return 32768 + 2 * (size_t)NT * kKC * 4; }

void set_smem_attrs(int device) {  // per device: the attribute applies to the current device
  static DeviceFlags done;
  if (done.done(device)) return;
  const int mx = (int)smem_bytes(256);
  ECCO_CUDA(cudaFuncSetAttribute(k_tc_fwd<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  ECCO_CUDA(cudaFuncSetAttribute(k_tc_fwd<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  ECCO_CUDA(cudaFuncSetAttribute(k_tc_fwd<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  ECCO_CUDA(cudaFuncSetAttribute(k_tc_dw1<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  ECCO_CUDA(cudaFuncSetAttribute(k_tc_dw1<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  ECCO_CUDA(cudaFuncSetAttribute(k_tc_dw1<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  done.mark(device);
}

}  // namespace

namespace tc {

void fwd_hidden(ecco_ctx* ctx, const uint16_t* xbase, const int64_t* row_off, const TcTile* tiles,
                int n_tiles, const int* steps, int step, const float* wbase, size_t wstride,
                float* Z, double live_rows) {
  if (n_tiles == 0) return;
  const int F = ctx->cfg.feat_dim, H = ctx->cfg.hidden_dim;
  const int NT = pick_nt(H, n_tiles);
  FwdArgs a{xbase, row_off, tiles, steps, step, wbase, wstride, Z, F, H, NT};
  const size_t sm = smem_bytes(NT);
  set_smem_attrs(ctx->cfg.device);
  const int kind = steps ? ECCO_KSTAT_TRAIN_STEP : ECCO_KSTAT_EVAL_MATRIX;
  const dim3 grid(n_tiles, H / NT);
  ECCO_TIMED(ctx, kind, 2.0 * live_rows * F * H, live_rows * F * 2.0 + (double)F * H * 4,
             (NT == 256   ? k_tc_fwd<256><<<grid, kThreads, sm, ctx->stream>>>(a)
              : NT == 128 ? k_tc_fwd<128><<<grid, kThreads, sm, ctx->stream>>>(a)
                          : k_tc_fwd<64><<<grid, kThreads, sm, ctx->stream>>>(a)));
  ECCO_LAUNCHED(ctx);
}

void fwd_hidden_bf16(ecco_ctx* ctx, const uint16_t* xbase, const int64_t* row_off,
                     const TcTile* tiles, int n_tiles, const int* steps, int step,
                     const uint16_t* w1t, size_t n_slots, const float* wbase, size_t wstride,
                     float* Z, double live_rows) {
  if (n_tiles == 0) return;
  const int F = ctx->cfg.feat_dim, H = ctx->cfg.hidden_dim;
  ECCO_REQUIRE(H % kBfNT == 0 && F % 64 == 0, "bf16 forward: H % 256 and F % 64");
  const CUtensorMap map = fused::tensor_map_bf16(w1t, n_slots * H, F, kBfNT);
  FwdBfArgs a{xbase, row_off, tiles, steps, step, wbase, wstride, Z, F, H};
  static DeviceFlags attr;  // per device
  if (!attr.done(ctx->cfg.device)) {
    ECCO_CUDA(cudaFuncSetAttribute(k_tc_fwd_bf16<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(2 * (size_t)(kBfA + kBfB))));
    ECCO_CUDA(cudaFuncSetAttribute(k_tc_fwd_bf16<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(4 * (size_t)(kBfA + kBfB))));
    attr.mark(ctx->cfg.device);
  }
  int sms = 0;
  ECCO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->cfg.device));
  const bool deep = (long)n_tiles * (H / kBfNT) * 2 <= sms;  // room for one CTA per SM
  const int kind = steps ? ECCO_KSTAT_TRAIN_STEP : ECCO_KSTAT_EVAL_MATRIX;
  const dim3 grid(n_tiles, H / kBfNT);
  ECCO_TIMED(ctx, kind, 2.0 * live_rows * F * H, live_rows * F * 2.0 + (double)F * H * 2,
             (deep ? k_tc_fwd_bf16<4><<<grid, kThreads, 4 * (size_t)(kBfA + kBfB), ctx->stream>>>(map, a)
                   : k_tc_fwd_bf16<2><<<grid, kThreads, 2 * (size_t)(kBfA + kBfB), ctx->stream>>>(map, a)));
  ECCO_LAUNCHED(ctx);
}

void dw1_update(ecco_ctx* ctx, const uint16_t* xbase, const int64_t* row_off, const int* slots,
                const int* steps, int step, int n_jobs, float* wbase, size_t wstride,
                const float* DH, int live_jobs, uint16_t* w1t) {
  if (n_jobs == 0) return;
  const int F = ctx->cfg.feat_dim, H = ctx->cfg.hidden_dim, B = ctx->cfg.minibatch;
  const int NT = pick_nt(H, n_jobs * (F / kM));
  Dw1Args a{xbase, row_off, slots, steps, step, wbase, wstride, DH, F, H, B, NT, ctx->cfg.sgd_lr, w1t};
  const size_t sm = smem_bytes(NT);
  set_smem_attrs(ctx->cfg.device);
  ECCO_TIMED(ctx, ECCO_KSTAT_TRAIN_DW1, 2.0 * live_jobs * F * H * B,
             (double)live_jobs * (B * F * 2.0 + B * H * 4.0 + 2.0 * F * H * 4),
             (NT == 256   ? k_tc_dw1<256><<<dim3(F / kM, H / NT, n_jobs), kThreads, sm, ctx->stream>>>(a)
              : NT == 128 ? k_tc_dw1<128><<<dim3(F / kM, H / NT, n_jobs), kThreads, sm, ctx->stream>>>(a)
                          : k_tc_dw1<64><<<dim3(F / kM, H / NT, n_jobs), kThreads, sm, ctx->stream>>>(a)));
  ECCO_LAUNCHED(ctx);
}

}  // namespace tc
