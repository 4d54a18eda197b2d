// Device helpers shared by the fused SGD chains (train_kernels.cu: the
// F <= 512 / C = 16 chain with TMEM-resident masters; wide_kernels.cu: the
// detection-head chain): DSMEM stores that complete on a remote mbarrier,
// bf16 operand rows, the branch-free expf of the owner softmax, L2
// prefetch, TMA gather4 of sampled frame rows.
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "sm100.cuh"

namespace chain {
using namespace sm100;

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
__device__ __forceinline__ void st_async_v2b32(uint32_t addr, uint32_t a, uint32_t b, uint32_t mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(addr),
      "r"(a), "r"(b), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t addr, float a, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(addr),
               "f"(a), "r"(mbar)
               : "memory");
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

// ecco_expf (learned_common.cuh) without its early-out branches: the same
// result for every argument, as straight-line code for the 16 classes.
__device__ __forceinline__ float expf_nb(float x) {
  const float xc = fminf(fmaxf(x, -87.0f), 88.0f);
  const float k = rintf(__fmul_rn(xc, 0x1.715476p+0f));
  float r = __fmaf_rn(k, -0x1.62e400p-1f, xc);
  r = __fmaf_rn(k, -0x1.7f7d1cp-20f, r);
  float q = 0x1.6c16c2p-10f;
  q = __fmaf_rn(q, r, 0x1.111112p-7f);
  q = __fmaf_rn(q, r, 0x1.555556p-5f);
  q = __fmaf_rn(q, r, 0x1.555556p-3f);
  q = __fmaf_rn(q, r, 0.5f);
  q = __fmaf_rn(q, r, 1.0f);
  q = __fmaf_rn(q, r, 1.0f);
  const float e = __fmul_rn(q, __uint_as_float((uint32_t)((int)k + 127) << 23));
  return x < -87.0f ? 0.0f : e;
}

__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
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

// TMA gather4 (sm_100a): four rows `r0..r3` of the 2-D frame table, columns
// [c0, c0 + 64), into four consecutive 128-byte rows of a 128B-swizzled tile.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int c0, int r0,
                                            int r1, int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// Bulk copy of `bytes` (16-byte multiple) from this CTA's shared memory to
// the shared memory of a CTA of the cluster (shared::cluster address),
// completing on that CTA's mbarrier; commit / wait until the source may be
// overwritten.
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src, uint32_t bytes,
                                         uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(src), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

}  // namespace chain
