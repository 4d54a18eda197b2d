// Bit-exact device port of the exp() the reference links against.
//
// The reference computes every similarity and every proficiency update with
// std::exp (reference proj/core/src/accuracy_model.cpp:33 and :107), which on
// the x86-64 hosts of this image resolves (glibc 2.39 ifunc) to the FMA build
// of glibc's table-driven exp: 128-entry 2^(k/128) table, degree-5 polynomial,
// and a fixed set of fused multiply-adds chosen by the compiler.  CUDA's own
// exp() is a different algorithm and disagrees in the last ulp on a fraction of
// inputs, which is enough to flip a strict '>' in find_cluster or the
// allocator.  This header restates the algorithm with the same FMA placement
// (derived from the ifunc's disassembly) so device
// results equal the reference's host results bit for bit.  Every operation is
// written with an explicit rounding intrinsic so the result does not depend on
// -fmad; the file is also compiled for the host to run the 1e8-sample
// equivalence test against libm (tests/test_exp_parity.py).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define ECCO_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define ECCO_HD static inline
#endif

namespace ecco_exp_detail {

#ifdef __CUDA_ARCH__
__device__ __forceinline__ double as_d(uint64_t u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ uint64_t as_u(double d) { return (uint64_t)__double_as_longlong(d); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fmad(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
static inline double as_d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static inline uint64_t as_u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
// volatile-free: the host build uses -ffp-contract=off so these stay unfused.
static inline double mul(double a, double b) { return a * b; }
static inline double add(double a, double b) { return a + b; }
static inline double sub(double a, double b) { return a - b; }
static inline double fmad(double a, double b, double c) { return fma(a, b, c); }
#endif

// glibc __exp_data constants (bit patterns).
#define ECCO_EXP_INVLN2N 0x40671547652b82feULL  /* 0x1.71547652b82fep7 = 128/ln2 */
#define ECCO_EXP_SHIFT 0x4338000000000000ULL    /* 0x1.8p52 */
#define ECCO_EXP_NEGLN2HIN 0xbf762e42fefa0000ULL
#define ECCO_EXP_NEGLN2LON 0xbd0cf79abc9e3b3aULL
#define ECCO_EXP_C2 0x3fdffffffffffdbdULL
#define ECCO_EXP_C3 0x3fc555555555543cULL
#define ECCO_EXP_C4 0x3fa55555cf172b91ULL
#define ECCO_EXP_C5 0x3f81111167a4d017ULL

// Scaling of results whose exponent leaves the normal range (k near +-1022).
ECCO_HD double specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    sbits -= 1009ULL << 52;
    double scale = as_d(sbits);
    double y = fmad(scale, tmp, scale);
    return mul(y, as_d(0x7f00000000000000ULL));  // 0x1p1009
  }
  sbits += 1022ULL << 52;
  double scale = as_d(sbits);
  double st = mul(scale, tmp);
  double y = add(scale, st);  // unfused in the FMA build as well
  if (y < 1.0) {
    double lo = add(sub(scale, y), st);
    double hi = add(y, 1.0);
    double t = add(add(sub(1.0, hi), y), lo);
    y = sub(add(t, hi), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return mul(y, as_d(0x0010000000000000ULL));  // 0x1p-1022
}

}  // namespace ecco_exp_detail

// exp(x) bit-identical to glibc 2.39's x86-64 FMA variant, with the table
// behind an accessor: tab.tail(i) / tab.sbits(i) are entries 2i / 2i+1 of the
// 256-entry table of exp_table.inc (i = ki & 127), wherever they live.
template <class Tab>
ECCO_HD double ecco_exp_with(double x, const Tab& tab) {
  using namespace ecco_exp_detail;
  uint64_t ix = as_u(x);
  uint32_t abstop = (uint32_t)((ix >> 52) & 0x7ff);
  bool special = false;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return add(x, 1.0);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                   // |x| >= 1024
      if (ix == 0xfff0000000000000ULL) return 0.0;            // -inf
      if (abstop >= 0x7ffu) return add(x, 1.0);               // inf or nan
      return (ix >> 63) ? 0.0 : as_d(0x7ff0000000000000ULL);  // under/overflow
    }
    special = true;  // large |x| that may still be representable
  }
  double kd = fmad(x, as_d(ECCO_EXP_INVLN2N), as_d(ECCO_EXP_SHIFT));
  uint64_t ki = as_u(kd);
  kd = sub(kd, as_d(ECCO_EXP_SHIFT));
  double r = fmad(kd, as_d(ECCO_EXP_NEGLN2HIN), x);
  r = fmad(kd, as_d(ECCO_EXP_NEGLN2LON), r);
  const uint32_t i = (uint32_t)(ki & 127u);
  uint64_t tail_bits, sbits0;
  tab.get(i, tail_bits, sbits0);
  uint64_t top = ki << 45;
  double tail = as_d(tail_bits);
  uint64_t sbits = sbits0 + top;
  double p23 = fmad(r, as_d(ECCO_EXP_C3), as_d(ECCO_EXP_C2));
  double rt = add(r, tail);
  double r2 = mul(r, r);
  double p45 = fmad(r, as_d(ECCO_EXP_C5), as_d(ECCO_EXP_C4));
  double tmp = fmad(p23, r2, rt);
  double r4 = mul(r2, r2);
  tmp = fmad(r4, p45, tmp);
  if (special) return specialcase(tmp, sbits, ki);
  double scale = as_d(sbits);
  return fmad(scale, tmp, scale);
}

// exp(x) bit-identical to glibc 2.39's x86-64 FMA variant. `tab` is the 256-entry
// table from exp_table.inc (global, constant or shared memory).
ECCO_HD double ecco_exp_tab(double x, const uint64_t* tab) {
  using namespace ecco_exp_detail;
  uint64_t ix = as_u(x);
  uint32_t abstop = (uint32_t)((ix >> 52) & 0x7ff);
  bool special = false;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return add(x, 1.0);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                   // |x| >= 1024
      if (ix == 0xfff0000000000000ULL) return 0.0;            // -inf
      if (abstop >= 0x7ffu) return add(x, 1.0);               // inf or nan
      return (ix >> 63) ? 0.0 : as_d(0x7ff0000000000000ULL);  // under/overflow
    }
    special = true;  // large |x| that may still be representable
  }
  double kd = fmad(x, as_d(ECCO_EXP_INVLN2N), as_d(ECCO_EXP_SHIFT));
  uint64_t ki = as_u(kd);
  kd = sub(kd, as_d(ECCO_EXP_SHIFT));
  double r = fmad(kd, as_d(ECCO_EXP_NEGLN2HIN), x);
  r = fmad(kd, as_d(ECCO_EXP_NEGLN2LON), r);
  uint32_t idx = 2u * (uint32_t)(ki & 127u);
  uint64_t top = ki << 45;
  double tail = as_d(tab[idx]);
  uint64_t sbits = tab[idx + 1] + top;
  double p23 = fmad(r, as_d(ECCO_EXP_C3), as_d(ECCO_EXP_C2));
  double rt = add(r, tail);
  double r2 = mul(r, r);
  double p45 = fmad(r, as_d(ECCO_EXP_C5), as_d(ECCO_EXP_C4));
  double tmp = fmad(p23, r2, rt);
  double r4 = mul(r2, r2);
  tmp = fmad(r4, p45, tmp);
  if (special) return specialcase(tmp, sbits, ki);
  double scale = as_d(sbits);
  return fmad(scale, tmp, scale);
}
