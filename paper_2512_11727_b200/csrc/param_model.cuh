// Device restatement of the reference's parametric accuracy model
// (proj/core/src/accuracy_model.cpp).  Compiled with -fmad=false: every
// expression keeps the reference's left-to-right evaluation order and
// rounding, and exp comes from the bit-exact glibc port in ecco_exp.cuh, so
// each function returns the same double the reference returns.
#pragma once
#include <math.h>
#include <stdint.h>

#include "ecco_exp.cuh"

#define ECCO_PMAX_D 8      // scene dimensions supported on the device
#define ECCO_PMAX_K 32     // cluster capacity supported on the device

struct PParams {
  double k, lambda, floor, ceil, thr;
  // 1/lambda when lambda is a power of two (the default 0.5): x / lambda and
  // x * (1/lambda) are then the correctly rounded value of the same exact
  // number, so the multiply is bit-identical and skips the fp64 division
  // (~20 dependent FP64 instructions per similarity); 0 = divide.
  double inv_lambda_pow2;
};

// 1/lambda if lambda is a power of two whose reciprocal is a normal double, else 0.
__host__ inline double exact_reciprocal_pow2(double lambda) {
  int e = 0;
  const double m = frexp(lambda, &e);  // lambda = m * 2^e, m in [0.5, 1)
  if (!(lambda > 0.0) || m != 0.5) return 0.0;
  const double inv = ldexp(1.0, 1 - e);
  return (inv > 2.2250738585072014e-308 && inv < 8.98846567431158e307) ? inv : 0.0;
}

// euclidean + similarity: accuracy_model.cpp:10-17, 28-34.
__device__ __forceinline__ double p_similarity(const double* a, const double* b, int d,
                                               const PParams& p, const uint64_t* tab) {
  double sq = 0.0;
  for (int i = 0; i < d; ++i) {
    const double t = __dsub_rn(a[i], b[i]);
    sq = __dadd_rn(sq, __dmul_rn(t, t));
  }
  const double ns = -__dsqrt_rn(sq);
  const double x = p.inv_lambda_pow2 != 0.0 ? __dmul_rn(ns, p.inv_lambda_pow2)
                                            : __ddiv_rn(ns, p.lambda);
  return ecco_exp_tab(x, tab);
}

// The exp table in shared memory, replicated 8 times with the (tail, sbits)
// pair of entry i of copy c at [i * 8 + c] (16 bytes): a 16-byte load is
// served 8 lanes per wavefront, and lane l reading copy l % 8 makes every
// wavefront bank-conflict-free whatever entries the lanes need (a single
// copy costs ~2.5x the wavefronts on random indices; ncu r2_k1).
struct RepTab {
  const ulonglong2* t;
  uint32_t c;
  __device__ __forceinline__ void get(uint32_t i, uint64_t& tail, uint64_t& sbits) const {
    const ulonglong2 v = t[i * 8u + c];
    tail = v.x;
    sbits = v.y;
  }
};

// similarity with a compile-time scene dimension (the scene stays in
// registers); same operation order as p_similarity.
template <int D, class Tab>
__device__ __forceinline__ double p_similarity_t(const double* a, const double* b,
                                                 const PParams& p, const Tab& tab) {
  double sq = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const double t = __dsub_rn(a[i], b[i]);
    sq = __dadd_rn(sq, __dmul_rn(t, t));
  }
  const double ns = -__dsqrt_rn(sq);
  const double x = p.inv_lambda_pow2 != 0.0 ? __dmul_rn(ns, p.inv_lambda_pow2)
                                            : __ddiv_rn(ns, p.lambda);
  return ecco_exp_with(x, tab);
}

// eval (accuracy_model.cpp:60-67) with find_cluster (:36-49) inlined, scene
// dimension D at compile time: bit-identical to p_eval.
template <int D, class Tab>
__device__ __forceinline__ double p_eval_t(int k, const double* cl, const double* prof, int clen,
                                           const double* cen, const double* scene,
                                           const PParams& p, const Tab& tab) {
  if (k == 0 || clen == 0) return p.floor;
  int best = -1;
  double best_sim = 0.0;
  for (int c = 0; c < k; ++c) {
    const double s = p_similarity_t<D>(cl + c * D, scene, p, tab);
    if (s > best_sim) {
      best_sim = s;
      best = c;
    }
  }
  const int c = (best >= 0 && best_sim >= p.thr) ? best : -1;
  const double pr = c < 0 ? 0.0 : prof[c];
  const double sim = p_similarity_t<D>(scene, cen, p, tab);
  return __dadd_rn(p.floor, __dmul_rn(__dmul_rn(__dsub_rn(p.ceil, p.floor), pr), sim));
}

// find_cluster: accuracy_model.cpp:36-49 (strict '>' from 0.0, then >= thr).
__device__ __forceinline__ int p_find_cluster(int k, const double* cl, int d, const double* scene,
                                              const PParams& p, const uint64_t* tab) {
  int best = -1;
  double best_sim = 0.0;
  for (int c = 0; c < k; ++c) {
    const double s = p_similarity(cl + c * d, scene, d, p, tab);
    if (s > best_sim) {
      best_sim = s;
      best = c;
    }
  }
  if (best >= 0 && best_sim >= p.thr) return best;
  return -1;
}

// eval: accuracy_model.cpp:60-67; floor + ((ceil - floor) * prof) * sim.
__device__ __forceinline__ double p_eval(int k, const double* cl, const double* prof, int clen,
                                         const double* cen, int d, const double* scene,
                                         const PParams& p, const uint64_t* tab) {
  if (k == 0 || clen == 0) return p.floor;
  const int c = p_find_cluster(k, cl, d, scene, p, tab);
  const double pr = c < 0 ? 0.0 : prof[c];
  const double sim = p_similarity(scene, cen, d, p, tab);
  return __dadd_rn(p.floor, __dmul_rn(__dmul_rn(__dsub_rn(p.ceil, p.floor), pr), sim));
}

// pixels_per_frame: types.cpp:11-13.
__device__ __forceinline__ double p_ppf(double q) {
  return __dmul_rn(q, __ddiv_rn(__dmul_rn(16.0, q), 9.0));
}

// effort of train_step: accuracy_model.cpp:82-86 (sources' throughputs in
// source order; mean = sequential sum / count).
__device__ __forceinline__ double p_effort(double fps, double res, double quality, double gpu_s,
                                           int n_src, const int* src_cam, const double* cam_tp) {
  const double supplied = __dmul_rn(fps, p_ppf(res));
  double required = 0.0;
  if (n_src > 0) {
    double sum = 0.0;
    for (int i = 0; i < n_src; ++i) sum = __dadd_rn(sum, cam_tp[src_cam[i]]);
    required = __ddiv_rn(sum, (double)n_src);
  }
  double suff = 1.0;
  if (required > 0.0) {
    const double r = __ddiv_rn(supplied, required);
    suff = r < 1.0 ? r : 1.0;  // std::min(1.0, r)
  }
  return __dmul_rn(__dmul_rn(gpu_s, suff), quality);
}

// p_train_step on a whole warp (same results bit for bit): the sources'
// cluster lookups against the clusters that exist at the step's start run
// on the lanes (one source each); lane 0 then walks the sources in map
// order, continuing each lookup over the clusters appended earlier in the
// step (the same ascending-c, strict-'>' sequence of comparisons as
// p_find_cluster), appending, and accumulating weights and the centroid;
// the per-cluster proficiency updates run on the lanes again.  Scratch:
// s_best / s_bsim [32], s_w [kmax] weights, s_kc [4] (k, rc, have_cen,
// touched mask; kmax <= 32).  Returns 0 or 2 (cluster capacity) on every
// lane; k / clen are updated on every lane.
__device__ __forceinline__ int p_train_step_warp(int* k, double* cl, double* prof, int* clen,
                                                 double* cen, int kmax, int d, double effort,
                                                 int n_src, const int* src_cam,
                                                 const double* src_frac, const double* cam_scenes,
                                                 const PParams& p, const uint64_t* tab, int* s_best,
                                                 double* s_bsim, double* s_w, int* s_kc) {
  if (!(effort > 0.0)) return 0;
  const int lane = threadIdx.x & 31;
  const int k0 = *k;
  for (int c = lane; c < kmax; c += 32) s_w[c] = 0.0;
  if (lane == 0) {
    s_kc[0] = k0;
    s_kc[1] = 0;  // rc
    s_kc[2] = 0;  // have_cen
    s_kc[3] = 0;  // touched clusters (bit c)
  }
  double acc_cen[ECCO_PMAX_D];
  for (int j = 0; j < d; ++j) acc_cen[j] = 0.0;
  __syncwarp();
  for (int base = 0; base < n_src; base += 32) {
    const int i = base + lane;
    int b = -1;
    double bs = 0.0;
    if (i < n_src) {
      const double* sc = cam_scenes + (size_t)src_cam[i] * d;
      for (int c = 0; c < k0; ++c) {
        const double sv = p_similarity(cl + c * d, sc, d, p, tab);
        if (sv > bs) {
          bs = sv;
          b = c;
        }
      }
    }
    s_best[lane] = b;
    s_bsim[lane] = bs;
    __syncwarp();
    if (lane == 0 && s_kc[1] == 0) {
      int kk = s_kc[0];
      const int cnt = n_src - base < 32 ? n_src - base : 32;
      for (int t = 0; t < cnt; ++t) {
        const int ii = base + t;
        const double* sc = cam_scenes + (size_t)src_cam[ii] * d;
        int bb = s_best[t];
        double bsv = s_bsim[t];
        for (int c = k0; c < kk; ++c) {  // clusters appended earlier in this step
          const double sv = p_similarity(cl + c * d, sc, d, p, tab);
          if (sv > bsv) {
            bsv = sv;
            bb = c;
          }
        }
        int c = (bb >= 0 && bsv >= p.thr) ? bb : -1;
        if (c < 0) {
          if (kk >= kmax) {
            s_kc[1] = 2;
            break;
          }
          for (int j = 0; j < d; ++j) cl[kk * d + j] = sc[j];
          prof[kk] = 0.0;
          c = kk++;
        }
        s_w[c] = __dadd_rn(s_w[c], src_frac[ii]);
        s_kc[3] = (int)((unsigned)s_kc[3] | (1u << c));
        s_kc[2] = 1;
        for (int j = 0; j < d; ++j) acc_cen[j] = __dadd_rn(acc_cen[j], __dmul_rn(src_frac[ii], sc[j]));
      }
      s_kc[0] = kk;
    }
    __syncwarp();
  }
  *k = s_kc[0];
  const int rc = s_kc[1];
  if (rc) return rc;
  for (int c = lane; c < *k; c += 32) {  // proficiencies of the touched clusters
    const double w = s_w[c];
    if (!(((unsigned)s_kc[3] >> c) & 1u) || w <= 0.0) continue;
    const double pr = prof[c];
    const double e = ecco_exp_tab(__dmul_rn(__dmul_rn(-p.k, effort), w), tab);
    prof[c] = __dsub_rn(1.0, __dmul_rn(__dsub_rn(1.0, pr), e));
  }
  if (lane == 0 && s_kc[2]) {
    for (int j = 0; j < d; ++j) cen[j] = acc_cen[j];
  }
  __syncwarp();
  if (s_kc[2]) *clen = d;
  return 0;
}

// train_step body after validation: accuracy_model.cpp:86-110.  The model
// (cl: kmax*d, prof: kmax) is updated in place.  Returns 0, or 2 when a new
// cluster would exceed kmax.
__device__ __forceinline__ int p_train_step(int* k, double* cl, double* prof, int* clen,
                                            double* cen, int kmax, int d, double effort,
                                            int n_src, const int* src_cam, const double* src_frac,
                                            const double* cam_scenes, const PParams& p,
                                            const uint64_t* tab) {
  if (!(effort > 0.0)) return 0;
  double weight[ECCO_PMAX_K];
  bool touched[ECCO_PMAX_K];
  for (int c = 0; c < kmax; ++c) {
    weight[c] = 0.0;
    touched[c] = false;
  }
  double acc_cen[ECCO_PMAX_D];
  bool have_cen = false;
  for (int i = 0; i < n_src; ++i) {
    const double* sc = cam_scenes + (size_t)src_cam[i] * d;
    int c = p_find_cluster(*k, cl, d, sc, p, tab);
    if (c < 0) {
      if (*k >= kmax) return 2;
      for (int j = 0; j < d; ++j) cl[*k * d + j] = sc[j];
      prof[*k] = 0.0;
      c = (*k)++;
    }
    weight[c] = __dadd_rn(weight[c], src_frac[i]);
    touched[c] = true;
    if (!have_cen) {
      for (int j = 0; j < d; ++j) acc_cen[j] = 0.0;
      have_cen = true;
    }
    for (int j = 0; j < d; ++j) acc_cen[j] = __dadd_rn(acc_cen[j], __dmul_rn(src_frac[i], sc[j]));
  }
  for (int c = 0; c < *k; ++c) {
    if (!touched[c] || weight[c] <= 0.0) continue;
    const double pr = prof[c];
    const double e = ecco_exp_tab(__dmul_rn(__dmul_rn(-p.k, effort), weight[c]), tab);
    prof[c] = __dsub_rn(1.0, __dmul_rn(__dsub_rn(1.0, pr), e));
  }
  if (have_cen) {
    for (int j = 0; j < d; ++j) cen[j] = acc_cen[j];
    *clen = d;
  }
  return 0;
}
