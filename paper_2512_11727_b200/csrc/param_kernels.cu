// Parametric backend kernels (sm_100a, fp64, bit-exact with the reference).
//
// K1  k_p_eval_matrix     camera x group matrix of eval()           accuracy_model.cpp:60-67
// K1' k_p_route_propose   same + group_request's masked argmax      grouping.cpp:30-39
// K2  k_p_trajectories    evaluate/train/evaluate chains per job    orchestrator.cpp:43-62
// K3  k_p_profile         build_profile_table x make_accuracy_probe transmission.cpp:52-118
//
// Work items are independent (pairs, jobs, camera-levels) so every kernel is
// a flat grid; the per-item work is a short chain of fp64 ops plus the
// table-driven exp, which runs from a shared-memory copy of the 2 KB table.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "ctx.cuh"
#include "param_model.cuh"

namespace {

__device__ const uint64_t g_exp_tab[256] = {
#include "exp_table.inc"
};

__device__ __forceinline__ void load_tab(uint64_t* s_tab) {
  for (int i = threadIdx.x + threadIdx.y * blockDim.x; i < 256; i += blockDim.x * blockDim.y)
    s_tab[i] = g_exp_tab[i];
  __syncthreads();
}

struct PDev {
  PParams p;
  int d, kmax, T;  // T = max_depth + 1 snapshot states per slot
  const int* k;
  const int* clen;
  const double* cl;
  const double* prof;
  const double* cen;
};

__device__ __forceinline__ double eval_slot(const PDev& m, int slot, const double* scene,
                                            const uint64_t* tab) {
  return p_eval(m.k[slot], m.cl + (size_t)slot * m.kmax * m.d, m.prof + (size_t)slot * m.kmax,
                m.clen[slot], m.cen + (size_t)slot * m.d, m.d, scene, m.p, tab);
}

// out[i, j] = eval(model(slot[j]), scene i); block = 32 jobs x 8 probes so a
// warp writes 32 consecutive doubles of one output row.
__global__ void __launch_bounds__(256) k_p_eval_matrix(PDev m, int n, const double* scenes,
                                                       int g, const int* slots,
                                                       const uint8_t* mask, double* out) {
  __shared__ uint64_t s_tab[256];
  load_tab(s_tab);
  const int j = blockIdx.x * 32 + threadIdx.x;
  const int i = blockIdx.y * 8 + threadIdx.y;
  if (i >= n || j >= g) return;
  const size_t o = (size_t)i * g + j;
  if (mask && !mask[o]) {
    out[o] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  double sc[ECCO_PMAX_D];
  for (int t = 0; t < m.d; ++t) sc[t] = scenes[(size_t)i * m.d + t];
  out[o] = eval_slot(m, slots[j], sc, s_tab);
}

// K1 for a compile-time scene dimension D (every fixture and BASELINE
// config has D = 2).  Block = 32 jobs x 8 probe rows; each block keeps its 32
// models and the 8-way replicated exp table in shared memory and walks probe
// rows i = blockIdx.y*8 + ty, stepping 8*gridDim.y (the table is loaded once
// per block, not once per 8 probes).  A warp writes 32 consecutive doubles of
// one output row.  Same arithmetic as k_p_eval_matrix, bit for bit (p_eval_t).
template <int D>
__global__ void __launch_bounds__(256) k_p_eval_matrix_t(PDev m, int n, const double* scenes,
                                                         int g, const int* slots,
                                                         const uint8_t* mask, double* out) {
  extern __shared__ __align__(16) uint8_t psm[];
  ulonglong2* s_rep = reinterpret_cast<ulonglong2*>(psm);      // 128 x 8 x 16 B
  const int K = m.kmax;
  const int stride = K * D + K + D;                             // doubles per model
  double* s_mod = reinterpret_cast<double*>(psm + 128 * 8 * 16);  // 32 models
  int* s_kc = reinterpret_cast<int*>(s_mod + 32 * stride);       // [32][2] k, clen
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < 128 * 8; e += 256) {
    const int i = e >> 3;
    s_rep[e] = make_ulonglong2(g_exp_tab[2 * i], g_exp_tab[2 * i + 1]);
  }
  const int j0 = blockIdx.x * 32;
  for (int e = tid; e < 32 * stride; e += 256) {
    const int jj = e / stride, q = e % stride;
    if (j0 + jj >= g) continue;
    const int slot = slots[j0 + jj];
    double v;
    if (q < K * D) v = m.cl[(size_t)slot * K * D + q];
    else if (q < K * D + K) v = m.prof[(size_t)slot * K + q - K * D];
    else v = m.cen[(size_t)slot * D + q - K * D - K];
    s_mod[e] = v;
  }
  if (tid < 32 && j0 + tid < g) {
    const int slot = slots[j0 + tid];
    s_kc[2 * tid] = m.k[slot];
    s_kc[2 * tid + 1] = m.clen[slot];
  }
  __syncthreads();
  const int j = j0 + threadIdx.x;
  if (j >= g) return;
  const double* md = s_mod + threadIdx.x * stride;
  const int k = s_kc[2 * threadIdx.x], clen = s_kc[2 * threadIdx.x + 1];
  const RepTab tab{s_rep, (uint32_t)(threadIdx.x & 7)};
  for (int i = blockIdx.y * 8 + threadIdx.y; i < n; i += 8 * gridDim.y) {
    const size_t o = (size_t)i * g + j;
    if (mask && !mask[o]) {
      out[o] = __longlong_as_double(0x7ff8000000000000LL);
      continue;
    }
    double sc[D];
#pragma unroll
    for (int t = 0; t < D; ++t) sc[t] = scenes[(size_t)i * D + t];
    out[o] = p_eval_t<D>(k, md, md + K * D, clen, md + K * D + K, sc, m.p, tab);
  }
}

// Sparse pairs: out[p] = eval(model(slot[p]), scene of probe p).
__global__ void __launch_bounds__(256) k_p_eval_pairs(PDev m, int n, const double* scenes,
                                                      const int* cams, const double* cam_scenes,
                                                      const int* slots, double* out) {
  __shared__ uint64_t s_tab[256];
  load_tab(s_tab);
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double* src = scenes ? scenes + (size_t)p * m.d : cam_scenes + (size_t)cams[p] * m.d;
  double sc[ECCO_PMAX_D];
  for (int t = 0; t < m.d; ++t) sc[t] = src[t];
  out[p] = eval_slot(m, slots[p], sc, s_tab);
}

// One warp per probe: every lane evaluates a strided subset of the jobs; the
// (acc, column) pairs are reduced with "higher acc, then lower column", which
// is exactly group_request's ascending scan with a strict '>'.
__global__ void __launch_bounds__(256) k_p_route_propose(PDev m, int n, const double* scenes,
                                                         const double* req, int g,
                                                         const int* slots, const uint8_t* mask,
                                                         int* best_col, double* best_acc) {
  __shared__ uint64_t s_tab[256];
  load_tab(s_tab);
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (i >= n) return;
  double sc[ECCO_PMAX_D];
  for (int t = 0; t < m.d; ++t) sc[t] = scenes[(size_t)i * m.d + t];
  const double r = req[i];
  int bc = -1;
  double ba = 0.0;
  for (int j = lane; j < g; j += 32) {
    if (mask && !mask[(size_t)i * g + j]) continue;
    const double a = eval_slot(m, slots[j], sc, s_tab);
    if (a < r) continue;
    if (bc < 0 || a > ba) {
      bc = j;
      ba = a;
    }
  }
  for (int off = 16; off; off >>= 1) {
    const int oc = __shfl_down_sync(0xffffffffu, bc, off);
    const double oa = __shfl_down_sync(0xffffffffu, ba, off);
    if (oc >= 0 && (bc < 0 || oa > ba || (oa == ba && oc < bc))) {
      bc = oc;
      ba = oa;
    }
  }
  if (lane == 0) {
    best_col[i] = bc;
    best_acc[i] = bc >= 0 ? ba : 0.0;
  }
}

// Mean of eval over a job's members: lanes evaluate, lane 0 sums in member
// order (orchestrator.cpp:46-49 sums sequentially, then divides).
__device__ double warp_mean_eval(int k, const double* cl, const double* prof, int clen,
                                 const double* cen, int d, const PParams& p, int nm,
                                 const int* mem, const double* cam_scenes, double* s_acc,
                                 const uint64_t* tab) {
  const int lane = threadIdx.x & 31;
  double sum = 0.0;
  for (int base = 0; base < nm; base += 32) {
    const int m = base + lane;
    if (m < nm) s_acc[lane] = p_eval(k, cl, prof, clen, cen, d, cam_scenes + (size_t)mem[m] * d, p, tab);
    __syncwarp();
    if (lane == 0) {
      const int cnt = nm - base < 32 ? nm - base : 32;
      for (int t = 0; t < cnt; ++t) sum = __dadd_rn(sum, s_acc[t]);
    }
    __syncwarp();
  }
  sum = __shfl_sync(0xffffffffu, sum, 0);
  return nm == 0 ? p.floor : __ddiv_rn(sum, (double)nm);
}

struct PTraj {
  PDev m;
  int* k;
  int* clen;
  double* cl;
  double* prof;
  double* cen;
  int* sk;
  int* sclen;
  double* scl;
  double* sprof;
  double* scen;
  const double* cam_scenes;
  const double* cam_tp;
  int* status;
};

constexpr int kWarpsPerBlock = 4;
constexpr int kModelDoubles = ECCO_PMAX_K * ECCO_PMAX_D + ECCO_PMAX_K + ECCO_PMAX_D;

__device__ void store_state(const PTraj& t, int slot, int idx, int k, int clen, const double* cl,
                            const double* prof, const double* cen) {
  const int lane = threadIdx.x & 31;
  const int d = t.m.d, K = t.m.kmax;
  const size_t st = (size_t)slot * t.m.T + idx;
  for (int q = lane; q < k * d; q += 32) t.scl[st * K * d + q] = cl[q];
  for (int q = lane; q < k; q += 32) t.sprof[st * K + q] = prof[q];
  for (int q = lane; q < d; q += 32) t.scen[st * d + q] = cen[q];
  if (lane == 0) {
    t.sk[st] = k;
    t.sclen[st] = clen;
  }
}

// One warp per job: acc[0] = evaluate; for each step train (lane 0, sources
// in map order) then evaluate.  Every intermediate model is kept as a
// snapshot for ecco_commit.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_p_trajectories(
    PTraj t, int n_jobs, const int* slots, const double* batch, const int* src_off,
    const int* src_cam, const double* src_frac, const int* mem_off, const int* mem_cam,
    double gpu_s, int depth, double* out) {
  __shared__ uint64_t s_tab[256];
  __shared__ double s_model[kWarpsPerBlock][kModelDoubles];
  __shared__ double s_acc[kWarpsPerBlock][32];
  __shared__ int s_kc[kWarpsPerBlock][4];
  __shared__ int s_best[kWarpsPerBlock][32];
  __shared__ double s_w[kWarpsPerBlock][ECCO_PMAX_K];
  load_tab(s_tab);
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int j = blockIdx.x * kWarpsPerBlock + w;
  if (j >= n_jobs) return;
  const int slot = slots[j];
  const int d = t.m.d, K = t.m.kmax;
  double* cl = s_model[w];
  double* prof = cl + ECCO_PMAX_K * ECCO_PMAX_D;
  double* cen = prof + ECCO_PMAX_K;
  int k = t.m.k[slot], clen = t.m.clen[slot];
  for (int q = lane; q < k * d; q += 32) cl[q] = t.m.cl[(size_t)slot * K * d + q];
  for (int q = lane; q < k; q += 32) prof[q] = t.m.prof[(size_t)slot * K + q];
  for (int q = lane; q < d; q += 32) cen[q] = t.m.cen[(size_t)slot * d + q];
  __syncwarp();
  store_state(t, slot, 0, k, clen, cl, prof, cen);
  const int m0 = mem_off[j], nm = mem_off[j + 1] - m0;
  const int s0 = src_off[j], ns = src_off[j + 1] - s0;
  out[(size_t)j * (depth + 1)] =
      warp_mean_eval(k, cl, prof, clen, cen, d, t.m.p, nm, mem_cam + m0, t.cam_scenes, s_acc[w], s_tab);
  const double effort = p_effort(batch[3 * j], batch[3 * j + 1], batch[3 * j + 2], gpu_s, ns,
                                 src_cam + s0, t.cam_tp);
  for (int step = 1; step <= depth; ++step) {
    // the step on the whole warp (p_train_step_warp: lookups on the lanes)
    const int rc = p_train_step_warp(&k, cl, prof, &clen, cen, K, d, effort, ns, src_cam + s0,
                                     src_frac + s0, t.cam_scenes, t.m.p, s_tab, s_best[w],
                                     s_acc[w], s_w[w], s_kc[w]);
    if (rc && lane == 0) atomicMax(t.status, rc);
    __syncwarp();
    store_state(t, slot, step, k, clen, cl, prof, cen);
    out[(size_t)j * (depth + 1) + step] = warp_mean_eval(k, cl, prof, clen, cen, d, t.m.p, nm,
                                                         mem_cam + m0, t.cam_scenes, s_acc[w], s_tab);
  }
}

__global__ void k_p_commit(PTraj t, int n_jobs, const int* slots, const int* granted) {
  const int j = blockIdx.x;
  if (j >= n_jobs) return;
  const int slot = slots[j], g = granted[j];
  if (g <= 0) return;
  const int d = t.m.d, K = t.m.kmax;
  const size_t st = (size_t)slot * t.m.T + g;
  const int k = t.sk[st];
  for (int q = threadIdx.x; q < k * d; q += blockDim.x) t.cl[(size_t)slot * K * d + q] = t.scl[st * K * d + q];
  for (int q = threadIdx.x; q < k; q += blockDim.x) t.prof[(size_t)slot * K + q] = t.sprof[st * K + q];
  for (int q = threadIdx.x; q < d; q += blockDim.x) t.cen[(size_t)slot * d + q] = t.scen[st * d + q];
  if (threadIdx.x == 0) {
    t.k[slot] = k;
    t.clen[slot] = t.sclen[st];
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_p_eval_jobs(
    PDev m, int n_jobs, const int* slots, const int* mem_off, const int* mem_cam,
    const double* cam_scenes, double* out) {
  __shared__ uint64_t s_tab[256];
  __shared__ double s_acc[kWarpsPerBlock][32];
  load_tab(s_tab);
  const int w = threadIdx.x / 32;
  const int j = blockIdx.x * kWarpsPerBlock + w;
  if (j >= n_jobs) return;
  const int slot = slots[j], d = m.d, K = m.kmax;
  const int m0 = mem_off[j], nm = mem_off[j + 1] - m0;
  const double r = warp_mean_eval(m.k[slot], m.cl + (size_t)slot * K * d, m.prof + (size_t)slot * K,
                                  m.clen[slot], m.cen + (size_t)slot * d, d, m.p, nm,
                                  mem_cam + m0, cam_scenes, s_acc[w], s_tab);
  if ((threadIdx.x & 31) == 0) out[j] = r;
}

// transmission.cpp:17-27
__device__ __forceinline__ bool preferred(double cf, double cq, double pf, double pq, int bias) {
  if (bias == 0) {
    if (cq != pq) return cq > pq;
    return cf > pf;
  }
  if (cf != pf) return cf > pf;
  return cq > pq;
}

// One thread per (camera, budget level): the whole build_profile_table row
// including every probe (seed at the floor, one train_step, eval).
__global__ void __launch_bounds__(128) k_p_profile(
    PParams p, int d, int n_cams, const int* cams, const int* bias, int n_levels,
    const double* levels, int n_grid, const double* gf, const double* gq, double window_s,
    double tie_eps, double ref_rate, double bpp_ref, const double* cam_scenes,
    const double* cam_tp, double* out_fps, double* out_res, uint8_t* out_feas) {
  __shared__ uint64_t s_tab[256];
  load_tab(s_tab);
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= n_cams * n_levels) return;
  const int ci = item / n_levels, l = item % n_levels;
  const int cam = cams[ci];
  const double* scene = cam_scenes + (size_t)cam * d;
  const double tp = cam_tp[cam];
  const double budget = levels[l];
  const double pixel_budget = __ddiv_rn(__dmul_rn(tp, budget), window_s);
  const double span = __dsub_rn(p.ceil, p.floor);
  double seed_prof = span > 0.0 ? __ddiv_rn(__dsub_rn(p.floor, p.floor), span) : 0.0;
  seed_prof = seed_prof < 0.0 ? 0.0 : (seed_prof > 1.0 ? 1.0 : seed_prof);
  // cheapest(grid), transmission.cpp:29-39
  int ch = 0;
  for (int i = 1; i < n_grid; ++i) {
    const double pr = __dmul_rn(gf[i], p_ppf(gq[i])), pb = __dmul_rn(gf[ch], p_ppf(gq[ch]));
    if (pr < pb || (pr == pb && (gq[i] < gq[ch] || (gq[i] == gq[ch] && gf[i] < gf[ch])))) ch = i;
  }
  double accs[64];
  bool found = false;
  double best = 0.0;
  const double one = 1.0;
  for (int i = 0; i < n_grid; ++i) {
    accs[i] = 0.0;
    if (__dmul_rn(gf[i], p_ppf(gq[i])) > pixel_budget) continue;
    double cl[ECCO_PMAX_D * 2], prof[2], cen[ECCO_PMAX_D];
    int k = 1, clen = d;
    for (int t = 0; t < d; ++t) cl[t] = cen[t] = scene[t];
    prof[0] = seed_prof;
    const double pixel_rate = __dmul_rn(gf[i], p_ppf(gq[i]));
    const double bpp = __ddiv_rn(ref_rate, pixel_rate);
    const double qr = __ddiv_rn(bpp, bpp_ref);
    const double quality = qr < 1.0 ? qr : 1.0;
    const double effort = p_effort(gf[i], gq[i], quality, budget, 1, &cam, cam_tp);
    // source camera index 0 of a one-entry table pointing at this camera
    p_train_step(&k, cl, prof, &clen, cen, 2, d, effort, 1, &cam, &one, cam_scenes, p, s_tab);
    accs[i] = p_eval(k, cl, prof, clen, cen, d, scene, p, s_tab);
    if (!found || accs[i] > best) best = accs[i];
    found = true;
  }
  const size_t o = (size_t)ci * n_levels + l;
  if (!found) {
    out_fps[o] = gf[ch];
    out_res[o] = gq[ch];
    out_feas[o] = 0;
    return;
  }
  bool have = false;
  double pf = 0.0, pq = 0.0;
  const int b = bias[ci];
  for (int i = 0; i < n_grid; ++i) {
    if (__dmul_rn(gf[i], p_ppf(gq[i])) > pixel_budget) continue;
    if (accs[i] < __dsub_rn(best, tie_eps)) continue;
    if (!have || preferred(gf[i], gq[i], pf, pq, b)) {
      pf = gf[i];
      pq = gq[i];
      have = true;
    }
  }
  out_fps[o] = pf;
  out_res[o] = pq;
  out_feas[o] = 1;
}

// seed_model, accuracy_model.cpp:124-134.
__global__ void k_p_seed(PTraj t, int n, const int* slots, const double* scenes,
                         const double* acc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int slot = slots[j], d = t.m.d, K = t.m.kmax;
  const PParams& p = t.m.p;
  const double span = __dsub_rn(p.ceil, p.floor);
  double pr = 0.0;
  if (span > 0.0) {
    pr = __ddiv_rn(__dsub_rn(acc[j], p.floor), span);
    pr = pr < 0.0 ? 0.0 : (pr > 1.0 ? 1.0 : pr);  // std::clamp(v, 0, 1)
  }
  for (int q = 0; q < d; ++q) {
    t.cl[(size_t)slot * K * d + q] = scenes[(size_t)j * d + q];
    t.cen[(size_t)slot * d + q] = scenes[(size_t)j * d + q];
  }
  t.prof[(size_t)slot * K] = pr;
  t.k[slot] = 1;
  t.clen[slot] = d;
}

PDev make_pdev(ecco_ctx* c) {
  PDev m;
  m.p = {c->cfg.params.learning_rate_k, c->cfg.params.similarity_lambda, c->cfg.params.acc_floor,
         c->cfg.params.acc_ceil, c->cfg.params.cluster_similarity_threshold,
         exact_reciprocal_pow2(c->cfg.params.similarity_lambda)};
  m.d = c->cfg.scene_dims;
  m.kmax = c->cfg.max_clusters;
  m.T = c->cfg.max_depth + 1;
  m.k = c->d_k;
  m.clen = c->d_clen;
  m.cl = c->d_cl;
  m.prof = c->d_prof;
  m.cen = c->d_cen;
  return m;
}

PTraj make_ptraj(ecco_ctx* c) {
  PTraj t;
  t.m = make_pdev(c);
  t.k = c->d_k;
  t.clen = c->d_clen;
  t.cl = c->d_cl;
  t.prof = c->d_prof;
  t.cen = c->d_cen;
  t.sk = c->d_sk;
  t.sclen = c->d_sclen;
  t.scl = c->d_scl;
  t.sprof = c->d_sprof;
  t.scen = c->d_scen;
  t.cam_scenes = c->d_scenes;
  t.cam_tp = c->d_tp;
  t.status = c->d_status;
  return t;
}

}  // namespace

namespace pbackend {

void eval_matrix(ecco_ctx* ctx, int n, const double* scenes, int g, const int* slots,
                 const uint8_t* mask, double* out) {
  if (n == 0 || g == 0) return;
  const PDev m = make_pdev(ctx);
  if (m.d == 2) {
    // ~8 resident blocks per SM (16 KB table + 32 models each); enough probe
    // rows per block to amortise loading them
    int sms = 0;
    ECCO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->cfg.device));
    const int gx = (g + 31) / 32;
    const int gy = std::max(1, std::min((n + 7) / 8, (sms * 8 + gx - 1) / gx));
    const size_t smem = 128 * 8 * 16 + 32 * (size_t)(m.kmax * 2 + m.kmax + 2) * 8 + 32 * 2 * 4;
    k_p_eval_matrix_t<2><<<dim3(gx, gy), dim3(32, 8), smem, ctx->stream>>>(m, n, scenes, g, slots,
                                                                            mask, out);
  } else {
    dim3 grid((g + 31) / 32, (n + 7) / 8), block(32, 8);
    k_p_eval_matrix<<<grid, block, 0, ctx->stream>>>(m, n, scenes, g, slots, mask, out);
  }
  ECCO_LAUNCHED(ctx);
}

void eval_pairs(ecco_ctx* ctx, int n, const double* scenes, const int* cams, const int* slots,
                double* out) {
  if (n == 0) return;
  k_p_eval_pairs<<<(n + 255) / 256, 256, 0, ctx->stream>>>(make_pdev(ctx), n, scenes, cams,
                                                           ctx->d_scenes, slots, out);
  ECCO_LAUNCHED(ctx);
}

void route_propose(ecco_ctx* ctx, int n, const double* scenes, const double* req, int g,
                   const int* slots, const uint8_t* mask, int* best, double* best_acc) {
  if (n == 0) return;
  k_p_route_propose<<<(n + 7) / 8, 256, 0, ctx->stream>>>(make_pdev(ctx), n, scenes, req, g,
                                                           slots, mask, best, best_acc);
  ECCO_LAUNCHED(ctx);
}

void trajectories(ecco_ctx* ctx, int n_jobs, const int* slots, const double* batch,
                  const int* src_off, const int* src_cam, const double* src_frac,
                  const int* mem_off, const int* mem_cam, double gpu_s, int depth, double* out) {
  if (n_jobs == 0) return;
  k_p_trajectories<<<(n_jobs + kWarpsPerBlock - 1) / kWarpsPerBlock, kWarpsPerBlock * 32, 0,
                     ctx->stream>>>(make_ptraj(ctx), n_jobs, slots, batch, src_off, src_cam,
                                    src_frac, mem_off, mem_cam, gpu_s, depth, out);
  ECCO_LAUNCHED(ctx);
}

void commit(ecco_ctx* ctx, int n_jobs, const int* slots, const int* granted) {
  if (n_jobs == 0) return;
  k_p_commit<<<n_jobs, 64, 0, ctx->stream>>>(make_ptraj(ctx), n_jobs, slots, granted);
  ECCO_LAUNCHED(ctx);
}

void eval_jobs(ecco_ctx* ctx, int n_jobs, const int* slots, const int* mem_off,
               const int* mem_cam, double* out) {
  if (n_jobs == 0) return;
  k_p_eval_jobs<<<(n_jobs + kWarpsPerBlock - 1) / kWarpsPerBlock, kWarpsPerBlock * 32, 0,
                  ctx->stream>>>(make_pdev(ctx), n_jobs, slots, mem_off, mem_cam, ctx->d_scenes,
                                 out);
  ECCO_LAUNCHED(ctx);
}

void profile(ecco_ctx* ctx, int n_cams, const int* cams, const int* bias, int n_levels,
             const double* levels, int n_grid, const double* gf, const double* gq,
             double window_s, double tie_eps, double ref_rate, double bpp_ref, double* fps,
             double* res, uint8_t* feas) {
  const long items = (long)n_cams * n_levels;
  if (items == 0) return;
  PDev m = make_pdev(ctx);
  k_p_profile<<<(unsigned)((items + 127) / 128), 128, 0, ctx->stream>>>(
      m.p, m.d, n_cams, cams, bias, n_levels, levels, n_grid, gf, gq, window_s, tie_eps,
      ref_rate, bpp_ref, ctx->d_scenes, ctx->d_tp, fps, res, feas);
  ECCO_LAUNCHED(ctx);
}

void seed(ecco_ctx* ctx, int n, const int* slots, const double* scenes, const double* acc) {
  if (n == 0) return;
  k_p_seed<<<(n + 127) / 128, 128, 0, ctx->stream>>>(make_ptraj(ctx), n, slots, scenes, acc);
  ECCO_LAUNCHED(ctx);
}

}  // namespace pbackend
