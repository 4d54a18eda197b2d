/*
 * ecco_oracle.c -- TEST INFRASTRUCTURE: CPU restatement used as the checker.
 *
 * Parametric part: a line-by-line restatement of the reference arithmetic
 * (/root/reference/proj/core/src/accuracy_model.cpp, transmission.cpp,
 * orchestrator.cpp), pinned against the reference's own known-answer tests
 * and against oracle/_ref/libecco_ref.so (tests/test_oracle_pinning.py).
 * Uses libm exp/sqrt exactly like the reference.  Compiled -ffp-contract=off.
 *
 * Learned part: the specification of backend L (synthetic camera streams,
 * frame sampler, MLP forward/backward/SGD, eval counts).  The reference has
 * no counterpart, so parity for it is pinned to this file only ("parity
 * unpinned by the reference").  Every reduction is sequential in
 * the order written here; the CUDA FFMA path reproduces it bit for bit.
 */
#include "ecco_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================= parametric backend ======================= */

/* euclidean + similarity, accuracy_model.cpp:10-17, 28-34 (sequential sum). */
double orc_similarity(const double* a, const double* b, int d, double lambda) {
  double sq = 0.0;
  for (int i = 0; i < d; ++i) {
    const double t = a[i] - b[i];
    sq += t * t;
  }
  return exp(-sqrt(sq) / lambda);
}

/* find_cluster, accuracy_model.cpp:36-49: strict '>' argmax from best_sim
 * 0.0, accepted iff >= threshold. */
int orc_find_cluster(int k, const double* clusters, int d, const double* scene,
                     const orc_params* p) {
  int best = -1;
  double best_sim = 0.0;
  for (int c = 0; c < k; ++c) {
    const double s = orc_similarity(clusters + c * d, scene, d, p->similarity_lambda);
    if (s > best_sim) {
      best_sim = s;
      best = c;
    }
  }
  if (best >= 0 && best_sim >= p->cluster_similarity_threshold) return best;
  return -1;
}

/* eval, accuracy_model.cpp:60-67. */
double orc_eval(int k, const double* clusters, const double* prof, int clen,
                const double* centroid, int d, const double* scene, const orc_params* p) {
  if (k == 0 || clen == 0) return p->acc_floor;
  const int cl = orc_find_cluster(k, clusters, d, scene, p);
  const double pr = cl < 0 ? 0.0 : prof[cl];
  const double sim = orc_similarity(scene, centroid, d, p->similarity_lambda);
  return p->acc_floor + (p->acc_ceil - p->acc_floor) * pr * sim;
}

/* pixels_per_frame, types.cpp:11-13. */
static double ppf(double q) { return q * (16.0 * q / 9.0); }

/* train_step, accuracy_model.cpp:69-111.  Returns 1 on invalid input, 2 when
 * the packed model runs out of cluster capacity. */
int orc_train_step(int* k, double* clusters, double* prof, int* clen, double* centroid, int kmax,
                   int d, double fps, double res, double quality, double gpu_s, int n_src,
                   const double* src_scenes, const double* src_tp, const double* src_frac,
                   const orc_params* p) {
  if (gpu_s < 0.0) return 1;
  double mix_total = 0.0;
  for (int i = 0; i < n_src; ++i) {
    if (src_frac[i] < 0.0) return 1;
    mix_total += src_frac[i];
  }
  if (n_src > 0 && fabs(mix_total - 1.0) > 1e-9) return 1;
  const double supplied = fps * ppf(res);
  double required = 0.0;
  if (n_src > 0) {
    double sum = 0.0;
    for (int i = 0; i < n_src; ++i) sum += src_tp[i];
    required = sum / (double)n_src;
  }
  const double sufficiency = required > 0.0 ? fmin(1.0, supplied / required) : 1.0;
  const double effort = gpu_s * sufficiency * quality;
  if (effort <= 0.0) return 0;

  /* cluster_weight is a std::map<int,double>: accumulate per cluster id, then
   * visit ascending ids.  New clusters are appended in source order. */
  double weight[64];
  int touched[64];
  if (kmax > 64) return 2;
  for (int c = 0; c < kmax; ++c) {
    weight[c] = 0.0;
    touched[c] = 0;
  }
  double cen[16];
  int have_cen = 0;
  for (int i = 0; i < n_src; ++i) {
    const double* sc = src_scenes + i * d;
    int cl = orc_find_cluster(*k, clusters, d, sc, p);
    if (cl < 0) {
      if (*k >= kmax) return 2;
      memcpy(clusters + (*k) * d, sc, sizeof(double) * d);
      prof[*k] = 0.0;
      cl = (*k)++;
    }
    weight[cl] += src_frac[i];
    touched[cl] = 1;
    if (!have_cen) {
      for (int j = 0; j < d; ++j) cen[j] = 0.0;
      have_cen = 1;
    }
    for (int j = 0; j < d; ++j) cen[j] += src_frac[i] * sc[j];
  }
  for (int c = 0; c < *k; ++c) {
    if (!touched[c] || weight[c] <= 0.0) continue;
    const double pr = prof[c];
    prof[c] = 1.0 - (1.0 - pr) * exp(-p->learning_rate_k * effort * weight[c]);
  }
  if (have_cen) {
    memcpy(centroid, cen, sizeof(double) * d);
    *clen = d;
  }
  return 0;
}

/* seed_model, accuracy_model.cpp:124-134. */
void orc_seed_model(const double* scene, int d, double device_acc, const orc_params* p,
                    double* cluster, double* prof) {
  const double span = p->acc_ceil - p->acc_floor;
  double pr = 0.0;
  if (span > 0.0) {
    pr = (device_acc - p->acc_floor) / span;
    if (pr < 0.0) pr = 0.0;
    if (pr > 1.0) pr = 1.0;
  }
  memcpy(cluster, scene, sizeof(double) * d);
  *prof = pr;
}

void orc_eval_matrix(int n, const double* scenes, int g, const int* ks, const double* clusters,
                     const double* profs, const int* clens, const double* centroids, int kmax,
                     int d, const orc_params* p, double* out) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < g; ++j)
      out[(long)i * g + j] =
          orc_eval(ks[j], clusters + (long)j * kmax * d, profs + (long)j * kmax, clens[j],
                   centroids + (long)j * d, d, scenes + (long)i * d, p);
}

/* Tie preference, transmission.cpp:17-27. */
static int preferred(double cf, double cq, double pf, double pq, int bias) {
  if (bias == 0) {
    if (cq != pq) return cq > pq;
    return cf > pf;
  }
  if (cf != pf) return cf > pf;
  return cq > pq;
}

/* build_profile_table (transmission.cpp:52-100) with make_accuracy_probe
 * (:102-118) and adapt_compression (:151-166). */
int orc_profile_table(const double* scene, int d, double throughput, int bias, int n_levels,
                      const double* levels_in, int n_grid, const double* gf, const double* gq,
                      double window_s, double tie_eps, double ref_rate, double bpp_ref,
                      const orc_params* p, double* out_budget, double* out_fps, double* out_res,
                      uint8_t* out_feasible) {
  if (n_grid <= 0 || n_levels <= 0 || !(window_s > 0.0) || !(ref_rate > 0.0)) return 1;
  double* levels = (double*)malloc(sizeof(double) * n_levels);
  double* accs = (double*)malloc(sizeof(double) * n_grid);
  memcpy(levels, levels_in, sizeof(double) * n_levels);
  /* std::sort ascending (insertion sort; values are distinct budget levels) */
  for (int i = 1; i < n_levels; ++i) {
    double v = levels[i];
    int j = i - 1;
    while (j >= 0 && levels[j] > v) {
      levels[j + 1] = levels[j];
      --j;
    }
    levels[j + 1] = v;
  }
  /* cheapest(grid), transmission.cpp:29-39 */
  int ch = 0;
  for (int i = 0; i < n_grid; ++i) {
    const double pr = gf[i] * ppf(gq[i]), pb = gf[ch] * ppf(gq[ch]);
    if (pr < pb || (pr == pb && (gq[i] < gq[ch] || (gq[i] == gq[ch] && gf[i] < gf[ch])))) ch = i;
  }
  int rc = 0;
  for (int l = 0; l < n_levels; ++l) {
    const double budget = levels[l];
    if (!(budget > 0.0)) {
      rc = 1;
      break;
    }
    const double pixel_budget = throughput * budget / window_s;
    int found = 0;
    double best = 0.0;
    for (int i = 0; i < n_grid; ++i) {
      accs[i] = 0.0;
      if (gf[i] * ppf(gq[i]) > pixel_budget) continue;
      /* probe: seed at the floor, one train_step(budget), eval */
      double cl[16], pr, cen[16];
      int k = 1, clen = d;
      orc_seed_model(scene, d, p->acc_floor, p, cl, &pr);
      memcpy(cen, scene, sizeof(double) * d);
      double quality = 0.0;
      {
        const double pixel_rate = gf[i] * ppf(gq[i]);
        const double bpp = ref_rate / pixel_rate;
        quality = fmin(1.0, bpp / bpp_ref);
      }
      const double frac = 1.0;
      double clusters[32];
      memcpy(clusters, cl, sizeof(double) * d);
      double prof[2] = {pr, 0.0};
      orc_train_step(&k, clusters, prof, &clen, cen, 2, d, gf[i], gq[i], quality, budget, 1,
                     scene, &throughput, &frac, p);
      accs[i] = orc_eval(k, clusters, prof, clen, cen, d, scene, p);
      if (!found || accs[i] > best) best = accs[i];
      found = 1;
    }
    out_budget[l] = budget;
    if (!found) {
      out_fps[l] = gf[ch];
      out_res[l] = gq[ch];
      out_feasible[l] = 0;
      continue;
    }
    int have = 0;
    double pf = 0.0, pq = 0.0;
    for (int i = 0; i < n_grid; ++i) {
      if (gf[i] * ppf(gq[i]) > pixel_budget) continue;
      if (accs[i] < best - tie_eps) continue;
      if (!have || preferred(gf[i], gq[i], pf, pq, bias)) {
        pf = gf[i];
        pq = gq[i];
        have = 1;
      }
    }
    out_fps[l] = pf;
    out_res[l] = pq;
    out_feasible[l] = 1;
  }
  free(levels);
  free(accs);
  return rc;
}

/* JobTrainingBackend::evaluate (orchestrator.cpp:43-50) and ::train (:52-62). */
int orc_param_trajectories(int n_jobs, int* ks, double* clusters, double* profs, int* clens,
                           double* centroids, int kmax, int d, const double* cam_scenes,
                           const double* cam_tp, const double* batches, const int* src_off,
                           const int* src_cam, const double* src_frac, const int* mem_off,
                           const int* mem_cam, double gpu_s, int depth, const orc_params* p,
                           double* out_acc) {
  double src_sc[64 * 16], src_t[64];
  for (int j = 0; j < n_jobs; ++j) {
    double* cl = clusters + (long)j * kmax * d;
    double* pr = profs + (long)j * kmax;
    double* ce = centroids + (long)j * d;
    const int ns = src_off[j + 1] - src_off[j];
    if (ns > 64 || d > 16) return 2;
    for (int s = 0; s < ns; ++s) {
      const int c = src_cam[src_off[j] + s];
      memcpy(src_sc + s * d, cam_scenes + (long)c * d, sizeof(double) * d);
      src_t[s] = cam_tp[c];
    }
    for (int t = 0; t <= depth; ++t) {
      if (t > 0) {
        const int rc = orc_train_step(&ks[j], cl, pr, &clens[j], ce, kmax, d, batches[3 * j],
                                      batches[3 * j + 1], batches[3 * j + 2], gpu_s, ns, src_sc,
                                      src_t, src_frac + src_off[j], p);
        if (rc) return rc;
      }
      const int nm = mem_off[j + 1] - mem_off[j];
      double acc;
      if (nm == 0) {
        acc = p->acc_floor;
      } else {
        double sum = 0.0;
        for (int m = 0; m < nm; ++m)
          sum += orc_eval(ks[j], cl, pr, clens[j], ce, d,
                          cam_scenes + (long)mem_cam[mem_off[j] + m] * d, p);
        acc = sum / nm;
      }
      out_acc[(long)j * (depth + 1) + t] = acc;
    }
  }
  return 0;
}

/* ======================= learned backend (spec) ======================= */

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

static float f_as(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint32_t u_as(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}

/* Deterministic expf shared with the device: range reduction by ln2 with a
 * two-constant split, degree-6 Taylor/Horner polynomial, fmaf throughout. */
float orc_expf(float x) {
  if (x < -87.0f) return 0.0f;
  if (x > 88.0f) x = 88.0f;
  const float k = rintf(x * 0x1.715476p+0f);
  float r = fmaf(k, -0x1.62e400p-1f, x);
  r = fmaf(k, -0x1.7f7d1cp-20f, r);
  float q = 0x1.6c16c2p-10f; /* 1/720 */
  q = fmaf(q, r, 0x1.111112p-7f);
  q = fmaf(q, r, 0x1.555556p-5f);
  q = fmaf(q, r, 0x1.555556p-3f);
  q = fmaf(q, r, 0.5f);
  q = fmaf(q, r, 1.0f);
  q = fmaf(q, r, 1.0f);
  const int ki = (int)k;
  return q * f_as((uint32_t)(ki + 127) << 23);
}

uint16_t orc_f32_to_bf16(float x) {
  uint32_t u = u_as(x);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float orc_bf16_to_f32(uint16_t b) { return f_as((uint32_t)b << 16); }

static float usym(uint32_t w) { return (float)(w >> 8) * 0x1p-23f - 1.0f; }

static void seed_key(const orc_lcfg* c, uint32_t salt, uint32_t key[2]) {
  key[0] = (uint32_t)c->seed ^ salt;
  key[1] = (uint32_t)(c->seed >> 32);
}

/* P[c][f] = U(-1,1); Q[c][d][f] = 4 * U(-1,1). */
void orc_prototypes(const orc_lcfg* c, float* P, float* Q) {
  uint32_t key[2], out[4];
  seed_key(c, 0u, key);
  for (int k = 0; k < c->C; ++k)
    for (int f = 0; f < c->F; ++f) {
      const uint32_t ctr[4] = {(uint32_t)f, (uint32_t)k, 0u, 0xFE000000u};
      orc_philox(ctr, key, out);
      P[(long)k * c->F + f] = usym(out[0]);
      for (int d = 0; d < c->D; ++d) {
        const uint32_t ctr2[4] = {(uint32_t)f, (uint32_t)k, 1u + d, 0xFE000000u};
        orc_philox(ctr2, key, out);
        Q[((long)k * c->D + d) * c->F + f] = usym(out[0]) * 4.0f;
      }
    }
}

/* x = bf16(P[y] + sum_d s_d Q[y][d] + sigma * tri_noise), label y = U{0..C-1}. */
void orc_gen_frames(const orc_lcfg* c, const float* P, const float* Q, int cam, int window,
                    int tag, int n_frames, const double* scene, uint16_t* x, int32_t* y) {
  uint32_t key[2], out[4];
  seed_key(c, 0u, key);
  float sd[16];
  for (int d = 0; d < c->D; ++d) sd[d] = (float)scene[d];
  const uint32_t wt = ((uint32_t)window & 0xFFFFFFu) | ((uint32_t)tag << 24);
  for (int r = 0; r < n_frames; ++r) {
    const uint32_t lc[4] = {0xFFFFFFFFu, (uint32_t)r, (uint32_t)cam, wt};
    orc_philox(lc, key, out);
    const int lab = (int)(out[0] % (uint32_t)c->C);
    y[r] = lab;
    for (int f4 = 0; f4 < c->F / 4; ++f4) {
      const uint32_t fc[4] = {(uint32_t)f4, (uint32_t)r, (uint32_t)cam, wt};
      orc_philox(fc, key, out);
      for (int i = 0; i < 4; ++i) {
        const int f = f4 * 4 + i;
        const float nz = (float)((out[i] & 0xFFFFu) + (out[i] >> 16)) * 0x1p-16f - 1.0f;
        float v = P[(long)lab * c->F + f];
        for (int d = 0; d < c->D; ++d) v = fmaf(sd[d], Q[((long)lab * c->D + d) * c->F + f], v);
        v = fmaf(c->noise, nz, v);
        x[(long)r * c->F + f] = orc_f32_to_bf16(v);
      }
    }
  }
}

void orc_sample(const orc_lcfg* c, int job_id, int n_src, const int* src_cams,
                const double* src_fracs, int window, int micro, int step, int* out_cam,
                int* out_frame) {
  uint32_t key[2], out[4];
  seed_key(c, (uint32_t)job_id * 0x9E3779B9u + 0x632BE5ABu, key);
  const uint32_t wt = ((uint32_t)window & 0xFFFFFFu) | (2u << 24);
  for (int s = 0; s < c->B; ++s) {
    const uint32_t ctr[4] = {(uint32_t)s, (uint32_t)step, (uint32_t)micro, wt};
    orc_philox(ctr, key, out);
    const double u = (double)(((uint64_t)out[0] << 21) | (out[1] >> 11)) * 0x1p-53;
    double cum = 0.0;
    int pick = n_src - 1;
    for (int i = 0; i < n_src; ++i) {
      cum += src_fracs[i];
      if (u < cum) {
        pick = i;
        break;
      }
    }
    out_cam[s] = src_cams[pick];
    out_frame[s] = (int)(out[2] % (uint32_t)c->R);
  }
}

/* The base model every new job starts from (the learned seed_model: an
 * untrained model, so a fresh job serves a camera exactly as well as an
 * ungrouped camera's own device model).  Kaiming-uniform, keyed by seed. */
void orc_init_weights(const orc_lcfg* c, float* w1, float* b1, float* w2, float* b2) {
  uint32_t key[2], out[4];
  seed_key(c, 0x27D4EB2Fu, key);
  const float a1 = sqrtf(6.0f / (float)c->F), a2 = sqrtf(6.0f / (float)c->H);
  for (int f = 0; f < c->F; ++f)
    for (int h = 0; h < c->H; ++h) {
      const uint32_t ctr[4] = {(uint32_t)h, (uint32_t)f, 1u, 3u << 24};
      orc_philox(ctr, key, out);
      w1[(long)f * c->H + h] = usym(out[0]) * a1;
    }
  for (int h = 0; h < c->H; ++h) b1[h] = 0.0f;
  for (int k = 0; k < c->H; ++k)
    for (int j = 0; j < c->C; ++j) {
      const uint32_t ctr[4] = {(uint32_t)j, (uint32_t)k, 2u, 3u << 24};
      orc_philox(ctr, key, out);
      w2[(long)k * c->C + j] = usym(out[0]) * a2;
    }
  for (int j = 0; j < c->C; ++j) b2[j] = 0.0f;
}

/* The learned step's arithmetic, fixed per output element: every dot
 * product is an fmaf chain in ascending contraction index from 0.0f, bias
 * added last; every gradient sum an fmaf (or +) chain in ascending sample
 * index.  The loops below keep exactly that sequence PER ELEMENT while
 * running the independent elements of a row in the inner loop (contiguous,
 * so the compiler vectorizes them with hardware FMA: the rounding of each
 * fmaf is the same single rounding whichever way it executes).  The device
 * FFMA path (learned_kernels.cu) follows the same sequences bit for bit. */

/* Forward of one sample: z (pre-activation, H), logits (C); acc: H floats
 * of scratch. */
static void fwd1(const orc_lcfg* c, const uint16_t* xs, const float* w1, const float* b1,
                 const float* w2, const float* b2, float* z, float* logit) {
  const int F = c->F, H = c->H, C = c->C;
  for (int h = 0; h < H; ++h) z[h] = 0.0f;
  for (int f = 0; f < F; ++f) {  /* z[h] = fmaf(x[f], W1[f][h], z[h]), f ascending */
    const float xf = orc_bf16_to_f32(xs[f]);
    const float* row = w1 + (long)f * H;
    for (int h = 0; h < H; ++h) z[h] = fmaf(xf, row[h], z[h]);
  }
  for (int h = 0; h < H; ++h) z[h] = z[h] + b1[h];
  float a[1024];
  for (int j = 0; j < C; ++j) a[j] = 0.0f;
  for (int k = 0; k < H; ++k) {  /* logit[j] = fmaf(relu(z[k]), W2[k][j], .), k ascending */
    const float hk = z[k] > 0.0f ? z[k] : 0.0f;
    const float* row = w2 + (long)k * C;
    for (int j = 0; j < C; ++j) a[j] = fmaf(hk, row[j], a[j]);
  }
  for (int j = 0; j < C; ++j) logit[j] = a[j] + b2[j];
}

float orc_sgd_step(const orc_lcfg* c, const uint16_t* x, const int32_t* y, float* w1, float* b1,
                   float* w2, float* b2) {
  const int B = c->B, F = c->F, H = c->H, C = c->C;
  float* z = (float*)malloc(sizeof(float) * B * H);
  float* dl = (float*)malloc(sizeof(float) * B * C);
  float* dh = (float*)malloc(sizeof(float) * B * H);
  float* w2t = (float*)malloc(sizeof(float) * C * H);
  float* acc = (float*)malloc(sizeof(float) * (H > C ? H : C));
  float* xf = (float*)malloc(sizeof(float) * B);
  float logit[1024];
  const float invB = 1.0f / (float)B;
  double loss = 0.0;
  for (int s = 0; s < B; ++s) {
    fwd1(c, x + (long)s * F, w1, b1, w2, b2, z + (long)s * H, logit);
    float m = logit[0];
    for (int j = 1; j < C; ++j) m = logit[j] > m ? logit[j] : m;
    float e[1024], sum = 0.0f;
    for (int j = 0; j < C; ++j) {
      e[j] = orc_expf(logit[j] - m);
      sum += e[j];
    }
    for (int j = 0; j < C; ++j) {
      const float pj = e[j] / sum;
      dl[(long)s * C + j] = (pj - (j == y[s] ? 1.0f : 0.0f)) * invB;
    }
    loss += (double)(logf(sum) - (logit[y[s]] - m));
  }
  /* dh[s][k] = relu'(z) * sum_j fmaf(dl[s][j], W2[k][j], .), j ascending, with
   * the pre-update W2 (transposed once so k runs contiguous) */
  for (int k = 0; k < H; ++k)
    for (int j = 0; j < C; ++j) w2t[(long)j * H + k] = w2[(long)k * C + j];
  for (int s = 0; s < B; ++s) {
    float* d = dh + (long)s * H;
    for (int k = 0; k < H; ++k) d[k] = 0.0f;
    for (int j = 0; j < C; ++j) {
      const float g = dl[(long)s * C + j];
      const float* row = w2t + (long)j * H;
      for (int k = 0; k < H; ++k) d[k] = fmaf(g, row[k], d[k]);
    }
    const float* zs = z + (long)s * H;
    for (int k = 0; k < H; ++k) d[k] = zs[k] > 0.0f ? d[k] : 0.0f;
  }
  /* W2[k][j] += -lr * sum_s fmaf(relu(z[s][k]), dl[s][j], .), s ascending */
  for (int k = 0; k < H; ++k) {
    for (int j = 0; j < C; ++j) acc[j] = 0.0f;
    for (int s = 0; s < B; ++s) {
      const float zk = z[(long)s * H + k];
      const float r = zk > 0.0f ? zk : 0.0f;
      const float* g = dl + (long)s * C;
      for (int j = 0; j < C; ++j) acc[j] = fmaf(r, g[j], acc[j]);
    }
    for (int j = 0; j < C; ++j) w2[(long)k * C + j] = fmaf(-c->lr, acc[j], w2[(long)k * C + j]);
  }
  for (int j = 0; j < C; ++j) acc[j] = 0.0f;
  for (int s = 0; s < B; ++s)
    for (int j = 0; j < C; ++j) acc[j] += dl[(long)s * C + j];
  for (int j = 0; j < C; ++j) b2[j] = fmaf(-c->lr, acc[j], b2[j]);
  /* W1[f][h] += -lr * sum_s fmaf(x[s][f], dh[s][h], .), s ascending */
  for (int f = 0; f < F; ++f) {
    for (int s = 0; s < B; ++s) xf[s] = orc_bf16_to_f32(x[(long)s * F + f]);
    for (int h = 0; h < H; ++h) acc[h] = 0.0f;
    for (int s = 0; s < B; ++s) {
      const float v = xf[s];
      const float* d = dh + (long)s * H;
      for (int h = 0; h < H; ++h) acc[h] = fmaf(v, d[h], acc[h]);
    }
    float* row = w1 + (long)f * H;
    for (int h = 0; h < H; ++h) row[h] = fmaf(-c->lr, acc[h], row[h]);
  }
  for (int h = 0; h < H; ++h) acc[h] = 0.0f;
  for (int s = 0; s < B; ++s)
    for (int h = 0; h < H; ++h) acc[h] += dh[(long)s * H + h];
  for (int h = 0; h < H; ++h) b1[h] = fmaf(-c->lr, acc[h], b1[h]);
  free(z);
  free(dl);
  free(dh);
  free(w2t);
  free(acc);
  free(xf);
  return (float)(loss / B);
}

int orc_count_correct(const orc_lcfg* c, const uint16_t* x, const int32_t* y, int n,
                      const float* w1, const float* b1, const float* w2, const float* b2) {
  float* z = (float*)malloc(sizeof(float) * c->H);
  float logit[1024];
  int correct = 0;
  for (int s = 0; s < n; ++s) {
    fwd1(c, x + (long)s * c->F, w1, b1, w2, b2, z, logit);
    int best = 0;
    for (int j = 1; j < c->C; ++j)
      if (logit[j] > logit[best]) best = j;
    correct += best == y[s];
  }
  free(z);
  return correct;
}

int orc_learned_steps(const orc_lcfg* c, double fps, double res, double quality, double gpu_s,
                      int n_src, const double* src_tp) {
  if (n_src <= 0) return 0;
  const double supplied = fps * ppf(res);
  double sum = 0.0;
  for (int i = 0; i < n_src; ++i) sum += src_tp[i];
  const double required = sum / (double)n_src;
  const double sufficiency = required > 0.0 ? fmin(1.0, supplied / required) : 1.0;
  const double effort = gpu_s * sufficiency * quality;
  if (effort <= 0.0) return 0;
  return (int)floor(effort * c->steps_per_gpu_s);
}
