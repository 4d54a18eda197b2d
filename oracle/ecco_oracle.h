/*
 * ecco_oracle.h -- TEST INFRASTRUCTURE: the CPU checker for the B200 path.
 *
 * A plain-C restatement of the reference's group-retraining arithmetic
 * (parametric backend: every function cites the reference file:line it
 * follows) and the specification of the learned backend.  The learned
 * backend has no reference counterpart: its parity is UNPINNED by the
 * reference ("parity unpinned") -- this restatement is
 * its specification.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load it.  The product never does.
 */
#ifndef ECCO_ORACLE_H_
#define ECCO_ORACLE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ModelParams, accuracy_model.hpp:18-24 (same layout as ecco_model_params). */
typedef struct {
  double learning_rate_k, similarity_lambda, acc_floor, acc_ceil, cluster_similarity_threshold;
} orc_params;

/* ---------------- parametric backend ---------------- */
double orc_similarity(const double* a, const double* b, int d, double lambda);
int orc_find_cluster(int k, const double* clusters, int d, const double* scene,
                     const orc_params* p);
double orc_eval(int k, const double* clusters, const double* prof, int clen,
                const double* centroid, int d, const double* scene, const orc_params* p);
int orc_train_step(int* k, double* clusters, double* prof, int* clen, double* centroid, int kmax,
                   int d, double fps, double res, double quality, double gpu_s, int n_src,
                   const double* src_scenes, const double* src_tp, const double* src_frac,
                   const orc_params* p);
void orc_seed_model(const double* scene, int d, double device_acc, const orc_params* p,
                    double* cluster, double* prof);
void orc_eval_matrix(int n, const double* scenes, int g, const int* ks, const double* clusters,
                     const double* profs, const int* clens, const double* centroids, int kmax,
                     int d, const orc_params* p, double* out);
int orc_profile_table(const double* scene, int d, double throughput, int bias, int n_levels,
                      const double* levels, int n_grid, const double* grid_fps,
                      const double* grid_res, double window_s, double tie_eps, double ref_rate,
                      double bpp_ref, const orc_params* p, double* out_budget, double* out_fps,
                      double* out_res, uint8_t* out_feasible);
/* Per-job trajectories of JobTrainingBackend (orchestrator.cpp:43-62):
 * acc[j][0] = evaluate; then depth x (train, evaluate).  Models are updated
 * in place (packed, stride kmax). */
int orc_param_trajectories(int n_jobs, int* ks, double* clusters, double* profs, int* clens,
                           double* centroids, int kmax, int d, const double* cam_scenes,
                           const double* cam_tp, const double* batches /* n_jobs*3 */,
                           const int* src_off, const int* src_cam, const double* src_frac,
                           const int* mem_off, const int* mem_cam, double gpu_s, int depth,
                           const orc_params* p, double* out_acc);

/* ---------------- learned backend specification ---------------- */
typedef struct {
  int F, H, C, D, B, R, S;
  float lr, noise;
  double steps_per_gpu_s;
  uint64_t seed;
} orc_lcfg;

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float orc_expf(float x);
uint16_t orc_f32_to_bf16(float x);
float orc_bf16_to_f32(uint16_t b);
/* Class prototypes P[C][F], Q[C][D][F] (fp32). */
void orc_prototypes(const orc_lcfg* c, float* P, float* Q);
/* Frames of one camera for one window: tag 0 = training ring (R frames),
 * tag 1 = labelled eval set (S frames).  Features are bf16 bits. */
void orc_gen_frames(const orc_lcfg* c, const float* P, const float* Q, int cam, int window,
                    int tag, int n_frames, const double* scene, uint16_t* x, int32_t* y);
void orc_sample(const orc_lcfg* c, int job_id, int n_src, const int* src_cams,
                const double* src_fracs, int window, int micro, int step, int* out_cam,
                int* out_frame);
void orc_init_weights(const orc_lcfg* c, float* w1, float* b1, float* w2, float* b2);
/* One SGD step on a gathered minibatch x[B*F] (bf16 bits), y[B]. Returns the
 * mean loss. */
float orc_sgd_step(const orc_lcfg* c, const uint16_t* x, const int32_t* y, float* w1, float* b1,
                   float* w2, float* b2);
int orc_count_correct(const orc_lcfg* c, const uint16_t* x, const int32_t* y, int n,
                      const float* w1, const float* b1, const float* w2, const float* b2);
/* Number of SGD steps one train(job, gpu_s) call runs (effort of
 * accuracy_model.cpp:82-86 times steps_per_gpu_s, floored). */
int orc_learned_steps(const orc_lcfg* c, double fps, double res, double quality, double gpu_s,
                      int n_src, const double* src_tp);

#ifdef __cplusplus
}
#endif
#endif
