/*
 * ecco_b200.h -- C-ABI of the B200-native group-retraining path of ECCO
 * (arXiv 2512.11727).
 *
 * The reference (a C++20 simulator, /root/reference/proj) drives this path
 * through three callback seams and a handful of free functions:
 *
 *   TrainingBackend::evaluate / ::train   proj/core/include/ecco/gpu_allocator.hpp:37-42
 *   ModelEvalFn                           proj/core/include/ecco/grouping.hpp:23
 *   ProbeFn (+ build_profile_table)       proj/core/include/ecco/transmission.hpp:46,52-56
 *   eval / train_step / seed_model        proj/core/include/ecco/accuracy_model.hpp:72-94
 *
 * Every entry point below replaces a batch of those per-item calls; the
 * comment on each names the reference interface it stands in for.  All
 * arguments are plain pointers and sizes; host buffers are copied
 * synchronously unless the name ends in _dev (device pointers, stream-ordered
 * on the context's stream).  Errors are reported as an ecco_status whose
 * values map 1:1 onto the reference's exception types (see ecco_status), with
 * the message available from ecco_last_error().  A context is not
 * thread-safe, matching the reference's single-owner contract
 * (proj/README.md:42-43).
 *
 * Two backends share the boundary:
 *   ECCO_BACKEND_PARAMETRIC  device restatement of accuracy_model.cpp, fp64,
 *                            bit-identical to the reference library;
 *   ECCO_BACKEND_LEARNED     real per-group MLPs (fwd + bwd + SGD) over
 *                            synthetic camera streams resident in HBM.
 */
#ifndef ECCO_B200_H_
#define ECCO_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ecco_ctx ecco_ctx;

/* Status codes; the C++ wrapper rethrows them as the reference's exceptions. */
typedef enum {
  ECCO_OK = 0,
  ECCO_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                  */
  ECCO_ERR_LOGIC = 2,            /* std::logic_error                       */
  ECCO_ERR_INFEASIBLE = 3,       /* ecco::InfeasibleScheduleError          */
  ECCO_ERR_SCHEMA = 4,           /* ecco::SchemaError                      */
  ECCO_ERR_CUDA = 5,             /* device failure (no reference analogue) */
  ECCO_ERR_RUNTIME = 6           /* std::runtime_error                     */
} ecco_status;

typedef enum { ECCO_BACKEND_PARAMETRIC = 0, ECCO_BACKEND_LEARNED = 1 } ecco_backend;

/* Arithmetic of the learned backend's dense contractions.
 *
 * ECCO_MATH_TC_BF16: tcgen05 tensor-core math with fp32 accumulation in TMEM
 * and fp32 master weights; the operands are bf16 (kind::f16) in the fused
 * SGD chain (train_kernels.cu, every contraction) and in the fused
 * evaluation kernels (eval_kernels.cu); shapes outside the fused chain
 * (tc_kernels.cu) run a bf16 forward and a kind::tf32 W1 gradient.  Results
 * are within the tolerances stated in DESIGN.md 2, not bit-exact.
 * ECCO_MATH_TC_TF32 is the round-1 name of the same mode (kept as an alias). */
typedef enum {
  ECCO_MATH_FFMA_EXACT = 0, /* fp32 FFMA in the oracle's order: bit-exact        */
  ECCO_MATH_TC_BF16 = 1,    /* tcgen05, bf16 operands (+tf32 dW1 off the chain)  */
  ECCO_MATH_TC_TF32 = 1     /* alias of ECCO_MATH_TC_BF16                        */
} ecco_math;

/* ModelParams (proj/core/include/ecco/accuracy_model.hpp:18-24). */
typedef struct {
  double learning_rate_k;
  double similarity_lambda;
  double acc_floor;
  double acc_ceil;
  double cluster_similarity_threshold;
} ecco_model_params;

typedef struct {
  int backend;          /* ecco_backend                                   */
  int device;           /* CUDA ordinal                                   */
  int scene_dims;       /* D, shared by every scene                       */
  int max_clusters;     /* P: cluster capacity per model (K_max)          */
  int max_jobs;         /* model slots                                    */
  int max_cameras;      /* camera table capacity                          */
  ecco_model_params params;
  /* learned backend */
  int math;             /* ecco_math                                      */
  int feat_dim;         /* F  (frame feature width)                       */
  int hidden_dim;       /* H                                              */
  int num_classes;      /* C                                              */
  int minibatch;        /* B samples per SGD step                         */
  int ring_frames;      /* R training frames per camera per window        */
  int eval_samples;     /* S labelled eval frames per camera              */
  int max_depth;        /* speculative trajectory depth kept as snapshots */
  float sgd_lr;
  float feature_noise;  /* sigma of the synthetic frame noise             */
  double steps_per_gpu_s; /* SGD steps one effective GPU-second buys      */
  uint64_t seed;
} ecco_config;

/* Defaults equal to the reference's ModelParams{} plus the learned-backend
 * classifier shape of SURVEY.md 8(a'): F=512, H=256, C=16, B=128. */
void ecco_default_config(ecco_config* cfg);

ecco_status ecco_create(const ecco_config* cfg, ecco_ctx** out);
void ecco_destroy(ecco_ctx* ctx);
const char* ecco_last_error(const ecco_ctx* ctx);
/* Number of kernels this context has launched (the bench's gpu_launches). */
uint64_t ecco_kernel_launches(const ecco_ctx* ctx);
/* Per-kernel device timing with CUDA events on the context stream (off by
 * default).  ecco_kernel_stat returns, for one tracked kernel family, the
 * launches, summed device milliseconds and the algorithmic flops and bytes of
 * those launches (units in DESIGN.md). */
typedef enum {
  ECCO_KSTAT_TRAIN_STEP = 0,   /* learned: fused SGD step (unfused math: hidden layer) */
  ECCO_KSTAT_TRAIN_DW1 = 1,    /* learned, unfused math: W1 gradient + SGD update   */
  ECCO_KSTAT_TRAIN_HEAD = 2,   /* learned, unfused math: logits/softmax/dH/W2       */
  ECCO_KSTAT_EVAL_MATRIX = 3,  /* learned: dense camera x group evaluation matrix   */
  ECCO_KSTAT_EVAL_PAIRS = 4,   /* learned: (camera, job) pair lists (chains, jobs)  */
  ECCO_KSTAT_P_EVAL = 5,       /* parametric eval matrix / pairs               */
  ECCO_KSTAT_P_TRAJ = 6,       /* parametric trajectories                      */
  ECCO_KSTAT_P_PROFILE = 7,    /* parametric profile tables                    */
  ECCO_KSTAT_FRAMES = 8,       /* synthetic stream generation                  */
  ECCO_KSTAT_COUNT = 9
} ecco_kstat;
ecco_status ecco_profile(ecco_ctx* ctx, int enable);
ecco_status ecco_kernel_stat(ecco_ctx* ctx, int which, uint64_t* launches, double* ms,
                             double* flops, double* bytes);
/* Host<->device bytes this context has copied (the bench's e2e accounting). */
ecco_status ecco_transfer_bytes(const ecco_ctx* ctx, uint64_t* h2d, uint64_t* d2h);
/* cudaStream_t the context launches on (as void*). */
void* ecco_stream(ecco_ctx* ctx);
ecco_status ecco_synchronize(ecco_ctx* ctx);

/* ---- camera table --------------------------------------------------------
 * CameraState (accuracy_model.hpp:27-34): scene + gpu_pixel_throughput.
 * Camera indices are positions in this table; the host keeps the
 * CameraId <-> index map and passes member lists in std::string order. */
ecco_status ecco_set_cameras(ecco_ctx* ctx, int n, const double* scenes /* n*D */,
                             const double* gpu_pixel_throughput /* n */);
/* apply_drift's scene change (accuracy_model.cpp:113-122) for a subset. */
ecco_status ecco_update_scenes(ecco_ctx* ctx, int n, const int* cam_idx,
                               const double* scenes /* n*D */);
/* Learned backend: (re)generate window `window`'s synthetic frame rings and
 * eval sets for every camera from (seed, camera, window, scene). */
ecco_status ecco_generate_frames(ecco_ctx* ctx, int window);
/* Learned backend, end-to-end path: upload frames produced on the host
 * (pinned or pageable) instead of generating them on the device.
 * frames: n*R*F bf16 bits, labels: n*R, eval: n*S*F bf16 bits, eval labels. */
ecco_status ecco_upload_frames(ecco_ctx* ctx, int n_cams, const uint16_t* frames,
                               const int32_t* labels, const uint16_t* eval_frames,
                               const int32_t* eval_labels);
/* Double-buffered window ingest, for overlapping the next window's upload
 * with the current window's kernels: ecco_stage_frames copies host frames
 * (same layouts as ecco_upload_frames; pinned memory for a truly
 * asynchronous DMA) into a back buffer on a separate copy stream and returns
 * immediately; ecco_swap_frames makes them current (the context stream
 * waits for the copy; no host synchronisation).  Kernels enqueued before the
 * swap keep reading the previous frames. */
ecco_status ecco_stage_frames(ecco_ctx* ctx, int n_cams, const uint16_t* frames,
                              const int32_t* labels, const uint16_t* eval_frames,
                              const int32_t* eval_labels);
ecco_status ecco_swap_frames(ecco_ctx* ctx);
/* The two parts of the staged ingest swap independently: bit 0 the frame
 * rings + their labels (what the SGD steps read), bit 1 the eval sets + their
 * labels (what the evaluation matrix and member evaluations read).  A staging
 * call stages the parts it copies (rings when ring cameras or sampled rows
 * are given, eval when n_eval > 0); ecco_swap_frames swaps every staged part,
 * ecco_swap_frame_parts the requested ones, so a window's eval sets can
 * become current for the regroup while its rings still stream in. */
ecco_status ecco_swap_frame_parts(ecco_ctx* ctx, int parts);
/* Allocates everything the staged ingest uses (back buffers of the frame
 * table and eval sets, copy stream, the sampled-row bitmap) up front, so the
 * first staging call does not pay for gigabytes of fresh device memory. */
ecco_status ecco_reserve_ingest(ecco_ctx* ctx);
/* Group-sharded variant of ecco_stage_frames: the frame rings of cameras
 * [ring_first, ring_first + ring_n) only (the members of this rank's groups:
 * a job trains on its own members' frames, orchestrator.cpp:52-62, 282-309)
 * and the eval sets of cameras [0, eval_n) (every camera is scored against
 * this rank's groups).  `frames` / `labels` point at camera ring_first's
 * ring.  Rings outside the range are left as they were in the back buffer. */
ecco_status ecco_stage_frames_range(ecco_ctx* ctx, int ring_first, int ring_n,
                                    const uint16_t* frames, const int32_t* labels, int eval_n,
                                    const uint16_t* eval_frames, const int32_t* eval_labels);
/* Copies the first n_cams cameras' resident frames back to the host (same
 * layouts as ecco_upload_frames; any pointer may be NULL). */
ecco_status ecco_read_frames(ecco_ctx* ctx, int n_cams, uint16_t* frames, int32_t* labels,
                             uint16_t* eval_frames, int32_t* eval_labels);
/* Same upload from device buffers already resident in HBM (stream-ordered). */
ecco_status ecco_upload_frames_dev(ecco_ctx* ctx, int n_cams, const void* frames,
                                   const void* labels, const void* eval_frames,
                                   const void* eval_labels);

/* ---- job models (RetrainJob::model, job.hpp:25-36) -----------------------
 * Parametric: ModelState = K clusters (K*D), K proficiencies, centroid (D;
 * centroid_len 0 = empty model).  Arrays are packed per job with stride
 * max_clusters. */
ecco_status ecco_put_models(ecco_ctx* ctx, int n, const int* job_ids,
                            const int* n_clusters, const double* clusters,
                            const double* proficiency, const double* centroid,
                            const int* centroid_len);
ecco_status ecco_get_models(ecco_ctx* ctx, int n, const int* job_ids, int* n_clusters,
                            double* clusters, double* proficiency, double* centroid,
                            int* centroid_len);
/* seed_model (accuracy_model.cpp:124-134) for new jobs: parametric seeds
 * cluster = centroid = scene, prof = clamp((acc - floor)/span); learned
 * initialises the MLP from (seed, job_id). */
ecco_status ecco_seed_models(ecco_ctx* ctx, int n, const int* job_ids,
                             const double* scenes /* n*D */, const double* device_acc);
/* Job termination (orchestrator.cpp:375): frees the slots. */
ecco_status ecco_drop_models(ecco_ctx* ctx, int n, const int* job_ids);
/* Learned backend: read / write the fp32 master weights of one job
 * (W1[F*H] row-major by feature, b1[H], W2[H*C], b2[C]). */
ecco_status ecco_get_weights(ecco_ctx* ctx, int job_id, float* w1, float* b1, float* w2,
                             float* b2);
ecco_status ecco_set_weights(ecco_ctx* ctx, int job_id, const float* w1, const float* b1,
                             const float* w2, const float* b2);

/* ---- TrainingBackend::evaluate (orchestrator.cpp:43-50) -------------------
 * Mean accuracy of each job's model over its members (camera indices in
 * member order, CSR); summed sequentially in that order, then divided. */
ecco_status ecco_eval_jobs(ecco_ctx* ctx, int n_jobs, const int* job_ids,
                           const int* member_offsets /* n_jobs+1 */,
                           const int* member_cams, double* out_mean /* n_jobs */);

/* ---- ModelEvalFn batch: the camera x group evaluation matrix ---------------
 * out[i*n_jobs + j] = eval(model(job_ids[j]), probe i).  A probe is a scene
 * (parametric: `scenes`, n_probes*D) or a camera's labelled eval set
 * (learned: `cam_idx`).  `mask` (nullable, n_probes*n_jobs bytes) skips
 * pairs rejected by correlation_filter (grouping.cpp:9-16); skipped entries
 * are written as NaN.  Replaces eval_job_on_scene (orchestrator.cpp:186-191)
 * called from group_request (grouping.cpp:33). */
ecco_status ecco_eval_matrix(ecco_ctx* ctx, int n_probes, const double* scenes,
                             const int* cam_idx, int n_jobs, const int* job_ids,
                             const uint8_t* mask, double* out);
/* Device-resident variant: out_dev is an n_probes*n_jobs fp64 device buffer;
 * stream-ordered on the context stream, returns without host synchronisation. */
ecco_status ecco_eval_matrix_dev(ecco_ctx* ctx, int n_probes, const double* scenes,
                                 const int* cam_idx, int n_jobs, const int* job_ids,
                                 const uint8_t* mask, void* out_dev);
/* The same matrix (learned backend, tensor-core math, camera probes)
 * enqueued on the context's own MATRIX stream, after everything enqueued on
 * the context stream so far (it evaluates the models committed by then), with
 * its evaluation grid leaving `reserve_sms` SMs free for the kernels the
 * context stream launches meanwhile; returns at once.  ecco_matrix_join makes
 * the context stream wait for it.  A model committed while it runs may be
 * read half-updated: its column must be re-evaluated after the join (what the
 * window-end regroup of paper_2512_11727_b200/window.py does for the groups
 * the allocator trained beyond the initial pass, overlapping the rest of the
 * matrix with their serial chains). */
ecco_status ecco_eval_matrix_dev_async(ecco_ctx* ctx, int n_probes, const int* cam_idx, int n_jobs,
                                       const int* job_ids, void* out_dev, int reserve_sms);
ecco_status ecco_matrix_join(ecco_ctx* ctx);
/* Sparse form of the same matrix: out[p] = eval(model(job_ids[p]), probe p)
 * where probe p is scenes[p] (parametric; nullable = the camera's current
 * scene cams[p]) or camera cams[p]'s eval set (learned).  Used for the
 * window-end per-member accuracies (orchestrator.cpp:330-341) and for
 * routing passes whose candidate pairs were pruned by the filter. */
ecco_status ecco_eval_pairs(ecco_ctx* ctx, int n_pairs, const double* scenes, const int* cams,
                            const int* job_ids, double* out);
/* Re-keys model slots (a model seeded under a provisional id becomes the
 * job the host commits it as). */
ecco_status ecco_rename_models(ecco_ctx* ctx, int n, const int* old_ids, const int* new_ids);
/* Fused epilogue of group_request (grouping.cpp:30-39): for each probe the
 * lowest-index job j (in job_ids order) maximising out[i,j] among unmasked
 * pairs with out[i,j] >= req_acc[i] (strict '>' between candidates);
 * best_col = -1 when none qualifies.  The host commits in request order. */
ecco_status ecco_route_propose(ecco_ctx* ctx, int n_probes, const double* scenes,
                               const int* cam_idx, const double* req_acc, int n_jobs,
                               const int* job_ids, const uint8_t* mask, int* best_col,
                               double* best_acc);

/* Diagnostic of the fused evaluation kernel (learned backend, tensor-core
 * math): the logits (+ b2) of every eval frame of cameras cam_idx[0..n)
 * under every model job_ids[0..g), as out[((i*S + s)*g + j)*C + c].  Exposed
 * for the numerics tests only. */
ecco_status ecco_debug_eval_logits(ecco_ctx* ctx, int n, const int* cam_idx, int g,
                                   const int* job_ids, float* out);

/* Epilogue alone, over a camera x group matrix already in HBM (e.g. the
 * all-gathered column blocks of every rank): the warp-reduced argmax /
 * threshold of group_request (grouping.cpp:30-39) per camera row.
 * matrix_dev: n_blocks column blocks of g_block columns, block b an n x
 * g_block row-major fp64 array at matrix_dev + b*n*g_block (NaN = masked);
 * n_blocks = 1 is a plain row-major n x g_block matrix, n_blocks = world size
 * the output of an all-gather of every rank's ecco_eval_matrix_dev block.
 * Column j = b*g_block + jb.  req_dev: n fp64 device accuracies (nullable =
 * 0); best_col_dev: n int32 (-1 = none qualifies); best_acc_dev: n fp64.
 * Stream-ordered on the context stream; no host synchronisation. */
ecco_status ecco_route_matrix_dev(ecco_ctx* ctx, int n, int g_block, int n_blocks,
                                  const void* matrix_dev, const void* req_dev, void* best_col_dev,
                                  void* best_acc_dev);

/* Same epilogue with a column -> group id map, for group placements where a
 * rank's block holds arbitrary groups (the cost-balanced placement of
 * SURVEY.md 8(e), paper_2512_11727_b200/shard.py): col_ids_dev holds
 * n_blocks*g_block int32 group ids in gathered column order (< 0 = padding
 * column, skipped).  best_id_dev receives the winning GROUP ID (-1 = none),
 * ties going to the lowest id -- group_request's order over jobs in
 * ascending id (grouping.cpp:30-39) -- whatever rank holds the group. */
ecco_status ecco_route_matrix_ids_dev(ecco_ctx* ctx, int n, int g_block, int n_blocks,
                                      const void* matrix_dev, const void* col_ids_dev,
                                      const void* req_dev, void* best_id_dev, void* best_acc_dev);

/* ---- TrainingBackend::train batches: marginal-gain probes ------------------
 * Batch description = TrainingBatchStats (accuracy_model.hpp:50-56) with the
 * source_mix flattened to CSR (cameras in std::map order). */
typedef struct {
  double delivered_frame_rate;
  double resolution;
  double quality_factor;
} ecco_batch;

/* Speculative trajectories: for every job, from its committed model,
 *   acc[j][0] = evaluate(j); for t = 1..depth: train(j, gpu_s); acc[j][t] =
 *   evaluate(j)
 * exactly as WindowAllocation::run_micro (gpu_allocator.cpp:125-135) would
 * observe them.  `micro_base[j]` is the job's count of already committed
 * micro-windows this window (keys the learned sampler; nullable = 0).  The
 * model after every step is kept as a snapshot (depth <= max_depth) for
 * ecco_commit.  Chains always start from the committed model: a caller that
 * needs a longer chain for a job commits the granted prefix and asks again
 * (the host replay only runs out of a chain when all of it was granted). */
ecco_status ecco_train_trajectories(
    ecco_ctx* ctx, int n_jobs, const int* job_ids, const ecco_batch* batches,
    const int* src_offsets /* n_jobs+1 */, const int* src_cams, const double* src_fracs,
    const int* member_offsets /* n_jobs+1 */, const int* member_cams,
    const int* micro_base, int window, double gpu_seconds, int depth,
    double* out_acc /* n_jobs*(depth+1) */);

/* Sampled-row variant of the staged ingest (the e2e path): the SGD draws of
 * the NEXT ecco_train_trajectories call (same job / batch / source-mix /
 * micro_base / window / gpu_s / depth arguments) are marked on the device,
 * and only those ring rows are read from `frames` (the full
 * [n_cams][R][F] table, which must be PINNED host memory: the copy stream
 * reads it zero-copy over PCIe) into the back buffer; all labels and the
 * first n_eval cameras' eval sets are copied as in ecco_stage_frames.  Rows
 * the trajectories never draw are not transferred (their back-buffer slots
 * are stale), so the trajectories' results equal a full upload's; once the
 * rings are current, a ecco_train_trajectories call that would draw an
 * unstaged row fails with ECCO_ERR_LOGIC (ecco_fetch_sampled_frames tops
 * them up).  Counts
 * the rows read into ecco_transfer_bytes.  The fetch runs as two CTAs
 * beside the window's kernels (the CTA-pair evaluation kernel schedules its
 * tiles dynamically around them).  Replaces, for the
 * learned path, the per-window frame delivery the reference models as
 * TrainingBatchStats (accuracy_model.hpp:36-44). */
ecco_status ecco_stage_sampled_frames(ecco_ctx* ctx, int n_jobs, const int* job_ids,
                                      const ecco_batch* batches, const int* src_off,
                                      const int* src_cams, const double* src_fracs,
                                      const int* micro_base, int window, double gpu_s, int depth,
                                      const uint16_t* frames, const int32_t* labels, int n_eval,
                                      const uint16_t* eval_frames, const int32_t* eval_labels);
/* Top-up of a sampled ingest: when the CURRENT rings came from
 * ecco_stage_sampled_frames (only the rows its trajectories draw), reads the
 * rows that THESE trajectories arguments draw and the rings lack from the
 * same pinned [n_cams][R][F] table, zero-copy, into the current rings
 * (stream-ordered on the context stream; returns after the fetch).  For
 * chains the caller did not foresee at staging time -- e.g. a chain the
 * allocator replay exhausts and extends (micro_base = micro-windows already
 * committed; depth may exceed max_depth -- up to 65535 micro-windows -- to
 * fetch the rows of chains that will follow).  A no-op when the current
 * rings are complete (generated,
 * uploaded or staged whole).  ecco_train_trajectories itself checks, when
 * the current rings are partial, that every row it draws was staged or
 * fetched, and fails with ECCO_ERR_LOGIC otherwise (no silent stale rows). */
ecco_status ecco_fetch_sampled_frames(ecco_ctx* ctx, int n_jobs, const int* job_ids,
                                      const ecco_batch* batches, const int* src_off,
                                      const int* src_cams, const double* src_fracs,
                                      const int* micro_base, int window, double gpu_s, int depth,
                                      const uint16_t* frames);
/* Makes the snapshot after granted[j] steps of the last chain (0 = keep the
 * committed model) the committed model. */
ecco_status ecco_commit(ecco_ctx* ctx, int n_jobs, const int* job_ids, const int* granted);
/* Learned backend: mean minibatch loss of the last speculative chain per step
 * (diagnostics; n_jobs*depth floats, NaN where no step ran). */
ecco_status ecco_last_losses(ecco_ctx* ctx, int n_jobs, const int* job_ids, int depth,
                             float* out);
/* Sample indices the learned sampler draws for one (job, micro, step):
 * out_cam/out_frame[B].  Exposed for the bit-exactness tests. */
ecco_status ecco_sample_indices(ecco_ctx* ctx, int job_id, int n_src, const int* src_cams,
                                const double* src_fracs, int window, int micro, int step,
                                int* out_cam, int* out_frame);

/* ---- ProbeFn batch: offline profile tables ---------------------------------
 * build_profile_table (transmission.cpp:52-100) with make_accuracy_probe
 * (transmission.cpp:102-118) for every camera in one launch, including the
 * tie_epsilon / bias tie-break.  bias[i]: 0 resolution, 1 frame_rate.
 * Outputs n_cams*n_levels rows in ascending budget order. */
ecco_status ecco_profile_tables(ecco_ctx* ctx, int n_cams, const int* cam_idx,
                                const int* bias, int n_levels, const double* levels,
                                int n_grid, const double* grid_fps, const double* grid_res,
                                double window_s, double tie_eps, double ref_rate_bps,
                                double bpp_ref, double* out_budget, double* out_fps,
                                double* out_res, uint8_t* out_feasible);

/* ---- whole-window driver (Simulation::step_window, orchestrator.cpp:211-413)
 * A host C++ restatement of the reference control loop that calls the
 * batched entry points above.  Scenario JSON follows proj/README.md:107-169. */
typedef struct ecco_sim ecco_sim;
typedef struct {
  int backend;         /* ecco_backend */
  int math;            /* ecco_math (learned) */
  int device;
  int spec_depth;      /* initial speculative depth for run_remaining */
  int feat_dim, hidden_dim, num_classes, minibatch, ring_frames, eval_samples;
  float sgd_lr;
  double steps_per_gpu_s;
  uint64_t seed;
  int host_frames;     /* learned: generate frames on the host and upload (e2e) */
  int full_matrix;     /* evaluate the dense camera x group matrix every routing pass */
} ecco_sim_options;
void ecco_sim_default_options(ecco_sim_options* opt);
ecco_status ecco_sim_create(const char* scenario_json, const ecco_sim_options* opt,
                            ecco_sim** out, char* err, size_t err_len);
void ecco_sim_destroy(ecco_sim* sim);
const char* ecco_sim_last_error(const ecco_sim* sim);
/* Returns 1 when a window ran, 0 when all windows have run. */
ecco_status ecco_sim_step_window(ecco_sim* sim, int* ran);
/* Timings of the last window in milliseconds: [0] whole window, [1] regroup
 * (window-end eval + update_grouping + reroute + next routing), [2] train
 * phase, [3] eval matrix, [4] host decision replay. */
ecco_status ecco_sim_last_timings(const ecco_sim* sim, double* out5);
/* Samples trained in the last window (sum over granted micro-windows). */
int64_t ecco_sim_last_samples(const ecco_sim* sim);
/* trace.csv / summary.json bytes (metrics.cpp:49-59, orchestrator.cpp:420-459).
 * Returns the required size; copies at most cap bytes. */
size_t ecco_sim_trace_csv(const ecco_sim* sim, char* buf, size_t cap);
size_t ecco_sim_summary_json(const ecco_sim* sim, char* buf, size_t cap);
ecco_ctx* ecco_sim_context(ecco_sim* sim);
/* Timings of the last window, up to n of: the five of ecco_sim_last_timings,
 * [5] netsim (simulate_window), [6] profile tables (first use of cameras),
 * [7] drift events, [8] routing of pending requests, [9] shares + config
 * selection + batch assembly (netsim and profiles excluded), [10] end-of-
 * window rows and statistics.  Returns the number written. */
int ecco_sim_last_timings_ex(const ecco_sim* sim, double* out, int n);

/* ---- allocator decisions (host, no device) --------------------------------
 * WindowAllocation (core/src/gpu_allocator.cpp:100-181: initial pass in job-id
 * order, then greedy pick_next / round robin until the micro-window budget is
 * spent) driven by fixed per-job accuracy trajectories -- the decision replay
 * the window driver runs on the device's speculative trajectories (SURVEY.md
 * H4/H8).  traj: n_jobs rows of traj_len accuracies in job_ids order (a job
 * trained i times reads traj[min(i, traj_len-1)]).  policy 0 ecco, 1 naive,
 * 2 total_acc_greedy.  Writes micro_windows records (job, acc before, after)
 * and, unless naive, the initial scores in ascending job id.  Errors as the
 * reference: invalid config -> ECCO_ERR_INVALID_ARGUMENT, no jobs or more
 * jobs than micro-windows -> ECCO_ERR_INFEASIBLE. */
ecco_status ecco_allocate_trajectories(int n_jobs, const int* job_ids, const int* members,
                                       const double* traj, int traj_len, double alpha, double beta,
                                       int micro_windows, double micro_s, int gpu_count, int bonus,
                                       int policy, int* out_job, double* out_before,
                                       double* out_after, double* out_initial_scores);

/* ---- network model (host, no device) ---------------------------------------
 * simulate_window's per-flow mean rates (core/src/netsim.cpp:64-94 with
 * aimd_step :45-62; replaces ecco::simulate_window's mean_rate_bps for the
 * window driver): n flows with additive increase alpha
 * (bits/s per RTT, > 0), decrease factor beta (in (0,1)) and local cap (<= 0
 * = uncapped, resolve_caps :33-40) over one shared bottleneck of `capacity`,
 * from zero rates for llround(duration_s / rtt_s) steps; mean over the
 * second half.  Bit-identical to the reference; `exact_steps` (optional)
 * receives how many steps needed the reference's sequential congestion sum.
 * Invalid arguments -> ECCO_ERR_INVALID_ARGUMENT (netsim.cpp:17-31). */
ecco_status ecco_netsim_mean_rates(int n, const double* alpha, const double* beta,
                                   const double* caps, double capacity, double rtt_s,
                                   double duration_s, double* mean_rates, int* exact_steps);

#ifdef __cplusplus
}
#endif

#endif /* ECCO_B200_H_ */
