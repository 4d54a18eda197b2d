// C-ABI of include/ecco_b200.h: argument validation with the reference's
// error semantics, host <-> device staging, and dispatch to the parametric
// (param_kernels.cu) or learned (learned_kernels.cu, tc_kernels.cu) backend.
#include <cstring>
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <optional>
#include <string>
#include <vector>

#include <cuda.h>

#include "ctx.cuh"

namespace {

// The message of the last failed ecco_create on this thread (there is no
// context to hold it): ecco_last_error(nullptr) returns it.
thread_local std::string g_create_error = "no context";

// The device address of pinned (mapped) host memory, nullptr for pageable
// memory -- asked of the pointer's attributes, so a refused pointer raises
// no CUDA API error (cudaHostGetDevicePointer would).
static void* mapped_device_ptr(const void* host) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// Makes the context's device current for the call and restores the caller's
// current device afterwards (several contexts on different GPUs in one
// process must not move the calling thread's device, e.g. torch's).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) (void)cudaGetLastError();
    if (cur != dev) {
      ECCO_CUDA(cudaSetDevice(dev));
      prev = cur;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class F>
ecco_status guarded(ecco_ctx* ctx, F&& f) {
  try {
    // every call runs on the context's device, whatever the calling thread
    // had current (several contexts on different GPUs in one process)
    std::optional<DeviceGuard> dg;
    if (ctx) dg.emplace(ctx->cfg.device);
    f();
    return ECCO_OK;
  } catch (const EccoError& e) {
    if (ctx) ctx->err = e.msg;
    (void)cudaGetLastError();  // a non-sticky CUDA error must not surface in the next call
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    (void)cudaGetLastError();
    return ECCO_ERR_RUNTIME;
  }
}

void free_all(ecco_ctx* c) {
  void* ptrs[] = {c->d_scenes, c->d_tp,     c->d_exp_tab, c->d_k,       c->d_clen,
                  c->d_cl,     c->d_prof,   c->d_cen,     c->d_sk,      c->d_sclen,
                  c->d_scl,    c->d_sprof,  c->d_scen,    c->d_status,  c->d_w,
                  c->d_wspec,  c->d_proto_p, c->d_proto_q, c->d_frames, c->d_labels,
                  c->d_eval,   c->d_eval_labels, c->d_losses, c->b_frames, c->b_labels,
                  c->b_eval,   c->b_eval_labels, c->d_zc_rows};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  fused::free_shadow(c->sh_commit);
  fused::free_shadow(c->sh_spec);
  fused::free_shadow(c->sh_spec2);
  fused::free_shadow(c->sh_pool);
  if (c->eval_stream) cudaStreamDestroy(c->eval_stream);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_chain[i]) cudaEventDestroy(c->ev_chain[i]);
    if (c->ev_eval[i]) cudaEventDestroy(c->ev_eval[i]);
  }
  delete (CUtensorMap*)c->map_x;
  for (auto& b : c->scratch) b.release();
  for (auto& b : c->train_scratch) b.release();
  for (auto& b : c->hscratch) b.release();
  for (auto& b : c->zc_args) b.release();
  c->zc_host.release();
  if (c->zc_host_free) cudaEventDestroy(c->zc_host_free);
  for (auto& b : c->traj_args) b.release();
  for (auto& b : c->em_args) b.release();
  c->tile_ctr.release();
  c->zc_flags.release();
  c->zc_flags_front.release();
  c->zc_topup.release();
  c->zc_missing.release();
  for (auto& b : c->commit_args) b.release();
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->copy_stream2) cudaStreamDestroy(c->copy_stream2);
  for (auto& b : c->side_scratch) b.release();
  for (auto& b : c->side_em_args) b.release();
  c->side_tile_ctr.release();
  if (c->matrix_stream) cudaStreamDestroy(c->matrix_stream);
  if (c->ev_matrix_in) cudaEventDestroy(c->ev_matrix_in);
  if (c->ev_matrix_done) cudaEventDestroy(c->ev_matrix_done);
  for (int i = 0; i < 2; ++i) {
    if (c->copy_done[i]) cudaEventDestroy(c->copy_done[i]);
    if (c->back_free[i]) cudaEventDestroy(c->back_free[i]);
  }
  if (c->stream) cudaStreamDestroy(c->stream);
}

// Zero-initialised device allocation.  The zeroing must be complete before
// any stream touches the buffer: the context's streams are non-blocking, so a
// legacy-stream cudaMemset (asynchronous with respect to the host) would NOT
// be ordered before their kernels -- a kernel could write the buffer (e.g.
// seed a model into d_w) and the late memset zero it again.  So: memset on
// the legacy stream and wait for it.
template <class T>
void dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  ECCO_CUDA(cudaMalloc((void**)p, n * sizeof(T)));
  ECCO_CUDA(cudaMemset(*p, 0, n * sizeof(T)));
  ECCO_CUDA(cudaStreamSynchronize(0));
}

bool learned(const ecco_ctx* c) { return c->cfg.backend == ECCO_BACKEND_LEARNED; }

// pixels_per_frame (types.cpp:11-13) and train_step's effort
// (accuracy_model.cpp:82-86); host copy used to plan learned SGD step counts.
double host_ppf(double q) { return q * (16.0 * q / 9.0); }

int learned_steps(const ecco_ctx* c, const ecco_batch& b, double gpu_s, int n_src,
                  const int* src_cam) {
  if (n_src <= 0) return 0;
  const double supplied = b.delivered_frame_rate * host_ppf(b.resolution);
  double sum = 0.0;
  for (int i = 0; i < n_src; ++i) sum += c->h_tp[src_cam[i]];
  const double required = sum / (double)n_src;
  const double suff = required > 0.0 ? std::min(1.0, supplied / required) : 1.0;
  const double effort = gpu_s * suff * b.quality_factor;
  if (effort <= 0.0) return 0;
  return (int)std::floor(effort * c->cfg.steps_per_gpu_s);
}

// train_step's input validation (accuracy_model.cpp:73-81), done on the host
// once per job before any device work.
void validate_batch(const ecco_ctx* c, int j, double gpu_s, int n_src, const int* src_cam,
                    const double* frac) {
  if (gpu_s < 0.0) ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "train_step: negative gpu_time");
  double total = 0.0;
  for (int i = 0; i < n_src; ++i) {
    if (frac[i] < 0.0)
      ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "train_step: negative source_mix fraction");
    total += frac[i];
  }
  if (n_src > 0 && std::abs(total - 1.0) > 1e-9)
    ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "train_step: source_mix fractions must sum to 1");
  for (int i = 0; i < n_src; ++i)
    if (src_cam[i] < 0 || src_cam[i] >= c->n_cams)
      ecco_throw(ECCO_ERR_INVALID_ARGUMENT,
                 "train_step: source_mix camera missing (job row " + std::to_string(j) + ")");
}

void check_cams(const ecco_ctx* c, int n, const int* cams, const char* what) {
  for (int i = 0; i < n; ++i)
    if (cams[i] < 0 || cams[i] >= c->n_cams)
      ecco_throw(ECCO_ERR_INVALID_ARGUMENT, std::string(what) + ": camera index out of range");
}

std::vector<int> slots_of(ecco_ctx* c, int n, const int* job_ids) {
  std::vector<int> s(n);
  for (int i = 0; i < n; ++i) s[i] = c->slot(job_ids[i]);
  return s;
}

}  // namespace

void ecco_ctx::check_device_status() {
  int st = 0;
  ECCO_CUDA(ctx_memcpy(this, &st, d_status, sizeof(int), cudaMemcpyDeviceToHost, stream));
  ECCO_CUDA(cudaStreamSynchronize(stream));
  if (st) {
    ECCO_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int), stream));
    if (st == 2) ecco_throw(ECCO_ERR_RUNTIME, "model cluster capacity (max_clusters) exceeded");
    ecco_throw(ECCO_ERR_RUNTIME, "device status " + std::to_string(st));
  }
}

extern "C" {

void ecco_default_config(ecco_config* c) {
  memset(c, 0, sizeof(*c));
  c->backend = ECCO_BACKEND_PARAMETRIC;
  c->device = 0;
  c->scene_dims = 2;
  c->max_clusters = 16;
  c->max_jobs = 1024;
  c->max_cameras = 16384;
  c->params = {0.05, 0.5, 0.1, 0.6, 0.9};
  c->math = ECCO_MATH_FFMA_EXACT;
  c->feat_dim = 512;
  c->hidden_dim = 256;
  c->num_classes = 16;
  c->minibatch = 128;
  c->ring_frames = 512;
  c->eval_samples = 64;
  c->max_depth = 8;
  c->sgd_lr = 0.05f;
  c->feature_noise = 1.0f;
  c->steps_per_gpu_s = 4.0;
  c->seed = 0x5eed0001ULL;
}

ecco_status ecco_create(const ecco_config* cfg, ecco_ctx** out) {
  *out = nullptr;
  ecco_ctx* c = new ecco_ctx();
  c->cfg = *cfg;
  const ecco_status st = guarded(c, [&] {
    const ecco_config& g = c->cfg;
    ECCO_REQUIRE(g.scene_dims >= 1 && g.scene_dims <= 8, "scene_dims must be in [1, 8]");
    ECCO_REQUIRE(g.max_clusters >= 1 && g.max_clusters <= 32, "max_clusters must be in [1, 32]");
    ECCO_REQUIRE(g.max_jobs >= 1 && g.max_cameras >= 1, "max_jobs/max_cameras must be positive");
    ECCO_REQUIRE(g.max_depth >= 1 && g.max_depth <= 64, "max_depth must be in [1, 64]");
    ECCO_REQUIRE(g.params.similarity_lambda > 0.0, "similarity: lambda must be positive");
    if (g.backend == ECCO_BACKEND_LEARNED) {
      ECCO_REQUIRE(g.feat_dim % 64 == 0 && g.feat_dim > 0, "feat_dim must be a multiple of 64");
      ECCO_REQUIRE(g.hidden_dim % 128 == 0 && g.hidden_dim > 0, "hidden_dim must be a multiple of 128");
      ECCO_REQUIRE(g.num_classes % 4 == 0 && g.num_classes >= 4 && g.num_classes <= 256,
                   "num_classes must be a multiple of 4 in [4, 256]");
      ECCO_REQUIRE(g.minibatch % 64 == 0 && g.minibatch > 0, "minibatch must be a multiple of 64");
      ECCO_REQUIRE(g.eval_samples % 64 == 0 && g.eval_samples > 0,
                   "eval_samples must be a multiple of 64");
      ECCO_REQUIRE(g.ring_frames > 0, "ring_frames must be positive");
      ECCO_REQUIRE(g.math == ECCO_MATH_FFMA_EXACT || g.math == ECCO_MATH_TC_BF16, "unknown math");
    }
    ECCO_CUDA(cudaSetDevice(g.device));
    ECCO_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    const int D = g.scene_dims, K = g.max_clusters, S = g.max_jobs, T = g.max_depth + 1;
    dalloc(&c->d_scenes, (size_t)g.max_cameras * D);
    dalloc(&c->d_tp, (size_t)g.max_cameras);
    dalloc(&c->d_status, 1);
    dalloc(&c->d_k, S);
    dalloc(&c->d_clen, S);
    for (int s = g.max_jobs - 1; s >= 0; --s) c->free_slots.push_back(s);
    if (g.backend == ECCO_BACKEND_PARAMETRIC) {
      dalloc(&c->d_cl, (size_t)S * K * D);
      dalloc(&c->d_prof, (size_t)S * K);
      dalloc(&c->d_cen, (size_t)S * D);
      dalloc(&c->d_sk, (size_t)S * T);
      dalloc(&c->d_sclen, (size_t)S * T);
      dalloc(&c->d_scl, (size_t)S * T * K * D);
      dalloc(&c->d_sprof, (size_t)S * T * K);
      dalloc(&c->d_scen, (size_t)S * T * D);
    } else {
      const size_t F = g.feat_dim, H = g.hidden_dim, C = g.num_classes;
      c->n_params = F * H + H + H * C + C;
      dalloc(&c->d_w, (size_t)S * c->n_params);
      dalloc(&c->d_wspec, (size_t)S * g.max_depth * c->n_params);
      dalloc(&c->d_losses, (size_t)S * g.max_depth);
      dalloc(&c->d_proto_p, C * F);
      dalloc(&c->d_proto_q, C * D * F);
      dalloc(&c->d_frames, (size_t)g.max_cameras * g.ring_frames * F);
      dalloc(&c->d_labels, (size_t)g.max_cameras * g.ring_frames);
      dalloc(&c->d_eval, (size_t)g.max_cameras * g.eval_samples * F);
      dalloc(&c->d_eval_labels, (size_t)g.max_cameras * g.eval_samples);
      lbackend::init(c);
    }
    ECCO_CUDA(cudaStreamSynchronize(c->stream));
  });
  if (st != ECCO_OK) {
    g_create_error = c->err;
    free_all(c);
    delete c;
    return st;
  }
  *out = c;
  return ECCO_OK;
}

void ecco_destroy(ecco_ctx* ctx) {
  if (!ctx) return;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_all(ctx);
  delete ctx;
  if (prev >= 0) cudaSetDevice(prev);
}

const char* ecco_last_error(const ecco_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

uint64_t ecco_kernel_launches(const ecco_ctx* ctx) { return ctx ? ctx->launches : 0; }

void* ecco_stream(ecco_ctx* ctx) { return (void*)ctx->stream; }

ecco_status ecco_profile(ecco_ctx* ctx, int enable) {
  return guarded(ctx, [&] {
    ctx->fold_stats();
    if (enable)
      for (auto& k : ctx->kstats) k.launches = 0, k.ms = k.flops = k.bytes = 0.0;
    ctx->profiling = enable != 0;
  });
}

ecco_status ecco_kernel_stat(ecco_ctx* ctx, int which, uint64_t* launches, double* ms,
                             double* flops, double* bytes) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(which >= 0 && which < ECCO_KSTAT_COUNT, "kernel_stat: unknown kernel family");
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->fold_stats();
    const KStat& k = ctx->kstats[which];
    *launches = k.launches;
    *ms = k.ms;
    *flops = k.flops;
    *bytes = k.bytes;
  });
}

ecco_status ecco_transfer_bytes(const ecco_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
  *h2d = ctx->h2d_bytes;
  *d2h = ctx->d2h_bytes;
  if (ctx->d_zc_rows) {  // + rows read from pinned host memory by the sampled-row fetch
    unsigned long long n = 0;
    if (cudaStreamSynchronize(ctx->copy_stream) != cudaSuccess ||
        (ctx->copy_stream2 && cudaStreamSynchronize(ctx->copy_stream2) != cudaSuccess) ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess ||  // (top-up fetches)
        cudaMemcpy(&n, ctx->d_zc_rows, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess)
      return ECCO_ERR_CUDA;
    *h2d += n * (uint64_t)ctx->cfg.feat_dim * 2;
  }
  return ECCO_OK;
}

ecco_status ecco_synchronize(ecco_ctx* ctx) {
  return guarded(ctx, [&] { ECCO_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

ecco_status ecco_set_cameras(ecco_ctx* ctx, int n, const double* scenes, const double* tp) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(n >= 0 && n <= ctx->cfg.max_cameras, "camera count exceeds max_cameras");
    const int D = ctx->cfg.scene_dims;
    ctx->n_cams = n;
    ctx->h_scenes.assign(scenes, scenes + (size_t)n * D);
    ctx->h_tp.assign(tp, tp + n);
    if (n == 0) return;
    ECCO_CUDA(ctx_memcpy(ctx, ctx->d_scenes, scenes, sizeof(double) * n * D, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, ctx->d_tp, tp, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_update_scenes(ecco_ctx* ctx, int n, const int* cam_idx, const double* scenes) {
  return guarded(ctx, [&] {
    check_cams(ctx, n, cam_idx, "update_scenes");
    const int D = ctx->cfg.scene_dims;
    for (int i = 0; i < n; ++i) {
      std::copy(scenes + (size_t)i * D, scenes + (size_t)(i + 1) * D,
                ctx->h_scenes.begin() + (size_t)cam_idx[i] * D);
      ECCO_CUDA(ctx_memcpy(ctx, ctx->d_scenes + (size_t)cam_idx[i] * D, scenes + (size_t)i * D,
                                sizeof(double) * D, cudaMemcpyHostToDevice, ctx->stream));
    }
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_generate_frames(ecco_ctx* ctx, int window) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "generate_frames: learned backend only");
    lbackend::generate_frames(ctx, window);
    ctx->ring_partial = false;
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

static void upload_frames_impl(ecco_ctx* ctx, int n, const void* frames, const void* labels,
                               const void* eval, const void* eval_labels, cudaMemcpyKind kind) {
  ECCO_REQUIRE(learned(ctx), "upload_frames: learned backend only");
  ECCO_REQUIRE(n >= 0 && n <= ctx->n_cams, "upload_frames: camera count");
  const ecco_config& g = ctx->cfg;
  const size_t fr = (size_t)n * g.ring_frames, ev = (size_t)n * g.eval_samples;
  ECCO_CUDA(ctx_memcpy(ctx, ctx->d_frames, frames, fr * g.feat_dim * 2, kind, ctx->stream));
  ECCO_CUDA(ctx_memcpy(ctx, ctx->d_labels, labels, fr * 4, kind, ctx->stream));
  ECCO_CUDA(ctx_memcpy(ctx, ctx->d_eval, eval, ev * g.feat_dim * 2, kind, ctx->stream));
  ECCO_CUDA(ctx_memcpy(ctx, ctx->d_eval_labels, eval_labels, ev * 4, kind, ctx->stream));
  ctx->ring_partial = false;
}

ecco_status ecco_upload_frames(ecco_ctx* ctx, int n, const uint16_t* frames, const int32_t* labels,
                               const uint16_t* eval, const int32_t* eval_labels) {
  return guarded(ctx, [&] {
    upload_frames_impl(ctx, n, frames, labels, eval, eval_labels, cudaMemcpyHostToDevice);
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_stage_frames(ecco_ctx* ctx, int n, const uint16_t* frames, const int32_t* labels,
                              const uint16_t* eval, const int32_t* eval_labels) {
  return ecco_stage_frames_range(ctx, 0, n, frames, labels, n, eval, eval_labels);
}

// Back buffers + copy stream of the double-buffered ingest (first use); the
// copy stream then waits until kernels of the previous window stop reading
// the back buffers of the parts about to be staged (bit 0 rings, bit 1 eval).
void open_back_buffers(ecco_ctx* ctx, int parts) {
  const ecco_config& g = ctx->cfg;
  if (!ctx->copy_stream) {
    ECCO_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    ECCO_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream2, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      ECCO_CUDA(cudaEventCreateWithFlags(&ctx->copy_done[i], cudaEventDisableTiming));
      ECCO_CUDA(cudaEventCreateWithFlags(&ctx->back_free[i], cudaEventDisableTiming));
    }
    const size_t fr = (size_t)g.max_cameras * g.ring_frames, ev = (size_t)g.max_cameras * g.eval_samples;
    dalloc(&ctx->b_frames, fr * g.feat_dim);
    dalloc(&ctx->b_labels, fr);
    dalloc(&ctx->b_eval, ev * g.feat_dim);
    dalloc(&ctx->b_eval_labels, ev);
  }
  for (int i = 0; i < 2; ++i) {
    if (!((parts >> i) & 1)) continue;
    ECCO_REQUIRE(!ctx->staged[i], i == 0 ? "stage_frames: staged rings not swapped in yet"
                                         : "stage_frames: staged eval sets not swapped in yet");
    if (ctx->back_busy[i]) ECCO_CUDA(cudaStreamWaitEvent(ctx->part_stream(i), ctx->back_free[i], 0));
  }
}

// Marks `parts` staged once the copies enqueued so far on the copy stream land.
void staged_parts(ecco_ctx* ctx, int parts) {
  for (int i = 0; i < 2; ++i)
    if ((parts >> i) & 1) {
      ECCO_CUDA(cudaEventRecord(ctx->copy_done[i], ctx->part_stream(i)));
      ctx->staged[i] = true;
    }
}

ecco_status ecco_stage_frames_range(ecco_ctx* ctx, int first, int n, const uint16_t* frames,
                                    const int32_t* labels, int n_eval, const uint16_t* eval,
                                    const int32_t* eval_labels) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "stage_frames: learned backend only");
    ECCO_REQUIRE(first >= 0 && n >= 0 && first + n <= ctx->n_cams, "stage_frames: camera range");
    ECCO_REQUIRE(n_eval >= 0 && n_eval <= ctx->n_cams, "stage_frames: eval camera count");
    const ecco_config& g = ctx->cfg;
    const int parts = (n > 0 || n_eval == 0 ? 1 : 0) | (n_eval > 0 ? 2 : 0);
    open_back_buffers(ctx, parts);
    const size_t fr = (size_t)n * g.ring_frames, ev = (size_t)n_eval * g.eval_samples;
    const size_t f0 = (size_t)first * g.ring_frames;
    const cudaMemcpyKind k = cudaMemcpyHostToDevice;
    ECCO_CUDA(ctx_memcpy(ctx, ctx->b_frames + f0 * g.feat_dim, frames, fr * g.feat_dim * 2, k,
                         ctx->copy_stream));
    ECCO_CUDA(ctx_memcpy(ctx, ctx->b_labels + f0, labels, fr * 4, k, ctx->copy_stream));
    ECCO_CUDA(ctx_memcpy(ctx, ctx->b_eval, eval, ev * g.feat_dim * 2, k, ctx->copy_stream2));
    ECCO_CUDA(ctx_memcpy(ctx, ctx->b_eval_labels, eval_labels, ev * 4, k, ctx->copy_stream2));
    staged_parts(ctx, parts);
    if (parts & 1) ctx->back_partial = false;  // whole rings (of the caller's range)
  });
}

ecco_status ecco_reserve_ingest(ecco_ctx* ctx) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "reserve_ingest: learned backend only");
    open_back_buffers(ctx, 0);  // the back buffers, copy stream and events
    if (!ctx->d_zc_rows) dalloc(&ctx->d_zc_rows, 1);
    const size_t rows = (size_t)ctx->cfg.max_cameras * ctx->cfg.ring_frames;
    ctx->zc_flags.get((rows + 31) / 32 * 4);
    ctx->zc_host.get(4096);
    ECCO_CUDA(cudaDeviceSynchronize());
  });
}

ecco_status ecco_stage_sampled_frames(ecco_ctx* ctx, int n_jobs, const int* job_ids,
                                      const ecco_batch* batches, const int* src_off,
                                      const int* src_cams, const double* src_fracs,
                                      const int* micro_base, int window, double gpu_s, int depth,
                                      const uint16_t* frames, const int32_t* labels, int n_eval,
                                      const uint16_t* eval, const int32_t* eval_labels) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "stage_sampled_frames: learned backend only");
    ECCO_REQUIRE(n_jobs >= 0 && depth >= 1 && depth <= ctx->cfg.max_depth,
                 "stage_sampled_frames: depth must be in [1, max_depth]");
    ECCO_REQUIRE(n_eval >= 0 && n_eval <= ctx->n_cams, "stage_sampled_frames: eval camera count");
    ECCO_REQUIRE(n_jobs == 0 || src_off[0] == 0, "CSR offsets must start at 0");
    for (int j = 0; j < n_jobs; ++j)
      validate_batch(ctx, j, gpu_s, src_off[j + 1] - src_off[j], src_cams + src_off[j],
                     src_fracs + src_off[j]);
    const ecco_config& g = ctx->cfg;
    void* fdev = nullptr;  // the device address of the pinned ring table
    fdev = mapped_device_ptr(frames);
    ECCO_REQUIRE(fdev != nullptr, "stage_sampled_frames: frames must be pinned (mapped) host memory");
    const int parts = 1 | (n_eval > 0 ? 2 : 0);
    open_back_buffers(ctx, parts);
    cudaStream_t st = ctx->copy_stream;
    if (!ctx->d_zc_rows) {
      dalloc(&ctx->d_zc_rows, 1);
      ECCO_CUDA(cudaDeviceSynchronize());
    }
    const cudaMemcpyKind k = cudaMemcpyHostToDevice;
    const size_t rows = (size_t)ctx->n_cams * g.ring_frames, words = (rows + 31) / 32;
    uint32_t* flags = (uint32_t*)ctx->zc_flags.get(words * 4);
    ECCO_CUDA(cudaMemsetAsync(flags, 0, words * 4, st));
    if (n_jobs > 0) {
      std::vector<int> steps(n_jobs), mb(n_jobs, 0);
      int max_steps = 0;
      for (int j = 0; j < n_jobs; ++j) {
        steps[j] = learned_steps(ctx, batches[j], gpu_s, src_off[j + 1] - src_off[j],
                                 src_cams + src_off[j]);
        max_steps = std::max(max_steps, steps[j]);
      }
      if (micro_base) mb.assign(micro_base, micro_base + n_jobs);
      const size_t nsrc = std::max(src_off[n_jobs], 1);
      // the arguments go through a pinned buffer: a pageable copy would make
      // the host wait for the copy stream (which waits for the previous
      // window's kernels); the previous call's copies have long read it
      if (!ctx->zc_host_free)
        ECCO_CUDA(cudaEventCreateWithFlags(&ctx->zc_host_free, cudaEventDisableTiming));
      else
        ECCO_CUDA(cudaEventSynchronize(ctx->zc_host_free));
      const size_t words_i = 4 * (size_t)n_jobs + 1 + nsrc, bytes_h = words_i * 4 + nsrc * 8 + 64;
      uint8_t* hb = (uint8_t*)ctx->zc_host.get(bytes_h);
      size_t ho = 0;
      auto up = [&](int i, const void* h, size_t bytes) {
        void* d = ctx->zc_args[i].get(bytes);
        ho = (ho + 7) & ~(size_t)7;
        std::memcpy(hb + ho, h, bytes);
        ECCO_CUDA(ctx_memcpy(ctx, d, hb + ho, bytes, k, st));
        ho += bytes;
        return d;
      };
      const int* d_j = (const int*)up(0, job_ids, sizeof(int) * n_jobs);
      const int* d_st = (const int*)up(1, steps.data(), sizeof(int) * n_jobs);
      const int* d_so = (const int*)up(2, src_off, sizeof(int) * (n_jobs + 1));
      const int* d_sc = (const int*)up(3, src_cams, sizeof(int) * nsrc);
      const double* d_sf = (const double*)up(4, src_fracs, sizeof(double) * nsrc);
      const int* d_mb = (const int*)up(5, mb.data(), sizeof(int) * n_jobs);
      stage::mark_sampled(ctx, st, n_jobs, d_j, d_st, max_steps, d_so, d_sc, d_sf, d_mb, depth,
                          window, flags);
      ECCO_CUDA(cudaEventRecord(ctx->zc_host_free, st));
    }
    // (the CTA-pair evaluation kernel schedules its super tiles dynamically:
    // pairs that cannot start beside the fetch simply take fewer tiles)
    stage::fetch_rows(ctx, st, (const uint16_t*)fdev, ctx->b_frames, flags, words, ctx->d_zc_rows);
    ECCO_CUDA(ctx_memcpy(ctx, ctx->b_labels, labels, rows * 4, k, st));
    const size_t ev = (size_t)n_eval * g.eval_samples;
    ECCO_CUDA(ctx_memcpy(ctx, ctx->b_eval, eval, ev * g.feat_dim * 2, k, ctx->copy_stream2));
    ECCO_CUDA(ctx_memcpy(ctx, ctx->b_eval_labels, eval_labels, ev * 4, k, ctx->copy_stream2));
    staged_parts(ctx, parts);
    ctx->back_partial = true;  // only the drawn rows: zc_flags says which
  });
}

ecco_status ecco_fetch_sampled_frames(ecco_ctx* ctx, int n_jobs, const int* job_ids,
                                      const ecco_batch* batches, const int* src_off,
                                      const int* src_cams, const double* src_fracs,
                                      const int* micro_base, int window, double gpu_s, int depth,
                                      const uint16_t* frames) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "fetch_sampled_frames: learned backend only");
    // (depth only bounds the draws marked: a caller may fetch ahead of the
    // chains it will run, e.g. a group's whole remaining budget at once)
    ECCO_REQUIRE(n_jobs >= 0 && depth >= 1 && depth <= 65535,
                 "fetch_sampled_frames: depth must be in [1, 65535]");
    ECCO_REQUIRE(n_jobs == 0 || src_off[0] == 0, "CSR offsets must start at 0");
    for (int j = 0; j < n_jobs; ++j)
      validate_batch(ctx, j, gpu_s, src_off[j + 1] - src_off[j], src_cams + src_off[j],
                     src_fracs + src_off[j]);
    if (!ctx->ring_partial || n_jobs == 0) return;  // complete rings: nothing to fetch
    void* fdev = nullptr;
    fdev = mapped_device_ptr(frames);
    ECCO_REQUIRE(fdev != nullptr, "fetch_sampled_frames: frames must be pinned (mapped) host memory");
    const ecco_config& g = ctx->cfg;
    cudaStream_t st = ctx->stream;
    std::vector<int> steps(n_jobs), mb(n_jobs, 0);
    int max_steps = 0;
    for (int j = 0; j < n_jobs; ++j) {
      steps[j] = learned_steps(ctx, batches[j], gpu_s, src_off[j + 1] - src_off[j],
                               src_cams + src_off[j]);
      max_steps = std::max(max_steps, steps[j]);
    }
    if (micro_base) mb.assign(micro_base, micro_base + n_jobs);
    const size_t nsrc = std::max(src_off[n_jobs], 1);
    DevBuf* b = ctx->traj_args;  // stream-ordered before the next trajectories' uploads
    auto up = [&](int i, const void* h, size_t bytes) {
      void* d = b[i].get(bytes);
      ECCO_CUDA(ctx_memcpy(ctx, d, h, bytes, cudaMemcpyHostToDevice, st));
      return d;
    };
    const int* d_j = (const int*)up(7, job_ids, sizeof(int) * n_jobs);
    const int* d_st = (const int*)up(9, steps.data(), sizeof(int) * n_jobs);
    const int* d_so = (const int*)up(1, src_off, sizeof(int) * (n_jobs + 1));
    const int* d_sc = (const int*)up(2, src_cams, sizeof(int) * nsrc);
    const double* d_sf = (const double*)up(3, src_fracs, sizeof(double) * nsrc);
    const int* d_mb = (const int*)up(8, mb.data(), sizeof(int) * n_jobs);
    const size_t rows = (size_t)ctx->n_cams * g.ring_frames, words = (rows + 31) / 32;
    uint32_t* want = (uint32_t*)ctx->zc_topup.get(words * 4);
    ECCO_CUDA(cudaMemsetAsync(want, 0, words * 4, st));
    stage::mark_sampled(ctx, st, n_jobs, d_j, d_st, max_steps, d_so, d_sc, d_sf, d_mb, depth,
                        window, want);
    if (!ctx->d_zc_rows) dalloc(&ctx->d_zc_rows, 1);
    stage::fetch_rows(ctx, st, (const uint16_t*)fdev, ctx->d_frames, want, words, ctx->d_zc_rows,
                      (uint32_t*)ctx->zc_flags_front.p);
    ECCO_CUDA(cudaStreamSynchronize(st));  // the caller's arguments are host memory
  });
}

static void swap_parts(ecco_ctx* ctx, int parts) {
  for (int i = 0; i < 2; ++i) {
    if (!((parts >> i) & 1)) continue;
    ECCO_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->copy_done[i], 0));
    if (i == 0) {
      std::swap(ctx->d_frames, ctx->b_frames);
      std::swap(ctx->d_labels, ctx->b_labels);
      std::swap(ctx->zc_flags, ctx->zc_flags_front);
      ctx->ring_partial = ctx->back_partial;
      ctx->back_partial = false;
    } else {
      std::swap(ctx->d_eval, ctx->b_eval);
      std::swap(ctx->d_eval_labels, ctx->b_eval_labels);
      delete (CUtensorMap*)ctx->map_x;  // rebuilt over the new eval buffer on next use
      ctx->map_x = nullptr;
    }
    // kernels enqueued so far read the old front (now back): the next
    // staging copy of this part waits for them
    ECCO_CUDA(cudaEventRecord(ctx->back_free[i], ctx->stream));
    ctx->back_busy[i] = true;
    ctx->staged[i] = false;
  }
}

ecco_status ecco_swap_frames(ecco_ctx* ctx) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(ctx->staged[0] || ctx->staged[1], "swap_frames: nothing staged");
    swap_parts(ctx, (ctx->staged[0] ? 1 : 0) | (ctx->staged[1] ? 2 : 0));
  });
}

ecco_status ecco_swap_frame_parts(ecco_ctx* ctx, int parts) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(parts >= 1 && parts <= 3, "swap_frame_parts: parts is a mask of 1 (rings), 2 (eval)");
    ECCO_REQUIRE(!(parts & 1) || ctx->staged[0], "swap_frame_parts: rings not staged");
    ECCO_REQUIRE(!(parts & 2) || ctx->staged[1], "swap_frame_parts: eval sets not staged");
    swap_parts(ctx, parts);
  });
}

ecco_status ecco_read_frames(ecco_ctx* ctx, int n, uint16_t* frames, int32_t* labels,
                             uint16_t* eval, int32_t* eval_labels) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "read_frames: learned backend only");
    ECCO_REQUIRE(n >= 0 && n <= ctx->n_cams, "read_frames: camera count");
    const ecco_config& g = ctx->cfg;
    const size_t fr = (size_t)n * g.ring_frames, ev = (size_t)n * g.eval_samples;
    const cudaMemcpyKind k = cudaMemcpyDeviceToHost;
    if (frames) ECCO_CUDA(ctx_memcpy(ctx, frames, ctx->d_frames, fr * g.feat_dim * 2, k, ctx->stream));
    if (labels) ECCO_CUDA(ctx_memcpy(ctx, labels, ctx->d_labels, fr * 4, k, ctx->stream));
    if (eval) ECCO_CUDA(ctx_memcpy(ctx, eval, ctx->d_eval, ev * g.feat_dim * 2, k, ctx->stream));
    if (eval_labels) ECCO_CUDA(ctx_memcpy(ctx, eval_labels, ctx->d_eval_labels, ev * 4, k, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_upload_frames_dev(ecco_ctx* ctx, int n, const void* frames, const void* labels,
                                   const void* eval, const void* eval_labels) {
  return guarded(ctx, [&] {
    upload_frames_impl(ctx, n, frames, labels, eval, eval_labels, cudaMemcpyDeviceToDevice);
  });
}

ecco_status ecco_put_models(ecco_ctx* ctx, int n, const int* job_ids, const int* n_clusters,
                            const double* clusters, const double* prof, const double* centroid,
                            const int* centroid_len) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(!learned(ctx), "put_models: parametric backend only (use ecco_set_weights)");
    const int D = ctx->cfg.scene_dims, K = ctx->cfg.max_clusters;
    for (int i = 0; i < n; ++i) {
      ECCO_REQUIRE(n_clusters[i] >= 0 && n_clusters[i] <= K, "put_models: cluster count");
      ECCO_REQUIRE(centroid_len[i] == 0 || centroid_len[i] == D, "put_models: centroid length");
      const int s = ctx->alloc_slot(job_ids[i]);
      ECCO_CUDA(ctx_memcpy(ctx, ctx->d_cl + (size_t)s * K * D, clusters + (size_t)i * K * D,
                                sizeof(double) * K * D, cudaMemcpyHostToDevice, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, ctx->d_prof + (size_t)s * K, prof + (size_t)i * K, sizeof(double) * K,
                                cudaMemcpyHostToDevice, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, ctx->d_cen + (size_t)s * D, centroid + (size_t)i * D, sizeof(double) * D,
                                cudaMemcpyHostToDevice, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, ctx->d_k + s, n_clusters + i, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, ctx->d_clen + s, centroid_len + i, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    }
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_get_models(ecco_ctx* ctx, int n, const int* job_ids, int* n_clusters,
                            double* clusters, double* prof, double* centroid, int* centroid_len) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(!learned(ctx), "get_models: parametric backend only");
    const int D = ctx->cfg.scene_dims, K = ctx->cfg.max_clusters;
    for (int i = 0; i < n; ++i) {
      const int s = ctx->slot(job_ids[i]);
      ECCO_CUDA(ctx_memcpy(ctx, clusters + (size_t)i * K * D, ctx->d_cl + (size_t)s * K * D,
                                sizeof(double) * K * D, cudaMemcpyDeviceToHost, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, prof + (size_t)i * K, ctx->d_prof + (size_t)s * K, sizeof(double) * K,
                                cudaMemcpyDeviceToHost, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, centroid + (size_t)i * D, ctx->d_cen + (size_t)s * D, sizeof(double) * D,
                                cudaMemcpyDeviceToHost, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, n_clusters + i, ctx->d_k + s, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, centroid_len + i, ctx->d_clen + s, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    }
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_seed_models(ecco_ctx* ctx, int n, const int* job_ids, const double* scenes,
                             const double* device_acc) {
  return guarded(ctx, [&] {
    if (n == 0) return;
    std::vector<int> s(n);
    for (int i = 0; i < n; ++i) s[i] = ctx->alloc_slot(job_ids[i]);
    for (int i = 0; i < n; ++i) ctx->mark_dirty(s[i]);
    int* d_s = ctx->upload(0, s.data(), n);
    if (learned(ctx)) {
      int* d_j = ctx->upload(1, job_ids, n);
      lbackend::seed(ctx, n, job_ids, d_s, d_j);
    } else {
      double* d_sc = ctx->upload(1, scenes, (size_t)n * ctx->cfg.scene_dims);
      double* d_a = ctx->upload(2, device_acc, n);
      pbackend::seed(ctx, n, d_s, d_sc, d_a);
    }
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_drop_models(ecco_ctx* ctx, int n, const int* job_ids) {
  return guarded(ctx, [&] {
    for (int i = 0; i < n; ++i) {
      auto it = ctx->slot_of.find(job_ids[i]);
      if (it == ctx->slot_of.end()) continue;
      ctx->free_slots.push_back(it->second);
      ctx->slot_of.erase(it);
    }
  });
}

ecco_status ecco_get_weights(ecco_ctx* ctx, int job_id, float* w1, float* b1, float* w2, float* b2) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "get_weights: learned backend only");
    const ecco_config& g = ctx->cfg;
    const size_t F = g.feat_dim, H = g.hidden_dim, C = g.num_classes;
    const float* base = ctx->d_w + (size_t)ctx->slot(job_id) * ctx->n_params;
    std::vector<float> tmp(ctx->w1_t ? F * H : 0);
    ECCO_CUDA(ctx_memcpy(ctx, ctx->w1_t ? tmp.data() : w1, base, F * H * 4, cudaMemcpyDeviceToHost,
                         ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, b1, base + F * H, H * 4, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, w2, base + F * H + H, H * C * 4, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, b2, base + F * H + H + H * C, C * 4, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->w1_t)  // [H][F] -> API layout W1[F][H]
      for (size_t h = 0; h < H; ++h)
        for (size_t f = 0; f < F; ++f) w1[f * H + h] = tmp[h * F + f];
  });
}

ecco_status ecco_set_weights(ecco_ctx* ctx, int job_id, const float* w1, const float* b1,
                             const float* w2, const float* b2) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "set_weights: learned backend only");
    const ecco_config& g = ctx->cfg;
    const size_t F = g.feat_dim, H = g.hidden_dim, C = g.num_classes;
    const int slot = ctx->alloc_slot(job_id);
    ctx->mark_dirty(slot);
    float* base = ctx->d_w + (size_t)slot * ctx->n_params;
    std::vector<float> tmp;
    if (ctx->w1_t) {  // API layout W1[F][H] -> [H][F]
      tmp.resize(F * H);
      for (size_t f = 0; f < F; ++f)
        for (size_t h = 0; h < H; ++h) tmp[h * F + f] = w1[f * H + h];
      w1 = tmp.data();
    }
    ECCO_CUDA(ctx_memcpy(ctx, base, w1, F * H * 4, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, base + F * H, b1, H * 4, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, base + F * H + H, w2, H * C * 4, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, base + F * H + H + H * C, b2, C * 4, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_eval_jobs(ecco_ctx* ctx, int n_jobs, const int* job_ids, const int* mem_off,
                           const int* mem_cams, double* out_mean) {
  return guarded(ctx, [&] {
    if (n_jobs == 0) return;
    ECCO_REQUIRE(mem_off[0] == 0, "member_offsets[0] must be 0");
    check_cams(ctx, mem_off[n_jobs], mem_cams, "eval_jobs");
    auto s = slots_of(ctx, n_jobs, job_ids);
    int* d_s = ctx->upload(0, s.data(), n_jobs);
    int* d_off = ctx->upload(1, mem_off, n_jobs + 1);
    int* d_mem = ctx->upload(2, mem_cams, std::max(mem_off[n_jobs], 1));
    double* d_out = (double*)ctx->scratch[3].get(sizeof(double) * n_jobs);
    if (learned(ctx)) {
      // learned eval_jobs uses scratch 0..7 internally; copy inputs aside
      DevBuf a, b, c2;
      int* ds = (int*)a.get(sizeof(int) * n_jobs);
      int* doff = (int*)b.get(sizeof(int) * (n_jobs + 1));
      int* dmem = (int*)c2.get(sizeof(int) * std::max(mem_off[n_jobs], 1));
      double* dout;
      DevBuf o;
      dout = (double*)o.get(sizeof(double) * n_jobs);
      ECCO_CUDA(ctx_memcpy(ctx, ds, d_s, sizeof(int) * n_jobs, cudaMemcpyDeviceToDevice, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, doff, d_off, sizeof(int) * (n_jobs + 1), cudaMemcpyDeviceToDevice, ctx->stream));
      ECCO_CUDA(ctx_memcpy(ctx, dmem, d_mem, sizeof(int) * std::max(mem_off[n_jobs], 1), cudaMemcpyDeviceToDevice, ctx->stream));
      lbackend::eval_jobs(ctx, n_jobs, ds, doff, dmem, dout);
      ECCO_CUDA(ctx_memcpy(ctx, out_mean, dout, sizeof(double) * n_jobs, cudaMemcpyDeviceToHost, ctx->stream));
      ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
      a.release(); b.release(); c2.release(); o.release();
      return;
    }
    pbackend::eval_jobs(ctx, n_jobs, d_s, d_off, d_mem, d_out);
    ECCO_CUDA(ctx_memcpy(ctx, out_mean, d_out, sizeof(double) * n_jobs, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

static void eval_matrix_impl(ecco_ctx* ctx, int n, const double* scenes, const int* cam_idx,
                             int g, const int* job_ids, const uint8_t* mask, double* d_out) {
  if (n == 0 || g == 0) return;
  auto s = slots_of(ctx, g, job_ids);
  DevBuf& bs = ctx->em_args[0];  // kept across calls: no cudaMalloc/cudaFree per window
  DevBuf& bp = ctx->em_args[1];
  DevBuf& bm = ctx->em_args[2];
  int* d_s = (int*)bs.get(sizeof(int) * g);
  ECCO_CUDA(ctx_memcpy(ctx, d_s, s.data(), sizeof(int) * g, cudaMemcpyHostToDevice, ctx->stream));
  uint8_t* d_m = nullptr;
  if (mask) {
    d_m = (uint8_t*)bm.get((size_t)n * g);
    ECCO_CUDA(ctx_memcpy(ctx, d_m, mask, (size_t)n * g, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (learned(ctx)) {
    ECCO_REQUIRE(cam_idx != nullptr, "eval_matrix: learned backend needs cam_idx");
    check_cams(ctx, n, cam_idx, "eval_matrix");
    int* d_c = (int*)bp.get(sizeof(int) * n);
    ECCO_CUDA(ctx_memcpy(ctx, d_c, cam_idx, sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
    lbackend::eval_matrix(ctx, n, d_c, g, d_s, d_m, d_out, s.data());
  } else {
    ECCO_REQUIRE(scenes != nullptr, "eval_matrix: parametric backend needs scenes");
    const int D = ctx->cfg.scene_dims;
    double* d_sc = (double*)bp.get(sizeof(double) * (size_t)n * D);
    ECCO_CUDA(ctx_memcpy(ctx, d_sc, scenes, sizeof(double) * n * D, cudaMemcpyHostToDevice, ctx->stream));
    pbackend::eval_matrix(ctx, n, d_sc, g, d_s, d_m, d_out);
  }
}

ecco_status ecco_eval_matrix(ecco_ctx* ctx, int n, const double* scenes, const int* cam_idx, int g,
                             const int* job_ids, const uint8_t* mask, double* out) {
  return guarded(ctx, [&] {
    if (n == 0 || g == 0) return;
    DevBuf o;
    double* d_out = (double*)o.get(sizeof(double) * (size_t)n * g);
    eval_matrix_impl(ctx, n, scenes, cam_idx, g, job_ids, mask, d_out);
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    ECCO_CUDA(cudaMemcpy(out, d_out, sizeof(double) * (size_t)n * g, cudaMemcpyDeviceToHost));
    o.release();
  });
}

ecco_status ecco_eval_matrix_dev(ecco_ctx* ctx, int n, const double* scenes, const int* cam_idx,
                                 int g, const int* job_ids, const uint8_t* mask, void* out_dev) {
  return guarded(ctx, [&] { eval_matrix_impl(ctx, n, scenes, cam_idx, g, job_ids, mask, (double*)out_dev); });
}

ecco_status ecco_eval_matrix_dev_async(ecco_ctx* ctx, int n, const int* cam_idx, int g,
                                       const int* job_ids, void* out_dev, int reserve_sms) {
  return guarded(ctx, [&] {
    const bool exact = learned(ctx) && !ctx->fused_eval && ctx->cfg.math == ECCO_MATH_FFMA_EXACT;
    ECCO_REQUIRE(learned(ctx) && (ctx->fused_eval || exact),
                 "eval_matrix_dev_async: learned backend with fused tensor-core or FFMA_EXACT math");
    ECCO_REQUIRE(reserve_sms >= 0, "eval_matrix_dev_async: reserve_sms must be >= 0");
    if (n == 0 || g == 0) return;
    if (!ctx->matrix_stream) {
      ECCO_CUDA(cudaStreamCreateWithFlags(&ctx->matrix_stream, cudaStreamNonBlocking));
      ECCO_CUDA(cudaEventCreateWithFlags(&ctx->ev_matrix_in, cudaEventDisableTiming));
      ECCO_CUDA(cudaEventCreateWithFlags(&ctx->ev_matrix_done, cudaEventDisableTiming));
    }
    // the committed models' evaluation shadows are rebuilt on the CONTEXT
    // stream first: the chains that run meanwhile evaluate from the same
    // shadows, and must not see one half rebuilt by the matrix stream
    // (FFMA_EXACT evaluates the fp32 masters themselves: the matrix reads a
    // copy taken here, so commits on the context stream meanwhile -- the
    // greedy's extended groups, whose columns the caller re-evaluates --
    // never race with its reads)
    float* wread = ctx->d_w;
    if (exact) {
      const size_t bytes = sizeof(float) * (size_t)ctx->cfg.max_jobs * ctx->n_params;
      wread = (float*)ctx->side_w.get(bytes);
      ECCO_CUDA(cudaMemcpyAsync(wread, ctx->d_w, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      auto s = slots_of(ctx, g, job_ids);
      lbackend::refresh_models(ctx, s.data(), g);
    }
    // the matrix sees everything the context stream has enqueued (committed models)
    ECCO_CUDA(cudaEventRecord(ctx->ev_matrix_in, ctx->stream));
    ECCO_CUDA(cudaStreamWaitEvent(ctx->matrix_stream, ctx->ev_matrix_in, 0));
    // enqueue with the side buffers swapped in: nothing the context stream
    // runs meanwhile shares a scratch buffer, argument buffer or tile counter
    cudaStream_t main_stream = ctx->stream;
    auto swap_side = [&] {
      for (int i = 0; i < 20; ++i) std::swap(ctx->scratch[i], ctx->side_scratch[i]);
      for (int i = 0; i < 3; ++i) std::swap(ctx->em_args[i], ctx->side_em_args[i]);
      std::swap(ctx->tile_ctr, ctx->side_tile_ctr);
    };
    swap_side();
    float* const w_main = ctx->d_w;
    ctx->stream = ctx->matrix_stream;
    ctx->reserve_sms = reserve_sms;
    ctx->d_w = wread;
    try {
      eval_matrix_impl(ctx, n, nullptr, cam_idx, g, job_ids, nullptr, (double*)out_dev);
    } catch (...) {
      ctx->stream = main_stream;
      ctx->reserve_sms = 0;
      ctx->d_w = w_main;
      swap_side();
      throw;
    }
    ctx->stream = main_stream;
    ctx->reserve_sms = 0;
    ctx->d_w = w_main;
    swap_side();
    ECCO_CUDA(cudaEventRecord(ctx->ev_matrix_done, ctx->matrix_stream));
  });
}

ecco_status ecco_matrix_join(ecco_ctx* ctx) {
  return guarded(ctx, [&] {
    if (ctx->matrix_stream) ECCO_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_matrix_done, 0));
  });
}

ecco_status ecco_eval_pairs(ecco_ctx* ctx, int n, const double* scenes, const int* cams,
                            const int* job_ids, double* out) {
  return guarded(ctx, [&] {
    if (n == 0) return;
    auto s = slots_of(ctx, n, job_ids);
    DevBuf bs, bc, bsc, bo;
    int* d_s = (int*)bs.get(sizeof(int) * n);
    ECCO_CUDA(ctx_memcpy(ctx, d_s, s.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
    int* d_c = nullptr;
    if (cams) {
      check_cams(ctx, n, cams, "eval_pairs");
      d_c = (int*)bc.get(sizeof(int) * n);
      ECCO_CUDA(ctx_memcpy(ctx, d_c, cams, sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
    }
    double* d_out = (double*)bo.get(sizeof(double) * n);
    if (learned(ctx)) {
      ECCO_REQUIRE(cams != nullptr, "eval_pairs: learned backend needs cams");
      lbackend::eval_pairs(ctx, n, d_c, d_s, d_out, s.data());
    } else {
      ECCO_REQUIRE(scenes != nullptr || cams != nullptr, "eval_pairs: need scenes or cams");
      double* d_sc = nullptr;
      if (scenes) {
        const int D = ctx->cfg.scene_dims;
        d_sc = (double*)bsc.get(sizeof(double) * (size_t)n * D);
        ECCO_CUDA(ctx_memcpy(ctx, d_sc, scenes, sizeof(double) * (size_t)n * D, cudaMemcpyHostToDevice, ctx->stream));
      }
      pbackend::eval_pairs(ctx, n, d_sc, d_c, d_s, d_out);
    }
    ECCO_CUDA(ctx_memcpy(ctx, out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    bs.release(); bc.release(); bsc.release(); bo.release();
  });
}

ecco_status ecco_rename_models(ecco_ctx* ctx, int n, const int* old_ids, const int* new_ids) {
  return guarded(ctx, [&] {
    for (int i = 0; i < n; ++i) {
      const int s = ctx->slot(old_ids[i]);
      ECCO_REQUIRE(!ctx->slot_of.count(new_ids[i]) || old_ids[i] == new_ids[i],
                   "rename_models: target id in use");
      ctx->slot_of.erase(old_ids[i]);
      ctx->slot_of[new_ids[i]] = s;
    }
  });
}

ecco_status ecco_debug_eval_logits(ecco_ctx* ctx, int n, const int* cam_idx, int g,
                                   const int* job_ids, float* out) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx) && ctx->fused_eval,
                 "debug_eval_logits: needs the learned backend with tensor-core math");
    if (n == 0 || g == 0) return;
    check_cams(ctx, n, cam_idx, "debug_eval_logits");
    auto s = slots_of(ctx, g, job_ids);
    lbackend::debug_logits(ctx, n, cam_idx, g, s.data(), out);
  });
}

ecco_status ecco_route_matrix_dev(ecco_ctx* ctx, int n, int g_block, int n_blocks,
                                  const void* matrix_dev, const void* req_dev, void* best_col_dev,
                                  void* best_acc_dev) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(n >= 0 && g_block >= 0 && n_blocks >= 1, "route_matrix: bad size");
    ECCO_REQUIRE(n == 0 || ((matrix_dev || g_block == 0) && best_col_dev && best_acc_dev),
                 "route_matrix: null buffer");
    lbackend::route_matrix(ctx, n, g_block, n_blocks, (const double*)matrix_dev,
                           (const double*)req_dev, nullptr, (int*)best_col_dev,
                           (double*)best_acc_dev);
  });
}

ecco_status ecco_route_matrix_ids_dev(ecco_ctx* ctx, int n, int g_block, int n_blocks,
                                      const void* matrix_dev, const void* col_ids_dev,
                                      const void* req_dev, void* best_id_dev, void* best_acc_dev) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(n >= 0 && g_block >= 0 && n_blocks >= 1, "route_matrix_ids: bad size");
    ECCO_REQUIRE(n == 0 || ((matrix_dev || g_block == 0) && best_id_dev && best_acc_dev &&
                            (col_ids_dev || g_block == 0)),
                 "route_matrix_ids: null buffer");
    lbackend::route_matrix(ctx, n, g_block, n_blocks, (const double*)matrix_dev,
                           (const double*)req_dev, (const int*)col_ids_dev, (int*)best_id_dev,
                           (double*)best_acc_dev);
  });
}

ecco_status ecco_route_propose(ecco_ctx* ctx, int n, const double* scenes, const int* cam_idx,
                               const double* req, int g, const int* job_ids, const uint8_t* mask,
                               int* best_col, double* best_acc) {
  return guarded(ctx, [&] {
    if (n == 0) return;
    auto s = slots_of(ctx, g, job_ids);
    DevBuf bs, bp, bm, br, bo1, bo2;
    int* d_s = (int*)bs.get(sizeof(int) * std::max(g, 1));
    if (g) ECCO_CUDA(ctx_memcpy(ctx, d_s, s.data(), sizeof(int) * g, cudaMemcpyHostToDevice, ctx->stream));
    uint8_t* d_m = nullptr;
    if (mask && g) {
      d_m = (uint8_t*)bm.get((size_t)n * g);
      ECCO_CUDA(ctx_memcpy(ctx, d_m, mask, (size_t)n * g, cudaMemcpyHostToDevice, ctx->stream));
    }
    double* d_r = (double*)br.get(sizeof(double) * n);
    ECCO_CUDA(ctx_memcpy(ctx, d_r, req, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    int* d_b = (int*)bo1.get(sizeof(int) * n);
    double* d_a = (double*)bo2.get(sizeof(double) * n);
    if (learned(ctx)) {
      check_cams(ctx, n, cam_idx, "route_propose");
      int* d_c = (int*)bp.get(sizeof(int) * n);
      ECCO_CUDA(ctx_memcpy(ctx, d_c, cam_idx, sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
      lbackend::route_propose(ctx, n, d_c, d_r, g, d_s, d_m, d_b, d_a);
    } else {
      const int D = ctx->cfg.scene_dims;
      double* d_sc = (double*)bp.get(sizeof(double) * (size_t)n * D);
      ECCO_CUDA(ctx_memcpy(ctx, d_sc, scenes, sizeof(double) * n * D, cudaMemcpyHostToDevice, ctx->stream));
      pbackend::route_propose(ctx, n, d_sc, d_r, g, d_s, d_m, d_b, d_a);
    }
    ECCO_CUDA(ctx_memcpy(ctx, best_col, d_b, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, best_acc, d_a, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_train_trajectories(ecco_ctx* ctx, int n_jobs, const int* job_ids,
                                    const ecco_batch* batches, const int* src_off,
                                    const int* src_cams, const double* src_fracs,
                                    const int* mem_off, const int* mem_cams,
                                    const int* micro_base, int window, double gpu_s, int depth,
                                    double* out_acc) {
  return guarded(ctx, [&] {
    if (n_jobs == 0) return;
    ECCO_REQUIRE(depth >= 0 && depth <= ctx->cfg.max_depth, "depth must be in [0, max_depth]");
    ECCO_REQUIRE(src_off[0] == 0 && mem_off[0] == 0, "CSR offsets must start at 0");
    for (int j = 0; j < n_jobs; ++j)
      validate_batch(ctx, j, gpu_s, src_off[j + 1] - src_off[j], src_cams + src_off[j],
                     src_fracs + src_off[j]);
    check_cams(ctx, mem_off[n_jobs], mem_cams, "train_trajectories members");
    auto s = slots_of(ctx, n_jobs, job_ids);
    const size_t nsrc = std::max(src_off[n_jobs], 1), nmem = std::max(mem_off[n_jobs], 1);
    DevBuf* b = ctx->traj_args;  // kept across calls: no cudaMalloc/cudaFree per window
    auto up = [&](int i, const void* h, size_t bytes) {
      void* d = b[i].get(bytes);
      ECCO_CUDA(ctx_memcpy(ctx, d, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
      return d;
    };
    int* d_s = (int*)up(0, s.data(), sizeof(int) * n_jobs);
    int* d_so = (int*)up(1, src_off, sizeof(int) * (n_jobs + 1));
    int* d_sc = (int*)up(2, src_cams, sizeof(int) * nsrc);
    double* d_sf = (double*)up(3, src_fracs, sizeof(double) * nsrc);
    int* d_mo = (int*)up(4, mem_off, sizeof(int) * (n_jobs + 1));
    int* d_mc = (int*)up(5, mem_cams, sizeof(int) * nmem);
    double* d_out = (double*)b[6].get(sizeof(double) * n_jobs * (depth + 1));
    if (learned(ctx)) {
      std::vector<int> steps(n_jobs);
      for (int j = 0; j < n_jobs; ++j)
        steps[j] = learned_steps(ctx, batches[j], gpu_s, src_off[j + 1] - src_off[j], src_cams + src_off[j]);
      int* d_j = (int*)up(7, job_ids, sizeof(int) * n_jobs);
      std::vector<int> mb(n_jobs, 0);
      if (micro_base) mb.assign(micro_base, micro_base + n_jobs);
      int* d_mb = (int*)up(8, mb.data(), sizeof(int) * n_jobs);
      if (ctx->ring_partial) {
        // the current rings hold only the rows a sampled staging fetched:
        // every draw of THIS call must be among them, or its arguments
        // differ from the staging call's (the chain would read stale rows)
        int max_steps = 0;
        for (int v : steps) max_steps = std::max(max_steps, v);
        int* d_st = (int*)up(9, steps.data(), sizeof(int) * n_jobs);
        unsigned* d_miss = (unsigned*)ctx->zc_missing.get(sizeof(unsigned));
        ECCO_CUDA(cudaMemsetAsync(d_miss, 0, sizeof(unsigned), ctx->stream));
        stage::mark_sampled(ctx, ctx->stream, n_jobs, d_j, d_st, max_steps, d_so, d_sc, d_sf, d_mb,
                            depth, window, nullptr, (const uint32_t*)ctx->zc_flags_front.p, d_miss);
        unsigned miss = 0;
        ECCO_CUDA(ctx_memcpy(ctx, &miss, d_miss, sizeof(unsigned), cudaMemcpyDeviceToHost,
                             ctx->stream));
        ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
        ECCO_REQUIRE_LOGIC(miss == 0, "train_trajectories: " + std::to_string(miss) +
                                          " sampled draws read ring rows that "
                                          "ecco_stage_sampled_frames did not stage (its arguments "
                                          "differ from this call's): stage them with "
                                          "ecco_fetch_sampled_frames first");
      }
      lbackend::trajectories(ctx, n_jobs, job_ids, d_s, d_j, steps.data(), d_so, d_sc, d_sf, d_mo,
                             d_mc, d_mb, window, depth, d_out);
    } else {
      std::vector<double> bt(3 * (size_t)n_jobs);
      for (int j = 0; j < n_jobs; ++j) {
        bt[3 * j] = batches[j].delivered_frame_rate;
        bt[3 * j + 1] = batches[j].resolution;
        bt[3 * j + 2] = batches[j].quality_factor;
      }
      double* d_bt = (double*)up(7, bt.data(), sizeof(double) * bt.size());
      pbackend::trajectories(ctx, n_jobs, d_s, d_bt, d_so, d_sc, d_sf, d_mo, d_mc, gpu_s, depth, d_out);
      ctx->check_device_status();
    }
    ECCO_CUDA(ctx_memcpy(ctx, out_acc, d_out, sizeof(double) * n_jobs * (depth + 1), cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_commit(ecco_ctx* ctx, int n_jobs, const int* job_ids, const int* granted) {
  return guarded(ctx, [&] {
    if (n_jobs == 0) return;
    for (int j = 0; j < n_jobs; ++j)
      ECCO_REQUIRE(granted[j] >= 0 && granted[j] <= ctx->cfg.max_depth, "commit: granted out of range");
    auto s = slots_of(ctx, n_jobs, job_ids);
    for (int j = 0; j < n_jobs; ++j)
      if (granted[j] > 0) ctx->mark_dirty(s[j]);
    int* d_s = (int*)ctx->commit_args[0].get(sizeof(int) * n_jobs);
    int* d_g = (int*)ctx->commit_args[1].get(sizeof(int) * n_jobs);
    ECCO_CUDA(ctx_memcpy(ctx, d_s, s.data(), sizeof(int) * n_jobs, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, d_g, granted, sizeof(int) * n_jobs, cudaMemcpyHostToDevice, ctx->stream));
    if (learned(ctx))
      lbackend::commit(ctx, n_jobs, d_s, d_g);
    else
      pbackend::commit(ctx, n_jobs, d_s, d_g);
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_last_losses(ecco_ctx* ctx, int n_jobs, const int* job_ids, int depth, float* out) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "last_losses: learned backend only");
    ECCO_REQUIRE(depth >= 0 && depth <= ctx->cfg.max_depth, "depth out of range");
    const int T = ctx->cfg.max_depth;
    for (int j = 0; j < n_jobs; ++j) {
      const int s = ctx->slot(job_ids[j]);
      ECCO_CUDA(ctx_memcpy(ctx, out + (size_t)j * depth, ctx->d_losses + (size_t)s * T,
                                sizeof(float) * depth, cudaMemcpyDeviceToHost, ctx->stream));
    }
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

ecco_status ecco_sample_indices(ecco_ctx* ctx, int job_id, int n_src, const int* src_cams,
                                const double* src_fracs, int window, int micro, int step,
                                int* out_cam, int* out_frame) {
  return guarded(ctx, [&] {
    ECCO_REQUIRE(learned(ctx), "sample_indices: learned backend only");
    ECCO_REQUIRE(n_src >= 1, "sample_indices: need a source");
    DevBuf a, b, c2, d;
    int* d_c = (int*)a.get(sizeof(int) * n_src);
    double* d_f = (double*)b.get(sizeof(double) * n_src);
    const int B = ctx->cfg.minibatch;
    int* d_oc = (int*)c2.get(sizeof(int) * B);
    int* d_of = (int*)d.get(sizeof(int) * B);
    ECCO_CUDA(ctx_memcpy(ctx, d_c, src_cams, sizeof(int) * n_src, cudaMemcpyHostToDevice, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, d_f, src_fracs, sizeof(double) * n_src, cudaMemcpyHostToDevice, ctx->stream));
    lbackend::sample_indices(ctx, job_id, n_src, d_c, d_f, window, micro, step, d_oc, d_of);
    ECCO_CUDA(ctx_memcpy(ctx, out_cam, d_oc, sizeof(int) * B, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, out_frame, d_of, sizeof(int) * B, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    a.release(); b.release(); c2.release(); d.release();
  });
}

ecco_status ecco_profile_tables(ecco_ctx* ctx, int n_cams, const int* cam_idx, const int* bias,
                                int n_levels, const double* levels, int n_grid,
                                const double* grid_fps, const double* grid_res, double window_s,
                                double tie_eps, double ref_rate_bps, double bpp_ref,
                                double* out_budget, double* out_fps, double* out_res,
                                uint8_t* out_feasible) {
  return guarded(ctx, [&] {
    // build_profile_table / make_accuracy_probe validation (transmission.cpp:56-61, 104-105)
    if (n_grid <= 0) ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "build_profile_table: empty config grid");
    if (n_levels <= 0) ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "build_profile_table: no budget levels");
    if (!(window_s > 0.0))
      ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "build_profile_table: window duration must be positive");
    if (!(ref_rate_bps > 0.0))
      ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "make_accuracy_probe: reference rate must be positive");
    ECCO_REQUIRE(n_grid <= 64, "profile: at most 64 grid configs on the device");
    check_cams(ctx, n_cams, cam_idx, "profile_tables");
    std::vector<double> lv(levels, levels + n_levels);
    std::sort(lv.begin(), lv.end());
    for (double b : lv)
      if (!(b > 0.0)) ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "build_profile_table: budget levels must be positive");
    if (n_cams == 0) return;
    DevBuf b[8];
    auto up = [&](int i, const void* h, size_t bytes) {
      void* d = b[i].get(bytes);
      ECCO_CUDA(ctx_memcpy(ctx, d, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
      return d;
    };
    std::vector<int> bz(n_cams, 0);
    if (bias) bz.assign(bias, bias + n_cams);
    int* d_c = (int*)up(0, cam_idx, sizeof(int) * n_cams);
    int* d_b = (int*)up(1, bz.data(), sizeof(int) * n_cams);
    double* d_l = (double*)up(2, lv.data(), sizeof(double) * n_levels);
    double* d_gf = (double*)up(3, grid_fps, sizeof(double) * n_grid);
    double* d_gq = (double*)up(4, grid_res, sizeof(double) * n_grid);
    const size_t rows = (size_t)n_cams * n_levels;
    double* d_f = (double*)b[5].get(sizeof(double) * rows);
    double* d_r = (double*)b[6].get(sizeof(double) * rows);
    uint8_t* d_fe = (uint8_t*)b[7].get(rows);
    pbackend::profile(ctx, n_cams, d_c, d_b, n_levels, d_l, n_grid, d_gf, d_gq, window_s, tie_eps,
                      ref_rate_bps, bpp_ref, d_f, d_r, d_fe);
    ECCO_CUDA(ctx_memcpy(ctx, out_fps, d_f, sizeof(double) * rows, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, out_res, d_r, sizeof(double) * rows, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(ctx_memcpy(ctx, out_feasible, d_fe, rows, cudaMemcpyDeviceToHost, ctx->stream));
    ECCO_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int c = 0; c < n_cams; ++c)
      for (int l = 0; l < n_levels; ++l) out_budget[(size_t)c * n_levels + l] = lv[l];
    for (auto& x : b) x.release();
  });
}

}  // extern "C"
