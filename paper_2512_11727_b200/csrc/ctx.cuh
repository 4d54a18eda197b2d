// Internal state of an ecco_ctx and the helpers shared by the .cu files.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ecco_b200.h"

// Status carried through the C++ layer as an exception, converted back to an
// ecco_status at the C-ABI boundary (abi.cu).
struct EccoError {
  ecco_status code;
  std::string msg;
};

[[noreturn]] inline void ecco_throw(ecco_status code, const std::string& msg) {
  throw EccoError{code, msg};
}

#define ECCO_CUDA(call)                                                                \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      ecco_throw(ECCO_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

#define ECCO_REQUIRE(cond, msg)                                        \
  do {                                                                 \
    if (!(cond)) ecco_throw(ECCO_ERR_INVALID_ARGUMENT, (msg));         \
  } while (0)
#define ECCO_REQUIRE_LOGIC(cond, msg)                                  \
  do {                                                                 \
    if (!(cond)) ecco_throw(ECCO_ERR_LOGIC, (msg));                    \
  } while (0)

// Growable device scratch buffer.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      size_t want = bytes < 4096 ? 4096 : bytes + bytes / 4;
      if (cudaMalloc(&p, want) != cudaSuccess) ecco_throw(ECCO_ERR_CUDA, "cudaMalloc scratch");
      cap = want;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Per-device "attribute already set" flags for cudaFuncSetAttribute (the
// attribute applies to the current device): thread-safe, and a device past
// the 64 cached ones is simply set again on every launch.
struct DeviceFlags {
  std::atomic<uint64_t> bits{0};
  bool done(int dev) const { return dev >= 0 && dev < 64 && ((bits.load() >> dev) & 1u); }
  void mark(int dev) {
    if (dev >= 0 && dev < 64) bits.fetch_or(1ull << dev);
  }
};

// Growable pinned host staging buffer.
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      size_t want = bytes < 4096 ? 4096 : bytes + bytes / 4;
      if (cudaMallocHost(&p, want) != cudaSuccess) ecco_throw(ECCO_ERR_CUDA, "cudaMallocHost");
      cap = want;
    }
    return p;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

inline cudaError_t ctx_memcpy(ecco_ctx* ctx, void* dst, const void* src, size_t bytes,
                              cudaMemcpyKind kind, cudaStream_t s);

// Per-kernel CUDA-event timing (enabled by ecco_profile): each tracked launch
// is bracketed by two events on the context stream; durations are folded in
// when the stats are read.  Algorithmic flops / bytes per launch are supplied
// by the launch site ("units of work").
struct KStat {
  uint64_t launches = 0;
  double ms = 0.0, flops = 0.0, bytes = 0.0;
  struct Pending {
    cudaEvent_t a, b;
    double flops, bytes;
  };
  std::vector<Pending> pending;
};

// bf16 shadow of a set of fp32 model slots for the fused tensor-core
// evaluation (eval_kernels.cu): W1^T [slot][H][F] (TMA map `map_w`) and the
// 128B-swizzled W2^T image per slot.
struct Shadow {
  uint16_t* w1t = nullptr;
  uint8_t* w2t = nullptr;
  void* map_w = nullptr;        // CUtensorMap*, {64, 128} boxes (evaluation)
  void* map_w_pair = nullptr;   // CUtensorMap*, {64, 64} boxes (CTA-pair evaluation)
  void* map_w2_pair = nullptr;  // CUtensorMap*, 5-D view of the W2^T images per CTA half
};

struct ecco_ctx {
  ecco_config cfg{};
  cudaStream_t stream = nullptr;
  std::string err;
  uint64_t launches = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;
  bool profiling = false;
  KStat kstats[ECCO_KSTAT_COUNT];
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t take_event() {
    if (event_pool.empty()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) ecco_throw(ECCO_ERR_CUDA, "cudaEventCreate");
      return e;
    }
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  void fold_stats() {
    for (auto& k : kstats) {
      for (auto& p : k.pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
          k.ms += ms;
          k.flops += p.flops;
          k.bytes += p.bytes;
          k.launches++;
        }
        event_pool.push_back(p.a);
        event_pool.push_back(p.b);
      }
      k.pending.clear();
    }
  }

  // camera table (replicated on every rank)
  int n_cams = 0;
  std::vector<double> h_scenes, h_tp;
  double* d_scenes = nullptr;  // max_cameras * D
  double* d_tp = nullptr;      // max_cameras
  uint64_t* d_exp_tab = nullptr;

  // model slots keyed by JobId
  std::unordered_map<int, int> slot_of;
  std::vector<int> free_slots;

  // parametric models: committed state + speculative chain (max_depth+1 states)
  int* d_k = nullptr;          // slots
  int* d_clen = nullptr;       // slots
  double* d_cl = nullptr;      // slots * K * D
  double* d_prof = nullptr;    // slots * K
  double* d_cen = nullptr;     // slots * D
  int* d_sk = nullptr;         // slots * (max_depth+1)
  int* d_sclen = nullptr;
  double* d_scl = nullptr;     // slots * (max_depth+1) * K * D
  double* d_sprof = nullptr;
  double* d_scen = nullptr;
  int* d_status = nullptr;     // device-side error flag

  // learned backend
  size_t n_params = 0;         // F*H + H + H*C + C
  float* d_w = nullptr;        // slots * n_params (committed fp32 masters)
  float* d_wspec = nullptr;    // slots * max_depth * n_params (snapshots)
  float* d_proto_p = nullptr;  // C * F
  float* d_proto_q = nullptr;  // C * D * F
  uint16_t* d_frames = nullptr;  // max_cameras * R * F (bf16 bits)
  int32_t* d_labels = nullptr;   // max_cameras * R
  uint16_t* d_eval = nullptr;    // max_cameras * S * F
  int32_t* d_eval_labels = nullptr;
  float* d_losses = nullptr;     // slots * max_depth
  int frames_window = -1;
  // back buffers of the double-buffered window ingest (ecco_stage_frames /
  // ecco_swap_frames), allocated on first use; copies run on copy_stream
  uint16_t* b_frames = nullptr;
  int32_t* b_labels = nullptr;
  uint16_t* b_eval = nullptr;
  int32_t* b_eval_labels = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaStream_t copy_stream2 = nullptr;  // the eval-set part: its DMA beside the rings' fetch
  cudaStream_t part_stream(int part) const { return part == 0 ? copy_stream : copy_stream2; }
  // per part (0: rings + labels, 1: eval sets + labels): the staged copy's
  // completion, and the point after which the back buffer is no longer read
  cudaEvent_t copy_done[2] = {nullptr, nullptr}, back_free[2] = {nullptr, nullptr};
  bool staged[2] = {false, false}, back_busy[2] = {false, false};
  // sampled-row ingest (ecco_stage_sampled_frames): the window's job
  // arguments on the copy stream, the bitmap of drawn ring rows, and the
  // running count of rows read from host memory over PCIe (zero-copy)
  DevBuf zc_args[6], zc_flags;
  // The bitmap of the rows present in the CURRENT ring buffer when it came
  // from a sampled staging (ring_partial): ecco_train_trajectories checks
  // every draw against it, ecco_fetch_sampled_frames tops it up.  Swapped
  // with zc_flags when the staged rings become current.
  DevBuf zc_flags_front, zc_topup, zc_missing;
  bool ring_partial = false, back_partial = false;
  HostBuf zc_host;                   // pinned staging of those arguments (truly async copies)
  cudaEvent_t zc_host_free = nullptr;  // the previous argument copy has read zc_host
  DevBuf traj_args[10];  // ecco_train_trajectories' uploaded arguments
  DevBuf commit_args[2];  // ecco_commit's
  DevBuf em_args[3];    // ecco_eval_matrix(_dev)'s uploaded arguments
  DevBuf tile_ctr;      // the CTA-pair evaluation kernel's dynamic super-tile counter
  // ecco_eval_matrix_dev_async: the matrix runs on its own stream with its own
  // scratch / argument buffers / tile counter (swapped in for the enqueue),
  // leaving reserve_sms SMs to what the context stream runs meanwhile
  cudaStream_t matrix_stream = nullptr;
  cudaEvent_t ev_matrix_in = nullptr, ev_matrix_done = nullptr;
  DevBuf side_scratch[20], side_em_args[3], side_tile_ctr;
  DevBuf side_w;  // FFMA_EXACT: the committed masters the async matrix reads
  int reserve_sms = 0;
  unsigned long long* d_zc_rows = nullptr;

  // fused evaluation: shadows of the committed models (refreshed lazily for
  // slots marked dirty) and of the speculative snapshot being evaluated
  bool fused_eval = false;
  bool fused_train = false;
  // fused mode keeps the fp32 W1 masters transposed, [slot][H][F], so the
  // fused SGD update reads and writes them coalesced; ecco_get/set_weights
  // translate to the API layout W1[F][H]
  bool w1_t = false;
  Shadow sh_commit, sh_spec, sh_spec2;  // (sh_spec / sh_spec2: alternate micro-windows)
  Shadow sh_pool;  // serial chains: the images of one job's max_depth snapshots
  cudaStream_t eval_stream = nullptr;    // member evaluations of a chain, beside its training
  cudaEvent_t ev_chain[2] = {nullptr, nullptr}, ev_eval[2] = {nullptr, nullptr};
  std::vector<char> sh_dirty;
  void* map_x = nullptr;  // CUtensorMap* over d_eval
  void mark_dirty(int slot) {
    if (slot >= 0 && slot < (int)sh_dirty.size()) sh_dirty[slot] = 1;
  }

  DevBuf scratch[26];  // 19-20: the general-path evaluation plan of a chain, 21-25: a serial chain's (learned_kernels.cu)
  // 0-10: general training path (learned_kernels.cu; 0-1 also the fused chains' sampled rows),
  // 11: the wide chain's gathered minibatch rows (wide_kernels.cu)
  DevBuf train_scratch[12];
  HostBuf hscratch[4];

  int slot(int job_id) const {
    auto it = slot_of.find(job_id);
    if (it == slot_of.end())
      ecco_throw(ECCO_ERR_INVALID_ARGUMENT, "unknown job id " + std::to_string(job_id));
    return it->second;
  }
  int alloc_slot(int job_id) {
    auto it = slot_of.find(job_id);
    if (it != slot_of.end()) return it->second;
    if (free_slots.empty()) ecco_throw(ECCO_ERR_RUNTIME, "model slots exhausted (max_jobs)");
    int s = free_slots.back();
    free_slots.pop_back();
    slot_of[job_id] = s;
    return s;
  }
  // Copies a host array to a fresh scratch device buffer (stream-ordered).
  template <class T>
  T* upload(int which, const T* h, size_t n) {
    if (n == 0) return nullptr;
    T* d = (T*)scratch[which].get(n * sizeof(T));
    ECCO_CUDA(ctx_memcpy(this, d, h, n * sizeof(T), cudaMemcpyHostToDevice, stream));
    return d;
  }
  void check_device_status();
};

// cudaMemcpyAsync that keeps the context's host<->device byte counters.
inline cudaError_t ctx_memcpy(ecco_ctx* ctx, void* dst, const void* src, size_t bytes,
                              cudaMemcpyKind kind, cudaStream_t s) {
  if (kind == cudaMemcpyHostToDevice) ctx->h2d_bytes += bytes;
  if (kind == cudaMemcpyDeviceToHost) ctx->d2h_bytes += bytes;
  return cudaMemcpyAsync(dst, src, bytes, kind, s);
}

// Wraps a tracked launch statement with profiling events.
#define ECCO_TIMED(ctx, id, fl, by, launch)                                 \
  do {                                                                      \
    if ((ctx)->profiling) {                                                 \
      cudaEvent_t a_ = (ctx)->take_event(), b_ = (ctx)->take_event();       \
      cudaEventRecord(a_, (ctx)->stream);                                   \
      launch;                                                               \
      cudaEventRecord(b_, (ctx)->stream);                                   \
      (ctx)->kstats[id].pending.push_back({a_, b_, (double)(fl), (double)(by)}); \
    } else {                                                                \
      launch;                                                               \
    }                                                                       \
  } while (0)

// Kernel launch bookkeeping (counts every launch for the bench's gpu_launches).
#define ECCO_LAUNCHED(ctx)                                  \
  do {                                                      \
    (ctx)->launches++;                                      \
    cudaError_t e_ = cudaGetLastError();                    \
    if (e_ != cudaSuccess)                                  \
      ecco_throw(ECCO_ERR_CUDA, cudaGetErrorString(e_));    \
  } while (0)

// ---- entry points implemented per backend ----
namespace pbackend {
void eval_matrix(ecco_ctx* ctx, int n_probes, const double* d_scenes_in, int n_jobs,
                 const int* d_slots, const uint8_t* d_mask, double* d_out);
void route_propose(ecco_ctx* ctx, int n_probes, const double* d_scenes_in, const double* d_req,
                   int n_jobs, const int* d_slots, const uint8_t* d_mask, int* d_best,
                   double* d_best_acc);
void trajectories(ecco_ctx* ctx, int n_jobs, const int* d_slots, const double* d_batch,
                  const int* d_src_off, const int* d_src_cam, const double* d_src_frac,
                  const int* d_mem_off, const int* d_mem_cam, double gpu_s, int depth,
                  double* d_out);
void commit(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_granted);
void eval_jobs(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_mem_off,
               const int* d_mem_cam, double* d_out);
void profile(ecco_ctx* ctx, int n_cams, const int* d_cam, const int* d_bias, int n_levels,
             const double* d_levels, int n_grid, const double* d_gf, const double* d_gq,
             double window_s, double tie_eps, double ref_rate, double bpp_ref, double* d_fps,
             double* d_res, uint8_t* d_feas);
void seed(ecco_ctx* ctx, int n, const int* d_slots, const double* d_scenes_in,
          const double* d_acc);
void eval_pairs(ecco_ctx* ctx, int n, const double* d_scenes_in, const int* d_cams,
                const int* d_slots, double* d_out);
}  // namespace pbackend

namespace fused {
bool supported(const ecco_ctx* ctx);
// Evaluation images for `images` model slots (cfg.max_jobs when 0).
void init_shadow(ecco_ctx* ctx, Shadow& sh, size_t images = 0);
void free_shadow(Shadow& sh);
// bf16 images of the models in `slots` (W1^T only for `w1t_slots` when
// given: the fused SGD chain writes the W1^T image of every model it trained)
// Same from device slot lists (no host upload: stream-ordered, the host
// does not wait), W1^T images for d_w1t_slots[0..n1) only.
void refresh_shadow_dev(ecco_ctx* ctx, Shadow& sh, const float* wbase, size_t wstride,
                        const int* d_slots, int n, const int* d_w1t_slots, int n1);
void refresh_shadow(ecco_ctx* ctx, Shadow& sh, const float* wbase, size_t wstride,
                    const std::vector<int>& slots, const std::vector<int>* w1t_slots = nullptr);
// Correct-prediction counts of (probe camera, model slot) pairs.  Dense mode
// (d_tile_ebeg == nullptr): every probe under every entry, counts[p*ld+col].
// Pairs mode: tile m walks entries [tile_ebeg[m], tile_ebeg[m+1]) and a probe
// row counts only under its own slot (d_probe_slot), counts[p].
void eval_counts(ecco_ctx* ctx, const Shadow& sh, const float* wbase, size_t wstride,
                 int n_probes, const int* d_cams, int n_ent, const int* d_ent_slot,
                 const int* d_ent_col, int n_tiles_override, const int* d_tile_ebeg,
                 const int* d_probe_slot, int ld, int* d_counts, float* dbg_logits,
                 double live_pairs, bool pair_tiles = false);
// The CTA-pair evaluation kernel applies (C == 16, not disabled): pair lists
// may then be cut into 256-row super tiles (pair_tiles = true).
bool pair_supported(const ecco_ctx* ctx);
// bf16 W1^T [slot][H][F] of the fp32 masters of `n` device slots.
void shadow_w1t(ecco_ctx* ctx, const int* d_slots, int n, const float* wbase, size_t wstride,
                uint16_t* w1t);
// 2-D bf16 [rows][cols] tensor map, {64, box_rows} boxes, 128-byte swizzle.
CUtensorMap tensor_map_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
void counts_to_acc(ecco_ctx* ctx, size_t n, const int* d_counts, const uint8_t* d_mask,
                   double* d_out);
bool train_supported(const ecco_ctx* ctx);
// Fused SGD chain for wide models (wide_kernels.cu: F <= 1024, H = 512 or
// 1024, C <= 128, the detection head of BASELINE configs[4]): a cluster of
// H/64 CTAs per job, fp32 masters read-modify-written in the snapshot (L2)
// every step.  Same contract as train_chain (which dispatches to it).
bool wide_supported(const ecco_ctx* ctx);
// The sampled rows chain_rows() drew, gathered into contiguous minibatches
// for the wide chain (called by chain_rows for wide shapes).
void wide_gather(ecco_ctx* ctx, int n_jobs, const int* d_steps, int max_steps, int n_micro);
void train_wide(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_steps,
                const int* h_steps, int micro, int n_micro, const float* wsrc, size_t wsrc_stride,
                float* wbase, size_t wstride, int loss_t, int n_launch = 1, size_t wmicro = 0);
// Fused SGD chain (train_kernels.cu): every job's steps[j] SGD steps of one
// micro-window in ONE launch, one thread-block cluster per job with the fp32
// masters resident in TMEM, starting from the models at wsrc and leaving them
// at wbase (a snapshot); writes the bf16 W1^T shadow `sh` (if given).
// chain_rows() first draws the sampled rows of all n_micro micro-windows of
// the call (micro-window `micro` of them is trained by train_chain).
void chain_rows(ecco_ctx* ctx, int n_jobs, const int* d_job_ids, const int* d_steps,
                const int* h_steps, const int* d_src_off, const int* d_src_cam,
                const double* d_src_frac, const int* d_micro_base, int n_micro, int window,
                bool wide_rows = true);
// Fused FP32 SGD chain (ffma_chain.cu): the oracle-exact math of the FFMA
// path in one launch per micro-window (same contract as train_chain, without
// shadows), one cluster of H/16 CTAs per job.
bool ffma_chain_supported(const ecco_ctx* ctx);
void train_ffma(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_steps,
                const int* h_steps, int micro, int n_micro, const float* wsrc, size_t wsrc_stride,
                float* wbase, size_t wstride, int loss_t, int n_launch = 1, size_t wmicro = 0);
void train_chain(ecco_ctx* ctx, const Shadow* sh, int n_jobs, const int* d_slots,
                 const int* d_steps, const int* h_steps, int micro, int n_micro,
                 const float* wsrc, size_t wsrc_stride, float* wbase, size_t wstride,
                 int loss_t, int n_launch = 1, size_t wmicro = 0);
}  // namespace fused

// Sampled-row ingest (stage_kernels.cu), on the given stream.
namespace stage {
// Marks, in a bitmap over ring rows (cam * R + frame), every row the fused
// or general SGD path will draw for micro-windows micro_base[j] + t,
// t < depth (the same counter-RNG draws as k_chain_rows / k_l_sample).
void mark_sampled(ecco_ctx* ctx, cudaStream_t st, int n_jobs, const int* d_job_ids,
                  const int* d_steps, int max_steps, const int* d_src_off, const int* d_src_cam,
                  const double* d_src_frac, const int* d_micro_base, int depth, int window,
                  uint32_t* d_flags, const uint32_t* d_have = nullptr,
                  unsigned* d_missing = nullptr);
// Copies every marked row (F bf16) from mapped pinned host memory into dst
// (same [row][F] layout), counting the rows into *d_count.  With d_have,
// rows already marked there are skipped and the copied ones are marked.
void fetch_rows(ecco_ctx* ctx, cudaStream_t st, const uint16_t* host_dev, uint16_t* dst,
                const uint32_t* d_flags, size_t n_words, unsigned long long* d_count,
                uint32_t* d_have = nullptr);
}  // namespace stage

namespace lbackend {
void init(ecco_ctx* ctx);
// Rebuilds the bf16 evaluation shadows of the committed models among the
// slots that changed since their last refresh (stream-ordered).
void refresh_models(ecco_ctx* ctx, const int* h_slots, int n);
void generate_frames(ecco_ctx* ctx, int window);
void seed(ecco_ctx* ctx, int n, const int* h_job_ids, const int* d_slots, const int* d_job_ids);
void eval_matrix(ecco_ctx* ctx, int n_probes, const int* d_cams, int n_jobs, const int* d_slots,
                 const uint8_t* d_mask, double* d_out, const int* h_slots = nullptr);
void route_propose(ecco_ctx* ctx, int n_probes, const int* d_cams, const double* d_req,
                   int n_jobs, const int* d_slots, const uint8_t* d_mask, int* d_best,
                   double* d_best_acc);
void eval_jobs(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_mem_off,
               const int* d_mem_cam, double* d_out);
void trajectories(ecco_ctx* ctx, int n_jobs, const int* h_job_ids, const int* d_slots,
                  const int* d_job_ids, const int* h_steps, const int* d_src_off,
                  const int* d_src_cam, const double* d_src_frac, const int* d_mem_off,
                  const int* d_mem_cam, const int* d_micro_base, int window, int depth,
                  double* d_out);
void commit(ecco_ctx* ctx, int n_jobs, const int* d_slots, const int* d_granted);
void eval_pairs(ecco_ctx* ctx, int n, const int* d_cams, const int* d_slots, double* d_out,
                const int* h_slots = nullptr);
void debug_logits(ecco_ctx* ctx, int n, const int* h_cams, int gj, const int* h_slots, float* out);
void route_matrix(ecco_ctx* ctx, int n, int gb, int n_blocks, const double* d_M,
                  const double* d_req, const int* d_ids, int* d_best, double* d_best_acc);
void sample_indices(ecco_ctx* ctx, int job_id, int n_src, const int* d_src_cam,
                    const double* d_src_frac, int window, int micro, int step, int* d_cam,
                    int* d_frame);
}  // namespace lbackend
