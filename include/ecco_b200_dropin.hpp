/* ecco_b200_dropin.hpp -- the reference-side C++ binding of the B200 path.
 *
 * Header-only; a maintainer adds it to the reference build (it includes the
 * reference's own headers "ecco/*.hpp" from proj/core/include) and links
 * libecco_b200.so.  It implements the reference's callback interfaces over
 * the C-ABI of ecco_b200.h, so the reference call sites stay unchanged:
 *
 *   ecco::TrainingBackend  (core/include/ecco/gpu_allocator.hpp:37-42)
 *       CudaTrainingBackend replaces JobTrainingBackend
 *       (core/src/orchestrator.cpp:31-70): every job's speculative chain of
 *       micro-windows is computed in one batched device call; evaluate() /
 *       train() replay it as WindowAllocation::run_micro
 *       (core/src/gpu_allocator.cpp:125-135) consumes it, and finish() commits
 *       the granted prefixes and writes the trained models back into the
 *       reference's JobMap.
 *   ecco::ModelEvalFn      (core/include/ecco/grouping.hpp:23)
 *       make_eval_fn replaces eval_job_on_scene (orchestrator.cpp:186-191).
 *   ecco::ProbeFn          (core/include/ecco/transmission.hpp:46)
 *       build_profile_tables replaces build_profile_table driven by
 *       make_accuracy_probe (transmission.cpp:52-118) for many cameras at
 *       once (Simulation::profile, orchestrator.cpp:94-116).
 *
 * Two backends behind the same classes:
 *   parametric  the reference's accuracy model, bit-identical: the job's
 *               ModelState is shipped to the device and written back;
 *   learned     real per-group MLPs resident on the device (Device(params,
 *               LearnedShape, ...)): a job's model is its device weights,
 *               keyed by JobId (seeded on first use), and the probe of a
 *               routing request is its CAMERA's labelled eval set.
 * BatchedRouter serves group_request's ModelEvalFn for a whole routing pass
 * from ONE ecco_eval_matrix call (both backends).
 * The status -> exception mapping mirrors core/include/ecco/types.hpp:29-48.
 * Verified against the unmodified reference by oracle/dropin_test.cpp
 * (parametric) and oracle/dropin_learned_test.cpp (learned, vs the CPU
 * oracle's trajectories).
 */
#ifndef ECCO_B200_DROPIN_HPP_
#define ECCO_B200_DROPIN_HPP_

#include <algorithm>
#include <functional>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "ecco/accuracy_model.hpp"
#include "ecco/gpu_allocator.hpp"
#include "ecco/grouping.hpp"
#include "ecco/job.hpp"
#include "ecco/transmission.hpp"
#include "ecco/types.hpp"
#include "ecco_b200.h"

namespace ecco_b200 {

inline void check(ecco_ctx* c, ecco_status s, int window = 0) {
  switch (s) {
    case ECCO_OK:
      return;
    case ECCO_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(ecco_last_error(c));
    case ECCO_ERR_LOGIC:
      throw std::logic_error(ecco_last_error(c));
    case ECCO_ERR_INFEASIBLE:
      throw ecco::InfeasibleScheduleError(window, ecco_last_error(c));
    case ECCO_ERR_SCHEMA:
      throw ecco::SchemaError("", ecco_last_error(c));
    default:
      throw std::runtime_error(ecco_last_error(c));
  }
}

// The learned backend's model and stream shape (ecco_config's learned
// fields; defaults = ecco_default_config's, SURVEY.md 8(a')).
struct LearnedShape {
  int feat_dim = 512, hidden_dim = 256, num_classes = 16, minibatch = 128;
  int ring_frames = 512, eval_samples = 64, max_depth = 64;
  float sgd_lr = 0.05f, feature_noise = 1.0f;
  double steps_per_gpu_s = 4.0;
  uint64_t seed = 0x5eed0001ULL;
  int math = ECCO_MATH_FFMA_EXACT;  // or ECCO_MATH_TC_BF16
};

// A device context plus the CameraId <-> index table and the job models it
// holds.
class Device {
 public:
  // parametric backend
  Device(const ecco::ModelParams& p, int scene_dims, int max_clusters, int max_jobs,
         int max_cameras, int device = 0)
      : D_(scene_dims), P_(max_clusters) {
    ecco_config c;
    ecco_default_config(&c);
    c.backend = ECCO_BACKEND_PARAMETRIC;
    c.device = device;
    c.scene_dims = scene_dims;
    c.max_clusters = max_clusters;
    c.max_jobs = max_jobs;
    c.max_cameras = max_cameras;
    c.params = {p.learning_rate_k, p.similarity_lambda, p.acc_floor, p.acc_ceil,
                p.cluster_similarity_threshold};
    c.max_depth = 64;
    check(nullptr, ecco_create(&c, &ctx_));
  }
  // learned backend
  Device(const ecco::ModelParams& p, const LearnedShape& shape, int scene_dims, int max_jobs,
         int max_cameras, int device = 0)
      : D_(scene_dims), P_(1), learned_(true) {
    ecco_config c;
    ecco_default_config(&c);
    c.backend = ECCO_BACKEND_LEARNED;
    c.device = device;
    c.scene_dims = scene_dims;
    c.max_jobs = max_jobs;
    c.max_cameras = max_cameras;
    c.params = {p.learning_rate_k, p.similarity_lambda, p.acc_floor, p.acc_ceil,
                p.cluster_similarity_threshold};
    c.math = shape.math;
    c.feat_dim = shape.feat_dim;
    c.hidden_dim = shape.hidden_dim;
    c.num_classes = shape.num_classes;
    c.minibatch = shape.minibatch;
    c.ring_frames = shape.ring_frames;
    c.eval_samples = shape.eval_samples;
    c.max_depth = shape.max_depth;
    c.sgd_lr = shape.sgd_lr;
    c.feature_noise = shape.feature_noise;
    c.steps_per_gpu_s = shape.steps_per_gpu_s;
    c.seed = shape.seed;
    check(nullptr, ecco_create(&c, &ctx_));
  }
  bool learned() const { return learned_; }
  // learned: the window's synthetic streams (frame rings + eval sets) of
  // every camera, from (seed, camera, window, scene)
  void generate_frames(int window) { check(ctx_, ecco_generate_frames(ctx_, window)); }
  // learned: a job's device model, seeded on first use (the learned
  // seed_model: the base model every new job starts from)
  void ensure_model(ecco::JobId id) {
    if (seeded_.count(id)) return;
    check(ctx_, ecco_seed_models(ctx_, 1, &id, nullptr, nullptr));
    seeded_.insert(id);
  }
  void drop_model(ecco::JobId id) {
    check(ctx_, ecco_drop_models(ctx_, 1, &id));
    seeded_.erase(id);
  }
  ~Device() { ecco_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  ecco_ctx* ctx() const { return ctx_; }
  int dims() const { return D_; }

  // CameraState table (accuracy_model.hpp:27-34): scenes and pixel throughput,
  // indexed in std::map (CameraId string) order.
  void set_cameras(const std::map<ecco::CameraId, ecco::CameraState>& cams) {
    index_.clear();
    std::vector<double> scenes, tp;
    for (const auto& [id, c] : cams) {
      if ((int)c.scene.size() != D_) throw std::invalid_argument("camera scene dimension");
      index_[id] = (int)index_.size();
      scenes.insert(scenes.end(), c.scene.begin(), c.scene.end());
      tp.push_back(c.gpu_pixel_throughput);
    }
    check(ctx_, ecco_set_cameras(ctx_, (int)tp.size(), scenes.data(), tp.data()));
  }
  int cam(const ecco::CameraId& id) const { return index_.at(id); }

  // RetrainJob::model <-> device slot.
  void put_model(ecco::JobId id, const ecco::ModelState& m) {
    const int k = (int)m.clusters.size();
    if (k > P_) throw std::invalid_argument("model has more clusters than max_clusters");
    std::vector<double> cl((size_t)P_ * D_, 0.0), pr(P_, 0.0), ce(D_, 0.0);
    for (int i = 0; i < k; ++i) {
      std::copy(m.clusters[i].begin(), m.clusters[i].end(), cl.begin() + (size_t)i * D_);
      pr[i] = m.proficiency[i];
    }
    std::copy(m.centroid.begin(), m.centroid.end(), ce.begin());
    const int clen = (int)m.centroid.size();
    check(ctx_, ecco_put_models(ctx_, 1, &id, &k, cl.data(), pr.data(), ce.data(), &clen));
  }
  ecco::ModelState get_model(ecco::JobId id) const {
    int k = 0, clen = 0;
    std::vector<double> cl((size_t)P_ * D_), pr(P_), ce(D_);
    check(ctx_, ecco_get_models(ctx_, 1, &id, &k, cl.data(), pr.data(), ce.data(), &clen));
    ecco::ModelState m;
    for (int i = 0; i < k; ++i) {
      m.clusters.emplace_back(cl.begin() + (size_t)i * D_, cl.begin() + (size_t)(i + 1) * D_);
      m.proficiency.push_back(pr[i]);
    }
    m.centroid.assign(ce.begin(), ce.begin() + clen);
    return m;
  }

 private:
  ecco_ctx* ctx_ = nullptr;
  int D_, P_;
  bool learned_ = false;
  std::map<ecco::CameraId, int> index_;
  std::set<ecco::JobId> seeded_;
};

// JobTrainingBackend (orchestrator.cpp:31-70) on the device.  Construct it
// where the reference constructs JobTrainingBackend, with the same JobMap,
// batches and bootstrap function; every train() must be for `micro_gpu_s`
// (the allocator's gpu_count * micro_window_duration_s, gpu_allocator.cpp:127).
class CudaTrainingBackend final : public ecco::TrainingBackend {
 public:
  CudaTrainingBackend(Device& dev, ecco::JobMap& jobs,
                      const std::map<ecco::JobId, ecco::TrainingBatchStats>& batches,
                      std::function<ecco::TrainingBatchStats(const ecco::RetrainJob&)> bootstrap,
                      double micro_gpu_s, int depth = 4, int window = 0)
      : dev_(dev), jobs_(jobs), gpu_s_(micro_gpu_s), depth_(std::max(1, depth)),
        window_(window) {
    for (auto& [id, job] : jobs_) {
      if (dev_.learned())
        dev_.ensure_model(id);  // the job's weights live on the device
      else
        dev_.put_model(id, job.model);
      Chain c;
      const auto it = batches.find(id);
      const ecco::TrainingBatchStats b = it != batches.end() ? it->second : bootstrap(job);
      c.batch = {b.delivered_frame_rate, b.resolution, b.quality_factor};
      for (const auto& [cam, frac] : b.source_mix) {  // std::map order, as train_step
        c.src.push_back(dev_.cam(cam));
        c.frac.push_back(frac);
      }
      for (const auto& m : job.members) c.mem.push_back(dev_.cam(m.camera));
      chains_[id] = std::move(c);
    }
  }

  double evaluate(ecco::JobId id) override {
    prepare();
    Chain& c = chain(id);
    return c.acc[c.used];
  }

  void train(ecco::JobId id, double gpu_seconds) override {
    if (gpu_seconds != gpu_s_)
      throw std::invalid_argument("CudaTrainingBackend: micro-window GPU time changed");
    prepare();
    Chain& c = chain(id);
    if (c.used + 1 >= (int)c.acc.size()) {  // chain spent: commit it, extend (depth doubling)
      const int next = std::min(64, 2 * ((int)c.acc.size() - 1));
      commit(id);
      run(id, next);
    }
    ++c.used;
  }

  // After run_remaining: commits every granted prefix and, parametric,
  // writes the trained models into the JobMap (what JobTrainingBackend::train
  // did in place); learned models stay on the device (ecco_get_weights).
  void finish() {
    for (auto& [id, c] : chains_) {
      commit(id);
      if (!dev_.learned()) jobs_.at(id).model = dev_.get_model(id);
    }
    prepared_ = false;
  }

 private:
  struct Chain {
    ecco_batch batch{};
    std::vector<int> src, mem;
    std::vector<double> frac, acc;
    int used = 0, base = 0;
  };

  Chain& chain(ecco::JobId id) { return chains_.at(id); }

  // Every job's chain in one batched device call (the first evaluate()).
  void prepare() {
    if (prepared_) return;
    prepared_ = true;
    std::vector<int> ids, so{0}, mo{0}, src, mem, base;
    std::vector<double> frac;
    std::vector<ecco_batch> bs;
    for (auto& [id, c] : chains_) {
      ids.push_back(id);
      bs.push_back(c.batch);
      src.insert(src.end(), c.src.begin(), c.src.end());
      frac.insert(frac.end(), c.frac.begin(), c.frac.end());
      mem.insert(mem.end(), c.mem.begin(), c.mem.end());
      so.push_back((int)src.size());
      mo.push_back((int)mem.size());
      base.push_back(c.base);
    }
    std::vector<double> acc(ids.size() * (depth_ + 1));
    check(dev_.ctx(), ecco_train_trajectories(dev_.ctx(), (int)ids.size(), ids.data(), bs.data(),
                                              so.data(), src.data(), frac.data(), mo.data(),
                                              mem.data(), base.data(), window_, gpu_s_, depth_,
                                              acc.data()));
    for (size_t j = 0; j < ids.size(); ++j) {
      Chain& c = chain(ids[j]);
      c.acc.assign(acc.begin() + j * (depth_ + 1), acc.begin() + (j + 1) * (depth_ + 1));
      c.used = 0;
    }
  }

  void run(ecco::JobId id, int depth) {
    Chain& c = chain(id);
    const int so[2] = {0, (int)c.src.size()}, mo[2] = {0, (int)c.mem.size()};
    c.acc.assign(depth + 1, 0.0);
    check(dev_.ctx(), ecco_train_trajectories(dev_.ctx(), 1, &id, &c.batch, so, c.src.data(),
                                              c.frac.data(), mo, c.mem.data(), &c.base,
                                              window_, gpu_s_, depth, c.acc.data()));
    c.used = 0;
  }

  void commit(ecco::JobId id) {
    Chain& c = chain(id);
    if (c.acc.empty()) return;
    check(dev_.ctx(), ecco_commit(dev_.ctx(), 1, &id, &c.used));
    c.base += c.used;
    c.acc.clear();
    c.used = 0;
  }

  Device& dev_;
  ecco::JobMap& jobs_;
  double gpu_s_;
  int depth_;
  int window_;
  std::map<ecco::JobId, Chain> chains_;
  bool prepared_ = false;
};

// eval_job_on_scene (orchestrator.cpp:186-191) on the device: eval(job.model,
// probe with `scene`), parametric backend.  Per call it ships the job's model
// and evaluates one pair; a routing pass that knows all its requests up front
// uses BatchedRouter (below) instead: one fused launch for the whole pass.
inline ecco::ModelEvalFn make_eval_fn(Device& dev) {
  if (dev.learned())
    throw std::invalid_argument("make_eval_fn: the learned probe is a camera, use BatchedRouter");
  return [&dev](const ecco::RetrainJob& job, const ecco::SceneVector& scene) {
    if ((int)scene.size() != dev.dims()) throw std::invalid_argument("scene dimension");
    dev.put_model(job.id, job.model);
    double out = 0.0;
    check(dev.ctx(),
          ecco_eval_matrix(dev.ctx(), 1, scene.data(), nullptr, 1, &job.id, nullptr, &out));
    return out;
  };
}

// Batched ModelEvalFn for a whole routing pass.  group_request
// (grouping.cpp:18-62) calls eval_fn(job, request.subsamples) for every
// correlated job, one request at a time; a routing pass
// (route_pending_requests, orchestrator.cpp:158-184, or update_grouping's
// reroute, grouping.cpp:113-118) knows its requests up front, so:
//
//   BatchedRouter router(dev, jobs, pending);  // ONE ecco_eval_matrix call
//   for (auto& req : pending) {                // in the reference's order
//     router.route_as(req);
//     auto a = ecco::group_request(jobs, req, cfg, params, router.eval_fn(), next_id);
//     if (a.created) router.created(jobs.at(a.job));
//   }
//
// The probe of a request is its scene (parametric: request.subsamples, as
// eval_job_on_scene, orchestrator.cpp:186-191) or its CAMERA's labelled eval
// set (learned).  The constructor evaluates every (request, job) pair in one
// fused launch; jobs created during the pass (seed_model / the learned base
// model) are evaluated on demand.  Values equal make_eval_fn's bit for bit.
class BatchedRouter {
 public:
  BatchedRouter(Device& dev, const ecco::JobMap& jobs,
                const std::vector<ecco::RetrainRequest>& requests)
      : dev_(dev) {
    std::vector<int> cams, ids;
    std::vector<double> scenes;
    for (const auto& r : requests) {
      if (row_.count(r.camera)) continue;
      row_[r.camera] = (int)row_.size();
      if (dev.learned()) cams.push_back(dev.cam(r.camera));  // the probe is its eval set
      else {
        if ((int)r.subsamples.size() != dev.dims()) throw std::invalid_argument("scene dimension");
        scenes.insert(scenes.end(), r.subsamples.begin(), r.subsamples.end());
      }
    }
    for (const auto& [id, j] : jobs) {
      if (dev.learned())
        dev.ensure_model(id);
      else
        dev.put_model(id, j.model);
      col_[id] = (int)ids.size();
      ids.push_back(id);
    }
    n_jobs_ = (int)ids.size();
    m_.assign(row_.size() * ids.size(), 0.0);
    if (!row_.empty() && !ids.empty())
      check(dev.ctx(), ecco_eval_matrix(dev.ctx(), (int)row_.size(),
                                        dev.learned() ? nullptr : scenes.data(),
                                        dev.learned() ? cams.data() : nullptr, (int)ids.size(),
                                        ids.data(), nullptr, m_.data()));
  }
  void route_as(const ecco::RetrainRequest& request) { cur_ = &request; }
  // a job group_request created in this pass (it may be a candidate for the
  // pass's later requests)
  void created(const ecco::RetrainJob& job) {
    if (dev_.learned())
      dev_.ensure_model(job.id);
    else
      dev_.put_model(job.id, job.model);
  }
  ecco::ModelEvalFn eval_fn() {
    return [this](const ecco::RetrainJob& job, const ecco::SceneVector& scene) {
      if (!cur_) throw std::logic_error("BatchedRouter: route_as() before group_request");
      const auto r = row_.find(cur_->camera);
      const auto c = col_.find(job.id);
      if (r != row_.end() && c != col_.end()) return m_[(size_t)r->second * n_jobs_ + c->second];
      created(job);
      const int id = job.id;
      double out = 0.0;
      if (dev_.learned()) {
        const int cam = dev_.cam(cur_->camera);
        check(dev_.ctx(), ecco_eval_pairs(dev_.ctx(), 1, nullptr, &cam, &id, &out));
      } else {
        if ((int)scene.size() != dev_.dims()) throw std::invalid_argument("scene dimension");
        check(dev_.ctx(),
              ecco_eval_matrix(dev_.ctx(), 1, scene.data(), nullptr, 1, &id, nullptr, &out));
      }
      return out;
    };
  }

 private:
  Device& dev_;
  std::map<ecco::CameraId, int> row_;
  std::map<ecco::JobId, int> col_;
  std::vector<double> m_;
  int n_jobs_ = 0;
  const ecco::RetrainRequest* cur_ = nullptr;
};

// build_profile_table(camera, budget_levels, grid, make_accuracy_probe(camera,
// params, reference_rate_bps, bpp_ref), opts) for every camera in one device
// launch (every grid probe of every level, the tie_epsilon / bias tie-break
// fused).  The cameras must be in the Device's camera table; the params are
// the Device's.
inline std::vector<ecco::ProfileTable> build_profile_tables(
    Device& dev, const std::vector<ecco::CameraState>& cameras,
    const std::vector<double>& budget_levels, const std::vector<ecco::SamplingConfig>& grid,
    const ecco::ProfilerOptions& opts, double reference_rate_bps, double bpp_ref) {
  if (grid.empty()) throw std::invalid_argument("build_profile_table: empty config grid");
  if (budget_levels.empty()) throw std::invalid_argument("build_profile_table: no budget levels");
  std::vector<double> levels = budget_levels;
  std::sort(levels.begin(), levels.end());  // rows in ascending budget order
  std::vector<int> idx, bias;
  for (const auto& c : cameras) {
    idx.push_back(dev.cam(c.id));
    bias.push_back(opts.bias == ecco::ProfileBias::frame_rate ? 1 : 0);
  }
  std::vector<double> gf, gr;
  for (const auto& g : grid) {
    gf.push_back(g.frame_rate);
    gr.push_back(g.resolution);
  }
  const size_t n = cameras.size() * levels.size();
  std::vector<double> ob(n), of(n), oq(n);
  std::vector<uint8_t> fe(n);
  check(dev.ctx(), ecco_profile_tables(dev.ctx(), (int)cameras.size(), idx.data(), bias.data(),
                                       (int)levels.size(), levels.data(), (int)grid.size(),
                                       gf.data(), gr.data(), opts.window_duration_s,
                                       opts.tie_epsilon, reference_rate_bps, bpp_ref, ob.data(),
                                       of.data(), oq.data(), fe.data()));
  std::vector<ecco::ProfileTable> out(cameras.size());
  for (size_t i = 0; i < cameras.size(); ++i) {
    out[i].camera = cameras[i].id;
    for (size_t l = 0; l < levels.size(); ++l) {
      const size_t o = i * levels.size() + l;
      ecco::ProfileRow r;
      r.budget_gpu_s = ob[o];
      r.config.frame_rate = of[o];
      r.config.resolution = oq[o];
      r.feasible = fe[o] != 0;
      out[i].rows.push_back(r);
    }
  }
  return out;
}

}  // namespace ecco_b200

#endif  // ECCO_B200_DROPIN_HPP_
