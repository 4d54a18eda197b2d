// accuracy_model_b200.cpp -- TEST INFRASTRUCTURE ONLY.
//
// ecco's accuracy-model API (core/include/ecco/accuracy_model.hpp:58-94) with
// eval, train_step and seed_model EXECUTED BY THE B200 BUILD: every call ships
// its model and cameras to a parametric device context of libecco_b200.so and
// runs the device kernels through the C-ABI (ecco_eval_pairs,
// ecco_train_trajectories + ecco_commit, ecco_seed_models).  The remaining
// helpers (similarity, find_cluster, find_or_add_cluster, apply_drift) and
// the argument checks are the C restatement (oracle/ecco_oracle.c) with the
// reference's exceptions.  oracle/Makefile links this object INSTEAD of the
// reference's accuracy_model.o into the reference's own unit tests
// (proj/tests/*.cpp) -> oracle/_ref/unit_tests_b200, so the reference's
// accuracy-model, allocator, grouping, transmission and orchestrator suites
// run against the device arithmetic (tests/test_reference_suite.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "ecco/accuracy_model.hpp"
#include "ecco_b200.h"
#include "ecco_oracle.h"

namespace ecco {
namespace {

constexpr int kP = 32;      // cluster capacity of a device model (ecco_config limit)
constexpr int kCams = 256;  // camera table capacity

struct Device {
  ecco_ctx* ctx = nullptr;
  int D = -1;
  ModelParams p{};
  ~Device() {
    if (ctx) ecco_destroy(ctx);
  }
};

void check(ecco_ctx* c, ecco_status s) {
  if (s == ECCO_OK) return;
  const std::string m = c ? ecco_last_error(c) : "ecco_create failed";
  if (s == ECCO_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
  if (s == ECCO_ERR_LOGIC) throw std::logic_error(m);
  throw std::runtime_error(m);
}

bool same_params(const ModelParams& a, const ModelParams& b) {
  return std::memcmp(&a, &b, sizeof(ModelParams)) == 0;
}

ecco_ctx* device(const ModelParams& p, int D) {
  static Device dev;
  if (dev.ctx && dev.D == D && same_params(dev.p, p)) return dev.ctx;
  if (dev.ctx) ecco_destroy(dev.ctx);
  dev.ctx = nullptr;
  ecco_config c;
  ecco_default_config(&c);
  c.backend = ECCO_BACKEND_PARAMETRIC;
  c.scene_dims = D;
  c.max_clusters = kP;
  c.max_jobs = 4;
  c.max_cameras = kCams;
  c.max_depth = 2;
  c.params = {p.learning_rate_k, p.similarity_lambda, p.acc_floor, p.acc_ceil,
              p.cluster_similarity_threshold};
  check(nullptr, ecco_create(&c, &dev.ctx));
  dev.D = D;
  dev.p = p;
  return dev.ctx;
}

void put(ecco_ctx* ctx, const ModelState& m, int D) {
  const int id = 1, k = (int)m.clusters.size(), clen = (int)m.centroid.size();
  if (k > kP) throw std::runtime_error("accuracy_model_b200: model exceeds the cluster capacity");
  std::vector<double> cl((size_t)kP * D, 0.0), pr(kP, 0.0), ce(D, 0.0);
  for (int i = 0; i < k; ++i) {
    if ((int)m.clusters[i].size() != D) throw std::invalid_argument("similarity: scene dimension mismatch");
    std::copy(m.clusters[i].begin(), m.clusters[i].end(), cl.begin() + (size_t)i * D);
    pr[i] = m.proficiency[i];
  }
  std::copy(m.centroid.begin(), m.centroid.end(), ce.begin());
  check(ctx, ecco_put_models(ctx, 1, &id, &k, cl.data(), pr.data(), ce.data(), &clen));
}

ModelState get(ecco_ctx* ctx, int D) {
  const int id = 1;
  int k = 0, clen = 0;
  std::vector<double> cl((size_t)kP * D), pr(kP), ce(D);
  check(ctx, ecco_get_models(ctx, 1, &id, &k, cl.data(), pr.data(), ce.data(), &clen));
  ModelState m;
  for (int i = 0; i < k; ++i) {
    m.clusters.emplace_back(cl.begin() + (size_t)i * D, cl.begin() + (size_t)(i + 1) * D);
    m.proficiency.push_back(pr[i]);
  }
  m.centroid.assign(ce.begin(), ce.begin() + clen);
  return m;
}

void set_cameras(ecco_ctx* ctx, const std::vector<const CameraState*>& cams, int D) {
  std::vector<double> sc, tp;
  for (const CameraState* c : cams) {
    if ((int)c->scene.size() != D) throw std::invalid_argument("similarity: scene dimension mismatch");
    sc.insert(sc.end(), c->scene.begin(), c->scene.end());
    tp.push_back(c->gpu_pixel_throughput);
  }
  check(ctx, ecco_set_cameras(ctx, (int)cams.size(), sc.data(), tp.data()));
}

int dims_of(const ModelState& m, const SceneVector& s) {
  if (!m.clusters.empty()) return (int)m.clusters[0].size();
  return (int)s.size();
}

}  // namespace

double similarity(const SceneVector& a, const SceneVector& b, double lambda) {
  if (a.size() != b.size()) throw std::invalid_argument("similarity: scene dimension mismatch");
  if (!(lambda > 0.0)) throw std::invalid_argument("similarity: lambda must be positive");
  return orc_similarity(a.data(), b.data(), (int)a.size(), lambda);
}

int find_cluster(const ModelState& model, const SceneVector& scene, const ModelParams& params) {
  int best = -1;
  double best_sim = 0.0;
  for (size_t i = 0; i < model.clusters.size(); ++i) {  // strict >: lowest id on ties
    const double s = similarity(model.clusters[i], scene, params.similarity_lambda);
    if (best < 0 || s > best_sim) {
      best = (int)i;
      best_sim = s;
    }
  }
  return best >= 0 && best_sim >= params.cluster_similarity_threshold ? best : -1;
}

int find_or_add_cluster(ModelState& model, const SceneVector& scene, const ModelParams& params) {
  const int c = find_cluster(model, scene, params);
  if (c >= 0) return c;
  model.clusters.push_back(scene);
  model.proficiency.push_back(0.0);
  return (int)model.clusters.size() - 1;
}

double eval(const ModelState& model, const CameraState& camera, const ModelParams& params) {
  const int D = dims_of(model, camera.scene);
  if ((int)camera.scene.size() != D) throw std::invalid_argument("similarity: scene dimension mismatch");
  if (!(params.similarity_lambda > 0.0))
    throw std::invalid_argument("similarity: lambda must be positive");
  ecco_ctx* ctx = device(params, D);
  put(ctx, model, D);
  set_cameras(ctx, {&camera}, D);
  const int cam = 0, id = 1;
  double out = 0.0;
  check(ctx, ecco_eval_pairs(ctx, 1, nullptr, &cam, &id, &out));
  return out;
}

ModelState train_step(const ModelState& model, const TrainingBatchStats& batch, double gpu_time_s,
                      const std::vector<CameraState>& cameras, const ModelParams& params) {
  // the reference's argument checks (accuracy_model.cpp:72-80, 94-100)
  if (gpu_time_s < 0.0) throw std::invalid_argument("train_step: negative gpu_time");
  double total = 0.0;
  for (const auto& [id, f] : batch.source_mix) {
    if (f < 0.0) throw std::invalid_argument("train_step: negative source_mix fraction");
    total += f;
  }
  if (!batch.source_mix.empty() && std::abs(total - 1.0) > 1e-9)
    throw std::invalid_argument("train_step: source_mix fractions must sum to 1");
  std::vector<const CameraState*> cams;
  for (const auto& c : cameras) cams.push_back(&c);
  std::vector<int> src;
  std::vector<double> frac;
  for (const auto& [id, f] : batch.source_mix) {
    int k = -1;
    for (size_t i = 0; i < cameras.size() && k < 0; ++i)
      if (cameras[i].id == id) k = (int)i;
    if (k < 0) throw std::invalid_argument("train_step: source_mix camera missing: " + id);
    src.push_back(k);
    frac.push_back(f);
  }
  int D = !model.clusters.empty() ? (int)model.clusters[0].size()
                                  : (!src.empty() ? (int)cameras[src[0]].scene.size() : 0);
  for (int k : src)
    if ((int)cameras[k].scene.size() != D)
      throw std::invalid_argument("train_step: scene dimension mismatch in batch");
  if (D == 0 || src.empty()) return model;  // no sources: nothing trains (accuracy_model.cpp:88-110)
  ecco_ctx* ctx = device(params, D);
  put(ctx, model, D);
  set_cameras(ctx, cams, D);
  const int id = 1, so[2] = {0, (int)src.size()}, mo[2] = {0, 1}, mem = src.empty() ? 0 : src[0];
  const ecco_batch b = {batch.delivered_frame_rate, batch.resolution, batch.quality_factor};
  double acc[2];
  check(ctx, ecco_train_trajectories(ctx, 1, &id, &b, so, src.data(), frac.data(), mo, &mem,
                                     nullptr, 0, gpu_time_s, 1, acc));
  const int one = 1;
  check(ctx, ecco_commit(ctx, 1, &id, &one));
  return get(ctx, D);
}

CameraState apply_drift(const CameraState& camera, const DriftEvent& event,
                        const ModelParams& params) {
  if (event.camera != camera.id)
    throw std::invalid_argument("apply_drift: event targets camera " + event.camera + ", not " +
                                camera.id);
  CameraState next = camera;
  next.scene = event.new_scene;
  next.local_model_acc = std::max(params.acc_floor, camera.local_model_acc - event.acc_drop);
  return next;
}

ModelState seed_model(const SceneVector& scene, double device_acc, const ModelParams& params) {
  const int D = (int)scene.size();
  ecco_ctx* ctx = device(params, D);
  const int id = 1;
  check(ctx, ecco_seed_models(ctx, 1, &id, scene.data(), &device_acc));
  return get(ctx, D);
}

}  // namespace ecco
