// dropin_test.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The reference-side C++ binding (include/ecco_b200_dropin.hpp) plugged into
// the UNMODIFIED reference library (oracle/_ref/libecco_ref.so, built from
// /root/reference/proj/core): the reference's own WindowAllocation
// (core/src/gpu_allocator.cpp:100-181) drives
//   (a) RefBackend, a restatement of the reference's JobTrainingBackend
//       (core/src/orchestrator.cpp:31-70, which lives in an anonymous
//       namespace there) over the reference's eval / train_step, and
//   (b) ecco_b200::CudaTrainingBackend over libecco_b200.so on the GPU,
// on the same randomly generated jobs, batches and cameras; the schedules
// (every micro-window record) and the trained models must be identical bit
// for bit.  The reference's group_request (core/src/grouping.cpp:18-62) is
// then run with the reference's eval_job_on_scene, with
// ecco_b200::make_eval_fn and with ecco_b200::BatchedRouter (one fused
// evaluation matrix per routing pass), and every camera's profile table is built by the
// reference's build_profile_table + make_accuracy_probe and by
// ecco_b200::build_profile_tables; assignments and rows must be identical.
//
// Built by oracle/Makefile (target `dropin`, where /root/reference exists)
// into oracle/_ref/dropin_test; run by tests/test_dropin.py on the GPU box.
// Usage: dropin_test [seed] [n_trials]; prints one line per trial, exit 0 iff
// every trial matched.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "ecco/accuracy_model.hpp"
#include "ecco/gpu_allocator.hpp"
#include "ecco/grouping.hpp"
#include "ecco/job.hpp"
#include "ecco/transmission.hpp"
#include "ecco_b200_dropin.hpp"

using namespace ecco;

namespace {

class RefBackend : public TrainingBackend {
 public:
  RefBackend(JobMap& jobs, const std::map<CameraId, CameraState>& cams,
             const std::map<JobId, TrainingBatchStats>& batches,
             std::function<TrainingBatchStats(const RetrainJob&)> boot, const ModelParams& p)
      : jobs_(jobs), cams_(cams), batches_(batches), boot_(std::move(boot)), p_(p) {}
  double evaluate(JobId id) override {
    const RetrainJob& job = jobs_.at(id);
    if (job.members.empty()) return p_.acc_floor;
    double sum = 0.0;
    for (const auto& m : job.members) sum += eval(job.model, cams_.at(m.camera), p_);
    return sum / job.member_count();
  }
  void train(JobId id, double gpu_s) override {
    RetrainJob& job = jobs_.at(id);
    const auto it = batches_.find(id);
    const TrainingBatchStats b = it != batches_.end() ? it->second : boot_(job);
    std::vector<CameraState> src;
    for (const auto& e : b.source_mix) src.push_back(cams_.at(e.first));
    job.model = train_step(job.model, b, gpu_s, src, p_);
  }

 private:
  JobMap& jobs_;
  const std::map<CameraId, CameraState>& cams_;
  const std::map<JobId, TrainingBatchStats>& batches_;
  std::function<TrainingBatchStats(const RetrainJob&)> boot_;
  const ModelParams& p_;
};

bool same(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

bool same_model(const ModelState& a, const ModelState& b) {
  if (a.clusters.size() != b.clusters.size() || a.centroid.size() != b.centroid.size())
    return false;
  for (size_t k = 0; k < a.clusters.size(); ++k) {
    if (!same(a.proficiency[k], b.proficiency[k])) return false;
    for (size_t d = 0; d < a.clusters[k].size(); ++d)
      if (!same(a.clusters[k][d], b.clusters[k][d])) return false;
  }
  for (size_t d = 0; d < a.centroid.size(); ++d)
    if (!same(a.centroid[d], b.centroid[d])) return false;
  return true;
}

char id_buf[32];
std::string cam_id(int i) {
  std::snprintf(id_buf, sizeof(id_buf), "cam%03d", i);
  return id_buf;
}

}  // namespace

int main(int argc, char** argv) {
  const int seed = argc > 1 ? std::atoi(argv[1]) : 1;
  const int trials = argc > 2 ? std::atoi(argv[2]) : 6;
  const ModelParams params;
  const std::vector<double> fps = {1, 2, 5, 10, 15, 30}, res = {360, 480, 720, 960, 1080};
  int failures = 0;
  for (int trial = 0; trial < trials; ++trial) {
    std::mt19937_64 rng(seed * 1000003ull + trial);  // test data only
    std::uniform_real_distribution<double> u(0.0, 1.0);
    auto grid = [&](double step) { return std::round(u(rng) / step) * step; };
    const int n_cams = 8 + (int)(u(rng) * 40), n_jobs = 2 + (int)(u(rng) * 10);
    std::map<CameraId, CameraState> cams;
    for (int i = 0; i < n_cams; ++i) {
      CameraState c;
      c.id = cam_id(i);
      c.scene = {grid(0.05), grid(0.05)};
      c.gpu_pixel_throughput = 8.192e6;
      cams[c.id] = c;
    }
    JobMap jobs;
    std::map<JobId, TrainingBatchStats> batches;
    for (int j = 0; j < n_jobs; ++j) {
      RetrainJob job;
      job.id = 3 * j + 1;
      const int nm = 1 + (int)(u(rng) * 5);
      for (int k = 0; k < nm; ++k) {
        RetrainRequest r;
        r.camera = cam_id((int)(u(rng) * n_cams));
        if (job.find_member(r.camera)) continue;
        r.subsamples = cams.at(r.camera).scene;
        job.insert_member(r);
      }
      job.model = seed_model(cams.at(job.members.front().camera).scene, 0.1 + 0.3 * u(rng),
                             params);
      if (u(rng) < 0.7) {  // a batch with a source mix over members (+ maybe one outsider)
        TrainingBatchStats b;
        b.delivered_frame_rate = fps[(int)(u(rng) * fps.size())] * job.member_count();
        b.resolution = res[(int)(u(rng) * res.size())];
        b.quality_factor = 0.3 + 0.7 * u(rng);
        double tot = 0.0;
        std::map<CameraId, double> w;
        for (const auto& m : job.members) w[m.camera] = 0.2 + u(rng);
        if (u(rng) < 0.3) w[cam_id((int)(u(rng) * n_cams))] += 0.5;
        for (const auto& [c, x] : w) tot += x;
        double acc = 0.0;
        int left = (int)w.size();
        for (const auto& [c, x] : w) {  // fractions summing to exactly 1
          b.source_mix[c] = --left ? x / tot : 1.0 - acc;
          acc += b.source_mix[c];
        }
        batches[job.id] = b;
      }
      jobs[job.id] = job;
    }
    auto boot = [&](const RetrainJob& job) {
      TrainingBatchStats b;  // bootstrap_batch (orchestrator.cpp:193-203)
      b.delivered_frame_rate = fps.front();
      b.resolution = res.front();
      b.quality_factor = 1.0;
      for (const auto& m : job.members) b.source_mix[m.camera] = 1.0 / job.member_count();
      return b;
    };
    AllocatorConfig cfg;
    cfg.micro_windows = n_jobs + (int)(u(rng) * 3 * n_jobs);
    cfg.micro_window_duration_s = 2.0 + 8.0 * u(rng);
    cfg.gpu_count = 1 + (int)(u(rng) * 2);
    const SchedulePolicy pol = trial % 3 == 0   ? SchedulePolicy::ecco
                               : trial % 3 == 1 ? SchedulePolicy::total_acc_greedy
                                                : SchedulePolicy::naive;
    std::vector<JobView> views;
    for (const auto& [id, j] : jobs) views.push_back({id, j.member_count()});

    JobMap ja = jobs, jb = jobs;
    RefBackend ref(ja, cams, batches, boot, params);
    WindowAllocation wa(views, cfg, pol);
    wa.run_initial_pass(ref);
    wa.run_remaining(ref);

    ecco_b200::Device dev(params, 2, 32, 64, n_cams);
    dev.set_cameras(cams);
    ecco_b200::CudaTrainingBackend cuda(dev, jb, batches, boot,
                                        cfg.gpu_count * cfg.micro_window_duration_s, 2);
    WindowAllocation wb(views, cfg, pol);
    wb.run_initial_pass(cuda);
    wb.run_remaining(cuda);
    cuda.finish();

    int bad = 0;
    const auto& ra = wa.schedule().records;
    const auto& rb = wb.schedule().records;
    if (ra.size() != rb.size()) ++bad;
    for (size_t i = 0; i < ra.size() && i < rb.size(); ++i)
      if (ra[i].job != rb[i].job || !same(ra[i].acc_before, rb[i].acc_before) ||
          !same(ra[i].acc_after, rb[i].acc_after))
        ++bad;
    for (const auto& [id, j] : ja)
      if (!same_model(j.model, jb.at(id).model)) ++bad;

    // ModelEvalFn: route fresh requests through the reference's group_request
    GroupingConfig gcfg;
    gcfg.delta_m = 1e9;  // every job passes the spatial filter
    ModelEvalFn eval_ref = [&](const RetrainJob& job, const SceneVector& scene) {
      CameraState probe;
      probe.scene = scene;
      return eval(job.model, probe, params);
    };
    const ModelEvalFn eval_b200 = ecco_b200::make_eval_fn(dev);
    JobMap ga = ja, gb = ja, gc = ja;
    JobId next_a = 1000, next_b = 1000, next_c = 1000;
    int routed = 0;
    // requests for cameras of the table (the device indexes probes by camera)
    std::vector<RetrainRequest> pending;
    for (int q = 0; q < 12; ++q) {
      RetrainRequest r;
      r.camera = cam_id((int)(u(rng) * n_cams));
      bool dup = false;
      for (const auto& p : pending) dup |= p.camera == r.camera;
      for (const auto& [id, j] : ga) dup |= j.find_member(r.camera) != nullptr;
      if (dup) continue;
      r.subsamples = {grid(0.05), grid(0.05)};
      r.acc = 0.1 + 0.3 * u(rng);
      pending.push_back(r);
    }
    ecco_b200::BatchedRouter router(dev, gc, pending);  // one fused matrix for the pass
    for (const auto& r : pending) {
      const GroupAssignment a = group_request(ga, r, gcfg, params, eval_ref, next_a);
      const GroupAssignment b = group_request(gb, r, gcfg, params, eval_b200, next_b);
      router.route_as(r);
      const GroupAssignment c = group_request(gc, r, gcfg, params, router.eval_fn(), next_c);
      if (c.created) router.created(gc.at(c.job));
      if (a.job != b.job || a.created != b.created || !same(a.acc, b.acc)) ++bad;
      if (a.job != c.job || a.created != c.created || !same(a.acc, c.acc)) ++bad;
      ++routed;
    }
    // ProbeFn: the profile tables of every camera (Simulation::profile's grid
    // and levels, orchestrator.cpp:94-116), reference vs one device launch
    std::vector<double> levels;
    for (int k = 1; k <= cfg.micro_windows; ++k)
      levels.push_back(k * cfg.gpu_count * cfg.micro_window_duration_s);
    const auto grid_cfgs = make_config_grid({1, 2, 5, 10, 15}, {360, 480, 720, 960});
    ProfilerOptions popts;
    popts.window_duration_s = cfg.micro_windows * cfg.micro_window_duration_s;
    popts.bias = trial % 2 ? ProfileBias::frame_rate : ProfileBias::resolution;
    std::vector<CameraState> cam_list;
    for (const auto& [id, c] : cams) cam_list.push_back(c);
    const auto tables = ecco_b200::build_profile_tables(dev, cam_list, levels, grid_cfgs, popts,
                                                        1e6, 0.1);
    int rows = 0;
    for (size_t i = 0; i < cam_list.size(); ++i) {
      const ProfileTable want = build_profile_table(
          cam_list[i], levels, grid_cfgs, make_accuracy_probe(cam_list[i], params, 1e6, 0.1), popts);
      if (want.rows.size() != tables[i].rows.size()) ++bad;
      for (size_t l = 0; l < want.rows.size() && l < tables[i].rows.size(); ++l, ++rows) {
        const auto &w = want.rows[l], &g = tables[i].rows[l];
        if (!same(w.budget_gpu_s, g.budget_gpu_s) || !same(w.config.frame_rate, g.config.frame_rate) ||
            !same(w.config.resolution, g.config.resolution) || w.feasible != g.feasible)
          ++bad;
      }
    }
    std::printf("trial %d: %zu micro-windows, %d jobs, %d routed requests, %d profile rows, "
                "policy %d: %s\n", trial, ra.size(), n_jobs, routed, rows, (int)pol,
                bad ? "MISMATCH" : "identical");
    failures += bad != 0;
  }
  return failures ? 1 : 0;
}
