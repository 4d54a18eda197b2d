// dropin_learned_test.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The reference-side C++ binding (include/ecco_b200_dropin.hpp) with the
// LEARNED backend, plugged into the UNMODIFIED reference library
// (oracle/_ref/libecco_ref.so): the reference's own WindowAllocation
// (core/src/gpu_allocator.cpp:100-181) drives
//   (a) OracleLearnedBackend: the learned backend's CPU oracle
//       (oracle/ecco_oracle.c: Philox frames and sampler, fp32 SGD step in the
//       FFMA order, correct-count evaluation), one job at a time exactly as
//       JobTrainingBackend (core/src/orchestrator.cpp:31-70) would call a
//       trainer: evaluate = mean over members (string order, summed, / n);
//       train = the micro-window's SGD steps on draws from the batch's
//       source mix;
//   (b) ecco_b200::CudaTrainingBackend over libecco_b200.so with FFMA math,
//       speculative chains on the GPU,
// on the same random jobs, batches and cameras: every micro-window record
// (job, accuracy before, after) and every job's trained weights must be
// identical bit for bit.  Then the reference's group_request
// (core/src/grouping.cpp:18-62) routes requests with an oracle ModelEvalFn
// (the request camera's eval set under the job's oracle weights) and with
// ecco_b200::BatchedRouter (one fused ecco_eval_matrix per pass): the
// assignments must be identical.
//
// Usage: dropin_learned_test [seed] [n_trials]; one line per trial, exit 0
// iff every trial matched.  Run by tests/test_dropin.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "ecco/gpu_allocator.hpp"
#include "ecco/grouping.hpp"
#include "ecco/job.hpp"
#include "ecco_b200_dropin.hpp"
extern "C" {
#include "ecco_oracle.h"
}

using namespace ecco;

namespace {

constexpr int kWindow = 3;

struct OracleStreams {
  orc_lcfg c{};
  std::vector<uint16_t> frames, eval;  // [cam][R][F], [cam][S][F]
  std::vector<int32_t> labels, eval_labels;
  std::vector<double> tp;
};

using Weights = std::vector<std::vector<float>>;  // W1, b1, W2, b2

Weights base_weights(const orc_lcfg& c) {
  Weights w = {std::vector<float>((size_t)c.F * c.H), std::vector<float>(c.H),
               std::vector<float>((size_t)c.H * c.C), std::vector<float>(c.C)};
  orc_init_weights(&c, w[0].data(), w[1].data(), w[2].data(), w[3].data());
  return w;
}

double count_acc(const OracleStreams& o, const Weights& w, int cam) {
  const orc_lcfg& c = o.c;
  const int n = orc_count_correct(&c, o.eval.data() + (size_t)cam * c.S * c.F,
                                  o.eval_labels.data() + (size_t)cam * c.S, c.S, w[0].data(),
                                  w[1].data(), w[2].data(), w[3].data());
  return (double)n / (double)c.S;
}

class OracleLearnedBackend : public TrainingBackend {
 public:
  OracleLearnedBackend(const OracleStreams& o, const JobMap& jobs,
                       const std::map<CameraId, int>& index,
                       const std::map<JobId, TrainingBatchStats>& batches,
                       std::function<TrainingBatchStats(const RetrainJob&)> boot, double floor)
      : o_(o), jobs_(jobs), index_(index), batches_(batches), boot_(std::move(boot)),
        floor_(floor) {
    for (const auto& [id, j] : jobs) w_[id] = base_weights(o.c);
  }
  double evaluate(JobId id) override {
    const RetrainJob& job = jobs_.at(id);
    if (job.members.empty()) return floor_;
    double sum = 0.0;
    for (const auto& m : job.members) sum += count_acc(o_, w_.at(id), index_.at(m.camera));
    return sum / job.member_count();
  }
  void train(JobId id, double gpu_s) override {
    const RetrainJob& job = jobs_.at(id);
    const auto it = batches_.find(id);
    const TrainingBatchStats b = it != batches_.end() ? it->second : boot_(job);
    std::vector<int> src;
    std::vector<double> frac, tp;
    for (const auto& [cam, f] : b.source_mix) {
      src.push_back(index_.at(cam));
      frac.push_back(f);
      tp.push_back(o_.tp[index_.at(cam)]);
    }
    const orc_lcfg& c = o_.c;
    const int steps = orc_learned_steps(&c, b.delivered_frame_rate, b.resolution, b.quality_factor,
                                        gpu_s, (int)src.size(), tp.data());
    const int micro = micro_[id]++;
    Weights& w = w_.at(id);
    std::vector<int> cams(c.B), fr(c.B);
    std::vector<uint16_t> x((size_t)c.B * c.F);
    std::vector<int32_t> y(c.B);
    for (int step = 0; step < steps; ++step) {
      orc_sample(&c, id, (int)src.size(), src.data(), frac.data(), kWindow, micro, step,
                 cams.data(), fr.data());
      for (int s = 0; s < c.B; ++s) {
        const size_t row = (size_t)cams[s] * c.R + fr[s];
        std::memcpy(x.data() + (size_t)s * c.F, o_.frames.data() + row * c.F, 2 * (size_t)c.F);
        y[s] = o_.labels[row];
      }
      orc_sgd_step(&c, x.data(), y.data(), w[0].data(), w[1].data(), w[2].data(), w[3].data());
    }
  }
  const Weights& weights(JobId id) const { return w_.at(id); }

 private:
  const OracleStreams& o_;
  const JobMap& jobs_;
  const std::map<CameraId, int>& index_;
  const std::map<JobId, TrainingBatchStats>& batches_;
  std::function<TrainingBatchStats(const RetrainJob&)> boot_;
  double floor_;
  std::map<JobId, Weights> w_;
  std::map<JobId, int> micro_;
};

bool same(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

char id_buf[32];
std::string cam_id(int i) {
  std::snprintf(id_buf, sizeof(id_buf), "cam%03d", i);
  return id_buf;
}

}  // namespace

int main(int argc, char** argv) {
  const int seed = argc > 1 ? std::atoi(argv[1]) : 1;
  const int trials = argc > 2 ? std::atoi(argv[2]) : 4;
  const int first = argc > 3 ? std::atoi(argv[3]) : 0;
  const ModelParams params;
  ecco_b200::LearnedShape shape;
  shape.feat_dim = 128;
  shape.hidden_dim = 128;
  shape.num_classes = 16;
  shape.minibatch = 64;
  shape.ring_frames = 96;
  shape.eval_samples = 64;
  shape.steps_per_gpu_s = 0.5;
  shape.math = ECCO_MATH_FFMA_EXACT;
  const std::vector<double> fps = {5, 10, 15, 30}, res = {480, 720, 960, 1080};
  int failures = 0;
  for (int trial = first; trial < first + trials; ++trial) {
    std::mt19937_64 rng(seed * 1000003ull + trial);  // test data only
    std::uniform_real_distribution<double> u(0.0, 1.0);
    auto grid = [&](double step) { return std::round(u(rng) / step) * step; };
    const int n_cams = 6 + (int)(u(rng) * 14), n_jobs = 2 + (int)(u(rng) * 5);
    std::map<CameraId, CameraState> cams;
    for (int i = 0; i < n_cams; ++i) {
      CameraState c;
      c.id = cam_id(i);
      c.scene = {grid(0.1), grid(0.1)};
      c.gpu_pixel_throughput = 8.192e6;
      cams[c.id] = c;
    }
    // the CPU oracle's streams, camera index = std::map order (as the Device)
    OracleStreams o;
    o.c = {shape.feat_dim, shape.hidden_dim, shape.num_classes, 2, shape.minibatch,
           shape.ring_frames, shape.eval_samples, shape.sgd_lr, shape.feature_noise,
           shape.steps_per_gpu_s, shape.seed};
    std::vector<float> P((size_t)o.c.C * o.c.F), Q((size_t)o.c.C * o.c.D * o.c.F);
    orc_prototypes(&o.c, P.data(), Q.data());
    o.frames.resize((size_t)n_cams * o.c.R * o.c.F);
    o.labels.resize((size_t)n_cams * o.c.R);
    o.eval.resize((size_t)n_cams * o.c.S * o.c.F);
    o.eval_labels.resize((size_t)n_cams * o.c.S);
    std::map<CameraId, int> index;
    {
      int i = 0;
      for (const auto& [id, c] : cams) {
        index[id] = i;
        o.tp.push_back(c.gpu_pixel_throughput);
        orc_gen_frames(&o.c, P.data(), Q.data(), i, kWindow, 0, o.c.R, c.scene.data(),
                       o.frames.data() + (size_t)i * o.c.R * o.c.F,
                       o.labels.data() + (size_t)i * o.c.R);
        orc_gen_frames(&o.c, P.data(), Q.data(), i, kWindow, 1, o.c.S, c.scene.data(),
                       o.eval.data() + (size_t)i * o.c.S * o.c.F,
                       o.eval_labels.data() + (size_t)i * o.c.S);
        ++i;
      }
    }
    JobMap jobs;
    std::map<JobId, TrainingBatchStats> batches;
    for (int j = 0; j < n_jobs; ++j) {
      RetrainJob job;
      job.id = 3 * j + 2;
      const int nm = 1 + (int)(u(rng) * 4);
      for (int k = 0; k < nm; ++k) {
        RetrainRequest r;
        r.camera = cam_id((int)(u(rng) * n_cams));
        if (job.find_member(r.camera)) continue;
        r.subsamples = cams.at(r.camera).scene;
        job.insert_member(r);
      }
      if (u(rng) < 0.7) {
        TrainingBatchStats b;
        b.delivered_frame_rate = fps[(int)(u(rng) * fps.size())] * job.member_count();
        b.resolution = res[(int)(u(rng) * res.size())];
        b.quality_factor = 0.5 + 0.5 * u(rng);
        double tot = 0.0;
        std::map<CameraId, double> w;
        for (const auto& m : job.members) w[m.camera] = 0.2 + u(rng);
        if (u(rng) < 0.3) w[cam_id((int)(u(rng) * n_cams))] += 0.5;
        for (const auto& [c, x] : w) tot += x;
        double acc = 0.0;
        int left = (int)w.size();
        for (const auto& [c, x] : w) {
          b.source_mix[c] = --left ? x / tot : 1.0 - acc;
          acc += b.source_mix[c];
        }
        batches[job.id] = b;
      }
      jobs[job.id] = job;
    }
    auto boot = [&](const RetrainJob& job) {
      TrainingBatchStats b;  // bootstrap_batch (orchestrator.cpp:193-203)
      b.delivered_frame_rate = 15.0 * job.member_count();
      b.resolution = 720;
      b.quality_factor = 1.0;
      for (const auto& m : job.members) b.source_mix[m.camera] = 1.0 / job.member_count();
      return b;
    };
    AllocatorConfig cfg;
    cfg.micro_windows = n_jobs + (int)(u(rng) * 3 * n_jobs);
    cfg.micro_window_duration_s = 2.0 + 6.0 * u(rng);
    cfg.gpu_count = 1 + (int)(u(rng) * 2);
    const SchedulePolicy pol = trial % 3 == 0   ? SchedulePolicy::ecco
                               : trial % 3 == 1 ? SchedulePolicy::total_acc_greedy
                                                : SchedulePolicy::naive;
    std::vector<JobView> views;
    for (const auto& [id, j] : jobs) views.push_back({id, j.member_count()});

    OracleLearnedBackend orc(o, jobs, index, batches, boot, params.acc_floor);
    WindowAllocation wa(views, cfg, pol);
    wa.run_initial_pass(orc);
    wa.run_remaining(orc);

    ecco_b200::Device dev(params, shape, 2, 64, n_cams);
    dev.set_cameras(cams);
    dev.generate_frames(kWindow);
    if (std::getenv("ECCO_DROPIN_VERBOSE")) {  // inputs of the two backends before any training
      std::vector<uint16_t> fr(o.frames.size()), ev(o.eval.size());
      std::vector<int32_t> lb(o.labels.size()), el(o.eval_labels.size());
      ecco_b200::check(dev.ctx(), ecco_read_frames(dev.ctx(), n_cams, fr.data(), lb.data(),
                                                   ev.data(), el.data()));
      std::printf("  frames equal %d %d %d %d\n", fr == o.frames, lb == o.labels, ev == o.eval,
                  el == o.eval_labels);
      for (const auto& [id, j] : jobs) {
        dev.ensure_model(id);
        std::vector<int> mo = {0}, mc;
        for (const auto& m : j.members) mc.push_back(index.at(m.camera));
        mo.push_back((int)mc.size());
        double got = 0.0;
        ecco_b200::check(dev.ctx(), ecco_eval_jobs(dev.ctx(), 1, &id, mo.data(), mc.data(), &got));
        OracleLearnedBackend fresh(o, jobs, index, batches, boot, params.acc_floor);
        std::printf("  job %d base eval: device %.17g oracle %.17g\n", (int)id, got,
                    fresh.evaluate(id));
      }
    }
    JobMap jb = jobs;
    ecco_b200::CudaTrainingBackend cuda(dev, jb, batches, boot,
                                        cfg.gpu_count * cfg.micro_window_duration_s, 2, kWindow);
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
          !same(ra[i].acc_after, rb[i].acc_after)) {
        if (!bad)
          std::printf("  micro %zu: oracle job %d %.17g -> %.17g, device job %d %.17g -> %.17g\n", i,
                      (int)ra[i].job, ra[i].acc_before, ra[i].acc_after, (int)rb[i].job,
                      rb[i].acc_before, rb[i].acc_after);
        ++bad;
      }
    for (const auto& [id, j] : jobs) {
      Weights got = {std::vector<float>((size_t)o.c.F * o.c.H), std::vector<float>(o.c.H),
                     std::vector<float>((size_t)o.c.H * o.c.C), std::vector<float>(o.c.C)};
      ecco_b200::check(dev.ctx(), ecco_get_weights(dev.ctx(), id, got[0].data(), got[1].data(),
                                                   got[2].data(), got[3].data()));
      const Weights& want = orc.weights(id);
      for (int t = 0; t < 4; ++t)
        if (std::memcmp(got[t].data(), want[t].data(), 4 * got[t].size()) != 0) {
          std::printf("  job %d tensor %d differs\n", (int)id, t);
          ++bad;
        }
    }

    // routing: group_request over the trained jobs, oracle eval vs BatchedRouter
    GroupingConfig gcfg;
    gcfg.delta_m = 1e9;  // every job passes the spatial filter
    std::vector<RetrainRequest> pending;
    for (int q = 0; q < 6; ++q) {
      RetrainRequest r;
      r.camera = cam_id((int)(u(rng) * n_cams));
      bool dup = false;
      for (const auto& p : pending) dup |= p.camera == r.camera;
      if (dup) continue;
      r.subsamples = cams.at(r.camera).scene;
      r.acc = 0.05 + 0.2 * u(rng);
      pending.push_back(r);
    }
    JobMap ga, gb;  // the trained jobs without the pending cameras
    for (const auto& [id, j] : jobs) {
      RetrainJob k = j;
      k.members.clear();
      for (const auto& m : j.members) {
        bool p = false;
        for (const auto& r : pending) p |= r.camera == m.camera;
        if (!p) k.insert_member(m);
      }
      if (!k.members.empty()) ga[id] = k;
    }
    gb = ga;
    std::map<JobId, Weights> ow;
    for (const auto& [id, j] : ga) ow[id] = orc.weights(id);
    const RetrainRequest* cur = nullptr;
    ModelEvalFn eval_orc = [&](const RetrainJob& job, const SceneVector&) {
      auto it = ow.find(job.id);
      if (it == ow.end()) it = ow.emplace(job.id, base_weights(o.c)).first;
      return count_acc(o, it->second, index.at(cur->camera));
    };
    ecco_b200::BatchedRouter router(dev, gb, pending);
    JobId next_a = 1000, next_b = 1000;
    int routed = 0;
    for (const auto& r : pending) {
      cur = &r;
      const GroupAssignment a = group_request(ga, r, gcfg, params, eval_orc, next_a);
      router.route_as(r);
      const GroupAssignment b = group_request(gb, r, gcfg, params, router.eval_fn(), next_b);
      if (b.created) router.created(gb.at(b.job));
      if (a.job != b.job || a.created != b.created || !same(a.acc, b.acc)) {
        std::printf("  route %s: oracle job %d (%d) %.17g, device job %d (%d) %.17g\n",
                    r.camera.c_str(), (int)a.job, (int)a.created, a.acc, (int)b.job,
                    (int)b.created, b.acc);
        ++bad;
      }
      ++routed;
    }
    if (std::getenv("ECCO_DROPIN_VERBOSE")) {
      for (const auto& [id, j] : jobs) {
        std::printf("  job %d members", (int)id);
        for (const auto& m : j.members) std::printf(" %s(%d)", m.camera.c_str(), index.at(m.camera));
        std::printf(" | oracle eval %.17g\n", orc.evaluate(id));
      }
    }
    std::printf("trial %d: %zu micro-windows, %d jobs, %d routed requests, policy %d: %s\n", trial,
                ra.size(), n_jobs, routed, (int)pol, bad ? "MISMATCH" : "identical");
    failures += bad != 0;
  }
  return failures ? 1 : 0;
}
