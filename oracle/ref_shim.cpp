// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, compiled by
// oracle/Makefile from the sources under /root/reference/proj/core into
// oracle/_ref/libecco_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's reference / cpu_baseline legs load it, as the checker or as the
// timed reference CPU path; the product never links it.
//
// Source ids: train_step's source_mix is a std::map<CameraId,double>; the
// shim names sources "s0000", "s0001", ... so map order equals index order.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "ecco/accuracy_model.hpp"
#include "ecco/gpu_allocator.hpp"
#include "ecco/grouping.hpp"
#include "ecco/metrics.hpp"
#include "ecco/netsim.hpp"
#include "ecco/orchestrator.hpp"
#include "ecco/scenario.hpp"
#include "ecco/transmission.hpp"

using namespace ecco;

namespace {

thread_local std::string g_err;

ModelParams mp(const double* p) {
  ModelParams m;
  m.learning_rate_k = p[0];
  m.similarity_lambda = p[1];
  m.acc_floor = p[2];
  m.acc_ceil = p[3];
  m.cluster_similarity_threshold = p[4];
  return m;
}

ModelState unpack(int k, const double* clusters, const double* prof, int clen,
                  const double* centroid, int d) {
  ModelState m;
  for (int c = 0; c < k; ++c) {
    m.clusters.emplace_back(clusters + c * d, clusters + (c + 1) * d);
    m.proficiency.push_back(prof[c]);
  }
  if (clen > 0) m.centroid.assign(centroid, centroid + clen);
  return m;
}

std::string src_id(int i) {
  char buf[16];
  std::snprintf(buf, sizeof buf, "s%04d", i);
  return buf;
}

int code_of(const std::exception& e) {
  if (dynamic_cast<const InfeasibleScheduleError*>(&e)) return 3;
  if (dynamic_cast<const SchemaError*>(&e)) return 4;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::logic_error*>(&e)) return 2;
  return 6;
}

// TrainingBackend replaying fixed per-job accuracy trajectories: train()
// advances the job's cursor, evaluate() reads traj[cursor].  Used to drive
// the reference WindowAllocation with trajectories produced elsewhere.
class TrajectoryBackend : public TrainingBackend {
 public:
  std::map<JobId, std::vector<double>> traj;
  std::map<JobId, int> cursor;
  double evaluate(JobId id) override {
    const auto& t = traj.at(id);
    return t.at(std::min<std::size_t>(cursor[id], t.size() - 1));
  }
  void train(JobId id, double) override { ++cursor[id]; }
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

double ref_similarity(const double* a, const double* b, int d, double lambda) {
  return similarity(SceneVector(a, a + d), SceneVector(b, b + d), lambda);
}

int ref_find_cluster(int k, const double* clusters, const double* prof, int d,
                     const double* scene, const double* params) {
  ModelState m = unpack(k, clusters, prof, 0, nullptr, d);
  return find_cluster(m, SceneVector(scene, scene + d), mp(params));
}

double ref_eval(int k, const double* clusters, const double* prof, int clen,
                const double* centroid, int d, const double* scene, const double* params) {
  ModelState m = unpack(k, clusters, prof, clen, centroid, d);
  CameraState cam;
  cam.scene.assign(scene, scene + d);
  return eval(m, cam, mp(params));
}

// N x G matrix of eval(model_j, scene_i); models packed with stride kmax.
// Returns elapsed seconds (the reference CPU eval-matrix baseline).
double ref_eval_matrix(int n, const double* scenes, int g, const int* ks,
                       const double* clusters, const double* profs, const int* clens,
                       const double* centroids, int kmax, int d, const double* params,
                       double* out) {
  std::vector<ModelState> models;
  for (int j = 0; j < g; ++j)
    models.push_back(unpack(ks[j], clusters + (size_t)j * kmax * d, profs + (size_t)j * kmax,
                            clens[j], centroids + (size_t)j * d, d));
  const ModelParams p = mp(params);
  std::vector<CameraState> cams(n);
  for (int i = 0; i < n; ++i) cams[i].scene.assign(scenes + (size_t)i * d, scenes + (size_t)(i + 1) * d);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < g; ++j) out[(size_t)i * g + j] = eval(models[j], cams[i], p);
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// train_step on a packed model (capacity kmax clusters).  Sources are
// scenes/throughputs/fractions in source order.  Returns 0 or an error code.
int ref_train_step(int* k, double* clusters, double* prof, int* clen, double* centroid,
                   int kmax, int d, double fps, double res, double quality, double gpu_s,
                   int n_src, const double* src_scenes, const double* src_tp,
                   const double* src_frac, const double* params) {
  try {
    ModelState m = unpack(*k, clusters, prof, *clen, centroid, d);
    TrainingBatchStats b;
    b.delivered_frame_rate = fps;
    b.resolution = res;
    b.quality_factor = quality;
    std::vector<CameraState> cams;
    for (int i = 0; i < n_src; ++i) {
      b.source_mix[src_id(i)] = src_frac[i];
      CameraState c;
      c.id = src_id(i);
      c.scene.assign(src_scenes + (size_t)i * d, src_scenes + (size_t)(i + 1) * d);
      c.gpu_pixel_throughput = src_tp[i];
      cams.push_back(c);
    }
    ModelState out = train_step(m, b, gpu_s, cams, mp(params));
    if ((int)out.clusters.size() > kmax) {
      g_err = "cluster capacity exceeded";
      return 1;
    }
    *k = (int)out.clusters.size();
    for (int c = 0; c < *k; ++c) {
      std::copy(out.clusters[c].begin(), out.clusters[c].end(), clusters + c * d);
      prof[c] = out.proficiency[c];
    }
    *clen = (int)out.centroid.size();
    std::copy(out.centroid.begin(), out.centroid.end(), centroid);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

int ref_seed_model(const double* scene, int d, double acc, const double* params,
                   double* cluster_out, double* prof_out) {
  ModelState m = seed_model(SceneVector(scene, scene + d), acc, mp(params));
  std::copy(m.clusters[0].begin(), m.clusters[0].end(), cluster_out);
  *prof_out = m.proficiency[0];
  return 0;
}

// build_profile_table + make_accuracy_probe for one camera.
int ref_profile_table(const double* scene, int d, double throughput, int bias, int n_levels,
                      const double* levels, int n_grid, const double* grid_fps,
                      const double* grid_res, double window_s, double tie_eps,
                      double ref_rate, double bpp_ref, const double* params, double* out_budget,
                      double* out_fps, double* out_res, unsigned char* out_feasible) {
  try {
    CameraState cam;
    cam.id = "cam";
    cam.scene.assign(scene, scene + d);
    cam.gpu_pixel_throughput = throughput;
    std::vector<SamplingConfig> grid;
    for (int i = 0; i < n_grid; ++i) grid.push_back({grid_fps[i], grid_res[i]});
    ProfilerOptions opts;
    opts.window_duration_s = window_s;
    opts.bias = bias ? ProfileBias::frame_rate : ProfileBias::resolution;
    opts.tie_epsilon = tie_eps;
    const ProbeFn probe = make_accuracy_probe(cam, mp(params), ref_rate, bpp_ref);
    const ProfileTable t =
        build_profile_table(cam, std::vector<double>(levels, levels + n_levels), grid, probe, opts);
    for (std::size_t r = 0; r < t.rows.size(); ++r) {
      out_budget[r] = t.rows[r].budget_gpu_s;
      out_fps[r] = t.rows[r].config.frame_rate;
      out_res[r] = t.rows[r].config.resolution;
      out_feasible[r] = t.rows[r].feasible ? 1 : 0;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// The reference WindowAllocation driven by fixed accuracy trajectories
// (traj: n_jobs rows of traj_len accuracies, row j for job_ids[j]).
// policy 0 ecco, 1 naive, 2 total_acc_greedy.  Writes W records.
int ref_allocate_trajectories(int n_jobs, const int* job_ids, const int* members,
                              const double* traj, int traj_len, double alpha, double beta,
                              int micro_windows, double micro_s, int gpu_count, int bonus,
                              int policy, int* out_job, double* out_before, double* out_after,
                              double* out_initial_scores) {
  try {
    AllocatorConfig cfg;
    cfg.obj_alpha = alpha;
    cfg.size_exponent_beta = beta;
    cfg.micro_windows = micro_windows;
    cfg.micro_window_duration_s = micro_s;
    cfg.gpu_count = gpu_count;
    cfg.fairness_bonus = bonus != 0;
    std::vector<JobView> views;
    TrajectoryBackend be;
    for (int j = 0; j < n_jobs; ++j) {
      views.push_back({job_ids[j], members[j]});
      be.traj[job_ids[j]].assign(traj + (size_t)j * traj_len, traj + (size_t)(j + 1) * traj_len);
    }
    const SchedulePolicy pol = policy == 0   ? SchedulePolicy::ecco
                               : policy == 1 ? SchedulePolicy::naive
                                             : SchedulePolicy::total_acc_greedy;
    WindowAllocation alloc(views, cfg, pol);
    alloc.run_initial_pass(be);
    if (out_initial_scores) {
      int j = 0;
      for (const auto& [id, s] : alloc.initial_scores()) out_initial_scores[j++] = s;
    }
    alloc.run_remaining(be);
    const auto& recs = alloc.schedule().records;
    for (std::size_t i = 0; i < recs.size(); ++i) {
      out_job[i] = recs[i].job;
      out_before[i] = recs[i].acc_before;
      out_after[i] = recs[i].acc_after;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// Runs a scenario end to end through Simulation.  policy_override < 0 keeps
// the file's policy.  Writes trace.csv and summary.json bytes (truncated to
// the capacities; the return value carries the full sizes via *_len).
int ref_run_scenario(const char* json, int policy_override, char* trace, size_t trace_cap,
                     size_t* trace_len, char* summary, size_t summary_cap,
                     size_t* summary_len) {
  try {
    ScenarioConfig cfg = parse_scenario_json(json);
    if (policy_override == 0) cfg.policy = SchedulePolicy::ecco;
    if (policy_override == 1) cfg.policy = SchedulePolicy::naive;
    if (policy_override == 2) cfg.policy = SchedulePolicy::total_acc_greedy;
    Simulation sim(cfg);
    sim.run();
    std::ostringstream os;
    sim.trace().write_csv(os);
    const std::string t = os.str();
    const std::string s = sim.summary_json();
    *trace_len = t.size();
    *summary_len = s.size();
    std::memcpy(trace, t.data(), std::min(trace_cap, t.size()));
    std::memcpy(summary, s.data(), std::min(summary_cap, s.size()));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// Times Simulation::step_window for a scenario: per-window wall seconds in
// out_s (n_windows entries).  The reference CPU baseline of the window loop.
int ref_time_windows(const char* json, int max_windows, double* out_s, int* n_run) {
  try {
    ScenarioConfig cfg = parse_scenario_json(json);
    Simulation sim(cfg);
    int w = 0;
    while (w < max_windows) {
      auto t0 = std::chrono::steady_clock::now();
      if (!sim.step_window()) break;
      out_s[w++] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    *n_run = w;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// ref_time_windows that also returns the run's trace.csv bytes (one run
// serves both the timing and the trace comparison).
int ref_time_windows_trace(const char* json, int max_windows, double* out_s, int* n_run,
                           char* trace, size_t trace_cap, size_t* trace_len) {
  try {
    ScenarioConfig cfg = parse_scenario_json(json);
    Simulation sim(cfg);
    int w = 0;
    while (w < max_windows) {
      auto t0 = std::chrono::steady_clock::now();
      if (!sim.step_window()) break;
      out_s[w++] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    *n_run = w;
    std::ostringstream os;
    sim.trace().write_csv(os);
    const std::string t = os.str();
    *trace_len = t.size();
    std::memcpy(trace, t.data(), std::min(trace_cap, t.size()));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// ecco::simulate_window (netsim.cpp:64-94) on n flows "f00000".. with local
// caps (<= 0 = absent); mean rates in flow order.  Returns 0 or the error code.
int ref_simulate_window(int n, const double* alpha, const double* beta, const double* caps,
                        double capacity, double rtt_s, double duration_s, double* mean) {
  try {
    std::vector<FlowParams> flows(n);
    NetTopology topo;
    topo.shared_capacity_bps = capacity;
    topo.rtt_s = rtt_s;
    char id[16];
    for (int i = 0; i < n; ++i) {
      std::snprintf(id, sizeof(id), "f%05d", i);
      flows[i].id = id;
      flows[i].alpha_bps_per_rtt = alpha[i];
      flows[i].beta = beta[i];
      if (caps[i] > 0.0) topo.local_caps_bps[id] = caps[i];
    }
    const FlowTrace t = simulate_window(flows, topo, duration_s);
    for (int i = 0; i < n; ++i) mean[i] = t.mean_rate_bps.at(flows[i].id);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

}  // extern "C"
