// sim.cpp -- host C++ window driver over the C-ABI.
//
// A restatement of the reference control loop (Simulation::step_window,
// proj/core/src/orchestrator.cpp:211-413) in which every accuracy-model call
// is served by the batched device entry points of include/ecco_b200.h:
//
//   routing / reroute (grouping.cpp:18-62, 64-121)
//       -> one ecco_eval_pairs over the filter-surviving (request, job)
//          pairs plus the provisional columns of jobs the pass may create;
//          the host commits requests in order ("device proposes, host
//          commits").
//   WindowAllocation (gpu_allocator.cpp:100-181) via JobTrainingBackend
//       -> ecco_train_trajectories for all jobs at once (initial pass, then
//          speculative chains); the greedy loop is replayed on the host on
//          the returned accuracies, which is exactly what the allocator
//          observes (tests/support/scripted_backend.hpp shows decisions depend
//          only on these numbers); ecco_commit keeps the granted prefix.
//   window-end accuracies (orchestrator.cpp:328-352) -> ecco_eval_pairs.
//   profile tables (orchestrator.cpp:94-116)          -> ecco_profile_tables.
//
// The transmission controller, AIMD network model, trace and summary stay
// scalar host code with the reference's arithmetic, so the trace of a
// parametric run is byte-identical to the reference's.
#include <immintrin.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <optional>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include <json.hpp>

#include "ecco_b200.h"

namespace {

using nlohmann::json;

// AIMD share of a learned job whose estimate_shares share is 0 (see the
// set_aimd_params call in step_window).
constexpr double kLearnedShareFloor = 1e-3;

struct SimError {
  ecco_status code;
  std::string msg;
};
[[noreturn]] void fail(ecco_status c, const std::string& m) { throw SimError{c, m}; }
[[noreturn]] void schema(const std::string& path, const std::string& what) {
  fail(ECCO_ERR_SCHEMA, path + ": " + what);
}
void check(ecco_ctx* ctx, ecco_status st) {
  if (st != ECCO_OK) fail(st, ecco_last_error(ctx));
}

// ------------------------------------------------------------- netsim --
namespace ecco_netsim {

// simulate_window's per-flow mean rates (netsim.cpp:64-94, aimd_step
// :45-62), bit-identical to the reference.  The only cross-flow coupling is
// the congestion test `sum(rates) >= capacity` with the sum taken
// sequentially in flow order; that sum is computed here with eight
// interleaved accumulators (vectorisable) and the sequential sum is redone
// only when the two could fall on different sides of the capacity: both
// differ from the exact sum by at most (n + n/8 + 3) u sum(|rate|) (rates
// are non-negative), so outside a 2.5 n u sum margin the decision is the
// reference's.  Returns the number of steps that needed the sequential sum.
// One pass over the flows per RTT: the previous decision's update, the
// measurement sum, then this step's clamp to the local cap and its partial
// sums (accumulator k takes flows f = k mod 8) -- per flow, exactly
// aimd_step's operations in its order.  An AVX2 version (IEEE add / mul / min
// lanes, no contraction) and a scalar one compute the same bits.
template <bool kCongested>
void netsim_pass(size_t n, double* r, const double* alpha, const double* beta,
                 const double* caps, double* mean, bool meas, double acc[8]) {
  for (size_t f = 0; f < n; ++f) {
    double x = kCongested ? r[f] * beta[f] : std::min(r[f] + alpha[f], caps[f]);
    if (meas) mean[f] += x;
    x = std::min(x, caps[f]);
    r[f] = x;
    acc[f & 7] += x;
  }
}

template <bool kCongested>
__attribute__((target("avx2"))) void netsim_pass_avx2(size_t n, double* r, const double* alpha,
                                                      const double* beta, const double* caps,
                                                      double* mean, bool meas, double acc[8]) {
  __m256d a0 = _mm256_loadu_pd(acc), a1 = _mm256_loadu_pd(acc + 4);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    for (int h = 0; h < 2; ++h) {
      const size_t f = i + 4 * h;
      const __m256d c = _mm256_loadu_pd(caps + f);
      __m256d x = _mm256_loadu_pd(r + f);
      // std::min(a, b) == (b < a) ? b : a == _mm256_min_pd(b, a)'s pick for non-NaN
      x = kCongested ? _mm256_mul_pd(x, _mm256_loadu_pd(beta + f))
                     : _mm256_min_pd(c, _mm256_add_pd(x, _mm256_loadu_pd(alpha + f)));
      if (meas) _mm256_storeu_pd(mean + f, _mm256_add_pd(_mm256_loadu_pd(mean + f), x));
      x = _mm256_min_pd(c, x);
      _mm256_storeu_pd(r + f, x);
      if (h == 0)
        a0 = _mm256_add_pd(a0, x);
      else
        a1 = _mm256_add_pd(a1, x);
    }
  }
  _mm256_storeu_pd(acc, a0);
  _mm256_storeu_pd(acc + 4, a1);
  if (i < n) netsim_pass<kCongested>(n - i, r + i, alpha + i, beta + i, caps + i, mean + i, meas, acc);
}

int mean_rates(size_t n, const double* alpha, const double* beta, const double* caps,
               double capacity, int steps, double* mean) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  std::vector<double> rates(n, 0.0);  // the current step's rates, clamped to the caps
  for (size_t i = 0; i < n; ++i) mean[i] = 0.0;
  const int from = steps / 2;
  const double margin_per = 2.5 * (double)n * 0x1p-53;
  int exact = 0;
  double par = 0.0;  // their sum, eight interleaved accumulators (step 0: all zero)
  for (int s = 0; s < steps; ++s) {
    const double margin = margin_per * par;
    bool congested;
    if (par - capacity > margin) {
      congested = true;
    } else if (capacity - par > margin) {
      congested = false;
    } else {  // too close to call: the reference's sequential sum
      double total = 0.0;
      for (size_t k = 0; k < n; ++k) total += rates[k];
      congested = total >= capacity;
      ++exact;
    }
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool meas = s >= from;
    double* r = rates.data();
    if (avx2) {
      if (congested)
        netsim_pass_avx2<true>(n, r, alpha, beta, caps, mean, meas, acc);
      else
        netsim_pass_avx2<false>(n, r, alpha, beta, caps, mean, meas, acc);
    } else {
      if (congested)
        netsim_pass<true>(n, r, alpha, beta, caps, mean, meas, acc);
      else
        netsim_pass<false>(n, r, alpha, beta, caps, mean, meas, acc);
    }
    par = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
  const int measured = std::max(1, steps - from);
  for (size_t k = 0; k < n; ++k) mean[k] = mean[k] / measured;
  return exact;
}

}  // namespace ecco_netsim

// ----------------------------------------------------------- allocator --
namespace ecco_alloc {

// cal_objective_gain, gpu_allocator.cpp:49-76 (jobs ascending by id).  The
// size weights are fixed within a window: coef[k] = alpha * w_k / ws with
// w_k = members_k^beta and ws summed in job order -- the reference's
// `alpha * w / ws * gain` evaluates left to right, so coef[k] * gain[k] is the
// same double.  They are computed once per window (the reference recomputes
// them, pow() included, on every greedy pick: O(J) pow per micro-window).
void size_coef(const std::vector<int>& members, double alpha, double beta,
               std::vector<double>& coef) {
  coef.resize(members.size());
  double ws = 0.0;
  for (int n : members) ws += std::pow((double)n, beta);
  for (size_t k = 0; k < members.size(); ++k)
    coef[k] = alpha * std::pow((double)members[k], beta) / ws;
}

// current_scores (gpu_allocator.cpp:137-144): total_acc_greedy scores
// member_count * gain, otherwise the objective gain with the fairness bonus
// on the least-accurate job (strict <, lowest id on ties).
void scores(bool total_acc, bool bonus, const std::vector<double>& coef,
            const std::vector<int>& ids, const std::vector<int>& members,
            const std::vector<double>& acc, const std::vector<double>& gain,
            std::vector<double>& out) {
  out.resize(ids.size());
  if (total_acc) {
    for (size_t k = 0; k < ids.size(); ++k) out[k] = members[k] * gain[k];
    return;
  }
  int min_k = 0;
  double min_acc = acc[0];
  for (size_t k = 0; k < ids.size(); ++k) {
    out[k] = coef[k] * gain[k];
    const double a = acc[k];
    if (a < min_acc || (a == min_acc && ids[k] < ids[min_k])) {
      min_acc = a;
      min_k = (int)k;
    }
  }
  if (bonus) out[min_k] += gain[min_k];
}

// pick_next (gpu_allocator.cpp:146-158): highest score, strict >, so the
// lowest id wins ties.
int argmax(const std::vector<double>& sc) {
  int k = 0;
  double b = sc[0];
  for (size_t q = 1; q < sc.size(); ++q)
    if (sc[q] > b) {
      b = sc[q];
      k = (int)q;
    }
  return k;
}

// Tournament tree over per-job keys for the greedy's repeated picks: after a
// micro-window only the granted job's acc / gain change, so each pick is
// O(log J) instead of the O(J) rescan.  `better(a, b)` is the scan's strict
// comparison (b replaces the running winner a only if strictly better), so
// the winner is the lowest index among the best keys -- the same job the
// linear scans above return whenever no key is NaN (callers check).
template <class Better>
struct Tourney {
  int n = 0, P = 1;
  std::vector<int> t;  // t[P + k] = k; internal nodes hold the subtree winner (-1: empty)
  Better better;
  explicit Tourney(int n_, Better b) : n(n_), better(b) {
    while (P < n) P <<= 1;
    t.assign(2 * P, -1);
    for (int k = 0; k < n; ++k) t[P + k] = k;
    for (int i = P - 1; i >= 1; --i) t[i] = pick(t[2 * i], t[2 * i + 1]);
  }
  int pick(int a, int b) const {
    if (a < 0) return b;
    if (b < 0) return a;
    return better(b, a) ? b : a;  // a has the lower index
  }
  void update(int k) {
    for (int i = (P + k) >> 1; i >= 1; i >>= 1) t[i] = pick(t[2 * i], t[2 * i + 1]);
  }
  int best() const { return t[1]; }
  int best_except(int x) const {  // winner over every index but x
    int w = -1;
    for (int i = P + x; i > 1; i >>= 1) {  // siblings along x's path, in index order
      const int sib = i ^ 1;
      w = (sib < i) ? pick(t[sib], w) : pick(w, t[sib]);
    }
    return w;
  }
};

}  // namespace ecco_alloc

// ------------------------------------------------------------ scenario --
// Restatement of the strict schema of proj/core/src/scenario.cpp:80-357.

enum Policy { kEcco = 0, kNaive = 1, kTotalAcc = 2 };

struct CamSpec {
  std::string id;
  double x = 0, y = 0;
  std::vector<double> scene;
  double acc = 0.0, cap = 0.0, tp = 8.192e6;
  int bias = 0;  // 0 resolution, 1 frame_rate
};

struct Event {
  std::string cam;
  int ci = -1;
  double t = 0.0;
  std::vector<double> scene;
  double drop = 0.0;
};

struct Scenario {
  std::string name;
  unsigned seed = 0;
  int num_windows = 1;
  int policy = kEcco;
  bool equal_bw = false;
  double drift_threshold = 0.25;
  std::optional<double> response_target;
  ecco_model_params model{0.05, 0.5, 0.1, 0.6, 0.9};
  double alpha = 1.0, beta = 0.5;
  int W = 10;
  double mu = 6.0;
  int gpus = 1;
  bool bonus = true;
  double eps = 120.0, delta = 500.0, drop_p = 0.2;
  std::vector<double> ladder{360, 480, 720, 960};
  std::vector<double> fps{1, 2, 5, 10, 15};
  double bpp_ref = 0.1, alpha_unit = 5e5, probe_rate = 1e6;
  double fixed_f = 5.0, fixed_q = 960.0;
  double capacity = 6e6, rtt = 0.05;
  std::vector<CamSpec> cams;
  std::vector<Event> events;
  double T() const { return W * mu; }
};

double num(const json& j, const std::string& p) {
  if (!j.is_number()) schema(p, "expected a number");
  return j.get<double>();
}
double opt_num(const json& o, const char* k, const std::string& p, double fb) {
  return o.contains(k) ? num(o.at(k), p + "." + k) : fb;
}
int opt_int(const json& o, const char* k, const std::string& p, int fb) {
  if (!o.contains(k)) return fb;
  if (!o.at(k).is_number_integer()) schema(p + "." + k, "expected an integer");
  return o.at(k).get<int>();
}
bool opt_bool(const json& o, const char* k, const std::string& p, bool fb) {
  if (!o.contains(k)) return fb;
  if (!o.at(k).is_boolean()) schema(p + "." + k, "expected a boolean");
  return o.at(k).get<bool>();
}
std::string str(const json& j, const std::string& p) {
  if (!j.is_string()) schema(p, "expected a string");
  return j.get<std::string>();
}
std::vector<double> nums(const json& j, const std::string& p) {
  if (!j.is_array()) schema(p, "expected an array of numbers");
  std::vector<double> v;
  for (size_t i = 0; i < j.size(); ++i) v.push_back(num(j[i], p + "[" + std::to_string(i) + "]"));
  return v;
}
void only(const json& o, const std::string& p, std::initializer_list<const char*> keys) {
  if (!o.is_object()) schema(p, "expected an object");
  for (const auto& [k, v] : o.items()) {
    bool ok = false;
    for (const char* q : keys) ok = ok || k == q;
    if (!ok) schema(p + "." + k, "unknown field");
  }
}

Scenario parse_scenario(const std::string& text) {
  json root;
  try {
    root = json::parse(text);
  } catch (const json::parse_error& e) {
    schema("scenario", std::string("invalid JSON: ") + e.what());
  }
  only(root, "scenario",
       {"name", "seed", "num_windows", "policy", "equal_bandwidth", "drift_threshold",
        "response_target_acc", "model", "allocator", "grouping", "transmission",
        "shared_capacity_bps", "rtt_s", "window_length_s", "cameras", "drift_events"});
  Scenario s;
  if (root.contains("name")) s.name = str(root.at("name"), "name");
  if (root.contains("seed")) {
    if (!root.at("seed").is_number_unsigned()) schema("seed", "expected a non-negative integer");
    s.seed = root.at("seed").get<unsigned>();
  }
  s.num_windows = opt_int(root, "num_windows", "", s.num_windows);
  if (root.contains("policy")) {
    const std::string n = str(root.at("policy"), "policy");
    if (n == "ecco") s.policy = kEcco;
    else if (n == "naive") s.policy = kNaive;
    else if (n == "total_acc_greedy") s.policy = kTotalAcc;
    else schema("policy", "unknown policy " + n + " (expected ecco|naive|total_acc_greedy)");
  }
  s.equal_bw = opt_bool(root, "equal_bandwidth", "", s.equal_bw);
  s.drift_threshold = opt_num(root, "drift_threshold", "", s.drift_threshold);
  if (root.contains("response_target_acc"))
    s.response_target = num(root.at("response_target_acc"), "response_target_acc");
  if (root.contains("model")) {
    const json& m = root.at("model");
    only(m, "model", {"learning_rate_k", "similarity_lambda", "acc_floor", "acc_ceil",
                      "cluster_similarity_threshold"});
    s.model.learning_rate_k = opt_num(m, "learning_rate_k", "model", s.model.learning_rate_k);
    s.model.similarity_lambda = opt_num(m, "similarity_lambda", "model", s.model.similarity_lambda);
    s.model.acc_floor = opt_num(m, "acc_floor", "model", s.model.acc_floor);
    s.model.acc_ceil = opt_num(m, "acc_ceil", "model", s.model.acc_ceil);
    s.model.cluster_similarity_threshold =
        opt_num(m, "cluster_similarity_threshold", "model", s.model.cluster_similarity_threshold);
  }
  if (root.contains("allocator")) {
    const json& a = root.at("allocator");
    only(a, "allocator", {"obj_alpha", "size_exponent_beta", "micro_windows",
                          "micro_window_duration_s", "gpu_count", "fairness_bonus"});
    s.alpha = opt_num(a, "obj_alpha", "allocator", s.alpha);
    s.beta = opt_num(a, "size_exponent_beta", "allocator", s.beta);
    s.W = opt_int(a, "micro_windows", "allocator", s.W);
    s.mu = opt_num(a, "micro_window_duration_s", "allocator", s.mu);
    s.gpus = opt_int(a, "gpu_count", "allocator", s.gpus);
    s.bonus = opt_bool(a, "fairness_bonus", "allocator", s.bonus);
  }
  if (root.contains("grouping")) {
    const json& g = root.at("grouping");
    only(g, "grouping", {"epsilon_s", "delta_m", "drop_threshold_p"});
    s.eps = opt_num(g, "epsilon_s", "grouping", s.eps);
    s.delta = opt_num(g, "delta_m", "grouping", s.delta);
    s.drop_p = opt_num(g, "drop_threshold_p", "grouping", s.drop_p);
  }
  if (root.contains("transmission")) {
    const json& t = root.at("transmission");
    only(t, "transmission", {"resolution_ladder", "frame_rates", "bpp_ref", "alpha_unit_bps",
                             "probe_reference_rate_bps", "fixed_config"});
    if (t.contains("resolution_ladder"))
      s.ladder = nums(t.at("resolution_ladder"), "transmission.resolution_ladder");
    if (t.contains("frame_rates")) s.fps = nums(t.at("frame_rates"), "transmission.frame_rates");
    s.bpp_ref = opt_num(t, "bpp_ref", "transmission", s.bpp_ref);
    s.alpha_unit = opt_num(t, "alpha_unit_bps", "transmission", s.alpha_unit);
    s.probe_rate = opt_num(t, "probe_reference_rate_bps", "transmission", s.probe_rate);
    if (t.contains("fixed_config")) {
      const json& fc = t.at("fixed_config");
      only(fc, "transmission.fixed_config", {"frame_rate", "resolution"});
      s.fixed_f = opt_num(fc, "frame_rate", "transmission.fixed_config", s.fixed_f);
      s.fixed_q = opt_num(fc, "resolution", "transmission.fixed_config", s.fixed_q);
    }
  }
  s.capacity = opt_num(root, "shared_capacity_bps", "", s.capacity);
  s.rtt = opt_num(root, "rtt_s", "", s.rtt);
  if (!root.contains("cameras")) schema("cameras", "required");
  const json& cams = root.at("cameras");
  if (!cams.is_array()) schema("cameras", "expected an array");
  for (size_t i = 0; i < cams.size(); ++i) {
    const std::string p = "cameras[" + std::to_string(i) + "]";
    const json& c = cams[i];
    only(c, p, {"id", "location", "scene", "local_model_acc", "local_uplink_cap_bps",
                "gpu_pixel_throughput", "profile_bias"});
    CamSpec cs;
    if (!c.contains("id")) schema(p + ".id", "required");
    cs.id = str(c.at("id"), p + ".id");
    if (cs.id.empty()) schema(p + ".id", "must not be empty");
    if (!c.contains("location")) schema(p + ".location", "required");
    const auto loc = nums(c.at("location"), p + ".location");
    if (loc.size() != 2) schema(p + ".location", "expected [x, y]");
    cs.x = loc[0];
    cs.y = loc[1];
    if (!c.contains("scene")) schema(p + ".scene", "required");
    cs.scene = nums(c.at("scene"), p + ".scene");
    if (cs.scene.empty()) schema(p + ".scene", "must not be empty");
    cs.acc = opt_num(c, "local_model_acc", p, cs.acc);
    cs.cap = opt_num(c, "local_uplink_cap_bps", p, cs.cap);
    cs.tp = opt_num(c, "gpu_pixel_throughput", p, cs.tp);
    if (c.contains("profile_bias")) {
      const std::string b = str(c.at("profile_bias"), p + ".profile_bias");
      if (b == "resolution") cs.bias = 0;
      else if (b == "frame_rate") cs.bias = 1;
      else schema(p + ".profile_bias", "unknown profile bias " + b);
    }
    s.cams.push_back(cs);
  }
  if (root.contains("drift_events")) {
    const json& evs = root.at("drift_events");
    if (!evs.is_array()) schema("drift_events", "expected an array");
    for (size_t i = 0; i < evs.size(); ++i) {
      const std::string p = "drift_events[" + std::to_string(i) + "]";
      const json& e = evs[i];
      only(e, p, {"camera", "time_s", "new_scene", "acc_drop"});
      Event ev;
      if (!e.contains("camera")) schema(p + ".camera", "required");
      ev.cam = str(e.at("camera"), p + ".camera");
      if (!e.contains("time_s")) schema(p + ".time_s", "required");
      ev.t = num(e.at("time_s"), p + ".time_s");
      if (!e.contains("new_scene")) schema(p + ".new_scene", "required");
      ev.scene = nums(e.at("new_scene"), p + ".new_scene");
      if (!e.contains("acc_drop")) schema(p + ".acc_drop", "required");
      ev.drop = num(e.at("acc_drop"), p + ".acc_drop");
      s.events.push_back(ev);
    }
  }
  if (root.contains("window_length_s")) {
    const double given = num(root.at("window_length_s"), "window_length_s");
    const double derived = s.T();
    if (std::abs(given - derived) > 1e-9 * std::max(1.0, derived))
      schema("window_length_s",
             "conflicts with micro_windows * micro_window_duration_s = " + std::to_string(derived));
  }
  // ScenarioConfig::validate (scenario.cpp:204-272)
  if (s.num_windows < 1) schema("num_windows", "must be >= 1");
  if (s.drift_threshold < 0.0 || s.drift_threshold > 1.0)
    schema("drift_threshold", "must be in [0, 1]");
  if (s.response_target && (*s.response_target <= 0.0 || *s.response_target > 1.0))
    schema("response_target_acc", "must be in (0, 1]");
  if (s.alpha < 0.0) schema("allocator", "allocator: obj_alpha must be >= 0");
  if (s.beta > 1.0) schema("allocator", "allocator: size_exponent_beta must be <= 1");
  if (s.W < 1) schema("allocator", "allocator: micro_windows must be positive");
  if (!(s.mu > 0.0)) schema("allocator", "allocator: micro_window_duration_s must be positive");
  if (s.gpus < 1) schema("allocator", "allocator: gpu_count must be positive");
  const auto& m = s.model;
  if (m.learning_rate_k <= 0.0) schema("model.learning_rate_k", "must be > 0");
  if (m.similarity_lambda <= 0.0) schema("model.similarity_lambda", "must be > 0");
  if (m.acc_floor < 0.0 || m.acc_floor >= m.acc_ceil || m.acc_ceil > 1.0)
    schema("model", "needs 0 <= acc_floor < acc_ceil <= 1");
  if (m.cluster_similarity_threshold <= 0.0 || m.cluster_similarity_threshold > 1.0)
    schema("model.cluster_similarity_threshold", "must be in (0, 1]");
  if (s.eps < 0.0) schema("grouping.epsilon_s", "must be >= 0");
  if (s.delta < 0.0) schema("grouping.delta_m", "must be >= 0");
  if (s.drop_p <= 0.0) schema("grouping.drop_threshold_p", "must be > 0");
  if (s.ladder.empty()) schema("transmission.resolution_ladder", "must not be empty");
  if (s.fps.empty()) schema("transmission.frame_rates", "must not be empty");
  for (double q : s.ladder)
    if (q <= 0.0) schema("transmission.resolution_ladder", "entries must be > 0");
  for (double f : s.fps)
    if (f <= 0.0) schema("transmission.frame_rates", "entries must be > 0");
  if (s.bpp_ref <= 0.0) schema("transmission.bpp_ref", "must be > 0");
  if (s.alpha_unit <= 0.0) schema("transmission.alpha_unit_bps", "must be > 0");
  if (s.probe_rate <= 0.0) schema("transmission.probe_reference_rate_bps", "must be > 0");
  if (s.fixed_f <= 0.0 || s.fixed_q <= 0.0) schema("transmission.fixed_config", "must be positive");
  if (s.capacity <= 0.0) schema("shared_capacity_bps", "must be > 0");
  if (s.rtt <= 0.0) schema("rtt_s", "must be > 0");
  if (s.cams.empty()) schema("cameras", "must not be empty");
  std::set<std::string> seen;
  const size_t dims = s.cams.front().scene.size();
  for (size_t i = 0; i < s.cams.size(); ++i) {
    const auto& c = s.cams[i];
    const std::string p = "cameras[" + std::to_string(i) + "]";
    if (!seen.insert(c.id).second) schema(p + ".id", "duplicate camera id");
    if (c.scene.size() != dims) schema(p + ".scene", "scene vectors must share one dimension");
    if (c.acc < 0.0 || c.acc > 1.0) schema(p + ".local_model_acc", "must be in [0, 1]");
    if (c.cap < 0.0) schema(p + ".local_uplink_cap_bps", "must be >= 0");
    if (c.tp <= 0.0) schema(p + ".gpu_pixel_throughput", "must be > 0");
  }
  for (size_t i = 0; i < s.events.size(); ++i) {
    const auto& e = s.events[i];
    const std::string p = "drift_events[" + std::to_string(i) + "]";
    if (!seen.count(e.cam)) schema(p + ".camera", "references unknown camera " + e.cam);
    if (e.t < 0.0) schema(p + ".time_s", "must be >= 0");
    if (e.scene.size() != dims) schema(p + ".new_scene", "scene vectors must share one dimension");
    if (e.drop < 0.0) schema(p + ".acc_drop", "must be >= 0");
  }
  return s;
}

const char* policy_name(int p) {
  return p == kEcco ? "ecco" : p == kNaive ? "naive" : "total_acc_greedy";
}

// --------------------------------------------------------------- trace --

enum Kind { kAccuracy, kRequest, kJoin, kNewJob, kRemove, kTerminate, kMicro, kJobWindow };
const char* kind_name(int k) {
  static const char* n[] = {"accuracy", "request", "join", "new_job",
                            "remove",   "terminate", "micro", "job_window"};
  return n[k];
}

struct Row {
  int kind = kAccuracy;
  int window = 0;
  double t = 0.0;
  int cam = -1;
  int job = -1;
  double v[5] = {0, 0, 0, 0, 0};
};

// format_value, metrics.cpp:42-47.
// format_value (metrics.cpp:42-47): "%.9g", with -0 written as 0.
// std::to_chars(general, 9) is specified as printf's %.9g in the C locale
// (same digits, exponent form and rounding) at a fraction of the cost.
void fmt_to(std::string& out, double v) {
  if (v == 0.0) {
    out += '0';
    return;
  }
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::general, 9);
  out.append(buf, r.ptr);
}
std::string fmt(double v) {
  std::string s;
  fmt_to(s, v);
  return s;
}

// ---------------------------------------------------------------- state --

struct Request {
  int cam = -1;
  double t = 0.0;
  double x = 0.0, y = 0.0;
  std::vector<double> scene;
  double acc = 0.0;
  std::vector<double> hist;
};

struct Job {
  int id = 0;
  std::vector<Request> members;  // ascending camera index == std::string order
  std::map<int, double> acc_per_member;
  std::vector<double> mean_hist;
  int find(int cam) const {
    for (size_t i = 0; i < members.size(); ++i)
      if (members[i].cam == cam) return (int)i;
    return -1;
  }
  void insert(Request r) {
    auto pos = std::lower_bound(members.begin(), members.end(), r,
                                [](const Request& a, const Request& b) { return a.cam < b.cam; });
    members.insert(pos, std::move(r));
  }
};

struct Batch {
  double fps = 0, res = 0, quality = 1.0;
  std::vector<int> src;  // ascending camera index (std::map order)
  std::vector<double> frac;
};

struct ProfRow {
  double budget, f, q;
  bool feasible;
};

struct Cam {
  std::string id;
  double x, y;
  std::vector<double> scene;
  double acc, cap, tp;
  int bias;
};

constexpr int kBaseModelId = INT_MIN + 7;  // learned backend's base model

}  // namespace

struct ecco_sim {
  Scenario cfg;
  ecco_sim_options opt{};
  ecco_ctx* ctx = nullptr;
  std::string err;
  std::vector<Cam> cams;
  std::map<std::string, int> cam_index;
  std::map<int, Job> jobs;
  std::vector<int> membership;  // camera -> job or -1
  std::map<int, Batch> batches;
  std::vector<std::optional<std::vector<ProfRow>>> profiles;
  std::vector<uint8_t> prof_sorted;  // budgets non-decreasing: select_config by bisection
  std::vector<double> sel_f, sel_q, rate_of;  // per-camera scratch of a window
  std::vector<double> coef;                    // objective size weights of a window
  std::vector<Event> events;
  size_t next_event = 0;
  std::vector<Request> pending;
  int next_job_id = 0;
  int window = 0;
  std::vector<Row> rows;
  double timings[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int64_t samples = 0;
  int D = 2;

  bool learned() const { return opt.backend == ECCO_BACKEND_LEARNED; }

  // ---------------------------------------------------------- grouping --
  // correlation_filter, grouping.cpp:9-16.
  bool correlated(const Job& j, const Request& r) const {
    for (const auto& m : j.members) {
      if (std::abs(m.t - r.t) > cfg.eps) return false;
      if (std::hypot(m.x - r.x, m.y - r.y) > cfg.delta) return false;
    }
    return true;
  }
  static bool correlated_pair(const Request& a, const Request& b, double eps, double delta) {
    return std::abs(a.t - b.t) <= eps && std::hypot(a.x - b.x, a.y - b.y) <= delta;
  }

  struct Assignment {
    int job = -1;
    bool created = false;
    double acc = 0.0;
  };

  // group_request over a whole ordered batch of requests (grouping.cpp:18-62),
  // with exclude[i] the job request i must not rejoin (-1 none).
  std::vector<Assignment> route_batch(std::vector<Request>& reqs, const std::vector<int>& exclude) {
    const int n = (int)reqs.size();
    std::vector<Assignment> out(n);
    if (n == 0) return out;
    // (a) candidate pairs against jobs existing at batch start (superset: a
    //     job's member set only grows during the pass).
    struct Box {
      double x0, y0, x1, y1, t0, t1;
    };
    std::vector<int> ids;
    std::vector<Box> boxes;
    for (const auto& [id, j] : jobs) {
      Box b{1e300, 1e300, -1e300, -1e300, 1e300, -1e300};
      for (const auto& m : j.members) {
        b.x0 = std::min(b.x0, m.x);
        b.y0 = std::min(b.y0, m.y);
        b.x1 = std::max(b.x1, m.x);
        b.y1 = std::max(b.y1, m.y);
        b.t0 = std::min(b.t0, m.t);
        b.t1 = std::max(b.t1, m.t);
      }
      ids.push_back(id);
      boxes.push_back(b);
    }
    // Candidate search over a uniform grid of job boxes (cell = delta): a
    // job is a candidate for request r only if r lies within delta of its
    // member box on both axes and within eps of its members' times (else
    // some member fails correlation_filter).  Pairs come out per request in
    // ascending job id (the JobMap order group_request walks), pair_off[r]
    // delimiting request r's run.
    std::vector<int> pair_job;
    std::vector<int> pair_req;
    std::vector<int> pair_off(n + 1, 0);
    {
      const double cell = std::max(cfg.delta, 1e-9);
      auto cidx = [&](double v) { return (long long)std::floor(v / cell); };
      auto ckey = [](long long gx, long long gy) {
        return (unsigned long long)(gx * 1000003LL + gy);
      };
      std::unordered_map<unsigned long long, std::vector<int>> grid;  // cell -> job positions
      std::vector<int> wide;  // boxes spanning too many cells: checked against every request
      for (size_t k = 0; k < ids.size(); ++k) {
        const Box& b = boxes[k];
        const long long x0 = cidx(b.x0 - cfg.delta), x1 = cidx(b.x1 + cfg.delta);
        const long long y0 = cidx(b.y0 - cfg.delta), y1 = cidx(b.y1 + cfg.delta);
        if ((x1 - x0 + 1) * (y1 - y0 + 1) > 64) {
          wide.push_back((int)k);
          continue;
        }
        for (long long gx = x0; gx <= x1; ++gx)
          for (long long gy = y0; gy <= y1; ++gy) grid[ckey(gx, gy)].push_back((int)k);
      }
      std::vector<int> cand;
      for (int r = 0; r < n; ++r) {
        const Request& q = reqs[r];
        cand.assign(wide.begin(), wide.end());
        auto it = grid.find(ckey(cidx(q.x), cidx(q.y)));
        if (it != grid.end()) cand.insert(cand.end(), it->second.begin(), it->second.end());
        std::sort(cand.begin(), cand.end());  // positions in ids: ascending job id
        for (int k : cand) {
          if (ids[k] == exclude[r]) continue;
          const Box& b = boxes[k];
          const double dx = q.x < b.x0 ? b.x0 - q.x : (q.x > b.x1 ? q.x - b.x1 : 0.0);
          const double dy = q.y < b.y0 ? b.y0 - q.y : (q.y > b.y1 ? q.y - b.y1 : 0.0);
          if (dx > cfg.delta || dy > cfg.delta) continue;
          if (q.t - b.t0 > cfg.eps || b.t1 - q.t > cfg.eps) continue;
          if (!correlated(jobs.at(ids[k]), q)) continue;
          pair_job.push_back(ids[k]);
          pair_req.push_back(r);
        }
        pair_off[r + 1] = (int)pair_job.size();
      }
    }
    // (b) provisional columns: a job founded by request a can only be a
    //     candidate for a later request b correlated with a.
    std::vector<int> has_later(n, 0);
    std::vector<std::pair<int, int>> prov;  // (founder a, later b)
    {
      const double cell = std::max(cfg.delta, 1e-9);
      std::unordered_map<long long, std::vector<int>> grid;
      auto key = [&](double x, double y) {
        const long long gx = (long long)std::floor(x / cell), gy = (long long)std::floor(y / cell);
        return gx * 1000003LL + gy;
      };
      for (int r = 0; r < n; ++r) grid[key(reqs[r].x, reqs[r].y)].push_back(r);
      for (int a = 0; a < n; ++a) {
        const long long gx = (long long)std::floor(reqs[a].x / cell),
                        gy = (long long)std::floor(reqs[a].y / cell);
        for (long long dx = -1; dx <= 1; ++dx)
          for (long long dy = -1; dy <= 1; ++dy) {
            auto it = grid.find((gx + dx) * 1000003LL + (gy + dy));
            if (it == grid.end()) continue;
            for (int b : it->second)
              if (b > a && correlated_pair(reqs[a], reqs[b], cfg.eps, cfg.delta)) {
                prov.push_back({a, b});
                has_later[a] = 1;
              }
          }
      }
    }
    // device: one pair evaluation over (a) and (b)
    std::vector<int> pj;
    std::vector<int> pc;
    std::vector<double> ps;
    auto add_pair = [&](int job, int r) {
      pj.push_back(job);
      pc.push_back(reqs[r].cam);
      ps.insert(ps.end(), reqs[r].scene.begin(), reqs[r].scene.end());
    };
    for (size_t i = 0; i < pair_job.size(); ++i) add_pair(pair_job[i], pair_req[i]);
    std::vector<int> prov_id(n, 0);
    if (!learned()) {
      std::vector<int> sid;
      std::vector<double> ssc, sacc;
      for (int a = 0; a < n; ++a)
        if (has_later[a]) {
          prov_id[a] = -1000000 - a;
          sid.push_back(prov_id[a]);
          ssc.insert(ssc.end(), reqs[a].scene.begin(), reqs[a].scene.end());
          sacc.push_back(reqs[a].acc);
        }
      if (!sid.empty())
        check(ctx, ecco_seed_models(ctx, (int)sid.size(), sid.data(), ssc.data(), sacc.data()));
      for (const auto& [a, b] : prov) add_pair(prov_id[a], b);
    } else {
      // every new learned job starts as the base model: one column per request
      for (const auto& [a, b] : prov) (void)a, (void)b;
      for (int r = 0; r < n; ++r) add_pair(kBaseModelId, r);
    }
    std::vector<double> vals(pj.size());
    if (!pj.empty())
      check(ctx, ecco_eval_pairs(ctx, (int)pj.size(), learned() ? nullptr : ps.data(), pc.data(),
                                 pj.data(), vals.data()));
    size_t off = pair_job.size();
    std::vector<double> base_val(n, 0.0);
    std::vector<double> prov_val(prov.size(), 0.0);
    if (!learned()) {
      for (size_t i = 0; i < prov.size(); ++i) prov_val[i] = vals[off + i];
    } else {
      for (int r = 0; r < n; ++r) base_val[r] = vals[off + r];
    }
    // founders a < b whose job may be a candidate for b, per b (ascending a:
    // jobs created in this pass get ascending ids in request order)
    std::vector<std::vector<int>> prov_of(n);  // indices into prov
    for (size_t i = 0; i < prov.size(); ++i) prov_of[prov[i].second].push_back((int)i);
    for (auto& v : prov_of)
      std::sort(v.begin(), v.end(), [&](int x, int y) { return prov[x].first < prov[y].first; });
    // camera -> job at batch start, kept current through the commit
    std::vector<int> mem_of(cams.size(), -1);
    for (const auto& [id, j] : jobs)
      for (const auto& m : j.members) mem_of[m.cam] = id;
    // host commit in request order (group_request, grouping.cpp:18-62): the
    // candidates are the pairs found above (existing jobs, ascending id; a
    // job's member set only grows, so correlation_filter is re-checked on the
    // current members) followed by the jobs this pass created for correlated
    // earlier requests (larger ids, ascending) -- the same jobs, in the same
    // order, that a walk over every job would accept
    std::vector<int> created_by(n, -1);  // request -> job it created
    std::map<int, int> founder;  // new job id -> founding request
    std::vector<int> created_ids, created_prov;
    for (int r = 0; r < n; ++r) {
      Request& q = reqs[r];
      if (mem_of[q.cam] >= 0)
        fail(ECCO_ERR_INVALID_ARGUMENT, "group_request: camera " + cams[q.cam].id +
                                            " is already a member of job " +
                                            std::to_string(mem_of[q.cam]));
      int best = -1;
      double best_acc = 0.0;
      auto consider = [&](int id, double acc) {
        if (acc < q.acc) return;
        if (best < 0 || acc > best_acc) {
          best = id;
          best_acc = acc;
        }
      };
      for (int i = pair_off[r]; i < pair_off[r + 1]; ++i) {
        const int id = pair_job[i];
        if (!correlated(jobs.at(id), q)) continue;
        consider(id, vals[i]);
      }
      for (int pi : prov_of[r]) {
        const int id = created_by[prov[pi].first];
        if (id < 0 || (exclude[r] >= 0 && id == exclude[r])) continue;
        if (!correlated(jobs.at(id), q)) continue;
        consider(id, learned() ? base_val[r] : prov_val[pi]);
      }
      if (best >= 0) {
        Job& j = jobs.at(best);
        q.hist.clear();
        const int cam = q.cam;
        j.insert(q);
        j.acc_per_member[cam] = best_acc;
        mem_of[cam] = best;
        out[r] = {best, false, best_acc};
      } else {
        Job j;
        j.id = next_job_id++;
        const double seed_acc = q.acc;
        const int cam = q.cam;
        q.hist.clear();
        j.insert(q);
        j.acc_per_member[cam] = seed_acc;
        founder[j.id] = r;
        created_by[r] = j.id;
        created_ids.push_back(j.id);
        mem_of[cam] = j.id;
        out[r] = {j.id, true, seed_acc};
        jobs.emplace(j.id, std::move(j));
      }
    }
    // device bookkeeping of created jobs
    if (!learned()) {
      std::vector<int> olds, news, unused, fresh_ids;
      std::vector<double> fresh_sc, fresh_acc;
      std::set<int> used_prov;
      for (int id : created_ids) {
        const int a = founder[id];
        if (has_later[a]) {
          olds.push_back(prov_id[a]);
          news.push_back(id);
          used_prov.insert(a);
        } else {
          fresh_ids.push_back(id);
          fresh_sc.insert(fresh_sc.end(), reqs[a].scene.begin(), reqs[a].scene.end());
          fresh_acc.push_back(reqs[a].acc);
        }
      }
      for (int a = 0; a < n; ++a)
        if (has_later[a] && !used_prov.count(a)) unused.push_back(prov_id[a]);
      if (!olds.empty()) check(ctx, ecco_rename_models(ctx, (int)olds.size(), olds.data(), news.data()));
      if (!unused.empty()) check(ctx, ecco_drop_models(ctx, (int)unused.size(), unused.data()));
      if (!fresh_ids.empty())
        check(ctx, ecco_seed_models(ctx, (int)fresh_ids.size(), fresh_ids.data(), fresh_sc.data(),
                                    fresh_acc.data()));
    } else if (!created_ids.empty()) {
      check(ctx, ecco_seed_models(ctx, (int)created_ids.size(), created_ids.data(), nullptr, nullptr));
    }
    return out;
  }

  void refresh_membership() {
    std::fill(membership.begin(), membership.end(), -1);
    for (const auto& [id, j] : jobs)
      for (const auto& m : j.members) membership[m.cam] = id;
  }

  void emit_request(const Request& r) {
    Row row;
    row.kind = kRequest;
    row.window = window;
    row.t = r.t;
    row.cam = r.cam;
    row.v[0] = r.acc;
    rows.push_back(row);
    pending.push_back(r);
  }

  Request detect(int ci, double now) const {
    Request r;
    r.cam = ci;
    r.t = now;
    r.x = cams[ci].x;
    r.y = cams[ci].y;
    r.scene = cams[ci].scene;
    r.acc = cams[ci].acc;
    return r;
  }

  bool is_pending(int ci) const {
    for (const auto& r : pending)
      if (r.cam == ci) return true;
    return false;
  }

  // apply_due_events, orchestrator.cpp:118-145.
  void apply_due_events(double t0) {
    std::vector<int> changed;
    while (next_event < events.size() && events[next_event].t <= t0) {
      const Event& ev = events[next_event++];
      Cam& c = cams[ev.ci];
      c.scene = ev.scene;
      c.acc = std::max(cfg.model.acc_floor, c.acc - ev.drop);
      changed.push_back(ev.ci);
      if (membership[ev.ci] >= 0) continue;
      if (is_pending(ev.ci)) continue;
      if (c.acc < cfg.drift_threshold) emit_request(detect(ev.ci, ev.t));
    }
    if (!changed.empty()) {
      std::vector<double> sc;
      for (int ci : changed) sc.insert(sc.end(), cams[ci].scene.begin(), cams[ci].scene.end());
      check(ctx, ecco_update_scenes(ctx, (int)changed.size(), changed.data(), sc.data()));
    }
    for (int ci = 0; ci < (int)cams.size(); ++ci) {
      if (membership[ci] >= 0) continue;
      if (is_pending(ci)) continue;
      if (cams[ci].acc < cfg.drift_threshold) emit_request(detect(ci, t0));
    }
  }

  // route_pending_requests, orchestrator.cpp:158-184.
  void route_pending(double t0) {
    std::stable_sort(pending.begin(), pending.end(), [](const Request& a, const Request& b) {
      if (a.t != b.t) return a.t < b.t;
      return a.cam < b.cam;
    });
    std::vector<int> excl(pending.size(), -1);
    const auto as = route_batch(pending, excl);
    for (size_t i = 0; i < pending.size(); ++i) {
      Row row;
      row.kind = as[i].created ? kNewJob : kJoin;
      row.window = window;
      row.t = t0;
      row.cam = pending[i].cam;
      row.job = as[i].job;
      row.v[0] = as[i].acc;
      rows.push_back(row);
    }
    pending.clear();
    refresh_membership();
  }

  // --------------------------------------------------------- allocator --
  Batch bootstrap(const Job& j) const {
    Batch b;
    b.fps = *std::min_element(cfg.fps.begin(), cfg.fps.end());
    b.res = *std::min_element(cfg.ladder.begin(), cfg.ladder.end());
    b.quality = 1.0;
    for (const auto& m : j.members) {
      b.src.push_back(m.cam);
      b.frac.push_back(1.0 / j.members.size());
    }
    return b;
  }

  double gpu_seconds() const { return cfg.gpus * cfg.mu; }

  int learned_steps(const Batch& b) const {
    if (b.src.empty()) return 0;
    const double supplied = b.fps * (b.res * (16.0 * b.res / 9.0));
    double sum = 0.0;
    for (int c : b.src) sum += cams[c].tp;
    const double required = sum / (double)b.src.size();
    const double suff = required > 0.0 ? std::min(1.0, supplied / required) : 1.0;
    const double effort = gpu_seconds() * suff * b.quality;
    if (effort <= 0.0) return 0;
    return (int)std::floor(effort * opt.steps_per_gpu_s);
  }

  // Trajectories from the committed models of `ids` (batches given).
  std::vector<std::vector<double>> trajectories(const std::vector<int>& ids,
                                                const std::vector<Batch>& bs,
                                                const std::vector<int>& micro_base, int depth) {
    const int n = (int)ids.size();
    std::vector<ecco_batch> eb(n);
    std::vector<int> so{0}, sc, mo{0}, mc;
    std::vector<double> sf;
    for (int i = 0; i < n; ++i) {
      eb[i] = {bs[i].fps, bs[i].res, bs[i].quality};
      sc.insert(sc.end(), bs[i].src.begin(), bs[i].src.end());
      sf.insert(sf.end(), bs[i].frac.begin(), bs[i].frac.end());
      so.push_back((int)sc.size());
      for (const auto& m : jobs.at(ids[i]).members) mc.push_back(m.cam);
      mo.push_back((int)mc.size());
    }
    std::vector<double> out((size_t)n * (depth + 1));
    check(ctx, ecco_train_trajectories(ctx, n, ids.data(), eb.data(), so.data(), sc.data(),
                                       sf.data(), mo.data(), mc.data(), micro_base.data(), window,
                                       gpu_seconds(), depth, out.data()));
    std::vector<std::vector<double>> tr(n);
    for (int i = 0; i < n; ++i)
      tr[i].assign(out.begin() + (size_t)i * (depth + 1), out.begin() + (size_t)(i + 1) * (depth + 1));
    return tr;
  }

  struct Micro {
    int index, job;
    double before, after;
  };

  void prepare_scores(const std::vector<int>& members) {
    ecco_alloc::size_coef(members, cfg.alpha, cfg.beta, coef);
  }
  void scores(const std::vector<int>& ids, const std::vector<int>& members,
              const std::vector<double>& acc, const std::vector<double>& gain,
              std::vector<double>& s) const {
    ecco_alloc::scores(cfg.policy == kTotalAcc, cfg.bonus, coef, ids, members, acc, gain, s);
  }

  // ------------------------------------------------------------ netsim --
  // simulate_window (netsim.cpp:64-94) keeping only the second-half sums.
  std::vector<double> simulate(const std::vector<double>& alpha, const std::vector<double>& beta,
                               const std::vector<double>& caps) const {
    if (!(cfg.capacity > 0.0)) fail(ECCO_ERR_INVALID_ARGUMENT, "netsim: shared capacity must be positive");
    const size_t n = alpha.size();
    for (size_t i = 0; i < n; ++i) {
      if (!(alpha[i] > 0.0)) fail(ECCO_ERR_INVALID_ARGUMENT, "netsim: alpha must be positive");
      if (!(beta[i] > 0.0 && beta[i] < 1.0)) fail(ECCO_ERR_INVALID_ARGUMENT, "netsim: beta must be in (0,1)");
    }
    const int steps = (int)std::llround(cfg.T() / cfg.rtt);
    std::vector<double> sums(n, 0.0);
    if (n == 0) return sums;
    ecco_netsim::mean_rates(n, alpha.data(), beta.data(), caps.data(), cfg.capacity, steps,
                            sums.data());
    return sums;
  }

  // Profile tables for every camera in `need` (orchestrator.cpp:94-116).
  void build_profiles(const std::vector<int>& need) {
    if (need.empty()) return;
    std::vector<double> levels;
    for (int k = 1; k <= cfg.W; ++k) levels.push_back(k * cfg.gpus * cfg.mu);
    std::vector<double> gf, gq;
    for (double f : cfg.fps)
      for (double q : cfg.ladder) {
        gf.push_back(f);
        gq.push_back(q);
      }
    std::vector<int> bias;
    for (int c : need) bias.push_back(cams[c].bias);
    const size_t rn = need.size() * levels.size();
    std::vector<double> ob(rn), of(rn), oq(rn);
    std::vector<uint8_t> fe(rn);
    check(ctx, ecco_profile_tables(ctx, (int)need.size(), need.data(), bias.data(),
                                   (int)levels.size(), levels.data(), (int)gf.size(), gf.data(),
                                   gq.data(), cfg.T(), 1e-9, cfg.probe_rate, cfg.bpp_ref,
                                   ob.data(), of.data(), oq.data(), fe.data()));
    for (size_t i = 0; i < need.size(); ++i) {
      std::vector<ProfRow> t;
      for (size_t l = 0; l < levels.size(); ++l) {
        const size_t o = i * levels.size() + l;
        t.push_back({ob[o], of[o], oq[o], fe[o] != 0});
      }
      bool sorted = true;
      for (size_t l = 1; l < t.size(); ++l) sorted = sorted && !(t[l].budget < t[l - 1].budget);
      if (prof_sorted.size() < profiles.size()) prof_sorted.resize(profiles.size(), 0);
      prof_sorted[need[i]] = sorted;
      profiles[need[i]] = std::move(t);
    }
  }

  // ---------------------------------------------------------- a window --
  bool step() {
    if (window >= cfg.num_windows) return false;
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto w0 = clk::now();
    samples = 0;
    const double T = cfg.T();
    const double t0 = window * T, t1 = t0 + T;
    apply_due_events(t0);
    const auto w_events = clk::now();
    if (learned() && !opt.host_frames) check(ctx, ecco_generate_frames(ctx, window));
    route_pending(t0);
    const auto w_routed = clk::now();
    double route_ms = ms(w0, w_routed);
    double net_ms = 0.0, prof_ms = 0.0, sel_ms = 0.0;
    struct Stats {
      int members = 0;
      double p = 0, c = 0, delivered = 0;
      int micros = 0;
    };
    std::map<int, Stats> wstats;
    double train_ms = 0.0, replay_ms = 0.0;
    if (!jobs.empty()) {
      const auto a0 = clk::now();
      std::vector<int> ids, members;
      for (const auto& [id, j] : jobs) {
        ids.push_back(id);
        members.push_back((int)j.members.size());
      }
      const int J = (int)ids.size();
      // WindowAllocation ctor checks (gpu_allocator.cpp:100-123)
      if (J > cfg.W)
        fail(ECCO_ERR_INFEASIBLE, "window " + std::to_string(window) + ": " + std::to_string(J) +
                                      " jobs exceed " + std::to_string(cfg.W) + " micro-windows");
      std::vector<Micro> recs;
      std::vector<int> per_job(J, 0);
      std::vector<double> acc(J), gain(J);
      int budget = cfg.W;
      // ---- initial pass: one micro per job, all jobs in one launch
      {
        std::vector<Batch> bs;
        for (int id : ids) {
          auto it = batches.find(id);
          bs.push_back(it != batches.end() ? it->second : bootstrap(jobs.at(id)));
        }
        std::vector<int> mb(J, 0);
        const auto tr = trajectories(ids, bs, mb, 1);
        std::vector<int> one(J, 1);
        check(ctx, ecco_commit(ctx, J, ids.data(), one.data()));
        for (int k = 0; k < J; ++k) {
          if (learned()) samples += (int64_t)learned_steps(bs[k]) * opt.minibatch;
          recs.push_back({(int)recs.size(), ids[k], tr[k][0], tr[k][1]});
          acc[k] = tr[k][1];
          gain[k] = tr[k][1] - tr[k][0];
          per_job[k] = 1;
          --budget;
        }
      }
      const auto a1 = clk::now();
      train_ms += ms(a0, a1);
      std::vector<double> init_scores;
      if (cfg.policy == kNaive) init_scores.assign(J, 1.0);
      else {
        prepare_scores(members);
        scores(ids, members, acc, gain, init_scores);
      }
      // estimate_shares (gpu_allocator.cpp:78-98)
      const double total_gpu_s = cfg.gpus * T;
      double total = 0.0;
      for (double g : init_scores) total += std::max(0.0, g);
      const bool uniform = !(total > 0.0);
      std::vector<double> p(J), c(J);
      for (int k = 0; k < J; ++k) {
        p[k] = uniform ? 1.0 / (double)J : std::max(0.0, init_scores[k]) / total;
        c[k] = p[k] * total_gpu_s;
      }
      // profiles needed this window (ecco / total_acc policies)
      if (cfg.policy != kNaive) {
        std::vector<int> need;
        for (int id : ids)
          for (const auto& m : jobs.at(id).members)
            if (!profiles[m.cam]) need.push_back(m.cam);
        std::sort(need.begin(), need.end());
        need.erase(std::unique(need.begin(), need.end()), need.end());
        const auto p0 = clk::now();
        build_profiles(need);
        prof_ms += ms(p0, clk::now());
      }
      // configs and flows (orchestrator.cpp:253-278)
      std::vector<double> fa, fb, fcap;
      std::vector<int> flow_cam;
      sel_f.assign(cams.size(), 0.0);  // (frame rate, resolution) per camera this window
      sel_q.assign(cams.size(), 0.0);
      for (int k = 0; k < J; ++k) {
        const Job& j = jobs.at(ids[k]);
        Stats& st = wstats[ids[k]];
        const int nm = (int)j.members.size();
        st.members = nm;
        st.p = p[k];
        st.c = c[k];
        for (const auto& m : j.members) {
          double f, q;
          if (cfg.policy == kNaive) {
            f = cfg.fixed_f;
            q = cfg.fixed_q;
          } else {
            // select_config, transmission.cpp:120-138
            // (the LAST row within budget; with non-decreasing budgets the rows
            // within budget are a prefix, so bisection finds the same row)
            const auto& t = *profiles[m.cam];
            const double lim = c[k] * (1.0 + 1e-12) + 1e-12;
            const ProfRow* row = nullptr;
            if (prof_sorted[m.cam]) {
              const auto it = std::partition_point(
                  t.begin(), t.end(), [lim](const ProfRow& r) { return r.budget <= lim; });
              if (it != t.begin()) row = &*(it - 1);
            } else {
              for (const auto& r : t)
                if (r.budget <= lim) row = &r;
            }
            if (!row) row = &t.front();
            f = row->f / nm;
            q = row->q;
          }
          sel_f[m.cam] = f;
          sel_q[m.cam] = q;
          const Cam& cm = cams[m.cam];
          fcap.push_back(cm.cap > 0.0 ? cm.cap : std::numeric_limits<double>::infinity());
          if (cfg.equal_bw) {
            fa.push_back(cfg.alpha_unit);
          } else {
            // set_aimd_params, transmission.cpp:140-149.  The parametric
            // model's gains are always > 0, so p_share > 0 there; a learned
            // job whose retrain did not raise its eval accuracy gets p = 0
            // from estimate_shares (gpu_allocator.cpp:93-95), which the
            // reference would reject.  The learned backend keeps such a
            // job's flow alive at a floor share ("deviations").
            if (learned() && !(p[k] > 0.0)) {
              fa.push_back(kLearnedShareFloor / nm * cfg.alpha_unit);
              fb.push_back(0.5);
              flow_cam.push_back(m.cam);
              continue;
            }
            if (!(p[k] > 0.0) || p[k] > 1.0 + 1e-9)
              fail(ECCO_ERR_INVALID_ARGUMENT, "set_aimd_params: p_share must be in (0,1]");
            fa.push_back(p[k] / nm * cfg.alpha_unit);
          }
          fb.push_back(0.5);
          flow_cam.push_back(m.cam);
        }
      }
      if (!(cfg.rtt > 0.0)) fail(ECCO_ERR_INVALID_ARGUMENT, "netsim: rtt must be positive");
      const auto n0 = clk::now();
      const std::vector<double> mean_rate = simulate(fa, fb, fcap);
      net_ms += ms(n0, clk::now());
      rate_of.assign(cams.size(), 0.0);
      for (size_t i = 0; i < flow_cam.size(); ++i) rate_of[flow_cam[i]] = mean_rate[i];
      // batch assembly (orchestrator.cpp:282-309)
      for (int k = 0; k < J; ++k) {
        const Job& j = jobs.at(ids[k]);
        double tf = 0, rs = 0, ql = 0, dl = 0;
        for (const auto& m : j.members) {
          const double f = sel_f[m.cam], q = sel_q[m.cam];
          const double rate = rate_of[m.cam];
          // adapt_compression, transmission.cpp:151-166
          double quality = 0.0;
          if (rate < 0.0) fail(ECCO_ERR_INVALID_ARGUMENT, "adapt_compression: negative rate");
          if (rate != 0.0) {
            const double pr = f * (q * (16.0 * q / 9.0));
            if (!(pr > 0.0)) fail(ECCO_ERR_INVALID_ARGUMENT, "adapt_compression: config has zero pixel rate");
            quality = std::min(1.0, rate / pr / cfg.bpp_ref);
          }
          tf += f;
          rs += f * q * q;
          ql += f * quality;
          dl += rate;
        }
        if (tf > 0.0) {
          Batch b;
          b.fps = tf;
          b.res = std::sqrt(rs / tf);
          b.quality = ql / tf;
          for (const auto& m : j.members) {
            b.src.push_back(m.cam);
            b.frac.push_back(sel_f[m.cam] / tf);
          }
          batches[ids[k]] = b;
        }
        wstats[ids[k]].delivered = dl;
      }
      // ---- remaining micro-windows: speculative chains + host replay
      const auto r0 = clk::now();
      sel_ms = ms(a1, r0);
      if (budget > 0) {
        std::vector<Batch> bs;
        for (int id : ids) {
          auto it = batches.find(id);
          bs.push_back(it != batches.end() ? it->second : bootstrap(jobs.at(id)));
        }
        const int maxd = std::max(1, opt_max_depth());
        int d0 = learned() ? std::max(1, std::min(maxd, opt.spec_depth)) : std::min(maxd, budget);
        std::vector<int> mb(J, 1);
        auto chains = trajectories(ids, bs, mb, std::min(d0, budget));
        std::vector<int> used(J, 0), depth_of(J, std::min(d0, budget)), base(J, 1);
        int rr = 0;
        std::vector<double> sc;
        while (budget > 0) {
          int k;
          if (cfg.policy == kNaive) {
            k = rr % J;
            ++rr;
          } else {
            scores(ids, members, acc, gain, sc);
            k = ecco_alloc::argmax(sc);
          }
          if (used[k] + 1 >= (int)chains[k].size()) {
            // chain exhausted: commit it and extend this job (depth doubling)
            check(ctx, ecco_commit(ctx, 1, &ids[k], &used[k]));
            base[k] += used[k];
            const int nd = std::min({maxd, budget, std::max(1, depth_of[k] * 2)});
            const auto ext = trajectories({ids[k]}, {bs[k]}, {base[k]}, nd);
            chains[k] = ext[0];
            used[k] = 0;
            depth_of[k] = nd;
          }
          const double before = chains[k][used[k]];
          const double after = chains[k][used[k] + 1];
          ++used[k];
          if (learned()) samples += (int64_t)learned_steps(bs[k]) * opt.minibatch;
          recs.push_back({(int)recs.size(), ids[k], before, after});
          acc[k] = after;
          gain[k] = after - before;
          per_job[k] += 1;
          --budget;
        }
        check(ctx, ecco_commit(ctx, J, ids.data(), used.data()));
      }
      const auto r1 = clk::now();
      train_ms += ms(r0, r1);
      replay_ms = 0.0;
      for (const auto& rec : recs) {
        Row row;
        row.kind = kMicro;
        row.window = window;
        row.t = t0 + (rec.index + 1) * cfg.mu;
        row.job = rec.job;
        row.v[0] = rec.index;
        row.v[1] = rec.before;
        row.v[2] = rec.after;
        rows.push_back(row);
      }
      for (int k = 0; k < J; ++k) wstats[ids[k]].micros = per_job[k];
    }
    // ---- window-end accuracies (orchestrator.cpp:328-352)
    const auto e0 = clk::now();
    {
      std::vector<int> pj, pc;
      for (const auto& [id, j] : jobs)
        for (const auto& m : j.members) {
          pj.push_back(id);
          pc.push_back(m.cam);
        }
      std::vector<double> v(pj.size());
      if (!pj.empty())
        check(ctx, ecco_eval_pairs(ctx, (int)pj.size(), nullptr, pc.data(), pj.data(), v.data()));
      size_t q = 0;
      for (auto& [id, j] : jobs) {
        double sum = 0.0;
        for (auto& m : j.members) {
          const double a = v[q++];
          j.acc_per_member[m.cam] = a;
          m.hist.push_back(a);
          cams[m.cam].acc = a;
          sum += a;
        }
        if (!j.members.empty()) j.mean_hist.push_back(sum / j.members.size());
      }
    }
    for (int ci = 0; ci < (int)cams.size(); ++ci) {
      Row row;
      row.kind = kAccuracy;
      row.window = window;
      row.t = t1;
      row.cam = ci;
      row.job = membership[ci];
      row.v[0] = cams[ci].acc;
      rows.push_back(row);
    }
    if (!jobs.empty()) regroup(t1);
    const auto e1 = clk::now();
    for (const auto& [job, st] : wstats) {
      Row row;
      row.kind = kJobWindow;
      row.window = window;
      row.t = t1;
      row.job = job;
      row.v[0] = st.members;
      row.v[1] = st.p;
      row.v[2] = st.c;
      row.v[3] = st.delivered;
      row.v[4] = st.micros;
      rows.push_back(row);
    }
    ++window;
    const auto w1 = clk::now();
    timings[0] = ms(w0, w1);
    timings[1] = route_ms + ms(e0, e1);
    timings[2] = train_ms;
    timings[3] = ms(e0, e1);
    timings[4] = replay_ms;
    timings[5] = net_ms;
    timings[6] = prof_ms;
    timings[7] = ms(w0, w_events);
    timings[8] = ms(w_events, w_routed);
    timings[9] = sel_ms - net_ms - prof_ms;
    timings[10] = ms(e1, w1);
    return true;
  }

  int opt_max_depth() const { return ecco_max_depth_cache; }
  int ecco_max_depth_cache = 8;

  // update_grouping, grouping.cpp:64-121, plus the orchestrator's rows.
  void regroup(double now) {
    if (!(cfg.drop_p > 0.0))
      fail(ECCO_ERR_INVALID_ARGUMENT, "update_grouping: drop_threshold_p must be positive");
    struct Removal {
      int cam, job;
      double drop;
      bool degenerate;
    };
    std::vector<Removal> removals;
    for (const auto& [id, j] : jobs)
      for (const auto& m : j.members) {
        const auto& h = m.hist;
        if (h.size() < 2) continue;
        const double prev = h[h.size() - 2], cur = h.back();
        if (prev <= 0.0) {
          removals.push_back({m.cam, id, 0.0, true});
          continue;
        }
        const double drop = (cur - prev) / prev;
        if (drop < -cfg.drop_p) removals.push_back({m.cam, id, drop, false});
      }
    std::vector<Request> evicted;
    std::vector<int> excl;
    for (const auto& rm : removals) {
      Job& j = jobs.at(rm.job);
      const int i = j.find(rm.cam);
      Request r = j.members[i];
      j.members.erase(j.members.begin() + i);
      j.acc_per_member.erase(rm.cam);
      const double last = r.hist.empty() ? r.acc : r.hist.back();
      r.t = now;
      r.x = cams[rm.cam].x;
      r.y = cams[rm.cam].y;
      r.scene = cams[rm.cam].scene;
      r.acc = std::max(0.0, last);
      r.hist.clear();
      evicted.push_back(std::move(r));
      excl.push_back(rm.job);
    }
    std::vector<int> terminated;
    for (auto it = jobs.begin(); it != jobs.end();) {
      if (it->second.members.empty()) {
        terminated.push_back(it->first);
        it = jobs.erase(it);
      } else {
        ++it;
      }
    }
    if (!terminated.empty()) check(ctx, ecco_drop_models(ctx, (int)terminated.size(), terminated.data()));
    const auto as = route_batch(evicted, excl);
    for (const auto& rm : removals) {
      Row row;
      row.kind = kRemove;
      row.window = window;
      row.t = now;
      row.cam = rm.cam;
      row.job = rm.job;
      row.v[0] = rm.drop;
      row.v[1] = rm.degenerate ? 1.0 : 0.0;
      rows.push_back(row);
    }
    for (int id : terminated) {
      batches.erase(id);
      Row row;
      row.kind = kTerminate;
      row.window = window;
      row.t = now;
      row.job = id;
      rows.push_back(row);
    }
    for (size_t i = 0; i < evicted.size(); ++i) {
      Row row;
      row.kind = as[i].created ? kNewJob : kJoin;
      row.window = window;
      row.t = now;
      row.cam = evicted[i].cam;
      row.job = as[i].job;
      row.v[0] = as[i].acc;
      rows.push_back(row);
    }
    refresh_membership();
  }

  // -------------------------------------------------------------- output --
  // trace.csv (metrics.cpp:49-59).  Rows are formatted once, incrementally:
  // a call formats only the rows appended since the previous one.
  const std::string& trace_csv() const {
    if (trace_text.empty()) trace_text = "record,window,time_s,camera,job,v1,v2,v3,v4,v5\n";
    char ib[24];
    for (; trace_rows < rows.size(); ++trace_rows) {
      const Row& r = rows[trace_rows];
      std::string& s = trace_text;
      s += kind_name(r.kind);
      s += ',';
      s.append(ib, std::to_chars(ib, ib + sizeof ib, r.window).ptr);
      s += ',';
      fmt_to(s, r.t);
      s += ',';
      if (r.cam >= 0) s += cams[r.cam].id;
      s += ',';
      if (r.job >= 0) s.append(ib, std::to_chars(ib, ib + sizeof ib, r.job).ptr);
      for (int k = 0; k < 5; ++k) {
        s += ',';
        fmt_to(s, r.v[k]);
      }
      s += '\n';
    }
    return trace_text;
  }
  mutable std::string trace_text;
  mutable size_t trace_rows = 0;

  std::string summary_json() const {
    json j;
    j["name"] = cfg.name;
    j["policy"] = policy_name(cfg.policy);
    j["seed"] = cfg.seed;
    j["equal_bandwidth"] = cfg.equal_bw;
    j["num_windows"] = cfg.num_windows;
    j["windows_run"] = window;
    j["window_length_s"] = cfg.T();
    json fa = json::object();
    for (const auto& c : cams) fa[c.id] = c.acc;
    j["final_accuracy"] = fa;
    // mean_accuracy_per_window, metrics.cpp:108-121
    std::map<int, std::pair<double, int>> per;
    for (const auto& r : rows)
      if (r.kind == kAccuracy) {
        auto& e = per[r.window];
        e.first += r.v[0];
        e.second += 1;
      }
    std::vector<double> means;
    for (const auto& [w, e] : per) means.push_back(e.first / std::max(1, e.second));
    j["mean_accuracy_per_window"] = means;
    json jl = json::array();
    for (const auto& [id, jb] : jobs) {
      json e;
      e["id"] = id;
      json mem = json::array();
      for (const auto& m : jb.members) mem.push_back(cams[m.cam].id);
      e["members"] = mem;
      e["mean_acc"] = jb.mean_hist.empty() ? 0.0 : jb.mean_hist.back();
      jl.push_back(e);
    }
    j["jobs"] = jl;
    if (cfg.response_target) {
      // response_time, metrics.cpp:130-149
      const double target = *cfg.response_target;
      std::map<std::string, std::pair<double, std::optional<double>>> res;
      for (const auto& r : rows) {
        if (r.kind != kRequest) continue;
        const std::string& id = cams[r.cam].id;
        if (res.count(id)) continue;
        std::optional<double> resp;
        if (r.v[0] >= target) resp = 0.0;
        res[id] = {r.t, resp};
      }
      for (const auto& r : rows) {
        if (r.kind != kAccuracy) continue;
        auto it = res.find(cams[r.cam].id);
        if (it == res.end() || it->second.second) continue;
        if (r.t >= it->second.first && r.v[0] >= target) it->second.second = r.t - it->second.first;
      }
      json rj = json::object();
      for (const auto& [id, e] : res) {
        if (e.second) rj[id] = *e.second;
        else rj[id] = nullptr;
      }
      j["response_time_s"] = rj;
    }
    return j.dump(2) + "\n";
  }
};

extern "C" {

void ecco_sim_default_options(ecco_sim_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->backend = ECCO_BACKEND_PARAMETRIC;
  o->math = ECCO_MATH_FFMA_EXACT;
  o->device = 0;
  o->spec_depth = 4;  // learned: 4 micro-windows per job up front (C4: 90 -> 64 ms per window)
  o->feat_dim = 512;
  o->hidden_dim = 256;
  o->num_classes = 16;
  o->minibatch = 128;
  o->ring_frames = 512;
  o->eval_samples = 64;
  o->sgd_lr = 0.05f;
  o->steps_per_gpu_s = 4.0;
  o->seed = 0x5eed0001ULL;
  o->host_frames = 0;
  o->full_matrix = 0;
}

ecco_status ecco_sim_create(const char* scenario_json, const ecco_sim_options* opt, ecco_sim** out,
                            char* err, size_t err_len) {
  *out = nullptr;
  auto* s = new ecco_sim();
  auto report = [&](ecco_status st, const std::string& m) {
    if (err && err_len) {
      std::snprintf(err, err_len, "%s", m.c_str());
    }
    if (s->ctx) ecco_destroy(s->ctx);
    delete s;
    return st;
  };
  try {
    s->cfg = parse_scenario(scenario_json);
    if (opt) s->opt = *opt;
    else ecco_sim_default_options(&s->opt);
    // cameras in std::string order: index order == the reference's map order
    std::vector<CamSpec> sorted = s->cfg.cams;
    std::sort(sorted.begin(), sorted.end(), [](const CamSpec& a, const CamSpec& b) { return a.id < b.id; });
    for (size_t i = 0; i < sorted.size(); ++i) {
      const auto& c = sorted[i];
      s->cam_index[c.id] = (int)i;
      s->cams.push_back({c.id, c.x, c.y, c.scene, c.acc, c.cap, c.tp, c.bias});
    }
    s->D = (int)s->cams[0].scene.size();
    s->membership.assign(s->cams.size(), -1);
    s->profiles.resize(s->cams.size());
    s->events = s->cfg.events;
    for (auto& e : s->events) e.ci = s->cam_index.at(e.cam);
    std::stable_sort(s->events.begin(), s->events.end(), [](const Event& a, const Event& b) {
      if (a.t != b.t) return a.t < b.t;
      return a.cam < b.cam;
    });
    ecco_config cfg;
    ecco_default_config(&cfg);
    cfg.backend = s->opt.backend;
    cfg.device = s->opt.device;
    cfg.scene_dims = s->D;
    cfg.params = s->cfg.model;
    cfg.max_cameras = (int)s->cams.size();
    cfg.max_jobs = 2 * (int)s->cams.size() + 16;
    cfg.math = s->opt.math;
    cfg.feat_dim = s->opt.feat_dim;
    cfg.hidden_dim = s->opt.hidden_dim;
    cfg.num_classes = s->opt.num_classes;
    cfg.minibatch = s->opt.minibatch;
    cfg.ring_frames = s->opt.ring_frames;
    cfg.eval_samples = s->opt.eval_samples;
    cfg.sgd_lr = s->opt.sgd_lr;
    cfg.steps_per_gpu_s = s->opt.steps_per_gpu_s;
    cfg.seed = s->opt.seed;
    cfg.max_depth = s->opt.backend == ECCO_BACKEND_LEARNED ? std::max(2, std::max(8, s->opt.spec_depth))
                                                            : std::min(64, std::max(1, s->cfg.W));
    s->ecco_max_depth_cache = cfg.max_depth;
    const ecco_status st = ecco_create(&cfg, &s->ctx);
    if (st != ECCO_OK) return report(st, "ecco_create failed");
    std::vector<double> sc, tp;
    for (const auto& c : s->cams) {
      sc.insert(sc.end(), c.scene.begin(), c.scene.end());
      tp.push_back(c.tp);
    }
    check(s->ctx, ecco_set_cameras(s->ctx, (int)s->cams.size(), sc.data(), tp.data()));
    if (s->learned()) {
      const int base = kBaseModelId;
      check(s->ctx, ecco_seed_models(s->ctx, 1, &base, nullptr, nullptr));
    }
  } catch (const SimError& e) {
    return report(e.code, e.msg);
  } catch (const std::exception& e) {
    return report(ECCO_ERR_RUNTIME, e.what());
  }
  *out = s;
  return ECCO_OK;
}

void ecco_sim_destroy(ecco_sim* s) {
  if (!s) return;
  if (s->ctx) ecco_destroy(s->ctx);
  delete s;
}

const char* ecco_sim_last_error(const ecco_sim* s) { return s ? s->err.c_str() : "no sim"; }

ecco_status ecco_sim_step_window(ecco_sim* s, int* ran) {
  try {
    *ran = s->step() ? 1 : 0;
    return ECCO_OK;
  } catch (const SimError& e) {
    s->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    s->err = e.what();
    return ECCO_ERR_RUNTIME;
  }
}

ecco_status ecco_sim_last_timings(const ecco_sim* s, double* out5) {
  for (int i = 0; i < 5; ++i) out5[i] = s->timings[i];
  return ECCO_OK;
}

int64_t ecco_sim_last_samples(const ecco_sim* s) { return s->samples; }

size_t ecco_sim_trace_csv(const ecco_sim* s, char* buf, size_t cap) {
  const std::string& t = s->trace_csv();
  if (buf && cap) std::memcpy(buf, t.data(), std::min(cap, t.size()));
  return t.size();
}

size_t ecco_sim_summary_json(const ecco_sim* s, char* buf, size_t cap) {
  const std::string t = s->summary_json();
  if (buf && cap) std::memcpy(buf, t.data(), std::min(cap, t.size()));
  return t.size();
}

ecco_ctx* ecco_sim_context(ecco_sim* s) { return s->ctx; }

}  // extern "C"

ecco_status ecco_netsim_mean_rates(int n, const double* alpha, const double* beta,
                                   const double* caps, double capacity, double rtt_s,
                                   double duration_s, double* mean_rates, int* exact_steps) {
  if (!(capacity > 0.0) || !(rtt_s > 0.0) || !(duration_s > 0.0) || n < 0)
    return ECCO_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < n; ++i)
    if (!(alpha[i] > 0.0) || !(beta[i] > 0.0 && beta[i] < 1.0)) return ECCO_ERR_INVALID_ARGUMENT;
  std::vector<double> c(caps, caps + n);
  for (double& x : c)
    if (!(x > 0.0)) x = std::numeric_limits<double>::infinity();  // resolve_caps (netsim.cpp:33-40)
  const int steps = (int)std::llround(duration_s / rtt_s);
  const int ex = n ? ecco_netsim::mean_rates((size_t)n, alpha, beta, c.data(), capacity, steps,
                                             mean_rates)
                   : 0;
  if (exact_steps) *exact_steps = ex;
  return ECCO_OK;
}

int ecco_sim_last_timings_ex(const ecco_sim* s, double* out, int n) {
  if (!s || !out) return 0;
  const int k = std::min(n, 11);
  for (int i = 0; i < k; ++i) out[i] = s->timings[i];
  return k;
}

ecco_status ecco_allocate_trajectories(int n_jobs, const int* job_ids, const int* members,
                                       const double* traj, int traj_len, double alpha, double beta,
                                       int micro_windows, double micro_s, int gpu_count, int bonus,
                                       int policy, int* out_job, double* out_before,
                                       double* out_after, double* out_initial_scores) {
  // AllocatorConfig::validate (gpu_allocator.cpp:19-30) and the
  // WindowAllocation constructor's checks (:100-123)
  if (alpha < 0.0 || beta > 1.0 || micro_windows < 1 || !(micro_s > 0.0) || gpu_count < 1 ||
      n_jobs < 0 || traj_len < 1 || policy < 0 || policy > 2)
    return ECCO_ERR_INVALID_ARGUMENT;
  std::vector<int> order(n_jobs);
  for (int j = 0; j < n_jobs; ++j) order[j] = j;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return job_ids[a] < job_ids[b]; });
  std::vector<int> ids(n_jobs), mem(n_jobs);
  for (int k = 0; k < n_jobs; ++k) {
    ids[k] = job_ids[order[k]];
    mem[k] = members[order[k]];
    if (mem[k] < 1) return ECCO_ERR_INVALID_ARGUMENT;
    if (k && ids[k] == ids[k - 1]) return ECCO_ERR_INVALID_ARGUMENT;
  }
  if (n_jobs == 0 || n_jobs > micro_windows) return ECCO_ERR_INFEASIBLE;
  std::vector<int> cursor(n_jobs, 0);
  std::vector<double> acc(n_jobs, 0.0), gain(n_jobs, 0.0), coef, sc;
  ecco_alloc::size_coef(mem, alpha, beta, coef);
  int budget = micro_windows, rec = 0;
  auto at = [&](int k, int c) { return traj[(size_t)order[k] * traj_len + std::min(c, traj_len - 1)]; };
  auto run_micro = [&](int k) {  // run_micro (:125-135) over the trajectory backend
    const double before = at(k, cursor[k]);
    ++cursor[k];
    const double after = at(k, cursor[k]);
    --budget;
    acc[k] = after;
    gain[k] = after - before;
    out_job[rec] = ids[k];
    out_before[rec] = before;
    out_after[rec] = after;
    ++rec;
  };
  for (int k = 0; k < n_jobs; ++k) run_micro(k);  // run_initial_pass (:160-166)
  if (policy != 1) {
    ecco_alloc::scores(policy == 2, bonus != 0, coef, ids, mem, acc, gain, sc);
    if (out_initial_scores)
      for (int k = 0; k < n_jobs; ++k) out_initial_scores[k] = sc[k];
  }
  int rr = 0;
  bool finite = true;  // the trees reproduce the scans' picks when no key is NaN
  for (size_t i = 0; i < (size_t)n_jobs * traj_len; ++i) finite = finite && !std::isnan(traj[i]);
  if (policy == 1 || !finite) {
    while (budget > 0) {  // run_remaining (:168-181)
      int k;
      if (policy == 1) {
        k = rr % n_jobs;
        ++rr;
      } else {
        ecco_alloc::scores(policy == 2, bonus != 0, coef, ids, mem, acc, gain, sc);
        k = ecco_alloc::argmax(sc);
      }
      run_micro(k);
    }
    return ECCO_OK;
  }
  // the same greedy, each pick from two tournament trees: the bonus-free
  // score (coef * gain, or members * gain for total_acc) and, for the
  // fairness bonus, the least-accurate job (lowest id on ties)
  std::vector<double> base(n_jobs);
  auto base_of = [&](int k) { return policy == 2 ? mem[k] * gain[k] : coef[k] * gain[k]; };
  for (int k = 0; k < n_jobs; ++k) base[k] = base_of(k);
  auto hi = [&](int a, int b) { return base[a] > base[b]; };
  auto lo = [&](int a, int b) { return acc[a] < acc[b]; };
  ecco_alloc::Tourney<decltype(hi)> top(n_jobs, hi);
  ecco_alloc::Tourney<decltype(lo)> low(n_jobs, lo);
  const bool with_bonus = policy == 0 && bonus != 0;
  while (budget > 0) {
    int k = top.best();
    if (with_bonus) {
      const int m = low.best();
      const double boosted = base[m] + gain[m];
      const int v = top.best_except(m);
      k = v < 0 || boosted > base[v] || (boosted == base[v] && m < v) ? m : v;
    }
    run_micro(k);
    base[k] = base_of(k);
    top.update(k);
    low.update(k);
  }
  return ECCO_OK;
}
