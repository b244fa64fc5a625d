// Host engine of the B200-native MoE-SpeQ decode path (C++; calls CUDA kernels only through
// the C-ABI in include/mspq_capi.h).
//
//  * perfmodel restatement (perfmodel.cpp:85-217): k_accept, t_draft, t_pcie_new, t_verify,
//    t_cycle, select_k, k_slo_from_ttft, update_acceptance -- the Amortization-Roofline
//    governor, evaluated on a HardwareProfile re-fit from measured B200 numbers.
//  * replay(): Engine::run (sim.cpp:98-432) with every cache decision made by the device
//    controller (K4, token-major) and the modeled two-lane timing restated on the host.
//  * Engine::generate(): live speculative decode -- draft step as a CUDA graph, per-row
//    planner launches, copy-engine H2D into the HBM slot pool, layer-major bf16 verify,
//    device accept scan, governor.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mspq_capi.h"
#include "json.hpp"
#include "host_common.h"
#include "status.h"

using json = nlohmann::ordered_json;

namespace mspq_host {

[[noreturn]] void fail(int code, const std::string& msg) { throw Err{code, msg}; }
#define CUDA_OK(x)                                                                     \
  do {                                                                                 \
    cudaError_t _e = (x);                                                              \
    if (_e != cudaSuccess) fail(MSPQ_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
  } while (0)
#define CAPI_OK(x)                                   \
  do {                                               \
    int _s = (x);                                    \
    if (_s) fail(_s, std::string(#x) + ": " + mspq_last_error()); \
  } while (0)

// ============================================================================ perfmodel
void Profile::validate() const {  // perfmodel.cpp:22-31
  if (pcie_bandwidth <= 0.0) fail(MSPQ_ERR_INVALID_CONFIG, "pcie_bandwidth must be > 0");
  if (pcie_init_latency < 0.0 || pcie_overhead < 0.0) fail(MSPQ_ERR_INVALID_CONFIG, "pcie latencies must be >= 0");
  if (expert_size_bytes == 0) fail(MSPQ_ERR_INVALID_CONFIG, "expert_size_bytes must be > 0");
  if (draft_base < 0.0 || draft_per_token <= 0.0) fail(MSPQ_ERR_INVALID_CONFIG, "draft costs must be positive");
  if (token_bytes <= 0.0) fail(MSPQ_ERR_INVALID_CONFIG, "token_bytes must be > 0");
  check_samples();
}
void Profile::check_samples() const {
  if (verify_samples.size() < 2) fail(MSPQ_ERR_INSUFFICIENT_SAMPLES, "need at least two verify samples");
  for (size_t i = 1; i < verify_samples.size(); ++i)
    if (verify_samples[i].first <= verify_samples[i - 1].first)
      fail(MSPQ_ERR_INVALID_CONFIG, "verify sample windows must be strictly increasing");
}
Profile Profile::from_json(const json& j) {  // perfmodel.cpp:33-63
  if (!j.is_object()) fail(MSPQ_ERR_INVALID_CONFIG, "profile must be a JSON object");
  Profile p;
  for (auto it = j.begin(); it != j.end(); ++it) {
    const std::string& k = it.key();
    if (k == "pcie_bandwidth_bytes_per_s") p.pcie_bandwidth = it->get<double>();
    else if (k == "pcie_init_latency_s") p.pcie_init_latency = it->get<double>();
    else if (k == "pcie_overhead_s") p.pcie_overhead = it->get<double>();
    else if (k == "expert_size_bytes") p.expert_size_bytes = it->get<uint64_t>();
    else if (k == "draft_base_s") p.draft_base = it->get<double>();
    else if (k == "draft_per_token_s") p.draft_per_token = it->get<double>();
    else if (k == "token_bytes") p.token_bytes = it->get<double>();
    else if (k == "verify_samples") {
      p.verify_samples.clear();
      for (const auto& s : *it) {
        if (!s.is_array() || s.size() != 2) fail(MSPQ_ERR_INVALID_CONFIG, "verify_samples entries must be [window, seconds]");
        p.verify_samples.emplace_back(s[0].get<double>(), s[1].get<double>());
      }
    } else
      fail(MSPQ_ERR_INVALID_CONFIG, "unknown profile field: " + k);
  }
  p.validate();
  return p;
}
json Profile::to_json() const {
  json j;
  j["pcie_bandwidth_bytes_per_s"] = pcie_bandwidth;
  j["pcie_init_latency_s"] = pcie_init_latency;
  j["pcie_overhead_s"] = pcie_overhead;
  j["expert_size_bytes"] = expert_size_bytes;
  j["draft_base_s"] = draft_base;
  j["draft_per_token_s"] = draft_per_token;
  j["token_bytes"] = token_bytes;
  j["verify_samples"] = json::array();
  for (auto& [w, s] : verify_samples) j["verify_samples"].push_back({w, s});
  return j;
}

double k_accept(const std::vector<double>& p, int k) {  // perfmodel.cpp:85-97
  if (k < 0 || k > (int)p.size()) fail(MSPQ_ERR_K_OUT_OF_RANGE, "k out of modeled positions");
  double sum = 0.0, prefix = 1.0;
  for (int i = 0; i < k; ++i) {
    prefix *= p[i];
    sum += prefix;
  }
  return sum;
}
double t_draft(const Profile& p, int k) { return p.draft_base + static_cast<double>(k) * p.draft_per_token; }
double t_pcie_new(const Profile& p, int n) {
  if (n < 0) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "num_new_experts must be >= 0");
  if (n == 0) return 0.0;
  return p.pcie_overhead + static_cast<double>(n) * static_cast<double>(p.expert_size_bytes) / p.pcie_bandwidth;
}
double t_verify(const Profile& p, double window) {
  const auto& s = p.verify_samples;
  p.check_samples();
  size_t hi = 1;
  while (hi + 1 < s.size() && s[hi].first < window) ++hi;
  const auto& [x0, y0] = s[hi - 1];
  const auto& [x1, y1] = s[hi];
  const double t = (window - x0) / (x1 - x0);
  return y0 + t * (y1 - y0);
}
double t_cycle(const Profile& p, int k, int n) {
  return std::max(t_draft(p, k), p.pcie_init_latency) + t_pcie_new(p, n) + t_verify(p, static_cast<double>(k + 1));
}
int select_k(const Profile& p, const std::vector<double>& acc, int k_min, int k_max, int k_slo, const Est& est) {
  const int hi = std::min(k_max, k_slo);
  if (k_min > hi) fail(MSPQ_ERR_EMPTY_RANGE, "k_min exceeds the SLO-constrained maximum");
  if (k_min < 1) fail(MSPQ_ERR_K_OUT_OF_RANGE, "k_min must be >= 1");
  int best_k = k_min;
  double best = -1.0;
  for (int k = k_min; k <= hi; ++k) {
    const double v = k_accept(acc, k) / t_cycle(p, k, est(k));
    if (v > best) {
      best = v;
      best_k = k;
    }
  }
  return best_k;
}
int k_slo_from_ttft(const Profile& p, double budget, const Est& est, int k_min, int k_max) {
  if (k_min < 1 || k_min > k_max) fail(MSPQ_ERR_EMPTY_RANGE, "invalid [k_min, k_max]");
  auto lat = [&](int k) { return t_cycle(p, k, est(k)); };
  if (budget < lat(k_min)) fail(MSPQ_ERR_INFEASIBLE_BUDGET, "budget below the k_min cycle latency");
  int lo = k_min, hi = k_max;
  while (lo < hi) {
    const int mid = lo + (hi - lo + 1) / 2;
    if (lat(mid) <= budget) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
std::vector<double> update_acceptance(const std::vector<double>& p, double a, const std::vector<bool>& o) {
  if (o.size() > p.size()) fail(MSPQ_ERR_K_OUT_OF_RANGE, "more outcomes than modeled positions");
  std::vector<double> q = p;
  for (size_t i = 0; i < o.size(); ++i) {
    q[i] = (1.0 - a) * q[i] + a * (o[i] ? 1.0 : 0.0);
    if (!o[i]) break;
  }
  return q;
}

// ============================================================================ config


int parse_policy(const std::string& s) {
  if (s == "lru") return 0;
  if (s == "lookahead") return 1;
  if (s == "sp-sooner") return 2;
  if (s == "sp-later") return 3;
  if (s == "speculative") return 4;
  fail(MSPQ_ERR_UNKNOWN_POLICY, s);
}
const char* policy_name(int p) {
  static const char* n[] = {"lru", "lookahead", "sp-sooner", "sp-later", "speculative"};
  return n[p];
}

HostCfg parse_host_cfg(const std::string& text) {
  json j = json::parse(text, nullptr, false);
  if (j.is_discarded() || !j.is_object()) fail(MSPQ_ERR_INVALID_CONFIG, "config is not a JSON object");
  HostCfg c;
  static const std::set<std::string> known = {"policy", "capacity_mode", "cache_capacity", "entropy_weighted_capacity",
                                              "k", "governor", "phases", "prefetch_budget", "rollback_s", "ema_alpha",
                                              "initial_accept", "seed", "collect_plans", "profile", "profile_path", "log",
                                              "generator", "verify_overlap", "estimator", "prefetch_defer",
                                              "refetch_from_hbm"};
  for (auto it = j.begin(); it != j.end(); ++it)
    if (!known.count(it.key())) fail(MSPQ_ERR_INVALID_CONFIG, "unknown key in run config: " + it.key());
  auto num = [&](const json& o, const char* k, double d) {
    if (!o.contains(k)) return d;
    if (!o[k].is_number()) fail(MSPQ_ERR_INVALID_CONFIG, std::string(k) + " must be a number");
    return o[k].get<double>();
  };
  auto integer = [&](const json& o, const char* k, long d) {
    if (!o.contains(k)) return d;
    if (!o[k].is_number_integer()) fail(MSPQ_ERR_INVALID_CONFIG, std::string(k) + " must be an integer");
    return o[k].get<long>();
  };
  if (j.contains("policy")) c.policy = parse_policy(j["policy"].get<std::string>());
  if (j.contains("capacity_mode")) {
    std::string m = j["capacity_mode"].get<std::string>();
    if (m == "per_layer") c.mode = 0;
    else if (m == "global") c.mode = 1;
    else fail(MSPQ_ERR_INVALID_CONFIG, "capacity_mode must be \"per_layer\" or \"global\"");
  }
  c.cache_capacity = integer(j, "cache_capacity", c.cache_capacity);
  if (j.contains("entropy_weighted_capacity")) c.entropy_weighted = j["entropy_weighted_capacity"].get<bool>();
  if (j.contains("k")) {
    if (j["k"].is_string() && j["k"].get<std::string>() == "governor") c.use_governor = true;
    else if (j["k"].is_number_integer()) {
      c.use_governor = false;
      c.fixed_k = j["k"].get<int>();
    } else
      fail(MSPQ_ERR_INVALID_CONFIG, "k must be an integer or \"governor\"");
  }
  if (j.contains("governor")) {
    const auto& g = j["governor"];
    for (auto it = g.begin(); it != g.end(); ++it)
      if (it.key() != "k_min" && it.key() != "k_max" && it.key() != "k_slo" && it.key() != "ttft_budget_s")
        fail(MSPQ_ERR_INVALID_CONFIG, "unknown key in governor: " + it.key());
    c.k_min = (int)integer(g, "k_min", c.k_min);
    c.k_max = (int)integer(g, "k_max", c.k_max);
    c.k_slo = (int)integer(g, "k_slo", c.k_slo);
    c.ttft_budget = num(g, "ttft_budget_s", c.ttft_budget);
  }
  if (j.contains("phases")) {  // run_config.cpp:142-146
    if (!j["phases"].is_object()) fail(MSPQ_ERR_INVALID_CONFIG, "phases must be an object");
    for (auto it = j["phases"].begin(); it != j["phases"].end(); ++it)
      if (it.key() != "f1" && it.key() != "f2") fail(MSPQ_ERR_INVALID_CONFIG, "unknown key in phases: " + it.key());
    c.f1 = num(j["phases"], "f1", c.f1);
    c.f2 = num(j["phases"], "f2", c.f2);
  }
  c.budget = (int)integer(j, "prefetch_budget", c.budget);
  c.rollback = num(j, "rollback_s", c.rollback);
  c.ema_alpha = num(j, "ema_alpha", c.ema_alpha);
  c.initial_accept = num(j, "initial_accept", c.initial_accept);
  if (j.contains("collect_plans")) c.collect_plans = j["collect_plans"].get<bool>();
  if (j.contains("log")) c.log = j["log"].get<bool>();
  if (j.contains("verify_overlap")) c.verify_overlap = j["verify_overlap"].get<bool>();
  if (j.contains("prefetch_defer")) c.prefetch_defer = j["prefetch_defer"].get<bool>();
  if (j.contains("refetch_from_hbm")) c.refetch_from_hbm = j["refetch_from_hbm"].get<bool>();
  // profile / profile_path (run_config.cpp:155-170): exclusive; a relative path resolves against
  // the caller's working directory (the reference's base_dir for an inline config)
  if (j.contains("profile") && j.contains("profile_path"))
    fail(MSPQ_ERR_INVALID_CONFIG, "give either profile or profile_path, not both");
  if (j.contains("profile")) {
    c.profile = Profile::from_json(j["profile"]);
    c.profile_given = true;
  } else if (j.contains("profile_path")) {
    if (!j["profile_path"].is_string()) fail(MSPQ_ERR_INVALID_CONFIG, "profile_path must be a string");
    const std::string path = j["profile_path"].get<std::string>();
    std::ifstream in(path);
    if (!in) fail(MSPQ_ERR_IO, "cannot open profile file: " + path);
    json pj = json::parse(in, nullptr, false);
    if (pj.is_discarded()) fail(MSPQ_ERR_INVALID_CONFIG, "profile file is not valid JSON: " + path);
    c.profile = Profile::from_json(pj);
    c.profile_given = true;
  }
  if (j.contains("estimator")) {  // governor |E_new(k)| estimator (not in the reference schema)
    if (!j["estimator"].is_string()) fail(MSPQ_ERR_INVALID_CONFIG, "estimator must be a string");
    const std::string e = j["estimator"].get<std::string>();
    if (e == "linear") c.estimator = 0;
    else if (e == "elb") c.estimator = 1;
    else fail(MSPQ_ERR_INVALID_CONFIG, "estimator must be \"linear\" or \"elb\"");
  }
  return c;
}

void validate_host_cfg(const HostCfg& c, int top_k) {  // SimConfig::validate, sim.cpp:436-456
  c.profile.validate();
  if (!c.use_governor && c.fixed_k < 1) fail(MSPQ_ERR_INVALID_CONFIG, "fixed k must be >= 1");
  if (c.use_governor) {
    if (c.k_min < 1 || c.k_min > c.k_max) fail(MSPQ_ERR_INVALID_CONFIG, "governor needs 1 <= k_min <= k_max");
    if (c.k_slo < c.k_min) fail(MSPQ_ERR_INVALID_CONFIG, "governor k_slo below k_min");
  }
  if (c.cache_capacity < top_k) fail(MSPQ_ERR_INVALID_CONFIG, "cache capacity below top_k cannot serve one step");
  if (c.f1 < 0.0 || c.f2 < c.f1 || c.f2 > 1.0) fail(MSPQ_ERR_INVALID_CONFIG, "phase boundaries need 0 <= f1 <= f2 <= 1");
  if (c.budget < 0) fail(MSPQ_ERR_INVALID_CONFIG, "prefetch budget must be >= 0");
  if (c.rollback < 0.0) fail(MSPQ_ERR_INVALID_CONFIG, "rollback must be >= 0");
  if (c.ema_alpha < 0.0 || c.ema_alpha > 1.0) fail(MSPQ_ERR_INVALID_CONFIG, "ema_alpha must be in [0, 1]");
  if (c.initial_accept < 0.0 || c.initial_accept > 1.0) fail(MSPQ_ERR_INVALID_CONFIG, "initial_accept must be in [0, 1]");
}

// ============================================================================ trace (JSONL)
struct Trace {
  int L = 0, N = 0, K = 0, shared = 0;
  uint64_t expert_bytes = 0;
  std::vector<int32_t> target, draft;  // [n][L][K]
  std::vector<double> gates;           // [n][L][K] if has_gates
  std::vector<char> acc;
  bool has_gates = false;
  int n = 0;
};

Trace parse_trace(const std::string& text) {  // trace.cpp:226-278 (structural checks)
  Trace t;
  std::istringstream in(text);
  std::string line;
  int line_no = 0;
  if (!std::getline(in, line)) fail(MSPQ_ERR_EMPTY_TRACE, "stream contains no header line");
  ++line_no;
  json h = json::parse(line, nullptr, false);
  if (h.is_discarded() || !h.is_object() || !h.contains("shape")) fail(MSPQ_ERR_MALFORMED_RECORD, "header (line 1)");
  const auto& sh = h["shape"];
  for (const char* f : {"L", "N", "top_k", "shared", "expert_bytes"})
    if (!sh.contains(f) || !sh[f].is_number()) fail(MSPQ_ERR_MALFORMED_RECORD, std::string("shape missing numeric field ") + f);
  t.L = sh["L"].get<int>();
  t.N = sh["N"].get<int>();
  t.K = sh["top_k"].get<int>();
  t.shared = sh["shared"].get<int>();
  t.expert_bytes = sh["expert_bytes"].get<uint64_t>();
  if (t.L < 1 || t.N < 1 || t.K < 1 || t.K > t.N || t.shared < 0) fail(MSPQ_ERR_SHAPE_VIOLATION, "shape");
  bool first = true;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    json r = json::parse(line, nullptr, false);
    if (r.is_discarded() || !r.is_object()) fail(MSPQ_ERR_MALFORMED_RECORD, "record is not a JSON object (line " + std::to_string(line_no) + ")");
    for (const char* f : {"pos", "target", "draft", "acc"})
      if (!r.contains(f)) fail(MSPQ_ERR_MALFORMED_RECORD, std::string("record missing field ") + f);
    if (r["pos"].get<int>() != t.n) fail(MSPQ_ERR_SHAPE_VIOLATION, "pos out of order (line " + std::to_string(line_no) + ")");
    auto routing = [&](const json& arr, std::vector<int32_t>& out) {
      if (!arr.is_array() || (int)arr.size() != t.L) fail(MSPQ_ERR_SHAPE_VIOLATION, "layer entries");
      size_t base = out.size();
      out.resize(base + (size_t)t.L * t.K, -1);
      for (const auto& ent : arr) {
        int l = ent[0].get<int>();
        if (l < 0 || l >= t.L) fail(MSPQ_ERR_SHAPE_VIOLATION, "layer out of range");
        const auto& es = ent[1];
        if ((int)es.size() != t.K) fail(MSPQ_ERR_SHAPE_VIOLATION, "top_k mismatch");
        for (int j = 0; j < t.K; ++j) {
          int e = es[j].get<int>();
          if (e < 0 || e >= t.N) fail(MSPQ_ERR_SHAPE_VIOLATION, "expert out of range");
          out[base + (size_t)l * t.K + j] = e;
        }
      }
    };
    routing(r["target"], t.target);
    routing(r["draft"], t.draft);
    const bool g = r.contains("gates");
    if (first) t.has_gates = g;
    first = false;
    if (g != t.has_gates) fail(MSPQ_ERR_SHAPE_VIOLATION, "gates present on some records only");
    if (g) {
      size_t base = t.gates.size();
      t.gates.resize(base + (size_t)t.L * t.K, 0.0);
      for (const auto& ent : r["gates"]) {
        int l = ent[0].get<int>();
        for (int j = 0; j < t.K; ++j) t.gates[base + (size_t)l * t.K + j] = ent[1][j].get<double>();
      }
    }
    t.acc.push_back(r["acc"].get<bool>() ? 1 : 0);
    ++t.n;
  }
  return t;
}

double layer_entropy(const Trace& t, int l) {  // trace.cpp:401-420
  std::vector<uint64_t> counts(t.N, 0);
  uint64_t total = 0;
  for (int i = 0; i < t.n; ++i)
    for (int j = 0; j < t.K; ++j) {
      ++counts[t.target[((size_t)i * t.L + l) * t.K + j]];
      ++total;
    }
  double h = 0.0;
  for (uint64_t c : counts) {
    if (!c) continue;
    const double p = static_cast<double>(c) / static_cast<double>(total);
    h -= p * std::log2(p);
  }
  return h;
}

std::vector<int> layer_caps(const HostCfg& c, const Trace* t, int L, int K) {  // sim.cpp:26-43
  std::vector<int> caps(L, (int)c.cache_capacity);
  if (c.mode != 0 || !c.entropy_weighted || !t || t->n == 0) return caps;
  std::vector<double> h(L);
  double mean = 0.0;
  for (int l = 0; l < L; ++l) {
    h[l] = layer_entropy(*t, l);
    mean += h[l];
  }
  mean /= static_cast<double>(L);
  if (mean <= 0.0) return caps;
  for (int l = 0; l < L; ++l) {
    const double scaled = static_cast<double>(c.cache_capacity) * h[l] / mean;
    caps[l] = (int)std::max<long long>(K, std::llround(scaled));
  }
  return caps;
}

json segment(const char* lane, const char* label, double start, double dur) {
  json s;
  s["lane"] = lane;
  s["label"] = label;
  s["start_s"] = start;
  s["duration_s"] = dur;
  return s;
}

// ============================================================================ replay
// run_simulation (sim.cpp:458-466) with the device control plane.
std::string replay(int device, const std::string& trace_text, const std::string& cfg_text) {
  CUDA_OK(cudaSetDevice(device));
  Trace t = parse_trace(trace_text);
  HostCfg c = parse_host_cfg(cfg_text);
  validate_host_cfg(c, t.K);
  json rep;
  auto finish_empty = [&]() {
    rep["total_tokens"] = 0;
    rep["total_time_s"] = 0.0;
    rep["tpot_s"] = 0.0;
    rep["ttft_s"] = 0.0;
    rep["mean_coverage"] = 0.0;
    rep["mean_step_coverage"] = 0.0;
    rep["mean_accepted"] = 0.0;
    rep["stall_time_s"] = 0.0;
    rep["total_new_experts"] = 0;
    rep["cycles"] = json::array();
    return rep.dump();
  };
  if (t.n == 0) return finish_empty();
  Profile prof = c.profile;
  if (t.expert_bytes > 0) prof.expert_size_bytes = t.expert_bytes;  // sim.cpp:54-55
  const int L = t.L, K = t.K, E = t.N, n = t.n;
  const int kcap = std::max(c.use_governor ? c.k_max : c.fixed_k, 1);
  std::vector<int> caps = layer_caps(c, &t, L, K);
  // device state
  cudaStream_t st;
  CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  mspq_cache* cache = nullptr;
  CAPI_OK(mspq_cache_create(L, E, K, kcap, L * E + 8, 0, &cache));
  struct Guard {
    mspq_cache* c;
    cudaStream_t s;
    std::vector<void*> d, h;
    ~Guard() {
      for (void* p : d) cudaFree(p);
      for (void* p : h) cudaFreeHost(p);
      mspq_cache_destroy(c);
      cudaStreamDestroy(s);
    }
  } guard{cache, st, {}, {}};
  CAPI_OK(mspq_cache_configure(cache, c.mode, c.policy, caps.data(), (int)c.cache_capacity, c.budget, c.f1, c.f2, st));
  int32_t *d_tgt, *d_dr;
  double* d_g = nullptr;
  const size_t ne = (size_t)n * L * K;
  CUDA_OK(cudaMalloc(&d_tgt, ne * 4));
  guard.d.push_back(d_tgt);
  CUDA_OK(cudaMalloc(&d_dr, ne * 4));
  guard.d.push_back(d_dr);
  CUDA_OK(cudaMemcpyAsync(d_tgt, t.target.data(), ne * 4, cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemcpyAsync(d_dr, t.draft.data(), ne * 4, cudaMemcpyHostToDevice, st));
  if (t.has_gates) {
    CUDA_OK(cudaMalloc(&d_g, ne * 8));
    guard.d.push_back(d_g);
    CUDA_OK(cudaMemcpyAsync(d_g, t.gates.data(), ne * 8, cudaMemcpyHostToDevice, st));
  }
  // per-cycle output block: counts | batches | jit_rows | cov | step
  const size_t o_counts = 0, o_batch = 8, o_jit = o_batch + (size_t)kcap * 3, o_cov = o_jit + (size_t)kcap * 2,
               o_step = o_cov + (size_t)L * 2, o_end = o_step + (size_t)(kcap + 1) * L * 2;
  int32_t *d_out, *d_flush, *h_out;
  CUDA_OK(cudaMalloc(&d_out, o_end * 4));
  guard.d.push_back(d_out);
  CUDA_OK(cudaMalloc(&d_flush, (size_t)L * E * 4));
  guard.d.push_back(d_flush);
  CUDA_OK(cudaHostAlloc((void**)&h_out, o_end * 4, 0));
  guard.h.push_back(h_out);
  mspq_cache_view view;
  CAPI_OK(mspq_cache_view_get(cache, &view));
  std::vector<int32_t> h_plan(view.plan_cap * 3), h_log;
  if (c.log) h_log.resize((size_t)view.log_cap * 6);

  std::vector<double> accept(kcap, c.initial_accept);
  double g = static_cast<double>(L) * static_cast<double>(K);
  auto est = [&g]() { return Est([gg = g](int k) { return static_cast<int>(std::llround(gg * static_cast<double>(k))); }); };
  int k_slo = c.k_slo;
  if (c.use_governor && c.ttft_budget > 0.0) k_slo = std::min(k_slo, k_slo_from_ttft(prof, c.ttft_budget, est(), c.k_min, c.k_max));

  // Without per-event logs or plans the whole trace runs in ONE device launch with the governor on
  // the device (mspq_cache_replay_all); the host then walks the per-cycle slices with the timing
  // model below and re-derives every k to check the device's choice.  With logs/plans (tests) each
  // cycle is one launch.
  const bool all_mode = !c.log && !c.collect_plans && (int)prof.verify_samples.size() <= 16;
  std::vector<int32_t> k_dev;
  int32_t* h_all = nullptr;
  if (all_mode) {
    std::vector<unsigned char> acc8(t.acc.begin(), t.acc.end());
    unsigned char* d_acc;
    int32_t *d_slices, *d_k, *d_nc;
    CUDA_OK(cudaMalloc(&d_acc, (size_t)n));
    guard.d.push_back(d_acc);
    CUDA_OK(cudaMalloc(&d_slices, (size_t)n * o_end * 4));
    guard.d.push_back(d_slices);
    CUDA_OK(cudaMalloc(&d_k, (size_t)n * 4));
    guard.d.push_back(d_k);
    CUDA_OK(cudaMalloc(&d_nc, 4));
    guard.d.push_back(d_nc);
    CUDA_OK(cudaMemcpyAsync(d_acc, acc8.data(), (size_t)n, cudaMemcpyHostToDevice, st));
    const int32_t gi[6] = {c.use_governor ? 1 : 0, c.fixed_k, c.k_min, c.k_max, k_slo, kcap};
    const double gr[8] = {c.ema_alpha, c.initial_accept, prof.pcie_bandwidth, prof.pcie_init_latency,
                          prof.pcie_overhead, static_cast<double>(prof.expert_size_bytes), prof.draft_base,
                          prof.draft_per_token};
    std::vector<double> vs;
    for (auto& [w, tv] : prof.verify_samples) {
      vs.push_back(w);
      vs.push_back(tv);
    }
    const int32_t offs[4] = {(int32_t)o_batch, (int32_t)o_jit, (int32_t)o_cov, (int32_t)o_step};
    CAPI_OK(mspq_cache_replay_all(cache, d_tgt, d_dr, d_g, d_acc, n, gi, gr, (int)prof.verify_samples.size(),
                                  vs.data(), d_slices, (int)o_end, offs, d_k, d_nc, d_flush, st));
    int32_t nc = 0;
    CUDA_OK(cudaMemcpyAsync(&nc, d_nc, 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (nc < 1 || nc > n) fail(MSPQ_ERR_INTERNAL, "replay_all: cycle count");
    k_dev.resize(nc);
    CUDA_OK(cudaHostAlloc((void**)&h_all, (size_t)nc * o_end * 4, 0));
    guard.h.push_back(h_all);
    CUDA_OK(cudaMemcpy(h_all, d_slices, (size_t)nc * o_end * 4, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(k_dev.data(), d_k, (size_t)nc * 4, cudaMemcpyDeviceToHost));
  }

  double now = 0.0, step_cov_total = 0.0, layer_cov_total = 0.0, stall = 0.0;
  uint64_t step_total = 0, layer_cov_count = 0, acc_total = 0, total_new = 0;
  int pos = 0, ci = 0, head_pos = -1;
  double channel_free = 0.0;
  json cycles = json::array();
  json logs = json::array();
  while (pos < n) {
    const int rem = n - pos;
    const int kk = c.use_governor ? select_k(prof, accept, c.k_min, c.k_max, k_slo, est()) : c.fixed_k;
    const int k_eff = std::min(kk, rem);
    const double t0 = now;
    json rec;
    rec["cycle"] = ci;
    rec["k"] = k_eff;
    json segs = json::array();
    const double draft_dur = t_draft(prof, k_eff), draft_end = t0 + draft_dur;
    segs.push_back(segment("compute", "draft", t0, draft_dur));
    if (all_mode) {
      if (ci >= (int)k_dev.size() || k_dev[ci] != k_eff)
        fail(MSPQ_ERR_INTERNAL, "replay_all: device governor chose a different k than the host");
      h_out = h_all + (size_t)ci * o_end;
    } else {
      CAPI_OK(mspq_cache_replay_cycle(cache, d_tgt, d_dr, d_g, pos, k_eff, head_pos, d_out + o_counts,
                                      d_out + o_batch, d_out + o_jit, d_out + o_cov, d_out + o_step, d_flush, st));
      CUDA_OK(cudaMemcpyAsync(h_out, d_out, o_end * 4, cudaMemcpyDeviceToHost, st));
      CUDA_OK(cudaStreamSynchronize(st));
    }
    const int32_t* cnt = h_out + o_counts;
    if (cnt[5]) fail(MSPQ_ERR_OVERFLOW, "device controller overflow");
    const int fetched = cnt[1], demand = cnt[2], nplan = cnt[3], nbatch = cnt[0];
    if (c.collect_plans && nplan > 0)
      CUDA_OK(cudaMemcpy(h_plan.data(), view.plan, (size_t)nplan * 12, cudaMemcpyDeviceToHost));
    if (c.log) {
      const int nl = std::min(cnt[4], view.log_cap);
      CUDA_OK(cudaMemcpy(h_log.data(), view.log, (size_t)nl * 24, cudaMemcpyDeviceToHost));
      json lj = json::array();
      for (int i = 0; i < nl; ++i) {
        const int32_t* ev = &h_log[(size_t)i * 6];
        lj.push_back({ev[0], ev[1], ev[2] / E, ev[2] % E, ev[3], ev[4] < 0 ? -1 : ev[4] / E, ev[4] < 0 ? -1 : ev[4] % E});
      }
      logs.push_back(lj);
    }
    // coverage at verify start
    json cov = json::array();
    for (int l = 0; l < L; ++l) {
      const double v = static_cast<double>(h_out[o_cov + l * 2]) / static_cast<double>(h_out[o_cov + l * 2 + 1]);
      cov.push_back(v);
      layer_cov_total += v;
      ++layer_cov_count;
    }
    const int nwin = (head_pos >= 0 ? 1 : 0) + k_eff;
    const int nslots = nwin * L;
    double step_cov_sum = 0.0;
    for (int s = 0; s < nslots; ++s)
      step_cov_sum += static_cast<double>(h_out[o_step + s * 2]) / static_cast<double>(h_out[o_step + s * 2 + 1]);
    // I/O lane (sim.cpp:302-347)
    auto draft_done_at = [&](int row) { return t0 + prof.draft_base + static_cast<double>(row + 1) * prof.draft_per_token; };
    struct B {
      double issue, start, end;
      int count;
      bool req;
    };
    std::vector<B> batches, jit;
    for (int b = 0; b < nbatch; ++b)
      batches.push_back({draft_done_at(h_out[o_batch + b * 3]), 0, 0, h_out[o_batch + b * 3 + 1], h_out[o_batch + b * 3 + 2] != 0});
    for (int r = 0; r < k_eff; ++r)
      if (h_out[o_jit + r * 2] > 0) jit.push_back({0, 0, 0, h_out[o_jit + r * 2], h_out[o_jit + r * 2 + 1] != 0});
    bool any_req = demand > 0;
    for (auto& b : batches) any_req = any_req || b.req;
    for (auto& b : jit) any_req = any_req || b.req;
    double p0 = draft_end, channel = std::max(t0, channel_free);
    if (any_req) {
      const double init_start = channel;
      channel = init_start + prof.pcie_init_latency;
      segs.push_back(segment("io", "io_init", init_start, prof.pcie_init_latency));
      p0 = std::max(draft_end, channel);
    }
    double required_drain = p0;
    const double S = static_cast<double>(prof.expert_size_bytes);
    for (auto& b : batches) {
      b.start = std::max(b.issue, channel);
      const double dur = prof.pcie_overhead + static_cast<double>(b.count) * S / prof.pcie_bandwidth;
      b.end = b.start + dur;
      channel = b.end;
      segs.push_back(segment("io", "io_new", b.start, dur));
      if (b.req) required_drain = std::max(required_drain, b.end);
    }
    for (auto& b : jit) {
      b.start = std::max(p0, channel);
      const double dur = prof.pcie_overhead + static_cast<double>(b.count) * S / prof.pcie_bandwidth;
      b.end = b.start + dur;
      channel = b.end;
      segs.push_back(segment("io", "io_new", b.start, dur));
      if (b.req) required_drain = std::max(required_drain, b.end);
    }
    const double sync_dur = t_pcie_new(prof, demand);
    double io_wait = std::max(0.0, required_drain - p0);
    if (demand > 0) io_wait = std::max(io_wait, channel - p0);
    if (sync_dur > 0.0) {
      segs.push_back(segment("io", "io_new", p0 + io_wait, sync_dur));
      channel = std::max(channel, p0 + io_wait + sync_dur);
    }
    channel_free = channel;
    const double verify_start = p0 + io_wait + sync_dur;
    const double verify_dur = t_verify(prof, static_cast<double>(k_eff + 1));
    segs.push_back(segment("compute", "verify", verify_start, verify_dur));
    double cycle_end = verify_start + verify_dur;
    int accepted = 0;
    while (accepted < k_eff && t.acc[pos + accepted]) ++accepted;
    if (accepted < k_eff && c.rollback > 0.0) {
      segs.push_back(segment("compute", "rollback", cycle_end, c.rollback));
      cycle_end += c.rollback;
    }
    const int consumed = std::min(accepted + 1, rem);
    const int bonus = consumed - std::min(accepted, consumed);
    rec["accepted"] = consumed - bonus;
    rec["bonus"] = bonus;
    rec["start_s"] = t0;
    rec["span_s"] = cycle_end - t0;
    rec["coverage"] = cov;
    rec["step_coverage"] = nslots > 0 ? step_cov_sum / nslots : 0.0;
    rec["steps"] = nslots;
    rec["new_experts"] = fetched;
    rec["bytes"] = static_cast<uint64_t>(fetched) * prof.expert_size_bytes;
    rec["io_wait_s"] = io_wait;
    rec["sync_fetch_s"] = sync_dur;
    rec["sync_count"] = demand;
    rec["segments"] = segs;
    if (c.collect_plans) {
      json pp = json::array();
      for (int i = 0; i < nplan; ++i) {
        json it;
        it["issue_after_token"] = h_plan[i * 3];
        it["layer"] = h_plan[i * 3 + 1] / E;
        it["expert"] = h_plan[i * 3 + 1] % E;
        it["phase"] = h_plan[i * 3 + 2];
        pp.push_back(it);
      }
      rec["prefetch_plan"] = pp;
      // reorder_verification (scheduler.cpp:339-357) on the verified window
      json ep = json::array();
      for (int l = 0; l < L; ++l) {
        std::map<int, std::vector<int>> groups;
        for (int w = 0; w < nwin; ++w) {
          const int vpos = head_pos >= 0 ? (w == 0 ? head_pos : pos + w - 1) : pos + w;
          for (int j = 0; j < K; ++j) groups[t.target[((size_t)vpos * L + l) * K + j]].push_back(vpos);
        }
        json lj;
        lj["layer"] = l;
        lj["groups"] = json::array();
        for (auto& [e, toks] : groups) {
          json gj;
          gj["expert"] = e;
          gj["tokens"] = toks;
          lj["groups"].push_back(gj);
        }
        ep.push_back(lj);
      }
      rec["execution_plan"] = ep;
    }
    head_pos = bonus > 0 ? pos + accepted : -1;
    std::vector<bool> outcomes;
    for (int i = 0; i < k_eff; ++i) {
      const bool ok = t.acc[pos + i];
      outcomes.push_back(ok);
      if (!ok) break;
    }
    if (outcomes.size() > accept.size()) outcomes.resize(accept.size());
    accept = update_acceptance(accept, c.ema_alpha, outcomes);
    g = static_cast<double>(fetched) / static_cast<double>(k_eff);
    stall += verify_start - draft_end;
    step_cov_total += step_cov_sum;
    step_total += nslots;
    acc_total += (uint64_t)(consumed - bonus);
    total_new += fetched;
    cycles.push_back(rec);
    now = cycle_end;
    pos += consumed;
    ++ci;
  }
  rep["total_tokens"] = pos;
  rep["total_time_s"] = now;
  rep["tpot_s"] = pos > 0 ? now / static_cast<double>(pos) : 0.0;
  rep["ttft_s"] = cycles.empty() ? 0.0 : cycles[0]["span_s"].get<double>();
  rep["mean_coverage"] = layer_cov_count > 0 ? layer_cov_total / static_cast<double>(layer_cov_count) : 0.0;
  rep["mean_step_coverage"] = step_total > 0 ? step_cov_total / static_cast<double>(step_total) : 0.0;
  rep["mean_accepted"] = cycles.empty() ? 0.0 : static_cast<double>(acc_total) / static_cast<double>(cycles.size());
  rep["stall_time_s"] = stall;
  rep["total_new_experts"] = total_new;
  rep["cycles"] = cycles;
  if (c.log) rep["log"] = logs;
  return rep.dump();
}

}  // namespace mspq_host

// ============================================================================ C-ABI (engine part)
namespace {
template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const mspq_host::Err& e) {
    return mspq::set_error(e.code, e.msg);
  } catch (const nlohmann::json::exception& e) {
    return mspq::set_error(MSPQ_ERR_INVALID_CONFIG, e.what());
  } catch (const std::exception& e) {
    return mspq::set_error(MSPQ_ERR_INTERNAL, e.what());
  }
}
char* dup(const std::string& s) {
  char* p = (char*)malloc(s.size() + 1);
  memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
}  // namespace

extern "C" int mspq_replay(int device, const char* trace_jsonl, const char* config_json, char** report_json) {
  return guarded([&] {
    *report_json = dup(mspq_host::replay(device, trace_jsonl, config_json));
    return MSPQ_OK;
  });
}

namespace mspq_host {
// Independent replays of one trace run CONCURRENTLY: each config gets its own host thread, device
// cache controller and stream, so the device executes the configs' launches side by side (the
// reference's compare_policies / sweep_k loop over run_simulation serially, sim.cpp:539-574).
// Rows come back in config order; the first failing config's error is rethrown.
std::vector<json> replay_many(int device, const char* trace_jsonl, const std::vector<json>& cfgs) {
  const size_t n = cfgs.size();
  std::vector<std::string> out(n);
  std::vector<std::exception_ptr> err(n);
  const size_t width = std::max<size_t>(1, std::min<size_t>(n, 32));
  for (size_t b = 0; b < n; b += width) {
    std::vector<std::thread> th;
    for (size_t i = b; i < std::min(n, b + width); ++i)
      th.emplace_back([&, i] {
        try {
          out[i] = replay(device, trace_jsonl, cfgs[i].dump());
        } catch (...) {
          err[i] = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
  }
  std::vector<json> reps;
  for (size_t i = 0; i < n; ++i) {
    if (err[i]) std::rethrow_exception(err[i]);
    reps.push_back(json::parse(out[i]));
  }
  return reps;
}
}  // namespace mspq_host

// compare_policies / sweep_k (sim.cpp:539-574) on the device control plane: run_simulation of
// the trace once per (policy, capacity) / per fixed k, rows as in PolicyRow / SweepRow
// (sim.hpp:88-109), the configs replayed concurrently (replay_many).  policies_json: ["lru", ...];
// capacities_json / ks_json: integer arrays.
extern "C" int mspq_compare_policies(int device, const char* trace_jsonl, const char* config_json,
                                     const char* policies_json, const char* capacities_json, char** rows_json) {
  using namespace mspq_host;
  return guarded([&] {
    json base = json::parse(config_json, nullptr, false);
    json pols = json::parse(policies_json, nullptr, false), caps = json::parse(capacities_json, nullptr, false);
    if (base.is_discarded() || !pols.is_array() || !caps.is_array())
      fail(MSPQ_ERR_INVALID_CONFIG, "compare_policies: config object, policy and capacity arrays");
    json rows = json::array();
    std::vector<json> cfgs;
    for (const auto& pol : pols)
      for (const auto& cap : caps) {
        json cfg = base;
        cfg["policy"] = pol;
        cfg["cache_capacity"] = cap;
        cfgs.push_back(cfg);
      }
    const std::vector<json> reps = replay_many(device, trace_jsonl, cfgs);
    for (size_t i = 0; i < cfgs.size(); ++i)
      rows.push_back({{"policy", cfgs[i]["policy"]}, {"capacity", cfgs[i]["cache_capacity"]},
                      {"coverage", reps[i]["mean_step_coverage"]}, {"tpot", reps[i]["tpot_s"]}});
    *rows_json = dup(rows.dump());
    return MSPQ_OK;
  });
}

extern "C" int mspq_sweep_k(int device, const char* trace_jsonl, const char* config_json, const char* ks_json,
                            char** rows_json) {
  using namespace mspq_host;
  return guarded([&] {
    json base = json::parse(config_json, nullptr, false);
    json ks = json::parse(ks_json, nullptr, false);
    if (base.is_discarded() || !ks.is_array()) fail(MSPQ_ERR_INVALID_CONFIG, "sweep_k: config object, k array");
    json rows = json::array();
    std::vector<json> cfgs;
    for (const auto& k : ks) {
      json cfg = base;
      cfg["k"] = k;  // fixed k: the governor is off (SimConfig use_governor = false)
      cfgs.push_back(cfg);
    }
    const std::vector<json> reps = replay_many(device, trace_jsonl, cfgs);
    for (size_t i = 0; i < cfgs.size(); ++i)
      rows.push_back({{"k", cfgs[i]["k"]}, {"tpot", reps[i]["tpot_s"]}, {"mean_accepted", reps[i]["mean_accepted"]},
                      {"coverage", reps[i]["mean_step_coverage"]}, {"ttft", reps[i]["ttft_s"]}});
    *rows_json = dup(rows.dump());
    return MSPQ_OK;
  });
}

// Governor evaluation for parity tests: same request/response schema as oracle/ref_shim.cpp's
// ref_governor (select_k, k_slo_from_ttft, t_cycle/k_accept/t_verify tables, EMA update).
extern "C" int mspq_governor(const char* request_json, char** out_json) {
  using namespace mspq_host;
  return guarded([&] {
    json r = json::parse(request_json);
    Profile prof = r.contains("profile") ? Profile::from_json(r["profile"]) : Profile{};
    std::vector<double> p = r["p"].get<std::vector<double>>();
    const double alpha = r.value("alpha", 0.1);
    const int k_min = r.value("k_min", 1), k_max = r.value("k_max", 16), k_slo = r.value("k_slo", 16);
    const double g = r.value("g", 0.0);
    Est est = [g](int k) { return static_cast<int>(std::llround(g * static_cast<double>(k))); };
    json out;
    out["select_k"] = select_k(prof, p, k_min, k_max, k_slo, est);
    const double budget = r.value("ttft_budget", 0.0);
    if (budget > 0.0) {
      try {
        out["k_slo_ttft"] = k_slo_from_ttft(prof, budget, est, k_min, k_max);
      } catch (const Err& e) {
        out["k_slo_ttft"] = std::string("error:") + std::to_string(e.code - 1);
      }
    }
    json tc = json::array(), ka = json::array(), tv = json::array();
    for (int k = 0; k <= k_max && k <= (int)p.size(); ++k) {
      tc.push_back(t_cycle(prof, k, est(k)));
      ka.push_back(k_accept(p, k));
      tv.push_back(t_verify(prof, static_cast<double>(k + 1)));
    }
    out["t_cycle"] = tc;
    out["k_accept"] = ka;
    out["t_verify"] = tv;
    if (r.contains("outcomes")) {
      std::vector<bool> o;
      for (const auto& b : r["outcomes"]) o.push_back(b.get<bool>());
      out["updated_p"] = update_acceptance(p, alpha, o);
    }
    *out_json = dup(out.dump());
    return MSPQ_OK;
  });
}

// ---- live engine entry points (implemented in live.cpp)
