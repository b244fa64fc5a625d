// Host-side types shared by engine.cpp (replay, governor) and live.cpp (generate).
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "json.hpp"

namespace mspq_host {
using json = nlohmann::ordered_json;

struct Err {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);

struct Profile {  // HardwareProfile, perfmodel.hpp:15-30
  double pcie_bandwidth = 16e9, pcie_init_latency = 20e-3, pcie_overhead = 2e-3;
  uint64_t expert_size_bytes = 25'000'000;
  double draft_base = 5e-3, draft_per_token = 3e-3;
  std::vector<std::pair<double, double>> verify_samples = {{1.0, 10e-3}, {5.0, 20e-3}, {9.0, 40e-3}, {17.0, 75e-3}};
  double token_bytes = 1.0;
  void validate() const;
  void check_samples() const;
  static Profile from_json(const json& j);
  json to_json() const;
};

using Est = std::function<int(int)>;
double k_accept(const std::vector<double>& p, int k);
double t_draft(const Profile& p, int k);
double t_pcie_new(const Profile& p, int n);
double t_verify(const Profile& p, double window);
double t_cycle(const Profile& p, int k, int n);
int select_k(const Profile& p, const std::vector<double>& acc, int k_min, int k_max, int k_slo, const Est& est);
int k_slo_from_ttft(const Profile& p, double budget, const Est& est, int k_min, int k_max);
std::vector<double> update_acceptance(const std::vector<double>& p, double a, const std::vector<bool>& o);

struct HostCfg {  // SimConfig (sim.hpp:15-34) from the run-config schema (run_config.cpp:94-174)
  int policy = 4;  // speculative
  int mode = 0;    // per-layer
  long cache_capacity = 8;
  bool entropy_weighted = false;
  int fixed_k = 4;
  bool use_governor = false;
  int k_min = 1, k_max = 16, k_slo = 16;
  double ttft_budget = 0.0;
  Profile profile;
  bool profile_given = false;
  double f1 = 0.25, f2 = 0.75;
  int budget = 2;
  double rollback = 0.0, ema_alpha = 0.1, initial_accept = 0.8;
  bool collect_plans = false;
  bool log = false;  // extension: emit the per-event hit/miss log
  // extension (live engine): run a verify layer's GEMM for the resident experts while the missing
  // ones are still on the link (two smaller K3 launches; +4% at cap 14/16, neutral at 4/16)
  bool verify_overlap = false;
  // extension (live engine): the governor's |E_new(k)| estimator. 0 = the reference's linear g*k
  // (sim.cpp:75-78, 404; the parity default); 1 = "elb": per layer, the expected union of the
  // draft-predicted routing over a (k+1)-token window minus the experts resident now
  int estimator = 0;
  // extension (live engine): issue a layer's plan prefetches behind the previous layer's demand
  // copies (per-layer capacity mode) instead of in plan order at draft time
  bool prefetch_defer = true;
  // a fetch of an expert whose first-request buffer of the same verify layer still holds it (evicted
  // and requested again inside one layer) is served HBM -> HBM from that buffer instead of the link
  bool refetch_from_hbm = true;
};
int parse_policy(const std::string& s);
const char* policy_name(int p);
HostCfg parse_host_cfg(const std::string& text);
void validate_host_cfg(const HostCfg& c, int top_k);
json segment(const char* lane, const char* label, double start, double dur);
}  // namespace mspq_host
