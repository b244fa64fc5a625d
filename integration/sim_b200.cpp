// Reference-side binding a maintainer adds to proj/ (INTEGRATION.md §2): run_simulation with every
// cache decision on the B200, same signature shape and the same SimReport.  Compiled here against
// the reference headers (oracle/Makefile -> oracle/_ref/sim_b200_check) so the snippet is real code.
#include "sim_b200.hpp"

#include <cstdlib>
#include <string>

#include "mspq_capi.h"
#include "moespeq/errors.hpp"

namespace moespeq {

namespace {
CycleRecord cycle_from_json(const nlohmann::ordered_json& c) {
  CycleRecord r;
  r.cycle_index = c["cycle"];
  r.k_used = c["k"];
  r.accepted_count = c["accepted"];
  r.bonus_token = c["bonus"];
  r.start_time = c["start_s"];
  r.span = c["span_s"];
  r.per_layer_coverage = c["coverage"].get<std::vector<double>>();
  r.step_coverage_mean = c["step_coverage"];
  r.step_count = c["steps"];
  r.new_experts_fetched = c["new_experts"];
  r.bytes_transferred = c["bytes"];
  r.io_wait = c["io_wait_s"];
  r.sync_fetch_time = c["sync_fetch_s"];
  r.sync_fetch_count = c["sync_count"];
  for (const auto& s : c["segments"])
    r.segments.push_back({s["label"].get<std::string>(), s["start_s"].get<double>(), s["duration_s"].get<double>(),
                          s["lane"].get<std::string>() == "io" ? 1 : 0});
  if (c.contains("prefetch_plan")) r.prefetch_plan = c["prefetch_plan"];
  if (c.contains("execution_plan")) r.execution_plan = c["execution_plan"];
  return r;
}
}  // namespace

SimReport run_simulation_b200(const Trace& trace, const nlohmann::json& run_config, int device) {
  char* out = nullptr;
  const std::string t = write_trace(trace), c = run_config.dump();
  if (const int s = mspq_replay(device, t.c_str(), c.c_str(), &out); s != 0)
    throw Error(s >= 1 && s <= 18 ? static_cast<ErrorCode>(s - 1) : ErrorCode::InvalidConfig, mspq_last_error());
  const nlohmann::ordered_json j = nlohmann::ordered_json::parse(out);  // keeps the plans' key order
  mspq_free(out);
  SimReport r;
  r.total_tokens = j["total_tokens"];
  r.total_time = j["total_time_s"];
  r.tpot = j["tpot_s"];
  r.ttft = j["ttft_s"];
  r.mean_coverage = j["mean_coverage"];
  r.mean_step_coverage = j["mean_step_coverage"];
  r.mean_accepted = j["mean_accepted"];
  r.stall_time = j["stall_time_s"];
  r.total_new_experts = j["total_new_experts"];
  for (const auto& cy : j["cycles"]) r.cycles.push_back(cycle_from_json(cy));
  return r;
}

}  // namespace moespeq
