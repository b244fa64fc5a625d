// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// C-ABI shim compiled together with the reference's own control-plane sources
// (/root/reference/proj/src/{trace,perfmodel,scheduler,sim,run_config}.cpp, built by
// oracle/Makefile into oracle/_ref/libmoespeq_ref.so).  It lets the Python tests call the
// UNMODIFIED reference implementation:
//   ref_generate_trace  -> generate_synthetic_trace   (trace.cpp:319-399)
//   ref_run_simulation  -> parse_trace + parse_run_config + run_simulation (sim.cpp:458-466)
//   ref_plan_prefetch   -> build_elb + plan_prefetch   (scheduler.cpp:41-63, 173-254)
//   ref_governor        -> select_k / k_slo_from_ttft / t_cycle / k_accept (perfmodel.cpp:85-204)
// Every function returns a malloc'd JSON string (free with ref_free) or nullptr with the
// error text retrievable through ref_last_error().
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "json.hpp"
#include "moespeq/perfmodel.hpp"
#include "moespeq/run_config.hpp"
#include "moespeq/scheduler.hpp"
#include "moespeq/sim.hpp"
#include "moespeq/trace.hpp"

using namespace moespeq;
using nlohmann::json;

namespace {
thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class F>
char* guarded(F&& f) {
  try {
    return dup(f());
  } catch (const Error& e) {
    g_err = std::string("moespeq::Error code=") + std::to_string(static_cast<int>(e.code())) +
            " " + e.what();
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

char* ref_generate_trace(int L, int N, int top_k, int shared, unsigned long long expert_bytes,
                         int tokens, double hard, double soft, double mismatch, double accept,
                         double skew, unsigned long long seed) {
  return guarded([&] {
    ModelShape shape{L, N, top_k, shared, expert_bytes};
    return write_trace(
        generate_synthetic_trace(shape, tokens, hard, soft, mismatch, accept, skew, seed));
  });
}

// config_json uses the reference run-config schema (run_config.hpp:30-50).
char* ref_run_simulation(const char* trace_jsonl, const char* config_json) {
  return guarded([&] {
    std::istringstream in(trace_jsonl);
    Trace trace = parse_trace(in);
    RunConfig cfg = parse_run_config(json::parse(config_json));
    return run_simulation(trace, cfg.sim).to_json().dump();
  });
}

char* ref_run_simulation_ex(const char* trace_jsonl, const char* config_json, int want_cycles_csv) {
  return guarded([&] {
    std::istringstream in(trace_jsonl);
    Trace trace = parse_trace(in);
    RunConfig cfg = parse_run_config(json::parse(config_json));
    SimReport r = run_simulation(trace, cfg.sim);
    json out;
    out["report"] = json::parse(r.to_json().dump());
    if (want_cycles_csv) {
      out["cycles_csv"] = r.cycles_csv();
      out["timeline_csv"] = r.timeline_csv();
    }
    return out.dump();
  });
}

// Plans over the first `k` trace tokens against a cache pre-populated with `resident`
// ([[layer,expert],...]).
char* ref_plan_prefetch(const char* trace_jsonl, int k, const char* resident_json, int budget,
                        double f1, double f2, int capacity) {
  return guarded([&] {
    std::istringstream in(trace_jsonl);
    Trace trace = parse_trace(in);
    auto elb = build_elb(std::span<const TokenRecord>(trace.tokens.data(), k),
                         trace.shape.num_moe_layers);
    CacheState cache(CapacityMode::PerLayer, static_cast<std::size_t>(capacity));
    for (const auto& kv : json::parse(resident_json)) cache.insert({kv[0].get<int>(), kv[1].get<int>()});
    return plan_prefetch(elb, cache, budget, f1, f2).to_json().dump();
  });
}

// Victim under the lookahead rule for a cache holding `resident`.
char* ref_select_victim(const char* trace_jsonl, int k, const char* resident_json, int now,
                        int layer_filter) {
  return guarded([&] {
    std::istringstream in(trace_jsonl);
    Trace trace = parse_trace(in);
    auto elb = build_elb(std::span<const TokenRecord>(trace.tokens.data(), k),
                         trace.shape.num_moe_layers);
    CacheState cache(CapacityMode::Global, 1u << 20);
    for (const auto& kv : json::parse(resident_json)) cache.insert({kv[0].get<int>(), kv[1].get<int>()});
    ExpertKey v = select_victim_lookahead(cache, elb, now, layer_filter);
    return json::array({v.layer, v.expert}).dump();
  });
}

// Governor: request {"profile":{...},"p":[...],"alpha":a,"k_min":..,"k_max":..,"k_slo":..,
// "g":g,"ttft_budget":b,"outcomes":[bool...]} -> {"select_k":..,"k_slo_ttft":..|null,
// "t_cycle":[...k=0..k_max],"k_accept":[...],"updated_p":[...]}
char* ref_governor(const char* request_json) {
  return guarded([&] {
    json r = json::parse(request_json);
    HardwareProfile prof = r.contains("profile") ? HardwareProfile::from_json(r["profile"])
                                                 : HardwareProfile{};
    AcceptanceModel m;
    m.p = r["p"].get<std::vector<double>>();
    m.ema_alpha = r.value("alpha", 0.1);
    GovernorConfig gov;
    gov.k_min = r.value("k_min", 1);
    gov.k_max = r.value("k_max", 16);
    gov.k_slo = r.value("k_slo", 16);
    const double g = r.value("g", 0.0);
    // "est": optional table est[k] (any |E_new(k)| estimator, e.g. the live engine's elb one)
    // fed to the reference's select_k in place of the linear g*k
    const std::vector<int> table = r.contains("est") ? r["est"].get<std::vector<int>>() : std::vector<int>{};
    NewExpertEstimator est = [g, table](int k) {
      if (!table.empty()) return table.at(static_cast<size_t>(k));
      return static_cast<int>(std::llround(g * static_cast<double>(k)));
    };
    json out;
    out["select_k"] = select_k(prof, m, gov, est);
    const double budget = r.value("ttft_budget", 0.0);
    if (budget > 0.0) {
      try {
        out["k_slo_ttft"] = k_slo_from_ttft(prof, budget, est, gov.k_min, gov.k_max);
      } catch (const Error& e) {
        out["k_slo_ttft"] = std::string("error:") + std::to_string(static_cast<int>(e.code()));
      }
    }
    json tc = json::array(), ka = json::array(), tv = json::array();
    for (int k = 0; k <= gov.k_max && k <= static_cast<int>(m.p.size()); ++k) {
      tc.push_back(t_cycle(prof, k, est(k)));
      ka.push_back(k_accept(m, k));
      tv.push_back(t_verify(prof, static_cast<double>(k + 1)));
    }
    out["t_cycle"] = tc;
    out["k_accept"] = ka;
    out["t_verify"] = tv;
    if (r.contains("outcomes")) {
      std::vector<bool> o;
      for (const auto& b : r["outcomes"]) o.push_back(b.get<bool>());
      out["updated_p"] = update_acceptance(m, o).p;
    }
    return out.dump();
  });
}

// compare_policies / sweep_k (sim.cpp:539-574) with the rows as JSON
char* ref_compare_policies(const char* trace_jsonl, const char* config_json, const char* policies_json,
                           const char* capacities_json) {
  return guarded([&] {
    std::istringstream in(trace_jsonl);
    const Trace trace = parse_trace(in);
    const RunConfig cfg = parse_run_config(json::parse(config_json));
    std::vector<Policy> pols;
    for (const auto& p : json::parse(policies_json)) pols.push_back(parse_policy(p.get<std::string>()));
    const std::vector<std::size_t> caps = json::parse(capacities_json).get<std::vector<std::size_t>>();
    json rows = json::array();
    for (const auto& r : compare_policies(trace, cfg.sim, pols, caps))
      rows.push_back({{"policy", to_string(r.policy)}, {"capacity", r.capacity}, {"coverage", r.coverage},
                      {"tpot", r.tpot}});
    return rows.dump();
  });
}

char* ref_sweep_k(const char* trace_jsonl, const char* config_json, const char* ks_json) {
  return guarded([&] {
    std::istringstream in(trace_jsonl);
    const Trace trace = parse_trace(in);
    const RunConfig cfg = parse_run_config(json::parse(config_json));
    const std::vector<int> ks = json::parse(ks_json).get<std::vector<int>>();
    json rows = json::array();
    for (const auto& r : sweep_k(trace, cfg.sim, ks))
      rows.push_back({{"k", r.k}, {"tpot", r.tpot}, {"mean_accepted", r.mean_accepted}, {"coverage", r.coverage},
                      {"ttft", r.first_cycle_latency}});
    return rows.dump();
  });
}

// classify_fidelity (both granularities) + layer_entropy of every layer (trace.cpp:401-462)
char* ref_trace_analysis(const char* trace_jsonl) {
  return guarded([&] {
    std::istringstream in(trace_jsonl);
    const Trace tr = parse_trace(in);
    json out;
    for (auto [name, gran] : {std::pair<const char*, FidelityGranularity>{"token_layer", FidelityGranularity::TokenLayer},
                              {"token", FidelityGranularity::Token}}) {
      const FidelityStats f = classify_fidelity(tr, gran);
      out["fidelity"][name] = {{"hard_rate", f.hard_rate}, {"soft_rate", f.soft_rate},
                               {"mismatch_rate", f.mismatch_rate}, {"hard_count", f.hard_count},
                               {"soft_count", f.soft_count}, {"mismatch_count", f.mismatch_count},
                               {"total", f.total}};
    }
    json ent = json::array();
    for (int l = 0; l < tr.shape.num_moe_layers; ++l) ent.push_back(layer_entropy(tr, l));
    out["layer_entropy"] = ent;
    return out.dump();
  });
}

}  // extern "C"
