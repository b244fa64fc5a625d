// the B200 run_simulation for the reference's C++ API (proj/include/moespeq).
#pragma once
#include "json.hpp"
#include "moespeq/sim.hpp"
#include "moespeq/trace.hpp"

namespace moespeq {
// Same inputs and SimReport as run_simulation (sim.hpp:86); the run-config JSON is the
// reference schema (run_config.hpp:30-50).  Throws moespeq::Error on a non-zero status.
SimReport run_simulation_b200(const Trace& trace, const nlohmann::json& run_config, int device = 0);
}  // namespace moespeq
