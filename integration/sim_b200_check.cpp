// TEST DRIVER (tests/test_integration_gpu.py): runs the reference run_simulation and the B200
// binding on the same trace file and run-config, prints "identical" when the two SimReport
// to_json() dumps are byte-equal, else the first differing line.  Usage: sim_b200_check trace.jsonl config.json
#include <fstream>
#include <iostream>
#include <sstream>

#include "moespeq/run_config.hpp"
#include "sim_b200.hpp"

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  std::ifstream tin(argv[1]), cin(argv[2]);
  const moespeq::Trace trace = moespeq::parse_trace(tin);
  const nlohmann::json cfg = nlohmann::json::parse(cin);
  const moespeq::RunConfig rc = moespeq::parse_run_config(cfg);
  const std::string want = moespeq::run_simulation(trace, rc.sim).to_json().dump(1);
  const std::string got = moespeq::run_simulation_b200(trace, cfg).to_json().dump(1);
  if (want == got) {
    std::cout << "identical " << want.size() << " bytes\n";
    return 0;
  }
  std::istringstream a(want), b(got);
  std::string la, lb;
  int n = 0;
  while (std::getline(a, la) && std::getline(b, lb)) {
    ++n;
    if (la != lb) {
      std::cout << "line " << n << ": reference " << la << " | b200 " << lb << "\n";
      break;
    }
  }
  return 1;
}
