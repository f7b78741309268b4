// esdg_run_main.cpp -- minimal driver around the reference's own run_case /
// run_ladder (core/src/runner.cpp, core/src/config.cpp): the reference's CLI
// (tools/esdg_main.cpp) needs the un-vendored CLI11 header, so the tests use
// this one instead. Built twice by oracle/Makefile from the SAME reference
// sources: against the reference's esdg/solver.hpp (esdg_run_cpu) and against
// the type-swap header include/esdg_b200/swap/esdg/solver.hpp (esdg_run_gpu).
//
//   esdg_run_{cpu,gpu} run|ladder <config file> [key value ...]
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "esdg/config.hpp"
#include "esdg/error.hpp"
#include "esdg/runner.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s run|ladder <config file> [key value ...]\n", argv[0]);
    return esdg::kExitConfigError;
  }
  try {
    esdg::RunConfig cfg = esdg::parse_config_file(argv[2]);
    std::vector<std::pair<std::string, std::string>> overrides;
    for (int i = 3; i + 1 < argc; i += 2) overrides.emplace_back(argv[i], argv[i + 1]);
    esdg::apply_overrides(cfg, overrides);
    return std::string(argv[1]) == "ladder" ? esdg::run_ladder(cfg) : esdg::run_case(cfg);
  } catch (const esdg::ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return esdg::kExitConfigError;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
