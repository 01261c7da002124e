// dppix::run_sweep (cli.hpp) on one PGM, CSV to stdout. Compiled twice from
// this one file: against include/dppix + libdppix_gpu.so (sweep_gpu) and
// against the reference's headers and sources (_ref_gate/sweep_ref), so the
// two CSVs can be compared column by column (runtime_ms aside).
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "dppix/cli.hpp"

template <class T>
static std::vector<T> list(const char* s) {
  std::vector<T> v;
  std::stringstream in(s);
  std::string tok;
  while (std::getline(in, tok, ','))
    if (!tok.empty()) {
      std::stringstream t(tok);
      T x{};
      t >> x;
      v.push_back(x);
    }
  return v;
}

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: %s image.pgm eps,.. m,.. b,.. seed,.. recon(0|1) u|a\n", argv[0]);
    return 2;
  }
  dppix::RunConfig cfg;
  cfg.input = argv[1];
  cfg.epsilon_list = list<double>(argv[2]);
  cfg.m_list = list<int>(argv[3]);
  cfg.b_list = list<int>(argv[4]);
  cfg.n_list = {1};
  cfg.seed_list = list<std::uint64_t>(argv[5]);
  cfg.reconstruct_check = std::atoi(argv[6]) != 0;
  cfg.mode = argv[7][0] == 'a' ? dppix::RunMode::adaptive : dppix::RunMode::uniform;
  try {
    const dppix::SweepResult r = dppix::run_sweep(cfg);
    std::fputs(r.csv.c_str(), stdout);
    return r.failures ? 1 : 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
