// egsolve_gpu.cpp — `egsolve solve` (proj/tools/egsolve.cpp:86-108) with the
// GPU variant: the reference loader (parse_arena, io.hpp:19) reads the arena
// file, solve_gpu solves it on the B200, and the reference output format
// (write_solution(make_solution(...)), io.hpp:35-37) goes to stdout.
//
//   egsolve_gpu <arena.eg> [--dense|--sparse] [--no-certify] [--timeout S]
// Exit codes as egsolve: 0 ok, 1 input/config error, 2 timeout.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "egsolve/errors.hpp"
#include "egsolve/io.hpp"
#include "solver_gpu.hpp"

using namespace egsolve;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <arena.eg> [--dense|--sparse] [--no-certify] [--timeout S]\n",
                 argv[0]);
    return 1;
  }
  GpuOptions g;
  SolverOptions o;
  for (int i = 2; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--dense")) g.mode = EGS_MODE_DENSE;
    else if (!std::strcmp(argv[i], "--sparse")) g.mode = EGS_MODE_SPARSE;
    else if (!std::strcmp(argv[i], "--no-certify")) g.certify = false;
    else if (!std::strcmp(argv[i], "--timeout") && i + 1 < argc) o.timeout_seconds = std::atof(argv[++i]);
  }
  try {
    std::ifstream in(argv[1], std::ios::binary);
    if (!in) throw Error(std::string("cannot open ") + argv[1]);
    std::stringstream ss;
    ss << in.rdbuf();
    const GameArena arena = parse_arena(ss.str());
    egs_gpu_stats st{};
    const SolveReport report = solve_gpu(arena, o, g, &st);
    const std::string text = write_solution(make_solution(arena, report));
    std::fwrite(text.data(), 1, text.size(), stdout);
    std::cerr << "gpu solved '" << argv[1] << "': lifts=" << report.lifts
              << " rounds=" << report.rounds << " certified=" << st.certified
              << " device=" << st.solve_seconds << "s time=" << report.wall_seconds << "s\n";
    return 0;
  } catch (const TimeoutError& e) {
    std::cerr << argv[1] << ": timed out (" << e.what() << ")\n";
    return 2;
  } catch (const Error& e) {
    std::cerr << argv[1] << ": " << e.what() << "\n";
    return 1;
  }
}
