// latency_main.cpp — per-call latency of the drop-in, measured the way the reference's own
// acceptance criterion 8 measures it (tests/acceptance.cpp:559-592): bitmm::bench_routine
// (/root/reference/proj/src/bench.cpp:91-170, unmodified; median of `reps` calls, each
// returning a fresh DenseMatrix) for 1/1, 1/2 and 2/2 at one shape. Linked against the
// drop-in (latency_b200) and against the reference's CPU library (latency_ref) by
// oracle/Makefile.
//
//   latency_* [m k n] [reps]      (default 1024 1024 1024, 9 reps, 2 warm-up)
#include <cstdlib>
#include <iostream>

#include "bitmm/bench.hpp"
#include "bitmm/kernels.hpp"

int main(int argc, char** argv) {
  bitmm::GemmProblem p{1024, 1024, 1024};
  if (argc >= 4) p = bitmm::GemmProblem{std::atoll(argv[1]), std::atoll(argv[2]), std::atoll(argv[3])};
  bitmm::BenchOptions opt;
  opt.reps = argc >= 5 ? std::atoi(argv[4]) : 9;
  opt.warmup = 2;
  opt.seed = 1;
  const bitmm::Routine rs[] = {bitmm::Routine::k1x1, bitmm::Routine::k1x2, bitmm::Routine::k2x2};
  const char* names[] = {"1x1", "1x2", "2x2"};
  for (int i = 0; i < 3; ++i) {
    const bitmm::BenchRecord r = bitmm::bench_routine(rs[i], p, opt);
    std::cout << names[i] << " m=" << p.m << " k=" << p.k << " n=" << p.n << " median_ms=" << r.seconds * 1e3
              << "\n";
  }
  return 0;
}
