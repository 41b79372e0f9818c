// verify_main.cpp — runs the reference's own verification sweep (bitmm::run_verification,
// /root/reference/proj/src/verify.cpp:352-376, unmodified) and prints its report the way the
// reference CLI's `verify` command does (tools/bitmm_main.cpp: exit 0 when every suite passes,
// 1 otherwise). Linked by oracle/Makefile three ways: against the reference's CPU library
// (verify_ref), against the drop-in with the GEMMs and packers on the B200 (verify_b200), and
// with the row ops on the B200 as well (verify_b200_rowops).
//
//   verify_* [--seed S] [--gemm-cases N] [--max-dim D] [--dot-n N] [--mbm-n N]
//            [--rowop-cases N] [--inject-fault]
#include <cstdlib>
#include <cstring>
#include <iostream>

#include "bitmm/verify.hpp"

int main(int argc, char** argv) {
  bitmm::VerifyOptions opt;
  for (int i = 1; i < argc; ++i) {
    const char* a = argv[i];
    auto next = [&]() -> long long {
      if (i + 1 >= argc) {
        std::cerr << "missing value for " << a << "\n";
        std::exit(2);
      }
      return std::atoll(argv[++i]);
    };
    if (!std::strcmp(a, "--inject-fault")) opt.inject_fault = true;
    else if (!std::strcmp(a, "--seed")) opt.seed = static_cast<std::uint64_t>(next());
    else if (!std::strcmp(a, "--gemm-cases")) opt.gemm_cases = static_cast<int>(next());
    else if (!std::strcmp(a, "--max-dim")) opt.gemm_max_dim = static_cast<int>(next());
    else if (!std::strcmp(a, "--dot-n")) opt.dot_exhaustive_n = static_cast<int>(next());
    else if (!std::strcmp(a, "--mbm-n")) opt.mbm_exhaustive_n = opt.mbm_class_n = static_cast<int>(next());
    else if (!std::strcmp(a, "--rowop-cases")) opt.random_rowop_cases = static_cast<int>(next());
    else {
      std::cerr << "unknown option " << a << "\n";
      return 2;
    }
  }
  const bitmm::VerifyReport report = bitmm::run_verification(opt);
  bitmm::print_report(std::cout, report);
  return report.passed ? 0 : 1;
}
