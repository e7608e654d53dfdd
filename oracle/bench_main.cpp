// TEST/BENCH INFRASTRUCTURE ONLY.
//
// `rvk bench` without CLI11 (absent from the image): the argument handling of
// run_bench_cmd (/root/reference/proj/tools/rvk_main.cpp:160-221, restated)
// around the reference's own harness rvk::run_bench / format_bench_table /
// write_bench_csv (src/bench.cpp:103-200, compiled unmodified). Linked twice
// by oracle/Makefile:
//   _ref/rvk_ref_bench     against the reference's run_ransac / estimate_all
//   _ref/rvk_dropin_bench  against librvk_dropin.so (link-time substitution,
//                          INTEGRATION.md): the harness's parallel_* columns
//                          then time the sm_100a path while the sequential_*
//                          columns stay the reference's 1-core CPU baselines --
//                          the GPU arm of the bench harness.
//
//   rvk_*_bench [--grid default|N1,N2xP1,P2] -o OUT.csv [--workers W] [--seed S]
//               [--reps R] [--warmups K]
#include <rvk/bench.hpp>

#include <cstdint>
#include <cstring>
#include <exception>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

bool parse_int_list(const std::string& text, std::vector<int>& out) {
  out.clear();
  std::size_t start = 0;
  while (start <= text.size()) {
    const std::size_t comma = text.find(',', start);
    const std::string token =
        text.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
    try {
      std::size_t used = 0;
      const int value = std::stoi(token, &used);
      if (used != token.size() || value < 1) return false;
      out.push_back(value);
    } catch (const std::exception&) {
      return false;
    }
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  return !out.empty();
}

}  // namespace

int main(int argc, char** argv) {
  std::string grid = "default", out_path;
  rvk::BenchConfig config;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (i + 1 >= argc) {
      std::cerr << "error: missing value for " << a << '\n';
      return 2;
    }
    const std::string v = argv[++i];
    try {
      if (a == "--grid") grid = v;
      else if (a == "-o" || a == "--output") out_path = v;
      else if (a == "--workers") config.workers = std::stoi(v);
      else if (a == "--seed") config.ransac.rng_seed = std::stoull(v);
      else if (a == "--reps") config.repetitions = std::stoi(v);
      else if (a == "--warmups") config.warmups = std::stoi(v);
      else {
        std::cerr << "error: unknown option " << a << '\n';
        return 2;
      }
    } catch (const std::exception&) {
      std::cerr << "error: bad value for " << a << '\n';
      return 2;
    }
  }
  if (out_path.empty()) {
    std::cerr << "error: -o is required\n";
    return 2;
  }
  if (grid != "default") {
    const std::size_t cross = grid.find('x');
    if (cross == std::string::npos || !parse_int_list(grid.substr(0, cross), config.cluster_counts) ||
        !parse_int_list(grid.substr(cross + 1), config.points_per_cluster)) {
      std::cerr << "error: grid must be 'default' or 'N1,N2,...xP1,P2,...'\n";
      return 2;
    }
  }
  std::vector<rvk::BenchRow> rows;
  try {
    rows = rvk::run_bench(config);
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 3;
  }
  std::cout << rvk::format_bench_table(rows);
  try {
    rvk::write_bench_csv(out_path, rows);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 3;
  }
  return 0;
}
