// Generates tests/golden/bench_grid.csv from the REFERENCE's own bench
// harness (proj/include/phgrms/bench.hpp), compiled in place from
// /root/reference (this container only):
//   g++ -O2 -std=c++20 -I/root/reference/proj/include tests/golden/make_bench_golden.cpp -pthread \
//       -o /tmp/mbg && /tmp/mbg > tests/golden/bench_grid.csv
// The total_ms column (a wall time) is replaced by "-"; every other column
// is deterministic and must match the drop-in (tests/cpp/test_dropin.cpp).
#include <cstdio>
#include <sstream>
#include <string>

#include "phgrms/bench.hpp"

int main() {
    phgrms::BenchConfig cfg;
    cfg.synth_sizes = {24, 64, 200};
    cfg.densities = {0.05, 0.30, 0.70};
    cfg.engines = {phgrms::EngineSpec::serial(), phgrms::EngineSpec::parallel(3)};
    cfg.repetitions = 1;
    cfg.seed = 5;
    auto res = phgrms::run_benchmark(cfg);
    for (auto& r : res.records) r.total_ms = 0.0;
    std::string csv = phgrms::write_csv(res.records);
    std::istringstream in(csv);
    std::string line;
    while (std::getline(in, line)) {
        // drop the 8th field (total_ms)
        std::string out;
        int field = 0;
        std::string cur;
        std::istringstream ls(line);
        while (std::getline(ls, cur, ',')) {
            if (field++ == 7) cur = "-";
            out += (out.empty() ? "" : ",") + cur;
        }
        std::printf("%s\n", out.c_str());
    }
    return 0;
}
