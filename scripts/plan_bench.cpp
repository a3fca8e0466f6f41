// CPU timing of the slab planner's host layout (csrc/slab_layout.cpp) on
// synthetic run lengths shaped like the bench's plans:
//   C4 dual:   1e6 W rows x 5 windows, ~10 entries per run
//   C4 primal: 1e4 W rows x 488 windows, ~10 entries per run
//   C2 dual:   1e4 W rows x 49 windows, ~20 entries per run
// g++ -O3 -std=c++17 -I paper_2311_07710_b200/csrc scripts/plan_bench.cpp \
//     paper_2311_07710_b200/csrc/slab_layout.cpp -lpthread -o /tmp/plan_bench && /tmp/plan_bench
#include <chrono>
#include <cstdio>
#include <random>

#include "slab_layout.hpp"

int main() {
  struct Case {
    const char* name;
    int nw, S;
    double mean;
    int order;  // 0 auto, 1 natural (the bench's C4 dual plan is natural: its real runs pad 1.113)
  } cases[] = {{"C4 dual", 1000000, 5, 10.0, 0}, {"C4 dual/n", 1000000, 5, 10.0, 1},
               {"C4 primal", 10000, 488, 10.2, 0}, {"C2 dual", 10000, 49, 20.0, 0}};
  for (const Case& c : cases) {
    std::mt19937_64 g(1);
    std::poisson_distribution<int> P(c.mean);
    std::vector<int32_t> len(static_cast<std::size_t>(c.nw) * c.S);
    for (auto& v : len) v = std::min(P(g), 512);
    for (int rep = 0; rep < 3; ++rep) {
      rb::SlabLayout lay;
      const auto t0 = std::chrono::steady_clock::now();
      const bool ok = rb::slab_layout(len.data(), c.nw, c.S, 2816, 512, c.order, 0, lay);
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      // FNV-1a over the tiles and the metadata: layout changes must keep it
      uint64_t h = 1469598103934665603ull;
      auto mix = [&](const void* p, std::size_t n) {
        for (std::size_t i = 0; i < n; ++i) h = (h ^ static_cast<const uint8_t*>(p)[i]) * 1099511628211ull;
      };
      mix(lay.tiles.data(), sizeof(rb::SlabTile) * lay.tiles.size());
      mix(lay.meta_data(), sizeof(uint16_t) * lay.meta_size());
      std::printf("%-10s %s tiles %zu entries %lld (%s) %.1f ms hash %016llx\n", c.name, ok ? "ok" : "FAIL",
                  lay.tiles.size(), static_cast<long long>(lay.entries), lay.sorted ? "sorted" : "natural", ms,
                  static_cast<unsigned long long>(h));
    }
  }
}
