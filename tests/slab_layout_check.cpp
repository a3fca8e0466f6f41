// Invariant checker for the slab planner's host layout (csrc/slab_layout.cpp),
// built and run by tests/test_slab_layout.py on the CPU. For synthetic run
// lengths of several shapes and each row order it checks that the tiles,
// offsets and metadata describe every (window, W row) run exactly once in the
// form slab.cuh reads them, and prints a hash of the layout so the test can
// compare runs with different thread counts (the layout must not depend on
// them). Exit status 1 on the first violated invariant.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "slab_layout.hpp"

namespace {

int fail(const char* what, int t) {
  std::printf("FAIL %s (tile %d)\n", what, t);
  std::exit(1);
}

uint64_t fnv(uint64_t h, const void* p, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) h = (h ^ static_cast<const uint8_t*>(p)[i]) * 1099511628211ull;
  return h;
}

// returns the layout hash
uint64_t check(const std::vector<int32_t>& len, int32_t nw, int S, int ecap, int rcap, int order, bool pinned_sink) {
  rb::SlabLayout lay;
  std::vector<uint16_t> sink;
  rb::MetaAlloc alloc;
  if (pinned_sink)
    alloc = [&](std::size_t n) {
      sink.assign(n, 0xabcd);  // garbage: every element must be written
      return sink.data();
    };
  if (!rb::slab_layout(len.data(), nw, S, ecap, rcap, order, 0, lay, alloc)) fail("layout does not fit", -1);
  const uint16_t* meta = lay.meta_data();
  const int nt = static_cast<int>(lay.tiles.size());
  if (order == 1 && lay.sorted) fail("order 1 must be natural", -1);
  if (order == 2 && !lay.sorted) fail("order 2 must be sorted", -1);
  std::vector<int32_t> seen(static_cast<std::size_t>(nw) * S, 0);
  int64_t cursor = 0, mcur = 0;
  int prev_s = -1, prev_minlen = 1 << 30;
  for (int t = 0; t < nt; ++t) {
    const rb::SlabTile& d = lay.tiles[t];
    if (d.s < prev_s || d.s >= S) fail("tiles not window-major", t);
    if (d.s != prev_s) prev_minlen = 1 << 30;
    prev_s = d.s;
    if (d.a != cursor) fail("entry offset", t);
    if (d.meta != mcur) fail("metadata offset", t);
    const int nr = d.nr, nsl = (nr + 31) / 32;
    if (nr <= 0 || nr > rcap) fail("rows per tile", t);
    if (d.m != 3 * nr + nsl + 1) fail("metadata size", t);
    if (d.n > lay.max_tile || d.m > lay.max_meta) fail("max_tile / max_meta", t);
    if (d.n > ecap && nr > 32) fail("tile over the entry cap could have been split", t);
    const uint16_t* m = meta + d.meta;
    const int32_t* L = len.data() + static_cast<int64_t>(d.s) * nw;
    int minlen = 1 << 30, maxlen = 0;
    for (int i = 0; i < nr; ++i) {
      const int32_t r = static_cast<int32_t>(m[2 * i] | (static_cast<uint32_t>(m[2 * i + 1]) << 16));
      if (r < 0 || r >= nw) fail("row id", t);
      if (L[r] <= 0) fail("row without a run", t);
      if (m[2 * nr + i] != L[r]) fail("run length", t);
      if (i > 0 && m[2 * nr + i] > m[2 * nr + i - 1]) fail("rows not sorted by run", t);
      if (seen[static_cast<int64_t>(d.s) * nw + r]++) fail("run placed twice", t);
      minlen = std::min(minlen, L[r]), maxlen = std::max(maxlen, L[r]);
    }
    int64_t off = 0;
    for (int q = 0; q < nsl; ++q) {
      if (m[3 * nr + q] != off) fail("slice offset", t);
      off += 32 * static_cast<int64_t>(m[2 * nr + 32 * q]);
    }
    if (m[3 * nr + nsl] != off || off != d.n) fail("tile entries", t);
    const int64_t mend = d.meta + ((d.m + 7) & ~7);
    for (int64_t j = d.meta + d.m; j < mend; ++j)
      if (meta[j] != 0) fail("metadata padding", t);
    // (natural tiles are index ranges of the window's rows, except that a tile
    // over the cap is split by run length, so only the sorted order is checked)
    if (lay.sorted && maxlen > prev_minlen) fail("sorted tiles out of run order", t);
    prev_minlen = minlen;
    cursor += d.n;
    mcur = mend;
  }
  if (cursor != lay.entries) fail("total entries", -1);
  if (lay.meta_size() != static_cast<std::size_t>(mcur) + 8) fail("metadata length", -1);
  for (std::size_t j = mcur; j < lay.meta_size(); ++j)
    if (meta[j] != 0) fail("metadata slack", -1);
  for (int64_t q = 0; q < static_cast<int64_t>(nw) * S; ++q)
    if ((len[q] > 0) != (seen[q] == 1)) fail("run missing", -1);
  uint64_t h = 1469598103934665603ull;
  h = fnv(h, lay.tiles.data(), sizeof(rb::SlabTile) * lay.tiles.size());
  h = fnv(h, meta, sizeof(uint16_t) * lay.meta_size());
  return h;
}

}  // namespace

int main() {
  struct Case {
    const char* name;
    int32_t nw;
    int S;
    int kind;  // 0 Poisson(mean), 1 skewed (few long runs), 2 mostly empty, 3 every run at the cap
    double mean;
  } cases[] = {{"tall", 200000, 5, 0, 10.0},     {"wide", 2000, 300, 0, 10.0}, {"skewed", 30000, 17, 1, 4.0},
               {"sparse", 50000, 9, 2, 3.0},     {"capped", 4000, 3, 3, 0.0},  {"one row", 1, 4, 0, 30.0},
               {"empty window", 5000, 6, 2, 0.0}};
  for (const Case& c : cases) {
    std::mt19937_64 g(12345);
    std::poisson_distribution<int> P(c.mean > 0 ? c.mean : 1.0);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<int32_t> len(static_cast<std::size_t>(c.nw) * c.S, 0);
    for (std::size_t q = 0; q < len.size(); ++q) {
      int v = 0;
      if (c.kind == 0) v = P(g);
      else if (c.kind == 1) v = U(g) < 0.02 ? 200 + static_cast<int>(300 * U(g)) : P(g);
      else if (c.kind == 2) v = U(g) < 0.1 ? 1 + P(g) : 0;
      else v = 512;
      if (c.kind == 2 && c.mean == 0.0 && q / c.nw == 2) v = 0;  // one window with no runs at all
      len[q] = std::min(v, 512);
    }
    for (int order = 0; order < 3; ++order)
      for (int sink = 0; sink < 2; ++sink) {
        const uint64_t h = check(len, c.nw, c.S, 2816, 512, order, sink == 1);
        std::printf("OK %s order %d sink %d %016llx\n", c.name, order, sink, static_cast<unsigned long long>(h));
      }
  }
  return 0;
}
