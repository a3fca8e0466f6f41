// slab_layout.hpp — host side of the slab tile planner (slab.cu): from the
// per-(window, W row) run lengths, the tiles (whole 32-row slices per stage),
// each tile's slot order and metadata, and where every run's entries go.
// Plain C++ (no CUDA), so it is also benchmarked on a CPU host
// (scripts/plan_bench.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <vector>

namespace rb {

// tile t (window-major: a CTA's contiguous tile range mostly shares one
// window, staged once)
struct SlabTile {
  int32_t a;     // first entry (8-aligned)
  int32_t n;     // entries (multiple of 8; jagged slices carry no padding)
  int32_t meta;  // first metadata element in SlabView::meta (8-aligned)
  int32_t k0;    // first W row of the chunk
  int32_t nr;    // rows of the chunk
  int32_t s;     // window
  int32_t m;     // metadata elements
  int32_t pad;
};

struct SlabLayout {
  std::vector<SlabTile> tiles;
  std::vector<int64_t> tile_bytes;  // staged bytes per tile (CTA balance)
  std::vector<int32_t> off, jx;     // per run (s * nw + k): tile base, jagged-offset slot (see fill_kernel)
  std::vector<int32_t> joff;        // per slice entry: offset inside the tile
  std::vector<uint16_t> meta;       // all tiles' metadata (8-aligned per tile, + 8 slack), unless meta_alloc
  uint16_t* meta_ptr = nullptr;     // where the metadata went (meta.data() or the meta_alloc buffer)
  std::size_t meta_len = 0;
  const uint16_t* meta_data() const { return meta_ptr; }
  std::size_t meta_size() const { return meta_len; }
  int64_t entries = 0;              // padded entries of all tiles
  int max_tile = 0, max_meta = 0;
  bool sorted = false;              // row order used (natural unless it pads too much)
};

// len: run lengths, window-major (len[s * nw + k]); ecap: tile entry cap
// (multiple of 32); rcap: rows per tile; order: 0 auto, 1 natural, 2 sorted;
// row_cost: CTA-balance cost per tile row. false when the layout does not fit
// the int32 offsets. meta_alloc (optional): where to write the metadata (the
// caller's upload staging, e.g. pinned memory: no copy, no zero fill).
using MetaAlloc = std::function<uint16_t*(std::size_t)>;
bool slab_layout(const int32_t* len, int32_t nw, int S, int ecap, int rcap, int order, int64_t row_cost,
                 SlabLayout& out, const MetaAlloc& meta_alloc = {});

// f(i) for i in [0, n) on host threads (RAPDHG_PLAN_THREADS, default half the cores)
int plan_threads();

}  // namespace rb
