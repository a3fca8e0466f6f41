// slab_layout.cpp — host side of the slab tile planner (see slab_layout.hpp).
//
// From the run lengths (entries of W row k in window s), per window:
//  * the row order: natural (index order; neighbouring rows share tiles, so
//    partial writes and the finish pass stay coalesced) or sorted by run
//    length (no padding, scattered partials) — natural unless its padding
//    would exceed kNaturalPad;
//  * greedy spans of whole 32-row groups up to the stage's entry budget and
//    the row cap;
//  * per span (tile) its rows sorted by run length (stable), so each 32-row
//    slice is as wide as its first lane's run, and the tile's metadata:
//    perm (W-row index, 2 x u16 per slot) | len (u16 per slot) | soff (slice
//    starts + end, u16; lane l's entry e of slice q sits at soff[q] + 32 e + l).
// Everything runs in place on one array of row indices per window and writes
// straight into the output arrays (no per-tile containers), in parallel over
// windows, spans and tiles.
#include "slab_layout.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <thread>

#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

namespace rb {

namespace {

constexpr double kNaturalPad = 1.12;  // natural order unless its slices pad more than this
constexpr int kRunCap = 512;          // longest run (slab.cuh kSlabRunCap)

template <class F>
void parallel_for(int64_t n, const F& f) {
  const int T = static_cast<int>(std::min<int64_t>(n, plan_threads()));
  if (T <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  // dynamic: items of very different cost (windows of a skewed pattern)
  std::atomic<int64_t> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&] {
      // below the solver's own thread, which launches the setup kernels the
      // plans overlap (the power iterations: one host sync every 8 steps)
      setpriority(PRIO_PROCESS, static_cast<id_t>(syscall(SYS_gettid)), 5);
      for (int64_t i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& x : th) x.join();
}

struct Span {
  int32_t s, b, e;  // window, range of order[s]
};

// Stable sort of rows r[0, n) by run length L[r] descending: a counting sort
// over the lengths' range (runs are short and the groups small, so this is
// linear where a comparison sort allocates and branches).
void sort_by_len_desc(int32_t* r, int32_t n, const int32_t* L, std::vector<int32_t>& cnt,
                      std::vector<int32_t>& tmp) {
  if (n <= 1) return;
  int32_t lo = L[r[0]], hi = lo;
  for (int32_t i = 1; i < n; ++i) lo = std::min(lo, L[r[i]]), hi = std::max(hi, L[r[i]]);
  if (lo == hi) return;
  const int32_t range = hi - lo + 1;
  cnt.assign(static_cast<std::size_t>(range) + 1, 0);
  for (int32_t i = 0; i < n; ++i) ++cnt[hi - L[r[i]] + 1];
  for (int32_t v = 1; v <= range; ++v) cnt[v] += cnt[v - 1];
  tmp.resize(n);
  for (int32_t i = 0; i < n; ++i) tmp[cnt[hi - L[r[i]]]++] = r[i];
  std::copy(tmp.begin(), tmp.end(), r);
}

// Padded entries of one natural tile whose run lengths are lens[0, n): sorted
// descending, each 32-row slice as wide as its first run.
int64_t padded_entries(const int32_t* lens, int32_t n, std::vector<int32_t>& cnt) {
  if (n == 0) return 0;
  int32_t lo = lens[0], hi = lo;
  for (int32_t i = 1; i < n; ++i) lo = std::min(lo, lens[i]), hi = std::max(hi, lens[i]);
  cnt.assign(static_cast<std::size_t>(hi - lo) + 1, 0);
  for (int32_t i = 0; i < n; ++i) ++cnt[hi - lens[i]];
  // walk lengths from the top: slice q starts at rank 32 q
  int64_t pad = 0, rank = 0, next = 0;
  for (int32_t b = 0; b <= hi - lo; ++b) {
    const int64_t c = cnt[b];
    while (next < rank + c) {  // slice starts falling in this bucket
      pad += 32 * static_cast<int64_t>(hi - b);
      next += 32;
    }
    rank += c;
  }
  return pad;
}

}  // namespace

int plan_threads() {
  static const int t = [] {
    const char* e = std::getenv("RAPDHG_PLAN_THREADS");
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    // the two ops' plans run concurrently: leave the solver thread a core
    return std::max(1, std::min(32, e ? std::atoi(e) : std::max(1, (hw - 1) / 2)));
  }();
  return t;
}

bool slab_layout(const int32_t* len, int32_t nw, int S, int ecap, int rcap, int order_mode, int64_t row_cost,
                 SlabLayout& out, const MetaAlloc& meta_alloc) {
  out = SlabLayout{};
  if (S <= 0 || nw <= 0) return true;
  // RAPDHG_TRACE: the phases' host times
  const bool trace = std::getenv("RAPDHG_TRACE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[slab layout] %d rows x %d windows: %-8s %.2f ms\n", nw, S, what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  // row order per window: rows with a non-empty run (natural index order);
  // windows cut into chunks of rows so that few, tall windows (C4's dual: 5 x
  // 1e6 rows) still spread over the threads: count per chunk, then fill
  constexpr int32_t kOrderChunk = 1 << 16;
  const int32_t nch = (nw + kOrderChunk - 1) / kOrderChunk;
  std::vector<int32_t> ccount(static_cast<std::size_t>(S) * nch + 1, 0);
  parallel_for(static_cast<int64_t>(S) * nch, [&](int64_t i) {
    const int64_t si = i / nch;
    const int32_t k0 = static_cast<int32_t>(i % nch) * kOrderChunk, k1 = std::min(nw, k0 + kOrderChunk);
    const int32_t* L = len + si * nw;
    int32_t cnt = 0;
    for (int32_t k = k0; k < k1; ++k) cnt += L[k] > 0;
    ccount[i] = cnt;
  });
  std::vector<std::vector<int32_t>> order(S);
  std::vector<int32_t> cstart(ccount.size(), 0);
  std::vector<int32_t> wcount(S);
  for (int s = 0; s < S; ++s) {
    int32_t c = 0;
    for (int32_t j = 0; j < nch; ++j) cstart[static_cast<std::size_t>(s) * nch + j] = c, c += ccount[static_cast<std::size_t>(s) * nch + j];
    wcount[s] = c;
  }
  parallel_for(S, [&](int64_t si) { order[si].resize(wcount[si]); });  // (fresh pages: fault them in parallel)
  parallel_for(static_cast<int64_t>(S) * nch, [&](int64_t i) {
    const int64_t si = i / nch;
    const int32_t k0 = static_cast<int32_t>(i % nch) * kOrderChunk, k1 = std::min(nw, k0 + kOrderChunk);
    const int32_t* L = len + si * nw;
    int32_t* o = order[si].data() + cstart[i];
    for (int32_t k = k0; k < k1; ++k)
      if (L[k] > 0) *o++ = k;
  });
  phase("order");
  // natural vs sorted: the padding natural tiles would have (each tile's runs
  // sorted, 32-row slices), estimated on a strided sample of up to 64 tiles'
  // worth of rows per window (the decision only needs the ratio)
  bool sorted = order_mode == 2;
  if (order_mode == 0) {
    std::vector<int64_t> pad_w(S, 0), raw_w(S, 0);
    parallel_for(S, [&](int64_t si) {
      const int32_t* L = len + si * nw;
      const std::vector<int32_t>& o = order[si];
      std::vector<int32_t> buf, cnt;
      buf.reserve(rcap);
      int64_t raw = 0, pad = 0, tot = 0;
      const int64_t no = static_cast<int64_t>(o.size());
      // sample: every step-th run of rows of one natural tile
      const int64_t sample_rows = 64 * static_cast<int64_t>(rcap);
      const int64_t stride_blocks = std::max<int64_t>(1, no / std::max<int64_t>(sample_rows, 1));
      auto flush = [&] {
        pad += padded_entries(buf.data(), static_cast<int32_t>(buf.size()), cnt);
        buf.clear();
        raw = 0;
      };
      for (int64_t blk = 0; blk * rcap < no; blk += stride_blocks) {  // blocks of rcap rows, strided
        for (int64_t i = blk * rcap; i < std::min(no, (blk + 1) * rcap); ++i) {
          const int32_t l = L[o[i]];
          if (buf.size() % 32 == 0 && !buf.empty() &&
              (raw + l > ecap * 7 / 8 || static_cast<int>(buf.size()) + 1 > rcap))
            flush();
          buf.push_back(l);
          raw += l;
          tot += l;
        }
        flush();
      }
      pad_w[si] = pad, raw_w[si] = tot;
    });
    int64_t padded = 0, actual = 0;
    for (int s = 0; s < S; ++s) padded += pad_w[s], actual += raw_w[s];
    sorted = static_cast<double>(padded) > kNaturalPad * static_cast<double>(std::max<int64_t>(actual, 1));
  }
  if (sorted)  // by run length, descending (stable: counting sort)
    parallel_for(S, [&](int64_t si) {
      const int32_t* L = len + si * nw;
      std::vector<int32_t>& o = order[si];
      std::vector<int32_t> start(kRunCap + 2, 0), tmp(o.size());
      for (int32_t k : o) ++start[kRunCap - std::min(L[k], kRunCap) + 1];
      for (int v = 1; v <= kRunCap + 1; ++v) start[v] += start[v - 1];
      for (int32_t k : o) tmp[start[kRunCap - std::min(L[k], kRunCap)]++] = k;
      o.swap(tmp);
    });
  phase("padding");
  // greedy spans of whole 32-row groups per window (sorted: the group's padded
  // width; natural: its raw entries against 7/8 of the budget)
  std::vector<std::vector<Span>> spans_w(S);
  parallel_for(S, [&](int64_t si) {
    const int32_t* L = len + si * nw;
    const std::vector<int32_t>& o = order[si];
    const int32_t no = static_cast<int32_t>(o.size());
    std::vector<Span>& sp = spans_w[si];
    int32_t b = 0;
    int64_t acc = 0;
    const int64_t cap = sorted ? ecap : ecap * 7 / 8;
    for (int32_t q = 0; q < no; q += 32) {
      const int32_t qe = std::min(no, q + 32);
      int64_t w = 0;
      if (sorted) w = 32 * static_cast<int64_t>(L[o[q]]);
      else
        for (int32_t i = q; i < qe; ++i) w += L[o[i]];
      if (q > b && (acc + w > cap || qe - b > rcap)) {
        sp.push_back({static_cast<int32_t>(si), b, q});
        b = q;
        acc = 0;
      }
      acc += w;
    }
    if (b < no) sp.push_back({static_cast<int32_t>(si), b, no});
  });
  std::vector<Span> spans;
  for (auto& v : spans_w) spans.insert(spans.end(), v.begin(), v.end());
  phase("spans");
  // tiles: rows sorted by run (in place), padded size; split any that overflow
  // (a sub-range of a sorted span is sorted: halves only need their size)
  auto padded = [&](const Span& sp) {
    const int32_t* L = len + static_cast<int64_t>(sp.s) * nw;
    const int32_t* r = order[sp.s].data();
    int64_t n = 0;
    for (int32_t q = sp.b; q < sp.e; q += 32) n += 32 * static_cast<int64_t>(L[r[q]]);
    return n;
  };
  std::vector<int64_t> tn(spans.size(), 0);
  parallel_for(static_cast<int64_t>(spans.size()), [&](int64_t t) {
    thread_local std::vector<int32_t> cnt, tmp;
    const Span& sp = spans[t];
    sort_by_len_desc(order[sp.s].data() + sp.b, sp.e - sp.b, len + static_cast<int64_t>(sp.s) * nw, cnt, tmp);
    tn[t] = padded(sp);
  });
  for (bool split = true; split;) {
    split = false;
    std::vector<Span> next;
    std::vector<int64_t> nn;
    next.reserve(spans.size());
    nn.reserve(spans.size());
    for (std::size_t t = 0; t < spans.size(); ++t) {
      const Span& sp = spans[t];
      if (tn[t] > ecap && sp.e - sp.b > 32) {
        const int32_t mid = sp.b + std::max<int32_t>(32, ((sp.e - sp.b) / 2) & ~31);
        next.push_back({sp.s, sp.b, mid});
        nn.push_back(padded(next.back()));
        next.push_back({sp.s, mid, sp.e});
        nn.push_back(padded(next.back()));
        split = true;
      } else {
        next.push_back(sp);
        nn.push_back(tn[t]);
      }
    }
    spans.swap(next);
    tn.swap(nn);
  }
  phase("tiles");
  // offsets (sequential prefix over tiles)
  const int32_t ntiles = static_cast<int32_t>(spans.size());
  out.tiles.resize(ntiles);
  out.tile_bytes.resize(ntiles);
  std::vector<int64_t> meta_at(ntiles + 1, 0);
  int64_t cursor = 0;
  for (int32_t t = 0; t < ntiles; ++t) {
    const Span& sp = spans[t];
    const int32_t nr = sp.e - sp.b, nsl = (nr + 31) / 32;
    SlabTile& d = out.tiles[t];
    d.a = static_cast<int32_t>(std::min<int64_t>(cursor, INT32_MAX));
    d.n = static_cast<int32_t>(tn[t]);
    d.meta = static_cast<int32_t>(std::min<int64_t>(meta_at[t], INT32_MAX));
    d.k0 = 0;
    d.nr = nr;
    d.s = sp.s;
    d.m = 3 * nr + nsl + 1;
    d.pad = 0;
    out.max_tile = std::max(out.max_tile, d.n);
    out.max_meta = std::max(out.max_meta, d.m);
    out.tile_bytes[t] = 10 * static_cast<int64_t>(d.n) + 2 * static_cast<int64_t>(d.m) + row_cost * nr + 16384;
    meta_at[t + 1] = meta_at[t] + ((static_cast<int64_t>(d.m) + 7) & ~int64_t{7});
    cursor += d.n;
  }
  out.entries = cursor;
  out.sorted = sorted;
  if (cursor > INT32_MAX || meta_at[ntiles] > INT32_MAX) return false;
  phase("offsets");
  // metadata, in parallel over tiles (disjoint ranges)
  // (written once: each tile zeroes its own 8-alignment tail, no fill pass)
  out.meta_len = static_cast<std::size_t>(meta_at[ntiles]) + 8;  // + slack: copies round up to 8
  if (meta_alloc) {
    out.meta_ptr = meta_alloc(out.meta_len);
  } else {
    out.meta.resize(out.meta_len);
    out.meta_ptr = out.meta.data();
  }
  uint16_t* const meta0 = out.meta_ptr;
  std::fill(meta0 + meta_at[ntiles], meta0 + out.meta_len, uint16_t{0});
  parallel_for(ntiles, [&](int64_t t) {
    const Span& sp = spans[t];
    const int32_t* L = len + static_cast<int64_t>(sp.s) * nw;
    const int32_t* r = order[sp.s].data() + sp.b;
    const int32_t nr = sp.e - sp.b, nsl = (nr + 31) / 32;
    uint16_t* m = meta0 + meta_at[t];
    std::fill(m + 3 * nr + nsl + 1, meta0 + meta_at[t + 1], uint16_t{0});
    for (int32_t i = 0; i < nr; ++i) {
      m[2 * i] = static_cast<uint16_t>(static_cast<uint32_t>(r[i]) & 0xffffu);
      m[2 * i + 1] = static_cast<uint16_t>(static_cast<uint32_t>(r[i]) >> 16);
      m[2 * nr + i] = static_cast<uint16_t>(L[r[i]]);
    }
    int64_t cur = 0;
    for (int32_t q = 0; q < nsl; ++q) {
      m[3 * nr + q] = static_cast<uint16_t>(cur);
      cur += 32 * static_cast<int64_t>(L[r[32 * q]]);
    }
    m[3 * nr + nsl] = static_cast<uint16_t>(cur);
  });
  phase("metadata");
  return true;
}

}  // namespace rb
