// slab.cu — setup of the slab tile plans (see slab.cuh).
#include <algorithm>
#include <climits>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "slab.cuh"

namespace rb {

namespace {

// Column histogram by window (integer counts: exact in any order). A block
// counts a grid-stride share in shared memory first — global atomics on a few
// dozen buckets from every entry serialise (8 ms on C2).
constexpr int kHistSmem = 8192;  // buckets counted in shared memory
__global__ void hist_kernel(const int32_t* ci, int64_t nnz, int width, int nb, int* hist) {
  __shared__ int sh[kHistSmem];
  const bool local = nb <= kHistSmem;
  if (local)
    for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = ci[k] / width;
    if (local) atomicAdd(&sh[b], 1);
    else atomicAdd(&hist[b], 1);
  }
  if (!local) return;
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// The plan's windows on the device. Windows start at multiples of `width`, so
// a column's window is one table lookup (lut: window of each aligned block of
// columns, or -1).
struct Wins {
  const Window* w;
  const int32_t* lut;
  int width, nlut, S;
  int stride = 0;  // resident plans: window s is staged at s * stride; all windows form ONE run
  __device__ __forceinline__ int of(int32_t c) const {
    const int b = c / width;
    if (b >= nlut) return -1;
    const int s = lut[b];
    return (s >= 0 && c - w[s].lo < w[s].len) ? s : -1;
  }
  __device__ __forceinline__ int run(int s) const { return stride ? 0 : s; }  // run index of window s
  __device__ __forceinline__ uint16_t offset(int s, int32_t c) const {        // column in the staged image
    return static_cast<uint16_t>((stride ? s * stride : 0) + (c - w[s].lo));
  }
};

// in-window entries of row r, per window (per: zeroed, stride apart; may be
// null) and in total; *maxrun = the longest per-window run. Columns are
// sorted, so a window's entries are one contiguous run.
__device__ __forceinline__ int in_window_count(const int32_t* rp, const int32_t* ci, int r, const Wins& wins,
                                               int* per, int64_t stride, int* maxrun = nullptr) {
  const int b = rp[r], e = rp[r + 1];
  int tot = 0, mx = 0, cur = -1, run = 0;
  for (int p = b; p < e; ++p) {
    const int w = wins.of(ci[p]);
    if (w < 0) continue;
    const int s = wins.run(w);
    if (s != cur) {
      if (cur >= 0 && per) per[cur * stride] = run;
      cur = s, run = 0;
    }
    ++run, ++tot;
    mx = max(mx, run);
  }
  if (cur >= 0 && per) per[cur * stride] = run;
  if (maxrun) *maxrun = mx;
  return tot;
}

// Rows [r0, r1): in-window entry count, or 0 when a window run or the rest
// (other entries of both segments) exceeds cap — such rows stay on the
// regular schedule, whose block/split bins spread long rows over a CTA.
__global__ void count_kernel(const int32_t* rp, const int32_t* ci, const int32_t* rp_o, int32_t r0, int32_t r1,
                             Wins wins, int cap, int32_t* cnt) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= r1 - r0) return;
  const int r = r0 + static_cast<int>(i);
  int mx = 0;
  const int tot = in_window_count(rp, ci, r, wins, nullptr, 0, &mx);
  const int rest = (rp[r + 1] - rp[r]) - tot + (rp_o ? rp_o[r + 1] - rp_o[r] : 0);
  cnt[i] = (mx <= cap && rest <= cap) ? tot : 0;
}

// per-(window, W row) counts (window-major, cnt[s * nw + k]) and rest counts
__global__ void seg_counts_kernel(const int32_t* rows, int32_t nw, const int32_t* rp_w, const int32_t* ci_w,
                                  const int32_t* rp_o, Wins wins, int32_t* cnt, int32_t* rest_w, int32_t* rest_o) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nw) return;
  const int r = rows[k];
  const int tot = in_window_count(rp_w, ci_w, r, wins, cnt + k, nw);
  rest_w[k] = (rp_w[r + 1] - rp_w[r]) - tot;
  rest_o[k] = rp_o ? rp_o[r + 1] - rp_o[r] : 0;
}

// thread per W row: scatter its entries into its slice lane (run (s, k): tile
// base off[s * nw + k]; jx = (index of its slice's jagged offsets in joff) *
// 32 + lane; entry e at base + joff[jx / 32 + e] + lane) and into the rest CSRs
__global__ void fill_kernel(const int32_t* rows, int32_t nw, const int32_t* rp_w, const int32_t* ci_w,
                            const int32_t* rp_o, const int32_t* ci_o, Wins wins, const int32_t* off,
                            const int32_t* jx, const int32_t* joff, uint16_t* col, int32_t* pos,
                            const int32_t* rrp_w, int32_t* rci_w, int32_t* rpos_w, const int32_t* rrp_o,
                            int32_t* rci_o, int32_t* rpos_o) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nw) return;
  const int r = rows[k];
  int cur = -1, e = 0;
  int rw = rrp_w[k];
  for (int p = rp_w[r]; p < rp_w[r + 1]; ++p) {
    const int32_t c = ci_w[p];
    const int w = wins.of(c);
    if (w >= 0) {
      const int s = wins.run(w);
      if (s != cur) cur = s, e = 0;
      const int64_t run = static_cast<int64_t>(s) * nw + k;
      const int64_t wp = off[run] + joff[(jx[run] >> 5) + e] + (jx[run] & 31);
      col[wp] = wins.offset(w, c);
      pos[wp] = p;
      ++e;
    } else {
      rci_w[rw] = c;
      rpos_w[rw] = p;
      ++rw;
    }
  }
  if (rp_o) {
    int ro = rrp_o[k];
    for (int p = rp_o[r]; p < rp_o[r + 1]; ++p, ++ro) {
      rci_o[ro] = ci_o[p];
      rpos_o[ro] = p;
    }
  }
}

__global__ void gather_kernel(double* dst, const double* src, const int32_t* pos, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = pos[i] >= 0 ? src[pos[i]] : 0.0;
}

inline unsigned g1(int64_t n) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, 256)); }

std::string slab_mode() {
  const char* e = std::getenv("RAPDHG_SLAB");
  return e ? e : "auto";
}
int slab_min_row() { return slab_mode() == "force" ? 1 : kSlabMinRow; }

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

template <class T>
std::vector<T> download(const DevBuf<T>& d, int64_t n, cudaStream_t st) {
  std::vector<T> h(static_cast<std::size_t>(n));
  if (n > 0) RB_CUDA(cudaMemcpyAsync(h.data(), d.get(), sizeof(T) * n, cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  return h;
}

std::vector<int32_t> scan_host(const std::vector<int32_t>& cnt) {
  std::vector<int32_t> rp(cnt.size() + 1, 0);
  for (std::size_t i = 0; i < cnt.size(); ++i) rp[i + 1] = rp[i] + cnt[i];
  return rp;
}

// One tile: W rows (indices k, runs already sorted by length, descending),
// 32 per slice, each slice as wide as its longest run (the per-window sort
// makes slices nearly uniform). meta (uint16) = perm (uint32 row index k per
// slot, 2 elements each) | len[nr] | soff[nsl + 1]; joff = per slice the start
// of each entry e (fill_kernel only); offsets relative to the tile's first
// entry.
struct TileLayout {
  std::vector<int32_t> rows;  // the tile's W rows in slot order
  std::vector<uint16_t> meta;
  std::vector<int32_t> joff;  // slice q's offsets start at joff[sj[q]]
  std::vector<int32_t> sj;
  int32_t n = 0;
};
TileLayout layout_tile(const int32_t* rows, const int32_t* len, int32_t nr) {
  TileLayout L;
  const int nsl = (nr + 31) / 32;
  L.meta.resize(3 * static_cast<std::size_t>(nr) + nsl + 1);
  for (int32_t i = 0; i < nr; ++i) {
    L.meta[2 * i] = static_cast<uint16_t>(static_cast<uint32_t>(rows[i]) & 0xffffu);
    L.meta[2 * i + 1] = static_cast<uint16_t>(static_cast<uint32_t>(rows[i]) >> 16);
    L.meta[2 * nr + i] = static_cast<uint16_t>(len[i]);
  }
  int64_t cur = 0;
  for (int q = 0; q < nsl; ++q) {
    L.meta[3 * nr + q] = static_cast<uint16_t>(cur);  // soff[q]
    L.sj.push_back(static_cast<int32_t>(L.joff.size()));
    const int Lm = len[32 * q];
    for (int e = 0; e < Lm; ++e) L.joff.push_back(static_cast<int32_t>(cur + 32 * e));
    cur += 32 * static_cast<int64_t>(Lm);
  }
  L.meta[3 * nr + nsl] = static_cast<uint16_t>(cur);
  L.n = static_cast<int32_t>(cur);  // a multiple of 32
  return L;
}

// f(0 .. n-1) on host threads: half the cores by default, as the two ops'
// plans are built concurrently (RAPDHG_PLAN_THREADS overrides)
int plan_threads() {
  static const int t = [] {
    const char* e = std::getenv("RAPDHG_PLAN_THREADS");
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    return std::max(1, std::min(32, e ? std::atoi(e) : std::max(1, hw / 2)));
  }();
  return t;
}
template <class F>
void parallel_for(int64_t n, const F& f) {
  const int T = static_cast<int>(std::min<int64_t>(n, plan_threads()));
  if (T <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (int64_t i = t; i < n; i += T) f(i);
    });
  for (auto& x : th) x.join();
}

}  // namespace

int slab_grid(const void* kernel, int smem_bytes) {
  int per_sm = 0;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSlabThreads, smem_bytes));
  return std::max(1, per_sm) * kSMs;
}

SlabChoice choose_slabs(const int32_t* rp, const int32_t* ci, int32_t rows, int64_t nnz, int32_t ncols,
                        cudaStream_t st) {
  (void)rp;
  SlabChoice ch;
  const std::string mode = slab_mode();
  if (mode == "off" || nnz <= 0 || ncols <= 0 || rows <= 0) return ch;
  // RAPDHG_SLAB_WIDTH: window width in columns (tuning; 16-bit offsets)
  const int width = std::min(std::max(env_int("RAPDHG_SLAB_WIDTH", kSlabWidth), 128), 65536);
  const int nb = static_cast<int>(ceil_div(ncols, width));
  DevBuf<int> hist(nb);
  hist.zero(st);
  hist_kernel<<<std::min<unsigned>(g1(nnz), 4 * kSMs), 256, 0, st>>>(ci, nnz, width, nb, hist.get());
  RB_LAUNCH_CHECK();
  const std::vector<int> h = download(hist, nb, st);
  // aligned windows, densest first, kept while they serve enough gathers per
  // column to repay staging (force: any non-empty window)
  const double min_density = mode == "force" ? 1e-9 : kSlabMinDensity;
  // RAPDHG_SLAB_MIN_WINDOWS: below this many windows the gathered range is
  // small enough for L1 to serve it (the regular kernel is as fast)
  std::vector<int> order(nb);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return h[a] > h[b]; });
  for (int b : order) {
    if (static_cast<int>(ch.windows.size()) == kMaxSlabs) break;
    const int32_t lo = b * width, len = std::min(width, ncols - lo) & ~1;  // even: 16 B bulk copies
    if (len == 0 || h[b] == 0) continue;
    if (h[b] < min_density * len) break;
    ch.windows.push_back(Window{lo, len});
  }
  ch.width = width;
  std::sort(ch.windows.begin(), ch.windows.end(), [](const Window& a, const Window& b) { return a.lo < b.lo; });
  const int min_windows = mode == "force" ? 1 : env_int("RAPDHG_SLAB_MIN_WINDOWS", kSlabMinWindows);
  if (static_cast<int>(ch.windows.size()) < min_windows) ch.windows.clear();
  if (std::getenv("RAPDHG_TRACE"))
    std::fprintf(stderr, "[slab] %d columns: %zu windows of %d\n", ncols, ch.windows.size(), width);
  return ch;
}

// Off by default (RAPDHG_SLAB_RESIDENT=1 enables): measured slower — one
// 174 KB CTA per SM holds only a few slices in flight, and each lane's
// in-kernel epilogue (row id, rest CSR chain, gather, epilogue inputs) is a
// chain of dependent global loads: C4's dual took 320 us against 134 us
// windowed (ncu: 14% warps active, long_scoreboard), C3's primal 82 vs 68 us.
bool slab_resident(const SlabChoice& choice) {
  const char* e = std::getenv("RAPDHG_SLAB_RESIDENT");
  if (!(e && e[0] == '1')) return false;
  const int S = static_cast<int>(choice.windows.size());
  return S > 0 && S <= kSlabResidentMax && S * choice.width <= 65536;  // 16-bit offsets into the image
}

void build_slab_plan(SlabPlan& plan, const SlabChoice& choice, int seg, const int32_t* rp1, const int32_t* ci1,
                     const int32_t* rp2, const int32_t* ci2, int32_t r0, int32_t r1, cudaStream_t st) {
  plan = SlabPlan{};
  const int nwin = static_cast<int>(choice.windows.size());
  if (nwin == 0 || r1 <= r0) return;
  // resident: every window staged at once (window s at s * width doubles),
  // each W row ONE run over all of them, finished inside the slab kernel
  const bool resident = slab_resident(choice);
  const int S = resident ? 1 : nwin;  // runs per W row
  Tracer tr(st);
  {
    const int nlut = choice.windows.back().lo / choice.width + 1;
    std::vector<int32_t> lut(nlut, -1);
    for (int s = 0; s < nwin; ++s) lut[choice.windows[s].lo / choice.width] = s;
    plan.win.alloc(nwin);
    plan.win.upload(choice.windows.data(), nwin, st);
    plan.lut.alloc(nlut);
    plan.lut.upload(lut.data(), nlut, st);
  }
  const Wins wins{plan.win.get(), plan.lut.get(), choice.width, choice.windows.back().lo / choice.width + 1, nwin,
                  resident ? choice.width : 0};
  const int32_t* rp_w = seg == 0 ? rp1 : rp2;  // windowed segment
  const int32_t* ci_w = seg == 0 ? ci1 : ci2;
  const int32_t* rp_o = seg == 0 ? rp2 : rp1;  // the other segment (rest only)
  const int32_t* ci_o = seg == 0 ? ci2 : ci1;
  const int32_t nr = r1 - r0;
  std::vector<int32_t> hc;
  {
    DevBuf<int32_t> cnt(nr);
    count_kernel<<<g1(nr), 256, 0, st>>>(rp_w, ci_w, rp_o, r0, r1, wins, kSlabRunCap, cnt.get());
    RB_LAUNCH_CHECK();
    hc = download(cnt, nr, st);
  }
  std::vector<int32_t> rows;
  const int min_row = slab_min_row();
  for (int32_t i = 0; i < nr; ++i)
    if (hc[i] >= min_row) rows.push_back(r0 + i);
  const int32_t nw = static_cast<int32_t>(rows.size());
  if (nw == 0) {
    if (std::getenv("RAPDHG_TRACE"))
      std::fprintf(stderr, "[slab] seg %d rows [%d,%d): %d windows, no W rows\n", seg, r0, r1, S);
    return;
  }
  plan.rows.alloc(nw);
  plan.rows.upload(rows.data(), nw, st);
  // per-(window, row) run lengths and rest counts
  const int64_t runs = static_cast<int64_t>(nw) * S;
  if (runs > kSlabMaxRuns) {  // ~20 B of plan state per (window, W row) pair
    if (std::getenv("RAPDHG_TRACE"))
      std::fprintf(stderr, "[slab] seg %d: %d W rows x %d windows exceeds the plan budget\n", seg, nw, S);
    plan = SlabPlan{};
    return;
  }
  DevBuf<int32_t> c2(runs), rw(nw), ro(nw);
  c2.zero(st);
  seg_counts_kernel<<<g1(nw), 256, 0, st>>>(plan.rows.get(), nw, rp_w, ci_w, rp_o, wins, c2.get(), rw.get(), ro.get());
  RB_LAUNCH_CHECK();
  const std::vector<int32_t> hc2 = download(c2, runs, st), hrw = download(rw, nw, st), hro = download(ro, nw, st);
  tr.mark("    counts");
  // Tiles, per window, of whole 32-row slices (slice-padded entries within
  // the stage, rows within the row cap), from one of two row orders:
  //  * natural: the window's W rows in index order, each tile's rows sorted
  //    by run length — neighbouring rows share tiles, so partial writes and
  //    the finish pass stay coalesced;
  //  * sorted: all the window's W rows sorted by run length first — slices of
  //    nearly equal runs, no padding, but scattered partial writes.
  // Natural unless its padding exceeds kSlabNaturalPad (RAPDHG_SLAB_ORDER=
  // natural|sorted forces). Rows with an empty run in a window appear in none
  // of its tiles (their partial stays the zero written at setup).
  const int ecap = (std::min(32736, std::max(256, env_int("RAPDHG_SLAB_TILE", kSlabTileCap))) + 31) & ~31;
  const int rcap = kSlabRowCap;
  struct TileSpan {
    int s;
    int32_t b, e;  // range of order[s]
  };
  auto build = [&](bool sorted, std::vector<std::vector<int32_t>>& order, std::vector<TileSpan>& spans,
                   std::vector<TileLayout>& lay) {
    order.assign(S, {});
    parallel_for(S, [&](int64_t si) {
      const int s = static_cast<int>(si);
      const int32_t* len = hc2.data() + static_cast<int64_t>(s) * nw;
      std::vector<int32_t> o;
      o.reserve(nw);
      if (sorted) {
        std::vector<int32_t> start(kSlabRunCap + 2, 0);
        for (int32_t k = 0; k < nw; ++k) ++start[kSlabRunCap - len[k] + 1];
        for (int v = 1; v <= kSlabRunCap + 1; ++v) start[v] += start[v - 1];
        o.resize(nw);
        for (int32_t k = 0; k < nw; ++k) o[start[kSlabRunCap - len[k]]++] = k;
        int32_t cnt = nw;
        while (cnt > 0 && len[o[cnt - 1]] == 0) --cnt;  // empty runs last
        o.resize(cnt);
      } else {
        for (int32_t k = 0; k < nw; ++k)
          if (len[k] > 0) o.push_back(k);
      }
      order[s] = std::move(o);
    });
    tr.mark("    row orders");
    spans.clear();
    for (int s = 0; s < S; ++s) {
      const std::vector<int32_t>& o = order[s];
      const int32_t* len = hc2.data() + static_cast<int64_t>(s) * nw;
      const int32_t no = static_cast<int32_t>(o.size());
      int32_t b = 0;
      int64_t acc = 0;
      for (int32_t q = 0; q < no; q += 32) {  // group of 32 rows starting at q
        const int32_t qe = std::min(no, q + 32);
        int64_t w = 0;  // sorted: the slice's padded width; natural: raw entries (7/8 budget below)
        if (sorted) w = 32 * static_cast<int64_t>(len[o[q]]);
        else
          for (int32_t i = q; i < qe; ++i) w += len[o[i]];
        const int64_t cap = sorted ? ecap : ecap * 7 / 8;
        if (q > b && (acc + w > cap || qe - b > rcap)) {
          spans.push_back({s, b, q});
          b = q;
          acc = 0;
        }
        acc += w;
      }
      if (b < no) spans.push_back({s, b, no});
    }
    tr.mark("    spans");
    for (;;) {  // lay out (rows of a tile sorted by run); split tiles that overflow
      lay.assign(spans.size(), TileLayout{});
      parallel_for(static_cast<int64_t>(spans.size()), [&](int64_t t) {
        const TileSpan& sp = spans[t];
        const int32_t* len = hc2.data() + static_cast<int64_t>(sp.s) * nw;
        std::vector<int32_t> rows_t(order[sp.s].begin() + sp.b, order[sp.s].begin() + sp.e);
        std::stable_sort(rows_t.begin(), rows_t.end(), [&](int32_t x, int32_t y) { return len[x] > len[y]; });
        std::vector<int32_t> len_t(rows_t.size());
        for (std::size_t i = 0; i < rows_t.size(); ++i) len_t[i] = len[rows_t[i]];
        lay[t] = layout_tile(rows_t.data(), len_t.data(), static_cast<int32_t>(rows_t.size()));
        lay[t].rows = std::move(rows_t);
      });
      std::vector<TileSpan> next;
      bool split = false;
      for (std::size_t t = 0; t < spans.size(); ++t) {
        const TileSpan& sp = spans[t];
        if (lay[t].n > ecap && sp.e - sp.b > 32) {
          const int32_t mid = sp.b + std::max<int32_t>(32, ((sp.e - sp.b) / 2) & ~31);
          next.push_back({sp.s, sp.b, mid});
          next.push_back({sp.s, mid, sp.e});
          split = true;
        } else {
          next.push_back(sp);
        }
      }
      if (!split) break;
      spans.swap(next);
    }
  };
  std::vector<std::vector<int32_t>> order;
  std::vector<TileSpan> spans;
  std::vector<TileLayout> lay;
  bool sorted = false;
  {
    const char* mode = std::getenv("RAPDHG_SLAB_ORDER");
    if (mode) {
      sorted = std::string(mode) == "sorted";
    } else {
      // natural unless it pads too much: the padding of natural tiles from the
      // run lengths alone (each tile's runs sorted, 32-row slices)
      int64_t padded = 0, actual = 0;
      for (int32_t c : hc2) actual += c;
      std::vector<int64_t> pad_w(S, 0);
      parallel_for(S, [&](int64_t si) {
        const int32_t* len = hc2.data() + si * nw;
        std::vector<int32_t> buf;
        int64_t raw = 0, pad = 0;
        auto flush = [&] {
          std::sort(buf.begin(), buf.end(), std::greater<int32_t>());
          for (std::size_t q = 0; q < buf.size(); q += 32) pad += 32 * static_cast<int64_t>(buf[q]);
          buf.clear();
          raw = 0;
        };
        for (int32_t k = 0; k < nw; ++k) {
          if (len[k] == 0) continue;
          if (buf.size() % 32 == 0 && !buf.empty() &&
              (raw + len[k] > ecap * 7 / 8 || static_cast<int>(buf.size()) + 1 > rcap))
            flush();
          buf.push_back(len[k]);
          raw += len[k];
        }
        flush();
        pad_w[si] = pad;
      });
      for (int64_t v : pad_w) padded += v;
      sorted = static_cast<double>(padded) > kSlabNaturalPad * static_cast<double>(std::max<int64_t>(actual, 1));
    }
    tr.mark("    padding estimate");
    build(sorted, order, spans, lay);
  }
  const int32_t ntiles = static_cast<int32_t>(spans.size());
  tr.mark("    tiles + layouts");
  // tile arrays: window-major, each tile 32-entry aligned; run (s, k): tile
  // base off[s * nw + k] and jx[s * nw + k] (see fill_kernel)
  std::vector<int32_t> off(runs, 0), jx(runs, 0);
  std::vector<SlabTile> tiles(ntiles);
  const int64_t row_cost = env_int("RAPDHG_SLAB_ROWCOST", kSlabRowCost);
  std::vector<int64_t> joff_at(ntiles + 1, 0), meta_at(ntiles + 1, 0);
  int64_t cursor = 0;
  int max_tile = 0, max_meta = 0;
  plan.tile_bytes.resize(ntiles);
  for (int32_t t = 0; t < ntiles; ++t) {  // offsets (sequential prefix)
    const TileSpan& sp = spans[t];
    const TileLayout& L = lay[t];
    SlabTile& d = tiles[t];
    d.a = static_cast<int32_t>(cursor);
    d.n = L.n;
    d.meta = static_cast<int32_t>(meta_at[t]);
    d.k0 = 0;
    d.nr = sp.e - sp.b;
    d.s = sp.s;
    d.m = static_cast<int32_t>(L.meta.size());
    max_tile = std::max(max_tile, d.n);
    max_meta = std::max(max_meta, d.m);
    // cost for balancing the CTAs' contiguous ranges: staged bytes, per-row
    // work (length/perm loads, the partial store), a fixed per-tile cost
    plan.tile_bytes[t] = 10 * static_cast<int64_t>(d.n) + 2 * static_cast<int64_t>(d.m) +
                         row_cost * static_cast<int64_t>(d.nr) + 16384;
    joff_at[t + 1] = joff_at[t] + static_cast<int64_t>(L.joff.size());
    meta_at[t + 1] = meta_at[t] + ((static_cast<int64_t>(L.meta.size()) + 7) & ~int64_t{7});
    cursor += d.n;
  }
  std::vector<int32_t> joff(joff_at[ntiles]);
  std::vector<uint16_t> meta(meta_at[ntiles], 0);
  parallel_for(ntiles, [&](int64_t t) {  // contents (disjoint per tile)
    const TileSpan& sp = spans[t];
    const TileLayout& L = lay[t];
    const int32_t n_r = sp.e - sp.b;
    for (int32_t slot = 0; slot < n_r; ++slot) {
      const int64_t run = static_cast<int64_t>(sp.s) * nw + L.rows[slot];
      off[run] = tiles[t].a;
      jx[run] = static_cast<int32_t>((joff_at[t] + L.sj[slot / 32]) * 32 + slot % 32);
    }
    std::copy(L.joff.begin(), L.joff.end(), joff.begin() + joff_at[t]);
    std::copy(L.meta.begin(), L.meta.end(), meta.begin() + meta_at[t]);
  });
  if (cursor > INT32_MAX || max_tile > ecap || max_meta > kSlabMetaCap ||
      static_cast<int64_t>(joff.size()) * 32 > INT32_MAX) {  // int32 offsets; tiles must fit a stage
    plan = SlabPlan{};
    return;
  }
  tr.mark("    tile arrays");
  meta.resize(meta.size() + 8, 0);  // slack: a tile's metadata copy rounds up to 8
  const int64_t total = std::max<int64_t>(cursor, 32);
  DevBuf<int32_t> doff(runs), djx(runs), djoff(joff.size());
  doff.upload(off.data(), runs, st);
  djx.upload(jx.data(), runs, st);
  djoff.upload(joff.data(), joff.size(), st);
  plan.tile.alloc(tiles.size());
  plan.tile.upload(tiles.data(), tiles.size(), st);
  plan.meta.alloc(meta.size());
  plan.meta.upload(meta.data(), meta.size(), st);
  plan.col.alloc(total), plan.pos.alloc(total), plan.val.alloc(total);
  RB_CUDA(cudaMemsetAsync(plan.col.get(), 0, sizeof(uint16_t) * total, st));
  RB_CUDA(cudaMemsetAsync(plan.pos.get(), 0xff, sizeof(int32_t) * total, st));  // padding: pos -1 -> 0.0
  const std::vector<int32_t> rrw = scan_host(hrw), rro = scan_host(hro);
  // rest CSRs keep the op's segment order: rest1 = segment 1, rest2 = segment 2
  DevBuf<int32_t>& rrp_w = seg == 0 ? plan.rrp1 : plan.rrp2;
  DevBuf<int32_t>& rci_w = seg == 0 ? plan.rci1 : plan.rci2;
  DevBuf<int32_t>& rpos_w = seg == 0 ? plan.rpos1 : plan.rpos2;
  DevBuf<int32_t>& rrp_o = seg == 0 ? plan.rrp2 : plan.rrp1;
  DevBuf<int32_t>& rci_o = seg == 0 ? plan.rci2 : plan.rci1;
  DevBuf<int32_t>& rpos_o = seg == 0 ? plan.rpos2 : plan.rpos1;
  rrp_w.alloc(nw + 1), rrp_o.alloc(nw + 1);
  rrp_w.upload(rrw.data(), nw + 1, st);
  rrp_o.upload(rro.data(), nw + 1, st);
  rci_w.alloc(rrw[nw]), rpos_w.alloc(rrw[nw]), rci_o.alloc(rro[nw]), rpos_o.alloc(rro[nw]);
  (seg == 0 ? plan.rval1 : plan.rval2).alloc(rrw[nw]);
  (seg == 0 ? plan.rval2 : plan.rval1).alloc(rro[nw]);
  fill_kernel<<<g1(nw), 256, 0, st>>>(plan.rows.get(), nw, rp_w, ci_w, rp_o, ci_o, wins, doff.get(), djx.get(),
                                      djoff.get(), plan.col.get(), plan.pos.get(), rrp_w.get(), rci_w.get(), rpos_w.get(),
                                      rp_o ? rrp_o.get() : nullptr, rci_o.get(), rpos_o.get());
  RB_LAUNCH_CHECK();
  tr.mark("    upload + fill");
  plan.partial.alloc(runs);
  plan.partial.zero(st);  // (window, row) pairs without entries keep 0
  {
    std::vector<int32_t> widx(nr, -1), wrow(nw);
    for (int32_t k = 0; k < nw; ++k) widx[rows[k] - r0] = k, wrow[k] = rows[k] - r0;
    plan.widx.alloc(nr);
    plan.widx.upload(widx.data(), nr, st);
    plan.wrow.alloc(nw);
    plan.wrow.upload(wrow.data(), nw, st);
  }
  SlabView& v = plan.view;
  v.nw = nw;
  v.S = S;
  v.J = ntiles;
  v.seg = seg;
  v.ecap = ecap;
  v.mcap = kSlabMetaCap;
  v.win_max = 0;
  for (int s = 0; s < nwin; ++s) v.win_max = std::max(v.win_max, choice.windows[s].len);
  v.win = plan.win.get();
  v.win_max = (v.win_max + 1) & ~1;  // keeps the value stage 16 B-aligned
  v.resident = resident ? nwin : 0;
  if (resident) v.win_max = nwin * choice.width;  // the whole image (window s at s * width)
  v.tile = plan.tile.get();
  v.meta = plan.meta.get();
  v.col = plan.col.get();
  v.val = plan.val.get();
  v.partial = plan.partial.get();
  v.wrow = plan.wrow.get();
  v.rest1 = CsrView{plan.rrp1.get(), plan.rci1.get(), plan.rval1.get()};
  v.rest2 = CsrView{plan.rrp2.get(), plan.rci2.get(), plan.rval2.get()};
  RB_CUDA(cudaStreamSynchronize(st));
  if (std::getenv("RAPDHG_TRACE"))
    std::fprintf(stderr, "[slab] seg %d rows [%d,%d): W rows %d windows %d%s chunks %d tiles %d entries %lld (%.3f padded, %s)\n",
                 seg, r0, r1, nw, nwin, resident ? " (resident)" : "", ntiles, ntiles, static_cast<long long>(cursor),
                 static_cast<double>(cursor) / std::max<int64_t>(1, [&] {
                   int64_t t = 0;
                   for (int32_t c : hc2) t += c;
                   return t;
                 }()),
                 sorted ? "sorted" : "natural");
}

void fill_slab_values(SlabPlan& plan, const double* v1, const double* v2, cudaStream_t st) {
  const SlabView& v = plan.view;
  if (!v.active()) return;
  const double* vw = v.seg == 0 ? v1 : v2;
  const int64_t n = plan.val.size();
  if (n) gather_kernel<<<g1(n), 256, 0, st>>>(plan.val.get(), vw, plan.pos.get(), n);
  if (plan.rval1.size() && v1) gather_kernel<<<g1(plan.rval1.size()), 256, 0, st>>>(plan.rval1.get(), v1, plan.rpos1.get(), plan.rval1.size());
  if (plan.rval2.size() && v2) gather_kernel<<<g1(plan.rval2.size()), 256, 0, st>>>(plan.rval2.get(), v2, plan.rpos2.get(), plan.rval2.size());
  RB_LAUNCH_CHECK();
}

void build_slab_phase(SlabPhase& ph, const SlabChoice& choice, int seg, const int32_t* rp1, const int32_t* ci1,
                      const int32_t* rp2, const int32_t* ci2, int32_t r0, int32_t r1, const int32_t* len,
                      cudaStream_t st) {
  ph = SlabPhase{};
  build_slab_plan(ph.plan, choice, seg, rp1, ci1, rp2, ci2, r0, r1, st);
  if (!ph.active()) return;
  const int32_t nr = r1 - r0;
  const std::vector<int32_t> widx = download(ph.plan.widx, nr, st);
  std::vector<int32_t> orr;
  for (int32_t i = 0; i < nr; ++i)
    if (widx[i] < 0) orr.push_back(i);
  if (!orr.empty()) {
    DevBuf<int32_t> d(orr.size());
    d.upload(orr.data(), orr.size(), st);
    build_schedule(ph.others, len, static_cast<int64_t>(orr.size()), false, st, d.get());
  }
  RB_CUDA(cudaStreamSynchronize(st));
}

void assign_slab_ctas(SlabPlan& plan, int grid, cudaStream_t st) {
  SlabView& v = plan.view;
  const int nt = v.tiles();
  std::vector<int64_t> pre(nt + 1, 0);
  for (int t = 0; t < nt; ++t) pre[t + 1] = pre[t] + plan.tile_bytes[t];
  std::vector<int32_t> cta(grid + 1, 0);
  for (int b = 1; b <= grid; ++b) {
    cta[b] = b == grid ? nt
                       : static_cast<int32_t>(std::lower_bound(pre.begin(), pre.end(), pre[nt] * b / grid) - pre.begin());
    cta[b] = std::max(cta[b], cta[b - 1]);
  }
  plan.cta.alloc(grid + 1);
  plan.cta.upload(cta.data(), grid + 1, st);
  v.cta = plan.cta.get();
  v.grid = grid;
  RB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace rb
