// slab.cu — setup of the slab tile plans (see slab.cuh).
#include <algorithm>
#include <climits>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "slab.cuh"
#include "slab_layout.hpp"

namespace rb {

namespace {

// widx[row - r0] = k and wrow[k] = row - r0 for the W rows (rows[k])
__global__ void wrow_kernel(const int32_t* rows, int32_t nw, int32_t r0, int32_t* widx, int32_t* wrow) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nw) return;
  const int32_t r = rows[k] - r0;
  widx[r] = k;
  wrow[k] = r;
}

__global__ void others_flag_kernel(const int32_t* widx, int32_t n, uint8_t* flag) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = widx[i] < 0;
}

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
// cap > 0 (with maxrun): stop as soon as a run or the out-of-window entries
// exceed cap — the row is then no W row whatever the rest holds (C3's
// 1e6-entry budget row took one thread 0.2 s to scan).
__device__ __forceinline__ int in_window_count(const int32_t* rp, const int32_t* ci, int r, const Wins& wins,
                                               int* per, int64_t stride, int* maxrun = nullptr, int cap = 0) {
  const int b = rp[r], e = rp[r + 1];
  int tot = 0, mx = 0, cur = -1, run = 0;
  // batches of 8 entries: their window lookups are independent loads, so a
  // long row (C4's 5,000-entry feature rows) keeps 8 in flight instead of 1
  constexpr int B = 8;
  for (int p0 = b; p0 < e; p0 += B) {
    int wv[B];
#pragma unroll
    for (int u = 0; u < B; ++u) wv[u] = p0 + u < e ? wins.of(ci[p0 + u]) : -2;
    bool stop = false;
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int w = wv[u];
      if (w == -2 || stop) break;
      const int p = p0 + u;
      if (w < 0) {
        if (cap > 0 && (p + 1 - b) - tot > cap) stop = true;
        continue;
      }
      const int s = wins.run(w);
      if (s != cur) {
        if (cur >= 0 && per) per[cur * stride] = run;
        cur = s, run = 0;
      }
      ++run, ++tot;
      mx = max(mx, run);
      if (cap > 0 && mx > cap) stop = true;
    }
    if (stop) break;
  }
  if (cur >= 0 && per) per[cur * stride] = run;
  if (maxrun) *maxrun = mx;
  return tot;
}

// Rows [r0, r1): in-window entry count, or 0 when a window run or the rest
// (other entries of both segments) exceeds cap — such rows stay on the
// regular schedule, whose block/split bins spread long rows over a CTA.
// Rows longer than this are counted by a block each (count_long_kernel,
// seg_counts_long_kernel): per window, two binary searches in the sorted
// columns instead of one thread walking every entry (C4's 1e4 feature rows of
// 5,000 entries: 18 ms of one-thread scans in the primal plan's counts).
constexpr int kLongRow = 2048;

__device__ __forceinline__ int32_t first_at_least(const int32_t* c, int32_t b, int32_t e, int64_t key) {
  while (b < e) {
    const int32_t mid = b + (e - b) / 2;
    if (c[mid] < key) b = mid + 1;
    else e = mid;
  }
  return b;
}

// Block-wide window counts of row r: per window s, c_s (via `per`, stride
// apart, or not at all), and the total and the longest run (thread 0).
template <class PerFn>
__device__ __forceinline__ void block_window_counts(const int32_t* rp, const int32_t* ci, int r, const Wins& wins,
                                                    PerFn per, int* tot_out, int* mx_out) {
  __shared__ int st[256], sm[256];
  const int b = rp[r], e = rp[r + 1];
  int tot = 0, mx = 0;
  for (int s = threadIdx.x; s < wins.S; s += blockDim.x) {
    const Window w = wins.w[s];
    const int c = first_at_least(ci, b, e, static_cast<int64_t>(w.lo) + w.len) - first_at_least(ci, b, e, w.lo);
    per(s, c);
    tot += c;
    mx = max(mx, c);
  }
  st[threadIdx.x] = tot, sm[threadIdx.x] = mx;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (static_cast<int>(threadIdx.x) < h)
      st[threadIdx.x] += st[threadIdx.x + h], sm[threadIdx.x] = max(sm[threadIdx.x], sm[threadIdx.x + h]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *tot_out = st[0], *mx_out = wins.stride ? st[0] : sm[0];  // resident: one run
  __syncthreads();
}

__global__ void count_long_kernel(const int32_t* list, const int32_t* nlist, const int32_t* rp, const int32_t* ci,
                                  const int32_t* rp_o, int32_t r0, Wins wins, int cap, int32_t* cnt) {
  __shared__ int tot, mx;
  for (int i = blockIdx.x; i < *nlist; i += gridDim.x) {
    const int r = list[i];
    block_window_counts(rp, ci, r, wins, [](int, int) {}, &tot, &mx);
    if (threadIdx.x == 0) {
      const int rest = (rp[r + 1] - rp[r]) - tot + (rp_o ? rp_o[r + 1] - rp_o[r] : 0);
      cnt[r - r0] = (mx <= cap && rest <= cap) ? tot : 0;
    }
  }
}

__global__ void count_kernel(const int32_t* rp, const int32_t* ci, const int32_t* rp_o, int32_t r0, int32_t r1,
                             Wins wins, int cap, int32_t* cnt, int32_t* long_list, int32_t* nlong) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= r1 - r0) return;
  const int r = r0 + static_cast<int>(i);
  const int len = rp[r + 1] - rp[r], len_o = rp_o ? rp_o[r + 1] - rp_o[r] : 0;
  if (len > kLongRow && len_o <= cap) {  // a block's work (count_long_kernel)
    long_list[atomicAdd(nlong, 1)] = r;
    return;
  }
  if (len_o > cap) {  // the other segment alone exceeds the rest cap
    cnt[i] = 0;
    return;
  }
  int mx = 0;
  const int tot = in_window_count(rp, ci, r, wins, nullptr, 0, &mx, cap);
  const int rest = len - tot + len_o;  // (an early stop leaves mx or rest above cap)
  cnt[i] = (mx <= cap && rest <= cap) ? tot : 0;
}

// per-(window, W row) counts (window-major, cnt[s * nw + k]) and rest counts
__global__ void seg_counts_kernel(const int32_t* rows, int32_t nw, const int32_t* rp_w, const int32_t* ci_w,
                                  const int32_t* rp_o, Wins wins, int32_t* cnt, int32_t* rest_w, int32_t* rest_o,
                                  int32_t* long_list, int32_t* nlong) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nw) return;
  const int r = rows[k];
  if (rp_w[r + 1] - rp_w[r] > kLongRow) {  // seg_counts_long_kernel
    long_list[atomicAdd(nlong, 1)] = static_cast<int32_t>(k);
    return;
  }
  const int tot = in_window_count(rp_w, ci_w, r, wins, cnt + k, nw);
  rest_w[k] = (rp_w[r + 1] - rp_w[r]) - tot;
  rest_o[k] = rp_o ? rp_o[r + 1] - rp_o[r] : 0;
}

__global__ void seg_counts_long_kernel(const int32_t* list, const int32_t* nlist, const int32_t* rows, int32_t nw,
                                       const int32_t* rp_w, const int32_t* ci_w, const int32_t* rp_o, Wins wins,
                                       int32_t* cnt, int32_t* rest_w, int32_t* rest_o) {
  __shared__ int tot, mx;
  for (int i = blockIdx.x; i < *nlist; i += gridDim.x) {
    const int k = list[i], r = rows[k];
    if (wins.stride) {  // resident: one run over every window
      block_window_counts(rp_w, ci_w, r, wins, [](int, int) {}, &tot, &mx);
      if (threadIdx.x == 0) cnt[k] = tot;
    } else {
      block_window_counts(rp_w, ci_w, r, wins, [&](int s, int c) { cnt[static_cast<int64_t>(s) * nw + k] = c; }, &tot,
                          &mx);
    }
    if (threadIdx.x == 0) {
      rest_w[k] = (rp_w[r + 1] - rp_w[r]) - tot;
      rest_o[k] = rp_o ? rp_o[r + 1] - rp_o[r] : 0;
    }
  }
}

// block per tile, thread per slot: the slot's W row k (perm) has its run in
// the tile's window (resident plans: all its in-window entries) as entries
// e = 0 .. len-1, placed at tile base + soff[slice] + 32 e + lane (the
// layout of slab_layout.cpp); padding keeps col 0 / pos -1 from the memsets.
__global__ void tile_fill_kernel(const SlabTile* tiles, const uint16_t* meta, const int32_t* rows,
                                 const int32_t* rp_w, const int32_t* ci_w, Wins wins, uint16_t* col, int32_t* pos) {
  const SlabTile d = tiles[blockIdx.x];
  const uint16_t* m = meta + d.meta;
  const uint32_t* perm = reinterpret_cast<const uint32_t*>(m);
  const uint16_t* len = m + 2 * d.nr;
  const uint16_t* soff = len + d.nr;
  for (int slot = threadIdx.x; slot < d.nr; slot += blockDim.x) {
    const int32_t k = static_cast<int32_t>(perm[slot]);
    const int L = len[slot];
    const int64_t base = static_cast<int64_t>(d.a) + soff[slot >> 5] + (slot & 31);
    const int r = rows[k];
    const int b = rp_w[r], e = rp_w[r + 1];
    if (wins.stride) {  // resident: every in-window entry, in column order
      int q = 0;
      for (int p = b; p < e && q < L; ++p) {
        const int w = wins.of(ci_w[p]);
        if (w < 0) continue;
        col[base + 32 * static_cast<int64_t>(q)] = wins.offset(w, ci_w[p]);
        pos[base + 32 * static_cast<int64_t>(q)] = p;
        ++q;
      }
    } else {  // the window's run: a contiguous range of the column-sorted row
      const Window w = wins.w[d.s];
      int lo = b, hi = e;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ci_w[mid] < w.lo) lo = mid + 1;
        else hi = mid;
      }
      for (int q = 0; q < L; ++q) {
        col[base + 32 * static_cast<int64_t>(q)] = static_cast<uint16_t>(ci_w[lo + q] - w.lo);
        pos[base + 32 * static_cast<int64_t>(q)] = lo + q;
      }
    }
  }
}

// thread per W row: its entries outside the windows (and its other segment)
// into the rest CSRs
__global__ void rest_fill_kernel(const int32_t* rows, int32_t nw, const int32_t* rp_w, const int32_t* ci_w,
                                 const int32_t* rp_o, const int32_t* ci_o, Wins wins, const int32_t* rrp_w,
                                 int32_t* rci_w, int32_t* rpos_w, const int32_t* rrp_o, int32_t* rci_o,
                                 int32_t* rpos_o) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nw) return;
  const int r = rows[k];
  int rw = rrp_w[k];
  for (int p = rp_w[r]; p < rp_w[r + 1]; ++p) {
    const int32_t c = ci_w[p];
    if (wins.of(c) < 0) {
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

// exclusive scan of n counts into n + 1 offsets on the device; returns the total
int32_t scan_dev(const int32_t* cnt, int32_t n, DevBuf<int32_t>& off, cudaStream_t st) {
  off.alloc(static_cast<std::size_t>(n) + 1);
  off.zero(st);
  if (n > 0) {
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, off.get() + 1, n, st));
    DevBuf<unsigned char> tmp(tb);
    RB_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, cnt, off.get() + 1, n, st));
  }
  int32_t tot = 0;
  RB_CUDA(cudaMemcpyAsync(&tot, off.get() + n, sizeof(tot), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  return tot;
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

std::vector<int32_t> download_len(const int32_t* d, int64_t n, cudaStream_t st) {
  std::vector<int32_t> h(static_cast<std::size_t>(n));
  if (n > 0) RB_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  return h;
}

template <class T>
std::vector<T> download(const DevBuf<T>& d, int64_t n, cudaStream_t st) {
  std::vector<T> h(static_cast<std::size_t>(n));
  if (n > 0) RB_CUDA(cudaMemcpyAsync(h.data(), d.get(), sizeof(T) * n, cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  return h;
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
  // per-row counts through pinned staging (C4's dual: 2e6 rows — a pageable
  // round trip of the counts and the W-row list cost several ms here)
  PinnedBuf<int32_t> hcb;
  hcb.alloc(static_cast<std::size_t>(nr));
  DevBuf<int32_t> long_list(nr), nlong(1);
  {
    DevBuf<int32_t> cnt(nr);
    nlong.zero(st);
    count_kernel<<<g1(nr), 256, 0, st>>>(rp_w, ci_w, rp_o, r0, r1, wins, kSlabRunCap, cnt.get(), long_list.get(),
                                         nlong.get());
    count_long_kernel<<<4 * kSMs, 256, 0, st>>>(long_list.get(), nlong.get(), rp_w, ci_w, rp_o, r0, wins, kSlabRunCap,
                                                cnt.get());
    RB_LAUNCH_CHECK();
    if (nr > 0) RB_CUDA(cudaMemcpyAsync(hcb.get(), cnt.get(), sizeof(int32_t) * nr, cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
  }
  tr.mark("    row counts");
  std::vector<int32_t> rows;
  const int min_row = slab_min_row();
  for (int32_t i = 0; i < nr; ++i)
    if (hcb[i] >= min_row) rows.push_back(r0 + i);
  const int32_t nw = static_cast<int32_t>(rows.size());
  if (nw == 0) {
    if (std::getenv("RAPDHG_TRACE"))
      std::fprintf(stderr, "[slab] seg %d rows [%d,%d): %d windows, no W rows\n", seg, r0, r1, S);
    return;
  }
  plan.rows.alloc(nw);
  std::memcpy(hcb.get(), rows.data(), sizeof(int32_t) * nw);  // (nw <= nr: the staging buffer fits)
  plan.rows.upload(hcb.get(), nw, st);
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
  nlong.zero(st);
  seg_counts_kernel<<<g1(nw), 256, 0, st>>>(plan.rows.get(), nw, rp_w, ci_w, rp_o, wins, c2.get(), rw.get(), ro.get(),
                                            long_list.get(), nlong.get());
  seg_counts_long_kernel<<<4 * kSMs, 256, 0, st>>>(long_list.get(), nlong.get(), plan.rows.get(), nw, rp_w, ci_w, rp_o,
                                                   wins, c2.get(), rw.get(), ro.get());
  RB_LAUNCH_CHECK();
  PinnedBuf<int32_t> hc2;  // the run lengths, for the host layout
  hc2.alloc(static_cast<std::size_t>(runs));
  RB_CUDA(cudaMemcpyAsync(hc2.get(), c2.get(), sizeof(int32_t) * runs, cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  tr.mark("    counts");
  // tiles, slot orders and metadata (slab_layout.cpp)
  const int ecap = (std::min(32736, std::max(256, env_int("RAPDHG_SLAB_TILE", kSlabTileCap))) + 31) & ~31;
  int order_mode = 0;
  if (const char* mode = std::getenv("RAPDHG_SLAB_ORDER")) order_mode = std::string(mode) == "sorted" ? 2 : 1;
  SlabLayout lay;
  PinnedBuf<uint16_t> hm;  // the metadata, written by the layout straight into pinned upload staging
  const bool fits = slab_layout(hc2.get(), nw, S, ecap, kSlabRowCap, order_mode,
                                env_int("RAPDHG_SLAB_ROWCOST", kSlabRowCost), lay, [&](std::size_t n) {
                                  hm.alloc(n);
                                  return hm.get();
                                });
  tr.mark("    layout (host)");
  if (!fits || lay.max_tile > ecap || lay.max_meta > kSlabMetaCap) {  // int32 offsets; tiles must fit a stage
    plan = SlabPlan{};
    return;
  }
  const int32_t ntiles = static_cast<int32_t>(lay.tiles.size());
  const int64_t cursor = lay.entries;
  const bool sorted = lay.sorted;
  plan.tile_bytes = lay.tile_bytes;
  const int64_t total = std::max<int64_t>(cursor, 32);
  {
    plan.meta.alloc(lay.meta_size());
    plan.meta.upload(hm.get(), lay.meta_size(), st);
    plan.tile.alloc(lay.tiles.size());
    plan.tile.upload(lay.tiles.data(), lay.tiles.size(), st);
    plan.col.alloc(total), plan.pos.alloc(total), plan.val.alloc(total);
    RB_CUDA(cudaMemsetAsync(plan.col.get(), 0, sizeof(uint16_t) * total, st));
    RB_CUDA(cudaMemsetAsync(plan.pos.get(), 0xff, sizeof(int32_t) * total, st));  // padding: pos -1 -> 0.0
    if (ntiles)
      tile_fill_kernel<<<static_cast<unsigned>(ntiles), 256, 0, st>>>(plan.tile.get(), plan.meta.get(),
                                                                      plan.rows.get(), rp_w, ci_w, wins,
                                                                      plan.col.get(), plan.pos.get());
    RB_LAUNCH_CHECK();
    RB_CUDA(cudaStreamSynchronize(st));  // the pinned staging is released below
  }
  // rest CSRs keep the op's segment order: rest1 = segment 1, rest2 = segment 2
  DevBuf<int32_t>& rrp_w = seg == 0 ? plan.rrp1 : plan.rrp2;
  DevBuf<int32_t>& rci_w = seg == 0 ? plan.rci1 : plan.rci2;
  DevBuf<int32_t>& rpos_w = seg == 0 ? plan.rpos1 : plan.rpos2;
  DevBuf<int32_t>& rrp_o = seg == 0 ? plan.rrp2 : plan.rrp1;
  DevBuf<int32_t>& rci_o = seg == 0 ? plan.rci2 : plan.rci1;
  DevBuf<int32_t>& rpos_o = seg == 0 ? plan.rpos2 : plan.rpos1;
  const int32_t nrw = scan_dev(rw.get(), nw, rrp_w, st), nro = scan_dev(ro.get(), nw, rrp_o, st);
  rci_w.alloc(nrw), rpos_w.alloc(nrw), rci_o.alloc(nro), rpos_o.alloc(nro);
  (seg == 0 ? plan.rval1 : plan.rval2).alloc(nrw);
  (seg == 0 ? plan.rval2 : plan.rval1).alloc(nro);
  rest_fill_kernel<<<g1(nw), 256, 0, st>>>(plan.rows.get(), nw, rp_w, ci_w, rp_o, ci_o, wins, rrp_w.get(),
                                           rci_w.get(), rpos_w.get(), rp_o ? rrp_o.get() : nullptr, rci_o.get(),
                                           rpos_o.get());
  RB_LAUNCH_CHECK();
  tr.mark("    upload + fill");
  plan.partial.alloc(runs);
  plan.partial.zero(st);  // (window, row) pairs without entries keep 0
  plan.widx.alloc(nr);  // on the device from the W rows (no host arrays of nr entries)
  RB_CUDA(cudaMemsetAsync(plan.widx.get(), 0xff, sizeof(int32_t) * nr, st));  // -1: no partials
  plan.wrow.alloc(nw);
  wrow_kernel<<<g1(nw), 256, 0, st>>>(plan.rows.get(), nw, r0, plan.widx.get(), plan.wrow.get());
  RB_LAUNCH_CHECK();
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
                   for (int64_t q = 0; q < runs; ++q) t += hc2[q];
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
  // the rows without partials: a rowwise schedule; RAPDHG_SELL_OTHERS=1 puts
  // the short ones (<= kSellMaxLen entries, a per-row rule, so shards agree)
  // on sliced ELL instead — measured neutral (C4 +0.6%, C3 -0.8%, C2 -2%:
  // these rows overlap the slab kernel either way), so off by default
  const char* so = std::getenv("RAPDHG_SELL_OTHERS");
  const bool sell = sell_enabled() && so && so[0] == '1';
  if (!sell) {  // the list on the device (C4's dual: 1e6 of 2e6 rows; no host round trip)
    DevBuf<uint8_t> flag(nr);
    others_flag_kernel<<<g1(nr), 256, 0, st>>>(ph.plan.widx.get(), nr, flag.get());
    RB_LAUNCH_CHECK();
    DevBuf<int32_t> list(nr), cnt(1);
    const thrust::counting_iterator<int32_t> idx(0);
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx, flag.get(), list.get(), cnt.get(), nr, st));
    DevBuf<unsigned char> tmp(tb);
    RB_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, idx, flag.get(), list.get(), cnt.get(), nr, st));
    int32_t no = 0;
    RB_CUDA(cudaMemcpyAsync(&no, cnt.get(), sizeof(no), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    if (no > 0) build_schedule(ph.others, len, no, false, st, list.get());
    RB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  const std::vector<int32_t> widx = download(ph.plan.widx, nr, st);
  const std::vector<int32_t> hlen = download_len(len, nr, st);
  std::vector<int32_t> orr, osh;
  for (int32_t i = 0; i < nr; ++i)
    if (widx[i] < 0) (sell && hlen[i] <= kSellMaxLen ? osh : orr).push_back(i);
  if (!orr.empty()) {
    DevBuf<int32_t> d(orr.size());
    d.upload(orr.data(), orr.size(), st);
    build_schedule(ph.others, len, static_cast<int64_t>(orr.size()), false, st, d.get());
  }
  if (!osh.empty()) {
    DevBuf<int32_t> d(osh.size());
    d.upload(osh.data(), osh.size(), st);
    build_sell_plan(ph.others_sell, rp1 ? rp1 + r0 : nullptr, ci1, rp2 ? rp2 + r0 : nullptr, ci2,
                    static_cast<int32_t>(osh.size()), st, d.get());
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
