// slab.cuh — window-tiled SpMV with the gathered vector staged in shared
// memory (fast mode).
//
// Why: a random fp64 gather touches its own 128 B line and the L1TEX tag stage
// retires ~1 line per cycle per SM, so a gather-heavy SpMV is bound at ~1
// gather/cycle/SM (C2: 1e7 gathers = 34 us) long before HBM. Shared memory
// serves a warp's 32 random 8 B reads in a few wavefronts, so reading the
// gathered vector from smem removes that bound whenever enough gathers land in
// a column range to repay staging it.
//
// Layout (slab.cu): the columns of one segment of the op's pattern are cut
// into aligned windows of kSlabWidth columns; windows receiving
// >= kSlabMinDensity gathers per column are kept (at most kMaxSlabs). "W rows"
// (>= kSlabMinRow in-window entries, every run and the rest <= kSlabRunCap)
// are cut into chunks so that each (chunk j, window s) tile fits one shared-
// memory stage. Inside a tile the chunk's rows are sorted by their run length
// in window s and grouped into slices of 32 rows, one row per lane; a slice
// stores its entries as jagged diagonals (entry e of the rows whose run is
// longer than e, contiguous; no padding; 16-bit column offsets + fp64 values,
// 10 B/nnz), so a warp reads its values and columns contiguously and only the
// window gather is random. Each W row also
// has a "rest" CSR: its entries outside the windows and its other segment.
//
// slab_kernel is persistent (2 CTAs per SM), double-buffered and warp-
// specialised: a producer warp bulk-copies (cp.async.bulk, mbarrier
// complete_tx) the next tile's window slice, values, columns and slice
// metadata into the free stage while 8 consumer warps compute the current
// tile from shared memory, writing one partial per (window, row). Then the finish pass (SlabFinishOp through rowwise_kernel)
// runs over all rows of the op: a W row sums its rest entries and its S
// partials, a non-W row is the op's own row, and both run the op's epilogue.
// A row's arithmetic depends only on the windows and its own entries (each
// window run is summed sequentially in column order) — not on chunking,
// slicing, tile order or CTA — so results are deterministic and a sharded
// solve that reuses the global windows stays bit-identical.
#pragma once

#include <cstdint>
#include <vector>

#include "ops.cuh"
#include "slab_layout.hpp"
#include "sell.cuh"

namespace rb {

constexpr int kMaxSlabs = 1024;     // windows per op (in device memory)
constexpr int64_t kSlabMaxRuns = int64_t{16} << 20;  // (window, W row) pairs per plan
constexpr int kSlabWidth = 2048;        // columns per window (16 KB of fp64)
constexpr int kSlabMinRow = 16;         // in-window entries that make a W row
constexpr double kSlabMinDensity = 16;  // gathers per column that keep a window
constexpr int kSlabTileCap = 2816;      // entries per tile (28 KB staged)
#ifndef RB_SLAB_STAGES
#define RB_SLAB_STAGES 3
#endif
constexpr int kSlabStages = RB_SLAB_STAGES;  // tile stages per CTA (one shared window)
constexpr int kSlabRowCap = 512;        // rows per chunk
constexpr int kSlabRunCap = 512;        // W rows: every window run and the rest <= this
constexpr int kSlabMinWindows = 1;     // RAPDHG_SLAB_MIN_WINDOWS overrides
constexpr int kSlabResidentMax = 8;    // resident plans: at most this many windows (128 KB) staged at once
constexpr int kSlabProf = 10;           // per-CTA profile slots (RB_SLAB_PROFILE)

// SlabTile (slab_layout.hpp): tile t, window-major (a CTA's contiguous tile
// range mostly shares one window, staged once)

// Per-tile metadata (uint16 elements): perm (uint32 W-row index per slot, 2
// elements each) | len[nr] (run length per slot) | soff[nsl + 1] (slice
// starts, entries relative to the tile). Lane l's entry e of slice q sits at
// soff[q] + 32 e + l. A window's tiles hold its W rows sorted by their run
// length there, so the 32 rows of a slice have nearly equal runs (≈ no
// padding) whatever the window.
constexpr int kSlabRowCost = 0;          // CTA balance: cost per tile row, in staged-byte units
constexpr int kSlabGroupedS = 16;        // finish: 8 warps share a row's partials from this many windows
constexpr double kSlabNaturalPad = 1.12;  // natural row order unless its slices pad more than this
constexpr int kSlabMetaCap = 3 * kSlabRowCap + kSlabRowCap / 32 + 8;  // per tile (multiple of 8)
struct SlabView {
  int32_t nw = 0;                  // W rows
  int32_t S = 0;                   // windows (even lengths)
  int32_t J = 0;                   // tiles
  int32_t seg = 0;                 // accumulator the windows feed (0: segment 1, 1: segment 2)
  int32_t win_max = 0;             // widest window (doubles, even)
  int32_t ecap = 0;                // tile entry capacity (multiple of 8)
  int32_t mcap = 0;                // tile metadata capacity (multiple of 8)
  int32_t grid = 0;                // persistent CTAs
  int32_t wfirst = 0;              // finish grid: W-row blocks first (launch_slab_phase)
  int32_t resident = 0;            // > 0: that many windows staged at once (window s at s * win_max / resident);
                                   // W rows are one run and finish in the slab kernel (no partials)
  const Window* win = nullptr;     // [S] (device)
  const SlabTile* tile = nullptr;   // [J]
  const int32_t* cta = nullptr;     // [grid + 1] tile ranges per CTA (balanced by bytes)
  const uint16_t* meta = nullptr;   // per-tile metadata
  const uint16_t* col = nullptr;    // column offset inside the window
  const double* val = nullptr;
  double* partial = nullptr;        // [S * nw] (window-major: a tile's partials are contiguous)
  const int32_t* wrow = nullptr;    // [nw] W rows' ids relative to the op's row base
  CsrView rest1{}, rest2{};         // rest CSRs over W rows (segment 1 / 2)
  unsigned long long* prof = nullptr;  // [grid * kSlabProf] phase times (RB_SLAB_PROFILE builds)
  unsigned long long* fprof = nullptr; // [4] finish kernel: max end of other rows, min/max W wait done, max W end
  unsigned long long* span = nullptr;  // [2 kMaxChunk] in-loop timing: step start (%globaltimer, min over CTAs)
  bool active() const { return nw > 0 && S > 0; }
  __host__ __device__ int tiles() const { return J; }
  // stage: [header 16 B][window][values][columns][metadata]
  // smem: [window][stage 0] .. [stage kSlabStages - 1];
  // stage: [header 16 B][values][columns][metadata]
  __host__ __device__ int stage_bytes() const { return 16 + ecap * 10 + mcap * 2; }
  int smem_bytes() const;
};

// Device arrays behind a SlabView (built by build_slab_plan).
struct SlabPlan {
  SlabView view;
  DevBuf<int32_t> rows, pos, wrow, widx, lut;
  DevBuf<Window> win;
  DevBuf<SlabTile> tile;
  DevBuf<int32_t> cta;
  std::vector<int64_t> tile_bytes;  // host: bytes each tile stages
  DevBuf<uint16_t> col, meta;
  DevBuf<double> val, partial;
  DevBuf<int32_t> rrp1, rci1, rpos1, rrp2, rci2, rpos2;  // rest CSRs (pos = source position)
  DevBuf<double> rval1, rval2;
  DevBuf<unsigned long long> prof;
};

// Which windows a matrix segment gets: chosen once on the whole matrix, reused
// unchanged for every shard so per-row arithmetic agrees.
struct SlabChoice {
  std::vector<Window> windows;  // each starts at a multiple of width
  int width = kSlabWidth;
  bool empty() const { return windows.empty(); }
};

// Windows over the columns of `m` (device CSR arrays, rows x ncols).
// RAPDHG_SLAB=off disables; =force keeps every non-empty window and W rows
// with a single in-window entry (tests reach the path at small sizes).
SlabChoice choose_slabs(const int32_t* rp, const int32_t* ci, int32_t rows, int64_t nnz,
                        int32_t ncols, cudaStream_t st);

// Plan for rows [r0, r1) of the two-segment pattern (seg1 = rp1/ci1, may be
// null; seg2 = rp2/ci2); the windows apply to segment `seg` (0 or 1). The
// other segment goes entirely to the rest CSR. The op's rows are numbered
// relative to r0 (a shard's ops index its slice); r0 = 0 on one GPU.
void build_slab_plan(SlabPlan& plan, const SlabChoice& choice, int seg, const int32_t* rp1,
                     const int32_t* ci1, const int32_t* rp2, const int32_t* ci2, int32_t r0,
                     int32_t r1, cudaStream_t st);

// (Re)fill the plan's values from value arrays laid out like seg1 / seg2.
void fill_slab_values(SlabPlan& plan, const double* v1, const double* v2, cudaStream_t st);


// Persistent grid for the slab kernel at this smem size.
int slab_grid(const void* kernel, int smem_bytes);

// ---- kernel -----------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One-shot mbarrier + 1-D bulk copies (TMA engine): global -> shared.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {  // no arrival
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Streamed once: evict-first in L2, so the tiles do not displace the iterate
// vectors the other kernels of the step gather.
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
}

// Producer, in two parts so the entries of the first tiles can be in flight
// before the previous kernel of the step has finished (they do not depend on
// it): slab_entries bulk-copies tile d's values, columns and metadata into the
// stage at `base` and announces their bytes; slab_commit adds the window when
// it changes and arrives, completing the stage's phase. The header is
// published to the consumers by the mbarrier.
__device__ __forceinline__ void slab_entries(const SlabView& sv, const SlabTile& d, unsigned char* base,
                                             uint64_t* bar) {
  int32_t* hdr = reinterpret_cast<int32_t*>(base);
  double* val = reinterpret_cast<double*>(base + 16);
  uint16_t* col = reinterpret_cast<uint16_t*>(val + sv.ecap);
  uint16_t* meta = col + sv.ecap;
  const uint32_t m8 = static_cast<uint32_t>(d.m + 7) & ~7u;
  hdr[0] = 0;
  hdr[1] = d.nr;
  hdr[2] = d.s;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic accesses of the buffers before
  mbar_expect_tx_only(bar, static_cast<uint32_t>(d.n) * 10u + m8 * 2u);
  if (d.n) {
    bulk_g2s_stream(val, sv.val + d.a, static_cast<uint32_t>(d.n) * 8u, bar);
    bulk_g2s_stream(col, sv.col + d.a, static_cast<uint32_t>(d.n) * 2u, bar);
  }
  bulk_g2s_stream(meta, sv.meta + d.meta, m8 * 2u, bar);
}
template <class Op>
__device__ __forceinline__ void slab_commit(const Op& op, const SlabView& sv, const SlabTile& d, double* win,
                                            uint64_t* bar, bool copy_window) {
  if (sv.resident) {  // the whole image, once (window s at s * stride)
    const int stride = sv.win_max / sv.resident;
    uint32_t bytes = 0;
    if (copy_window)
      for (int s = 0; s < sv.resident; ++s) bytes += static_cast<uint32_t>(sv.win[s].len) * 8u;
    mbar_expect_tx(bar, bytes);
    if (copy_window)
      for (int s = 0; s < sv.resident; ++s) {
        const Window w = sv.win[s];
        bulk_g2s(win + s * stride, op.gather_src(sv.seg) + w.lo, static_cast<uint32_t>(w.len) * 8u, bar);
      }
    return;
  }
  const Window w = copy_window ? sv.win[d.s] : Window{};
  const uint32_t wbytes = static_cast<uint32_t>(w.len) * 8u;
  mbar_expect_tx(bar, wbytes);  // arrive (+ the window's bytes)
  if (wbytes) bulk_g2s(win, op.gather_src(sv.seg) + w.lo, wbytes, bar);
}

#ifdef RB_SLAB_PROFILE
// per-CTA phase times (thread 0, %globaltimer ns): [0] start, [2] waiting for
// copies, [3] tile compute, [6] end, [7] tiles
__device__ __forceinline__ unsigned long long slab_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SLAB_T(var) const unsigned long long var = threadIdx.x == 0 && sv.prof ? slab_now() : 0ull
#define SLAB_ADD(slot, v) \
  if (threadIdx.x == 0 && sv.prof) sv.prof[blockIdx.x * kSlabProf + (slot)] += (v)
#define SLAB_SET(slot, v) \
  if (threadIdx.x == 0 && sv.prof) sv.prof[blockIdx.x * kSlabProf + (slot)] = (v)
#else
#define SLAB_T(var)
#define SLAB_ADD(slot, v)
#define SLAB_SET(slot, v)
#endif

constexpr int kSlabConsumers = 8;                        // consumer warps
constexpr int kSlabThreads = 32 * (kSlabConsumers + 1);  // + one producer warp

// Warp-specialised: warp kSlabConsumers (lane 0) bulk-copies tiles into
// kSlabStages stages (full barrier: bytes landed) and, when a tile's window
// differs from the one held, first waits until every issued tile is consumed
// and then reloads the shared window with it; the consumer warps wait for a
// stage, take every kSlabConsumers-th slice of it (dealt on a counter that
// runs across tiles, so the warps share the work evenly without a CTA-wide
// barrier) and arrive on the stage's empty barrier when done.
template <class Op>
__global__ void __launch_bounds__(kSlabThreads) slab_kernel(const Op op, const SlabView sv) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kSlabStages], empty[kSlabStages];
  // power-iteration batches past the stop (uniform over the grid; the gate
  // was written by an earlier, completed grid)
  if (HasGate<Op>::closed(op)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* win = reinterpret_cast<double*>(smem_raw);
  unsigned char* stages = smem_raw + sv.win_max * 8;
  const int sb = sv.stage_bytes();
  SLAB_T(t_start);
#ifdef RB_SLAB_PROFILE
  if (threadIdx.x == 0 && sv.prof)
    for (int q = 0; q < kSlabProf; ++q) sv.prof[blockIdx.x * kSlabProf + q] = 0ull;
  if (threadIdx.x == 0 && blockIdx.x == 0 && sv.fprof) {
    sv.fprof[0] = 0ull, sv.fprof[1] = ~0ull, sv.fprof[2] = 0ull, sv.fprof[3] = 0ull;
    __threadfence();
  }
#endif
  SLAB_SET(0, t_start);
  if (threadIdx.x == 0)
    for (int q = 0; q < kSlabStages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kSlabConsumers);
    }
  __syncthreads();  // barriers initialised
  // this CTA's tiles: a contiguous range of the window-major tile order, so
  // consecutive tiles mostly share their window
  const int t0 = sv.cta[blockIdx.x], t1 = sv.cta[blockIdx.x + 1];
  if (warp == kSlabConsumers) {  // producer
    if (lane == 0) {
      // This launch may start while the previous kernel of the step still
      // runs (programmatic dependent launch): the entries of the first tiles
      // sharing the first window go out at once; the window (written by the
      // previous kernels) only after griddepcontrol.wait. Consumers cannot
      // pass stage 0 before its window lands, so everything they do follows
      // the previous kernels.
      SlabTile pend[kSlabStages];
      int pre = 0;
      if (t0 < t1) {
        SlabTile d = sv.tile[t0];
        while (true) {
          pend[pre] = d;
          slab_entries(sv, d, stages + pre * sb, &full[pre]);
          ++pre;
          if (pre == kSlabStages || t0 + pre >= t1) break;
          d = sv.tile[t0 + pre];
          if (d.s != pend[0].s) break;
        }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      // the finish kernel may launch once every CTA is past the wait (so its
      // rows without partials see this step's inputs complete)
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      if (sv.span) {  // in-loop timing: the step starts when its inputs are complete
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        atomicMin(&sv.span[2 * op.it + Op::kPhase], now);
      }
      int held = -1;  // window in the shared buffer
      for (int q = 0; q < pre; ++q) {
        slab_commit(op, sv, pend[q], win, &full[q], q == 0);
        held = pend[0].s;
      }
      if (t0 + pre < t1) {
        SlabTile d = sv.tile[t0 + pre];
        for (int t = t0 + pre, i = pre; t < t1; ++t, ++i) {
          const int st = i % kSlabStages;
          const SlabTile cur = d;
          if (t + 1 < t1) d = sv.tile[t + 1];  // prefetch the next descriptor
          if (i >= kSlabStages) mbar_wait(&empty[st], (i / kSlabStages - 1) & 1);  // stage free
          const bool change = cur.s != held;
          if (change && held >= 0)  // drain: the tiles in flight still read the old window
            for (int q = 1; q < kSlabStages && i - q >= 0; ++q) {
              const int p = i - q;
              mbar_wait(&empty[p % kSlabStages], (p / kSlabStages) & 1);
            }
          slab_entries(sv, cur, stages + st * sb, &full[st]);
          slab_commit(op, sv, cur, win, &full[st], change);
          held = cur.s;
        }
      }
    }
    return;
  }
  int i = 0, deal = 0;  // deal: slices dealt so far, mod kSlabConsumers
  for (int t = t0; t < t1; ++t, ++i) {
    const int st = i % kSlabStages;
    const unsigned char* base = stages + st * sb;
    SLAB_T(t_w0);
    mbar_wait(&full[st], (i / kSlabStages) & 1);
    SLAB_T(t_w1);
    SLAB_ADD(2, t_w1 - t_w0);
    SLAB_ADD(7, 1);
    const int32_t* hdr = reinterpret_cast<const int32_t*>(base);
    const int nr = hdr[1], s = hdr[2];
    const double* val = reinterpret_cast<const double*>(base + 16);
    const uint16_t* col = reinterpret_cast<const uint16_t*>(val + sv.ecap);
    const uint32_t* perm = reinterpret_cast<const uint32_t*>(col + sv.ecap);
    const uint16_t* len = reinterpret_cast<const uint16_t*>(perm + nr);
    const uint16_t* soff = len + nr;
    double* partial = sv.partial + static_cast<int64_t>(s) * sv.nw;
    const int nsl = (nr + 31) >> 5;
    for (int q = (warp - deal + kSlabConsumers) % kSlabConsumers; q < nsl; q += kSlabConsumers) {
      const int slot = (q << 5) + lane;
      const int L = slot < nr ? len[slot] : 0;
      // resident: this lane's row finishes here; its epilogue inputs are
      // requested before the tile's entries so their latency overlaps
      int r = 0;
      typename Op::Pre pre{};
      if (sv.resident && slot < nr) {
        r = sv.wrow[perm[slot]];
        pre = op.prefetch(r);
      }
      const int Lm = len[q << 5];  // the slice's longest run (lane 0: sorted)
      const double* vq = val + soff[q] + lane;
      const uint16_t* cq = col + soff[q] + lane;
      double part = 0.0;
      for (int e = 0; e < Lm; e += 4) {
        double v[4], x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = L > e + u;
          v[u] = ok ? vq[(e + u) << 5] : 0.0;
          x[u] = ok ? win[cq[(e + u) << 5]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) part = fma(v[u], x[u], part);
      }
      if (sv.resident) {  // the row's entries outside the windows, then the epilogue
        if (slot < nr) {
          const int k = static_cast<int>(perm[slot]);
          const Op rest = op.with_views(sv.rest1, sv.rest2);
          const Gather gl[2] = {Gather{rest.gather_src(0), nullptr, 0, 0u}, Gather{rest.gather_src(1), nullptr, 0, 0u}};
          typename Op::AccT a;
          a.zero();
          rest.template accumulate<kUnroll>(k, 0, rest.len(k), 0, 1, a, gl);
          if (sv.seg == 0) a.v[0] += part;
          else a.v[Op::AccT::kK - 1] += part;
          op.finish(r, a, pre);
        }
      } else if (slot < nr) {
        partial[perm[slot]] = part;
      }
    }
    deal = (deal + nsl) % kSlabConsumers;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done reading the stage (and the window)
    SLAB_T(t_c1);
    SLAB_ADD(3, t_c1 - t_w1);
  }
  SLAB_T(t_end);
  SLAB_SET(6, t_end);
#ifdef RB_SLAB_PROFILE
  if (threadIdx.x == 0 && sv.prof) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    sv.prof[blockIdx.x * kSlabProf + 8] = smid;
  }
#endif
}

inline int SlabView::smem_bytes() const { return win_max * 8 + kSlabStages * stage_bytes(); }

// The rows of Op after the slab kernel, one launch (a programmatic dependent
// launch of the slab kernel):
//  * the last wblocks blocks: W rows, 32 per block — epilogue inputs and the
//    rest entries before the wait, then the S window partials (warp g sums
//    windows g, g + 8, ..., the 8 sums added in order), then the epilogue;
//    the per-row order depends only on S, so results are deterministic and
//    shard-invariant;
//  * the first blocks: ordinary rowwise tiles of the rows without partials
//    (no wait: they overlap the slab kernel; scheduled first so the waiting
//    W blocks do not hold SM slots while the slab kernel still runs).
// Visibility of the rows without partials: they gather vectors written two
// grids earlier (the previous step's finish kernel F). This grid is launched
// only once every CTA of the slab kernel S between them has triggered, and
// S's CTAs trigger after their own griddepcontrol.wait on F returned, so F
// has completed and its writes have been flushed to L2 before any block here
// starts. PTX promises visibility of F's writes only to S, so this relies on
// the flush at F's completion reaching every later reader (and on no stale L1
// line surviving into this grid); the GPU tests (test_gpu_slab.py) hold this
// schedule to the fully serialised one (RAPDHG_PDL=0) bit for bit over
// thousands of steps at the bench's size.
template <class Op>
__global__ void __launch_bounds__(kBlock) slab_finish_kernel(const Op op, const Op rest, const SlabView sv,
                                                             const SchedView others, int wblocks,
                                                             const SellView osell) {
  if (HasGate<Op>::closed(op)) return;  // see slab_kernel
  // the next kernel (the next slab kernel, a programmatic dependent launch)
  // may start prefetching its tiles; it waits for this grid before using y / w
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int ob = others.total_blocks > 0 ? others.total_blocks : 0;
  const int sb = static_cast<int>((osell.nslices + kBlock / 32 - 1) / (kBlock / 32));
  // block order: others, SELL slices, W rows — or (wfirst) the W-row blocks
  // first, so they are resident and have loaded their rest entries and
  // epilogue inputs when the slab grid completes (the arithmetic per row is
  // the same either way)
  int bid = static_cast<int>(blockIdx.x);
  if (sv.wfirst) bid = bid < wblocks ? ob + sb + bid : bid - wblocks;
  if (bid < ob) {  // the rows without partials (they start at once)
    const Gather g[2] = {Gather{op.gather_src(0), nullptr, 0, 0u}, Gather{op.gather_src(1), nullptr, 0, 0u}};
    rowwise_tile(op, others, bid, g);
#ifdef RB_SLAB_PROFILE
    if (threadIdx.x == 0 && sv.fprof) atomicMax(&sv.fprof[0], slab_now());
#endif
    return;
  }
  if (bid < ob + sb) {  // the short ones of them: sliced ELL, a slice per warp
    const int64_t q = static_cast<int64_t>(bid - ob) * (kBlock / 32) + (threadIdx.x >> 5);
    if (q < osell.nslices) sell_slice(op, osell, q, threadIdx.x & 31);
    return;
  }
  if (sv.resident) {  // W rows finished in the slab kernel: one block only waits for it, so
    // this grid completes after the slab grid (the next step's wait is transitive)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  // last: the W rows, whose blocks wait for the slab grid. The epilogue
  // inputs and the rest entries (independent of the slab kernel) are loaded
  // and summed before the wait. With many windows (S >= kSlabGroupedS) a
  // block takes 32 rows and warp g sums the partials of windows g, g + 8, ...
  // (one round of independent loads; warp 0 adds the 8 sums in order); with
  // few, a thread takes one row and sums its S partials in order.
  const bool grouped = sv.S >= kSlabGroupedS;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int wb = bid - ob - sb;  // W-row block
  const int k = grouped ? wb * 32 + lane : wb * kBlock + threadIdx.x;
  const bool valid = k < sv.nw;
  const bool owner = valid && (!grouped || g == 0);  // runs the row's epilogue
  typename Op::AccT a;
  a.zero();
  typename Op::Pre pre{};
  int r = 0;
  if (owner) {
    r = sv.wrow[k];
    pre = op.prefetch(r);
    const Gather gl[2] = {Gather{rest.gather_src(0), nullptr, 0, 0u}, Gather{rest.gather_src(1), nullptr, 0, 0u}};
    rest.template accumulate<kUnroll>(k, 0, rest.len(k), 0, 1, a, gl);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the slab kernel's partials are complete
#ifdef RB_SLAB_PROFILE
  if (threadIdx.x == 0 && sv.fprof) {
    const unsigned long long t = slab_now();
    atomicMin(&sv.fprof[1], t);
    atomicMax(&sv.fprof[2], t);
  }
#endif
  double tot = 0.0;
  if (grouped) {
    __shared__ double grp[kBlock / 32][32];
    constexpr int G = kBlock / 32;
    double t = 0.0;
    if (valid)
      for (int s0 = g; s0 < sv.S; s0 += 8 * G) {  // windows g, g + G, ... in order, 8 loads in flight
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int s = s0 + u * G;
          v[u] = s < sv.S ? __ldcg(sv.partial + static_cast<int64_t>(s) * sv.nw + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) t += v[u];
      }
    grp[g][lane] = t;
    __syncthreads();
    if (!owner) return;
    tot = grp[0][lane];
#pragma unroll
    for (int q = 1; q < G; ++q) tot += grp[q][lane];
  } else {
    if (!owner) return;
    const double* p = sv.partial + k;
    int q = 0;
    for (; q + 8 <= sv.S; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + static_cast<int64_t>(q + u) * sv.nw);
#pragma unroll
      for (int u = 0; u < 8; ++u) tot += v[u];
    }
    for (; q < sv.S; ++q) tot += __ldcg(p + static_cast<int64_t>(q) * sv.nw);
  }
  if (sv.seg == 0) a.v[0] += tot;
  else a.v[Op::AccT::kK - 1] += tot;
  op.finish(r, a, pre);
#ifdef RB_SLAB_PROFILE
  if (sv.fprof) atomicMax(&sv.fprof[3], slab_now());
#endif
}

// Raise the dynamic smem limit of the slab kernel of Op (once, outside stream
// capture) and return the persistent grid for that smem size.
template <class Op>
inline int prepare_slab(int smem_bytes) {
  const void* k = reinterpret_cast<const void*>(&slab_kernel<Op>);
  RB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  return slab_grid(k, smem_bytes);
}

// A slab-tiled op: the plan and the finish schedule over all of its rows.
struct SlabPhase {
  SlabPlan plan;
  Schedule others;     // rows without partials (the op's own rows) longer than kSellMaxLen
  SellPlan others_sell;  // the short ones, sliced ELL (sell.cuh); RAPDHG_SELL=0: all in `others`
  bool active() const { return plan.view.active(); }
};

// Plan + finish schedule for rows [r0, r1) of the op (see build_slab_plan);
// `len`: the op's row lengths for those rows. Leaves `ph` inactive when there
// are no W rows.
void build_slab_phase(SlabPhase& ph, const SlabChoice& choice, int seg, const int32_t* rp1, const int32_t* ci1,
                      const int32_t* rp2, const int32_t* ci2, int32_t r0, int32_t r1, const int32_t* len,
                      cudaStream_t st);

// Per-CTA contiguous tile ranges for `grid` persistent CTAs, balanced by the
// bytes each tile stages (after the grid is known).
void assign_slab_ctas(SlabPlan& plan, int grid, cudaStream_t st);

// One slab-tiled op: the slab kernel, then the finish kernel as a programmatic
// dependent launch (rows without partials start while the slab kernel runs;
// W rows wait for it). Returns kernels launched.
// RAPDHG_PDL=0: launch the slab and finish kernels without programmatic
// stream serialization (every kernel waits for the previous grid; the
// griddepcontrol instructions become no-ops). Results must not change: the
// tests compare both schedules bit for bit (see slab_finish_kernel).
inline bool pdl_enabled() {  // read per launch (launches are captured into graphs once)
  const char* e = std::getenv("RAPDHG_PDL");
  return !(e && e[0] == '0');
}

template <class Op>
inline int launch_slab_phase(const Op& op, const SlabPhase& ph, cudaStream_t st,
                             unsigned long long* span = nullptr) {
  SlabView sv = ph.plan.view;
  const unsigned pdl = pdl_enabled() ? 1u : 0u;
  sv.span = span;
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(sv.grid));
    cfg.blockDim = dim3(kSlabThreads);
    cfg.dynamicSmemBytes = static_cast<std::size_t>(sv.smem_bytes());
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RB_CUDA(cudaLaunchKernelEx(&cfg, slab_kernel<Op>, op, sv));
  }
  const SchedView& o = ph.others.view;
  const SellView& osell = ph.others_sell.view;
  const int wblocks = sv.resident ? 1 : static_cast<int>(ceil_div(sv.nw, sv.S >= kSlabGroupedS ? 32 : kBlock));
  const int sblocks = static_cast<int>(ceil_div(osell.nslices, kBlock / 32));
  {  // W-row blocks first when they fit two per SM (C3's dual: 32 blocks, step 62 -> 55 us; with
     // more of them, e.g. C4's 3,907 + 313, they would hold the SMs idle in their wait while the
     // rows without partials queue behind them: C4 129 -> 140 us). RAPDHG_FINISH_WFIRST=0|1 forces.
    const char* e = std::getenv("RAPDHG_FINISH_WFIRST");  // per launch (graphs capture it once)
    sv.wfirst = e && (e[0] == '0' || e[0] == '1') ? e[0] == '1' : wblocks <= 2 * kSMs;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(wblocks + sblocks + (o.total_blocks > 0 ? o.total_blocks : 0)));
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RB_CUDA(cudaLaunchKernelEx(&cfg, slab_finish_kernel<Op>, op, op.with_views(sv.rest1, sv.rest2), sv, o, wblocks,
                             osell));
  return 2;
}

}  // namespace rb
