// rowwise.cuh — the one SpMV engine behind every sparse product on the path.
//
// Every hot operation of the rAPDHG iteration is a row gather over a CSR
// matrix (or over the horizontal concatenation [Q | A'] of two CSRs sharing a
// row index) followed by a per-row epilogue: the dual step (A*w then the
// projected dual update, solver.hpp:164-167,178), the primal step (Q*x_md and
// A'*y then the gradient step and averages, solver.hpp:169-177) and the KKT
// products (kkt.hpp:32-39). rowwise_kernel<Op> runs any such "Op" with:
//
//  * a length-binned schedule: rows are grouped by nnz (SURVEY §7 hard part 1:
//    C3 has a 1e6-nnz row next to 1e6 singleton rows) and each bin uses
//    V = 1,2,4,...,32 lanes per row, a whole 256-thread block per row, or —
//    for rows longer than kSplitLen — several blocks per row whose partial
//    sums are combined by the last-arriving block in a FIXED order;
//  * deterministic reductions: a row's sum depends only on its length (which
//    fixes V) — never on timing — so every run is bit-reproducible (SPEC AC10)
//    without float atomics;
//  * a strict mode (Op::kStrict) with one thread per row summing sequentially
//    from +0.0 in CSR order with round-to-nearest mul/add and no FMA: that is
//    exactly sparse.hpp:84-86, so results are bit-identical to the reference.
//
// One launch covers all bins (the block index selects the bin), so each SpMV
// is one kernel node in the per-chunk CUDA graph.
#pragma once

#include <type_traits>

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace rb {

constexpr int kBlock = 256;
constexpr int kNumVBins = 6;      // V = 1,2,4,8,16,32
constexpr int kBinBlock = 6;      // one block per row
constexpr int kBinSplit = 7;      // several blocks per row
constexpr int kNumBins = 8;
constexpr int kSplitLen = 16384;  // nnz per block in split mode

struct BinDesc {
  int32_t row_begin, row_end;  // slots in perm
  int32_t blk_begin, blk_end;  // blocks of the launch
};

// A window [lo, lo + len) of a gathered vector's index space that the kernel
// stages in shared memory (len = 0: none). Random fp64 gathers through L1TEX
// cost one wavefront (~1 cycle/SM) per distinct 128 B line; from shared memory
// a warp's 32 random 8 B reads cost ~a bank-conflict degree (~4-5 cycles), so
// gathers that land in the window are ~6x cheaper. Chosen per matrix pattern at
// setup from a column histogram (schedule.cu).
struct Window {
  int32_t lo = 0, len = 0;
};

struct SchedView {
  const int32_t* perm;  // row order by bin; nullptr = identity (strict)
  BinDesc bins[kNumBins];
  // split-mode segments (one block each)
  const int32_t* seg_row;
  const int32_t* seg_lo;
  const int32_t* seg_hi;
  const int32_t* seg_first;  // first segment index of the segment's row
  const int32_t* seg_count;  // segments of that row
  double* seg_partial;       // [nseg * kMaxAcc]
  unsigned* seg_ticket;      // [nseg], used at index seg_first
  int32_t total_blocks;      // tiles; the persistent grid strides over them
  Window win[2];             // staged gather windows of segment 1 / 2 columns
};

constexpr int kMaxAcc = 8;

// ---- arithmetic ------------------------------------------------------------
// Strict: product rounded, then sum rounded (no contraction) = the reference's
// `s += v * x` compiled with -ffp-contract=off. Fast: one fused multiply-add.
template <bool Strict>
__device__ __forceinline__ double madd(double acc, double v, double x) {
  if constexpr (Strict)
    return __dadd_rn(acc, __dmul_rn(v, x));
  else
    return fma(v, x, acc);
}

// Streaming loads for matrix data (read once per product: evict-first so the
// gathered vectors keep their L2/L1 lines); read-only cached loads for the
// gathered vectors.
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ double ld_gather(const double* p) { return __ldg(p); }

// K accumulators combined by + (sums) or by max (Max = true, order-free).
template <int K, bool Max = false>
struct Acc {
  static constexpr int kK = K;
  double v[K];
  __device__ __forceinline__ static double comb(double a, double b) { return Max ? fmax(a, b) : a + b; }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = 0.0;
  }
  // Butterfly over the V lanes of a row group (fixed pattern -> deterministic).
  template <int V>
  __device__ __forceinline__ void reduce_lanes() {
#pragma unroll
    for (int off = V / 2; off > 0; off >>= 1)
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = comb(v[k], __shfl_xor_sync(0xffffffffu, v[k], off));
  }
};

constexpr int kUnroll = 4;  // loads in flight per lane (narrow rows, block/split)
// Ops whose long rows (>= 16 lanes) want more loads in flight declare
// kWideUnroll = 8 (costs registers, so only where it measured faster).

// First position >= target in the progression p0, p0 + stride, ... (p0 >= 0).
__device__ __forceinline__ int next_pos(int p0, int stride, int target) {
  return target <= p0 ? p0 : p0 + ((target - p0 + stride - 1) / stride) * stride;
}

// Accumulation of sum_k vals[k] * x[cols[k]] over positions p, p+stride, ...
// < end of one CSR segment (index = base + position). Predicated unroll: all
// kUnroll loads of a lane are issued together even when the lane has fewer
// elements left (short rows keep their memory-level parallelism); inactive
// slots contribute 0*0 = +0, which never changes a sum that started at +0.0
// (such a sum is never -0), so the adds stay in position order and strict
// mode remains the reference's sequential sum exactly.
#ifndef RB_PIPELINE
#define RB_PIPELINE 1
#endif

template <int U>
__device__ __forceinline__ void load_batch(const double* __restrict__ vals,
                                           const int32_t* __restrict__ cols, int64_t base, int p,
                                           int end, int stride, int32_t* c, double* v) {
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const bool ok = p + k * stride < end;
    const int64_t i = base + p + k * stride;
    c[k] = ok ? ld_stream(cols + i) : 0;
    v[k] = ok ? ld_stream(vals + i) : 0.0;
  }
}

// Gathered-vector access: the staged window from shared memory, the rest
// through the read-only path.
struct Gather {
  const double* __restrict__ x;
  const double* sm;
  int32_t lo;
  uint32_t len;
  __device__ __forceinline__ double operator()(int32_t c) const {
    const uint32_t k = static_cast<uint32_t>(c - lo);
    return k < len ? sm[k] : ld_gather(x + c);
  }
};

template <bool Strict, int U = kUnroll>
__device__ __forceinline__ double seg_dot(const double* __restrict__ vals,
                                          const int32_t* __restrict__ cols, const Gather& x,
                                          int64_t base, int p, int end, int stride, double acc) {
  if (p >= end) return acc;
  int32_t c[U];
  double v[U];
  load_batch<U>(vals, cols, base, p, end, stride, c, v);
  for (; p < end; p += U * stride) {
    // Software pipeline: the next batch's indices/values are requested before
    // this batch's gathers, so a lane keeps two batches of streaming loads and
    // one of gathers in flight instead of paying the two round trips in turn.
    int32_t cn[U];
    double vn[U], xv[U];
    if (RB_PIPELINE) load_batch<U>(vals, cols, base, p + U * stride, end, stride, cn, vn);
#pragma unroll
    for (int k = 0; k < U; ++k) xv[k] = (p + k * stride < end) ? x(c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < U; ++k) acc = madd<Strict>(acc, v[k], xv[k]);
    if (!RB_PIPELINE) load_batch<U>(vals, cols, base, p + U * stride, end, stride, cn, vn);
#pragma unroll
    for (int k = 0; k < U; ++k) c[k] = cn[k], v[k] = vn[k];
  }
  return acc;
}

// Two right-hand sides in one pass over the matrix (the relKKT products of the
// current iterate and of the average, kkt.hpp:32-39). With Split, entries
// whose column is < split go to (a[0], a[1]) and the others to (a[2], a[3])
// — the inequality / equality blocks of A'y (kkt.hpp:35-38); otherwise
// a[0] += v*xa, a[1] += v*xb. Same predicated unroll as seg_dot.
template <bool Strict, bool Split, int U = kUnroll>
__device__ __forceinline__ void seg_dot2(const double* __restrict__ vals,
                                         const int32_t* __restrict__ cols,
                                         const double2* __restrict__ x, int64_t base, int p,
                                         int end, int stride, int split, double* a) {
  for (; p < end; p += U * stride) {
    int32_t c[U];
    double v[U], ua[U], ub[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const bool ok = p + k * stride < end;
      const int64_t i = base + p + k * stride;
      c[k] = ok ? ld_stream(cols + i) : 0;
      v[k] = ok ? ld_stream(vals + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const bool ok = p + k * stride < end;
      const double2 u = ok ? __ldg(x + c[k]) : make_double2(0.0, 0.0);  // one 16 B gather for both points
      ua[k] = u.x;
      ub[k] = u.y;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (Split && c[k] >= split) {
        a[2] = madd<Strict>(a[2], v[k], ua[k]);
        a[3] = madd<Strict>(a[3], v[k], ub[k]);
      } else {
        a[0] = madd<Strict>(a[0], v[k], ua[k]);
        a[1] = madd<Strict>(a[1], v[k], ub[k]);
      }
    }
  }
}

// ---- the kernel --------------------------------------------------------------
//
// Persistent: the grid is sized to the resident capacity and each CTA walks
// tiles t = blockIdx.x, + gridDim.x, ... (heavy bins own the lowest tile
// indices, so every CTA starts on heavy work). A tile's result never depends on
// which CTA computes it, so the schedule stays deterministic. Each CTA stages
// the Op's gathered-vector windows in shared memory once, before its first
// tile.

// Ops may declare `Pre prefetch(r)` (epilogue inputs) and
// `finish(r, acc, pre)`: the kernel loads them before the row's gathers.
struct NoPre {};
template <class Op, class = void>
struct HasPre : std::false_type {};
template <class Op>
struct HasPre<Op, std::void_t<typename Op::Pre>> : std::true_type {};
template <class Op>
__device__ __forceinline__ auto prefetch_of(const Op& op, int r) {
  if constexpr (HasPre<Op>::value) return op.prefetch(r);
  else return NoPre{};
}
template <class Op, class P>
__device__ __forceinline__ void finish_with(const Op& op, int r, const typename Op::AccT& a, const P& pre) {
  if constexpr (HasPre<Op>::value) op.finish(r, a, pre);
  else op.finish(r, a);
}

template <class Op, int V>
__device__ __forceinline__ void run_vlane(const Op& op, const SchedView& s, const BinDesc& bd,
                                          int tile, const Gather* g) {
  constexpr int kRowsPerBlock = kBlock / V;
  const int grp = threadIdx.x / V;
  const int lane = threadIdx.x % V;
  const int slot = bd.row_begin + (tile - bd.blk_begin) * kRowsPerBlock + grp;
  const bool valid = slot < bd.row_end;
  const int r = valid ? (s.perm ? s.perm[slot] : slot) : 0;
  decltype(prefetch_of(op, r)) pre{};
  if (valid && lane == 0) pre = prefetch_of(op, r);
  typename Op::AccT a;
  a.zero();
  if (valid) op.template accumulate<(V >= 16 ? Op::kWideUnroll : kUnroll)>(r, 0, op.len(r), lane, V, a, g);
  a.template reduce_lanes<V>();  // all lanes participate (invalid ones hold 0)
  if (valid && lane == 0) finish_with(op, r, a, pre);
}

template <class Op>
__device__ __forceinline__ void block_reduce(typename Op::AccT& a) {
  __shared__ double sm[kBlock / 32][Op::AccT::kK > 0 ? Op::AccT::kK : 1];
  a.template reduce_lanes<32>();
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < Op::AccT::kK; ++k) sm[w][k] = a.v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < Op::AccT::kK; ++k) {
      double t = sm[0][k];
      for (int j = 1; j < kBlock / 32; ++j) t = Op::AccT::comb(t, sm[j][k]);  // fixed order
      a.v[k] = t;
    }
  }
  __syncthreads();  // sm is reused by the CTA's next tile
}

template <class Op>
__device__ __forceinline__ void run_block_row(const Op& op, const SchedView& s, const BinDesc& bd,
                                              int tile, const Gather* g) {
  const int slot = bd.row_begin + (tile - bd.blk_begin);
  const int r = s.perm ? s.perm[slot] : slot;
  decltype(prefetch_of(op, r)) pre{};
  if (threadIdx.x == 0) pre = prefetch_of(op, r);
  typename Op::AccT a;
  a.zero();
  op.template accumulate<kUnroll>(r, 0, op.len(r), threadIdx.x, kBlock, a, g);
  block_reduce<Op>(a);
  if (threadIdx.x == 0) finish_with(op, r, a, pre);
}

template <class Op>
__device__ __forceinline__ void run_split(const Op& op, const SchedView& s, const BinDesc& bd,
                                          int tile, const Gather* g) {
  constexpr int K = Op::AccT::kK;
  const int seg = tile - bd.blk_begin;
  const int r = s.seg_row[seg];
  typename Op::AccT a;
  a.zero();
  op.template accumulate<kUnroll>(r, s.seg_lo[seg], s.seg_hi[seg], threadIdx.x, kBlock, a, g);
  block_reduce<Op>(a);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) s.seg_partial[(int64_t)seg * kMaxAcc + k] = a.v[k];
    __threadfence();
    const int first = s.seg_first[seg], cnt = s.seg_count[seg];
    const unsigned t = atomicAdd(&s.seg_ticket[first], 1u);
    if (t == static_cast<unsigned>(cnt - 1)) {  // last segment of the row to finish
      __threadfence();
      typename Op::AccT tot;
      tot.zero();
      for (int j = 0; j < cnt; ++j)  // fixed segment order
#pragma unroll
        for (int k = 0; k < K; ++k)
          tot.v[k] = Op::AccT::comb(tot.v[k], __ldcg(&s.seg_partial[(int64_t)(first + j) * kMaxAcc + k]));
      s.seg_ticket[first] = 0u;  // re-arm for the next launch / graph replay
      op.finish(r, tot);
    }
  }
}

// One tile of a schedule (all kBlock threads of the CTA take part).
template <class Op>
__device__ __forceinline__ void rowwise_tile(const Op& op, const SchedView& s, int tile, const Gather* g) {
  int bin = 0;  // bins occupy disjoint tile ranges (heavy bins first, see schedule.cu)
#pragma unroll
  for (int b = 1; b < kNumBins; ++b)
    if (tile >= s.bins[b].blk_begin && tile < s.bins[b].blk_end) bin = b;
  const BinDesc bd = s.bins[bin];
  if constexpr (Op::kStrict) {
    run_vlane<Op, 1>(op, s, bd, tile, g);  // strict schedules hold a single V=1 bin
  } else {
    switch (bin) {
      case 0: run_vlane<Op, 1>(op, s, bd, tile, g); break;
      case 1: run_vlane<Op, 2>(op, s, bd, tile, g); break;
      case 2: run_vlane<Op, 4>(op, s, bd, tile, g); break;
      case 3: run_vlane<Op, 8>(op, s, bd, tile, g); break;
      case 4: run_vlane<Op, 16>(op, s, bd, tile, g); break;
      case 5: run_vlane<Op, 32>(op, s, bd, tile, g); break;
      case 6: run_block_row<Op>(op, s, bd, tile, g); break;
      default: run_split<Op>(op, s, bd, tile, g); break;
    }
  }
}

template <class Op, bool Win>
__global__ void __launch_bounds__(kBlock) rowwise_kernel(const Op op, const SchedView s) {
  extern __shared__ double win_smem[];
  // programmatic dependent launch (launch_rowwise(.., pdl)): the previous
  // kernel's writes are visible after the wait; the next kernel may be
  // scheduled at once (its own wait holds it). Both are no-ops otherwise.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (HasGate<Op>::closed(op)) return;  // uniform over the grid
  Gather g[2];
  int off = 0;
#pragma unroll
  for (int slot = 0; slot < 2; ++slot) {
    const Window w = s.win[slot];
    const bool use = Win && w.len > 0;  // Win = false compiles the smem path out
    const double* src = op.gather_src(slot);
    g[slot] = Gather{src, win_smem + off, w.lo, use ? static_cast<uint32_t>(w.len) : 0u};
    if (use) {
      for (int k = threadIdx.x; k < w.len; k += kBlock) win_smem[off + k] = __ldcg(src + w.lo + k);
      off += w.len;
    }
  }
  if (Win) __syncthreads();
  for (int tile = blockIdx.x; tile < s.total_blocks; tile += gridDim.x) rowwise_tile(op, s, tile, g);
}

// Resident CTAs per SM for a kernel instance at a dynamic smem size (cached).
int resident_ctas(const void* kernel, int smem_bytes);

template <class Op>
inline void launch_rowwise(const Op& op, const SchedView& s, cudaStream_t st, bool pdl = false) {
  if (s.total_blocks <= 0) return;
  const int wins = Op::kStageWindows ? s.win[0].len + s.win[1].len : 0;
  if (wins == 0 && pdl) {  // as a programmatic dependent launch of the previous kernel
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(static_cast<unsigned>(s.total_blocks));
    lc.blockDim = dim3(kBlock);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    RB_CUDA(cudaLaunchKernelEx(&lc, rowwise_kernel<Op, false>, op, s));
  } else if (wins == 0) {
    // one tile per CTA: the hardware scheduler balances heavy and light tiles
    rowwise_kernel<Op, false><<<s.total_blocks, kBlock, 0, st>>>(op, s);
  } else {
    // persistent: each resident CTA stages the windows once, then strides tiles
    const int smem = wins * static_cast<int>(sizeof(double));
    const void* k = reinterpret_cast<const void*>(&rowwise_kernel<Op, true>);
    const int grid = std::min(s.total_blocks, resident_ctas(k, smem) * kSMs);
    rowwise_kernel<Op, true><<<grid, kBlock, smem, st>>>(op, s);
  }
  RB_LAUNCH_CHECK();
}

// ---- schedule ---------------------------------------------------------------

// Owns the device arrays behind a SchedView. Built on the device from a row
// length functor (see schedule.cu).
struct Schedule {
  DevBuf<int32_t> perm;
  DevBuf<int32_t> seg_row, seg_lo, seg_hi, seg_first, seg_count;
  DevBuf<double> seg_partial;
  DevBuf<unsigned> seg_ticket;
  SchedView view{};
  int64_t rows = 0;
  int32_t bin_rows[kNumBins] = {};
};

// Bin of a row of length L (fast mode): the fewest lanes V (power of two, up to
// a warp) that leave each lane at most `epl` elements; rows longer than
// `block_min` get a whole block, rows longer than kSplitLen several blocks.
__host__ __device__ inline int bin_of_len(int64_t L, int epl, int block_min) {
  for (int b = 0; b < kNumVBins - 1; ++b)
    if (L <= static_cast<int64_t>(epl) << b) return b;
  if (L <= block_min) return kNumVBins - 1;
  if (L <= kSplitLen) return kBinBlock;
  return kBinSplit;
}

// Schedule tuning (env RAPDHG_EPL / RAPDHG_BLOCK_MIN override the defaults).
struct SchedParams {
  int epl = 16;
  int block_min = 4096;
  static SchedParams from_env();
};

// lengths: device array of per-row lengths (int32). strict: single V=1 bin in
// natural row order.
// Pick the staged gather window of each segment (1: cols1 of a matrix with
// ncols1 columns, 2: cols2 / ncols2; nnz2 = 0 for single-segment schedules)
// from a device column histogram: the densest range of at most kWinMax
// columns, kept only if it serves enough gathers to repay staging it in every
// resident CTA. RAPDHG_WINDOW=off disables, =force keeps any non-empty window.
constexpr int kWinMax = 12288;  // doubles (96 KB): 2 CTAs/SM
void choose_windows(Schedule& sch, const int32_t* cols1, int64_t nnz1, int32_t ncols1,
                    const int32_t* cols2, int64_t nnz2, int32_t ncols2, cudaStream_t st);

// d_subset (optional, fast mode): schedule only these row ids (rows = their
// count); d_len is indexed by row id.
void build_schedule(Schedule& sch, const int32_t* d_len, int64_t rows, bool strict,
                    cudaStream_t st, const int32_t* d_subset = nullptr);

}  // namespace rb
