// sell.cuh — sliced-ELL (SELL-32-sigma) layout for ops whose rows are all
// short (fast mode).
//
// Why: rowwise_kernel gives a row of <= 16 entries one lane, so the 32 lanes
// of a warp walk 32 different rows and every index / value load of the warp
// touches a different sector: on C5 (rows of 4-12 entries, 1.6e8 random
// gathers per iteration) the matrix stream then costs about twice the L1TEX
// wavefronts of the gathers themselves (ncu: 8.6e7 sectors for 3e7 entries of
// one pass, LSU wavefronts at 67% of peak).
//
// Layout: rows in index order (RAPDHG_SELL_SIGMA = s > 32: sorted by length
// within chunks of s rows), cut into slices of 32 rows; a slice stores its
// entries entry-major (entry e of lane l at off[q] + 32 e + l; padding col 0,
// value 0), so a warp's index and value loads are contiguous (4 + 8 sectors
// per 32 entries) and only the gathers are scattered. A row keeps its entries
// in CSR order, segment 1 (e < l1) then segment 2, each summed sequentially
// with fma into its own accumulator: the arithmetic depends only on the row,
// so results are deterministic and a sharded solve that builds the same
// layout over its rows stays bit-identical. The epilogue runs in the same
// warp (lane = row), its inputs requested before the row's entries.
#pragma once

#include <cstdint>

#include "ops.cuh"

namespace rb {

constexpr int kSellMaxLen = 64;    // rows up to this many entries (all rows of a SELL op)
// Rows per sorting chunk: 32 = index order. Sorting (less padding) scatters
// the epilogue's vector accesses over the chunk, and on C5's epilogue-heavy
// final primal pass that doubled its DRAM traffic (2.2 vs 1.0 GB): index
// order costs only idle lanes in a slice's last entries (no extra loads).
constexpr int kSellSigma = 32;

struct SellView {
  int64_t nslots = 0;               // rows (slots beyond are padding)
  int64_t nslices = 0;
  const int64_t* off = nullptr;     // [nslices + 1] entry offsets (multiples of 32)
  const int32_t* row = nullptr;     // [nslices * 32] op row per slot
  const int32_t* len = nullptr;     // entries per slot
  const int32_t* l1 = nullptr;      // segment-1 entries per slot
  const int32_t* col = nullptr;
  const double* val = nullptr;
  bool active() const { return nslices > 0; }
};

// Device arrays behind a SellView. pos: source of each entry's value (segment
// 1 positions as is, segment 2 positions + kSellSeg2; -1 padding).
constexpr int64_t kSellSeg2 = int64_t{1} << 40;
struct SellPlan {
  SellView view;
  DevBuf<int64_t> off, pos;
  DevBuf<int32_t> row, len, l1, col;
  DevBuf<double> val;
  bool active() const { return view.active(); }
};

// Plan over rows [0, rows) of the two-segment pattern (rp2 may be null; row
// pointers may be offset views, positions stay absolute). Leaves the plan
// the caller decides with sell_eligible (rows longer than kSellMaxLen would
// pad whole slices).
void build_sell_plan(SellPlan& plan, const int32_t* rp1, const int32_t* ci1, const int32_t* rp2, const int32_t* ci2,
                     int32_t rows, cudaStream_t st, const int32_t* subset = nullptr);
// subset (device, `rows` ids in increasing order): the plan covers only those
// rows of the pattern (slot s holds subset[s]).
bool sell_enabled();
// (Re)fill the values from arrays laid out like segment 1 / segment 2.
void fill_sell_values(SellPlan& plan, const double* v1, const double* v2, cudaStream_t st);
// Whether every row of the pattern has at most kSellMaxLen entries (and
// RAPDHG_SELL is not 0): decided once on the whole matrix, so every shard of a
// sharded solve takes the decision one GPU takes.
bool sell_eligible(const int32_t* rp1, const int32_t* rp2, int32_t rows, cudaStream_t st);

// One warp computes slice q (lane = row) and runs the op's epilogue.
template <class Op>
__device__ __forceinline__ void sell_slice(const Op& op, const SellView& sv, int64_t q, int lane) {
  constexpr int U = 4;
  const double* g0 = op.gather_src(0);
  const double* g1 = op.gather_src(1);
  const int64_t slot = (q << 5) + lane;
  const bool valid = slot < sv.nslots;
  int r = 0, L = 0, l1 = 0;
  typename Op::Pre pre{};
  if (valid) {
    r = sv.row[slot];
    L = sv.len[slot];
    l1 = sv.l1[slot];
    pre = op.prefetch(r);
  }
  const int64_t o = sv.off[q];
  const int W = static_cast<int>((sv.off[q + 1] - o) >> 5);
  const int32_t* cq = sv.col + o + lane;
  const double* vq = sv.val + o + lane;
  double a0 = 0.0, a1 = 0.0;
  int32_t c[U];
  double v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool ok = u < L;
    c[u] = ok ? __ldcs(cq + (u << 5)) : 0;
    v[u] = ok ? __ldcs(vq + (u << 5)) : 0.0;
  }
  for (int e = 0; e < W; e += U) {
    // next batch's indices / values in flight before this batch's gathers
    int32_t cn[U];
    double vn[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = e + U + u < L;
      cn[u] = ok ? __ldcs(cq + ((e + U + u) << 5)) : 0;
      vn[u] = ok ? __ldcs(vq + ((e + U + u) << 5)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = e + u < L ? __ldg((e + u < l1 ? g0 : g1) + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e + u < l1) a0 = fma(v[u], x[u], a0);
      else if (e + u < L) a1 = fma(v[u], x[u], a1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = cn[u], v[u] = vn[u];
  }
  if (valid) {
    typename Op::AccT acc;
    acc.zero();
    acc.v[0] = a0;
    if constexpr (Op::AccT::kK > 1) acc.v[Op::AccT::kK - 1] = a1;
    op.finish(r, acc, pre);
  }
}

template <class Op>
__global__ void __launch_bounds__(kBlock) sell_kernel(const Op op, const SellView sv) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see rowwise_kernel (no-ops without PDL)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kBlock / 32);
  for (int64_t q = (blockIdx.x * static_cast<int64_t>(kBlock) + threadIdx.x) >> 5; q < sv.nslices; q += nwarps)
    sell_slice(op, sv, q, lane);
}

template <class Op>
inline void launch_sell(const Op& op, const SellPlan& plan, cudaStream_t st, bool pdl = false) {
  const int64_t warps_needed = plan.view.nslices;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps_needed, kBlock / 32),
                                                                                       16 * kSMs)));
  if (pdl) {  // programmatic dependent launch (see launch_rowwise)
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kBlock);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    RB_CUDA(cudaLaunchKernelEx(&lc, sell_kernel<Op>, op, plan.view));
  } else {
    sell_kernel<Op><<<grid, kBlock, 0, st>>>(op, plan.view);
  }
  RB_LAUNCH_CHECK();
}

}  // namespace rb
