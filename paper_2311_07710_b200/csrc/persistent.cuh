// persistent.cuh — a whole chunk of inner steps in ONE cooperative launch,
// for problems so small that launching is the cost (C1: 1.3 MB per iteration,
// 2 kernels of ~1 us of work behind ~5 us of launch each).
//
// The CTAs of a grid that fits the GPU at once walk the dual step's rows,
// meet at a grid-wide barrier, walk the primal step's rows, meet again, and
// so on for every step of the chunk (the prologue first). Rows go through
// rowwise_tile or sell_slice — the functions the per-step kernels run — so
// every row is computed exactly as there: the results are bit-identical to the
// graph-replayed chunk (tests/test_gpu_parity.py), only the launches go.
// Opt-in (RAPDHG_PERSISTENT=1): on B200 the two grid-wide barriers per step
// cost more than the graph's launches (C1: 68k against 96k it/s).
#pragma once

#include <cooperative_groups.h>

#include "ops.cuh"
#include "rowwise.cuh"
#include "sell.cuh"

namespace rb {

// One step's rows: the sliced-ELL slices (a warp each, as sell_kernel) when
// the op has a SELL plan, else the rowwise tiles (a CTA each).
template <class Op>
__device__ __forceinline__ void chunk_pass(const Op& op, const SchedView& s, const SellView& sv) {
  if (sv.nslices > 0) {
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kBlock / 32);
    for (int64_t q = (blockIdx.x * static_cast<int64_t>(kBlock) + threadIdx.x) >> 5; q < sv.nslices; q += nwarps)
      sell_slice(op, sv, q, threadIdx.x & 31);
  } else {
    const Gather g[2] = {Gather{op.gather_src(0), nullptr, 0, 0u}, Gather{op.gather_src(1), nullptr, 0, 0u}};
    for (int t = blockIdx.x; t < s.total_blocks; t += gridDim.x) rowwise_tile(op, s, t, g);
  }
}

template <class DualOp, class PrimalOp>
__global__ void __launch_bounds__(kBlock) chunk_kernel(DualOp d, SchedView sd, SellView dsell, PrimalOp p0,
                                                       PrimalOp p1, SchedView sp, SellView psell, const double* x,
                                                       const double* xp, const double* xb, double* w, double* xmd,
                                                       const IterParams* P, int n, int len, int cur) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  {  // prologue_kernel (elementwise.cuh): w and x_md of the chunk's first step
    const IterParams& q = P[0];
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n; j += nthreads) {
      const double xj = x[j];
      w[j] = q.theta * (xj - xp[j]) + xj;
      xmd[j] = q.omib * xb[j] + q.ib * xj;
    }
  }
  grid.sync();
  for (int it = 0; it < len; ++it) {
    DualOp dop = d;
    dop.it = it;
    chunk_pass(dop, sd, dsell);
    grid.sync();
    PrimalOp pop = ((cur + it) & 1) ? p1 : p0;
    pop.it = it;
    chunk_pass(pop, sp, psell);
    grid.sync();
  }
}

}  // namespace rb
