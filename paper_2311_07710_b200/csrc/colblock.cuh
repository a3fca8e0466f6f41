// colblock.cuh — L2-sized column blocking of a gather-bound row op (fast mode).
//
// Why: a row op that gathers from a vector larger than what L2 keeps resident
// next to the streamed matrix (C5: w is 80 MB; the step also streams y, ybar
// and writes them back, 200+ MB per launch through a 126 MB L2) misses L2 on
// most gathers, and each miss moves a 64 B DRAM burst for 8 useful bytes:
// ncu on C5's dual step shows 4.2 GB read for 1.0 GB of algorithmic bytes.
//
// How: the gathered segment's columns are cut into nb blocks of at most
// kL2BlockBytes. Block b is a CSR over all rows holding, per row, the row's
// entries with columns in block b (a contiguous sub-run of the column-sorted
// row, values in their original order). Passes 0 .. nb-2 run SpmvOp over one
// block each (its slice of the vector stays L2-resident for the pass) and
// write per-row partial sums; the last pass runs the step op itself over the
// last block and, through PartialsOp, adds the earlier partials (prefetched
// with the epilogue inputs, summed in block order) before the epilogue.
// A row's value is ((p_0 + p_1) + ...) + s_last — fixed by the blocking, so
// results are deterministic.
#pragma once

#include <cstdint>
#include <vector>

#include "device_csr.cuh"
#include "ops.cuh"
#include "rowwise.cuh"
#include "sell.cuh"

namespace rb {

constexpr std::size_t kL2BlockBytes = std::size_t{48} << 20;

struct ColBlocks {
  int nb = 1;
  std::vector<int32_t> cut;  // nb + 1 column cuts
  std::vector<DevCsr> blk;   // block CSRs (rows of the op, all columns)
  std::vector<DevBuf<int32_t>> pos;  // per block: source position of each entry
  bool active() const { return nb >= 2; }
};

// Blocks for a segment with `ncols` columns gathered from 8-byte values:
// nb = ceil(8 * ncols / kL2BlockBytes) (RAPDHG_L2BLOCK_KB overrides the block
// size, RAPDHG_L2BLOCK=0 disables); nb < 2 leaves `cb` inactive.
int colblock_count(int64_t ncols);
void build_colblocks(ColBlocks& cb, int nb, const int32_t* rp, const int32_t* ci, int32_t rows, int32_t ncols,
                     cudaStream_t st);
void fill_colblock_values(ColBlocks& cb, const double* vals, cudaStream_t st);

// Fraction of entries whose column lies within 1/16 of the matrix width of the
// row's diagonal position: gathers of a "local" pattern (>= 1/2) already hit
// L2 in row order, and blocking would only add passes.
double pattern_locality(const int32_t* rp, const int32_t* ci, int32_t rows, int32_t ncols, int64_t nnz,
                        cudaStream_t st);

// Op over the last column blocks plus the partial sums of the earlier blocks
// of its first (part0, np0 blocks) and last (part1, np1 blocks) accumulators;
// partial q of row r at part[q * rows + r].
template <class Op>
struct PartialsOp {
  static constexpr bool kStrict = false;
  static constexpr int kWideUnroll = Op::kWideUnroll;
  static constexpr bool kStageWindows = false;
  using AccT = typename Op::AccT;
  Op op;
  const double* part0;
  const double* part1;
  int32_t np0, np1;
  int64_t rows;
  struct Pre {
    typename Op::Pre inner;
    double t0, t1;
  };
  __device__ __forceinline__ int len(int r) const { return op.len(r); }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride, AccT& acc,
                                             const Gather* g) const {
    op.template accumulate<U>(r, lo, hi, lane, stride, acc, g);
  }
  __device__ __forceinline__ const double* gather_src(int slot) const { return op.gather_src(slot); }
  __device__ __forceinline__ static double sum_parts(const double* p, int np, int64_t rows, int r) {
    double t = 0.0;
    if (np > 0) {
      t = __ldcs(p + r);
      for (int q = 1; q < np; ++q) t += __ldcs(p + q * rows + r);
    }
    return t;
  }
  __device__ __forceinline__ Pre prefetch(int r) const {
    return Pre{op.prefetch(r), sum_parts(part0, np0, rows, r), sum_parts(part1, np1, rows, r)};
  }
  __device__ __forceinline__ void finish(int r, const AccT& acc) const { finish(r, acc, prefetch(r)); }
  __device__ __forceinline__ void finish(int r, const AccT& acc, const Pre& pre) const {
    AccT a = acc;
    if (np0 > 0) a.v[0] = pre.t0 + a.v[0];
    if (np1 > 0) a.v[AccT::kK - 1] = pre.t1 + a.v[AccT::kK - 1];
    op.finish(r, a, pre.inner);
  }
};

// Column-blocked dual step over rows [0, rows) of a row view of A (rp offset
// to the first row; positions stay absolute, so values come from the full
// arrays): passes 0 .. nb-2 write partials, the last runs DualStepOp.
struct ColBlockedDual {
  ColBlocks cb;
  DevBuf<double> part;
  std::vector<Schedule> sch;
  std::vector<SellPlan> sell;  // per block, when the op's rows are short (sell.cuh)
  int64_t rows = 0;
  bool active() const { return cb.active(); }
};
void build_colblocked_dual(ColBlockedDual& d, int nb, const int32_t* rp, const int32_t* ci, int32_t rows,
                           int32_t ncols, const double* vals, bool sell, cudaStream_t st);

// `op`: the step op over the same rows with the unblocked views. Returns kernels launched.
inline int launch_colblocked_dual(const DualStepOp<false>& op, const ColBlockedDual& d, cudaStream_t st) {
  const int nb = d.cb.nb;
  const bool sell = !d.sell.empty();
  int n = 0;
  for (int b = 0; b + 1 < nb; ++b) {
    const SpmvOp<false> sp{d.cb.blk[b].view(), op.w, d.part.get() + static_cast<int64_t>(b) * d.rows};
    if (sell) launch_sell(sp, d.sell[b], st);
    else launch_rowwise(sp, d.sch[b].view, st);
    ++n;
  }
  DualStepOp<false> last = op;
  last.a = d.cb.blk[nb - 1].view();
  const PartialsOp<DualStepOp<false>> fin{last, d.part.get(), nullptr, nb - 1, 0, d.rows};
  if (sell) launch_sell(fin, d.sell[nb - 1], st);
  else launch_rowwise(fin, d.sch[nb - 1].view, st);
  return n + 1;
}

// Column-blocked primal step over rows [0, rows) of row views of Q and A':
// Q blocks 0 .. nq-2 and A' blocks as partial passes, then PrimalStepOp over
// the last Q block (+ the last A' block unless A'y is all partial passes,
// which it is whenever Q is blocked, so the last pass gathers one block).
struct ColBlockedPrimal {
  ColBlocks q, at;
  DevBuf<double> part_q, part_at;
  std::vector<Schedule> sch_q, sch_at;  // partial passes
  Schedule fin;
  std::vector<SellPlan> sell_q, sell_at;  // partial passes (when the op's rows are short)
  SellPlan sell_fin;
  bool at_all_partial = false;
  DevBuf<int32_t> zero_rp;  // empty rows for an all-partial A'
  int64_t rows = 0;
  bool on = false;
  bool active() const { return on; }
};
void build_colblocked_primal(ColBlockedPrimal& p, int nq, int na, const int32_t* rpq, const int32_t* ciq,
                             const double* qvals, const int32_t* rpat, const int32_t* ciat, const double* atvals,
                             int32_t rows, int32_t n, int32_t m, bool sell, cudaStream_t st);

inline int launch_colblocked_primal(const PrimalStepOp<false>& op, const ColBlockedPrimal& p, cudaStream_t st) {
  int n = 0;
  const bool sell = p.sell_fin.active();
  for (int b = 0; b + 1 < p.q.nb && p.q.active(); ++b) {
    const SpmvOp<false> sp{p.q.blk[b].view(), op.xmd, p.part_q.get() + static_cast<int64_t>(b) * p.rows};
    if (sell) launch_sell(sp, p.sell_q[b], st);
    else launch_rowwise(sp, p.sch_q[b].view, st);
    ++n;
  }
  const int npa = static_cast<int>(p.sch_at.size());
  for (int b = 0; b < npa; ++b) {
    const CsrView at = p.at.active() ? p.at.blk[b].view() : op.at;
    const SpmvOp<false> sp{at, op.y, p.part_at.get() + static_cast<int64_t>(b) * p.rows};
    if (sell) launch_sell(sp, p.sell_at[b], st);
    else launch_rowwise(sp, p.sch_at[b].view, st);
    ++n;
  }
  PrimalStepOp<false> last = op;
  if (p.q.active()) last.q = p.q.blk[p.q.nb - 1].view();
  if (p.at_all_partial) last.at = CsrView{p.zero_rp.get(), op.at.ci, op.at.v};
  else if (p.at.active()) last.at = p.at.blk[p.at.nb - 1].view();
  const PartialsOp<PrimalStepOp<false>> fin{last, p.part_q.get(), p.part_at.get(), p.q.active() ? p.q.nb - 1 : 0,
                                            npa, p.rows};
  if (sell) launch_sell(fin, p.sell_fin, st);
  else launch_rowwise(fin, p.fin.view, st);
  return n + 1;
}

}  // namespace rb
