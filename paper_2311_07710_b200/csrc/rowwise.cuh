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

#include <cuda_runtime.h>

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
  int32_t total_blocks;
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
template <bool Strict, int U = kUnroll>
__device__ __forceinline__ double seg_dot(const double* __restrict__ vals,
                                          const int32_t* __restrict__ cols,
                                          const double* __restrict__ x, int64_t base, int p,
                                          int end, int stride, double acc) {
  for (; p < end; p += U * stride) {
    int32_t c[U];
    double v[U], xv[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const bool ok = p + k * stride < end;
      const int64_t i = base + p + k * stride;
      c[k] = ok ? ld_stream(cols + i) : 0;
      v[k] = ok ? ld_stream(vals + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) xv[k] = (p + k * stride < end) ? ld_gather(x + c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < U; ++k) acc = madd<Strict>(acc, v[k], xv[k]);
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
                                         const double* __restrict__ xa,
                                         const double* __restrict__ xb, int64_t base, int p,
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
      ua[k] = ok ? ld_gather(xa + c[k]) : 0.0;
      ub[k] = ok ? ld_gather(xb + c[k]) : 0.0;
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

template <class Op, int V>
__device__ __forceinline__ void run_vlane(const Op& op, const SchedView& s, const BinDesc& bd) {
  constexpr int kRowsPerBlock = kBlock / V;
  const int g = threadIdx.x / V;
  const int lane = threadIdx.x % V;
  const int slot = bd.row_begin + (blockIdx.x - bd.blk_begin) * kRowsPerBlock + g;
  const bool valid = slot < bd.row_end;
  const int r = valid ? (s.perm ? s.perm[slot] : slot) : 0;
  typename Op::AccT a;
  a.zero();
  if (valid) op.template accumulate<(V >= 16 ? Op::kWideUnroll : kUnroll)>(r, 0, op.len(r), lane, V, a);
  a.template reduce_lanes<V>();  // all lanes participate (invalid ones hold 0)
  if (valid && lane == 0) op.finish(r, a);
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
}

template <class Op>
__device__ __forceinline__ void run_block_row(const Op& op, const SchedView& s, const BinDesc& bd) {
  const int slot = bd.row_begin + (blockIdx.x - bd.blk_begin);
  const int r = s.perm ? s.perm[slot] : slot;
  typename Op::AccT a;
  a.zero();
  op.template accumulate<kUnroll>(r, 0, op.len(r), threadIdx.x, kBlock, a);
  block_reduce<Op>(a);
  if (threadIdx.x == 0) op.finish(r, a);
}

template <class Op>
__device__ __forceinline__ void run_split(const Op& op, const SchedView& s, const BinDesc& bd) {
  constexpr int K = Op::AccT::kK;
  const int seg = blockIdx.x - bd.blk_begin;
  const int r = s.seg_row[seg];
  typename Op::AccT a;
  a.zero();
  op.template accumulate<kUnroll>(r, s.seg_lo[seg], s.seg_hi[seg], threadIdx.x, kBlock, a);
  block_reduce<Op>(a);
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) s.seg_partial[(int64_t)seg * kMaxAcc + k] = a.v[k];
    __threadfence();
    const int first = s.seg_first[seg], cnt = s.seg_count[seg];
    const unsigned t = atomicAdd(&s.seg_ticket[first], 1u);
    last = (t == static_cast<unsigned>(cnt - 1));
    if (last) {
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

template <class Op>
__global__ void __launch_bounds__(kBlock) rowwise_kernel(const Op op, const SchedView s) {
  // bins occupy disjoint block ranges (heavy bins first, see schedule.cu)
  int bin = 0;
#pragma unroll
  for (int b = 1; b < kNumBins; ++b)
    if (static_cast<int>(blockIdx.x) >= s.bins[b].blk_begin &&
        static_cast<int>(blockIdx.x) < s.bins[b].blk_end)
      bin = b;
  const BinDesc bd = s.bins[bin];
  if (static_cast<int>(blockIdx.x) < bd.blk_begin || static_cast<int>(blockIdx.x) >= bd.blk_end) return;
  if constexpr (Op::kStrict) {
    run_vlane<Op, 1>(op, s, bd);  // strict schedules hold a single V=1 bin
  } else {
    switch (bin) {
      case 0: run_vlane<Op, 1>(op, s, bd); break;
      case 1: run_vlane<Op, 2>(op, s, bd); break;
      case 2: run_vlane<Op, 4>(op, s, bd); break;
      case 3: run_vlane<Op, 8>(op, s, bd); break;
      case 4: run_vlane<Op, 16>(op, s, bd); break;
      case 5: run_vlane<Op, 32>(op, s, bd); break;
      case 6: run_block_row<Op>(op, s, bd); break;
      default: run_split<Op>(op, s, bd); break;
    }
  }
}

template <class Op>
inline void launch_rowwise(const Op& op, const SchedView& s, cudaStream_t st) {
  if (s.total_blocks <= 0) return;
  rowwise_kernel<Op><<<s.total_blocks, kBlock, 0, st>>>(op, s);
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
void build_schedule(Schedule& sch, const int32_t* d_len, int64_t rows, bool strict,
                    cudaStream_t st);

}  // namespace rb
