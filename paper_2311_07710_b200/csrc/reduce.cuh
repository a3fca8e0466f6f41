// reduce.cuh — deterministic vector reductions (dots, norms, maxima).
//
// The reference sums sequentially (vec.hpp:14-35, kkt.hpp:43-69). Two modes:
//  * strict: one thread walks i = 0..N-1 in order — the reference's exact
//    association, bit-identical results;
//  * fast: a grid whose size is a fixed function of N; thread t sums i = t,
//    t+G*256, ... in order, the block combines lanes by a fixed butterfly and
//    warps in index order, and the LAST-arriving block (ticket counter) sums
//    the per-block partials in block order. The result never depends on
//    scheduling, so runs are bit-reproducible without float atomics.
// Maxima are order-free and therefore identical in both modes.
//
// A functor F supplies the terms: `void operator()(int64_t i, double* s,
// double* mx) const` adds its contributions to NS sums and NM maxima.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace rb {

constexpr int kRedBlock = 256;
constexpr int kRedMaxGrid = 2 * kSMs;

inline int reduce_grid(int64_t n) {
  const int64_t g = ceil_div(n, kRedBlock * 4);
  return static_cast<int>(g < 1 ? 1 : (g > kRedMaxGrid ? kRedMaxGrid : g));
}

template <int NS, int NM, class F>
__global__ void reduce_seq_kernel(F f, int64_t n, double* out) {
  double s[NS > 0 ? NS : 1], mx[NM > 0 ? NM : 1];
  for (int k = 0; k < NS; ++k) s[k] = 0.0;
  for (int k = 0; k < NM; ++k) mx[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) f(i, s, mx);
  for (int k = 0; k < NS; ++k) out[k] = s[k];
  for (int k = 0; k < NM; ++k) out[NS + k] = mx[k];
}

template <int NS, int NM, class F>
__global__ void __launch_bounds__(kRedBlock) reduce_par_kernel(F f, int64_t n, double* partials,
                                                                unsigned* ticket, double* out) {
  constexpr int NT = NS + NM;
  double s[NS > 0 ? NS : 1], mx[NM > 0 ? NM : 1];
#pragma unroll
  for (int k = 0; k < NS; ++k) s[k] = 0.0;
#pragma unroll
  for (int k = 0; k < NM; ++k) mx[k] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kRedBlock;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRedBlock + threadIdx.x; i < n; i += stride)
    f(i, s, mx);
  // warp butterfly
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] += __shfl_xor_sync(0xffffffffu, s[k], off);
#pragma unroll
    for (int k = 0; k < NM; ++k) mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
  }
  __shared__ double sm[kRedBlock / 32][NT > 0 ? NT : 1];
  __shared__ bool am_last;
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) sm[w][k] = s[k];
#pragma unroll
    for (int k = 0; k < NM; ++k) sm[w][NS + k] = mx[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < NT; ++k) {
      double t = sm[0][k];
      for (int j = 1; j < kRedBlock / 32; ++j) t = k < NS ? t + sm[j][k] : fmax(t, sm[j][k]);
      partials[static_cast<int64_t>(blockIdx.x) * NT + k] = t;
    }
    __threadfence();
    am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    // warp w combines outputs k = w, w + 8, ...: lane l sums partials
    // l, l + 32, ... in order, then a fixed butterfly — deterministic.
    const int lane = threadIdx.x & 31;
    for (int k = w; k < NT; k += kRedBlock / 32) {
      const bool is_sum = k < NS;
      double t = 0.0;
      for (unsigned b = lane; b < gridDim.x; b += 32) {
        const double v = __ldcg(&partials[static_cast<int64_t>(b) * NT + k]);
        t = is_sum ? t + v : fmax(t, v);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, t, off);
        t = is_sum ? t + o : fmax(t, o);
      }
      if (lane == 0) out[k] = t;
    }
    if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next launch / graph replay
  }
}

// Scratch for reductions: partials for up to kRedMaxGrid blocks x 32 values.
struct ReduceScratch {
  DevBuf<double> partials;
  DevBuf<unsigned> ticket;
  void init(cudaStream_t st) {
    partials.alloc(static_cast<std::size_t>(kRedMaxGrid) * 32);
    ticket.alloc(1);
    ticket.zero(st);
  }
};

// Launch a reduction writing NS sums then NM maxima to d_out.
template <int NS, int NM, class F>
inline void launch_reduce(const F& f, int64_t n, bool strict, ReduceScratch& rs, double* d_out,
                          cudaStream_t st) {
  static_assert(NS + NM <= 32, "too many reduction outputs");
  if (strict) {
    reduce_seq_kernel<NS, NM, F><<<1, 1, 0, st>>>(f, n, d_out);
  } else {
    reduce_par_kernel<NS, NM, F>
        <<<reduce_grid(n), kRedBlock, 0, st>>>(f, n, rs.partials.get(), rs.ticket.get(), d_out);
  }
  RB_LAUNCH_CHECK();
}

}  // namespace rb
