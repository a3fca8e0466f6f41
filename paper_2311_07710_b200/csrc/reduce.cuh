// reduce.cuh — deterministic vector reductions (dots, norms, maxima).
//
// The reference sums sequentially (vec.hpp:14-35, kkt.hpp:43-69). Two modes:
//  * strict: one thread walks i = 0..N-1 in order — the reference's exact
//    association, bit-identical results;
//  * fast: the index space is cut into fixed CHUNKS of kRedChunk elements
//    (chunk c = [c*kRedChunk, (c+1)*kRedChunk) in GLOBAL indices). One block
//    reduces one chunk with a fixed pattern (thread-sequential, lane butterfly,
//    warps in order) into partial[c]; the partials are then combined by a
//    fixed lane-strided pass + butterfly. The result depends only on N — not
//    on scheduling, and not on how the index space is split across GPUs as
//    long as shard boundaries are multiples of kRedChunk (the row-sharded
//    solver aligns them), so a sharded solve reduces bit-identically to the
//    single-GPU one. No float atomics.
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
constexpr int kRedChunk = 2048;  // elements per chunk (8 per thread)
constexpr int kRedMaxOut = 32;

inline int64_t reduce_chunks(int64_t n) { return n > 0 ? ceil_div(n, kRedChunk) : 1; }

template <int NS, int NM, class F>
__global__ void reduce_seq_kernel(F f, int64_t n, double* out) {
  if (HasGate<F>::closed(f)) return;
  double s[NS > 0 ? NS : 1], mx[NM > 0 ? NM : 1];
  for (int k = 0; k < NS; ++k) s[k] = 0.0;
  for (int k = 0; k < NM; ++k) mx[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) f(i, s, mx);
  for (int k = 0; k < NS; ++k) out[k] = s[k];
  for (int k = 0; k < NM; ++k) out[NS + k] = mx[k];
}

// Fixed combine of partials[0..nchunks) (row-major, NT values each) into out,
// run by one block: warp w handles outputs k = w, w+8, ...; lane l folds
// partials l, l+32, ... in order, then a fixed butterfly.
template <int NS, int NT>
__device__ __forceinline__ void combine_partials(const double* partials, int64_t nchunks,
                                                 double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  for (int k = w; k < NT; k += kRedBlock / 32) {
    const bool is_sum = k < NS;
    double t = 0.0;
    for (int64_t b = lane; b < nchunks; b += 32) {
      const double v = __ldcg(&partials[b * NT + k]);
      t = is_sum ? t + v : fmax(t, v);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, t, off);
      t = is_sum ? t + o : fmax(t, o);
    }
    if (lane == 0) out[k] = t;
  }
}

// Phase 1: block b reduces chunk (chunk0 + b) of the functor's index space
// [0, n) into partials[(chunk0 + b) * NT ...]. With Combine (single launch),
// the last-arriving block then runs the fixed combine over all chunks.
template <int NS, int NM, class F, bool Combine>
__global__ void __launch_bounds__(kRedBlock) reduce_chunks_kernel(F f, int64_t n, double* partials,
                                                                   int64_t chunk0, unsigned* ticket,
                                                                   double* out) {
  constexpr int NT = NS + NM;
  // programmatic dependent launch (launch_reduce(.., pdl)); no-ops otherwise
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (HasGate<F>::closed(f)) return;  // uniform over the grid: no ticket taken
  double s[NS > 0 ? NS : 1], mx[NM > 0 ? NM : 1];
#pragma unroll
  for (int k = 0; k < NS; ++k) s[k] = 0.0;
#pragma unroll
  for (int k = 0; k < NM; ++k) mx[k] = 0.0;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRedChunk;
#pragma unroll
  for (int j = 0; j < kRedChunk / kRedBlock; ++j) {
    const int64_t i = base + j * kRedBlock + threadIdx.x;
    if (i < n) f(i, s, mx);
  }
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
  if (threadIdx.x < NT) {
    const int k = threadIdx.x;
    double t = sm[0][k];
    for (int j = 1; j < kRedBlock / 32; ++j) t = k < NS ? t + sm[j][k] : fmax(t, sm[j][k]);
    partials[(chunk0 + blockIdx.x) * NT + k] = t;
  }
  if constexpr (Combine) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (am_last) {
      __threadfence();
      combine_partials<NS, NT>(partials, gridDim.x, out);
      if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next launch / graph replay
    }
  }
}

template <int NS, int NT>
__global__ void __launch_bounds__(kRedBlock) reduce_combine_kernel(const double* partials,
                                                                    int64_t nchunks, double* out) {
  combine_partials<NS, NT>(partials, nchunks, out);
}

// Scratch for reductions: partials for up to `max_elems` elements x 32 values.
struct ReduceScratch {
  DevBuf<double> partials;
  DevBuf<unsigned> ticket;
  void init(int64_t max_elems, cudaStream_t st) {
    partials.alloc(static_cast<std::size_t>(reduce_chunks(max_elems)) * kRedMaxOut);
    ticket.alloc(1);
    ticket.zero(st);
  }
};

// Launch a reduction over [0, n) writing NS sums then NM maxima to d_out.
template <int NS, int NM, class F>
inline void launch_reduce(const F& f, int64_t n, bool strict, ReduceScratch& rs, double* d_out,
                          cudaStream_t st, bool pdl = false) {
  static_assert(NS + NM <= kRedMaxOut, "too many reduction outputs");
  if (strict) {
    reduce_seq_kernel<NS, NM, F><<<1, 1, 0, st>>>(f, n, d_out);
  } else if (pdl) {  // as a programmatic dependent launch of the previous kernel
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(static_cast<unsigned>(reduce_chunks(n)));
    lc.blockDim = dim3(kRedBlock);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    double* partials = rs.partials.get();
    unsigned* ticket = rs.ticket.get();
    RB_CUDA(cudaLaunchKernelEx(&lc, reduce_chunks_kernel<NS, NM, F, true>, f, n, partials, int64_t{0}, ticket, d_out));
  } else {
    reduce_chunks_kernel<NS, NM, F, true><<<static_cast<unsigned>(reduce_chunks(n)), kRedBlock, 0, st>>>(
        f, n, rs.partials.get(), 0, rs.ticket.get(), d_out);
  }
  RB_LAUNCH_CHECK();
}

// Sharded phase 1: the chunks of a local range that starts at global chunk
// `chunk0` (shard offsets are multiples of kRedChunk); partials land in the
// global partial array of `rs` at their global chunk index.
template <int NS, int NM, class F>
inline void launch_reduce_partials(const F& f, int64_t n_local, int64_t chunk0, ReduceScratch& rs,
                                   cudaStream_t st) {
  if (n_local <= 0) return;
  reduce_chunks_kernel<NS, NM, F, false><<<static_cast<unsigned>(ceil_div(n_local, kRedChunk)), kRedBlock,
                                           0, st>>>(f, n_local, rs.partials.get(), chunk0, nullptr, nullptr);
  RB_LAUNCH_CHECK();
}

// Sharded phase 2: combine the full (exchanged) partial array.
template <int NS, int NM>
inline void launch_reduce_combine(int64_t n_global, ReduceScratch& rs, double* d_out, cudaStream_t st) {
  reduce_combine_kernel<NS, NS + NM><<<1, kRedBlock, 0, st>>>(rs.partials.get(), reduce_chunks(n_global), d_out);
  RB_LAUNCH_CHECK();
}

}  // namespace rb
