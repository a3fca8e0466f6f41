// elementwise.cuh — per-element kernels of the iteration state, shared by the
// single-GPU and the row-sharded engines (a shard passes pointers offset to
// its slice). Internal linkage: each translation unit gets its own copy.
#pragma once

#include "ops.cuh"

namespace rb {
namespace {

// w = theta (x - x_prev) + x ; x_md = (1 - 1/beta) xbar + (1/beta) x
// (solver.hpp:163,169) for the first iteration of a chunk.
__global__ void prologue_kernel(const double* __restrict__ x, const double* __restrict__ xp,
                                const double* __restrict__ xb, double* __restrict__ w,
                                double* __restrict__ xmd, const IterParams* P, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const IterParams& q = P[0];
  const double xj = x[j];
  w[j] = q.theta * (xj - xp[j]) + xj;
  xmd[j] = q.omib * xb[j] + q.ib * xj;
}

// unscale_point (scaling.hpp:126-133) of the current iterate and the average.
// (xi / yi, when given: the same pairs interleaved for the KKT products'
// 16 B gathers)
__global__ void unscale_kernel(const double* x, const double* xb, const double* y,
                               const double* yb, const double* d, double* xuc, double* xua,
                               double* yuc, double* yua, int n, int m, double2* xi = nullptr,
                               double2* yi = nullptr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double f = d[i];
    const double c = x[i] * f, a = xb[i] * f;
    xuc[i] = c;
    xua[i] = a;
    if (xi) xi[i] = make_double2(c, a);
  } else if (i < n + m) {
    const int r = i - n;
    const double f = d[i];
    const double c = y[r] * f, a = yb[r] * f;
    yuc[r] = c;
    yua[r] = a;
    if (yi) yi[r] = make_double2(c, a);
  }
}

// (a[i], b[i]) pairs, so one 16 B gather serves both KKT points.
__global__ void interleave_kernel(const double* a, const double* b, double2* out, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = make_double2(a[i], b[i]);
}

// Restart (solver.hpp:442-448): optionally x <- xbar, y <- ybar; then
// x_prev <- x, xbar <- x, ybar <- y.
__global__ void restart_kernel(double* x, double* xp, double* xb, double* y, double* yb,
                               int from_avg, int n, int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double v = from_avg ? xb[i] : x[i];
    x[i] = v;
    xp[i] = v;
    xb[i] = v;
  } else if (i < n + m) {
    const int r = i - n;
    const double v = from_avg ? yb[r] : y[r];
    y[r] = v;
    yb[r] = v;
  }
}

}  // namespace
}  // namespace rb
