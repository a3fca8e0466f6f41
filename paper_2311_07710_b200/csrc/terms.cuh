// terms.cuh — reduction functors (reduce.cuh) shared by the single-GPU and
// the row-sharded engines. Indices are local to the range being reduced, so a
// shard passes pointers offset to its slice.
#pragma once

#include <cstdint>

namespace rb {

// Products are rounded before the add (--fmad=false), as the reference's
// `s += a[i] * b[i]` (vec.hpp:16).

struct SumSq {  // sum a_i^2 (norm2, vec.hpp:20)
  const double* a;
  __device__ void operator()(int64_t i, double* s, double*) const { s[0] += a[i] * a[i]; }
};

struct DotAndSumSq {  // s0 = v.w, s1 = w.w (opnorm.hpp:51-52, 77-78)
  const double* v;
  const double* w;
  StepGate gate{};
  __device__ void operator()(int64_t i, double* s, double*) const {
    s[0] += v[i] * w[i];
    s[1] += w[i] * w[i];
  }
};

// sum (x_i - e_i)^2 (dist2, vec.hpp:28-35), then e_i <- x_i (solver.hpp:459)
struct DistAndAdvance {
  const double* x;
  double* e;
  __device__ void operator()(int64_t i, double* s, double*) const {
    const double d = x[i] - e[i];
    s[0] += d * d;
    e[i] = x[i];
  }
};

// Dual-side relKKT terms for two points (kkt.hpp:44-53, 67):
// sums  by_i(c), by_e(c), by_i(a), by_e(a)
// maxes viol(c), viol(a), |ax|(c), |ax|(a), |b|
struct KktDualTerms {
  const double *axc, *axa, *b, *yc, *ya;
  int mi;
  __device__ void operator()(int64_t i, double* s, double* mx) const {
    const double bi = b[i];
    if (i < mi) {
      s[0] += bi * yc[i];
      s[2] += bi * ya[i];
      mx[0] = fmax(mx[0], axc[i] - bi);
      mx[1] = fmax(mx[1], axa[i] - bi);
    } else {
      s[1] += bi * yc[i];
      s[3] += bi * ya[i];
      mx[0] = fmax(mx[0], fabs(axc[i] - bi));
      mx[1] = fmax(mx[1], fabs(axa[i] - bi));
    }
    mx[2] = fmax(mx[2], fabs(axc[i]));
    mx[3] = fmax(mx[3], fabs(axa[i]));
    mx[4] = fmax(mx[4], fabs(bi));
  }
};

// Primal-side relKKT terms for two points (kkt.hpp:57-66):
// sums  x.qx(c), x.qx(a), c.x(c), c.x(a), then (box_projection) l.g+(c),
//       l.g+(a), u.g-(c), u.g-(a)
// maxes |qx+aty+c - lambda|(c), (a), |qx|(c), (a), |aty|(c), (a), |c|
// Without bounds (lo = hi = null: the reference's form) lambda = 0 and the
// bound sums stay 0. With bounds, lambda_j = max(g_j, 0) when l_j is finite
// plus min(g_j, 0) when u_j is finite (g = qx + aty + c): the bound
// multipliers that best fit stationarity; they enter the dual objective as
// l.max(g,0) + u.min(g,0) over the finite bounds.
struct KktPrimalTerms {
  const double *qxc, *qxa, *atc, *ata, *xc, *xa, *c;
  const double* lo = nullptr;  // original bounds (box_projection), null = none
  const double* hi = nullptr;
  __device__ void operator()(int64_t j, double* s, double* mx) const {
    const double cj = c[j];
    s[0] += xc[j] * qxc[j];
    s[1] += xa[j] * qxa[j];
    s[2] += cj * xc[j];
    s[3] += cj * xa[j];
    double gc = qxc[j] + atc[j] + cj, ga = qxa[j] + ata[j] + cj;
    if (lo || hi) {
      const double l = lo ? lo[j] : -INFINITY, u = hi ? hi[j] : INFINITY;
      if (l > -INFINITY) {
        s[4] += l * fmax(gc, 0.0);
        s[5] += l * fmax(ga, 0.0);
      }
      if (u < INFINITY) {
        s[6] += u * fmin(gc, 0.0);
        s[7] += u * fmin(ga, 0.0);
      }
      const double lc = (l > -INFINITY ? fmax(gc, 0.0) : 0.0) + (u < INFINITY ? fmin(gc, 0.0) : 0.0);
      const double la = (l > -INFINITY ? fmax(ga, 0.0) : 0.0) + (u < INFINITY ? fmin(ga, 0.0) : 0.0);
      gc = gc - lc;
      ga = ga - la;
    }
    mx[0] = fmax(mx[0], fabs(gc));
    mx[1] = fmax(mx[1], fabs(ga));
    mx[2] = fmax(mx[2], fabs(qxc[j]));
    mx[3] = fmax(mx[3], fabs(qxa[j]));
    mx[4] = fmax(mx[4], fabs(atc[j]));
    mx[5] = fmax(mx[5], fabs(ata[j]));
    mx[6] = fmax(mx[6], fabs(cj));
  }
};
constexpr int kKktPrimalSums = 8, kKktPrimalMaxes = 7;

}  // namespace rb
