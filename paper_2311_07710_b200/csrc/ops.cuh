// ops.cuh — the row operations run by rowwise_kernel (rowwise.cuh).
//
// Each Op describes, for one logical row r: its length (nnz over its one or two
// CSR segments), how to accumulate a lane's share of positions
// [lo, hi) (stride = lanes working on the row), and the epilogue `finish`
// run once per row with the fully reduced sums. Epilogue arithmetic is written
// exactly as the reference writes it; the library is compiled with
// --fmad=false so `a*b + c` is never contracted and the epilogues are
// bit-identical to the reference in both modes. Only the SpMV accumulation of
// fast mode uses explicit fma() (madd<false>).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rowwise.cuh"

#ifndef RB_DUAL_UNROLL
#define RB_DUAL_UNROLL 4  // 8 measured slower on C2/C4 (register pressure)
#endif

namespace rb {

// Per-iteration scalars of one inner step, computed on the host for a whole
// check interval (they depend only on k, eta_{k-1}, ||Q||, ||A||, omega:
// solver.hpp:347-368) and uploaded once per chunk.
struct IterParams {
  double theta;           // extrapolation theta_k (solver.hpp:163)
  double ib, omib;        // 1/beta_k and 1 - 1/beta_k (solver.hpp:160,169,177-178)
  double eta, tau;        // primal / dual step (solver.hpp:166,175)
  double theta_n;         // next iteration's theta, ...
  double ib_n, omib_n;    // ... and weights, to emit w and x_md for it
  long long t;            // global iteration index (NaN flag)
  int emit_next;          // 0 on the last iteration of a chunk
  int pad;
};

__device__ __forceinline__ void flag_nonfinite(double v, long long t, long long* bad) {
  if (!isfinite(v)) atomicMin(bad, t);
}

struct CsrView {
  const int32_t* rp;
  const int32_t* ci;
  const double* v;
};

// ---------------------------------------------------------------------------
// Dual step over rows of the stacked scaled A (solver.hpp:164-167, 178):
//   aw_i = sum A_ik w_k;  y_i += tau (aw_i - b_i);  y_i = max(y_i, 0) for
//   i < m_ineq;  ybar_i = (1 - 1/beta) ybar_i + (1/beta) y_i.
template <bool Strict>
struct DualStepOp {
  static constexpr bool kStrict = Strict;
  static constexpr int kPhase = 0;  // slot of the step in an iteration (in-loop timing)
  static constexpr int kWideUnroll = RB_DUAL_UNROLL;  // long A rows: loads in flight per lane
  static constexpr bool kStageWindows = true;
  using AccT = Acc<1>;
  CsrView a;
  const double* w;
  const double* b;
  double* y;
  double* yb;
  int m_ineq;
  const IterParams* P;
  int it;
  long long* bad;
  __device__ __forceinline__ int len(int r) const { return a.rp[r + 1] - a.rp[r]; }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather* g) const {
    acc.v[0] = seg_dot<Strict, U>(a.v, a.ci, g[0], a.rp[r], lo + lane, hi, stride, acc.v[0]);
  }
  __device__ __forceinline__ const double* gather_src(int) const { return w; }
  // same op over other CSR arrays (the rest CSR of a slab plan)
  __host__ __device__ DualStepOp with_views(CsrView s1, CsrView) const {
    DualStepOp o = *this;
    o.a = s1;
    return o;
  }
  // epilogue inputs, loaded before the row's gathers so their latency overlaps
  struct Pre {
    double y, b, yb;
  };
  __device__ __forceinline__ Pre prefetch(int i) const { return Pre{y[i], b[i], yb[i]}; }
  __device__ __forceinline__ void finish(int i, const AccT& acc) const { finish(i, acc, prefetch(i)); }
  __device__ __forceinline__ void finish(int i, const AccT& acc, const Pre& pre) const {
    const IterParams& q = P[it];
    double yi = pre.y;
    yi += q.tau * (acc.v[0] - pre.b);
    if (i < m_ineq) yi = yi > 0.0 ? yi : 0.0;
    y[i] = yi;
    yb[i] = q.omib * pre.yb + q.ib * yi;
    flag_nonfinite(yi, q.t, bad);
  }
};

// ---------------------------------------------------------------------------
// Primal step over rows j of [Q~ | A~'] (solver.hpp:169-177):
//   qx_j = sum Q_jk xmd_k;  aty_j = sum A'_ji y_i;
//   x+_j = x_j - eta ((qx_j + c_j) + aty_j);  xbar_j = (1-1/b) xbar_j + (1/b) x+_j
// and, when another iteration follows in the chunk, the next extrapolation
// w_j = theta' (x+_j - x_j) + x+_j and x_md_j = (1-1/b') xbar_j + (1/b') x+_j
// (solver.hpp:163,169 of the next call), so the next dual/primal kernels
// gather them directly.
template <bool Strict>
struct PrimalStepOp {
  static constexpr bool kStrict = Strict;
  static constexpr int kPhase = 1;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = true;
  using AccT = Acc<2>;
  CsrView q, at;
  const double* xmd;  // gathered by Q
  const double* y;    // gathered by A'
  const double* x_in;
  double* x_out;
  double* xb;
  const double* c;
  double* w_out;
  double* xmd_out;
  const IterParams* P;
  int it;
  long long* bad;
  // box_projection (B200 extension): x+ projected onto [lo, hi] (scaled
  // bounds, null = unbounded); the reference has no such step (its bounds
  // are rows), so this is never used in a parity mode
  const double* lo = nullptr;
  const double* hi = nullptr;
  __device__ __forceinline__ int len(int r) const {
    return (q.rp[r + 1] - q.rp[r]) + (at.rp[r + 1] - at.rp[r]);
  }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather* g) const {
    const int q0 = q.rp[r];
    const int L1 = q.rp[r + 1] - q0;
    const int p = lo + lane;
    acc.v[0] = seg_dot<Strict, U>(q.v, q.ci, g[0], q0, p, hi < L1 ? hi : L1, stride, acc.v[0]);
    acc.v[1] = seg_dot<Strict, U>(at.v, at.ci, g[1], static_cast<int64_t>(at.rp[r]) - L1,
                               next_pos(p, stride, L1), hi, stride,
                               acc.v[1]);
  }
  __device__ __forceinline__ const double* gather_src(int slot) const { return slot ? y : xmd; }
  __host__ __device__ PrimalStepOp with_views(CsrView s1, CsrView s2) const {
    PrimalStepOp o = *this;
    o.q = s1;
    o.at = s2;
    return o;
  }
  // epilogue inputs, loaded before the row's gathers so their latency overlaps
  struct Pre {
    double x, c, xb;
  };
  __device__ __forceinline__ Pre prefetch(int j) const { return Pre{x_in[j], c[j], xb[j]}; }
  __device__ __forceinline__ void finish(int j, const AccT& acc) const { finish(j, acc, prefetch(j)); }
  __device__ __forceinline__ void finish(int j, const AccT& acc, const Pre& pre) const {
    const IterParams& p = P[it];
    const double xo = pre.x;
    double xn = xo - p.eta * (acc.v[0] + pre.c + acc.v[1]);
    if (lo || hi) {  // the flag sees the unprojected value (a clamp would hide a NaN)
      flag_nonfinite(xn, p.t, bad);
      if (lo) xn = fmax(xn, lo[j]);
      if (hi) xn = fmin(xn, hi[j]);
    }
    x_out[j] = xn;
    const double xbn = p.omib * pre.xb + p.ib * xn;
    xb[j] = xbn;
    if (p.emit_next) {
      w_out[j] = p.theta_n * (xn - xo) + xn;
      xmd_out[j] = p.omib_n * xbn + p.ib_n * xn;
    }
    flag_nonfinite(xn, p.t, bad);
  }
};

// ---------------------------------------------------------------------------
// Plain y = M x (sparse.hpp:79-88); M' x uses the transposed CSR, which is
// bit-identical to the reference's scatter.
template <bool Strict>
struct SpmvOp {
  static constexpr bool kStrict = Strict;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = true;
  using AccT = Acc<1>;
  CsrView m;
  const double* x;
  double* y;
  StepGate gate{};  // power-iteration batches (engine.cu); default: always open
  __device__ __forceinline__ int len(int r) const { return m.rp[r + 1] - m.rp[r]; }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather* g) const {
    acc.v[0] = seg_dot<Strict, U>(m.v, m.ci, g[0], m.rp[r], lo + lane, hi, stride, acc.v[0]);
  }
  __device__ __forceinline__ const double* gather_src(int) const { return x; }
  struct Pre {};
  __device__ __forceinline__ Pre prefetch(int) const { return Pre{}; }
  __device__ __forceinline__ void finish(int r, const AccT& acc) const { y[r] = acc.v[0]; }
  __device__ __forceinline__ void finish(int r, const AccT& acc, const Pre&) const { y[r] = acc.v[0]; }
};

// ---------------------------------------------------------------------------
// y = M x of the power iteration (opnorm.hpp:44-46) over the rows of a slab
// phase (slab.cuh), so the norm estimate can use the step's plans once they
// are built: K = 1 for the rows of A (gathers x1); K = 2 for the rows of
// [Q | A'] (the primal step's plan), where only segment 2 (A' x2) is kept —
// the Q part is summed and dropped (C4: 1e4 of its 5.2e7 entries).
template <int K>
struct PhaseSpmvOp {
  static constexpr bool kStrict = false;
  static constexpr int kPhase = 0;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = true;
  using AccT = Acc<K>;
  CsrView s1, s2;  // s2: unused for K = 1
  const double* x1;
  const double* x2;
  double* y;
  StepGate gate{};
  int it = 0;
  __device__ __forceinline__ int len(int r) const {
    return (s1.rp[r + 1] - s1.rp[r]) + (K > 1 ? s2.rp[r + 1] - s2.rp[r] : 0);
  }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather* g) const {
    if constexpr (K == 1) {
      acc.v[0] = seg_dot<false, U>(s1.v, s1.ci, g[0], s1.rp[r], lo + lane, hi, stride, acc.v[0]);
    } else {
      const int q0 = s1.rp[r];
      const int L1 = s1.rp[r + 1] - q0;
      const int p = lo + lane;
      acc.v[0] = seg_dot<false, U>(s1.v, s1.ci, g[0], q0, p, hi < L1 ? hi : L1, stride, acc.v[0]);
      acc.v[1] = seg_dot<false, U>(s2.v, s2.ci, g[1], static_cast<int64_t>(s2.rp[r]) - L1,
                                   next_pos(p, stride, L1), hi, stride, acc.v[1]);
    }
  }
  __device__ __forceinline__ const double* gather_src(int slot) const { return slot ? x2 : x1; }
  __host__ __device__ PhaseSpmvOp with_views(CsrView a, CsrView b) const {
    PhaseSpmvOp o = *this;
    o.s1 = a;
    o.s2 = b;
    return o;
  }
  struct Pre {};
  __device__ __forceinline__ Pre prefetch(int) const { return Pre{}; }
  __device__ __forceinline__ void finish(int r, const AccT& acc) const { y[r] = acc.v[K - 1]; }
  __device__ __forceinline__ void finish(int r, const AccT& acc, const Pre&) const { y[r] = acc.v[K - 1]; }
};

// ---------------------------------------------------------------------------
// KKT products, two points (current and average) per matrix pass
// (kkt.hpp:32-39, called twice by evaluate_candidate solver.hpp:255-264).
// Rows of the ORIGINAL stacked A: ax_c = A xu_c, ax_a = A xu_a.
template <bool Strict>
struct KktAxOp {
  static constexpr bool kStrict = Strict;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = false;
  __device__ __forceinline__ const double* gather_src(int) const { return nullptr; }
  using AccT = Acc<2>;
  CsrView a;
  const double2* x;  // (current, average) interleaved
  double* axc;
  double* axa;
  __device__ __forceinline__ int len(int r) const { return a.rp[r + 1] - a.rp[r]; }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather* g) const {
    seg_dot2<Strict, false, U>(a.v, a.ci, x, a.rp[r], lo + lane, hi, stride, 0, acc.v);
  }
  __device__ __forceinline__ void finish(int r, const AccT& acc) const {
    axc[r] = acc.v[0];
    axa[r] = acc.v[1];
  }
};

// Rows j of the ORIGINAL [Q | A']: qx = Q xu, and A'y split into the
// inequality and equality blocks (kkt.hpp:35-38: aty = aty_i + 1.0*aty_e),
// for both points.
template <bool Strict>
struct KktQAtyOp {
  static constexpr bool kStrict = Strict;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = false;
  __device__ __forceinline__ const double* gather_src(int) const { return nullptr; }
  using AccT = Acc<6>;
  CsrView q, at;
  int m_ineq;
  const double2 *x, *y;  // (current, average) interleaved
  double *qxc, *qxa, *atyc, *atya;
  __device__ __forceinline__ int len(int r) const {
    return (q.rp[r + 1] - q.rp[r]) + (at.rp[r + 1] - at.rp[r]);
  }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather* g) const {
    // acc: [0] Qx cur, [1] Qx avg, [2] A_i'y cur, [3] A_i'y avg, [4] A_e'y cur, [5] A_e'y avg
    const int q0 = q.rp[r];
    const int L1 = q.rp[r + 1] - q0;
    const int p = lo + lane;
    seg_dot2<Strict, false, U>(q.v, q.ci, x, q0, p, hi < L1 ? hi : L1, stride, 0, acc.v);
    seg_dot2<Strict, true, U>(at.v, at.ci, y, static_cast<int64_t>(at.rp[r]) - L1,
                           next_pos(p, stride, L1), hi, stride, m_ineq, acc.v + 2);
  }
  __device__ __forceinline__ void finish(int j, const AccT& acc) const {
    qxc[j] = acc.v[0];
    qxa[j] = acc.v[1];
    atyc[j] = acc.v[2] + 1.0 * acc.v[4];
    atya[j] = acc.v[3] + 1.0 * acc.v[5];
  }
};

// ---------------------------------------------------------------------------
// Row measures of the stacked symmetric [[Q, A'], [A, 0]] (scaling.hpp:49-62):
// primal row j = Q row j then A' row j, dual row i = A row i. Kind 0 max-abs,
// 1 l2 (sqrt of sum of squares), 2 l1.
template <bool Strict, int Kind>
struct MeasureOp {
  static constexpr bool kStrict = Strict;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = false;
  __device__ __forceinline__ const double* gather_src(int) const { return nullptr; }
  using AccT = Acc<1, Kind == 0>;
  CsrView s1, s2;  // s2.rp == nullptr: single segment
  double* out;
  __device__ __forceinline__ int len1(int r) const { return s1.rp[r + 1] - s1.rp[r]; }
  __device__ __forceinline__ int len(int r) const {
    return len1(r) + (s2.rp ? s2.rp[r + 1] - s2.rp[r] : 0);
  }
  __device__ __forceinline__ static double term(double acc, double v) {
    const double a = fabs(v);
    if constexpr (Kind == 0) return acc < a ? a : acc;  // std::max(m, a)
    else if constexpr (Kind == 1) return Strict ? __dadd_rn(acc, __dmul_rn(a, a)) : acc + a * a;
    else return acc + a;
  }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather* g) const {
    const int L1 = len1(r);
    int p = lo + lane;
    const int e1 = hi < L1 ? hi : L1;
    for (; p < e1; p += stride) acc.v[0] = term(acc.v[0], s1.v[s1.rp[r] + p]);
    if (s2.rp)
      for (; p < hi; p += stride) acc.v[0] = term(acc.v[0], s2.v[static_cast<int64_t>(s2.rp[r]) - L1 + p]);
  }
  __device__ __forceinline__ void finish(int r, const AccT& acc) const {
    out[r] = Kind == 1 ? sqrt(acc.v[0]) : acc.v[0];
  }
};

// One scaling sweep that first applies the previous pass's factors to the
// working values (apply_pass, scaling.hpp:70: v *= f_row * f_col, the
// product of factors first) and then takes this pass's row measure of the
// scaled values (MeasureOp): the same operations on every entry as an apply
// sweep followed by a measure sweep, in one read and one write of the values.
// Segment s (s1 = Q or A rows, s2 = A' rows): row factor f[ro_s + r], column
// factor f[co_s + col].
template <bool Strict, int Kind>
struct ApplyMeasureOp {
  static constexpr bool kStrict = Strict;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = false;
  __device__ __forceinline__ const double* gather_src(int) const { return nullptr; }
  using AccT = Acc<1, Kind == 0>;
  CsrView s1, s2;  // s2.rp == nullptr: single segment
  double* w1;      // working values of segment 1 / 2 (updated in place)
  double* w2;
  const double* f;
  int ro1, co1, ro2, co2;
  double* out;
  __device__ __forceinline__ int len1(int r) const { return s1.rp[r + 1] - s1.rp[r]; }
  __device__ __forceinline__ int len(int r) const {
    return len1(r) + (s2.rp ? s2.rp[r + 1] - s2.rp[r] : 0);
  }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride,
                                             AccT& acc, const Gather*) const {
    const int L1 = len1(r);
    int p = lo + lane;
    const int e1 = hi < L1 ? hi : L1;
    const double fr1 = f[ro1 + r];
    for (; p < e1; p += stride) {
      const int64_t k = s1.rp[r] + p;
      const double v = w1[k] * (fr1 * f[co1 + s1.ci[k]]);
      w1[k] = v;
      acc.v[0] = MeasureOp<Strict, Kind>::term(acc.v[0], v);
    }
    if (s2.rp) {
      const double fr2 = f[ro2 + r];
      for (; p < hi; p += stride) {
        const int64_t k = static_cast<int64_t>(s2.rp[r]) - L1 + p;
        const double v = w2[k] * (fr2 * f[co2 + s2.ci[k]]);
        w2[k] = v;
        acc.v[0] = MeasureOp<Strict, Kind>::term(acc.v[0], v);
      }
    }
  }
  __device__ __forceinline__ void finish(int r, const AccT& acc) const {
    out[r] = Kind == 1 ? sqrt(acc.v[0]) : acc.v[0];
  }
};

}  // namespace rb
