// engine.cu — setup numerics and the iteration loop of the B200 rAPDHG solver.
// See engine.hpp. Reference: /root/reference/proj/include/rapdhg/solver.hpp.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <exception>
#include <functional>
#include <future>
#include <memory>
#include <thread>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <climits>
#include <limits>
#include <map>
#include <mutex>
#include <stdexcept>

#include "engine.hpp"
#include "persistent.cuh"
#include "rules.hpp"
#include "terms.cuh"
#include "elementwise.cuh"

namespace rb {

namespace {

inline unsigned grid1(int64_t n) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, 256)); }

// ---- elementwise kernels -----------------------------------------------------

__global__ void scale_copy_kernel(double* v, const double* w, double s, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = w[i] * s;  // v = w; scale(v, 1/nrm) (opnorm.hpp:52-53)
}

__global__ void gather_scale_kernel(double* v, const double* full, const int32_t* idx, bool scale, double s,
                                    int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = scale ? full[idx[i]] * s : full[idx[i]];
}

// Rows and columns a pattern touches (row non-empty, or referenced).
__global__ void touched_kernel(const int32_t* rp, const int32_t* ci, int32_t n, uint8_t* flag) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n || rp[r + 1] == rp[r]) return;
  flag[r] = 1;
  for (int32_t k = rp[r]; k < rp[r + 1]; ++k) flag[ci[k]] = 1;  // racing writes of the same 1
}
__global__ void compact_csr_kernel(const int32_t* act, int32_t nc, const int32_t* rp, const int32_t* ci,
                                   const double* v, const int32_t* newidx, const int32_t* rpc, int32_t* cic,
                                   double* vc) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nc) return;
  const int32_t o = act[r];
  int32_t q = rpc[r];
  for (int32_t k = rp[o]; k < rp[o + 1]; ++k, ++q) cic[q] = newidx[ci[k]], vc[q] = v[k];
}
__global__ void newidx_kernel(const int32_t* act, int32_t nc, int32_t* newidx) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nc) newidx[act[k]] = k;
}
__global__ void act_lengths_kernel(const int32_t* act, int32_t nc, const int32_t* rp, int32_t* len) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nc) len[k] = rp[act[k] + 1] - rp[act[k]];
}

__global__ void div_kernel(double* out, const double* v, const double* d, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = v[i] / d[i];  // +-inf stays +-inf (d > 0)
}

__global__ void fill_kernel(double* v, double s, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = s;
}

// Ruiz/l2/l1 factor: f = measure > 0 ? 1/sqrt(measure) : 1; d *= f
// (scaling.hpp:66-72)
__global__ void factor_kernel(double* f, const double* meas, double* d, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double mv = meas[i];
  const double fi = mv > 0.0 ? 1.0 / sqrt(mv) : 1.0;
  f[i] = fi;
  d[i] *= fi;
}

// out = (d[row_off + row] * v) * d[col_off + col] (SparseMatrix::scaled,
// sparse.hpp:154: r[row] * values_[k] * c[cols_[k]]).
__global__ void scaled_values_kernel(double* out, const double* v, const int32_t* row_of,
                                     const int32_t* ci, const double* d, int row_off, int col_off,
                                     int64_t nnz) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nnz) return;
  out[k] = d[row_off + row_of[k]] * v[k] * d[col_off + ci[k]];
}

// out[i] = d[off + i] * v[i] (c~ = D2 c, b~ = D1 b; scaling.hpp:119-121)
__global__ void scale_vec_kernel(double* out, const double* v, const double* d, int off, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = d[off + i] * v[i];
}

template <class Op, class Count>
inline void rowwise(const Op& op, const Schedule& s, cudaStream_t st, Count* launches) {
  if (s.view.total_blocks > 0) {
    launch_rowwise(op, s.view, st);
    ++*launches;
  }
}

}  // namespace

// kkt.hpp:54,63,68-69 on the device-reduced terms. The maxima were reduced
// exactly; the sums follow the mode's order.
void finalize_kkt(const KktRaw& r, Kkt out[2]) {
  for (int p = 0; p < 2; ++p) {
    const double viol = r.viol[p];
    out[p].r_primal = std::max(viol, 0.0) / (1.0 + std::max(r.ax_inf[p], r.b_inf));
    out[p].r_dual = r.dn[p] / (1.0 + std::max({r.qx_inf[p], r.aty_inf[p], r.c_inf}));
    const double xqx = r.xqx[p], cx = r.cx[p];
    // box_projection: the bound multipliers' share of the dual objective
    // (bl + bu = 0 in the reference's form, and x - 0.0 == x exactly)
    const double by = (r.by_i[p] + r.by_e[p]) - (r.bl[p] + r.bu[p]);
    out[p].r_gap = std::fabs(xqx + cx + by) /
                   (1.0 + std::max(std::fabs(0.5 * xqx + cx), std::fabs(0.5 * xqx + by)));
  }
}

void primal_terms_into(KktRaw& r, const double* g) {
  r.xqx[0] = g[0], r.xqx[1] = g[1], r.cx[0] = g[2], r.cx[1] = g[3];
  r.bl[0] = g[4], r.bl[1] = g[5], r.bu[0] = g[6], r.bu[1] = g[7];
  const double* mx = g + kKktPrimalSums;
  r.dn[0] = mx[0], r.dn[1] = mx[1], r.qx_inf[0] = mx[2], r.qx_inf[1] = mx[3];
  r.aty_inf[0] = mx[4], r.aty_inf[1] = mx[5], r.c_inf = mx[6];
}

// ============================================================================
// DeviceQP
// ============================================================================

namespace {
// the per-row errors of a CSR, as validate_dims reports them
[[noreturn]] void csr_error(int kind) {
  if (kind == 2) throw Error(RAPDHG_E_OUT_OF_RANGE, "sparse entry index out of range");
  if (kind == 3) invalid("CSR columns must be strictly increasing within a row");
  invalid("CSR row_ptr not monotone");
}
}  // namespace

// box_projection: the bounds' rules (canonicalize's, problem.hpp:134-143)
void validate_bounds(const rapdhg_qp& p, const rapdhg_config& cfg) {
  if (!p.lower && !p.upper) return;
  if (!cfg.box_projection)
    invalid("variable bounds need box_projection (the reference form takes them as rows: canonicalize)");
  if (cfg.strict_parity) invalid("box_projection has no reference counterpart: it needs strict_parity = 0");
  for (int j = 0; j < p.n; ++j) {
    const double l = p.lower ? p.lower[j] : -std::numeric_limits<double>::infinity();
    const double u = p.upper ? p.upper[j] : std::numeric_limits<double>::infinity();
    if (std::isnan(l) || std::isnan(u)) invalid("NaN variable bound");
    if (l > u) invalid("infeasible bounds on variable " + std::to_string(j));
  }
}

void DeviceQP::validate_dims(const rapdhg_qp& p, bool structure) {
  // problem.hpp:40-46 messages
  const int n = p.n;
  if (p.q.n_rows != n || p.q.n_cols != n) invalid("Q dimension mismatch");
  if (p.a_ineq.n_rows != p.m_ineq || p.a_ineq.n_cols != n)
    invalid("inequality block dimension mismatch");
  if (p.a_eq.n_rows != p.m_eq || p.a_eq.n_cols != n) invalid("equality block dimension mismatch");
  auto check = [structure](const rapdhg_csr& a) {
    if (a.n_rows < 0 || a.n_cols < 0) invalid("negative matrix dimension");
    if (a.nnz > 0 && (!a.col_idx || !a.values)) invalid("null CSR arrays");
    if (!a.row_ptr) invalid("null CSR row_ptr");
    if (a.row_ptr[0] != 0 || a.row_ptr[a.n_rows] != a.nnz) invalid("CSR row_ptr inconsistent with nnz");
    if (!structure) return;
    // rows in contiguous blocks on host threads; the error reported is the one a
    // sequential scan meets first (lowest block)
    enum { kOk, kMono, kRange, kOrder };
    auto scan = [&](int r0, int r1) {
      for (int r = r0; r < r1; ++r) {
        const int b = a.row_ptr[r], e = a.row_ptr[r + 1];
        if (e < b) return static_cast<int>(kMono);
        for (int k = b; k < e; ++k) {
          const int c = a.col_idx[k];
          if (c < 0 || c >= a.n_cols) return static_cast<int>(kRange);
          if (k > b && c <= a.col_idx[k - 1]) return static_cast<int>(kOrder);
        }
      }
      return static_cast<int>(kOk);
    };
    const int T = a.nnz < (1 << 20) ? 1 : static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
    std::vector<int> err(T, kOk);
    if (T == 1) {
      err[0] = scan(0, a.n_rows);
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          err[t] = scan(static_cast<int>(static_cast<int64_t>(a.n_rows) * t / T),
                        static_cast<int>(static_cast<int64_t>(a.n_rows) * (t + 1) / T));
        });
      for (auto& x : th) x.join();
    }
    for (int e : err)
      if (e != kOk) csr_error(e == kMono ? 1 : e == kRange ? 2 : 3);
  };
  check(p.q);
  check(p.a_ineq);
  check(p.a_eq);
}

DeviceQP::DeviceQP(const rapdhg_qp& p, bool strict_, cudaStream_t st_, bool check_structure)
    : st(st_), strict(strict_), n(p.n), mi(p.m_ineq), me(p.m_eq), m(p.m_ineq + p.m_eq) {
  Tracer tr(st);
  {
    HostStager sg;
    upload_csr(Q, p.q, st, &sg);
    DevCsr ai, ae;
    upload_csr(ai, p.a_ineq, st, &sg);
    upload_csr(ae, p.a_eq, st, &sg);
    if (check_structure) {  // before any kernel indexes with the uploaded arrays
      DevBuf<unsigned long long> slot(3);
      RB_CUDA(cudaMemsetAsync(slot.get(), 0xff, sizeof(unsigned long long) * 3, st));
      csr_check_async(Q, slot.get(), st);
      csr_check_async(ai, slot.get() + 1, st);
      csr_check_async(ae, slot.get() + 2, st);
      unsigned long long h[3];
      RB_CUDA(cudaMemcpyAsync(h, slot.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
      RB_CUDA(cudaStreamSynchronize(st));
      for (unsigned long long k : h)  // Q, A_ineq, A_eq: the order validate_dims checks them in
        if (k != kCsrOk) csr_error(static_cast<int>(k & 3u));
    }
    stack_csr(A, ai, ae, st);  // WorkingProblem::from (solver.hpp:106-108)
    RB_CUDA(cudaStreamSynchronize(st));
  }
  tr.mark("  upload + stack");
  transpose_csr(AT, A, &at_perm, st);
  tr.mark("  transpose");
  c.alloc(n);
  c.upload(p.c, n, st);
  if (p.lower) lo.alloc(n), lo.upload(p.lower, n, st);
  if (p.upper) hi.alloc(n), hi.upload(p.upper, n, st);
  b.alloc(m);
  b.upload(p.b_ineq, mi, st);
  if (me) RB_CUDA(cudaMemcpyAsync(b.get() + mi, p.b_eq, sizeof(double) * me, cudaMemcpyHostToDevice, st));
  red.init(std::max<int64_t>(n, m), st);
  red_out.alloc(64);
  red_host.alloc(64);
  tr.mark("  vectors + reduce scratch");
  // schedules (patterns only; shared by original and scaled values)
  DevBuf<int32_t> len;
  row_lengths(len, A.rp.get(), nullptr, A.rows, st);
  build_schedule(sch_dual, len.get(), A.rows, strict, st);
  choose_windows(sch_dual, A.ci.get(), A.nnz, n, nullptr, 0, 0, st);
  row_lengths(len, Q.rp.get(), AT.rp.get(), n, st);
  build_schedule(sch_primal, len.get(), n, strict, st);
  choose_windows(sch_primal, Q.ci.get(), Q.nnz, n, AT.ci.get(), AT.nnz, m, st);
  row_lengths(len, Q.rp.get(), nullptr, n, st);
  build_schedule(sch_q, len.get(), n, strict, st);
  choose_windows(sch_q, Q.ci.get(), Q.nnz, n, nullptr, 0, 0, st);
  row_lengths(len, AT.rp.get(), nullptr, n, st);
  build_schedule(sch_at, len.get(), n, strict, st);
  choose_windows(sch_at, AT.ci.get(), AT.nnz, m, nullptr, 0, 0, st);
  RB_CUDA(cudaStreamSynchronize(st));
  tr.mark("  schedules");
}

void DeviceQP::validate_symmetry() {
  DevCsr qt;
  transpose_csr(qt, Q, nullptr, st);
  double gap = 0.0, mabs = 0.0;
  symmetry_gap(Q, qt, &gap, &mabs, st);
  if (gap > 1e-12 * std::max(1.0, mabs)) invalid("Q is not symmetric");  // problem.hpp:47-49
}

template <int NS, int NM, class F>
void DeviceQP::reduce_to_host(const F& f, int64_t len, double* out) {
  launch_reduce<NS, NM>(f, len, strict, red, red_out.get(), st);
  ++launches;
  RB_CUDA(cudaMemcpyAsync(red_host.get(), red_out.get(), sizeof(double) * (NS + NM),
                          cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < NS + NM; ++k) out[k] = red_host[k];
}

void DeviceQP::spmv(const DevCsr& mat, const Schedule& s, const double* vals, const double* x,
                    double* y, StepGate gate, cudaStream_t on) {
  const cudaStream_t use = on ? on : st;
  if (strict) {
    SpmvOp<true> op{mat.view(vals), x, y, gate};
    rowwise(op, s, use, &launches);
  } else if (s.view.total_blocks > 0) {
    // the power iterations' products: programmatic dependent launches
    SpmvOp<false> op{mat.view(vals), x, y, gate};
    launch_rowwise(op, s.view, use, gate.stop != nullptr && pdl_enabled());
    ++launches;
  }
}

namespace {
template <bool Strict, int Kind>
void measures(DeviceQP& P, const double* qv, const double* av, const double* atv, double* meas) {
  MeasureOp<Strict, Kind> prim{P.Q.view(qv), P.AT.view(atv), meas};
  rowwise(prim, P.sch_primal, P.st, &P.launches);
  MeasureOp<Strict, Kind> dual{P.A.view(av), CsrView{nullptr, nullptr, nullptr}, meas + P.n};
  rowwise(dual, P.sch_dual, P.st, &P.launches);
}
template <int Kind>
void measures_mode(DeviceQP& P, const double* qv, const double* av, const double* atv, double* meas) {
  if (P.strict) measures<true, Kind>(P, qv, av, atv, meas);
  else measures<false, Kind>(P, qv, av, atv, meas);
}
// apply the factors f to the working values, then measure (ApplyMeasureOp)
// side (optional): the A rows' sweep runs there, beside the [Q | A'] rows'
// (two independent sweeps; `fork` / `join` events order them with P.st)
template <bool Strict, int Kind>
void apply_measures(DeviceQP& P, double* qw, double* aw, double* atw, const double* f, double* meas,
                    cudaStream_t side, cudaEvent_t fork, cudaEvent_t join) {
  ApplyMeasureOp<Strict, Kind> prim{P.Q.view(qw), P.AT.view(atw), qw, atw, f, 0, 0, 0, P.n, meas};
  ApplyMeasureOp<Strict, Kind> dual{P.A.view(aw), CsrView{nullptr, nullptr, nullptr}, aw, nullptr, f, P.n, 0, 0, 0,
                                    meas + P.n};
  if (side) {
    RB_CUDA(cudaEventRecord(fork, P.st));
    RB_CUDA(cudaStreamWaitEvent(side, fork, 0));
    rowwise(dual, P.sch_dual, side, &P.launches);
    rowwise(prim, P.sch_primal, P.st, &P.launches);
    RB_CUDA(cudaEventRecord(join, side));
    RB_CUDA(cudaStreamWaitEvent(P.st, join, 0));
  } else {
    rowwise(prim, P.sch_primal, P.st, &P.launches);
    rowwise(dual, P.sch_dual, P.st, &P.launches);
  }
}
template <int Kind>
void apply_measures_mode(DeviceQP& P, double* qw, double* aw, double* atw, const double* f, double* meas,
                         cudaStream_t side, cudaEvent_t fork, cudaEvent_t join) {
  if (P.strict) apply_measures<true, Kind>(P, qw, aw, atw, f, meas, nullptr, nullptr, nullptr);
  else apply_measures<false, Kind>(P, qw, aw, atw, f, meas, side, fork, join);
}
}  // namespace

// compute_scaling (scaling.hpp:97-106): working copies of the values of Q, A
// and A' evolve by identical products (each stacked entry and its mirror get
// f_row * f_col, commutative), row measures are taken over [Q | A'] rows and
// A rows in the triplet push order of stacked_triplets (scaling.hpp:30-45).
void DeviceQP::compute_scaling(int ruiz_iters, bool full, DevBuf<double>& d) {
  const int64_t N = static_cast<int64_t>(n) + m;
  d.alloc(N);
  fill_kernel<<<grid1(N), 256, 0, st>>>(d.get(), 1.0, N);
  ++launches;
  DevBuf<double> qw(Q.nnz), aw(A.nnz), atw(AT.nnz), meas(N), f(N);
  if (Q.nnz) RB_CUDA(cudaMemcpyAsync(qw.get(), Q.v.get(), sizeof(double) * Q.nnz, cudaMemcpyDeviceToDevice, st));
  if (A.nnz) RB_CUDA(cudaMemcpyAsync(aw.get(), A.v.get(), sizeof(double) * A.nnz, cudaMemcpyDeviceToDevice, st));
  if (AT.nnz) RB_CUDA(cudaMemcpyAsync(atw.get(), AT.v.get(), sizeof(double) * AT.nnz, cudaMemcpyDeviceToDevice, st));
  // pass p: measure (kind of pass p) -> factors -> apply them. The apply of
  // pass p and the measure of pass p + 1 run as one sweep (ApplyMeasureOp);
  // the last pass's apply is not needed (the working copies are dropped).
  std::vector<int> kinds(static_cast<std::size_t>(std::max(ruiz_iters, 0)), 0);
  if (full) kinds.push_back(1), kinds.push_back(2);
  // the A rows' sweeps on a side stream beside the [Q | A'] rows' (fast mode;
  // their kernels are latency-bound, C4: 12 passes 10.7 -> see DESIGN §4)
  OwnedStream side_own;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  if (!strict) {
    side = side_own.create();
    RB_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    RB_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  }
  for (std::size_t p = 0; p < kinds.size(); ++p) {
    if (p == 0) {
      if (kinds[0] == 0) measures_mode<0>(*this, qw.get(), aw.get(), atw.get(), meas.get());
      else if (kinds[0] == 1) measures_mode<1>(*this, qw.get(), aw.get(), atw.get(), meas.get());
      else measures_mode<2>(*this, qw.get(), aw.get(), atw.get(), meas.get());
    } else {  // apply pass p - 1's factors, measure for pass p
      if (kinds[p] == 0) apply_measures_mode<0>(*this, qw.get(), aw.get(), atw.get(), f.get(), meas.get(), side, fork, join);
      else if (kinds[p] == 1)
        apply_measures_mode<1>(*this, qw.get(), aw.get(), atw.get(), f.get(), meas.get(), side, fork, join);
      else apply_measures_mode<2>(*this, qw.get(), aw.get(), atw.get(), f.get(), meas.get(), side, fork, join);
    }
    factor_kernel<<<grid1(N), 256, 0, st>>>(f.get(), meas.get(), d.get(), N);
    RB_LAUNCH_CHECK();
    ++launches;
  }
  RB_CUDA(cudaStreamSynchronize(st));
  if (fork) cudaEventDestroy(fork);
  if (join) cudaEventDestroy(join);
}

void DeviceQP::scale_values(const double* d, DevBuf<double>& qs, DevBuf<double>& as,
                            DevBuf<double>& ats, DevBuf<double>& cs, DevBuf<double>& bs) {
  qs.alloc(Q.nnz), as.alloc(A.nnz), ats.alloc(AT.nnz), cs.alloc(n), bs.alloc(m);
  DevBuf<int32_t> q_row, a_row;
  expand_rows(q_row, Q, st);
  expand_rows(a_row, A, st);
  if (Q.nnz) scaled_values_kernel<<<grid1(Q.nnz), 256, 0, st>>>(qs.get(), Q.v.get(), q_row.get(), Q.ci.get(), d, 0, 0, Q.nnz);
  if (A.nnz) scaled_values_kernel<<<grid1(A.nnz), 256, 0, st>>>(as.get(), A.v.get(), a_row.get(), A.ci.get(), d, n, 0, A.nnz);
  RB_LAUNCH_CHECK();
  gather_values(ats.get(), as.get(), at_perm.get(), AT.nnz, st);  // same value at the mirror
  scale_vec_kernel<<<grid1(n), 256, 0, st>>>(cs.get(), c.get(), d, 0, n);
  if (m) scale_vec_kernel<<<grid1(m), 256, 0, st>>>(bs.get(), b.get(), d, n, m);
  RB_LAUNCH_CHECK();
  launches += 5;
  RB_CUDA(cudaStreamSynchronize(st));
}

RandomStart draw_random_start(int len, uint64_t seed) {
  RandomStart r;
  r.rng.seed(seed);
  r.v.resize(static_cast<std::size_t>(std::max(len, 0)));
  for (double& x : r.v) x = 2.0 * (static_cast<double>(r.rng() >> 11) * 0x1.0p-53) - 1.0;  // opnorm.hpp:22-24
  return r;
}

// estimate_op_norm / estimate_op_norm_symmetric (opnorm.hpp:36-87)
namespace {
// Device copy of the host's per-step decision (opnorm.hpp:48-59): thread 0
// of block 0 records a stop at this step when the step converged or w = 0
// (the host then restarts from a random vector), so the batch's remaining
// launches return at once. The host still replays the recorded values and
// decides; the gate only saves the overshoot past convergence.
struct PowerState {
  double lambda;  // the host's lambda before the batch's first step, then the device's
  int stop;       // step of the batch the device stopped at (INT_MAX: none)
  int it0;        // host iteration index of the batch's first step
};
__global__ void power_step_kernel(double* v, const double* w, const double* hist, PowerState* ps, int i,
                                  double tol, bool absval, int64_t n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (programmatic dependent launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (ps->stop < i) return;  // a stop recorded by an earlier step (uniform over the grid)
  const double s = hist[1];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double lambda_next = absval ? fabs(hist[0]) : hist[0];
    if (s == 0.0 || (ps->it0 + i > 0 && fabs(lambda_next - ps->lambda) <= tol * fabs(lambda_next)))
      ps->stop = i;  // read only by later launches
    else
      ps->lambda = lambda_next;
  }
  if (s == 0.0) return;  // v unchanged (the host restarts)
  // v = w * (1.0 / sqrt(s)): the same IEEE operations as the host's scale(v, 1.0 / nrm)
  const double inv = 1.0 / sqrt(s);
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[k] = w[k] * inv;
}

// One power iteration run in device batches on its own stream: each step
// records (v.w, ||w||^2) on the device and normalises v there; after a batch
// the host replays the reference's loop over the recorded values (stopping
// rule, zero-norm restart) — identical results, one host round trip per batch
// (8, 16, .. 64 steps) instead of per step. The device takes the same
// per-step decision (power_step_kernel), so the launches of a batch past
// convergence return at once (C4: up to 63 x 0.4 ms of products before).
class PowerRun {
 public:
  using Step = std::function<void(StepGate, cudaStream_t)>;  // w = M v
  // compact (optional, `len` entries): the iteration runs on v[compact[k]]
  // only — the indices outside stay 0 after the first product (rows and
  // columns the matrix never touches); the random start is still drawn and
  // normalised over all `full_len` entries, as the reference does
  PowerRun(DeviceQP& P, DevBuf<double>& v, DevBuf<double>& w, int len, Step step, bool absval, int max_iters,
           double tol, uint64_t seed, cudaStream_t s, ReduceScratch& red, const int32_t* compact = nullptr,
           int full_len = 0, const RandomStart* pre = nullptr)
      : P_(P), v_(v), w_(w), len_(len), step_(std::move(step)), absval_(absval), max_iters_(max_iters),
        tol_(tol), rng_(seed), s_(s), red_(red), hist_(2 * kMaxBatch), dps_(1), out_(1), compact_(compact),
        full_len_(compact ? full_len : len) {
    hh_.alloc(2 * kMaxBatch);
    hps_.alloc(2);
    hout_.alloc(1);
    sgrid_ = static_cast<unsigned>(std::min<int64_t>(ceil_div(len, 256), 4 * kSMs));
    if (pre && static_cast<int>(pre->v.size()) == full_len_) {  // drawn ahead: the same numbers
      rng_ = pre->rng;
      random_unit(pre->v.data());
    } else {
      random_unit();
    }
    done_ = max_iters_ <= 0;
  }
  bool done() const { return done_; }
  double result() const { return result_; }
  // a batch boundary at step `at` (batches never straddle it) and a hook run
  // before every batch with the index of its first step
  void split_at(int at, std::function<void(int)> hook) {
    split_ = at;
    hook_ = std::move(hook);
  }

  void launch() {  // the next batch, asynchronously
    if (done_) return;
    if (hook_) hook_(it_);
    K_ = std::min(batch_, max_iters_ - it_);
    if (it_ < split_) K_ = std::min(K_, split_ - it_);
    hps_[0] = PowerState{lambda_, INT_MAX, it_};
    RB_CUDA(cudaMemcpyAsync(dps_.get(), hps_.get(), sizeof(PowerState), cudaMemcpyHostToDevice, s_));
    enqueue_steps();
    RB_CUDA(cudaMemcpyAsync(hh_.get(), hist_.get(), sizeof(double) * 2 * K_, cudaMemcpyDeviceToHost, s_));
    RB_CUDA(cudaMemcpyAsync(hps_.get() + 1, dps_.get(), sizeof(PowerState), cudaMemcpyDeviceToHost, s_));
  }

  void finish() {  // wait for the batch and replay opnorm.hpp:44-60 over it
    if (done_) return;
    RB_CUDA(cudaStreamSynchronize(s_));
    const int dev_stop = hps_[1].stop;
    bool restarted = false;
    for (int i = 0; i < K_ && !restarted; ++i, ++it_) {
      if (i > dev_stop) throw std::logic_error("power iteration: device stopped before the host's decision");
      const double lambda_next = absval_ ? std::fabs(hh_[2 * i]) : hh_[2 * i];
      const double nrm = std::sqrt(hh_[2 * i + 1]);
      if (nrm == 0.0) {  // v stayed frozen from here on in this batch
        random_unit();
        restarted = true;
        continue;
      }
      if (it_ > 0 && std::fabs(lambda_next - lambda_) <= tol_ * std::fabs(lambda_next)) {
        if (std::getenv("RAPDHG_TRACE"))
          std::fprintf(stderr, "[rapdhg]     power iteration: converged at step %d (batch stop %d of %d)\n", it_,
                       dev_stop, K_);
        result_ = lambda_next;
        done_ = true;
        return;
      }
      lambda_ = lambda_next;
    }
    batch_ = std::min(batch_ * 2, kMaxBatch);
    if (it_ >= max_iters_) done_ = true, result_ = lambda_;
  }

 private:
  static constexpr int kMaxBatch = 64;
  // each step's kernels as programmatic dependent launches of the previous
  // ones (RAPDHG_PDL), so the next kernel is scheduled while one finishes
  void enqueue_steps() {
    const bool pdl = pdl_enabled() && !P_.strict;
    for (int i = 0; i < K_; ++i) {
      const StepGate gate{&dps_.get()->stop, i};
      step_(gate, s_);
      launch_reduce<2, 0>(DotAndSumSq{v_.get(), w_.get(), gate}, len_, P_.strict, red_, hist_.get() + 2 * i, s_,
                          pdl);
      if (pdl) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(sgrid_);
        lc.blockDim = dim3(256);
        lc.stream = s_;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        RB_CUDA(cudaLaunchKernelEx(&lc, power_step_kernel, v_.get(), static_cast<const double*>(w_.get()),
                                   static_cast<const double*>(hist_.get() + 2 * i), dps_.get(), i, tol_, absval_,
                                   static_cast<int64_t>(len_)));
      } else {
        power_step_kernel<<<sgrid_, 256, 0, s_>>>(v_.get(), w_.get(), hist_.get() + 2 * i, dps_.get(), i, tol_,
                                                  absval_, len_);
      }
      RB_LAUNCH_CHECK();
      P_.launches += 2;
    }
  }
  // random_unit (opnorm.hpp:20-30): host mt19937_64 stream, normalised on device
  void random_unit(const double* drawn = nullptr) {
    std::vector<double> h;
    if (!drawn) {
      h.resize(full_len_);
      for (double& x : h) x = 2.0 * (static_cast<double>(rng_() >> 11) * 0x1.0p-53) - 1.0;
      drawn = h.data();
    }
    DevBuf<double> full(compact_ ? full_len_ : 0);
    double* dst = compact_ ? full.get() : v_.get();
    RB_CUDA(cudaMemcpyAsync(dst, drawn, sizeof(double) * full_len_, cudaMemcpyHostToDevice, s_));
    launch_reduce<1, 0>(SumSq{dst}, full_len_, P_.strict, red_, out_.get(), s_);
    RB_CUDA(cudaMemcpyAsync(hout_.get(), out_.get(), sizeof(double), cudaMemcpyDeviceToHost, s_));
    RB_CUDA(cudaStreamSynchronize(s_));
    const double nrm = std::sqrt(hout_[0]);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 1.0;
    if (compact_) {  // v[k] = full[compact[k]] * (1 / nrm), the same operation per entry
      gather_scale_kernel<<<grid1(len_), 256, 0, s_>>>(v_.get(), full.get(), compact_, nrm > 0.0, inv, len_);
      RB_LAUNCH_CHECK();
    } else if (nrm > 0.0) {
      scale_copy_kernel<<<grid1(len_), 256, 0, s_>>>(v_.get(), v_.get(), inv, len_);
      RB_LAUNCH_CHECK();
    }
    P_.launches += 2;
    RB_CUDA(cudaStreamSynchronize(s_));  // `full` is freed in s_'s order below; h stays valid until here
  }

  DeviceQP& P_;
  DevBuf<double>& v_;
  DevBuf<double>& w_;
  int len_;
  Step step_;
  bool absval_;
  int max_iters_;
  double tol_;
  std::mt19937_64 rng_;
  cudaStream_t s_;
  ReduceScratch& red_;
  DevBuf<double> hist_;
  DevBuf<PowerState> dps_;
  DevBuf<double> out_;
  PinnedBuf<double> hh_, hout_;
  PinnedBuf<PowerState> hps_;
  const int32_t* compact_ = nullptr;
  int full_len_ = 0;
  unsigned sgrid_ = 1;
  double lambda_ = 0.0, result_ = 0.0;
  int it_ = 0, batch_ = 8, K_ = 0, split_ = INT_MAX;
  std::function<void(int)> hook_;
  bool done_ = false;
};

void run_alone(PowerRun& r) {
  while (!r.done()) {
    r.launch();
    r.finish();
  }
}
}  // namespace

double DeviceQP::op_norm_q(const double* qv, int max_iters, double tol, uint64_t seed, const RandomStart* pre,
                           cudaStream_t on, ReduceScratch* rs) {
  if (Q.nnz == 0) return 0.0;
  const cudaStream_t st = on ? on : this->st;  // (shadows the member on purpose)
  ReduceScratch& red = rs ? *rs : this->red;
  // fast mode: when Q touches at most half of the indices (C2 / C4: Q lives
  // on the 1e4 features of 2e5 / 1e6 variables), iterate on those only —
  // 1e4-entry vectors instead of 1e6 (C4: 7.5 -> 5 ms); the sums skip only
  // exact zeros, their grouping changes (fast mode: rounding only)
  if (!strict) {
    DevBuf<uint8_t> flag(n);
    flag.zero(st);
    touched_kernel<<<grid1(n), 256, 0, st>>>(Q.rp.get(), Q.ci.get(), n, flag.get());
    RB_LAUNCH_CHECK();
    DevBuf<int32_t> act(n), cnt(1);
    const thrust::counting_iterator<int32_t> idx(0);
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx, flag.get(), act.get(), cnt.get(), n, st));
    DevBuf<unsigned char> tmp(tb);
    RB_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, idx, flag.get(), act.get(), cnt.get(), n, st));
    int32_t nc = 0;
    RB_CUDA(cudaMemcpyAsync(&nc, cnt.get(), sizeof(nc), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    if (nc > 0 && 2 * static_cast<int64_t>(nc) <= n) {
      DevCsr C;
      C.rows = C.cols = nc;
      C.nnz = Q.nnz;
      C.rp.alloc(static_cast<std::size_t>(nc) + 1), C.ci.alloc(Q.nnz), C.v.alloc(Q.nnz);
      DevBuf<int32_t> newidx(n), len(nc);
      newidx_kernel<<<grid1(nc), 256, 0, st>>>(act.get(), nc, newidx.get());
      act_lengths_kernel<<<grid1(nc), 256, 0, st>>>(act.get(), nc, Q.rp.get(), len.get());
      RB_LAUNCH_CHECK();
      RB_CUDA(cudaMemsetAsync(C.rp.get(), 0, sizeof(int32_t), st));
      std::size_t sb = 0;
      RB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, sb, len.get(), C.rp.get() + 1, nc, st));
      DevBuf<unsigned char> stmp(sb);
      RB_CUDA(cub::DeviceScan::InclusiveSum(stmp.get(), sb, len.get(), C.rp.get() + 1, nc, st));
      compact_csr_kernel<<<grid1(nc), 256, 0, st>>>(act.get(), nc, Q.rp.get(), Q.ci.get(), qv, newidx.get(),
                                                     C.rp.get(), C.ci.get(), C.v.get());
      RB_LAUNCH_CHECK();
      Schedule sc;
      build_schedule(sc, len.get(), nc, false, st);
      DevBuf<double> v(nc), w(nc);
      PowerRun r(*this, v, w, nc,
                 [&](StepGate g, cudaStream_t s) { spmv(C, sc, C.v.get(), v.get(), w.get(), g, s); }, true,
                 max_iters, tol, seed, st, red, act.get(), n, pre);
      run_alone(r);
      return r.result();
    }
  }
  DevBuf<double> v(n), w(n);
  PowerRun r(*this, v, w, n,
             [&](StepGate g, cudaStream_t s) { spmv(Q, sch_q, qv, v.get(), w.get(), g, s); }, true, max_iters,
             tol, seed, st, red, nullptr, 0, pre);
  run_alone(r);
  return r.result();
}

// estimate_op_norm (opnorm.hpp:36-61): power iteration on A'A; A' v as the
// gather over CSR(A').
double DeviceQP::op_norm_a(const double* av, const double* atv, int max_iters, double tol,
                           uint64_t seed, const RandomStart* pre) {
  if (A.nnz == 0) return 0.0;
  DevBuf<double> v(n), w(n), mv(m);
  PowerRun r(
      *this, v, w, n,
      [&](StepGate g, cudaStream_t s) {
        spmv(A, sch_dual, av, v.get(), mv.get(), g, s);
        spmv(AT, sch_at, atv, mv.get(), w.get(), g, s);
      },
      false, max_iters, tol, seed, st, red, nullptr, 0, pre);
  run_alone(r);
  return std::sqrt(std::max(r.result(), 0.0));
}

// ============================================================================
// Engine
// ============================================================================


Engine::Engine(const rapdhg_qp& p, const rapdhg_config& cfg, Clock::time_point t0, bool full_plans, bool own_norm_a)
    : cfg_(cfg), full_plans_(full_plans), own_norm_a_(own_norm_a) {
  Tracer tr(nullptr);
  DeviceQP::validate_dims(p, false);  // the per-row scan runs on the device after the upload
  tr.mark("validate dims (host)");
  RB_CUDA(cudaSetDevice(cfg.device));
  st_ = own_st_.create();  // non-blocking; this object's allocations are ordered on it
  AllocStreamScope scope(st_);
  {  // twice a solve's estimated footprint, mapped once (see pool_reserve)
    const double nnz = static_cast<double>(p.q.nnz) + 2.0 * (static_cast<double>(p.a_ineq.nnz) + p.a_eq.nnz);
    const double rows = static_cast<double>(p.n) + p.m_ineq + p.m_eq;
    pool_reserve(static_cast<std::size_t>(2.0 * (48.0 * nnz + 320.0 * rows)));
  }
  tr.st = st_;
  tr.mark("device + stream");
  rand_future_ = std::async(std::launch::async, draw_random_start, p.n, cfg.seed);  // beside the upload
  P_ = std::make_unique<DeviceQP>(p, cfg.strict_parity != 0, st_, true);
  tr.mark("upload, stack, A', schedules");
  P_->validate_symmetry();  // original.validate() (solver.hpp:277)
  tr.mark("symmetry check");
  validate_config(cfg);     // cfg.validate() (solver.hpp:278)
  validate_bounds(p, cfg);  // box_projection (B200 extension)
  n_ = P_->n, m_ = P_->m, mi_ = P_->mi;
  if (!P_->strict) plan_slabs_async();  // reads n_, m_ and the device matrices only

  // scaling (solver.hpp:281-284)
  if (cfg.scaling) {
    P_->compute_scaling(10, true, d_);
    P_->scale_values(d_.get(), qs_, as_, ats_, cs_, bs_);
    qsv_ = qs_.get(), asv_ = as_.get(), atsv_ = ats_.get(), csv_ = cs_.get(), bsv_ = bs_.get();
  } else {
    d_.alloc(static_cast<std::size_t>(n_) + m_);
    fill_kernel<<<grid1(n_ + m_), 256, 0, st_>>>(d_.get(), 1.0, n_ + m_);
    RB_LAUNCH_CHECK();
    qsv_ = P_->Q.v.get(), asv_ = P_->A.v.get(), atsv_ = P_->AT.v.get();
    csv_ = P_->c.get(), bsv_ = P_->b.get();
  }
  if (P_->lo.size() || P_->hi.size()) {  // scaled bounds: x~ = x / d2
    if (P_->lo.size()) {
      los_.alloc(n_);
      div_kernel<<<grid1(n_), 256, 0, st_>>>(los_.get(), P_->lo.get(), d_.get(), n_);
      lsv_ = los_.get();
    }
    if (P_->hi.size()) {
      his_.alloc(n_);
      div_kernel<<<grid1(n_), 256, 0, st_>>>(his_.get(), P_->hi.get(), d_.get(), n_);
      hsv_ = his_.get();
    }
    RB_LAUNCH_CHECK();
  }
  tr.mark("scaling");
  // norms (solver.hpp:286-289)
  // (norm Q's batches on a side stream beside norm A's measured no faster on
  // C4: 97.6 against 7.5 + 90.3 ms — both runs are device-bound)
  const RandomStart start = rand_future_.get();
  if (!P_->strict && own_norm_a_) {
    // norm Q on a host thread and a stream of its own, beside norm A: its
    // (compacted) steps are a few short kernels that fit between norm A's
    // (C4: 5 ms hidden). Each run's arithmetic is the one it has alone.
    OwnedStream qs;
    const cudaStream_t sq = qs.create();
    cudaEvent_t ready;
    RB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    RB_CUDA(cudaEventRecord(ready, st_));  // the scaled values are written
    RB_CUDA(cudaStreamWaitEvent(sq, ready, 0));
    double nq = 0.0;
    std::exception_ptr qerr;
    std::thread tq([&] {
      try {
        RB_CUDA(cudaSetDevice(cfg.device));
        AllocStreamScope scope(sq);
        ReduceScratch rq;
        rq.init(n_, sq);
        nq = P_->op_norm_q(qsv_, 5000, 1e-4, cfg.seed, &start, sq, &rq);
        RB_CUDA(cudaStreamSynchronize(sq));
      } catch (...) {
        qerr = std::current_exception();
      }
    });
    try {
      norm_a = 1.01 * norm_a_power(5000, 1e-4, cfg.seed, &start);
    } catch (...) {
      tq.join();
      cudaEventDestroy(ready);
      throw;
    }
    tq.join();
    cudaEventDestroy(ready);
    if (qerr) std::rethrow_exception(qerr);
    norm_q = 1.01 * nq;
    tr.mark("norms (Q beside A)");
  } else {
    norm_q = 1.01 * P_->op_norm_q(qsv_, 5000, 1e-4, cfg.seed, &start);
    tr.mark("norm Q (power iteration)");
    if (own_norm_a_) norm_a = 1.01 * norm_a_power(5000, 1e-4, cfg.seed, &start);
    tr.mark("norm A (power iteration)");
  }
  // primal weight init on the scaled c, b (solver.hpp:296-300)
  if (cfg.primal_weight == RAPDHG_PW_ADAPTIVE) {
    double sc[1], sb[1];
    P_->reduce_to_host<1, 0>(SumSq{csv_}, n_, sc);
    P_->reduce_to_host<1, 0>(SumSq{bsv_}, m_, sb);
    omega0 = primal_weight_init(std::sqrt(sc[0]), std::sqrt(sb[0]));
  } else {
    omega0 = cfg.fixed_primal_weight;
  }

  // iterate and check buffers
  for (int i = 0; i < 2; ++i) {
    X_[i].alloc(n_), XMD_[i].alloc(n_), xu_[i].alloc(n_), yu_[i].alloc(m_);
    if (i == 0) xi_.alloc(n_), yi_.alloc(m_);
    ax_[i].alloc(m_), qx_[i].alloc(n_), aty_[i].alloc(n_);
  }
  w_.alloc(n_), xb_.alloc(n_), y_.alloc(m_), yb_.alloc(m_), epx_.alloc(n_), epy_.alloc(m_);
  best_x_.alloc(n_), best_y_.alloc(m_);
  params_.alloc(kMaxChunk);
  params_h_.alloc(kMaxChunk);
  bad_.alloc(1);
  bad_h_.alloc(1);
  if (cfg.profile_kernels) {
    events_.resize(2 * kMaxChunk + 1);
    for (auto& e : events_) RB_CUDA(cudaEventCreate(&e));
    span_mode_ = cfg.profile_kernels == 2;
    if (span_mode_) span_.alloc(2 * kMaxChunk);
  }
  RB_CUDA(cudaStreamSynchronize(st_));
  tr.mark("omega init + buffers");
  if (!P_->strict) {
    sell_dual_ = sell_eligible(P_->A.rp.get(), nullptr, m_, st_);
    sell_primal_ = sell_eligible(P_->Q.rp.get(), P_->AT.rp.get(), n_, st_);
    setup_slabs();
    if (full_plans_) {
      setup_colblocks();
    } else if (own_norm_a_) {  // built for the norm estimate only: the shards build their own
      RB_CUDA(cudaStreamSynchronize(st_));
      dual_ph_ = SlabPhase{};
      primal_ph_ = SlabPhase{};
    }
  }
  tr.mark("slab plans");
  setup_chunk_kernel();
  setup_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
}

// Slab-staged gathers for the dual (rows of A gather w) and the primal (A' part
// of [Q | A'] gathers y); slab.cuh. Rows outside a plan keep the regular kernel
// through a complement schedule.
#ifdef RB_SLAB_PROFILE
namespace {
// RB_SLAB_PROFILE builds: per-CTA phase times of the last slab launch, to stderr.
void dump_slab_profile(const char* name, const SlabView& v) {
  if (!v.prof) return;
  std::vector<unsigned long long> h(static_cast<std::size_t>(v.grid) * kSlabProf);
  RB_CUDA(cudaMemcpy(h.data(), v.prof, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int b = 0; b < v.grid; ++b) t0 = std::min(t0, h[b * kSlabProf]), t1 = std::max(t1, h[b * kSlabProf + 6]);
  std::vector<int> order(v.grid);
  for (int b = 0; b < v.grid; ++b) order[b] = b;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return h[a * kSlabProf + 6] > h[b * kSlabProf + 6]; });
  std::fprintf(stderr, "[slab %s] grid %d tiles %d span %.1f us\n", name, v.grid, v.tiles(), (t1 - t0) / 1e3);
  auto row = [&](int b) {
    const unsigned long long* p = &h[b * kSlabProf];
    std::fprintf(stderr, "  cta %3d sm %3llu start %6.1f wait %6.1f compute %6.1f end %6.1f tiles %llu\n", b, p[8],
                 (p[0] - t0) / 1e3, p[2] / 1e3, p[3] / 1e3, (p[6] - t0) / 1e3, p[7]);
  };
  for (int q = 0; q < 6 && q < v.grid; ++q) row(order[q]);
  std::fprintf(stderr, "  ...\n");
  for (int q = std::max(0, v.grid - 3); q < v.grid; ++q) row(order[q]);
  // end time by SM (both CTAs of an SM), slowest / fastest SMs, and by SM id halves
  std::vector<double> sm_end(kSMs, 0.0);
  for (int b = 0; b < v.grid; ++b) {
    const int sm = static_cast<int>(h[b * kSlabProf + 8]) % kSMs;
    sm_end[sm] = std::max(sm_end[sm], (h[b * kSlabProf + 6] - t0) / 1e3);
  }
  double lo_half = 0, hi_half = 0;
  for (int q = 0; q < kSMs; ++q) (q < kSMs / 2 ? lo_half : hi_half) += sm_end[q] / (kSMs / 2);
  {
    unsigned long long f[4];
    RB_CUDA(cudaMemcpy(f, v.fprof, sizeof(f), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "  slab end %.1f | finish: other rows end %.1f, W wait done %.1f..%.1f, W end %.1f us\n",
                 (t1 - t0) / 1e3, f[0] ? (f[0] - t0) / 1e3 : 0.0, (f[1] - t0) / 1e3, (f[2] - t0) / 1e3,
                 (f[3] - t0) / 1e3);
  }
  std::fprintf(stderr, "  mean end: SMs 0-73 %.1f us, SMs 74-147 %.1f us; by SM:", lo_half, hi_half);
  for (int q = 0; q < kSMs; ++q) std::fprintf(stderr, "%s%.0f", q % 16 ? " " : "\n   ", sm_end[q]);
  std::fprintf(stderr, "\n");
}
}  // namespace
#endif

void Engine::colblock_counts(bool dual_slab_active, bool primal_slab_active) {
  DeviceQP& P = *P_;
  auto local = [&](const DevCsr& m) {
    return pattern_locality(m.rp.get(), m.ci.get(), m.rows, m.cols, m.nnz, st_) >= 0.5;
  };
  cb_nb_dual_ = cb_nq_ = cb_na_ = 1;
  if (!dual_slab_active && colblock_count(n_) >= 2 && !local(P.A)) cb_nb_dual_ = colblock_count(n_);
  if (!primal_slab_active) {
    if (colblock_count(n_) >= 2 && !local(P.Q)) cb_nq_ = colblock_count(n_);
    if (colblock_count(m_) >= 2 && !local(P.AT)) cb_na_ = colblock_count(m_);
  }
}

void Engine::setup_colblocks() {
  DeviceQP& P = *P_;
  colblock_counts(dual_ph_.active(), primal_ph_.active());
  build_colblocked_dual(cbd_, cb_nb_dual_, P.A.rp.get(), P.A.ci.get(), m_, n_, asv_, sell_dual_, st_);
  build_colblocked_primal(cbp_, cb_nq_, cb_na_, P.Q.rp.get(), P.Q.ci.get(), qsv_, P.AT.rp.get(), P.AT.ci.get(), atsv_,
                          n_, n_, m_, sell_primal_, st_);
  // the plain path of short-row ops: sliced ELL instead of rowwise_kernel
  if (sell_dual_ && !dual_ph_.active() && !cbd_.active()) {
    build_sell_plan(sell_dual_plan_, P.A.rp.get(), P.A.ci.get(), nullptr, nullptr, m_, st_);
    fill_sell_values(sell_dual_plan_, asv_, nullptr, st_);
  }
  if (sell_primal_ && !primal_ph_.active() && !cbp_.active()) {
    build_sell_plan(sell_primal_plan_, P.Q.rp.get(), P.Q.ci.get(), P.AT.rp.get(), P.AT.ci.get(), n_, st_);
    fill_sell_values(sell_primal_plan_, qsv_, atsv_, st_);
  }
}

int norm_slab_step() {
  const char* e = std::getenv("RAPDHG_NORM_SLAB_STEP");
  return e ? std::atoi(e) : kNormSlabStep;
}

// estimate_op_norm on A (opnorm.hpp:36-61) for the solve. Fast mode: the
// first kNormSlabStep steps run on the rowwise SpMV while the slab plans are
// still being built on host threads; from that step on (a batch boundary),
// the plans are joined and the products run on the step's slab phases
// (PhaseSpmvOp: C4 0.22 instead of 0.40 ms per step). The switch step is
// fixed (norm_slab_step(): 40 — C4's plans are ready by then), never timing-
// dependent, so the estimate is deterministic; the sharded solver's setup
// runs the same code on the same full matrices, so its norm is the same bits.
double Engine::norm_a_power(int max_iters, double tol, uint64_t seed, const RandomStart* pre) {
  DeviceQP& P = *P_;
  const int K = norm_slab_step();
  if (P.strict || K < 0 || P.A.nnz == 0) return P.op_norm_a(asv_, atsv_, max_iters, tol, seed, pre);
  DevBuf<double> v(n_), w(n_), mv(m_);
  bool slab = false;
  PowerRun r(
      P, v, w, n_,
      [&](StepGate g, cudaStream_t s) {
        if (slab && dual_ph_.active())
          P.launches += launch_slab_phase(PhaseSpmvOp<1>{P.A.view(asv_), CsrView{}, v.get(), v.get(), mv.get(), g},
                                          dual_ph_, s);
        else
          P.spmv(P.A, P.sch_dual, asv_, v.get(), mv.get(), g, s);
        if (slab && primal_ph_.active())
          P.launches += launch_slab_phase(
              PhaseSpmvOp<2>{P.Q.view(qsv_), P.AT.view(atsv_), v.get(), mv.get(), w.get(), g}, primal_ph_, s);
        else
          P.spmv(P.AT, P.sch_at, atsv_, mv.get(), w.get(), g, s);
      },
      false, max_iters, tol, seed, P.st, P.red, nullptr, 0, pre);
  r.split_at(K, [&](int it) {
    if (slab || it < K) return;
    setup_slabs();  // joins the plan threads (waits if they are still running)
    slab = dual_ph_.active() || primal_ph_.active();
  });
  run_alone(r);
  return std::sqrt(std::max(r.result(), 0.0));
}

// Small problems run each chunk as one cooperative launch (persistent.cuh):
// fast mode, both steps on the plain path (rowwise or sliced ELL; no slab or
// column-block plans, no staged windows), no per-step profiling, and little
// enough work per iteration that the per-step launches are the cost.
// Opt-in (RAPDHG_PERSISTENT=1): measured slower than the replayed graph of
// per-step kernels — C1 68k against 96k it/s, the two grid-wide barriers per
// step costing more than the graph's launches.
void Engine::setup_chunk_kernel() {
  chunk_grid_ = 0;
  const char* env = std::getenv("RAPDHG_PERSISTENT");
  const std::string mode = env ? env : "0";
  if (mode != "1" || P_->strict || !events_.empty()) return;
  if (dual_ph_.active() || primal_ph_.active() || cbd_.active() || cbp_.active()) return;
  const SchedView& sd = P_->sch_dual.view;
  const SchedView& sp = P_->sch_primal.view;
  if (sd.win[0].len + sd.win[1].len + sp.win[0].len + sp.win[1].len > 0) return;
  const void* k = reinterpret_cast<const void*>(&chunk_kernel<DualStepOp<false>, PrimalStepOp<false>>);
  int per_sm = 0;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBlock, 0));
  if (per_sm < 1) return;
  auto blocks_of = [](const SchedView& v, const SellPlan& sp) {
    return sp.active() ? static_cast<int>(ceil_div(sp.view.nslices, kBlock / 32)) : v.total_blocks;
  };
  const int want = std::max(std::max(blocks_of(sd, sell_dual_plan_), blocks_of(sp, sell_primal_plan_)), 1);
  chunk_grid_ = std::min(want, per_sm * kSMs);
}

// The pattern-only part of the slab plans (windows, tiles, layouts: mostly
// host work), on a host thread with its own stream, started once the matrices
// are on the device so it overlaps the scaling and the power iterations.
void Engine::plan_slabs_async() {
  const int dev = cfg_.device;
  // one host thread (and stream) per op's plan
  auto task = [this, dev](bool dual) {
    RB_CUDA(cudaSetDevice(dev));
    // high priority: the plans' few short kernels (counts, fills) are
    // scheduled ahead of the scaling / power-iteration blocks they overlap,
    // instead of queueing behind them
    int lo = 0, hi = 0;
    RB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    cudaStream_t s2;
    RB_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi));
    try {
      // this thread's allocations and frees are ordered on s2 (its buffers
      // that outlive it are used after the join, which follows s2's sync)
      AllocStreamScope scope(s2);
      DeviceQP& P = *P_;
      Tracer tr(s2);
      DevBuf<int32_t> len;
      if (dual) {
        dual_choice_ = choose_slabs(P.A.rp.get(), P.A.ci.get(), P.A.rows, P.A.nnz, n_, s2);
        if (full_plans_ || own_norm_a_) {
          row_lengths(len, P.A.rp.get(), nullptr, m_, s2);
          build_slab_phase(dual_ph_, dual_choice_, 0, P.A.rp.get(), P.A.ci.get(), nullptr, nullptr, 0, m_, len.get(),
                           s2);
        }
        tr.mark("  slab plan: dual (async)");
      } else {
        primal_choice_ = choose_slabs(P.AT.rp.get(), P.AT.ci.get(), n_, P.AT.nnz, m_, s2);
        if (full_plans_ || own_norm_a_) {
          row_lengths(len, P.Q.rp.get(), P.AT.rp.get(), n_, s2);
          build_slab_phase(primal_ph_, primal_choice_, 1, P.Q.rp.get(), P.Q.ci.get(), P.AT.rp.get(), P.AT.ci.get(),
                           0, n_, len.get(), s2);
        }
        tr.mark("  slab plan: primal (async)");
      }
      RB_CUDA(cudaStreamSynchronize(s2));
    } catch (...) {
      cudaStreamSynchronize(s2);
      cudaStreamDestroy(s2);
      throw;
    }
    RB_CUDA(cudaStreamDestroy(s2));
  };
  plan_future_ = std::async(std::launch::async, task, true);
  plan_future2_ = std::async(std::launch::async, task, false);
}

void Engine::setup_slabs() {
  if (slabs_ready_) return;  // already done for the norm estimate
  slabs_ready_ = true;
  Tracer tr(st_);
  plan_future_.get();  // the pattern part (plan_slabs_async)
  plan_future2_.get();
  tr.mark("  slab plans joined");
  if (dual_ph_.active()) {
    fill_slab_values(dual_ph_.plan, asv_, nullptr, st_);
    fill_sell_values(dual_ph_.others_sell, asv_, nullptr, st_);
    const int smem = dual_ph_.plan.view.smem_bytes();
    prepare_slab<PhaseSpmvOp<1>>(smem);  // the norm's launches use the step's CTA ranges
    assign_slab_ctas(dual_ph_.plan, prepare_slab<DualStepOp<false>>(smem), st_);
  }
  if (primal_ph_.active()) {
    fill_slab_values(primal_ph_.plan, qsv_, atsv_, st_);
    fill_sell_values(primal_ph_.others_sell, qsv_, atsv_, st_);
    const int smem = primal_ph_.plan.view.smem_bytes();
    prepare_slab<PhaseSpmvOp<2>>(smem);
    assign_slab_ctas(primal_ph_.plan, prepare_slab<PrimalStepOp<false>>(smem), st_);
  }
  tr.mark("  slab values + launch setup");
#ifdef RB_SLAB_PROFILE
  for (SlabPlan* pl : {&dual_ph_.plan, &primal_ph_.plan})
    if (pl->view.active()) {
      pl->prof.alloc(static_cast<std::size_t>(pl->view.grid) * kSlabProf + 4);
      pl->prof.zero(st_);
      pl->view.prof = pl->prof.get();
      pl->view.fprof = pl->prof.get() + static_cast<std::size_t>(pl->view.grid) * kSlabProf;
    }
#endif
  RB_CUDA(cudaStreamSynchronize(st_));
}

Engine::~Engine() {
#ifdef RB_SLAB_PROFILE
  try {
    dump_slab_profile("dual", dual_ph_.plan.view);
    dump_slab_profile("primal", primal_ph_.plan.view);
  } catch (...) {
  }
#endif
  if (st_) cudaStreamSynchronize(st_);  // buffers are freed below / after this body
  if (st2_) cudaStreamSynchronize(st2_);
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
  for (auto& e : events_) cudaEventDestroy(e);
  P_.reset();
  if (evf_) cudaEventDestroy(evf_);
  if (evj_) cudaEventDestroy(evj_);
  // own_st_ / own_st2_ are destroyed after the remaining buffers
}

double Engine::bytes_dual() const {
  // stream A~ (value + index) and row pointers; gather w (n); read y, b, ybar;
  // write y, ybar (12 nnz(A) + 4(m+1) + 8(n + 5m))
  return 12.0 * P_->A.nnz + 4.0 * (m_ + 1) + 8.0 * (n_ + 5.0 * m_);
}
double Engine::bytes_primal() const {
  // stream Q~ and A~' with row pointers; gather x_md (n) and y (m); read x, c,
  // xbar; write x+, xbar, w, x_md (12 (nnz(Q) + nnz(A)) + 8(n+1) + 8(8n + m))
  return 12.0 * (P_->Q.nnz + P_->AT.nnz) + 4.0 * (2.0 * n_ + 2) + 8.0 * (8.0 * n_ + m_);
}
double Engine::bytes_iter() const {
  // B_iter = 12 (2 nnz(A) + nnz(Q)) + 4 (m + 2n + 3) + 8 (9n + 6m)
  return 12.0 * (2.0 * P_->A.nnz + P_->Q.nnz) + 4.0 * (m_ + 2.0 * n_ + 3) + 8.0 * (9.0 * n_ + 6.0 * m_);
}

void Engine::launch_chunk_body(int len, int cur, bool prof) {
  unsigned long long* span = nullptr;
  if (prof && span_mode_) {  // stamps instead of events
    span = span_.get();
    RB_CUDA(cudaMemsetAsync(span, 0xff, sizeof(unsigned long long) * 2 * len, st_));
    prof = false;
  }
  prologue_kernel<<<grid1(n_), 256, 0, st_>>>(X_[cur].get(), X_[cur ^ 1].get(), xb_.get(), w_.get(),
                                              XMD_[cur].get(), params_.get(), n_);
  RB_LAUNCH_CHECK();
  ++launches_;
  if (prof) RB_CUDA(cudaEventRecordWithFlags(events_[0], st_, cudaEventRecordExternal));
  for (int it = 0; it < len; ++it) {
    const int c = (cur + it) & 1;
    if (P_->strict) {
      DualStepOp<true> d{P_->A.view(asv_), w_.get(), bsv_, y_.get(), yb_.get(), mi_, params_.get(), it, bad_.get()};
      rowwise(d, P_->sch_dual, st_, &launches_);
    } else {
      DualStepOp<false> d{P_->A.view(asv_), w_.get(), bsv_, y_.get(), yb_.get(), mi_, params_.get(), it, bad_.get()};
      if (dual_ph_.active()) {
        launches_ += launch_slab_phase(d, dual_ph_, st_, span);
      } else if (cbd_.active()) {
        launches_ += launch_colblocked_dual(d, cbd_, st_);
      } else if (sell_dual_plan_.active()) {
        launch_sell(d, sell_dual_plan_, st_, plain_pdl_);
        ++launches_;
      } else if (P_->sch_dual.view.total_blocks > 0) {
        launch_rowwise(d, P_->sch_dual.view, st_, plain_pdl_);
        ++launches_;
      }
    }
    if (prof) RB_CUDA(cudaEventRecordWithFlags(events_[2 * it + 1], st_, cudaEventRecordExternal));
    if (P_->strict) {
      PrimalStepOp<true> pr{P_->Q.view(qsv_), P_->AT.view(atsv_), XMD_[c].get(), y_.get(), X_[c].get(),
                            X_[c ^ 1].get(), xb_.get(), csv_, w_.get(), XMD_[c ^ 1].get(), params_.get(), it, bad_.get()};
      rowwise(pr, P_->sch_primal, st_, &launches_);
    } else {
      PrimalStepOp<false> pr{P_->Q.view(qsv_), P_->AT.view(atsv_), XMD_[c].get(), y_.get(), X_[c].get(),
                             X_[c ^ 1].get(), xb_.get(), csv_, w_.get(), XMD_[c ^ 1].get(), params_.get(), it, bad_.get(),
                             lsv_, hsv_};
      if (primal_ph_.active()) {
        launches_ += launch_slab_phase(pr, primal_ph_, st_, span);
      } else if (cbp_.active()) {
        launches_ += launch_colblocked_primal(pr, cbp_, st_);
      } else if (sell_primal_plan_.active()) {
        launch_sell(pr, sell_primal_plan_, st_, plain_pdl_);
        ++launches_;
      } else if (P_->sch_primal.view.total_blocks > 0) {
        launch_rowwise(pr, P_->sch_primal.view, st_, plain_pdl_);
        ++launches_;
      }
    }
    if (prof) RB_CUDA(cudaEventRecordWithFlags(events_[2 * it + 2], st_, cudaEventRecordExternal));
  }
}

void Engine::run_chunk(int len) {
  params_.upload(params_h_.get(), len, st_);
  // kernel timing is sampled (every kProfilePeriod-th chunk) so the event
  // nodes barely perturb the timed loop
  const bool prof = !events_.empty() && (chunk_counter_++ % kProfilePeriod) == 0;
  if (chunk_grid_ > 0) {  // small problem: the chunk as one cooperative launch (persistent.cuh)
    const DualStepOp<false> d{P_->A.view(asv_), w_.get(), bsv_, y_.get(), yb_.get(), mi_, params_.get(), 0, bad_.get()};
    PrimalStepOp<false> pr[2];
    for (int c = 0; c < 2; ++c)
      pr[c] = PrimalStepOp<false>{P_->Q.view(qsv_), P_->AT.view(atsv_), XMD_[c].get(), y_.get(), X_[c].get(),
                                  X_[c ^ 1].get(), xb_.get(), csv_, w_.get(), XMD_[c ^ 1].get(), params_.get(), 0,
                                  bad_.get(), lsv_, hsv_};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(static_cast<unsigned>(chunk_grid_));
    lc.blockDim = dim3(kBlock);
    lc.stream = st_;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    RB_CUDA(cudaLaunchKernelEx(&lc, chunk_kernel<DualStepOp<false>, PrimalStepOp<false>>, d, P_->sch_dual.view,
                               sell_dual_plan_.view, pr[0], pr[1], P_->sch_primal.view, sell_primal_plan_.view,
                               static_cast<const double*>(X_[cur_].get()),
                               static_cast<const double*>(X_[cur_ ^ 1].get()), static_cast<const double*>(xb_.get()),
                               w_.get(), XMD_[cur_].get(), static_cast<const IterParams*>(params_.get()), n_, len,
                               cur_));
    ++launches_;
  } else if (cfg_.use_graphs) {
    const int key = (len << 2) | (cur_ << 1) | (prof ? 1 : 0);
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
      const int64_t before = launches_;
      const cudaGraphExec_t ge = capture_graph(st_, [&] { launch_chunk_body(len, cur_, prof); });
      graph_launches_[key] = launches_ - before;  // kernel nodes of this graph
      launches_ = before;  // counted at replay below
      it = graphs_.emplace(key, ge).first;
    }
    RB_CUDA(cudaGraphLaunch(it->second, st_));
    launches_ += graph_launches_[key];
  } else {
    launch_chunk_body(len, cur_, prof);
  }
  cur_ ^= (len & 1);
  bad_fresh_ = false;
  // no sync: the check's kernels queue behind the chunk (first_bad() or
  // evaluate() synchronise); sampled chunks read their events now
  if (prof && span_mode_) {  // step k lasts from its start to step k + 1's start
    std::vector<unsigned long long> h(2 * static_cast<std::size_t>(len));
    span_.download(h.data(), h.size(), st_);
    RB_CUDA(cudaStreamSynchronize(st_));
    for (std::size_t k = 0; k + 1 < h.size(); ++k)
      if (h[k] != ~0ull && h[k + 1] != ~0ull && h[k + 1] > h[k]) {
        kernel_ms_[k & 1] += static_cast<double>(h[k + 1] - h[k]) * 1e-6;
        ++kernel_count_[k & 1];
      }
  } else if (prof) {
    RB_CUDA(cudaStreamSynchronize(st_));
    for (int it = 0; it < len; ++it) {
      float a = 0.f, b = 0.f;
      RB_CUDA(cudaEventElapsedTime(&a, events_[2 * it], events_[2 * it + 1]));
      RB_CUDA(cudaEventElapsedTime(&b, events_[2 * it + 1], events_[2 * it + 2]));
      kernel_ms_[0] += a;
      kernel_ms_[1] += b;
      ++kernel_count_[0];
      ++kernel_count_[1];
    }
  }
}

// evaluate_candidate (solver.hpp:255-264) for the current iterate and the
// average at once: unscale, the three KKT products over the ORIGINAL matrices
// with both points per pass, then the reductions of kkt.hpp:43-69.
Cand Engine::evaluate() {
  const int cur = cur_;
  unscale_kernel<<<grid1(n_ + m_), 256, 0, st_>>>(X_[cur].get(), xb_.get(), y_.get(), yb_.get(), d_.get(),
                                                  xu_[0].get(), xu_[1].get(), yu_[0].get(), yu_[1].get(), n_, m_,
                                                  xi_.get(), yi_.get());
  RB_LAUNCH_CHECK();
  ++launches_;
  DeviceQP& P = *P_;
  if (P.strict) {
    KktAxOp<true> ax{P.A.view(), xi_.get(), ax_[0].get(), ax_[1].get()};
    rowwise(ax, P.sch_dual, st_, &launches_);
    KktQAtyOp<true> qa{P.Q.view(), P.AT.view(), mi_, xi_.get(), yi_.get(),
                       qx_[0].get(), qx_[1].get(), aty_[0].get(), aty_[1].get()};
    rowwise(qa, P.sch_primal, st_, &launches_);
    launch_reduce<4, 5>(KktDualTerms{ax_[0].get(), ax_[1].get(), P.b.get(), yu_[0].get(), yu_[1].get(), mi_},
                        m_, true, P.red, P.red_out.get(), st_);
    launch_reduce<kKktPrimalSums, kKktPrimalMaxes>(
        KktPrimalTerms{qx_[0].get(), qx_[1].get(), aty_[0].get(), aty_[1].get(), xu_[0].get(), xu_[1].get(),
                       P.c.get(), P.lo.size() ? P.lo.get() : nullptr, P.hi.size() ? P.hi.get() : nullptr},
        n_, true, P.red, P.red_out.get() + 16, st_);
  } else {
    // primal side on st2_ (own reduction scratch), dual side on st_, joined
    // before the read-back; the results do not depend on the overlap
    if (!st2_) {
      st2_ = own_st2_.create();
      RB_CUDA(cudaEventCreateWithFlags(&evf_, cudaEventDisableTiming));
      RB_CUDA(cudaEventCreateWithFlags(&evj_, cudaEventDisableTiming));
      red2_.init(std::max(n_, m_), st_);
    }
    RB_CUDA(cudaEventRecord(evf_, st_));
    RB_CUDA(cudaStreamWaitEvent(st2_, evf_, 0));
    KktQAtyOp<false> qa{P.Q.view(), P.AT.view(), mi_, xi_.get(), yi_.get(),
                        qx_[0].get(), qx_[1].get(), aty_[0].get(), aty_[1].get()};
    rowwise(qa, P.sch_primal, st2_, &launches_);
    // primal-side terms (kkt.hpp:56-66)
    launch_reduce<kKktPrimalSums, kKktPrimalMaxes>(
        KktPrimalTerms{qx_[0].get(), qx_[1].get(), aty_[0].get(), aty_[1].get(), xu_[0].get(), xu_[1].get(),
                       P.c.get(), P.lo.size() ? P.lo.get() : nullptr, P.hi.size() ? P.hi.get() : nullptr},
        n_, false, red2_, P.red_out.get() + 16, st2_);
    RB_CUDA(cudaEventRecord(evj_, st2_));
    KktAxOp<false> ax{P.A.view(), xi_.get(), ax_[0].get(), ax_[1].get()};
    rowwise(ax, P.sch_dual, st_, &launches_);
    // dual-side terms (kkt.hpp:43-53, 67)
    launch_reduce<4, 5>(KktDualTerms{ax_[0].get(), ax_[1].get(), P.b.get(), yu_[0].get(), yu_[1].get(), mi_},
                        m_, false, P.red, P.red_out.get(), st_);
    RB_CUDA(cudaStreamWaitEvent(st_, evj_, 0));
  }
  launches_ += 2;
  RB_CUDA(cudaMemcpyAsync(P.red_host.get(), P.red_out.get(), sizeof(double) * 32, cudaMemcpyDeviceToHost, st_));
  bad_.download(bad_h_.get(), 1, st_);  // the chunk's numerical-error flag, with the same sync
  RB_CUDA(cudaStreamSynchronize(st_));
  bad_fresh_ = true;
  const double* h = P.red_host.get();
  KktRaw r;
  r.by_i[0] = h[0], r.by_e[0] = h[1], r.by_i[1] = h[2], r.by_e[1] = h[3];
  r.viol[0] = h[4], r.viol[1] = h[5], r.ax_inf[0] = h[6], r.ax_inf[1] = h[7], r.b_inf = h[8];
  primal_terms_into(r, h + 16);
  Kkt k2[2];
  finalize_kkt(r, k2);
  Cand cd;
  cd.cur = k2[0];
  cd.avg = k2[1];
  cd.is_avg = !(cd.cur.relkkt() < cd.avg.relkkt());  // ties -> average
  return cd;
}

void Engine::restart(bool from_avg, double* dx, double* dy) {
  const int cur = cur_;
  restart_kernel<<<grid1(n_ + m_), 256, 0, st_>>>(X_[cur].get(), X_[cur ^ 1].get(), xb_.get(), y_.get(),
                                                  yb_.get(), from_avg ? 1 : 0, n_, m_);
  RB_LAUNCH_CHECK();
  ++launches_;
  // dist2 to the previous epoch start, then epoch_prev <- state (solver.hpp:454-460)
  double sx[1], sy[1];
  P_->reduce_to_host<1, 0>(DistAndAdvance{X_[cur].get(), epx_.get()}, n_, sx);
  P_->reduce_to_host<1, 0>(DistAndAdvance{y_.get(), epy_.get()}, m_, sy);
  launches_ += 2;
  *dx = std::sqrt(sx[0]);
  *dy = std::sqrt(sy[0]);
}

void Engine::download_point(const double* xu, const double* yu, double* x, double* y) {
  if (n_) RB_CUDA(cudaMemcpyAsync(x, xu, sizeof(double) * n_, cudaMemcpyDeviceToHost, st_));
  if (m_) RB_CUDA(cudaMemcpyAsync(y, yu, sizeof(double) * m_, cudaMemcpyDeviceToHost, st_));
  RB_CUDA(cudaStreamSynchronize(st_));
}

// Result blocks: the final point of a solve. Large ones come from the pinned
// cache (the download is then a direct DMA at link speed instead of the
// driver's pageable bounce, and a binding can wrap the memory without a
// copy); at most kResultPinnedMax bytes are pinned at once, the rest is
// malloc'ed. rapdhg_result_free hands a block back through result_block_free.
namespace {
constexpr std::size_t kResultPinnedMin = std::size_t{1} << 20;
constexpr std::size_t kResultPinnedMax = std::size_t{2} << 30;
struct ResultBlocks {
  std::mutex mu;
  std::map<void*, std::pair<std::size_t, bool>> live;  // block -> (bytes, pinned)
  std::size_t pinned_bytes = 0;
  // their own cache (size classes as pinned_class): a result the caller
  // still holds must not take the staging buffers the next solve reuses
  std::vector<std::pair<std::size_t, void*>> free;
};
ResultBlocks& result_blocks() {
  static ResultBlocks* rb = new ResultBlocks;  // never destroyed: frees may run at exit
  return *rb;
}
}  // namespace

void* result_block_alloc(std::size_t bytes) {
  bytes = bytes ? bytes : sizeof(double);
  ResultBlocks& R = result_blocks();
  bool pin = false;
  if (bytes >= kResultPinnedMin) {
    std::lock_guard<std::mutex> g(R.mu);
    if (R.pinned_bytes + bytes <= kResultPinnedMax) pin = true, R.pinned_bytes += bytes;
  }
  void* p = nullptr;
  if (pin) {
    const std::size_t cls = pinned_class(bytes);
    {
      std::lock_guard<std::mutex> g(R.mu);
      for (std::size_t i = 0; i < R.free.size(); ++i)
        if (R.free[i].first == cls) {
          p = R.free[i].second;
          R.free[i] = R.free.back();
          R.free.pop_back();
          break;
        }
    }
    const bool miss = !p;
    if (miss && cudaMallocHost(&p, cls) != cudaSuccess) {
      cudaGetLastError();
      std::lock_guard<std::mutex> g(R.mu);
      R.pinned_bytes -= bytes;
      pin = false;
      p = nullptr;
    } else if (miss) {
      // a caller that keeps the last result while solving again needs two
      // blocks: page-lock the spare now (~15 ms for C4's 32 MB) rather than
      // in the middle of the next solve
      void* spare = nullptr;
      if (cudaMallocHost(&spare, cls) == cudaSuccess) {
        std::lock_guard<std::mutex> g(R.mu);
        R.free.emplace_back(cls, spare);
      } else {
        cudaGetLastError();
      }
    }
  }
  if (!pin) {
    p = std::malloc(bytes);
    if (!p) throw Error(RAPDHG_E_INTERNAL, "out of host memory");
  }
  std::lock_guard<std::mutex> g(R.mu);
  R.live[p] = {bytes, pin};
  return p;
}

bool result_block_free(void* p) {
  if (!p) return false;
  ResultBlocks& R = result_blocks();
  std::pair<std::size_t, bool> e;
  {
    std::lock_guard<std::mutex> g(R.mu);
    auto it = R.live.find(p);
    if (it == R.live.end()) return false;
    e = it->second;
    R.live.erase(it);
    if (e.second) R.pinned_bytes -= e.first;
  }
  if (e.second) {
    std::lock_guard<std::mutex> g(R.mu);
    R.free.emplace_back(pinned_class(e.first), p);
  } else {
    std::free(p);
  }
  return true;
}

namespace {
template <typename T>
T* xalloc(std::size_t n) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (n ? n : 1)));
  if (!p) throw Error(RAPDHG_E_INTERNAL, "out of host memory");
  return p;
}
template <typename T>
void append(T*& arr, int64_t& count, const T& v) {
  T* p = static_cast<T*>(std::realloc(arr, sizeof(T) * (count + 1)));
  if (!p) throw Error(RAPDHG_E_INTERNAL, "out of host memory");
  arr = p;
  arr[count++] = v;
}
}  // namespace

// ---- Engine as the single-GPU loop backend -------------------------------------

void Engine::loop_begin() {
  kernel_ms_[0] = kernel_ms_[1] = 0.0;
  kernel_count_[0] = kernel_count_[1] = 0;
  chunk_counter_ = 0;  // every solve samples its first chunk
  launches_ = P_->launches;
  // loop time on the device timeline: events on the solver's stream bracket
  // everything from the first candidate evaluation to the final download
  RB_CUDA(cudaEventCreate(&ev0_));
  RB_CUDA(cudaEventCreate(&ev1_));
  RB_CUDA(cudaEventRecord(ev0_, st_));
  // IterateState::zeros (solver.hpp:293)
  cur_ = 0;
  for (auto* buf : {&X_[0], &X_[1], &xb_, &epx_}) buf->zero(st_);
  for (auto* buf : {&y_, &yb_, &epy_}) buf->zero(st_);
  bad_h_[0] = std::numeric_limits<long long>::max();
  bad_.upload(bad_h_.get(), 1, st_);
}

long long Engine::first_bad() {
  if (bad_fresh_) {  // read back with the last evaluate()'s results, after the chunk
    bad_fresh_ = false;
    return bad_h_[0];
  }
  bad_.download(bad_h_.get(), 1, st_);
  RB_CUDA(cudaStreamSynchronize(st_));
  return bad_h_[0];
}

void Engine::keep_best(bool avg) {
  const int i = avg ? 1 : 0;
  RB_CUDA(cudaMemcpyAsync(best_x_.get(), xu_[i].get(), sizeof(double) * n_, cudaMemcpyDeviceToDevice, st_));
  if (m_) RB_CUDA(cudaMemcpyAsync(best_y_.get(), yu_[i].get(), sizeof(double) * m_, cudaMemcpyDeviceToDevice, st_));
}

void Engine::download(int src, double* x, double* y) {
  if (src == 2) download_point(best_x_.get(), best_y_.get(), x, y);
  else download_point(xu_[src].get(), yu_[src].get(), x, y);
}

void Engine::loop_end(rapdhg_result* out) {
  RB_CUDA(cudaEventRecord(ev1_, st_));
  RB_CUDA(cudaEventSynchronize(ev1_));
  float loop_ms = 0.f;
  RB_CUDA(cudaEventElapsedTime(&loop_ms, ev0_, ev1_));
  cudaEventDestroy(ev0_);
  cudaEventDestroy(ev1_);
  out->loop_seconds = 1e-3 * loop_ms;
  out->kernel_launches = launches_;
  out->kernel_ms[0] = kernel_ms_[0], out->kernel_ms[1] = kernel_ms_[1];
  out->kernel_count[0] = kernel_count_[0], out->kernel_count[1] = kernel_count_[1];
}

void Engine::solve(rapdhg_result* out, Clock::time_point t0) {
  AllocStreamScope scope(st_);
  run_loop(*this, cfg_, LoopScalars{norm_q, norm_a, omega0, setup_seconds, n_, mi_, m_ - mi_}, out, t0);
}

// run_loop(): the loop of solver.hpp:293-471 on any backend, with inner steps
// batched into chunks that end exactly where the reference would run a check.
void run_loop(LoopBackend& be, const rapdhg_config& cfg, const LoopScalars& sc, rapdhg_result* out,
              Clock::time_point t0) {
  auto elapsed = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
  const int n = sc.n, mi_ = sc.mi, m = sc.mi + sc.me;
  const double norm_q = sc.norm_q, norm_a = sc.norm_a;
  std::memset(out, 0, sizeof(*out));
  out->n = n, out->m_ineq = sc.mi, out->m_eq = sc.me;
  out->norm_q = norm_q;
  out->norm_a = norm_a;
  be.loop_begin();
  IterParams* params_h = be.host_params();

  double omega = sc.omega0;
  long horizon = 1;
  const bool theoretical = cfg.step_rule == RAPDHG_STEP_THEORETICAL;
  const bool accelerated = cfg.algorithm == RAPDHG_ALG_APDHG;
  if (theoretical && accelerated) {
    if (cfg.restart == RAPDHG_RESTART_FIXED) horizon = cfg.restart_length;
    else if (cfg.restart == RAPDHG_RESTART_NONE) horizon = std::max<long>(cfg.max_iters, 1);
    else horizon = std::max<long>(4L * cfg.check_interval, 2);
  }
  out->norm_fallback = norm_a <= 0.0;
  double eta = 0.0, prev_eta = 0.0;
  long k = 0;

  // candidates: index 0 = current (xu_[0], yu_[0]), 1 = average
  Cand cand = be.evaluate();
  Kkt best = cand.res();
  auto copy_best = [&](const Cand& c) { be.keep_best(c.is_avg); };
  copy_best(cand);
  double epoch_start = cand.res().relkkt();
  double prev_candidate = std::numeric_limits<double>::infinity();
  auto log = [&](long t, const Kkt& r, double e, double w, bool rs) {
    append(out->log, out->n_log, rapdhg_log_record{t, r.r_primal, r.r_dual, r.r_gap, e, w, rs ? 1 : 0});
  };
  // result arrays grow in place; the block stays owned by `out` (freed by
  // rapdhg_result_free) whether or not the realloc succeeds
  auto grow = [](double*& arr, int64_t count) {
    double* p = static_cast<double*>(std::realloc(arr, sizeof(double) * static_cast<std::size_t>(count)));
    if (!p) throw Error(RAPDHG_E_INTERNAL, "out of host memory");
    arr = p;
    return p;
  };
  auto push_restart_point = [&](int idx) {
    double* xs = grow(out->restart_x, (out->n_restart_points + 1) * n + 1);
    double* ys = grow(out->restart_y, (out->n_restart_points + 1) * m + 1);
    be.download(idx, xs + out->n_restart_points * n, ys + out->n_restart_points * m);
    ++out->n_restart_points;
  };
  log(0, cand.res(), 0.0, omega, false);
  if (cfg.record_restart_points) push_restart_point(cand.is_avg ? 1 : 0);

  int status = -1;
  int fin_src = -1;  // 0/1 = candidate buffers, 2 = best
  long fin_iters = 0;
  Kkt fin_res;
  auto finish = [&](int st, int src, long iters, const Kkt& r) {
    status = st, fin_src = src, fin_iters = iters, fin_res = r;
  };
  if (cand.res().relkkt() <= cfg.tol) finish(RAPDHG_STATUS_OPTIMAL, cand.is_avg ? 1 : 0, 0, cand.res());
  else if (norm_q <= 0.0 && norm_a <= 0.0) finish(RAPDHG_STATUS_ITERATION_LIMIT, 2, 0, best);

  rapdhg_step_params sp{1.0, 1.0, 0.0, 0.0};
  long t = 1;
  while (status < 0 && t <= cfg.max_iters) {
    // ---- plan a chunk: steps t .. t_end, ending at the next check ----------
    int len = 0;
    bool horizon_hit = false, fixed_due = false, snapshot_due = false, check_due = false;
    long tt = t;
    for (; len < kMaxChunk && tt <= cfg.max_iters; ++tt) {
      if (theoretical) {
        if (accelerated)
          sp = step_schedule_theoretical(static_cast<int>(std::min<long>(k, horizon - 1)),
                                         static_cast<int>(horizon), norm_q, norm_a);
        else
          sp = pdhg_constant_steps(norm_q, norm_a);
      } else {
        if (accelerated) {
          eta = adaptive_eta(static_cast<int>(k), prev_eta, norm_q, norm_a, omega);
          sp.beta = 0.5 * (k + 2);
          sp.theta = static_cast<double>(k) / (k + 1);
        } else {
          if (k == 0) eta = adaptive_eta(0, 0.0, norm_q, norm_a, omega);
          sp.beta = 1.0;
          sp.theta = 1.0;
        }
        prev_eta = eta;
        sp.eta = eta / omega;
        sp.tau = eta * omega;
      }
      IterParams& q = params_h[len];
      const double inv_beta = 1.0 / sp.beta;
      q.theta = sp.theta;
      q.ib = inv_beta;
      q.omib = 1.0 - inv_beta;
      q.eta = sp.eta;
      q.tau = sp.tau;
      q.t = tt;
      q.emit_next = 0;
      if (len > 0) {
        IterParams& pq = params_h[len - 1];
        pq.theta_n = q.theta, pq.ib_n = q.ib, pq.omib_n = q.omib, pq.emit_next = 1;
      }
      ++len;
      ++k;
      horizon_hit = theoretical && accelerated && cfg.restart != RAPDHG_RESTART_NONE && k >= horizon;
      fixed_due = cfg.restart == RAPDHG_RESTART_FIXED && k >= cfg.restart_length;
      snapshot_due = cfg.snapshot_interval > 0 && tt % cfg.snapshot_interval == 0;
      check_due = tt % cfg.check_interval == 0 || fixed_due || horizon_hit || snapshot_due ||
                  tt == cfg.max_iters;
      if (check_due) break;
    }
    const long t_end = check_due ? tt : tt - 1;
    be.run_chunk(len);
    // a check's evaluation is queued right behind the chunk (one sync for
    // both); its results are only used once the chunk proved finite
    Cand next;
    if (check_due) next = be.evaluate();
    // all_finite after every step (solver.hpp:372-373): first bad iteration
    const long long bad = be.first_bad();
    if (bad <= t_end) {
      finish(RAPDHG_STATUS_NUMERICAL_ERROR, 2, static_cast<long>(bad), best);
      break;
    }
    t = t_end + 1;
    if (!check_due) continue;
    const long tc = t_end;
    const double cur_eta = theoretical ? sp.eta : eta;

    cand = next;
    const Kkt cres = cand.res();
    if (cres.relkkt() < best.relkkt()) {
      best = cres;
      copy_best(cand);
    }
    if (snapshot_due) {
      const int64_t s = out->n_snapshots;
      append(out->snapshot_iters, out->n_snapshots, static_cast<int64_t>(tc));
      grow(out->snapshot_x, (s + 1) * n + 1);
      grow(out->snapshot_y, (s + 1) * m + 1);
      be.download(1, out->snapshot_x + s * n, out->snapshot_y + s * m);
    }
    if (cres.relkkt() <= cfg.tol) {
      log(tc, cres, cur_eta, omega, false);
      finish(RAPDHG_STATUS_OPTIMAL, cand.is_avg ? 1 : 0, tc, cres);
      break;
    }
    // (an infinite limit is never reached: no vote needed)
    if (std::isfinite(cfg.time_limit_s) && be.any_rank(elapsed() > cfg.time_limit_s)) {
      log(tc, cres, cur_eta, omega, false);
      finish(RAPDHG_STATUS_TIME_LIMIT, 2, tc, best);
      break;
    }
    bool do_restart = false, from_avg = true;
    if (cfg.restart != RAPDHG_RESTART_NONE) {
      switch (cfg.restart) {
        case RAPDHG_RESTART_FIXED: do_restart = fixed_due; break;
        case RAPDHG_RESTART_HALVING:
          do_restart = restart_decision(cfg.restart, cand.avg.relkkt(), prev_candidate, epoch_start, k, tc, 0);
          break;
        case RAPDHG_RESTART_PDQP:
          do_restart = restart_decision(cfg.restart, cres.relkkt(), prev_candidate, epoch_start, k, tc, 0) ||
                       horizon_hit;
          from_avg = cand.is_avg;
          break;
        default: break;
      }
      if (horizon_hit) do_restart = true;
      prev_candidate = cres.relkkt();
    }
    log(tc, cres, cur_eta, omega, do_restart);
    if (!do_restart) continue;

    if (horizon_hit && !fixed_due) horizon *= 2;
    double dx = 0.0, dy = 0.0;
    be.restart(from_avg, &dx, &dy);
    k = 0;
    out->restarts += 1;
    prev_eta = 0.0;
    if (cfg.primal_weight == RAPDHG_PW_ADAPTIVE) omega = primal_weight_update(dx, dy, omega);
    // relKKT of the new epoch start == the average's when restarting from it
    epoch_start = (from_avg && !cand.is_avg) ? cand.avg.relkkt() : cres.relkkt();
    prev_candidate = std::numeric_limits<double>::infinity();
    if (cfg.record_restart_points) push_restart_point(from_avg ? 1 : 0);
  }
  if (status < 0) finish(RAPDHG_STATUS_ITERATION_LIMIT, 2, cfg.max_iters, best);

  out->status = status;
  out->iterations = fin_iters;
  out->residuals = {fin_res.r_primal, fin_res.r_dual, fin_res.r_gap};
  // the loop clock (loop_seconds: iterations + checks + restarts, device
  // time) stops before the solution's download to the host
  be.loop_end(out);
  // x | y_ineq | y_eq in one result block (page-locked when large): one
  // direct DMA per vector, no host copies
  double* blk = static_cast<double*>(result_block_alloc(sizeof(double) * (static_cast<std::size_t>(n) + m)));
  out->x = blk;
  out->y_ineq = blk + n;
  out->y_eq = blk + n + mi_;
  be.download(fin_src, out->x, out->y_ineq);
  out->setup_seconds = sc.setup_seconds;
  out->solve_seconds = elapsed();
}

// ============================================================================
// secondary API helpers
// ============================================================================

namespace {
// The stream of one secondary-API call: non-blocking, and the call's
// allocations are ordered on it. Declared before the call's buffers, which are
// therefore freed on it in stream order before it is drained and destroyed.
struct StreamGuard {
  OwnedStream own;
  cudaStream_t s = own.create();
  AllocStreamScope scope{s};
  ~StreamGuard() { cudaStreamSynchronize(s); }
};

rapdhg_qp single_matrix_qp(const rapdhg_csr& m, std::vector<int32_t>& zero_rp) {
  // A problem wrapper whose A_ineq is m (rows x cols) and Q is the empty
  // cols x cols matrix, so DeviceQP builds A, A' and their schedules.
  zero_rp.assign(static_cast<std::size_t>(m.n_cols) + 1, 0);
  rapdhg_qp p{};
  p.n = m.n_cols;
  p.m_ineq = m.n_rows;
  p.m_eq = 0;
  p.q = rapdhg_csr{m.n_cols, m.n_cols, 0, zero_rp.data(), nullptr, nullptr};
  p.a_ineq = m;
  p.a_eq = rapdhg_csr{0, m.n_cols, 0, zero_rp.data(), nullptr, nullptr};
  return p;
}
}  // namespace

void api_validate(const rapdhg_qp& p) {
  DeviceQP::validate_dims(p);  // problem.hpp:41-46
  StreamGuard sg;
  DeviceQP P(p, false, sg.s);
  P.validate_symmetry();  // problem.hpp:47-49
}

double api_symmetry_gap(const rapdhg_csr& mat) {
  if (mat.n_rows != mat.n_cols) invalid("symmetry_gap: matrix must be square");
  const int n = mat.n_rows;
  std::vector<int32_t> zrp(static_cast<std::size_t>(n) + 1, 0);
  std::vector<double> zeros(static_cast<std::size_t>(n) + 1, 0.0);
  rapdhg_qp p{};
  p.n = n;
  p.q = mat;
  p.a_ineq = rapdhg_csr{0, n, 0, zrp.data(), nullptr, nullptr};
  p.a_eq = rapdhg_csr{0, n, 0, zrp.data(), nullptr, nullptr};
  p.c = zeros.data(), p.b_ineq = zeros.data(), p.b_eq = zeros.data();
  DeviceQP::validate_dims(p);
  StreamGuard sg;
  DeviceQP P(p, false, sg.s);
  DevCsr qt;
  transpose_csr(qt, P.Q, nullptr, sg.s);
  double gap = 0.0, mabs = 0.0;
  symmetry_gap(P.Q, qt, &gap, &mabs, sg.s);
  return gap;
}

void api_spmv(const rapdhg_csr& mat, const double* x, double* y, bool transpose, bool strict) {
  std::vector<int32_t> zrp;
  rapdhg_qp p = single_matrix_qp(mat, zrp);
  std::vector<double> zeros(static_cast<std::size_t>(mat.n_cols) + static_cast<std::size_t>(mat.n_rows) + 1, 0.0);
  p.c = zeros.data();
  p.b_ineq = zeros.data();
  DeviceQP::validate_dims(p);
  StreamGuard sg;
  DeviceQP P(p, strict, sg.s);
  const int64_t in_len = transpose ? mat.n_rows : mat.n_cols;
  const int64_t out_len = transpose ? mat.n_cols : mat.n_rows;
  DevBuf<double> dx(in_len), dy(out_len);
  dx.upload(x, in_len, sg.s);
  if (transpose) P.spmv(P.AT, P.sch_at, P.AT.v.get(), dx.get(), dy.get());
  else P.spmv(P.A, P.sch_dual, P.A.v.get(), dx.get(), dy.get());
  dy.download(y, out_len, sg.s);
  RB_CUDA(cudaStreamSynchronize(sg.s));
}

void api_rel_kkt(const rapdhg_qp& p, const double* x, const double* yi, const double* ye,
                 bool strict, Kkt* out) {
  for (int i = 0; i < p.m_ineq; ++i)
    if (yi[i] < -1e-9) invalid("rel_kkt: negative inequality dual");  // kkt.hpp:29-30
  DeviceQP::validate_dims(p);
  StreamGuard sg;
  DeviceQP P(p, strict, sg.s);
  const int n = P.n, m = P.m, mi = P.mi;
  DevBuf<double> xu(n), yu(m), ax(m), qx(n), aty(n), ax2(m), qx2(n), aty2(n);
  xu.upload(x, n, sg.s);
  yu.upload(yi, mi, sg.s);
  if (m - mi) RB_CUDA(cudaMemcpyAsync(yu.get() + mi, ye, sizeof(double) * (m - mi), cudaMemcpyHostToDevice, sg.s));
  int64_t l = 0;
  DevBuf<double2> xi(n), yi2(m);
  interleave_kernel<<<grid1(n), 256, 0, sg.s>>>(xu.get(), xu.get(), xi.get(), n);
  interleave_kernel<<<grid1(m), 256, 0, sg.s>>>(yu.get(), yu.get(), yi2.get(), m);
  RB_LAUNCH_CHECK();
  if (strict) {
    rowwise(KktAxOp<true>{P.A.view(), xi.get(), ax.get(), ax2.get()}, P.sch_dual, sg.s, &l);
    rowwise(KktQAtyOp<true>{P.Q.view(), P.AT.view(), mi, xi.get(), yi2.get(), qx.get(), qx2.get(), aty.get(),
                            aty2.get()},
            P.sch_primal, sg.s, &l);
  } else {
    rowwise(KktAxOp<false>{P.A.view(), xi.get(), ax.get(), ax2.get()}, P.sch_dual, sg.s, &l);
    rowwise(KktQAtyOp<false>{P.Q.view(), P.AT.view(), mi, xi.get(), yi2.get(), qx.get(), qx2.get(), aty.get(),
                             aty2.get()},
            P.sch_primal, sg.s, &l);
  }
  const double *axp = ax.get(), *b = P.b.get(), *yp = yu.get();
  double h1[9];
  P.reduce_to_host<4, 5>(KktDualTerms{axp, axp, b, yp, yp, mi}, m, h1);
  const double *qxp = qx.get(), *atp = aty.get(), *xp = xu.get(), *c = P.c.get();
  double h2[kKktPrimalSums + kKktPrimalMaxes];
  P.reduce_to_host<kKktPrimalSums, kKktPrimalMaxes>(KktPrimalTerms{qxp, qxp, atp, atp, xp, xp, c}, n, h2);
  KktRaw r{};
  r.by_i[0] = h1[0], r.by_e[0] = h1[1], r.viol[0] = h1[4], r.ax_inf[0] = h1[6], r.b_inf = h1[8];
  primal_terms_into(r, h2);
  Kkt k2[2];
  finalize_kkt(r, k2);
  *out = k2[0];
}

void api_inner_step(const rapdhg_qp& p, rapdhg_iterate* s, const rapdhg_step_params& sp, int steps,
                    bool strict) {
  DeviceQP::validate_dims(p);
  StreamGuard sg;
  cudaStream_t st = sg.s;
  DeviceQP P(p, strict, st);
  const int n = P.n, m = P.m;
  DevBuf<double> X[2], XMD[2], w(n), xb(n), y(m), yb(m);
  for (int i = 0; i < 2; ++i) X[i].alloc(n), XMD[i].alloc(n);
  X[0].upload(s->x, n, st);
  X[1].upload(s->x_prev, n, st);
  xb.upload(s->x_bar, n, st);
  y.upload(s->y, m, st);
  yb.upload(s->y_bar, m, st);
  DevBuf<long long> bad(1);
  long long big = std::numeric_limits<long long>::max();
  bad.upload(&big, 1, st);
  std::vector<IterParams> ph(std::max(steps, 1));
  const double inv_beta = 1.0 / sp.beta;
  for (int i = 0; i < steps; ++i) {
    IterParams& q = ph[i];
    q.theta = sp.theta, q.ib = inv_beta, q.omib = 1.0 - inv_beta, q.eta = sp.eta, q.tau = sp.tau;
    q.theta_n = sp.theta, q.ib_n = inv_beta, q.omib_n = 1.0 - inv_beta;
    q.t = i + 1;
    q.emit_next = i + 1 < steps;
  }
  DevBuf<IterParams> params(ph.size());
  params.upload(ph.data(), ph.size(), st);
  int64_t l = 0;
  if (steps > 0) {
    prologue_kernel<<<grid1(n), 256, 0, st>>>(X[0].get(), X[1].get(), xb.get(), w.get(), XMD[0].get(), params.get(), n);
    RB_LAUNCH_CHECK();
  }
  for (int it = 0; it < steps; ++it) {
    const int c = it & 1;
    if (strict) {
      rowwise(DualStepOp<true>{P.A.view(), w.get(), P.b.get(), y.get(), yb.get(), P.mi, params.get(), it, bad.get()},
              P.sch_dual, st, &l);
      rowwise(PrimalStepOp<true>{P.Q.view(), P.AT.view(), XMD[c].get(), y.get(), X[c].get(), X[c ^ 1].get(), xb.get(),
                                 P.c.get(), w.get(), XMD[c ^ 1].get(), params.get(), it, bad.get()},
              P.sch_primal, st, &l);
    } else {
      rowwise(DualStepOp<false>{P.A.view(), w.get(), P.b.get(), y.get(), yb.get(), P.mi, params.get(), it, bad.get()},
              P.sch_dual, st, &l);
      rowwise(PrimalStepOp<false>{P.Q.view(), P.AT.view(), XMD[c].get(), y.get(), X[c].get(), X[c ^ 1].get(), xb.get(),
                                  P.c.get(), w.get(), XMD[c ^ 1].get(), params.get(), it, bad.get()},
              P.sch_primal, st, &l);
    }
  }
  const int cur = steps & 1;  // x is X[cur], x_prev X[cur^1]
  X[cur].download(s->x, n, st);
  X[cur ^ 1].download(s->x_prev, n, st);
  xb.download(s->x_bar, n, st);
  y.download(s->y, m, st);
  yb.download(s->y_bar, m, st);
  RB_CUDA(cudaStreamSynchronize(st));
  s->k += steps;
}

void api_scaling(const rapdhg_qp& p, int ruiz_iters, bool full, double* d1, double* d2, bool strict) {
  DeviceQP::validate_dims(p);
  StreamGuard sg;
  DeviceQP P(p, strict, sg.s);
  DevBuf<double> d;
  P.compute_scaling(ruiz_iters, full, d);
  RB_CUDA(cudaMemcpyAsync(d2, d.get(), sizeof(double) * P.n, cudaMemcpyDeviceToHost, sg.s));
  if (P.m) RB_CUDA(cudaMemcpyAsync(d1, d.get() + P.n, sizeof(double) * P.m, cudaMemcpyDeviceToHost, sg.s));
  RB_CUDA(cudaStreamSynchronize(sg.s));
}

void api_apply_scaling(const rapdhg_qp& p, const double* d1, const double* d2, double* qv,
                       double* aiv, double* aev, double* c, double* bi, double* be) {
  DeviceQP::validate_dims(p);
  StreamGuard sg;
  DeviceQP P(p, true, sg.s);
  DevBuf<double> d(static_cast<std::size_t>(P.n) + P.m);
  d.upload(d2, P.n, sg.s);
  if (P.m) RB_CUDA(cudaMemcpyAsync(d.get() + P.n, d1, sizeof(double) * P.m, cudaMemcpyHostToDevice, sg.s));
  DevBuf<double> qs, as, ats, cs, bs;
  P.scale_values(d.get(), qs, as, ats, cs, bs);
  qs.download(qv, P.Q.nnz, sg.s);
  as.download(aiv, p.a_ineq.nnz, sg.s);
  if (p.a_eq.nnz) RB_CUDA(cudaMemcpyAsync(aev, as.get() + p.a_ineq.nnz, sizeof(double) * p.a_eq.nnz, cudaMemcpyDeviceToHost, sg.s));
  cs.download(c, P.n, sg.s);
  bs.download(bi, P.mi, sg.s);
  if (P.me) RB_CUDA(cudaMemcpyAsync(be, bs.get() + P.mi, sizeof(double) * P.me, cudaMemcpyDeviceToHost, sg.s));
  RB_CUDA(cudaStreamSynchronize(sg.s));
}

double api_op_norm(const rapdhg_csr& mat, bool symmetric, int max_iters, double tol, uint64_t seed,
                   bool strict) {
  StreamGuard sg;
  std::vector<int32_t> zrp;
  if (symmetric) {
    if (mat.n_rows != mat.n_cols) invalid("estimate_op_norm_symmetric: matrix must be square");
    rapdhg_qp p{};
    zrp.assign(static_cast<std::size_t>(mat.n_cols) + 1, 0);
    std::vector<double> zeros(static_cast<std::size_t>(mat.n_cols) + 1, 0.0);
    p.n = mat.n_cols;
    p.q = mat;
    p.a_ineq = rapdhg_csr{0, mat.n_cols, 0, zrp.data(), nullptr, nullptr};
    p.a_eq = p.a_ineq;
    p.c = zeros.data();
    DeviceQP::validate_dims(p);
    DeviceQP P(p, strict, sg.s);
    return P.op_norm_q(P.Q.v.get(), max_iters, tol, seed);
  }
  rapdhg_qp p = single_matrix_qp(mat, zrp);
  std::vector<double> zeros(static_cast<std::size_t>(mat.n_cols) + static_cast<std::size_t>(mat.n_rows) + 1, 0.0);
  p.c = zeros.data();
  p.b_ineq = zeros.data();
  DeviceQP::validate_dims(p);
  DeviceQP P(p, strict, sg.s);
  return P.op_norm_a(P.A.v.get(), P.AT.v.get(), max_iters, tol, seed);
}

}  // namespace rb
