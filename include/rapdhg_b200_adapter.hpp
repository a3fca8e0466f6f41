// rapdhg_b200_adapter.hpp — reference-side binding (what a maintainer of the
// reference C++ solver adds to switch `rapdhg::solve` to the B200 library).
//
// Include AFTER the reference headers. canonicalize() is the drop-in for
// rapdhg::canonicalize (host-side, problem.hpp:131-198). Converts the reference's
// QuadraticProgram / SolverConfig (problem.hpp:24-34, solver.hpp:38-55) into
// the flat C-ABI structs of rapdhg_b200.h, calls rapdhg_solve(), and converts
// the result back into rapdhg::SolveResult (solver.hpp:76-89), re-throwing the
// reference's exception types with the library's message.
//
//   #include "rapdhg/solver.hpp"
//   #include "rapdhg_b200_adapter.hpp"
//   auto r = rapdhg_b200::solve(qp, cfg);          // same signature as rapdhg::solve
//
// Link with -L<repo>/paper_2311_07710_b200 -lrapdhg_b200.
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rapdhg/solver.hpp"
#include "rapdhg_b200.h"

namespace rapdhg_b200 {

// SparseMatrix keeps its CSR private (sparse.hpp:164-169); for_each walks it in
// row-major order, which is exactly CSR order.
struct CsrArrays {
  std::vector<int32_t> row_ptr, col_idx;
  std::vector<double> values;
  rapdhg_csr view(int rows, int cols) const {
    return rapdhg_csr{rows, cols, static_cast<int64_t>(values.size()), row_ptr.data(),
                      col_idx.data(), values.data()};
  }
};

inline CsrArrays to_csr(const rapdhg::SparseMatrix& m) {
  CsrArrays a;
  a.row_ptr.assign(static_cast<std::size_t>(m.rows()) + 1, 0);
  a.col_idx.reserve(m.nnz());
  a.values.reserve(m.nnz());
  m.for_each([&](int r, int c, double v) {
    ++a.row_ptr[r + 1];
    a.col_idx.push_back(c);
    a.values.push_back(v);
  });
  for (int r = 0; r < m.rows(); ++r) a.row_ptr[r + 1] += a.row_ptr[r];
  return a;
}

inline rapdhg_config to_config(const rapdhg::SolverConfig& c, int device = 0, bool strict = false) {
  rapdhg_config o;
  rapdhg_config_default(&o);
  o.algorithm = static_cast<int32_t>(c.algorithm);
  o.restart = static_cast<int32_t>(c.restart);
  o.restart_length = c.restart_length;
  o.step_rule = static_cast<int32_t>(c.step_rule);
  o.primal_weight = static_cast<int32_t>(c.primal_weight);
  o.fixed_primal_weight = c.fixed_primal_weight;
  o.tol = c.tol;
  o.max_iters = c.max_iters;
  o.time_limit_s = c.time_limit_s;
  o.check_interval = c.check_interval;
  o.scaling = c.scaling ? 1 : 0;
  o.seed = c.seed;
  o.snapshot_interval = c.snapshot_interval;
  o.record_restart_points = c.record_restart_points ? 1 : 0;
  o.device = device;
  o.strict_parity = strict ? 1 : 0;
  return o;
}

[[noreturn]] inline void rethrow(int rc) {
  const std::string msg = rapdhg_last_error();
  if (rc == RAPDHG_E_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == RAPDHG_E_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

inline std::vector<const char*> c_strs(const std::vector<std::string>& v) {
  std::vector<const char*> o;
  for (const std::string& x : v) o.push_back(x.c_str());
  return o;
}

inline rapdhg::SparseMatrix from_owned(const rapdhg_csr_owned& m) {
  std::vector<rapdhg::Triplet> t;
  for (int r = 0; r < m.n_rows; ++r)
    for (int64_t k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k) t.push_back({r, m.col_idx[k], m.values[k]});
  return rapdhg::SparseMatrix(m.n_rows, m.n_cols, std::move(t));
}

// Drop-in for rapdhg::canonicalize (problem.hpp:131-198) through
// rapdhg_canonicalize: RawProblem in, CanonicalProblem (qp + map) out.
inline rapdhg::CanonicalProblem canonicalize(const rapdhg::RawProblem& raw) {
  const CsrArrays q = to_csr(raw.q), a = to_csr(raw.a);
  std::vector<int32_t> types;
  for (rapdhg::RowType t : raw.row_types)
    types.push_back(t == rapdhg::RowType::kEq ? RAPDHG_ROW_EQ : t == rapdhg::RowType::kLe ? RAPDHG_ROW_LE
                                                                                          : RAPDHG_ROW_GE);
  const std::vector<const char*> rn = c_strs(raw.row_names), vn = c_strs(raw.var_names);
  rapdhg_raw_problem r{};
  r.n = raw.num_vars();
  r.m = raw.num_rows();
  r.q = q.view(raw.q.rows(), raw.q.cols());
  r.c = raw.c.data();
  r.obj_offset = raw.obj_offset;
  r.a = a.view(raw.a.rows(), raw.a.cols());
  r.row_types = types.data();
  r.rhs = raw.rhs.data();
  r.range = raw.range.empty() ? nullptr : raw.range.data();
  r.lower = raw.lower.data();
  r.upper = raw.upper.data();
  r.name = raw.name.c_str();
  r.row_names = rn.size() == raw.row_names.size() && !rn.empty() ? rn.data() : nullptr;
  r.var_names = vn.size() == raw.var_names.size() && !vn.empty() ? vn.data() : nullptr;
  rapdhg_qp_owned o{};
  rapdhg_canonical_map mp{};
  const int rc = rapdhg_canonicalize(&r, &o, &mp);
  if (rc != RAPDHG_OK) rethrow(rc);
  rapdhg::CanonicalProblem out;
  out.qp.q = from_owned(o.q);
  out.qp.a_ineq = from_owned(o.a_ineq);
  out.qp.a_eq = from_owned(o.a_eq);
  out.qp.c.assign(o.c, o.c + o.n);
  out.qp.b_ineq.assign(o.b_ineq, o.b_ineq + o.m_ineq);
  out.qp.b_eq.assign(o.b_eq, o.b_eq + o.m_eq);
  out.qp.obj_offset = o.obj_offset;
  if (o.name) out.qp.name = o.name;
  if (o.var_names)
    for (int j = 0; j < o.n; ++j) out.qp.var_names.emplace_back(o.var_names[j]);
  for (int i = 0; i < mp.n_ineq; ++i) out.map.ineq_labels.emplace_back(mp.ineq_labels[i]);
  for (int i = 0; i < mp.n_eq; ++i) out.map.eq_labels.emplace_back(mp.eq_labels[i]);
  rapdhg_qp_free(&o);
  rapdhg_canonical_map_free(&mp);
  return out;
}

// Drop-in for rapdhg::solve (solver.hpp:272).
inline rapdhg::SolveResult solve(const rapdhg::QuadraticProgram& p, const rapdhg::SolverConfig& cfg,
                                 int device = 0, bool strict_parity = false) {
  const CsrArrays q = to_csr(p.q), ai = to_csr(p.a_ineq), ae = to_csr(p.a_eq);
  const std::vector<const char*> vn = c_strs(p.var_names);
  rapdhg_qp qp{};
  qp.n = p.num_vars();
  qp.m_ineq = p.num_ineq();
  qp.m_eq = p.num_eq();
  qp.q = q.view(p.q.rows(), p.q.cols());
  qp.a_ineq = ai.view(p.a_ineq.rows(), p.a_ineq.cols());
  qp.a_eq = ae.view(p.a_eq.rows(), p.a_eq.cols());
  qp.c = p.c.data();
  qp.b_ineq = p.b_ineq.data();
  qp.b_eq = p.b_eq.data();
  qp.obj_offset = p.obj_offset;
  qp.name = p.name.c_str();
  qp.var_names = vn.size() == static_cast<std::size_t>(p.num_vars()) && !vn.empty() ? vn.data() : nullptr;
  const rapdhg_config c = to_config(cfg, device, strict_parity);
  rapdhg_result r{};
  const int rc = rapdhg_solve(&qp, &c, &r);
  if (rc != RAPDHG_OK) rethrow(rc);
  rapdhg::SolveResult out;
  out.status = static_cast<rapdhg::SolveStatus>(r.status);
  const int n = r.n, mi = r.m_ineq, me = r.m_eq, m = mi + me;
  auto point = [&](const double* x, const double* y) {
    rapdhg::PrimalDualPoint z;
    z.x.assign(x, x + n);
    z.y_ineq.assign(y, y + mi);
    z.y_eq.assign(y + mi, y + m);
    return z;
  };
  out.point.x.assign(r.x, r.x + n);
  out.point.y_ineq.assign(r.y_ineq, r.y_ineq + mi);
  out.point.y_eq.assign(r.y_eq, r.y_eq + me);
  out.residuals = {r.residuals.r_primal, r.residuals.r_dual, r.residuals.r_gap};
  out.iterations = r.iterations;
  out.restarts = r.restarts;
  out.solve_seconds = r.solve_seconds;
  out.norm_q = r.norm_q;
  out.norm_a = r.norm_a;
  out.norm_fallback = r.norm_fallback != 0;
  for (int64_t i = 0; i < r.n_log; ++i) {
    const rapdhg_log_record& L = r.log[i];
    out.log.push_back({L.iteration, L.r_primal, L.r_dual, L.r_gap, L.eta, L.omega, L.restarted != 0});
  }
  for (int64_t s = 0; s < r.n_snapshots; ++s)
    out.snapshots.emplace_back(r.snapshot_iters[s], point(r.snapshot_x + s * n, r.snapshot_y + s * m));
  for (int64_t s = 0; s < r.n_restart_points; ++s)
    out.restart_points.push_back(point(r.restart_x + s * n, r.restart_y + s * m));
  rapdhg_result_free(&r);
  return out;
}

}  // namespace rapdhg_b200
