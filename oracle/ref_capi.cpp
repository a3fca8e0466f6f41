// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the checker, never shipped).
//
// A thin extern "C" wrapper that compiles the UNMODIFIED reference solver
// headers in place (-I /root/reference/proj/include; nothing is copied into
// this repo) into oracle/_ref/libref_rapdhg.so, so that tests and the
// bench's CPU-baseline arm can run the reference's own code on the same
// CSR arrays the GPU consumes. Only tests/, __graft_entry__.smoke() and
// bench.py's reference/cpu_baseline legs may load the result.
//
// Built by oracle/Makefile with `g++ -O2 -std=c++20 -ffp-contract=off` and no
// -march, so the reference never contracts a*b+c into an FMA,
// which is what makes the strict GPU mode bit-comparable.
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "rapdhg/kkt.hpp"
#include "rapdhg/opnorm.hpp"
#include "rapdhg/problem.hpp"
#include "rapdhg/qps.hpp"
#include "rapdhg/scaling.hpp"
#include "rapdhg/solver.hpp"
#include "rapdhg/sparse.hpp"
#include "rapdhg/stepsize.hpp"
#include "rapdhg_b200.h"

using namespace rapdhg;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return RAPDHG_E_OUT_OF_RANGE;
  } catch (const QpsParseError& e) {
    g_err = e.what();
    return RAPDHG_E_PARSE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RAPDHG_E_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RAPDHG_E_INTERNAL;
  }
}

SparseMatrix to_sparse(const rapdhg_csr& m) {
  std::vector<Triplet> t;
  t.reserve(static_cast<std::size_t>(m.nnz));
  for (int r = 0; r < m.n_rows; ++r)
    for (int k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k) t.push_back({r, m.col_idx[k], m.values[k]});
  return SparseMatrix(m.n_rows, m.n_cols, std::move(t));
}

Vec to_vec(const double* p, int n) { return n > 0 ? Vec(p, p + n) : Vec(); }

QuadraticProgram to_qp(const rapdhg_qp* p) {
  QuadraticProgram qp;
  qp.q = to_sparse(p->q);
  qp.c = to_vec(p->c, p->n);
  qp.a_ineq = to_sparse(p->a_ineq);
  qp.b_ineq = to_vec(p->b_ineq, p->m_ineq);
  qp.a_eq = to_sparse(p->a_eq);
  qp.b_eq = to_vec(p->b_eq, p->m_eq);
  qp.obj_offset = p->obj_offset;
  if (p->name) qp.name = p->name;
  if (p->var_names)
    for (int j = 0; j < p->n; ++j) qp.var_names.emplace_back(p->var_names[j] ? p->var_names[j] : "");
  return qp;
}

char* dup_str(const std::string& v) {
  char* p = static_cast<char*>(std::malloc(v.size() + 1));
  std::memcpy(p, v.c_str(), v.size() + 1);
  return p;
}

char** dup_strs(const std::vector<std::string>& v) {
  char** p = static_cast<char**>(std::calloc(v.size() ? v.size() : 1, sizeof(char*)));
  for (std::size_t i = 0; i < v.size(); ++i) p[i] = dup_str(v[i]);
  return p;
}

SolverConfig to_cfg(const rapdhg_config* c) {
  SolverConfig s;
  s.algorithm = static_cast<Algorithm>(c->algorithm);
  s.restart = static_cast<RestartPolicy>(c->restart);
  s.restart_length = c->restart_length;
  s.step_rule = static_cast<StepRule>(c->step_rule);
  s.primal_weight = static_cast<PrimalWeightMode>(c->primal_weight);
  s.fixed_primal_weight = c->fixed_primal_weight;
  s.tol = c->tol;
  s.max_iters = c->max_iters;
  s.time_limit_s = c->time_limit_s;
  s.check_interval = c->check_interval;
  s.scaling = c->scaling != 0;
  s.seed = c->seed;
  s.snapshot_interval = c->snapshot_interval;
  s.record_restart_points = c->record_restart_points != 0;
  return s;
}

template <typename T>
T* dup(const T* src, std::size_t n) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (n ? n : 1)));
  if (n) std::memcpy(p, src, sizeof(T) * n);
  return p;
}

void fill_csr(const SparseMatrix& m, rapdhg_csr_owned* o) {
  o->n_rows = m.rows();
  o->n_cols = m.cols();
  o->nnz = static_cast<int64_t>(m.nnz());
  o->row_ptr = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (m.rows() + 1)));
  o->col_idx = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (m.nnz() ? m.nnz() : 1)));
  o->values = static_cast<double*>(std::malloc(sizeof(double) * (m.nnz() ? m.nnz() : 1)));
  for (int r = 0; r <= m.rows(); ++r) o->row_ptr[r] = 0;
  std::size_t k = 0;
  m.for_each([&](int r, int c, double v) {
    ++o->row_ptr[r + 1];
    o->col_idx[k] = c;
    o->values[k] = v;
    ++k;
  });
  for (int r = 0; r < m.rows(); ++r) o->row_ptr[r + 1] += o->row_ptr[r];
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_solve(const rapdhg_qp* p, const rapdhg_config* c, rapdhg_result* out) {
  return guard([&] {
    const QuadraticProgram qp = to_qp(p);
    const SolveResult r = solve(qp, to_cfg(c));
    std::memset(out, 0, sizeof(*out));
    out->status = static_cast<int32_t>(r.status);
    out->n = qp.num_vars();
    out->m_ineq = qp.num_ineq();
    out->m_eq = qp.num_eq();
    out->x = dup(r.point.x.data(), r.point.x.size());
    out->y_ineq = dup(r.point.y_ineq.data(), r.point.y_ineq.size());
    out->y_eq = dup(r.point.y_eq.data(), r.point.y_eq.size());
    out->residuals = {r.residuals.r_primal, r.residuals.r_dual, r.residuals.r_gap};
    out->iterations = r.iterations;
    out->restarts = r.restarts;
    out->solve_seconds = r.solve_seconds;
    out->norm_q = r.norm_q;
    out->norm_a = r.norm_a;
    out->norm_fallback = r.norm_fallback;
    out->n_log = static_cast<int64_t>(r.log.size());
    out->log = static_cast<rapdhg_log_record*>(
        std::malloc(sizeof(rapdhg_log_record) * (r.log.size() ? r.log.size() : 1)));
    for (std::size_t i = 0; i < r.log.size(); ++i) {
      const LogRecord& L = r.log[i];
      out->log[i] = {L.iteration, L.r_primal, L.r_dual, L.r_gap, L.eta, L.omega, L.restarted};
    }
    const std::size_t n = qp.num_vars(), m = qp.num_rows();
    out->n_snapshots = static_cast<int64_t>(r.snapshots.size());
    out->snapshot_iters = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (r.snapshots.size() + 1)));
    out->snapshot_x = static_cast<double*>(std::malloc(sizeof(double) * (r.snapshots.size() * n + 1)));
    out->snapshot_y = static_cast<double*>(std::malloc(sizeof(double) * (r.snapshots.size() * m + 1)));
    for (std::size_t s = 0; s < r.snapshots.size(); ++s) {
      out->snapshot_iters[s] = r.snapshots[s].first;
      const PrimalDualPoint& z = r.snapshots[s].second;
      std::copy(z.x.begin(), z.x.end(), out->snapshot_x + s * n);
      std::copy(z.y_ineq.begin(), z.y_ineq.end(), out->snapshot_y + s * m);
      std::copy(z.y_eq.begin(), z.y_eq.end(), out->snapshot_y + s * m + z.y_ineq.size());
    }
    out->n_restart_points = static_cast<int64_t>(r.restart_points.size());
    out->restart_x = static_cast<double*>(std::malloc(sizeof(double) * (r.restart_points.size() * n + 1)));
    out->restart_y = static_cast<double*>(std::malloc(sizeof(double) * (r.restart_points.size() * m + 1)));
    for (std::size_t s = 0; s < r.restart_points.size(); ++s) {
      const PrimalDualPoint& z = r.restart_points[s];
      std::copy(z.x.begin(), z.x.end(), out->restart_x + s * n);
      std::copy(z.y_ineq.begin(), z.y_ineq.end(), out->restart_y + s * m);
      std::copy(z.y_eq.begin(), z.y_eq.end(), out->restart_y + s * m + z.y_ineq.size());
    }
  });
}

void ref_result_free(rapdhg_result* r) {
  if (!r) return;
  std::free(r->x);
  std::free(r->y_ineq);
  std::free(r->y_eq);
  std::free(r->log);
  std::free(r->snapshot_iters);
  std::free(r->snapshot_x);
  std::free(r->snapshot_y);
  std::free(r->restart_x);
  std::free(r->restart_y);
  std::memset(r, 0, sizeof(*r));
}

int ref_spmv(const rapdhg_csr* m, const double* x, int64_t x_len, double* y) {
  return guard([&] {
    const SparseMatrix s = to_sparse(*m);
    Vec out;
    s.multiply(to_vec(x, static_cast<int>(x_len)), out);
    std::copy(out.begin(), out.end(), y);
  });
}

int ref_spmv_t(const rapdhg_csr* m, const double* x, int64_t x_len, double* y) {
  return guard([&] {
    const SparseMatrix s = to_sparse(*m);
    Vec out;
    s.multiply_transpose(to_vec(x, static_cast<int>(x_len)), out);
    std::copy(out.begin(), out.end(), y);
  });
}

int ref_transpose(const rapdhg_csr* m, rapdhg_csr_owned* out) {
  return guard([&] { fill_csr(to_sparse(*m).transpose(), out); });
}

int ref_symmetry_gap(const rapdhg_csr* m, double* out) {
  return guard([&] { *out = to_sparse(*m).symmetry_gap(); });
}

int ref_inner_step(const rapdhg_qp* p, rapdhg_iterate* s, const rapdhg_step_params* sp,
                   int32_t steps) {
  return guard([&] {
    const QuadraticProgram qp = to_qp(p);
    const WorkingProblem wp = WorkingProblem::from(qp);
    const int n = qp.num_vars(), m = qp.num_rows();
    IterateState st;
    st.x = to_vec(s->x, n);
    st.x_prev = to_vec(s->x_prev, n);
    st.y = to_vec(s->y, m);
    st.x_bar = to_vec(s->x_bar, n);
    st.y_bar = to_vec(s->y_bar, m);
    st.k = s->k;
    st.n = s->n;
    StepParams params{sp->beta, sp->theta, sp->eta, sp->tau};
    StepWorkspace ws;
    for (int i = 0; i < steps; ++i) inner_step_inplace(st, wp, params, ws);
    std::copy(st.x.begin(), st.x.end(), s->x);
    std::copy(st.x_prev.begin(), st.x_prev.end(), s->x_prev);
    std::copy(st.y.begin(), st.y.end(), s->y);
    std::copy(st.x_bar.begin(), st.x_bar.end(), s->x_bar);
    std::copy(st.y_bar.begin(), st.y_bar.end(), s->y_bar);
    s->k = st.k;
    s->n = st.n;
  });
}

int ref_rel_kkt(const rapdhg_qp* p, const double* x, const double* y_ineq, const double* y_eq,
                rapdhg_kkt* out) {
  return guard([&] {
    const QuadraticProgram qp = to_qp(p);
    PrimalDualPoint z;
    z.x = to_vec(x, qp.num_vars());
    z.y_ineq = to_vec(y_ineq, qp.num_ineq());
    z.y_eq = to_vec(y_eq, qp.num_eq());
    const KktResiduals r = rel_kkt(qp, z);
    *out = {r.r_primal, r.r_dual, r.r_gap};
  });
}

int ref_compute_scaling(const rapdhg_qp* p, double* d1, double* d2) {
  return guard([&] {
    const ScalingInfo s = compute_scaling(to_qp(p));
    std::copy(s.d1.begin(), s.d1.end(), d1);
    std::copy(s.d2.begin(), s.d2.end(), d2);
  });
}

int ref_ruiz_scaling(const rapdhg_qp* p, int32_t iterations, double* d1, double* d2) {
  return guard([&] {
    const ScalingInfo s = ruiz_scaling(to_qp(p), iterations);
    std::copy(s.d1.begin(), s.d1.end(), d1);
    std::copy(s.d2.begin(), s.d2.end(), d2);
  });
}

// Scaled problem values (scaling.hpp:109-123). Patterns are unchanged unless a
// scaled entry underflows to exactly 0 (then SparseMatrix drops it); *dropped
// reports how many entries the reference dropped.
int ref_apply_scaling(const rapdhg_qp* p, const double* d1, const double* d2, double* qv,
                      double* aiv, double* aev, double* c, double* bi, double* be,
                      int64_t* dropped) {
  return guard([&] {
    const QuadraticProgram qp = to_qp(p);
    ScalingInfo s;
    s.d1 = to_vec(d1, qp.num_rows());
    s.d2 = to_vec(d2, qp.num_vars());
    const QuadraticProgram o = apply_scaling(qp, s);
    int64_t k = 0;
    o.q.for_each([&](int, int, double v) { qv[k++] = v; });
    int64_t d = static_cast<int64_t>(qp.q.nnz()) - k;
    k = 0;
    o.a_ineq.for_each([&](int, int, double v) { aiv[k++] = v; });
    d += static_cast<int64_t>(qp.a_ineq.nnz()) - k;
    k = 0;
    o.a_eq.for_each([&](int, int, double v) { aev[k++] = v; });
    d += static_cast<int64_t>(qp.a_eq.nnz()) - k;
    std::copy(o.c.begin(), o.c.end(), c);
    std::copy(o.b_ineq.begin(), o.b_ineq.end(), bi);
    std::copy(o.b_eq.begin(), o.b_eq.end(), be);
    if (dropped) *dropped = d;
  });
}

int ref_estimate_op_norm(const rapdhg_csr* m, int32_t max_iters, double tol, uint64_t seed,
                         double* out) {
  return guard([&] {
    PowerIterOptions o;
    o.max_iters = max_iters;
    o.tol = tol;
    o.seed = seed;
    *out = estimate_op_norm(to_sparse(*m), o);
  });
}

int ref_estimate_op_norm_symmetric(const rapdhg_csr* m, int32_t max_iters, double tol,
                                   uint64_t seed, double* out) {
  return guard([&] {
    PowerIterOptions o;
    o.max_iters = max_iters;
    o.tol = tol;
    o.seed = seed;
    *out = estimate_op_norm_symmetric(to_sparse(*m), o);
  });
}

int ref_step_schedule_theoretical(int32_t k, int32_t horizon, double nq, double na,
                                  rapdhg_step_params* out) {
  return guard([&] {
    const StepParams s = step_schedule_theoretical(k, horizon, nq, na);
    *out = {s.beta, s.theta, s.eta, s.tau};
  });
}

int ref_pdhg_constant_steps(double nq, double na, rapdhg_step_params* out) {
  return guard([&] {
    const StepParams s = pdhg_constant_steps(nq, na);
    *out = {s.beta, s.theta, s.eta, s.tau};
  });
}

int ref_adaptive_eta(int32_t k, double prev, double nq, double na, double omega, double* out) {
  return guard([&] { *out = adaptive_eta(k, prev, nq, na, omega); });
}

int ref_primal_weight_init(const double* c, int64_t n, const double* b, int64_t m, double* out) {
  return guard([&] { *out = primal_weight_init(to_vec(c, (int)n), to_vec(b, (int)m)); });
}

int ref_primal_weight_update(double dx, double dy, double omega_prev, double* out) {
  return guard([&] { *out = primal_weight_update(dx, dy, omega_prev); });
}

int ref_restart_decision(int32_t policy, double cand, double cand_prev, double start, int64_t k,
                         int64_t total, int64_t fixed_length) {
  int result = 0;
  const int rc = guard([&] {
    RestartContext ctx;
    ctx.relkkt_candidate = cand;
    ctx.relkkt_candidate_prev = cand_prev;
    ctx.relkkt_epoch_start = start;
    ctx.k = k;
    ctx.total_iters = total;
    result = restart_decision(static_cast<RestartPolicy>(policy), ctx, fixed_length) ? 1 : 0;
  });
  return rc ? rc : result;
}

int ref_csr_from_triplets(int32_t n_rows, int32_t n_cols, int64_t nnz, const int32_t* rows,
                          const int32_t* cols, const double* vals, rapdhg_csr_owned* out) {
  return guard([&] {
    std::vector<Triplet> t(static_cast<std::size_t>(nnz));
    for (int64_t i = 0; i < nnz; ++i) t[i] = {rows[i], cols[i], vals[i]};
    fill_csr(SparseMatrix(n_rows, n_cols, std::move(t)), out);
  });
}

void fill_canonical(const CanonicalProblem& cp, rapdhg_qp_owned* out, rapdhg_canonical_map* map) {
  const QuadraticProgram& qp = cp.qp;
  std::memset(out, 0, sizeof(*out));
  out->n = qp.num_vars();
  out->m_ineq = qp.num_ineq();
  out->m_eq = qp.num_eq();
  fill_csr(qp.q, &out->q);
  fill_csr(qp.a_ineq, &out->a_ineq);
  fill_csr(qp.a_eq, &out->a_eq);
  out->c = dup(qp.c.data(), qp.c.size());
  out->b_ineq = dup(qp.b_ineq.data(), qp.b_ineq.size());
  out->b_eq = dup(qp.b_eq.data(), qp.b_eq.size());
  out->obj_offset = qp.obj_offset;
  out->name = dup_str(qp.name);
  if (!qp.var_names.empty()) out->var_names = dup_strs(qp.var_names);
  if (map) {
    map->n_ineq = static_cast<int32_t>(cp.map.ineq_labels.size());
    map->n_eq = static_cast<int32_t>(cp.map.eq_labels.size());
    map->ineq_labels = dup_strs(cp.map.ineq_labels);
    map->eq_labels = dup_strs(cp.map.eq_labels);
  }
}

// RawProblem (problem.hpp:76-92) from its C view, then canonicalize
// (problem.hpp:131-198) itself.
int ref_canonicalize(const rapdhg_raw_problem* r, rapdhg_qp_owned* out, rapdhg_canonical_map* map) {
  return guard([&] {
    RawProblem raw;
    if (r->name) raw.name = r->name;
    raw.q = to_sparse(r->q);
    raw.c = to_vec(r->c, r->n);
    raw.obj_offset = r->obj_offset;
    raw.a = to_sparse(r->a);
    for (int i = 0; i < r->m; ++i)
      raw.row_types.push_back(r->row_types[i] == RAPDHG_ROW_EQ ? RowType::kEq
                              : r->row_types[i] == RAPDHG_ROW_LE ? RowType::kLe : RowType::kGe);
    raw.rhs = to_vec(r->rhs, r->m);
    raw.range = r->range ? to_vec(r->range, r->m) : Vec(r->m, std::nan(""));
    raw.lower = to_vec(r->lower, r->n);
    raw.upper = to_vec(r->upper, r->n);
    if (r->row_names)
      for (int i = 0; i < r->m; ++i) raw.row_names.emplace_back(r->row_names[i]);
    if (r->var_names)
      for (int j = 0; j < r->n; ++j) raw.var_names.emplace_back(r->var_names[j]);
    fill_canonical(canonicalize(raw), out, map);
  });
}

int ref_parse_qps_map(const char* text, rapdhg_qp_owned* out, rapdhg_canonical_map* map) {
  return guard([&] {
    std::istringstream in{std::string(text)};
    fill_canonical(canonicalize(parse_qps(in)), out, map);
  });
}

void ref_canonical_map_free(rapdhg_canonical_map* map) {
  for (int i = 0; i < map->n_ineq; ++i) std::free(map->ineq_labels[i]);
  for (int i = 0; i < map->n_eq; ++i) std::free(map->eq_labels[i]);
  std::free(map->ineq_labels);
  std::free(map->eq_labels);
  std::memset(map, 0, sizeof(*map));
}

// QPS text -> canonical QP (qps.hpp:69-298 then problem.hpp:131-198).
int ref_parse_qps_canonical(const char* text, rapdhg_qp_owned* out) {
  return guard([&] {
    std::istringstream in{std::string(text)};
    const RawProblem raw = parse_qps(in);
    const CanonicalProblem cp = canonicalize(raw);
    const QuadraticProgram& qp = cp.qp;
    std::memset(out, 0, sizeof(*out));
    out->n = qp.num_vars();
    out->m_ineq = qp.num_ineq();
    out->m_eq = qp.num_eq();
    fill_csr(qp.q, &out->q);
    fill_csr(qp.a_ineq, &out->a_ineq);
    fill_csr(qp.a_eq, &out->a_eq);
    out->c = dup(qp.c.data(), qp.c.size());
    out->b_ineq = dup(qp.b_ineq.data(), qp.b_ineq.size());
    out->b_eq = dup(qp.b_eq.data(), qp.b_eq.size());
    out->obj_offset = qp.obj_offset;
  });
}

// write_qps (qps.hpp:320-381) of a canonical problem; free with ref_free.
int ref_write_qps(const rapdhg_qp* p, char** out) {
  return guard([&] {
    const std::string s = write_qps_string(to_qp(p));
    *out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out, s.c_str(), s.size() + 1);
  });
}

void ref_free(void* p) { std::free(p); }

void ref_csr_free(rapdhg_csr_owned* m) {
  if (!m) return;
  std::free(m->row_ptr);
  std::free(m->col_idx);
  std::free(m->values);
  std::memset(m, 0, sizeof(*m));
}

void ref_qp_free(rapdhg_qp_owned* p) {
  if (!p) return;
  ref_csr_free(&p->q);
  ref_csr_free(&p->a_ineq);
  ref_csr_free(&p->a_eq);
  std::free(p->c);
  std::free(p->b_ineq);
  std::free(p->b_eq);
  std::free(p->name);
  if (p->var_names)
    for (int j = 0; j < p->n; ++j) std::free(p->var_names[j]);
  std::free(p->var_names);
  std::memset(p, 0, sizeof(*p));
}

}  // extern "C"
