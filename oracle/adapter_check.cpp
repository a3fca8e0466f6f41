// oracle/adapter_check.cpp — TEST ONLY. Drop-in demonstration: the same
// rapdhg::QuadraticProgram / SolverConfig go to the reference's rapdhg::solve
// (compiled in place from /root/reference) and to rapdhg_b200::solve (the B200
// library through include/rapdhg_b200_adapter.hpp). Strict mode must give a
// bit-identical SolveResult; fast mode the same status and KKT within 1e-6.
// Exit code 0 = pass. Built by oracle/Makefile into _ref/adapter_check.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <random>

#include "rapdhg/solver.hpp"
#include "rapdhg_b200_adapter.hpp"

using namespace rapdhg;

static QuadraticProgram random_qp(unsigned seed, int n, int mi, int me) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> N(0.0, 1.0);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<Triplet> pt, qt, ai, ae;
  for (int r = 0; r < n / 2; ++r)
    for (int c = 0; c < n; ++c)
      if (U(g) < 0.1) pt.push_back({r, c, N(g)});
  SparseMatrix P(n / 2, n, pt);
  std::vector<std::vector<std::pair<int, double>>> rows(n / 2);
  P.for_each([&](int r, int c, double v) { rows[r].push_back({c, v}); });
  for (auto& row : rows)
    for (auto& a : row)
      for (auto& b : row) qt.push_back({a.first, b.first, a.second * b.second});
  for (int i = 0; i < n; ++i) qt.push_back({i, i, 1e-2});
  std::vector<double> x0(n);
  for (double& v : x0) v = N(g);
  QuadraticProgram p;
  p.q = SparseMatrix(n, n, qt);
  for (int r = 0; r < mi; ++r)
    for (int c = 0; c < n; ++c)
      if (U(g) < 0.15) ai.push_back({r, c, N(g)});
  for (int r = 0; r < me; ++r)
    for (int c = 0; c < n; ++c)
      if (U(g) < 0.15) ae.push_back({r, c, N(g)});
  p.a_ineq = SparseMatrix(mi, n, ai);
  p.a_eq = SparseMatrix(me, n, ae);
  p.b_ineq = spmv(p.a_ineq, x0);
  for (double& v : p.b_ineq) v += U(g);
  p.b_eq = spmv(p.a_eq, x0);
  p.c.resize(n);
  for (double& v : p.c) v = N(g);
  return p;
}

// rapdhg::canonicalize vs rapdhg_b200::canonicalize on typed rows, ranges
// and bounds: identical canonical problems and labels (host only).
static int check_canonicalize() {
  std::mt19937_64 g(7);
  std::normal_distribution<double> N(0.0, 1.0);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  const int n = 9, m = 7;
  RawProblem raw;
  raw.name = "adapter";
  std::vector<Triplet> at, qt;
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < n; ++c)
      if (U(g) < 0.4) at.push_back({r, c, N(g)});
  for (int i = 0; i < n; ++i) qt.push_back({i, i, 1.0 + U(g)});
  raw.q = SparseMatrix(n, n, qt);
  raw.a = SparseMatrix(m, n, at);
  for (int j = 0; j < n; ++j) {
    raw.c.push_back(N(g));
    raw.lower.push_back(U(g) < 0.3 ? -kInf : -U(g));
    raw.upper.push_back(U(g) < 0.3 ? kInf : U(g));
    raw.var_names.push_back("v" + std::to_string(j));
  }
  for (int i = 0; i < m; ++i) {
    raw.row_types.push_back(static_cast<RowType>(i % 3));
    raw.rhs.push_back(N(g));
    raw.range.push_back(U(g) < 0.5 ? std::nan("") : 2 * N(g));
    raw.row_names.push_back("row" + std::to_string(i));
  }
  const CanonicalProblem a = canonicalize(raw);
  const CanonicalProblem b = rapdhg_b200::canonicalize(raw);
  auto same_m = [](const SparseMatrix& x, const SparseMatrix& y) {
    const std::vector<Triplet> tx = x.triplets(), ty = y.triplets();
    return x.rows() == y.rows() && x.cols() == y.cols() && tx.size() == ty.size() &&
           std::equal(tx.begin(), tx.end(), ty.begin(), [](const Triplet& p, const Triplet& q) {
             return p.row == q.row && p.col == q.col && p.value == q.value;
           });
  };
  const bool same = same_m(a.qp.q, b.qp.q) && same_m(a.qp.a_ineq, b.qp.a_ineq) && same_m(a.qp.a_eq, b.qp.a_eq) &&
                    a.qp.c == b.qp.c && a.qp.b_ineq == b.qp.b_ineq && a.qp.b_eq == b.qp.b_eq &&
                    a.qp.name == b.qp.name && a.qp.var_names == b.qp.var_names &&
                    a.map.ineq_labels == b.map.ineq_labels && a.map.eq_labels == b.map.eq_labels;
  std::printf("canonicalize: %s (%d ineq, %d eq rows)\n", same ? "identical" : "DIFFERENT", a.qp.num_ineq(),
              a.qp.num_eq());
  return same ? 0 : 1;
}

int main() {
  int fails = check_canonicalize();
  for (unsigned seed : {1u, 2u, 3u}) {
    const QuadraticProgram p = random_qp(seed, 50, 25, 6);
    SolverConfig cfg;
    cfg.tol = 1e-7;
    cfg.snapshot_interval = 40;
    cfg.record_restart_points = true;
    const SolveResult a = solve(p, cfg);
    const SolveResult b = rapdhg_b200::solve(p, cfg, 0, /*strict_parity=*/true);
    bool same = a.status == b.status && a.iterations == b.iterations && a.restarts == b.restarts &&
                a.point.x == b.point.x && a.point.y_ineq == b.point.y_ineq && a.point.y_eq == b.point.y_eq &&
                a.log.size() == b.log.size() && a.snapshots.size() == b.snapshots.size();
    for (std::size_t i = 0; same && i < a.log.size(); ++i)
      same = a.log[i].r_primal == b.log[i].r_primal && a.log[i].r_dual == b.log[i].r_dual &&
             a.log[i].r_gap == b.log[i].r_gap && a.log[i].omega == b.log[i].omega &&
             a.log[i].restarted == b.log[i].restarted;
    const SolveResult f = rapdhg_b200::solve(p, cfg, 0, false);
    const bool fast_ok = f.status == a.status && f.residuals.relkkt() <= cfg.tol &&
                         std::fabs(p.objective(f.point.x) - p.objective(a.point.x)) <=
                             1e-6 * std::max(1.0, std::fabs(p.objective(a.point.x)));
    std::printf("seed %u: reference %s %ld it, b200 strict %s (%ld it), fast %s (%ld it)\n", seed,
                to_string(a.status), a.iterations, same ? "bit-identical" : "DIFFERENT", b.iterations,
                fast_ok ? "ok" : "BAD", f.iterations);
    fails += !same + !fast_ok;
  }
  bool threw = false;
  try {
    QuadraticProgram bad = random_qp(4, 10, 3, 0);
    bad.b_ineq.push_back(1.0);
    rapdhg_b200::solve(bad, SolverConfig{});
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "inequality block dimension mismatch";
  }
  std::printf("invalid_argument rethrown: %s\n", threw ? "yes" : "NO");
  return fails + !threw;
}
