/*
 * oracle/rapdhg_oracle.c — TEST INFRASTRUCTURE ONLY (the checker).
 *
 * A plain-C restatement of the reference rAPDHG solver path
 * (/root/reference/proj/include/rapdhg/*.hpp), written from the reference's
 * algorithm, function by function, each citing the file:line it follows.
 * It is pinned two ways by tests/test_oracle.py:
 *   1. bit-for-bit against the reference itself, compiled unmodified into
 *      oracle/_ref/libref_rapdhg.so (oracle/Makefile), on seeded instances;
 *   2. against the SPEC.md known-answer examples.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it; the product (paper_2311_07710_b200/) never links it.
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction) like the reference.
 * Sums are sequential in the reference's order so results are bit-identical.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "rapdhg_b200.h"

static const char* g_err = "";
const char* orc_last_error(void) { return g_err; }

#define FAIL(msg)          \
  do {                     \
    g_err = (msg);         \
    return RAPDHG_E_INVALID_ARGUMENT; \
  } while (0)

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* ---- vec.hpp -------------------------------------------------------- */
/* vec.hpp:14-18 */
static double v_dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
/* vec.hpp:20 */
static double v_norm2(const double* a, int64_t n) { return sqrt(v_dot(a, a, n)); }
/* vec.hpp:28-35 */
static double v_dist2(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  return sqrt(s);
}
/* vec.hpp:53-57 */
static int v_all_finite(const double* a, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

/* ---- sparse.hpp ----------------------------------------------------- */
/* sparse.hpp:79-88: sequential row gather from +0.0 */
static void csr_mul(const rapdhg_csr* m, const double* x, double* y) {
  for (int r = 0; r < m->n_rows; ++r) {
    double s = 0.0;
    for (int k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k) s += m->values[k] * x[m->col_idx[k]];
    y[r] = s;
  }
}
/* sparse.hpp:91-100: scatter in increasing row order, skipping x[r] == 0 */
static void csr_mul_t(const rapdhg_csr* m, const double* x, double* y) {
  for (int c = 0; c < m->n_cols; ++c) y[c] = 0.0;
  for (int r = 0; r < m->n_rows; ++r) {
    const double xr = x[r];
    if (xr == 0.0) continue;
    for (int k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k) y[m->col_idx[k]] += m->values[k] * xr;
  }
}

int orc_spmv(const rapdhg_csr* m, const double* x, int64_t x_len, double* y) {
  if (x_len != m->n_cols) FAIL("spmv: vector length does not match column count");
  csr_mul(m, x, y);
  return 0;
}
int orc_spmv_t(const rapdhg_csr* m, const double* x, int64_t x_len, double* y) {
  if (x_len != m->n_rows) FAIL("spmv_t: vector length does not match row count");
  csr_mul_t(m, x, y);
  return 0;
}

/* Owned CSR used internally (stacked A, transposes). */
typedef struct {
  int32_t rows, cols;
  int64_t nnz;
  int32_t* rp;
  int32_t* ci;
  double* v;
} ocsr;

static rapdhg_csr view(const ocsr* o) {
  rapdhg_csr c = {o->rows, o->cols, o->nnz, o->rp, o->ci, o->v};
  return c;
}
static void ocsr_free(ocsr* o) {
  free(o->rp);
  free(o->ci);
  free(o->v);
}

/* WorkingProblem::from (solver.hpp:101-112): [A_ineq; A_eq] stacked */
static ocsr stack_rows(const rapdhg_csr* a, const rapdhg_csr* b, int n) {
  ocsr o;
  o.rows = a->n_rows + b->n_rows;
  o.cols = n;
  o.nnz = a->nnz + b->nnz;
  o.rp = (int32_t*)malloc(sizeof(int32_t) * (o.rows + 1));
  o.ci = (int32_t*)malloc(sizeof(int32_t) * (o.nnz + 1));
  o.v = (double*)malloc(sizeof(double) * (o.nnz + 1));
  for (int r = 0; r <= a->n_rows; ++r) o.rp[r] = a->row_ptr[r];
  for (int r = 1; r <= b->n_rows; ++r) o.rp[a->n_rows + r] = (int32_t)a->nnz + b->row_ptr[r];
  if (a->nnz) memcpy(o.ci, a->col_idx, sizeof(int32_t) * a->nnz);
  if (a->nnz) memcpy(o.v, a->values, sizeof(double) * a->nnz);
  if (b->nnz) memcpy(o.ci + a->nnz, b->col_idx, sizeof(int32_t) * b->nnz);
  if (b->nnz) memcpy(o.v + a->nnz, b->values, sizeof(double) * b->nnz);
  return o;
}

/* SparseMatrix::transpose (sparse.hpp:102-108): stable counting sort by column
 * keeps entries of each transposed row in increasing original-row order. */
static ocsr transpose(const rapdhg_csr* m) {
  ocsr o;
  o.rows = m->n_cols;
  o.cols = m->n_rows;
  o.nnz = m->nnz;
  o.rp = (int32_t*)calloc(o.rows + 1, sizeof(int32_t));
  o.ci = (int32_t*)malloc(sizeof(int32_t) * (o.nnz + 1));
  o.v = (double*)malloc(sizeof(double) * (o.nnz + 1));
  for (int64_t k = 0; k < m->nnz; ++k) o.rp[m->col_idx[k] + 1]++;
  for (int r = 0; r < o.rows; ++r) o.rp[r + 1] += o.rp[r];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (o.rows + 1));
  memcpy(fill, o.rp, sizeof(int32_t) * (o.rows + 1));
  for (int r = 0; r < m->n_rows; ++r)
    for (int k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k) {
      const int32_t p = fill[m->col_idx[k]]++;
      o.ci[p] = r;
      o.v[p] = m->values[k];
    }
  free(fill);
  return o;
}

/* symmetry_gap (sparse.hpp:119-138): max |M_ij - M_ji| over the union. */
static double symmetry_gap(const rapdhg_csr* m) {
  ocsr t = transpose(m);
  double gap = 0.0;
  for (int r = 0; r < m->n_rows; ++r) {
    int i = m->row_ptr[r], ie = m->row_ptr[r + 1], j = t.rp[r], je = t.rp[r + 1];
    while (i < ie || j < je) {
      if (j == je || (i < ie && m->col_idx[i] < t.ci[j])) {
        gap = dmax(gap, fabs(m->values[i]));
        ++i;
      } else if (i == ie || t.ci[j] < m->col_idx[i]) {
        gap = dmax(gap, fabs(t.v[j]));
        ++j;
      } else {
        gap = dmax(gap, fabs(m->values[i] - t.v[j]));
        ++i;
        ++j;
      }
    }
  }
  ocsr_free(&t);
  return gap;
}
/* sparse.hpp:140-144 */
static double max_abs(const rapdhg_csr* m) {
  double r = 0.0;
  for (int64_t k = 0; k < m->nnz; ++k) r = dmax(r, fabs(m->values[k]));
  return r;
}

int orc_symmetry_gap(const rapdhg_csr* m, double* out) {
  *out = symmetry_gap(m);
  return 0;
}

/* QuadraticProgram::validate (problem.hpp:40-50) */
static int validate_qp(const rapdhg_qp* p) {
  const int n = p->n;
  if (p->q.n_rows != n || p->q.n_cols != n) FAIL("Q dimension mismatch");
  if (p->a_ineq.n_rows != p->m_ineq || p->a_ineq.n_cols != n)
    FAIL("inequality block dimension mismatch");
  if (p->a_eq.n_rows != p->m_eq || p->a_eq.n_cols != n) FAIL("equality block dimension mismatch");
  const double gap = symmetry_gap(&p->q);
  if (gap > 1e-12 * dmax(1.0, max_abs(&p->q))) FAIL("Q is not symmetric");
  return 0;
}

/* ---- stepsize.hpp --------------------------------------------------- */
/* stepsize.hpp:31-42 */
int orc_step_schedule_theoretical(int32_t k, int32_t horizon, double nq, double na,
                                  rapdhg_step_params* sp) {
  if (horizon < 1) FAIL("step schedule: horizon must be >= 1");
  if (k < 0 || k >= horizon) FAIL("step schedule: k out of range");
  if (na <= 0.0) na = nq / horizon;
  if (na <= 0.0) FAIL("step schedule: both norms are zero");
  sp->beta = 0.5 * (k + 2);
  sp->theta = (double)k / (k + 1);
  sp->eta = (k + 1) / (2.0 * (nq + horizon * na));
  sp->tau = (k + 1) / (2.0 * horizon * na);
  return 0;
}
/* stepsize.hpp:47-54 */
int orc_pdhg_constant_steps(double nq, double na, rapdhg_step_params* sp) {
  if (na <= 0.0) {
    if (nq <= 0.0) FAIL("pdhg steps: both norms are zero");
    sp->beta = 1.0, sp->theta = 1.0, sp->eta = 1.0 / nq, sp->tau = 0.0;
    return 0;
  }
  sp->beta = 1.0, sp->theta = 1.0, sp->eta = 1.0 / (nq + 2.0 * na), sp->tau = 1.0 / (2.0 * na);
  return 0;
}
/* stepsize.hpp:59-68 */
int orc_adaptive_eta(int32_t k, double prev, double nq, double na, double omega, double* out) {
  if (omega <= 0.0) FAIL("adaptive_eta: omega must be positive");
  if (nq <= 0.0 && na <= 0.0) FAIL("adaptive_eta: both norms are zero");
  const double qw = nq / omega;
  if (k == 0) {
    *out = 1.98 / (qw + sqrt(4.0 * na * na + qw * qw));
    return 0;
  }
  const double fresh = 0.99 * (k + 2) / (qw + sqrt(na * na * (k + 2.0) * (k + 2.0) + qw * qw));
  const double grow = (1.0 + 1.0 / k) * prev;
  *out = (fresh < grow) ? fresh : grow; /* std::min(grow, fresh) */
  return 0;
}
/* stepsize.hpp:73-78 */
int orc_primal_weight_init(const double* c, int64_t n, const double* b, int64_t m, double* out) {
  const double nc = v_norm2(c, n), nb = v_norm2(b, m);
  *out = (nc > 1e-10 && nb > 1e-10) ? nc / nb : 1.0;
  return 0;
}
/* stepsize.hpp:83-88 */
int orc_primal_weight_update(double dx, double dy, double w, double* out) {
  if (w <= 0.0) FAIL("primal weight must be positive");
  if (dx <= 1e-10 || dy <= 1e-10) {
    *out = w;
    return 0;
  }
  *out = exp(0.2 * log(dy / dx) + (1.0 - 0.2) * log(w));
  return 0;
}

/* solver.hpp:218-235 */
int orc_restart_decision(int32_t policy, double cand, double cand_prev, double start, int64_t k,
                         int64_t total, int64_t fixed_length) {
  switch (policy) {
    case RAPDHG_RESTART_NONE: return 0;
    case RAPDHG_RESTART_FIXED: return k >= fixed_length;
    case RAPDHG_RESTART_HALVING: return cand <= 0.5 * start;
    case RAPDHG_RESTART_PDQP:
      if (cand <= 0.2 * start) return 1;
      if (cand <= 0.8 * start && cand > cand_prev) return 1;
      return k >= 0.36 * (double)total;
  }
  return 0;
}

/* ---- kkt.hpp:28-72 -------------------------------------------------- */
int orc_rel_kkt(const rapdhg_qp* p, const double* x, const double* yi, const double* ye,
                rapdhg_kkt* out) {
  const int n = p->n, mi = p->m_ineq, me = p->m_eq;
  for (int i = 0; i < mi; ++i)
    if (yi[i] < -1e-9) FAIL("rel_kkt: negative inequality dual");
  double* ax_i = (double*)malloc(sizeof(double) * (mi + 1));
  double* ax_e = (double*)malloc(sizeof(double) * (me + 1));
  double* qx = (double*)malloc(sizeof(double) * (n + 1));
  double* aty = (double*)malloc(sizeof(double) * (n + 1));
  double* aty_e = (double*)malloc(sizeof(double) * (n + 1));
  csr_mul(&p->a_ineq, x, ax_i);
  csr_mul(&p->a_eq, x, ax_e);
  csr_mul(&p->q, x, qx);
  csr_mul_t(&p->a_ineq, yi, aty);
  csr_mul_t(&p->a_eq, ye, aty_e);
  for (int j = 0; j < n; ++j) aty[j] += 1.0 * aty_e[j]; /* axpy(1.0, ...) vec.hpp:38 */

  double viol = 0.0, ax_inf = 0.0, b_inf = 0.0;
  for (int i = 0; i < mi; ++i) {
    viol = dmax(viol, ax_i[i] - p->b_ineq[i]);
    ax_inf = dmax(ax_inf, fabs(ax_i[i]));
    b_inf = dmax(b_inf, fabs(p->b_ineq[i]));
  }
  for (int i = 0; i < me; ++i) {
    viol = dmax(viol, fabs(ax_e[i] - p->b_eq[i]));
    ax_inf = dmax(ax_inf, fabs(ax_e[i]));
    b_inf = dmax(b_inf, fabs(p->b_eq[i]));
  }
  out->r_primal = dmax(viol, 0.0) / (1.0 + dmax(ax_inf, b_inf));

  double dn = 0.0, qi = 0.0, ai = 0.0, ci = 0.0;
  for (int j = 0; j < n; ++j) {
    dn = dmax(dn, fabs(qx[j] + aty[j] + p->c[j]));
    qi = dmax(qi, fabs(qx[j]));
    ai = dmax(ai, fabs(aty[j]));
    ci = dmax(ci, fabs(p->c[j]));
  }
  out->r_dual = dn / (1.0 + dmax(dmax(qi, ai), ci));

  const double xqx = v_dot(x, qx, n);
  const double cx = v_dot(p->c, x, n);
  const double by = v_dot(p->b_ineq, yi, mi) + v_dot(p->b_eq, ye, me);
  out->r_gap = fabs(xqx + cx + by) / (1.0 + dmax(fabs(0.5 * xqx + cx), fabs(0.5 * xqx + by)));
  free(ax_i), free(ax_e), free(qx), free(aty), free(aty_e);
  return 0;
}

/* ---- scaling.hpp ---------------------------------------------------- */
/* Row measures of the stacked [[Q, A'],[A, 0]] in the triplet push order of
 * stacked_triplets (scaling.hpp:30-45) + row_measures (:49-62): primal row j
 * sees Q row j then A' row j (ineq rows before eq rows), dual row i sees A row
 * i. Values live in three working copies (Q, A, A') updated by apply_pass
 * (:66-72) with v *= f[row] * f[col]. kind: 0 max-abs, 1 l2, 2 l1. */
typedef struct {
  int n, m;
  ocsr q, a, at; /* working copies */
} stacked;

static void measures(const stacked* s, int kind, double* meas) {
  for (int j = 0; j < s->n + s->m; ++j) meas[j] = 0.0;
  for (int j = 0; j < s->n; ++j) {
    double acc = 0.0;
    for (int k = s->q.rp[j]; k < s->q.rp[j + 1]; ++k) {
      const double a = fabs(s->q.v[k]);
      acc = kind == 0 ? dmax(acc, a) : kind == 1 ? acc + a * a : acc + a;
    }
    for (int k = s->at.rp[j]; k < s->at.rp[j + 1]; ++k) {
      const double a = fabs(s->at.v[k]);
      acc = kind == 0 ? dmax(acc, a) : kind == 1 ? acc + a * a : acc + a;
    }
    meas[j] = acc;
  }
  for (int i = 0; i < s->m; ++i) {
    double acc = 0.0;
    for (int k = s->a.rp[i]; k < s->a.rp[i + 1]; ++k) {
      const double a = fabs(s->a.v[k]);
      acc = kind == 0 ? dmax(acc, a) : kind == 1 ? acc + a * a : acc + a;
    }
    meas[s->n + i] = acc;
  }
  if (kind == 1)
    for (int j = 0; j < s->n + s->m; ++j) meas[j] = sqrt(meas[j]);
}

static void apply_pass(stacked* s, double* d, const double* meas, double* f) {
  const int N = s->n + s->m;
  for (int j = 0; j < N; ++j) f[j] = meas[j] > 0.0 ? 1.0 / sqrt(meas[j]) : 1.0;
  for (int r = 0; r < s->n; ++r)
    for (int k = s->q.rp[r]; k < s->q.rp[r + 1]; ++k) s->q.v[k] *= f[r] * f[s->q.ci[k]];
  for (int i = 0; i < s->m; ++i)
    for (int k = s->a.rp[i]; k < s->a.rp[i + 1]; ++k) s->a.v[k] *= f[s->n + i] * f[s->a.ci[k]];
  for (int j = 0; j < s->n; ++j)
    for (int k = s->at.rp[j]; k < s->at.rp[j + 1]; ++k) s->at.v[k] *= f[j] * f[s->n + s->at.ci[k]];
  for (int j = 0; j < N; ++j) d[j] *= f[j];
}

static ocsr ocsr_copy(const rapdhg_csr* m) {
  ocsr o;
  o.rows = m->n_rows, o.cols = m->n_cols, o.nnz = m->nnz;
  o.rp = (int32_t*)malloc(sizeof(int32_t) * (o.rows + 1));
  o.ci = (int32_t*)malloc(sizeof(int32_t) * (o.nnz + 1));
  o.v = (double*)malloc(sizeof(double) * (o.nnz + 1));
  memcpy(o.rp, m->row_ptr, sizeof(int32_t) * (o.rows + 1));
  if (o.nnz) memcpy(o.ci, m->col_idx, sizeof(int32_t) * o.nnz);
  if (o.nnz) memcpy(o.v, m->values, sizeof(double) * o.nnz);
  return o;
}

/* ruiz_iters Ruiz passes, then (full) one l2 and one l1 pass:
 * compute_scaling scaling.hpp:97-106 / ruiz_scaling :88-95 */
static void scaling_impl(const rapdhg_qp* p, int ruiz_iters, int full, double* d1, double* d2) {
  stacked s;
  s.n = p->n;
  s.m = p->m_ineq + p->m_eq;
  s.q = ocsr_copy(&p->q);
  s.a = stack_rows(&p->a_ineq, &p->a_eq, p->n);
  rapdhg_csr av = view(&s.a);
  s.at = transpose(&av);
  const int N = s.n + s.m;
  double* d = (double*)malloc(sizeof(double) * (N + 1));
  double* meas = (double*)malloc(sizeof(double) * (N + 1));
  double* f = (double*)malloc(sizeof(double) * (N + 1));
  for (int j = 0; j < N; ++j) d[j] = 1.0;
  for (int it = 0; it < ruiz_iters; ++it) {
    measures(&s, 0, meas);
    apply_pass(&s, d, meas, f);
  }
  if (full) {
    measures(&s, 1, meas);
    apply_pass(&s, d, meas, f);
    measures(&s, 2, meas);
    apply_pass(&s, d, meas, f);
  }
  memcpy(d2, d, sizeof(double) * s.n);
  if (s.m) memcpy(d1, d + s.n, sizeof(double) * s.m);
  free(d), free(meas), free(f);
  ocsr_free(&s.q), ocsr_free(&s.a), ocsr_free(&s.at);
}

int orc_compute_scaling(const rapdhg_qp* p, double* d1, double* d2) {
  scaling_impl(p, 10, 1, d1, d2);
  return 0;
}
int orc_ruiz_scaling(const rapdhg_qp* p, int32_t iters, double* d1, double* d2) {
  scaling_impl(p, iters, 0, d1, d2);
  return 0;
}

/* apply_scaling (scaling.hpp:109-123) via SparseMatrix::scaled
 * (sparse.hpp:147-156): (r[row] * v) * c[col]. */
int orc_apply_scaling(const rapdhg_qp* p, const double* d1, const double* d2, double* qv,
                      double* aiv, double* aev, double* c, double* bi, double* be) {
  for (int r = 0; r < p->n; ++r)
    for (int k = p->q.row_ptr[r]; k < p->q.row_ptr[r + 1]; ++k)
      qv[k] = d2[r] * p->q.values[k] * d2[p->q.col_idx[k]];
  for (int r = 0; r < p->m_ineq; ++r)
    for (int k = p->a_ineq.row_ptr[r]; k < p->a_ineq.row_ptr[r + 1]; ++k)
      aiv[k] = d1[r] * p->a_ineq.values[k] * d2[p->a_ineq.col_idx[k]];
  for (int r = 0; r < p->m_eq; ++r)
    for (int k = p->a_eq.row_ptr[r]; k < p->a_eq.row_ptr[r + 1]; ++k)
      aev[k] = d1[p->m_ineq + r] * p->a_eq.values[k] * d2[p->a_eq.col_idx[k]];
  for (int j = 0; j < p->n; ++j) c[j] = d2[j] * p->c[j];
  for (int i = 0; i < p->m_ineq; ++i) bi[i] = d1[i] * p->b_ineq[i];
  for (int i = 0; i < p->m_eq; ++i) be[i] = d1[p->m_ineq + i] * p->b_eq[i];
  return 0;
}

/* ---- opnorm.hpp ----------------------------------------------------- */
/* std::mt19937_64 (the C++ standard's parameters), restated. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;
static void mt_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}
static uint64_t mt_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
/* opnorm.hpp:20-30 */
static void random_unit(double* v, int n, mt64* g) {
  for (int i = 0; i < n; ++i) v[i] = 2.0 * ((double)(mt_next(g) >> 11) * 0x1.0p-53) - 1.0;
  const double nrm = v_norm2(v, n);
  if (nrm > 0.0) {
    const double s = 1.0 / nrm;
    for (int i = 0; i < n; ++i) v[i] *= s;
  }
}

/* opnorm.hpp:36-61 */
int orc_estimate_op_norm(const rapdhg_csr* m, int32_t max_iters, double tol, uint64_t seed,
                         double* out) {
  if (m->nnz == 0) {
    *out = 0.0;
    return 0;
  }
  mt64 g;
  mt_seed(&g, seed);
  const int n = m->n_cols;
  double* v = (double*)malloc(sizeof(double) * (n + 1));
  double* w = (double*)malloc(sizeof(double) * (n + 1));
  double* mv = (double*)malloc(sizeof(double) * (m->n_rows + 1));
  random_unit(v, n, &g);
  double lambda = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    csr_mul(m, v, mv);
    csr_mul_t(m, mv, w);
    const double ln = v_dot(v, w, n);
    const double nrm = v_norm2(w, n);
    if (nrm == 0.0) {
      random_unit(v, n, &g);
      continue;
    }
    const double s = 1.0 / nrm;
    for (int i = 0; i < n; ++i) v[i] = w[i] * s;
    if (it > 0 && fabs(ln - lambda) <= tol * fabs(ln)) {
      lambda = ln;
      break;
    }
    lambda = ln;
  }
  free(v), free(w), free(mv);
  *out = sqrt(dmax(lambda, 0.0));
  return 0;
}

/* opnorm.hpp:64-87 */
int orc_estimate_op_norm_symmetric(const rapdhg_csr* m, int32_t max_iters, double tol,
                                   uint64_t seed, double* out) {
  if (m->nnz == 0) {
    *out = 0.0;
    return 0;
  }
  mt64 g;
  mt_seed(&g, seed);
  const int n = m->n_cols;
  double* v = (double*)malloc(sizeof(double) * (n + 1));
  double* w = (double*)malloc(sizeof(double) * (n + 1));
  random_unit(v, n, &g);
  double lambda = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    csr_mul(m, v, w);
    const double ln = fabs(v_dot(v, w, n));
    const double nrm = v_norm2(w, n);
    if (nrm == 0.0) {
      random_unit(v, n, &g);
      continue;
    }
    const double s = 1.0 / nrm;
    for (int i = 0; i < n; ++i) v[i] = w[i] * s;
    if (it > 0 && fabs(ln - lambda) <= tol * fabs(ln)) {
      lambda = ln;
      break;
    }
    lambda = ln;
  }
  free(v), free(w);
  *out = lambda;
  return 0;
}

/* ---- solver.hpp ----------------------------------------------------- */
typedef struct {
  ocsr a; /* stacked, scaled */
  rapdhg_csr q;
  const double* c;
  double* b;
  int num_ineq;
  int n, m;
} working;

/* inner_step_inplace (solver.hpp:156-180); w/aw/qx/aty are workspaces.
 * x and x_prev are swapped by pointer as std::swap does. */
static void inner_step(double** x, double** x_prev, double* y, double* x_bar, double* y_bar,
                       int64_t* k, const working* wp, const rapdhg_step_params* sp, double* w,
                       double* aw, double* qx, double* aty) {
  const int n = wp->n, m = wp->m;
  const double ib = 1.0 / sp->beta;
  double* X = *x;
  double* XP = *x_prev;
  for (int j = 0; j < n; ++j) w[j] = sp->theta * (X[j] - XP[j]) + X[j];
  rapdhg_csr av = view(&wp->a);
  csr_mul(&av, w, aw);
  for (int i = 0; i < m; ++i) y[i] += sp->tau * (aw[i] - wp->b[i]);
  for (int i = 0; i < wp->num_ineq; ++i) y[i] = y[i] > 0.0 ? y[i] : 0.0;
  for (int j = 0; j < n; ++j) w[j] = (1.0 - ib) * x_bar[j] + ib * X[j];
  csr_mul(&wp->q, w, qx);
  csr_mul_t(&av, y, aty);
  /* swap(x, x_prev) */
  *x = XP;
  *x_prev = X;
  for (int j = 0; j < n; ++j) XP[j] = X[j] - sp->eta * (qx[j] + wp->c[j] + aty[j]);
  for (int j = 0; j < n; ++j) x_bar[j] = (1.0 - ib) * x_bar[j] + ib * XP[j];
  for (int i = 0; i < m; ++i) y_bar[i] = (1.0 - ib) * y_bar[i] + ib * y[i];
  ++*k;
}

int orc_inner_step(const rapdhg_qp* p, rapdhg_iterate* s, const rapdhg_step_params* sp,
                   int32_t steps) {
  working wp;
  wp.n = p->n;
  wp.m = p->m_ineq + p->m_eq;
  wp.num_ineq = p->m_ineq;
  wp.a = stack_rows(&p->a_ineq, &p->a_eq, p->n);
  wp.q = p->q;
  wp.c = p->c;
  wp.b = (double*)malloc(sizeof(double) * (wp.m + 1));
  if (p->m_ineq) memcpy(wp.b, p->b_ineq, sizeof(double) * p->m_ineq);
  if (p->m_eq) memcpy(wp.b + p->m_ineq, p->b_eq, sizeof(double) * p->m_eq);
  const int n = wp.n, m = wp.m;
  double* w = (double*)malloc(sizeof(double) * (n + 1));
  double* aw = (double*)malloc(sizeof(double) * (m + 1));
  double* qx = (double*)malloc(sizeof(double) * (n + 1));
  double* aty = (double*)malloc(sizeof(double) * (n + 1));
  double* x = (double*)malloc(sizeof(double) * (n + 1));
  double* xp = (double*)malloc(sizeof(double) * (n + 1));
  memcpy(x, s->x, sizeof(double) * n);
  memcpy(xp, s->x_prev, sizeof(double) * n);
  for (int it = 0; it < steps; ++it) inner_step(&x, &xp, s->y, s->x_bar, s->y_bar, &s->k, &wp, sp, w, aw, qx, aty);
  memcpy(s->x, x, sizeof(double) * n);
  memcpy(s->x_prev, xp, sizeof(double) * n);
  free(w), free(aw), free(qx), free(aty), free(x), free(xp), free(wp.b);
  ocsr_free(&wp.a);
  return 0;
}

/* One candidate = unscaled point + residuals (solver.hpp:249-264). */
typedef struct {
  double *x, *y; /* unscaled; y = [y_ineq | y_eq] */
  rapdhg_kkt res;
  int is_average;
} cand_t;

static double relkkt(const rapdhg_kkt* r) { return dmax(dmax(r->r_primal, r->r_dual), r->r_gap); }

/* unscale_point (scaling.hpp:126-133) then rel_kkt on the ORIGINAL problem */
static void eval_point(const rapdhg_qp* orig, const double* xs, const double* ys, const double* d1,
                       const double* d2, int n, int m, double* xu, double* yu, rapdhg_kkt* res) {
  for (int j = 0; j < n; ++j) xu[j] = xs[j] * d2[j];
  for (int i = 0; i < m; ++i) yu[i] = ys[i] * d1[i];
  orc_rel_kkt(orig, xu, yu, yu + orig->m_ineq, res);
}

static void push_log(rapdhg_result* r, int64_t it, const rapdhg_kkt* k, double eta, double omega,
                     int restarted) {
  r->log = (rapdhg_log_record*)realloc(r->log, sizeof(rapdhg_log_record) * (r->n_log + 1));
  rapdhg_log_record L = {it, k->r_primal, k->r_dual, k->r_gap, eta, omega, restarted};
  r->log[r->n_log++] = L;
}

static void push_point(int64_t* count, double** xs, double** ys, const double* x, const double* y,
                       int n, int m) {
  *xs = (double*)realloc(*xs, sizeof(double) * ((*count + 1) * n + 1));
  *ys = (double*)realloc(*ys, sizeof(double) * ((*count + 1) * m + 1));
  memcpy(*xs + *count * n, x, sizeof(double) * n);
  memcpy(*ys + *count * m, y, sizeof(double) * m);
  ++*count;
}

/* solve (solver.hpp:272-471). solve_seconds is not measured (oracle). */
int orc_solve(const rapdhg_qp* orig, const rapdhg_config* cfg, rapdhg_result* out) {
  memset(out, 0, sizeof(*out));
  int rc = validate_qp(orig);
  if (rc) return rc;
  if (cfg->tol <= 0.0) FAIL("tol must be positive");
  if (cfg->restart == RAPDHG_RESTART_FIXED && cfg->restart_length < 1)
    FAIL("fixed restart requires restart_length >= 1");
  if (cfg->check_interval < 1) FAIL("check_interval must be >= 1");
  if (cfg->max_iters < 0) FAIL("max_iters must be >= 0");

  const int n = orig->n, mi = orig->m_ineq, me = orig->m_eq, m = mi + me;
  out->n = n, out->m_ineq = mi, out->m_eq = me;
  double* d1 = (double*)malloc(sizeof(double) * (m + 1));
  double* d2 = (double*)malloc(sizeof(double) * (n + 1));
  if (cfg->scaling) {
    orc_compute_scaling(orig, d1, d2);
  } else {
    for (int i = 0; i < m; ++i) d1[i] = 1.0;
    for (int j = 0; j < n; ++j) d2[j] = 1.0;
  }
  /* scaled problem (apply_scaling) + WorkingProblem */
  double* qv = (double*)malloc(sizeof(double) * (orig->q.nnz + 1));
  double* aiv = (double*)malloc(sizeof(double) * (orig->a_ineq.nnz + 1));
  double* aev = (double*)malloc(sizeof(double) * (orig->a_eq.nnz + 1));
  double* cs = (double*)malloc(sizeof(double) * (n + 1));
  double* bs = (double*)malloc(sizeof(double) * (m + 1));
  if (cfg->scaling) {
    orc_apply_scaling(orig, d1, d2, qv, aiv, aev, cs, bs, bs + mi);
  } else {
    if (orig->q.nnz) memcpy(qv, orig->q.values, sizeof(double) * orig->q.nnz);
    if (orig->a_ineq.nnz) memcpy(aiv, orig->a_ineq.values, sizeof(double) * orig->a_ineq.nnz);
    if (orig->a_eq.nnz) memcpy(aev, orig->a_eq.values, sizeof(double) * orig->a_eq.nnz);
    memcpy(cs, orig->c, sizeof(double) * n);
    if (mi) memcpy(bs, orig->b_ineq, sizeof(double) * mi);
    if (me) memcpy(bs + mi, orig->b_eq, sizeof(double) * me);
  }
  rapdhg_csr qsc = orig->q, aisc = orig->a_ineq, aesc = orig->a_eq;
  qsc.values = qv, aisc.values = aiv, aesc.values = aev;
  working wp;
  wp.n = n, wp.m = m, wp.num_ineq = mi;
  wp.a = stack_rows(&aisc, &aesc, n);
  wp.q = qsc;
  wp.c = cs;
  wp.b = bs;
  rapdhg_csr av = view(&wp.a);

  double norm_q, norm_a;
  orc_estimate_op_norm_symmetric(&wp.q, 5000, 1e-4, cfg->seed, &norm_q);
  orc_estimate_op_norm(&av, 5000, 1e-4, cfg->seed, &norm_a);
  norm_q *= 1.01;
  norm_a *= 1.01;
  out->norm_q = norm_q, out->norm_a = norm_a;

  double* x = (double*)calloc(n + 1, sizeof(double));
  double* xp = (double*)calloc(n + 1, sizeof(double));
  double* xb = (double*)calloc(n + 1, sizeof(double));
  double* y = (double*)calloc(m + 1, sizeof(double));
  double* yb = (double*)calloc(m + 1, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (n + 1));
  double* aw = (double*)malloc(sizeof(double) * (m + 1));
  double* qx = (double*)malloc(sizeof(double) * (n + 1));
  double* aty = (double*)malloc(sizeof(double) * (n + 1));
  double* epx = (double*)calloc(n + 1, sizeof(double));
  double* epy = (double*)calloc(m + 1, sizeof(double));
  /* candidate buffers: cur, avg, best */
  cand_t cur, avg, best;
  cur.x = (double*)malloc(sizeof(double) * (n + 1)), cur.y = (double*)malloc(sizeof(double) * (m + 1));
  avg.x = (double*)malloc(sizeof(double) * (n + 1)), avg.y = (double*)malloc(sizeof(double) * (m + 1));
  best.x = (double*)malloc(sizeof(double) * (n + 1)), best.y = (double*)malloc(sizeof(double) * (m + 1));
  int64_t k = 0;

  double omega = cfg->primal_weight == RAPDHG_PW_ADAPTIVE ? 1.0 : cfg->fixed_primal_weight;
  if (cfg->primal_weight == RAPDHG_PW_ADAPTIVE) orc_primal_weight_init(cs, n, bs, m, &omega);

  long horizon = 1;
  const int theoretical = cfg->step_rule == RAPDHG_STEP_THEORETICAL;
  const int accelerated = cfg->algorithm == RAPDHG_ALG_APDHG;
  if (theoretical && accelerated) {
    if (cfg->restart == RAPDHG_RESTART_FIXED)
      horizon = cfg->restart_length;
    else if (cfg->restart == RAPDHG_RESTART_NONE)
      horizon = cfg->max_iters > 1 ? cfg->max_iters : 1;
    else
      horizon = 4 * cfg->check_interval > 2 ? 4 * cfg->check_interval : 2;
  }
  out->norm_fallback = norm_a <= 0.0;
  double eta = 0.0, prev_eta = 0.0;

  /* evaluate_candidate at t = 0 (solver.hpp:255-264) */
#define EVAL_CAND(chosen)                                                              \
  do {                                                                                 \
    eval_point(orig, x, y, d1, d2, n, m, cur.x, cur.y, &cur.res);                      \
    eval_point(orig, xb, yb, d1, d2, n, m, avg.x, avg.y, &avg.res);                    \
    cur.is_average = 0, avg.is_average = 1;                                            \
    chosen = relkkt(&cur.res) < relkkt(&avg.res) ? &cur : &avg;                        \
  } while (0)
#define COPY_CAND(dst, src)                          \
  do {                                               \
    memcpy((dst).x, (src)->x, sizeof(double) * n);   \
    memcpy((dst).y, (src)->y, sizeof(double) * m);   \
    (dst).res = (src)->res;                          \
    (dst).is_average = (src)->is_average;            \
  } while (0)

  cand_t* cand;
  EVAL_CAND(cand);
  COPY_CAND(best, cand);
  double epoch_start = relkkt(&cand->res);
  double prev_cand = INFINITY;
  push_log(out, 0, &cand->res, 0.0, omega, 0);
  if (cfg->record_restart_points) push_point(&out->n_restart_points, &out->restart_x, &out->restart_y, cand->x, cand->y, n, m);

  int status = -1;
  cand_t* fin = NULL;
  int64_t fin_iters = 0;
  if (relkkt(&cand->res) <= cfg->tol) {
    status = RAPDHG_STATUS_OPTIMAL, fin = cand, fin_iters = 0;
  } else if (norm_q <= 0.0 && norm_a <= 0.0) {
    status = RAPDHG_STATUS_ITERATION_LIMIT, fin = &best, fin_iters = 0;
  }
  rapdhg_step_params sp = {1.0, 1.0, 0.0, 0.0};
  for (int64_t t = 1; status < 0 && t <= cfg->max_iters; ++t) {
    if (theoretical) {
      if (accelerated)
        orc_step_schedule_theoretical((int)(k < horizon - 1 ? k : horizon - 1), (int)horizon, norm_q, norm_a, &sp);
      else
        orc_pdhg_constant_steps(norm_q, norm_a, &sp);
    } else {
      if (accelerated) {
        orc_adaptive_eta((int)k, prev_eta, norm_q, norm_a, omega, &eta);
        sp.beta = 0.5 * (k + 2);
        sp.theta = (double)k / (k + 1);
      } else {
        if (k == 0) orc_adaptive_eta(0, 0.0, norm_q, norm_a, omega, &eta);
        sp.beta = 1.0;
        sp.theta = 1.0;
      }
      prev_eta = eta;
      sp.eta = eta / omega;
      sp.tau = eta * omega;
    }
    inner_step(&x, &xp, y, xb, yb, &k, &wp, &sp, w, aw, qx, aty);
    if (!v_all_finite(x, n) || !v_all_finite(y, m)) {
      status = RAPDHG_STATUS_NUMERICAL_ERROR, fin = &best, fin_iters = t;
      break;
    }
    const int horizon_hit = theoretical && accelerated && cfg->restart != RAPDHG_RESTART_NONE && k >= horizon;
    const int fixed_due = cfg->restart == RAPDHG_RESTART_FIXED && k >= cfg->restart_length;
    const int snapshot_due = cfg->snapshot_interval > 0 && t % cfg->snapshot_interval == 0;
    const int check_due = t % cfg->check_interval == 0 || fixed_due || horizon_hit || snapshot_due || t == cfg->max_iters;
    if (!check_due) continue;
    const double cur_eta = theoretical ? sp.eta : eta;

    EVAL_CAND(cand);
    if (relkkt(&cand->res) < relkkt(&best.res)) COPY_CAND(best, cand);
    if (snapshot_due) {
      out->snapshot_iters = (int64_t*)realloc(out->snapshot_iters, sizeof(int64_t) * (out->n_snapshots + 1));
      out->snapshot_iters[out->n_snapshots] = t;
      int64_t cnt = out->n_snapshots;
      push_point(&cnt, &out->snapshot_x, &out->snapshot_y, avg.x, avg.y, n, m);
      out->n_snapshots = cnt;
    }
    if (relkkt(&cand->res) <= cfg->tol) {
      push_log(out, t, &cand->res, cur_eta, omega, 0);
      status = RAPDHG_STATUS_OPTIMAL, fin = cand, fin_iters = t;
      break;
    }
    if (cfg->time_limit_s <= 0.0) {
      /* elapsed() > time_limit_s (solver.hpp:394): the oracle keeps no clock,
       * so only a limit <= 0 (always exceeded) trips it */
      push_log(out, t, &cand->res, cur_eta, omega, 0);
      status = RAPDHG_STATUS_TIME_LIMIT, fin = &best, fin_iters = t;
      break;
    }
    int do_restart = 0, from_avg = 1;
    if (cfg->restart != RAPDHG_RESTART_NONE) {
      switch (cfg->restart) {
        case RAPDHG_RESTART_FIXED: do_restart = fixed_due; break;
        case RAPDHG_RESTART_HALVING:
          do_restart = orc_restart_decision(cfg->restart, relkkt(&avg.res), prev_cand, epoch_start, k, t, 0);
          break;
        case RAPDHG_RESTART_PDQP:
          do_restart = orc_restart_decision(cfg->restart, relkkt(&cand->res), prev_cand, epoch_start, k, t, 0) || horizon_hit;
          from_avg = cand->is_average;
          break;
        default: break;
      }
      if (horizon_hit) do_restart = 1;
      prev_cand = relkkt(&cand->res);
    }
    push_log(out, t, &cand->res, cur_eta, omega, do_restart);
    if (!do_restart) continue;

    if (horizon_hit && !fixed_due) horizon *= 2;
    if (from_avg) {
      memcpy(x, xb, sizeof(double) * n);
      memcpy(y, yb, sizeof(double) * m);
    }
    memcpy(xp, x, sizeof(double) * n);
    memcpy(xb, x, sizeof(double) * n);
    memcpy(yb, y, sizeof(double) * m);
    k = 0;
    out->restarts += 1;
    prev_eta = 0.0;
    if (cfg->primal_weight == RAPDHG_PW_ADAPTIVE) {
      const double dx = v_dist2(x, epx, n), dy = v_dist2(y, epy, m);
      orc_primal_weight_update(dx, dy, omega, &omega);
    }
    memcpy(epx, x, sizeof(double) * n);
    if (m) memcpy(epy, y, sizeof(double) * m);
    /* rel_kkt of the restart point == the average's residuals when restarting
     * from the average (same unscale + rel_kkt), else the candidate's. */
    epoch_start = (from_avg && !cand->is_average) ? relkkt(&avg.res) : relkkt(&cand->res);
    prev_cand = INFINITY;
    if (cfg->record_restart_points) {
      const cand_t* src = from_avg ? &avg : &cur;
      push_point(&out->n_restart_points, &out->restart_x, &out->restart_y, src->x, src->y, n, m);
    }
  }
  if (status < 0) status = RAPDHG_STATUS_ITERATION_LIMIT, fin = &best, fin_iters = cfg->max_iters;

  out->status = status;
  out->iterations = fin_iters;
  out->residuals = fin->res;
  out->x = (double*)malloc(sizeof(double) * (n + 1));
  out->y_ineq = (double*)malloc(sizeof(double) * (mi + 1));
  out->y_eq = (double*)malloc(sizeof(double) * (me + 1));
  memcpy(out->x, fin->x, sizeof(double) * n);
  if (mi) memcpy(out->y_ineq, fin->y, sizeof(double) * mi);
  if (me) memcpy(out->y_eq, fin->y + mi, sizeof(double) * me);

  free(d1), free(d2), free(qv), free(aiv), free(aev), free(cs), free(bs);
  free(x), free(xp), free(xb), free(y), free(yb), free(w), free(aw), free(qx), free(aty), free(epx), free(epy);
  free(cur.x), free(cur.y), free(avg.x), free(avg.y), free(best.x), free(best.y);
  ocsr_free(&wp.a);
  return 0;
}

void orc_result_free(rapdhg_result* r) {
  free(r->x), free(r->y_ineq), free(r->y_eq), free(r->log), free(r->snapshot_iters);
  free(r->snapshot_x), free(r->snapshot_y), free(r->restart_x), free(r->restart_y);
  memset(r, 0, sizeof(*r));
}
