// host.cpp — host-side utilities of the C-ABI: canonical CSR construction and
// the synthetic instance generators of SURVEY §8(d) (the reference ships none;
// SPEC.md:417-489 names the classes). Pure C++ (no CUDA), so these also work
// on a CPU-only host for building test inputs.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "rapdhg_b200.h"

// rapdhg_last_error() storage lives in capi.cu
void rb_set_error(const char* msg);

namespace {

struct HostError : std::runtime_error {
  int code;
  HostError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <typename F>
int hguard(F&& f) {
  try {
    f();
    return RAPDHG_OK;
  } catch (const HostError& e) {
    rb_set_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    rb_set_error("out of memory");
    return RAPDHG_E_INTERNAL;
  } catch (const std::exception& e) {
    rb_set_error(e.what());
    return RAPDHG_E_INTERNAL;
  }
}

template <typename T>
T* xalloc(std::size_t n) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (n ? n : 1)));
  if (!p) throw std::bad_alloc();
  return p;
}

// ---- RNG: splitmix64-seeded xoshiro256**, Box-Muller normals --------------
struct Rng {
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    uint64_t z = seed;
    for (auto& v : s) {
      z += 0x9E3779B97F4A7C15ULL;
      uint64_t x = z;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
      v = x ^ (x >> 31);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // [0,1)
  uint64_t below(uint64_t n) { return static_cast<uint64_t>(uniform() * static_cast<double>(n)); }
  bool has_spare = false;
  double spare = 0.0;
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 6.283185307179586 * u2;
    spare = r * std::sin(th);
    has_spare = true;
    return r * std::cos(th);
  }
};

// Triplet accumulation -> canonical CSR: rows by counting sort (stable), each
// row's entries stably sorted by column, duplicates summed in insertion order,
// exact zeros dropped — the contract of SparseMatrix(n_rows, n_cols, triplets)
// (sparse.hpp:31-62).
struct Triplets {
  int32_t rows, cols;
  std::vector<int32_t> r, c;
  std::vector<double> v;
  Triplets(int32_t rows_, int32_t cols_) : rows(rows_), cols(cols_) {}
  void add(int32_t i, int32_t j, double x) {
    r.push_back(i);
    c.push_back(j);
    v.push_back(x);
  }
  void reserve(std::size_t n) {
    r.reserve(n), c.reserve(n), v.reserve(n);
  }
};

void build_csr(int32_t rows, int32_t cols, std::size_t nnz, const int32_t* tr, const int32_t* tc,
               const double* tv, rapdhg_csr_owned* out) {
  if (rows < 0 || cols < 0) throw HostError(RAPDHG_E_INVALID_ARGUMENT, "negative matrix dimension");
  for (std::size_t k = 0; k < nnz; ++k)
    if (tr[k] < 0 || tr[k] >= rows || tc[k] < 0 || tc[k] >= cols)
      throw HostError(RAPDHG_E_OUT_OF_RANGE, "sparse entry index out of range");
  std::vector<int64_t> start(static_cast<std::size_t>(rows) + 1, 0);
  for (std::size_t k = 0; k < nnz; ++k) ++start[tr[k] + 1];
  for (int32_t i = 0; i < rows; ++i) start[i + 1] += start[i];
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  std::vector<int32_t> oc(nnz);
  std::vector<double> ov(nnz);
  for (std::size_t k = 0; k < nnz; ++k) {
    const int64_t p = fill[tr[k]]++;
    oc[p] = tc[k];
    ov[p] = tv[k];
  }
  out->n_rows = rows;
  out->n_cols = cols;
  out->row_ptr = xalloc<int32_t>(static_cast<std::size_t>(rows) + 1);
  out->col_idx = xalloc<int32_t>(nnz);
  out->values = xalloc<double>(nnz);
  std::vector<int32_t> idx;
  int64_t w = 0;
  for (int32_t i = 0; i < rows; ++i) {
    out->row_ptr[i] = static_cast<int32_t>(w);
    const int64_t b = start[i], e = start[i + 1];
    idx.resize(static_cast<std::size_t>(e - b));
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t bb) { return oc[b + a] < oc[b + bb]; });
    for (std::size_t q = 0; q < idx.size();) {
      const int32_t col = oc[b + idx[q]];
      double s = ov[b + idx[q]];
      ++q;
      while (q < idx.size() && oc[b + idx[q]] == col) s += ov[b + idx[q++]];
      if (s != 0.0) {
        out->col_idx[w] = col;
        out->values[w] = s;
        ++w;
      }
    }
  }
  out->row_ptr[rows] = static_cast<int32_t>(w);
  out->nnz = w;
}

void build_csr(Triplets& t, rapdhg_csr_owned* out) {
  build_csr(t.rows, t.cols, t.v.size(), t.r.data(), t.c.data(), t.v.data(), out);
  Triplets empty(0, 0);
  std::swap(t.r, empty.r), std::swap(t.c, empty.c), std::swap(t.v, empty.v);
}

double* vec_copy(const std::vector<double>& v) {
  double* p = xalloc<double>(v.size());
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(double) * v.size());
  return p;
}

// y = M x for an owned CSR (host; generator use only: b = A x0 + s).
std::vector<double> host_mv(const rapdhg_csr_owned& m, const std::vector<double>& x) {
  std::vector<double> y(m.n_rows, 0.0);
  for (int32_t r = 0; r < m.n_rows; ++r) {
    double s = 0.0;
    for (int32_t k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k) s += m.values[k] * x[m.col_idx[k]];
    y[r] = s;
  }
  return y;
}

void empty_csr(int32_t rows, int32_t cols, rapdhg_csr_owned* out) {
  Triplets t(rows, cols);
  build_csr(t, out);
}

// Distinct sorted columns for one row: k samples in [lo, lo+width).
void sample_cols(Rng& g, int32_t k, int32_t lo, int32_t width, std::vector<int32_t>& cols) {
  cols.clear();
  for (int32_t i = 0; i < k; ++i) cols.push_back(lo + static_cast<int32_t>(g.below(width)));
  std::sort(cols.begin(), cols.end());
  cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
}

// ---- C1: random QP (OSQP random QP) ----------------------------
void gen_random_qp(double scale, uint64_t seed, rapdhg_qp_owned* out) {
  Rng g(seed);
  const int32_t n = std::max<int32_t>(2, static_cast<int32_t>(std::lround(1000 * scale)));
  const int32_t m = std::max<int32_t>(1, n / 2);
  const double dens = 0.01;
  // P: n x n sparse Gaussian; Q = P'P + 1e-2 I (sum of row outer products)
  Triplets q(n, n);
  std::vector<int32_t> cols;
  std::vector<double> vals;
  for (int32_t r = 0; r < n; ++r) {
    const int32_t k = std::max<int32_t>(1, static_cast<int32_t>(std::lround(dens * n)));
    sample_cols(g, k, 0, n, cols);
    vals.resize(cols.size());
    for (auto& v : vals) v = g.normal();
    for (std::size_t a = 0; a < cols.size(); ++a)
      for (std::size_t b = 0; b < cols.size(); ++b) q.add(cols[a], cols[b], vals[a] * vals[b]);
  }
  for (int32_t i = 0; i < n; ++i) q.add(i, i, 1e-2);
  Triplets a(m, n);
  for (int32_t r = 0; r < m; ++r) {
    const int32_t k = std::max<int32_t>(1, static_cast<int32_t>(std::lround(dens * n)));
    sample_cols(g, k, 0, n, cols);
    for (int32_t cidx : cols) a.add(r, cidx, g.normal());
  }
  std::vector<double> x0(n), c(n);
  for (auto& v : x0) v = g.normal();
  for (auto& v : c) v = g.normal();
  build_csr(q, &out->q);
  build_csr(a, &out->a_ineq);
  std::vector<double> b = host_mv(out->a_ineq, x0);
  for (auto& v : b) v += g.uniform();
  empty_csr(0, n, &out->a_eq);
  out->n = n, out->m_ineq = m, out->m_eq = 0;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(b);
  out->b_eq = vec_copy({});
}

// ---- C2: Lasso  min y'y + lambda 1't  s.t. A_d x - y = b, x - t <= 0, -x - t <= 0
// variables [x (nf) | y (ns) | t (nf)]
void gen_lasso(double scale, uint64_t seed, rapdhg_qp_owned* out) {
  Rng g(seed);
  const int32_t nf = std::max<int32_t>(2, static_cast<int32_t>(std::lround(100000 * scale)));
  const int32_t ns = std::max<int32_t>(1, static_cast<int32_t>(std::lround(10000 * scale)));
  const int32_t n = 2 * nf + ns;
  const int32_t per_row = std::max<int32_t>(1, static_cast<int32_t>(std::lround(0.01 * nf)));
  std::vector<double> v(nf);
  for (auto& x : v) x = (g.uniform() < 0.5) ? 0.0 : g.normal() / std::sqrt(static_cast<double>(nf));
  Triplets ad(ns, nf);
  ad.reserve(static_cast<std::size_t>(ns) * per_row);
  std::vector<int32_t> cols;
  for (int32_t r = 0; r < ns; ++r) {
    sample_cols(g, per_row, 0, nf, cols);
    for (int32_t c : cols) ad.add(r, c, g.normal());
  }
  rapdhg_csr_owned Ad{};
  build_csr(ad, &Ad);
  std::vector<double> b = host_mv(Ad, v);
  for (auto& x : b) x += g.normal();
  // lambda = ||A_d' b||_inf / 5
  std::vector<double> atb(nf, 0.0);
  for (int32_t r = 0; r < ns; ++r)
    for (int32_t k = Ad.row_ptr[r]; k < Ad.row_ptr[r + 1]; ++k) atb[Ad.col_idx[k]] += Ad.values[k] * b[r];
  double lam = 0.0;
  for (double x : atb) lam = std::max(lam, std::fabs(x));
  lam /= 5.0;
  // equality block: [A_d, -I, 0]
  Triplets eq(ns, n);
  eq.reserve(Ad.nnz + ns);
  for (int32_t r = 0; r < ns; ++r) {
    for (int32_t k = Ad.row_ptr[r]; k < Ad.row_ptr[r + 1]; ++k) eq.add(r, Ad.col_idx[k], Ad.values[k]);
    eq.add(r, nf + r, -1.0);
  }
  std::free(Ad.row_ptr), std::free(Ad.col_idx), std::free(Ad.values);
  // inequality block: x_j - t_j <= 0 ; -x_j - t_j <= 0
  Triplets in(2 * nf, n);
  in.reserve(4 * static_cast<std::size_t>(nf));
  for (int32_t j = 0; j < nf; ++j) {
    in.add(j, j, 1.0), in.add(j, nf + ns + j, -1.0);
    in.add(nf + j, j, -1.0), in.add(nf + j, nf + ns + j, -1.0);
  }
  Triplets q(n, n);
  for (int32_t i = 0; i < ns; ++i) q.add(nf + i, nf + i, 2.0);  // y'y = 1/2 y'(2I)y
  std::vector<double> c(n, 0.0);
  for (int32_t j = 0; j < nf; ++j) c[nf + ns + j] = lam;
  build_csr(q, &out->q);
  build_csr(in, &out->a_ineq);
  build_csr(eq, &out->a_eq);
  out->n = n, out->m_ineq = 2 * nf, out->m_eq = ns;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(std::vector<double>(2 * nf, 0.0));
  out->b_eq = vec_copy(b);
}

// ---- C3: Markowitz  min x'Dx + y'y - mu'x  s.t. y - F'x = 0, 1'x = 1, x >= 0
// variables [x (na) | y (k)]
void gen_portfolio(double scale, uint64_t seed, rapdhg_qp_owned* out) {
  Rng g(seed);
  const int32_t na = std::max<int32_t>(4, static_cast<int32_t>(std::lround(1000000 * scale)));
  const int32_t k = std::max<int32_t>(2, static_cast<int32_t>(std::lround(1000 * scale)));
  const int32_t per_asset = std::min<int32_t>(20, k);
  const int32_t n = na + k;
  Triplets eq(k + 1, n);
  eq.reserve(static_cast<std::size_t>(na) * (per_asset + 1) + k);
  std::vector<int32_t> cols;
  // factor rows: y_f - sum_i F_if x_i = 0, built column-by-column (asset order)
  for (int32_t i = 0; i < na; ++i) {
    sample_cols(g, per_asset, 0, k, cols);
    for (int32_t f : cols) eq.add(f, i, -g.normal());
  }
  for (int32_t f = 0; f < k; ++f) eq.add(f, na + f, 1.0);
  for (int32_t i = 0; i < na; ++i) eq.add(k, i, 1.0);  // budget row 1'x = 1
  Triplets in(na, n);
  in.reserve(na);
  for (int32_t i = 0; i < na; ++i) in.add(i, i, -1.0);  // -x <= 0
  Triplets q(n, n);
  q.reserve(n);
  const double sk = std::sqrt(static_cast<double>(k));
  for (int32_t i = 0; i < na; ++i) q.add(i, i, 2.0 * (g.uniform() * sk));
  for (int32_t f = 0; f < k; ++f) q.add(na + f, na + f, 2.0);
  std::vector<double> c(n, 0.0);
  for (int32_t i = 0; i < na; ++i) c[i] = -g.normal();
  std::vector<double> beq(k + 1, 0.0);
  beq[k] = 1.0;
  build_csr(q, &out->q);
  build_csr(in, &out->a_ineq);
  build_csr(eq, &out->a_eq);
  out->n = n, out->m_ineq = na, out->m_eq = k + 1;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(std::vector<double>(na, 0.0));
  out->b_eq = vec_copy(beq);
}

// ---- C4: SVM  min x'x + lambda 1't  s.t. diag(l) A_s x - t <= -1, -t <= 0
// variables [x (nf) | t (ns)]
void gen_svm(double scale, uint64_t seed, rapdhg_qp_owned* out) {
  Rng g(seed);
  const int32_t ns = std::max<int32_t>(2, static_cast<int32_t>(std::lround(1000000 * scale)));
  const int32_t nf = std::max<int32_t>(2, static_cast<int32_t>(std::lround(10000 * scale)));
  const int32_t per_row = std::min<int32_t>(50, nf);
  const int32_t n = nf + ns;
  const double lam = 0.5;
  const double sd = std::sqrt(1.0 / nf);
  Triplets in(2 * ns, n);
  in.reserve(static_cast<std::size_t>(ns) * (per_row + 2));
  std::vector<int32_t> cols;
  for (int32_t r = 0; r < ns; ++r) {
    const double label = r < ns / 2 ? 1.0 : -1.0;
    sample_cols(g, per_row, 0, nf, cols);
    for (int32_t c : cols) in.add(r, c, label * (label / nf + sd * g.normal()));
    in.add(r, nf + r, -1.0);
  }
  for (int32_t r = 0; r < ns; ++r) in.add(ns + r, nf + r, -1.0);
  Triplets q(n, n);
  for (int32_t j = 0; j < nf; ++j) q.add(j, j, 2.0);
  std::vector<double> c(n, 0.0);
  for (int32_t r = 0; r < ns; ++r) c[nf + r] = lam;
  std::vector<double> b(2 * ns, 0.0);
  for (int32_t r = 0; r < ns; ++r) b[r] = -1.0;
  build_csr(q, &out->q);
  build_csr(in, &out->a_ineq);
  empty_csr(0, n, &out->a_eq);
  out->n = n, out->m_ineq = 2 * ns, out->m_eq = 0;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(b);
  out->b_eq = vec_copy({});
}

// ---- C5: large random QP, uniform (U) or 95%-block-local (L) columns --------
void gen_large(double scale, uint64_t seed, bool local, rapdhg_qp_owned* out) {
  Rng g(seed);
  const int32_t n = std::max<int32_t>(16, static_cast<int32_t>(std::lround(1e7 * scale)));
  const int32_t m = std::max<int32_t>(8, n / 2);
  const int32_t blocks = 8;
  auto col_for = [&](int32_t home_block) -> int32_t {
    if (local && g.uniform() < 0.95) {
      const int32_t lo = static_cast<int32_t>(static_cast<int64_t>(n) * home_block / blocks);
      const int32_t hi = static_cast<int32_t>(static_cast<int64_t>(n) * (home_block + 1) / blocks);
      return lo + static_cast<int32_t>(g.below(hi - lo));
    }
    return static_cast<int32_t>(g.below(n));
  };
  // A: 12 per row
  Triplets a(m, n);
  a.reserve(static_cast<std::size_t>(m) * 12);
  std::vector<int32_t> cols;
  for (int32_t r = 0; r < m; ++r) {
    const int32_t home = static_cast<int32_t>(static_cast<int64_t>(blocks) * r / m);
    cols.clear();
    for (int i = 0; i < 12; ++i) cols.push_back(col_for(home));
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    for (int32_t c : cols) a.add(r, c, g.normal());
  }
  // Q: 1.5 n off-diagonal pairs, mirrored; diagonal 1e-2 + sum |Q_ij|
  const int64_t pairs = static_cast<int64_t>(1.5 * n);
  Triplets q(n, n);
  q.reserve(static_cast<std::size_t>(2 * pairs + n));
  std::vector<double> diag(n, 1e-2);
  for (int64_t p = 0; p < pairs; ++p) {
    const int32_t i = static_cast<int32_t>(g.below(n));
    const int32_t home = static_cast<int32_t>(static_cast<int64_t>(blocks) * i / n);
    int32_t j = col_for(home);
    if (j == i) continue;
    const double v = g.normal();
    q.add(i, j, v);
    q.add(j, i, v);
    diag[i] += std::fabs(v);
    diag[j] += std::fabs(v);
  }
  for (int32_t i = 0; i < n; ++i) q.add(i, i, diag[i]);
  std::vector<double> x0(n), c(n);
  for (auto& v : x0) v = g.normal();
  for (auto& v : c) v = g.normal();
  build_csr(q, &out->q);
  build_csr(a, &out->a_ineq);
  std::vector<double> b = host_mv(out->a_ineq, x0);
  for (auto& v : b) v += g.uniform();
  empty_csr(0, n, &out->a_eq);
  out->n = n, out->m_ineq = m, out->m_eq = 0;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(b);
  out->b_eq = vec_copy({});
}

}  // namespace

extern "C" {

int rapdhg_csr_from_triplets(int32_t n_rows, int32_t n_cols, int64_t nnz, const int32_t* rows,
                             const int32_t* cols, const double* vals, rapdhg_csr_owned* out) {
  return hguard([&] {
    std::memset(out, 0, sizeof(*out));
    build_csr(n_rows, n_cols, static_cast<std::size_t>(nnz), rows, cols, vals, out);
  });
}

void rapdhg_csr_free(rapdhg_csr_owned* m) {
  if (!m) return;
  std::free(m->row_ptr);
  std::free(m->col_idx);
  std::free(m->values);
  std::memset(m, 0, sizeof(*m));
}

void rapdhg_qp_free(rapdhg_qp_owned* p) {
  if (!p) return;
  rapdhg_csr_free(&p->q);
  rapdhg_csr_free(&p->a_ineq);
  rapdhg_csr_free(&p->a_eq);
  std::free(p->c);
  std::free(p->b_ineq);
  std::free(p->b_eq);
  std::memset(p, 0, sizeof(*p));
}

void rapdhg_qp_view(const rapdhg_qp_owned* p, rapdhg_qp* v) {
  auto cv = [](const rapdhg_csr_owned& o) {
    return rapdhg_csr{o.n_rows, o.n_cols, o.nnz, o.row_ptr, o.col_idx, o.values};
  };
  v->n = p->n, v->m_ineq = p->m_ineq, v->m_eq = p->m_eq;
  v->q = cv(p->q), v->a_ineq = cv(p->a_ineq), v->a_eq = cv(p->a_eq);
  v->c = p->c, v->b_ineq = p->b_ineq, v->b_eq = p->b_eq;
  v->obj_offset = p->obj_offset;
}

int rapdhg_generate(int32_t kind, double scale, uint64_t seed, rapdhg_qp_owned* out) {
  return hguard([&] {
    if (!out) throw HostError(RAPDHG_E_INVALID_ARGUMENT, "null out");
    std::memset(out, 0, sizeof(*out));
    if (!(scale > 0.0)) throw HostError(RAPDHG_E_INVALID_ARGUMENT, "scale must be positive");
    switch (kind) {
      case RAPDHG_GEN_RANDOM_QP: gen_random_qp(scale, seed, out); break;
      case RAPDHG_GEN_LASSO: gen_lasso(scale, seed, out); break;
      case RAPDHG_GEN_PORTFOLIO: gen_portfolio(scale, seed, out); break;
      case RAPDHG_GEN_SVM: gen_svm(scale, seed, out); break;
      case RAPDHG_GEN_LARGE: gen_large(scale, seed, false, out); break;
      case RAPDHG_GEN_LARGE_LOCAL: gen_large(scale, seed, true, out); break;
      default: throw HostError(RAPDHG_E_INVALID_ARGUMENT, "unknown generator kind");
    }
  });
}

}  // extern "C"
