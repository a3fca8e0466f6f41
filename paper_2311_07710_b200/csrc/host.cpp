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
#include <thread>
#include <vector>

#include "rapdhg_b200.h"
#include "crng.h"

// rapdhg_last_error() storage lives in capi.cu
void rb_set_error(const char* msg);

namespace rb {
bool gen_large_device(double scale, uint64_t seed, bool local, rapdhg_qp_owned* out);  // gen_device.cu
bool gen_svm_a_device(int32_t ns, int32_t nf, int32_t per_row, uint64_t seed, rapdhg_csr_owned* a);
bool gen_lasso_core_device(int32_t nf, int32_t ns, int32_t per_row, uint64_t seed, rapdhg_csr_owned* ad, double* b,
                           double* lam);
bool gen_portfolio_eq_device(int32_t na, int32_t k, int32_t per_asset, uint64_t seed, rapdhg_csr_owned* eq);
}

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

// The counter-based generators (C4, C5) have device versions (gen_device.cu)
// that build the same arrays; they run for large instances when a device is
// visible (RAPDHG_GEN_DEVICE=1 / 0 forces them on / off).
bool use_device_generator(bool large) {
  const char* e = std::getenv("RAPDHG_GEN_DEVICE");
  return e ? e[0] == '1' : large;
}

// f(r) for r in [0, rows) on up to 16 host threads (contiguous ranges)
template <typename F>
void parallel_rows(int64_t rows, const F& f) {
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>({16, static_cast<int64_t>(std::thread::hardware_concurrency()),
                                                            rows / 4096 + 1}));
  std::vector<std::thread> th;
  for (int64_t t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (int64_t r = rows * t / T; r < rows * (t + 1) / T; ++r) f(r);
    });
  for (auto& x : th) x.join();
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
// variables [x (nf) | y (ns) | t (nf)]. Counter-based (crng.h), so the device
// generator (gen_device.cu) builds bit-identical arrays. Exact algorithm:
//  * v_j = 0 if uniform(kLassoV, j, 0) < 1/2, else normal(kLassoV, j, 1) / sqrt(nf);
//  * A_d row r: `per_row` draws q, column below(uniform(kLassoCol, r, q), nf),
//    value normal(kLassoVal, r, q); sorted by (column, q), duplicate columns
//    summed in that order (a zero sum dropped);
//  * b_r = (sum over the row's entries in column order of a * v_col, unfused)
//    + normal(kLassoNoise, r, 0);
//  * lambda = max_c |sum over rows r ascending of A_d[r, c] * b_r| / 5 (each
//    column summed sequentially in row order, unfused).
struct LassoDims {
  int32_t nf, ns, per_row;
};
LassoDims lasso_dims(double scale) {
  const int32_t nf = std::max<int32_t>(2, static_cast<int32_t>(std::lround(100000 * scale)));
  const int32_t ns = std::max<int32_t>(1, static_cast<int32_t>(std::lround(10000 * scale)));
  return {nf, ns, std::max<int32_t>(1, static_cast<int32_t>(std::lround(0.01 * nf)))};
}

// the structure around A_d, b and lambda (shared by the host and device paths)
void lasso_assemble(const LassoDims& d, const rapdhg_csr_owned& Ad, const std::vector<double>& b, double lam,
                    rapdhg_qp_owned* out) {
  const int32_t nf = d.nf, ns = d.ns, n = 2 * nf + ns;
  // equality block: [A_d, -I, 0] (the -1 is after every A_d column)
  rapdhg_csr_owned& eq = out->a_eq;
  eq.n_rows = ns, eq.n_cols = n, eq.nnz = Ad.nnz + ns;
  eq.row_ptr = xalloc<int32_t>(static_cast<std::size_t>(ns) + 1);
  eq.col_idx = xalloc<int32_t>(static_cast<std::size_t>(eq.nnz));
  eq.values = xalloc<double>(static_cast<std::size_t>(eq.nnz));
  eq.row_ptr[0] = 0;
  for (int32_t r = 0; r < ns; ++r) {
    int64_t w = eq.row_ptr[r];
    for (int32_t k = Ad.row_ptr[r]; k < Ad.row_ptr[r + 1]; ++k, ++w) eq.col_idx[w] = Ad.col_idx[k], eq.values[w] = Ad.values[k];
    eq.col_idx[w] = nf + r, eq.values[w] = -1.0;
    eq.row_ptr[r + 1] = static_cast<int32_t>(w + 1);
  }
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
  out->n = n, out->m_ineq = 2 * nf, out->m_eq = ns;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(std::vector<double>(2 * static_cast<std::size_t>(nf), 0.0));
  out->b_eq = vec_copy(b);
}

void gen_lasso(double scale, uint64_t seed, rapdhg_qp_owned* out) {
  using namespace rb::crng;
  const LassoDims d = lasso_dims(scale);
  const int32_t nf = d.nf, ns = d.ns, per_row = d.per_row;
  {  // A_d, b and lambda on the device for large instances
    rapdhg_csr_owned Ad{};
    std::vector<double> b(ns);
    double lam = 0.0;
    if (use_device_generator(scale >= 0.05) && rb::gen_lasso_core_device(nf, ns, per_row, seed, &Ad, b.data(), &lam)) {
      lasso_assemble(d, Ad, b, lam, out);
      std::free(Ad.row_ptr), std::free(Ad.col_idx), std::free(Ad.values);
      return;
    }
  }
  const double sq = std::sqrt(static_cast<double>(nf));
  std::vector<double> v(nf);
  parallel_rows(nf, [&](int64_t j) {
    v[j] = uniform(seed, kLassoV, j, 0) < 0.5 ? 0.0 : normal(seed, kLassoV, j, 1) / sq;
  });
  // A_d rows: sort each row's draws by (column, draw), merge duplicates
  std::vector<std::vector<int32_t>> rc(ns);
  std::vector<std::vector<double>> rv(ns);
  std::vector<double> b(ns);
  parallel_rows(ns, [&](int64_t r) {
    std::vector<std::pair<int32_t, int32_t>> e(per_row);
    for (int32_t q = 0; q < per_row; ++q)
      e[q] = {static_cast<int32_t>(below(uniform(seed, kLassoCol, r, q), static_cast<uint64_t>(nf))), q};
    std::sort(e.begin(), e.end());
    double acc = 0.0;
    for (int32_t k = 0; k < per_row;) {
      double x = normal(seed, kLassoVal, r, e[k].second);
      int32_t q = k + 1;
      for (; q < per_row && e[q].first == e[k].first; ++q) x = x + normal(seed, kLassoVal, r, e[q].second);
      if (x != 0.0) {
        rc[r].push_back(e[k].first), rv[r].push_back(x);
        acc = acc + x * v[e[k].first];
      }
      k = q;
    }
    b[r] = acc + normal(seed, kLassoNoise, r, 0);
  });
  rapdhg_csr_owned Ad{};
  Ad.n_rows = ns, Ad.n_cols = nf;
  Ad.row_ptr = xalloc<int32_t>(static_cast<std::size_t>(ns) + 1);
  Ad.row_ptr[0] = 0;
  for (int32_t r = 0; r < ns; ++r) Ad.row_ptr[r + 1] = Ad.row_ptr[r] + static_cast<int32_t>(rc[r].size());
  Ad.nnz = Ad.row_ptr[ns];
  Ad.col_idx = xalloc<int32_t>(static_cast<std::size_t>(Ad.nnz));
  Ad.values = xalloc<double>(static_cast<std::size_t>(Ad.nnz));
  for (int32_t r = 0; r < ns; ++r) {
    std::copy(rc[r].begin(), rc[r].end(), Ad.col_idx + Ad.row_ptr[r]);
    std::copy(rv[r].begin(), rv[r].end(), Ad.values + Ad.row_ptr[r]);
  }
  // lambda = ||A_d' b||_inf / 5, each column summed in row order
  std::vector<double> atb(nf, 0.0);
  for (int32_t r = 0; r < ns; ++r)
    for (int32_t k = Ad.row_ptr[r]; k < Ad.row_ptr[r + 1]; ++k) atb[Ad.col_idx[k]] = atb[Ad.col_idx[k]] + Ad.values[k] * b[r];
  double lam = 0.0;
  for (double x : atb) lam = std::max(lam, std::fabs(x));
  lam /= 5.0;
  lasso_assemble(d, Ad, b, lam, out);
  std::free(Ad.row_ptr), std::free(Ad.col_idx), std::free(Ad.values);
}

// ---- C3: Markowitz  min x'Dx + y'y - mu'x  s.t. y - F'x = 0, 1'x = 1, x >= 0
// variables [x (na) | y (k)]. Counter-based (crng.h; device: gen_device.cu):
//  * asset i draws q < per_asset: factor f = below(uniform(kPfF, i, q), k),
//    loading -normal(kPfVal, i, q); factor row f holds its entries in asset
//    order, duplicates (same f, i) summed in draw order (a zero sum dropped),
//    then (f, na + f) = 1;
//  * budget row k: (k, i) = 1; bounds -x_i <= 0;
//  * Q = diag(2 (uniform(kPfD, i, 0) sqrt(k))) on x, 2 on y; c_i = -normal(kPfMu, i, 0).
void gen_portfolio(double scale, uint64_t seed, rapdhg_qp_owned* out) {
  using namespace rb::crng;
  const int32_t na = std::max<int32_t>(4, static_cast<int32_t>(std::lround(1000000 * scale)));
  const int32_t k = std::max<int32_t>(2, static_cast<int32_t>(std::lround(1000 * scale)));
  const int32_t per_asset = std::min<int32_t>(20, k);
  const int32_t n = na + k;
  rapdhg_csr_owned& eq = out->a_eq;
  if (!(use_device_generator(scale >= 0.05) && rb::gen_portfolio_eq_device(na, k, per_asset, seed, &eq))) {
    // factor rows by counting sort of the draws (stable: asset order, then draw order)
    std::vector<int32_t> f(static_cast<std::size_t>(na) * per_asset);
    parallel_rows(na, [&](int64_t i) {
      for (int32_t q = 0; q < per_asset; ++q)
        f[i * per_asset + q] = static_cast<int32_t>(below(uniform(seed, kPfF, i, q), static_cast<uint64_t>(k)));
    });
    std::vector<int64_t> start(static_cast<std::size_t>(k) + 1, 0);
    for (int32_t x : f) ++start[x + 1];
    for (int32_t g = 0; g < k; ++g) start[g + 1] += start[g];
    std::vector<int64_t> slot(start.begin(), start.end() - 1), draw(f.size());
    for (int64_t t = 0; t < static_cast<int64_t>(f.size()); ++t) draw[slot[f[t]]++] = t;  // t = i * per_asset + q
    std::vector<std::vector<int32_t>> rc(k + 1);
    std::vector<std::vector<double>> rv(k + 1);
    parallel_rows(k, [&](int64_t g) {
      for (int64_t a = start[g]; a < start[g + 1];) {
        const int64_t i = draw[a] / per_asset;
        double x = -normal(seed, kPfVal, i, static_cast<uint32_t>(draw[a] % per_asset));
        int64_t b2 = a + 1;
        for (; b2 < start[g + 1] && draw[b2] / per_asset == i; ++b2)
          x = x + -normal(seed, kPfVal, i, static_cast<uint32_t>(draw[b2] % per_asset));
        if (x != 0.0) rc[g].push_back(static_cast<int32_t>(i)), rv[g].push_back(x);
        a = b2;
      }
      rc[g].push_back(na + static_cast<int32_t>(g)), rv[g].push_back(1.0);
    });
    for (int32_t i = 0; i < na; ++i) rc[k].push_back(i), rv[k].push_back(1.0);  // budget row 1'x = 1
    eq.n_rows = k + 1, eq.n_cols = n;
    eq.row_ptr = xalloc<int32_t>(static_cast<std::size_t>(k) + 2);
    eq.row_ptr[0] = 0;
    for (int32_t g = 0; g <= k; ++g) eq.row_ptr[g + 1] = eq.row_ptr[g] + static_cast<int32_t>(rc[g].size());
    eq.nnz = eq.row_ptr[k + 1];
    eq.col_idx = xalloc<int32_t>(static_cast<std::size_t>(eq.nnz));
    eq.values = xalloc<double>(static_cast<std::size_t>(eq.nnz));
    for (int32_t g = 0; g <= k; ++g) {
      std::copy(rc[g].begin(), rc[g].end(), eq.col_idx + eq.row_ptr[g]);
      std::copy(rv[g].begin(), rv[g].end(), eq.values + eq.row_ptr[g]);
    }
  }
  Triplets in(na, n);
  in.reserve(na);
  for (int32_t i = 0; i < na; ++i) in.add(i, i, -1.0);  // -x <= 0
  std::vector<double> qd(n, 2.0), c(n, 0.0);
  const double sk = std::sqrt(static_cast<double>(k));
  parallel_rows(na, [&](int64_t i) {
    qd[i] = 2.0 * (uniform(seed, kPfD, i, 0) * sk);
    c[i] = -normal(seed, kPfMu, i, 0);
  });
  Triplets q(n, n);
  q.reserve(n);
  for (int32_t i = 0; i < n; ++i) q.add(i, i, qd[i]);
  std::vector<double> beq(k + 1, 0.0);
  beq[k] = 1.0;
  build_csr(q, &out->q);
  build_csr(in, &out->a_ineq);
  out->n = n, out->m_ineq = na, out->m_eq = k + 1;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(std::vector<double>(na, 0.0));
  out->b_eq = vec_copy(beq);
}

// ---- C4: SVM  min x'x + lambda 1't  s.t. diag(l) A_s x - t <= -1, -t <= 0
// variables [x (nf) | t (ns)]. Counter-based (crng.h), so the device
// generator (gen_device.cu) and the numpy restatement that feeds the
// reference arm (oracle/synth.py) build bit-identical arrays. Exact algorithm:
//  * sample row r < ns has label l = +1 for r < ns/2 else -1 and `per_row`
//    draws k: column below(uniform(kSvmCol, r, k), nf), value
//    l * (l / nf + sqrt(1/nf) * normal(kSvmVal, r, k)); the draws are sorted
//    by (column, k) and duplicate columns merged by summing in that order
//    (a zero sum is dropped); then the entry (r, nf + r) = -1 (t_r);
//  * row ns + r: (ns + r, nf + r) = -1 (t_r >= 0 as a bound row);
//  * Q = 2 I on x, c = lambda on t, b = -1 on the sample rows, 0 below.
int32_t svm_row(uint64_t seed, int64_t r, int32_t ns, int32_t nf, int32_t per_row, int32_t* ci, double* v) {
  using namespace rb::crng;
  const double label = r < ns / 2 ? 1.0 : -1.0;
  const double sd = std::sqrt(1.0 / nf);
  int32_t c[64], k[64];
  for (int32_t q = 0; q < per_row; ++q)
    c[q] = static_cast<int32_t>(below(uniform(seed, kSvmCol, r, q), static_cast<uint64_t>(nf))), k[q] = q;
  for (int32_t q = 1; q < per_row; ++q)  // insertion sort by (column, draw)
    for (int32_t p = q; p > 0 && (c[p - 1] > c[p] || (c[p - 1] == c[p] && k[p - 1] > k[p])); --p)
      std::swap(c[p - 1], c[p]), std::swap(k[p - 1], k[p]);
  auto val = [&](int32_t kk) { return label * (label / nf + sd * normal(seed, kSvmVal, r, kk)); };
  int32_t w = 0;
  for (int32_t q = 0; q < per_row;) {
    double x = val(k[q]);
    int32_t e = q + 1;
    for (; e < per_row && c[e] == c[q]; ++e) x = x + val(k[e]);
    if (x != 0.0) ci[w] = c[q], v[w] = x, ++w;
    q = e;
  }
  ci[w] = nf + static_cast<int32_t>(r), v[w] = -1.0;
  return w + 1;
}

void gen_svm(double scale, uint64_t seed, rapdhg_qp_owned* out) {
  const int32_t ns = std::max<int32_t>(2, static_cast<int32_t>(std::lround(1000000 * scale)));
  const int32_t nf = std::max<int32_t>(2, static_cast<int32_t>(std::lround(10000 * scale)));
  const int32_t per_row = std::min<int32_t>(50, nf);
  const int32_t n = nf + ns, m = 2 * ns, slot = per_row + 1;
  rapdhg_csr_owned& a = out->a_ineq;
  if (!(use_device_generator(ns >= 20000) && rb::gen_svm_a_device(ns, nf, per_row, seed, &a))) {
  std::vector<int32_t> cnt(ns), tci(static_cast<std::size_t>(ns) * slot);
  std::vector<double> tv(static_cast<std::size_t>(ns) * slot);
  parallel_rows(ns, [&](int64_t r) {
    cnt[r] = svm_row(seed, r, ns, nf, per_row, &tci[r * slot], &tv[r * slot]);
  });
  a.n_rows = m, a.n_cols = n;
  a.row_ptr = xalloc<int32_t>(static_cast<std::size_t>(m) + 1);
  a.row_ptr[0] = 0;
  for (int32_t r = 0; r < ns; ++r) a.row_ptr[r + 1] = a.row_ptr[r] + cnt[r];
  for (int32_t r = 0; r < ns; ++r) a.row_ptr[ns + r + 1] = a.row_ptr[ns + r] + 1;
  a.nnz = a.row_ptr[m];
  a.col_idx = xalloc<int32_t>(static_cast<std::size_t>(a.nnz));
  a.values = xalloc<double>(static_cast<std::size_t>(a.nnz));
  parallel_rows(ns, [&](int64_t r) {
    std::memcpy(a.col_idx + a.row_ptr[r], &tci[r * slot], sizeof(int32_t) * cnt[r]);
    std::memcpy(a.values + a.row_ptr[r], &tv[r * slot], sizeof(double) * cnt[r]);
    a.col_idx[a.row_ptr[ns + r]] = nf + static_cast<int32_t>(r), a.values[a.row_ptr[ns + r]] = -1.0;
  });
  }
  Triplets q(n, n);
  for (int32_t j = 0; j < nf; ++j) q.add(j, j, 2.0);
  std::vector<double> c(n, 0.0);
  for (int32_t r = 0; r < ns; ++r) c[nf + r] = 0.5;  // lambda
  std::vector<double> b(m, 0.0);
  for (int32_t r = 0; r < ns; ++r) b[r] = -1.0;
  build_csr(q, &out->q);
  empty_csr(0, n, &out->a_eq);
  out->n = n, out->m_ineq = m, out->m_eq = 0;
  out->c = vec_copy(c);
  out->b_ineq = vec_copy(b);
  out->b_eq = vec_copy({});
}

// ---- C5: large random QP, uniform (U) or 95%-block-local (L) columns --------
// C5: A m x n with 12 draws per row, Q with 1.5 n mirrored
// off-diagonal pairs and a dominant diagonal, pattern U (uniform columns) or L
// (95% of a row's columns in its home block of n / 8). Counter-based
// (crng.h): every draw is a function of (seed, tag, index), so the device
// generator (gen_device.cu) produces bit-identical arrays; this host version
// is its reference. Exact algorithm (both sides):
//  * A row r: 12 (column, value) draws, sorted by (column, draw), duplicate
//    columns merged by summing their values in draw order;
//  * Q: pair p draws (i, j != i, v); triplets (i, j, v), (j, i, v) sorted by
//    (row, column, triplet index), duplicates summed in that order; Q_ii =
//    1e-2 + the sum of |v| over row i's triplets in that order;
//  * x0_i, c_i ~ normal; b_r = (A x0)_r (sequential, unfused) + uniform slack.
void gen_large(double scale, uint64_t seed, bool local, rapdhg_qp_owned* out) {
  using namespace rb::crng;
  const int32_t n = std::max<int32_t>(16, static_cast<int32_t>(std::lround(1e7 * scale)));
  const int32_t m = std::max<int32_t>(8, n / 2);
  const int32_t blocks = 8;
  // A
  std::vector<int32_t> arp(static_cast<std::size_t>(m) + 1, 0), aci;
  std::vector<double> av;
  aci.reserve(static_cast<std::size_t>(m) * 12);
  av.reserve(static_cast<std::size_t>(m) * 12);
  for (int32_t r = 0; r < m; ++r) {
    const int32_t home = static_cast<int32_t>(static_cast<int64_t>(blocks) * r / m);
    std::pair<int32_t, int32_t> e[12];
    for (int k = 0; k < 12; ++k) e[k] = {large_col(seed, kACol, r, k, n, home, blocks, local), k};
    std::sort(e, e + 12);
    for (int k = 0; k < 12;) {
      double v = normal(seed, kAVal, r, e[k].second);
      int q = k + 1;
      for (; q < 12 && e[q].first == e[k].first; ++q) v = v + normal(seed, kAVal, r, e[q].second);
      if (v != 0.0) aci.push_back(e[k].first), av.push_back(v);
      k = q;
    }
    arp[r + 1] = static_cast<int32_t>(aci.size());
  }
  // Q
  const int64_t pairs = static_cast<int64_t>(1.5 * n);
  std::vector<std::pair<uint64_t, int64_t>> trip;  // ((row << 32) | col, triplet index)
  trip.reserve(static_cast<std::size_t>(2 * pairs));
  for (int64_t p = 0; p < pairs; ++p) {
    const int32_t i = static_cast<int32_t>(below(uniform(seed, kQPair, p, 0), n));
    const int32_t home = static_cast<int32_t>(static_cast<int64_t>(blocks) * i / n);
    const int32_t j = large_col(seed, kQPair, p, 1, n, home, blocks, local);
    if (j == i) continue;
    trip.push_back({(static_cast<uint64_t>(i) << 32) | static_cast<uint32_t>(j), 2 * p});
    trip.push_back({(static_cast<uint64_t>(j) << 32) | static_cast<uint32_t>(i), 2 * p + 1});
  }
  std::stable_sort(trip.begin(), trip.end(),
                   [](const std::pair<uint64_t, int64_t>& x, const std::pair<uint64_t, int64_t>& y) {
                     return x.first < y.first;
                   });
  std::vector<int32_t> qrp(static_cast<std::size_t>(n) + 1, 0), qci;
  std::vector<double> qv;
  qci.reserve(trip.size() + n);
  qv.reserve(trip.size() + n);
  std::size_t t = 0;
  for (int32_t i = 0; i < n; ++i) {
    std::size_t te = t;
    while (te < trip.size() && static_cast<int32_t>(trip[te].first >> 32) == i) ++te;
    double diag = 1e-2;
    for (std::size_t q = t; q < te; ++q) diag = diag + std::fabs(normal(seed, kQVal, trip[q].second >> 1, 0));
    bool placed = false;
    for (std::size_t q = t; q < te;) {
      const int32_t col = static_cast<int32_t>(trip[q].first & 0xffffffffu);
      if (!placed && col > i) qci.push_back(i), qv.push_back(diag), placed = true;
      double v = normal(seed, kQVal, trip[q].second >> 1, 0);
      std::size_t r2 = q + 1;
      for (; r2 < te && trip[r2].first == trip[q].first; ++r2) v = v + normal(seed, kQVal, trip[r2].second >> 1, 0);
      if (v != 0.0) qci.push_back(col), qv.push_back(v);
      q = r2;
    }
    if (!placed) qci.push_back(i), qv.push_back(diag);
    qrp[i + 1] = static_cast<int32_t>(qci.size());
    t = te;
  }
  // c, b
  std::vector<double> c(n), b(m);
  for (int32_t i = 0; i < n; ++i) c[i] = normal(seed, kC, i, 0);
  for (int32_t r = 0; r < m; ++r) {
    double acc = 0.0;
    for (int32_t k = arp[r]; k < arp[r + 1]; ++k) acc = acc + av[k] * normal(seed, kX0, aci[k], 0);
    b[r] = acc + uniform(seed, kSlack, r, 0);
  }
  auto own = [](int32_t rows, int32_t cols, std::vector<int32_t>& rp, std::vector<int32_t>& ci,
                std::vector<double>& v, rapdhg_csr_owned* o) {
    o->n_rows = rows, o->n_cols = cols, o->nnz = static_cast<int64_t>(ci.size());
    o->row_ptr = xalloc<int32_t>(rp.size());
    std::memcpy(o->row_ptr, rp.data(), sizeof(int32_t) * rp.size());
    o->col_idx = xalloc<int32_t>(ci.size());
    if (!ci.empty()) std::memcpy(o->col_idx, ci.data(), sizeof(int32_t) * ci.size());
    o->values = vec_copy(v);
  };
  own(n, n, qrp, qci, qv, &out->q);
  own(m, n, arp, aci, av, &out->a_ineq);
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
  std::free(p->name);
  std::free(p->lower);
  std::free(p->upper);
  if (p->var_names)
    for (int32_t j = 0; j < p->n; ++j) std::free(p->var_names[j]);
  std::free(p->var_names);
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
  v->name = p->name;
  v->var_names = p->var_names;
  v->lower = p->lower;
  v->upper = p->upper;
}

// unscale_point / scale_point (scaling.hpp:126-143): x = D2 x~, y = D1 y~
// and the inverse, elementwise in place.
int rapdhg_unscale_point(const double* d1, const double* d2, int32_t n, int32_t m_ineq, int32_t m_eq, double* x,
                         double* y_ineq, double* y_eq) {
  return hguard([&] {
    if (n < 0 || m_ineq < 0 || m_eq < 0) throw HostError(RAPDHG_E_INVALID_ARGUMENT, "negative dimensions");
    for (int32_t j = 0; j < n; ++j) x[j] *= d2[j];
    for (int32_t i = 0; i < m_ineq; ++i) y_ineq[i] *= d1[i];
    for (int32_t i = 0; i < m_eq; ++i) y_eq[i] *= d1[m_ineq + i];
  });
}

int rapdhg_scale_point(const double* d1, const double* d2, int32_t n, int32_t m_ineq, int32_t m_eq, double* x,
                       double* y_ineq, double* y_eq) {
  return hguard([&] {
    if (n < 0 || m_ineq < 0 || m_eq < 0) throw HostError(RAPDHG_E_INVALID_ARGUMENT, "negative dimensions");
    for (int32_t j = 0; j < n; ++j) x[j] /= d2[j];
    for (int32_t i = 0; i < m_ineq; ++i) y_ineq[i] /= d1[i];
    for (int32_t i = 0; i < m_eq; ++i) y_eq[i] /= d1[m_ineq + i];
  });
}

// primal_weight_init (stepsize.hpp:73-78) with norm2 = sqrt of the
// sequential dot (vec.hpp:14-20)
int rapdhg_primal_weight_init(const double* c, int64_t n, const double* b, int64_t m, double* out) {
  return hguard([&] {
    if (!out || (n && !c) || (m && !b)) throw HostError(RAPDHG_E_INVALID_ARGUMENT, "null argument");
    double sc = 0.0, sb = 0.0;
    for (int64_t j = 0; j < n; ++j) sc += c[j] * c[j];
    for (int64_t i = 0; i < m; ++i) sb += b[i] * b[i];
    const double nc = std::sqrt(sc), nb = std::sqrt(sb);
    *out = (nc > 1e-10 && nb > 1e-10) ? nc / nb : 1.0;
  });
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
      case RAPDHG_GEN_LARGE:
      case RAPDHG_GEN_LARGE_LOCAL: {
        const bool local = kind == RAPDHG_GEN_LARGE_LOCAL;
        if (!(use_device_generator(scale >= 0.02) && rb::gen_large_device(scale, seed, local, out)))
          gen_large(scale, seed, local, out);
        break;
      }
      default: throw HostError(RAPDHG_E_INVALID_ARGUMENT, "unknown generator kind");
    }
  });
}

}  // extern "C"
