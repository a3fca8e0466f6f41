// gen_device.cu — C5 generator on the device.
//
// The same counter-based algorithm as gen_large in host.cpp (see the comment
// there): A rows sorted and merged by one thread per row; Q's mirrored
// triplets ordered by a stable radix sort of (row, column) keys over the
// triplet indices, then merged per row with the dominant diagonal inserted.
// Every draw is a function of (seed, tag, index) (crng.h) and every sum runs
// in the host's order with unfused operations, so the arrays are
// bit-identical to the host reference (tests/test_gpu_generators.py) while a
// 1e8-nonzero instance takes well under a second instead of ~10 s.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "crng.h"
#include "rapdhg_b200.h"

namespace rb {

namespace {

using namespace crng;

constexpr int kBlocks = 8;  // home blocks of the local pattern

inline unsigned g1(int64_t n) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, 256)); }

// A: row r -> up to 12 merged (column, value) entries in slots [12 r, 12 r + cnt)
__global__ void a_rows_kernel(int32_t m, int32_t n, uint64_t seed, bool local, int32_t* cnt, int32_t* tc,
                              double* tv) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  const int32_t home = static_cast<int32_t>(static_cast<int64_t>(kBlocks) * r / m);
  int32_t c[12], k[12];
  for (int q = 0; q < 12; ++q) c[q] = large_col(seed, kACol, r, q, n, home, kBlocks, local), k[q] = q;
  for (int q = 1; q < 12; ++q)  // insertion sort by (column, draw)
    for (int p = q; p > 0 && (c[p - 1] > c[p] || (c[p - 1] == c[p] && k[p - 1] > k[p])); --p) {
      const int32_t tc0 = c[p - 1], tk0 = k[p - 1];
      c[p - 1] = c[p], k[p - 1] = k[p], c[p] = tc0, k[p] = tk0;
    }
  int w = 0;
  for (int q = 0; q < 12;) {
    double v = normal(seed, kAVal, r, k[q]);
    int e = q + 1;
    for (; e < 12 && c[e] == c[q]; ++e) v = v + normal(seed, kAVal, r, k[e]);
    if (v != 0.0) tc[12 * r + w] = c[q], tv[12 * r + w] = v, ++w;
    q = e;
  }
  cnt[r] = w;
}

__global__ void a_compact_kernel(int32_t m, const int32_t* rp, const int32_t* tc, const double* tv, int32_t* ci,
                                 double* v) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  for (int q = 0; q < rp[r + 1] - rp[r]; ++q) ci[rp[r] + q] = tc[12 * r + q], v[rp[r] + q] = tv[12 * r + q];
}

// b_r = (A x0)_r + slack (sequential, unfused); c_i
__global__ void b_kernel(int32_t m, const int32_t* rp, const int32_t* ci, const double* v, uint64_t seed,
                         double* b) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  double acc = 0.0;
  for (int k = rp[r]; k < rp[r + 1]; ++k) acc = __dadd_rn(acc, __dmul_rn(v[k], normal(seed, kX0, ci[k], 0)));
  b[r] = acc + uniform(seed, kSlack, r, 0);
}
__global__ void c_kernel(int32_t n, uint64_t seed, double* c) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) c[i] = normal(seed, kC, i, 0);
}

// Q: pair p -> triplets 2p = (i, j), 2p + 1 = (j, i); skipped pairs sort last
__global__ void q_pairs_kernel(int64_t pairs, int32_t n, uint64_t seed, bool local, uint64_t* key, int32_t* idx) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= pairs) return;
  const int32_t i = static_cast<int32_t>(below(uniform(seed, kQPair, p, 0), n));
  const int32_t home = static_cast<int32_t>(static_cast<int64_t>(kBlocks) * i / n);
  const int32_t j = large_col(seed, kQPair, p, 1, n, home, kBlocks, local);
  const bool skip = j == i;
  key[2 * p] = skip ? ~0ull : (static_cast<uint64_t>(i) << 32) | static_cast<uint32_t>(j);
  key[2 * p + 1] = skip ? ~0ull : (static_cast<uint64_t>(j) << 32) | static_cast<uint32_t>(i);
  idx[2 * p] = static_cast<int32_t>(2 * p);
  idx[2 * p + 1] = static_cast<int32_t>(2 * p + 1);
}

__global__ void q_row_start_kernel(int32_t n, const uint64_t* key, int64_t nt, int64_t* rs) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i > n) return;
  const uint64_t k = static_cast<uint64_t>(i) << 32;
  int64_t lo = 0, hi = nt;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  rs[i] = lo;
}

// per row: merged off-diagonal entries (+ the diagonal); count or write
template <bool Write>
__global__ void q_rows_kernel(int32_t n, const uint64_t* key, const int32_t* idx, const int64_t* rs, uint64_t seed,
                              int32_t* cnt, const int32_t* rp, int32_t* ci, double* v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t t0 = rs[i], t1 = rs[i + 1];
  double diag = 1e-2;
  if (Write)
    for (int64_t q = t0; q < t1; ++q) diag = diag + fabs(normal(seed, kQVal, idx[q] >> 1, 0));
  int w = 0;
  bool placed = false;
  for (int64_t q = t0; q < t1;) {
    const int32_t col = static_cast<int32_t>(key[q] & 0xffffffffu);
    if (!placed && col > i) {
      if (Write) ci[rp[i] + w] = static_cast<int32_t>(i), v[rp[i] + w] = diag;
      ++w, placed = true;
    }
    double s = normal(seed, kQVal, idx[q] >> 1, 0);
    int64_t e = q + 1;
    for (; e < t1 && key[e] == key[q]; ++e) s = s + normal(seed, kQVal, idx[e] >> 1, 0);
    if (s != 0.0) {
      if (Write) ci[rp[i] + w] = col, v[rp[i] + w] = s;
      ++w;
    }
    q = e;
  }
  if (!placed) {
    if (Write) ci[rp[i] + w] = static_cast<int32_t>(i), v[rp[i] + w] = diag;
    ++w;
  }
  if (!Write) cnt[i] = w;
}

// C4 SVM sample row r -> its merged entries + the t entry, in slots
// [slot r, slot r + cnt) (the host's svm_row, host.cpp)
__global__ void svm_rows_kernel(int32_t ns, int32_t nf, int32_t per_row, uint64_t seed, int32_t* cnt, int32_t* tc,
                                double* tv) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= ns) return;
  const int32_t slot = per_row + 1;
  const double label = r < ns / 2 ? 1.0 : -1.0;
  const double sd = sqrt(1.0 / nf);
  int32_t c[50], k[50];
  for (int32_t q = 0; q < per_row; ++q)
    c[q] = static_cast<int32_t>(below(uniform(seed, kSvmCol, r, q), static_cast<uint64_t>(nf))), k[q] = q;
  for (int32_t q = 1; q < per_row; ++q)
    for (int32_t p = q; p > 0 && (c[p - 1] > c[p] || (c[p - 1] == c[p] && k[p - 1] > k[p])); --p) {
      const int32_t c0 = c[p - 1], k0 = k[p - 1];
      c[p - 1] = c[p], k[p - 1] = k[p], c[p] = c0, k[p] = k0;
    }
  int32_t w = 0;
  int32_t* oc = tc + r * slot;
  double* ov = tv + r * slot;
  for (int32_t q = 0; q < per_row;) {
    double x = __dmul_rn(label, __dadd_rn(label / nf, __dmul_rn(sd, normal(seed, kSvmVal, r, k[q]))));
    int32_t e = q + 1;
    for (; e < per_row && c[e] == c[q]; ++e)
      x = __dadd_rn(x, __dmul_rn(label, __dadd_rn(label / nf, __dmul_rn(sd, normal(seed, kSvmVal, r, k[e])))));
    if (x != 0.0) oc[w] = c[q], ov[w] = x, ++w;
    q = e;
  }
  oc[w] = nf + static_cast<int32_t>(r), ov[w] = -1.0;
  cnt[r] = w + 1;
}

// A = [sample rows (compacted slots); bound rows (ns + r, nf + r) = -1]
__global__ void svm_compact_kernel(int32_t ns, int32_t nf, int32_t slot, const int32_t* rp, const int32_t* tc,
                                   const double* tv, int32_t* ci, double* v) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= ns) return;
  const int32_t b = rp[r], len = rp[r + 1] - b;
  for (int32_t q = 0; q < len; ++q) ci[b + q] = tc[r * slot + q], v[b + q] = tv[r * slot + q];
  const int32_t o = rp[ns] + static_cast<int32_t>(r);
  ci[o] = nf + static_cast<int32_t>(r), v[o] = -1.0;
}

__global__ void iota_kernel(int32_t* p, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = static_cast<int32_t>(i);
}
__global__ void fill_one_kernel(int32_t* p, int32_t v) { *p = v; }

// ---- C2 Lasso (host.cpp gen_lasso) ----------------------------------------
__global__ void lasso_v_kernel(int32_t nf, uint64_t seed, double* v) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= nf) return;
  const double sq = sqrt(static_cast<double>(nf));
  v[j] = uniform(seed, kLassoV, j, 0) < 0.5 ? 0.0 : normal(seed, kLassoV, j, 1) / sq;
}
// draw t = r * per_row + q: key (row, column), payload t
__global__ void lasso_draw_kernel(int32_t ns, int32_t nf, int32_t per_row, uint64_t seed, uint64_t* key,
                                  int32_t* idx) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= static_cast<int64_t>(ns) * per_row) return;
  const int64_t r = t / per_row;
  const uint32_t q = static_cast<uint32_t>(t % per_row);
  const uint32_t c = static_cast<uint32_t>(below(uniform(seed, kLassoCol, r, q), static_cast<uint64_t>(nf)));
  key[t] = (static_cast<uint64_t>(r) << 32) | c;
  idx[t] = static_cast<int32_t>(t);
}
// rows of the key-sorted draws: merged duplicates (count, or write + b_r)
template <bool Write>
__global__ void lasso_rows_kernel(int32_t ns, int32_t per_row, uint64_t seed, const uint64_t* key, const int32_t* idx,
                                  const int32_t* rp, const double* v, int32_t* cnt, int32_t* ci, double* val,
                                  double* b) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= ns) return;
  const int64_t t0 = r * per_row, t1 = t0 + per_row;  // a row's draws stay within its per_row slots
  int w = 0;
  double acc = 0.0;
  for (int64_t a = t0; a < t1;) {
    double x = normal(seed, kLassoVal, r, static_cast<uint32_t>(idx[a] % per_row));
    int64_t e = a + 1;
    for (; e < t1 && key[e] == key[a]; ++e) x = __dadd_rn(x, normal(seed, kLassoVal, r, static_cast<uint32_t>(idx[e] % per_row)));
    if (x != 0.0) {
      const int32_t c = static_cast<int32_t>(key[a] & 0xffffffffu);
      if (Write) {
        ci[rp[r] + w] = c, val[rp[r] + w] = x;
        acc = __dadd_rn(acc, __dmul_rn(x, v[c]));
      }
      ++w;
    }
    a = e;
  }
  if (Write) b[r] = __dadd_rn(acc, normal(seed, kLassoNoise, r, 0));
  else cnt[r] = w;
}
__global__ void row_of_kernel(int32_t rows, const int32_t* rp, int32_t* row_of) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  for (int k = rp[r]; k < rp[r + 1]; ++k) row_of[k] = static_cast<int32_t>(r);
}
// |(A_d' b)_c|: column c's entries in ascending row order (stable transpose
// sort), summed sequentially and unfused
__global__ void lasso_atb_kernel(int32_t nf, const int32_t* cs, int64_t nnz, const int32_t* pos, const double* val,
                                 const int32_t* row_of, const double* b, double* out) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nf) return;
  int64_t lo = 0, hi = nnz;  // first sorted entry of column c
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cs[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  double acc = 0.0;
  for (int64_t k = lo; k < nnz && cs[k] == c; ++k) acc = __dadd_rn(acc, __dmul_rn(val[pos[k]], b[row_of[pos[k]]]));
  out[c] = fabs(acc);
}

// ---- C3 portfolio factor rows (host.cpp gen_portfolio) ----------------------
__global__ void pf_draw_kernel(int32_t na, int32_t k, int32_t per_asset, uint64_t seed, uint64_t* key, int32_t* idx) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= static_cast<int64_t>(na) * per_asset) return;
  const int64_t i = t / per_asset;
  const uint32_t q = static_cast<uint32_t>(t % per_asset);
  const uint64_t f = below(uniform(seed, kPfF, i, q), static_cast<uint64_t>(k));
  key[t] = (f << 32) | static_cast<uint64_t>(i);
  idx[t] = static_cast<int32_t>(t);
}
__global__ void key_row_start_kernel(int32_t rows, const uint64_t* key, int64_t nt, int64_t* rs) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r > rows) return;
  const uint64_t kk = static_cast<uint64_t>(r) << 32;
  int64_t lo = 0, hi = nt;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < kk) lo = mid + 1;
    else hi = mid;
  }
  rs[r] = lo;
}
template <bool Write>
__global__ void pf_rows_kernel(int32_t k, int32_t na, int32_t per_asset, uint64_t seed, const uint64_t* key,
                               const int32_t* idx, const int64_t* rs, const int32_t* rp, int32_t* cnt, int32_t* ci,
                               double* val) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= k) return;
  int w = 0;
  for (int64_t a = rs[f]; a < rs[f + 1];) {
    const int64_t i = idx[a] / per_asset;
    double x = -normal(seed, kPfVal, i, static_cast<uint32_t>(idx[a] % per_asset));
    int64_t e = a + 1;
    for (; e < rs[f + 1] && key[e] == key[a]; ++e)
      x = __dadd_rn(x, -normal(seed, kPfVal, i, static_cast<uint32_t>(idx[e] % per_asset)));
    if (x != 0.0) {
      if (Write) ci[rp[f] + w] = static_cast<int32_t>(i), val[rp[f] + w] = x;
      ++w;
    }
    a = e;
  }
  if (Write) ci[rp[f] + w] = na + static_cast<int32_t>(f), val[rp[f] + w] = 1.0;
  else cnt[f] = w + 1;
}
__global__ void pf_budget_kernel(int32_t na, int32_t base, int32_t* ci, double* val) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na) return;
  ci[base + i] = static_cast<int32_t>(i), val[base + i] = 1.0;
}

// exclusive scan of `cnt` (rows entries) into rp (rows + 1 entries)
void scan_rows(DevBuf<int32_t>& cnt, int64_t rows, DevBuf<int32_t>& rp, cudaStream_t st) {
  rp.alloc(rows + 1);
  rp.zero(st);
  std::size_t temp = 0;
  RB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, cnt.get(), rp.get() + 1, rows, st));
  DevBuf<unsigned char> tmp(temp);
  RB_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), temp, cnt.get(), rp.get() + 1, rows, st));
}

template <class T>
T* to_host(const DevBuf<T>& d, std::size_t n, cudaStream_t st) {
  T* h = static_cast<T*>(std::malloc(sizeof(T) * (n ? n : 1)));
  if (!h) throw Error(RAPDHG_E_INTERNAL, "out of host memory");
  if (n) RB_CUDA(cudaMemcpyAsync(h, d.get(), sizeof(T) * n, cudaMemcpyDeviceToHost, st));
  return h;
}

}  // namespace

// C5 on the device (device 0 of the calling thread's current device); false
// when no device is visible. Arrays are malloc'ed like the host generator's.
bool gen_large_device(double scale, uint64_t seed, bool local, rapdhg_qp_owned* out) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return false;
  }
  const int32_t n = std::max<int32_t>(16, static_cast<int32_t>(std::lround(1e7 * scale)));
  const int32_t m = std::max<int32_t>(8, n / 2);
  OwnedStream own;  // destroyed after the buffers below, which are freed on it
  cudaStream_t st = own.create();
  AllocStreamScope scope(st);
  // A
  DevBuf<int32_t> acnt(m), tc(static_cast<std::size_t>(m) * 12), arp, aci;
  DevBuf<double> tv(static_cast<std::size_t>(m) * 12), av, b(m), c(n);
  a_rows_kernel<<<g1(m), 256, 0, st>>>(m, n, seed, local, acnt.get(), tc.get(), tv.get());
  RB_LAUNCH_CHECK();
  scan_rows(acnt, m, arp, st);
  int32_t annz = 0;
  RB_CUDA(cudaMemcpyAsync(&annz, arp.get() + m, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  aci.alloc(annz), av.alloc(annz);
  a_compact_kernel<<<g1(m), 256, 0, st>>>(m, arp.get(), tc.get(), tv.get(), aci.get(), av.get());
  b_kernel<<<g1(m), 256, 0, st>>>(m, arp.get(), aci.get(), av.get(), seed, b.get());
  c_kernel<<<g1(n), 256, 0, st>>>(n, seed, c.get());
  RB_LAUNCH_CHECK();
  // Q
  const int64_t pairs = static_cast<int64_t>(1.5 * n), nt = 2 * pairs;
  DevBuf<uint64_t> key(nt), key_s(nt);
  DevBuf<int32_t> idx(nt), idx_s(nt), qcnt(n), qrp, qci;
  DevBuf<int64_t> rs(static_cast<std::size_t>(n) + 1);
  DevBuf<double> qv;
  q_pairs_kernel<<<g1(pairs), 256, 0, st>>>(pairs, n, seed, local, key.get(), idx.get());
  RB_LAUNCH_CHECK();
  {
    std::size_t temp = 0;
    RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, key.get(), key_s.get(), idx.get(), idx_s.get(), nt, 0,
                                            64, st));
    DevBuf<unsigned char> tmp(temp);
    RB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), temp, key.get(), key_s.get(), idx.get(), idx_s.get(), nt, 0,
                                            64, st));
  }
  q_row_start_kernel<<<g1(static_cast<int64_t>(n) + 1), 256, 0, st>>>(n, key_s.get(), nt, rs.get());
  q_rows_kernel<false><<<g1(n), 256, 0, st>>>(n, key_s.get(), idx_s.get(), rs.get(), seed, qcnt.get(), nullptr,
                                              nullptr, nullptr);
  RB_LAUNCH_CHECK();
  scan_rows(qcnt, n, qrp, st);
  int32_t qnnz = 0;
  RB_CUDA(cudaMemcpyAsync(&qnnz, qrp.get() + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  qci.alloc(qnnz), qv.alloc(qnnz);
  q_rows_kernel<true><<<g1(n), 256, 0, st>>>(n, key_s.get(), idx_s.get(), rs.get(), seed, nullptr, qrp.get(),
                                             qci.get(), qv.get());
  RB_LAUNCH_CHECK();
  // to the host (malloc'ed, freed by rapdhg_qp_free)
  out->n = n, out->m_ineq = m, out->m_eq = 0;
  out->q.n_rows = n, out->q.n_cols = n, out->q.nnz = qnnz;
  out->q.row_ptr = to_host(qrp, static_cast<std::size_t>(n) + 1, st);
  out->q.col_idx = to_host(qci, qnnz, st);
  out->q.values = to_host(qv, qnnz, st);
  out->a_ineq.n_rows = m, out->a_ineq.n_cols = n, out->a_ineq.nnz = annz;
  out->a_ineq.row_ptr = to_host(arp, static_cast<std::size_t>(m) + 1, st);
  out->a_ineq.col_idx = to_host(aci, annz, st);
  out->a_ineq.values = to_host(av, annz, st);
  out->a_eq.n_rows = 0, out->a_eq.n_cols = n, out->a_eq.nnz = 0;
  out->a_eq.row_ptr = static_cast<int32_t*>(std::calloc(1, sizeof(int32_t)));
  out->a_eq.col_idx = static_cast<int32_t*>(std::malloc(sizeof(int32_t)));
  out->a_eq.values = static_cast<double*>(std::malloc(sizeof(double)));
  out->c = to_host(c, n, st);
  out->b_ineq = to_host(b, m, st);
  out->b_eq = static_cast<double*>(std::malloc(sizeof(double)));
  RB_CUDA(cudaStreamSynchronize(st));
  return true;
}

}  // namespace rb

namespace rb {

// C4 SVM's constraint matrix A on the device (the dominant cost of the
// generator: 5e7 entries of 12-uniform normals); the host builds Q, c, b.
// false when no device is visible.
bool gen_svm_a_device(int32_t ns, int32_t nf, int32_t per_row, uint64_t seed, rapdhg_csr_owned* a) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return false;
  }
  if (per_row > 50) return false;
  OwnedStream own;
  cudaStream_t st = own.create();
  AllocStreamScope scope(st);
  const int32_t slot = per_row + 1, m = 2 * ns;
  DevBuf<int32_t> cnt(ns), tc(static_cast<std::size_t>(ns) * slot), rp, ci;
  DevBuf<double> tv(static_cast<std::size_t>(ns) * slot), v;
  svm_rows_kernel<<<g1(ns), 256, 0, st>>>(ns, nf, per_row, seed, cnt.get(), tc.get(), tv.get());
  RB_LAUNCH_CHECK();
  scan_rows(cnt, ns, rp, st);
  int32_t nnz_top = 0;
  RB_CUDA(cudaMemcpyAsync(&nnz_top, rp.get() + ns, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  const int64_t nnz = static_cast<int64_t>(nnz_top) + ns;
  ci.alloc(nnz), v.alloc(nnz);
  svm_compact_kernel<<<g1(ns), 256, 0, st>>>(ns, nf, slot, rp.get(), tc.get(), tv.get(), ci.get(), v.get());
  RB_LAUNCH_CHECK();
  a->n_rows = m, a->n_cols = nf + ns, a->nnz = nnz;
  a->col_idx = to_host(ci, nnz, st);
  a->values = to_host(v, nnz, st);
  int32_t* top = to_host(rp, static_cast<std::size_t>(ns) + 1, st);
  RB_CUDA(cudaStreamSynchronize(st));
  a->row_ptr = static_cast<int32_t*>(std::realloc(top, sizeof(int32_t) * (static_cast<std::size_t>(m) + 1)));
  if (!a->row_ptr) {
    std::free(top);
    throw Error(RAPDHG_E_INTERNAL, "out of host memory");
  }
  for (int32_t r = 0; r < ns; ++r) a->row_ptr[ns + r + 1] = nnz_top + r + 1;
  return true;
}

}  // namespace rb

namespace rb {

namespace {
bool have_device() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return false;
  }
  return true;
}
void sort_u64_pairs(DevBuf<uint64_t>& key, DevBuf<uint64_t>& key_s, DevBuf<int32_t>& idx, DevBuf<int32_t>& idx_s,
                    int64_t nt, int end_bit, cudaStream_t st) {
  std::size_t temp = 0;
  RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, key.get(), key_s.get(), idx.get(), idx_s.get(), nt, 0,
                                          end_bit, st));
  DevBuf<unsigned char> tmp(temp);
  RB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), temp, key.get(), key_s.get(), idx.get(), idx_s.get(), nt, 0,
                                          end_bit, st));
}
int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}
}  // namespace

// C2 Lasso: A_d (host arrays), b and lambda (host.cpp gen_lasso assembles the rest).
bool gen_lasso_core_device(int32_t nf, int32_t ns, int32_t per_row, uint64_t seed, rapdhg_csr_owned* ad, double* bh,
                           double* lam) {
  if (!have_device()) return false;
  OwnedStream own;
  cudaStream_t st = own.create();
  AllocStreamScope scope(st);
  const int64_t nt = static_cast<int64_t>(ns) * per_row;
  DevBuf<double> v(nf), b(ns), atb(nf), mx(1);
  DevBuf<uint64_t> key(nt), key_s(nt);
  DevBuf<int32_t> idx(nt), idx_s(nt), cnt(ns), rp, ci, row_of;
  DevBuf<double> val;
  lasso_v_kernel<<<g1(nf), 256, 0, st>>>(nf, seed, v.get());
  lasso_draw_kernel<<<g1(nt), 256, 0, st>>>(ns, nf, per_row, seed, key.get(), idx.get());
  RB_LAUNCH_CHECK();
  sort_u64_pairs(key, key_s, idx, idx_s, nt, 32 + bits_for(static_cast<uint64_t>(ns)), st);
  lasso_rows_kernel<false><<<g1(ns), 256, 0, st>>>(ns, per_row, seed, key_s.get(), idx_s.get(), nullptr, nullptr,
                                                   cnt.get(), nullptr, nullptr, nullptr);
  RB_LAUNCH_CHECK();
  scan_rows(cnt, ns, rp, st);
  int32_t nnz = 0;
  RB_CUDA(cudaMemcpyAsync(&nnz, rp.get() + ns, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  ci.alloc(nnz), val.alloc(nnz), row_of.alloc(nnz);
  lasso_rows_kernel<true><<<g1(ns), 256, 0, st>>>(ns, per_row, seed, key_s.get(), idx_s.get(), rp.get(), v.get(),
                                                  nullptr, ci.get(), val.get(), b.get());
  row_of_kernel<<<g1(ns), 256, 0, st>>>(ns, rp.get(), row_of.get());
  RB_LAUNCH_CHECK();
  {  // transpose order: entries by column, stable (ascending position = ascending row)
    DevBuf<int32_t> pos(nnz), pos_s(nnz), cs(nnz);
    iota_kernel<<<g1(nnz), 256, 0, st>>>(pos.get(), nnz);
    std::size_t temp = 0;
    RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, ci.get(), cs.get(), pos.get(), pos_s.get(), nnz, 0,
                                            bits_for(static_cast<uint64_t>(nf)), st));
    DevBuf<unsigned char> tmp(temp);
    RB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), temp, ci.get(), cs.get(), pos.get(), pos_s.get(), nnz, 0,
                                            bits_for(static_cast<uint64_t>(nf)), st));
    lasso_atb_kernel<<<g1(nf), 256, 0, st>>>(nf, cs.get(), nnz, pos_s.get(), val.get(), row_of.get(), b.get(),
                                             atb.get());
    RB_LAUNCH_CHECK();
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceReduce::Max(nullptr, tb, atb.get(), mx.get(), nf, st));
    DevBuf<unsigned char> tmp2(tb);
    RB_CUDA(cub::DeviceReduce::Max(tmp2.get(), tb, atb.get(), mx.get(), nf, st));
  }
  double hm = 0.0;
  RB_CUDA(cudaMemcpyAsync(&hm, mx.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaMemcpyAsync(bh, b.get(), sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
  ad->n_rows = ns, ad->n_cols = nf, ad->nnz = nnz;
  ad->row_ptr = to_host(rp, static_cast<std::size_t>(ns) + 1, st);
  ad->col_idx = to_host(ci, nnz, st);
  ad->values = to_host(val, nnz, st);
  RB_CUDA(cudaStreamSynchronize(st));
  *lam = hm / 5.0;
  return true;
}

// C3 portfolio: the equality block (factor rows + budget row), host arrays.
bool gen_portfolio_eq_device(int32_t na, int32_t k, int32_t per_asset, uint64_t seed, rapdhg_csr_owned* eq) {
  if (!have_device()) return false;
  OwnedStream own;
  cudaStream_t st = own.create();
  AllocStreamScope scope(st);
  const int64_t nt = static_cast<int64_t>(na) * per_asset;
  DevBuf<uint64_t> key(nt), key_s(nt);
  DevBuf<int32_t> idx(nt), idx_s(nt), cnt(static_cast<std::size_t>(k) + 1), rp, ci;
  DevBuf<int64_t> rs(static_cast<std::size_t>(k) + 1);
  DevBuf<double> val;
  pf_draw_kernel<<<g1(nt), 256, 0, st>>>(na, k, per_asset, seed, key.get(), idx.get());
  RB_LAUNCH_CHECK();
  sort_u64_pairs(key, key_s, idx, idx_s, nt, 32 + bits_for(static_cast<uint64_t>(k)), st);
  key_row_start_kernel<<<g1(static_cast<int64_t>(k) + 1), 256, 0, st>>>(k, key_s.get(), nt, rs.get());
  pf_rows_kernel<false><<<g1(k), 256, 0, st>>>(k, na, per_asset, seed, key_s.get(), idx_s.get(), rs.get(), nullptr,
                                               cnt.get(), nullptr, nullptr);
  RB_LAUNCH_CHECK();
  fill_one_kernel<<<1, 1, 0, st>>>(cnt.get() + k, na);  // the budget row
  scan_rows(cnt, static_cast<int64_t>(k) + 1, rp, st);
  int32_t nnz = 0;
  RB_CUDA(cudaMemcpyAsync(&nnz, rp.get() + k + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  ci.alloc(nnz), val.alloc(nnz);
  pf_rows_kernel<true><<<g1(k), 256, 0, st>>>(k, na, per_asset, seed, key_s.get(), idx_s.get(), rs.get(), rp.get(),
                                              nullptr, ci.get(), val.get());
  pf_budget_kernel<<<g1(na), 256, 0, st>>>(na, nnz - na, ci.get(), val.get());
  RB_LAUNCH_CHECK();
  eq->n_rows = k + 1, eq->n_cols = na + k, eq->nnz = nnz;
  eq->row_ptr = to_host(rp, static_cast<std::size_t>(k) + 2, st);
  eq->col_idx = to_host(ci, nnz, st);
  eq->values = to_host(val, nnz, st);
  RB_CUDA(cudaStreamSynchronize(st));
  return true;
}

}  // namespace rb
