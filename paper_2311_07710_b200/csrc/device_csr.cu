// device_csr.cu — structural CSR setup on the device (see device_csr.cuh).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "device_csr.cuh"

namespace rb {

namespace {

__global__ void offset_rowptr_kernel(int32_t* out, const int32_t* in, int64_t n, int32_t offset) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = in[i] + offset;
}

__global__ void iota_kernel(int32_t* p, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = static_cast<int32_t>(i);
}

// row_of[k]: upper_bound(rp, k) - 1
// row_of[k] = the row of entry k: each non-empty row writes its id at its
// first entry (row_of zeroed first), then an inclusive max-scan carries it
// over the row's other entries (a binary search per entry: 0.39 ms on C4's
// 5.2e7 entries).
__global__ void row_starts_kernel(int32_t* row_of, const int32_t* rp, int32_t rows) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int32_t b = rp[r];
  if (rp[r + 1] > b) row_of[b] = static_cast<int32_t>(r);
}

__global__ void transpose_fill_kernel(int32_t* out_ci, double* out_v, const int32_t* perm,
                                      const int32_t* row_of, const double* v, int64_t nnz) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nnz) return;
  const int32_t src = perm[k];
  out_ci[k] = row_of[src];
  out_v[k] = v[src];
}

// out_rp[c] = lower_bound(sorted_cols, c) for c in [0, cols]
__global__ void rowptr_from_sorted_kernel(int32_t* out_rp, const int32_t* sorted, int64_t nnz,
                                          int32_t cols) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c > cols) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  out_rp[c] = static_cast<int32_t>(lo);
}

__global__ void gather_values_kernel(double* dst, const double* src, const int32_t* perm,
                                     int64_t nnz) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < nnz) dst[k] = src[perm[k]];
}

__global__ void row_lengths_kernel(int32_t* len, const int32_t* rp1, const int32_t* rp2,
                                   int64_t rows) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  len[r] = (rp1[r + 1] - rp1[r]) + (rp2 ? rp2[r + 1] - rp2[r] : 0);
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
  atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}

// One thread per row merges row r of M with row r of M' (both column-sorted).
__global__ void symmetry_gap_kernel(CsrView m, CsrView t, int32_t rows, unsigned long long* gap,
                                    unsigned long long* mabs) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  int i = m.rp[r], ie = m.rp[r + 1], j = t.rp[r], je = t.rp[r + 1];
  double g = 0.0, a = 0.0;
  for (int k = i; k < ie; ++k) a = fmax(a, fabs(m.v[k]));
  while (i < ie || j < je) {
    if (j == je || (i < ie && m.ci[i] < t.ci[j])) {
      g = fmax(g, fabs(m.v[i]));
      ++i;
    } else if (i == ie || t.ci[j] < m.ci[i]) {
      g = fmax(g, fabs(t.v[j]));
      ++j;
    } else {
      g = fmax(g, fabs(m.v[i] - t.v[j]));
      ++i, ++j;
    }
  }
  atomic_max_nonneg(gap, g);  // max is order-free: exact and deterministic
  atomic_max_nonneg(mabs, a);
}

inline unsigned grid_for(int64_t n, int b = 256) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, b)); }

}  // namespace

HostStager::HostStager() {
  const char* e = std::getenv("RAPDHG_STAGE");
  on_ = !(e && e[0] == '0');
  if (const char* t = std::getenv("RAPDHG_STAGE_THREADS")) threads_ = std::min(kMaxThreads, std::max(1, std::atoi(t)));
}

HostStager::~HostStager() {
  if (last_) cudaStreamSynchronize(last_);  // the DMAs out of the buffers are done
  for (int s = 0; s < 2 * kMaxThreads; ++s) {
    if (ev_[s]) cudaEventDestroy(ev_[s]);
    pinned_release(buf_[s], kChunk);
  }
}

namespace {
// Whether [p, p + bytes) is page-locked host memory (cudaHostAlloc'ed or
// registered): then the DMA engines read it directly, at full link speed.
bool host_pinned(const void* p, std::size_t bytes) {
  for (const char* q : {static_cast<const char*>(p), static_cast<const char*>(p) + bytes - 1}) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
      cudaGetLastError();  // clear: a plain pageable pointer on old drivers
      return false;
    }
    if (a.type != cudaMemoryTypeHost) return false;
  }
  return true;
}
}  // namespace

void HostStager::upload(void* dst, const void* src, std::size_t bytes, cudaStream_t st) {
  if (!on_ || bytes < 2 * kChunk || host_pinned(src, bytes)) {
    if (bytes) RB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  last_ = st;
  const std::size_t nch = (bytes + kChunk - 1) / kChunk;
  const int T = static_cast<int>(std::min<std::size_t>(
      nch, std::min<unsigned>(threads_, std::max(1u, std::thread::hardware_concurrency()))));
  for (int s = 0; s < 2 * T; ++s)
    if (!buf_[s]) {
      buf_[s] = pinned_acquire(kChunk);
      RB_CUDA(cudaEventCreateWithFlags(&ev_[s], cudaEventDisableTiming));
    }
  int dev = 0;
  RB_CUDA(cudaGetDevice(&dev));
  std::atomic<int> failed{0};
  // thread t takes chunks t, t + T, ... alternating its two buffers; a buffer
  // is refilled once the event recorded after its previous DMA has passed
  auto work = [&](int t) {
    if (cudaSetDevice(dev) != cudaSuccess) {
      failed = 1;
      return;
    }
    int use = 0;
    for (std::size_t c = t; c < nch && !failed; c += T, ++use) {
      const int s = 2 * t + (use & 1);
      if (used_[s] && cudaEventSynchronize(ev_[s]) != cudaSuccess) failed = 1;  // its last DMA (any call)
      used_[s] = true;
      const std::size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      std::memcpy(buf_[s], static_cast<const char*>(src) + off, len);
      if (cudaMemcpyAsync(static_cast<char*>(dst) + off, buf_[s], len, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaEventRecord(ev_[s], st) != cudaSuccess)
        failed = 1;
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  if (failed) {
    const cudaError_t e = cudaGetLastError();
    RB_CUDA(e != cudaSuccess ? e : cudaErrorUnknown);
  }
}

namespace {
__global__ void csr_check_kernel(const int32_t* rp, const int32_t* ci, int32_t rows, int32_t ncols, int64_t nnz,
                                 unsigned long long* slot) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows; r += warps) {
    const int64_t b = rp[r], e = rp[r + 1];
    unsigned long long key = kCsrOk;
    if (e < b || b < 0 || e > nnz) {
      key = (static_cast<unsigned long long>(r) << 2) | 1u;
    } else {
      int64_t first = INT64_MAX;  // first offending position of the row (this lane's, then the warp's)
      int kind = 0;
      for (int64_t k = b + lane; k < e && k < first; k += 32) {
        const int32_t c = ci[k];
        if (c < 0 || c >= ncols) first = k, kind = 2;
        else if (k > b && c <= ci[k - 1]) first = k, kind = 3;
      }
      for (int off = 16; off > 0; off >>= 1) {
        const int64_t f2 = __shfl_xor_sync(0xffffffffu, first, off);
        const int k2 = __shfl_xor_sync(0xffffffffu, kind, off);
        if (f2 < first) first = f2, kind = k2;
      }
      if (kind) key = (static_cast<unsigned long long>(r) << 2) | static_cast<unsigned>(kind);
    }
    if (lane == 0 && key != kCsrOk) atomicMin(slot, key);
  }
}
}  // namespace

void csr_check_async(const DevCsr& m, unsigned long long* slot, cudaStream_t st) {
  if (m.rows <= 0) return;
  const int64_t blocks = std::min<int64_t>(ceil_div(static_cast<int64_t>(m.rows) * 32, 256), 16 * kSMs);
  csr_check_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(m.rp.get(), m.ci.get(), m.rows, m.cols, m.nnz, slot);
  RB_LAUNCH_CHECK();
}

void upload_csr(DevCsr& d, const rapdhg_csr& h, cudaStream_t st, HostStager* sg) {
  d.rows = h.n_rows;
  d.cols = h.n_cols;
  d.nnz = h.nnz;
  d.rp.alloc(static_cast<std::size_t>(h.n_rows) + 1);
  d.ci.alloc(static_cast<std::size_t>(h.nnz));
  d.v.alloc(static_cast<std::size_t>(h.nnz));
  if (!sg) {
    d.rp.upload(h.row_ptr, static_cast<std::size_t>(h.n_rows) + 1, st);
    d.ci.upload(h.col_idx, static_cast<std::size_t>(h.nnz), st);
    d.v.upload(h.values, static_cast<std::size_t>(h.nnz), st);
    return;
  }
  sg->upload(d.rp.get(), h.row_ptr, sizeof(int32_t) * (static_cast<std::size_t>(h.n_rows) + 1), st);
  sg->upload(d.ci.get(), h.col_idx, sizeof(int32_t) * static_cast<std::size_t>(h.nnz), st);
  sg->upload(d.v.get(), h.values, sizeof(double) * static_cast<std::size_t>(h.nnz), st);
}

void stack_csr(DevCsr& out, const DevCsr& top, const DevCsr& bot, cudaStream_t st) {
  out.rows = top.rows + bot.rows;
  out.cols = top.cols;
  out.nnz = top.nnz + bot.nnz;
  out.rp.alloc(static_cast<std::size_t>(out.rows) + 1);
  out.ci.alloc(static_cast<std::size_t>(out.nnz));
  out.v.alloc(static_cast<std::size_t>(out.nnz));
  RB_CUDA(cudaMemcpyAsync(out.rp.get(), top.rp.get(), sizeof(int32_t) * (top.rows + 1),
                          cudaMemcpyDeviceToDevice, st));
  if (bot.rows > 0) {
    offset_rowptr_kernel<<<grid_for(bot.rows), 256, 0, st>>>(out.rp.get() + top.rows + 1,
                                                             bot.rp.get() + 1, bot.rows,
                                                             static_cast<int32_t>(top.nnz));
    RB_LAUNCH_CHECK();
  }
  if (top.nnz) {
    RB_CUDA(cudaMemcpyAsync(out.ci.get(), top.ci.get(), sizeof(int32_t) * top.nnz, cudaMemcpyDeviceToDevice, st));
    RB_CUDA(cudaMemcpyAsync(out.v.get(), top.v.get(), sizeof(double) * top.nnz, cudaMemcpyDeviceToDevice, st));
  }
  if (bot.nnz) {
    RB_CUDA(cudaMemcpyAsync(out.ci.get() + top.nnz, bot.ci.get(), sizeof(int32_t) * bot.nnz, cudaMemcpyDeviceToDevice, st));
    RB_CUDA(cudaMemcpyAsync(out.v.get() + top.nnz, bot.v.get(), sizeof(double) * bot.nnz, cudaMemcpyDeviceToDevice, st));
  }
}

void expand_rows(DevBuf<int32_t>& row_of, const DevCsr& m, cudaStream_t st) {
  row_of.alloc(static_cast<std::size_t>(m.nnz));
  if (!m.nnz) return;
  if (m.nnz > INT_MAX) throw Error(RAPDHG_E_INTERNAL, "expand_rows: more than 2^31 entries");
  DevBuf<int32_t> starts(static_cast<std::size_t>(m.nnz));
  RB_CUDA(cudaMemsetAsync(starts.get(), 0, sizeof(int32_t) * static_cast<std::size_t>(m.nnz), st));
  row_starts_kernel<<<grid_for(m.rows), 256, 0, st>>>(starts.get(), m.rp.get(), m.rows);
  RB_LAUNCH_CHECK();
  std::size_t tb = 0;
  RB_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, starts.get(), row_of.get(), cub::Max(),
                                         static_cast<int>(m.nnz), st));
  DevBuf<unsigned char> temp(tb);
  RB_CUDA(cub::DeviceScan::InclusiveScan(temp.get(), tb, starts.get(), row_of.get(), cub::Max(),
                                         static_cast<int>(m.nnz), st));
}

void transpose_csr(DevCsr& out, const DevCsr& m, DevBuf<int32_t>* perm_out, cudaStream_t st) {
  out.rows = m.cols;
  out.cols = m.rows;
  out.nnz = m.nnz;
  out.rp.alloc(static_cast<std::size_t>(out.rows) + 1);
  out.ci.alloc(static_cast<std::size_t>(m.nnz));
  out.v.alloc(static_cast<std::size_t>(m.nnz));
  DevBuf<int32_t> keys_sorted(static_cast<std::size_t>(m.nnz));
  DevBuf<int32_t> iota(static_cast<std::size_t>(m.nnz));
  DevBuf<int32_t> perm(static_cast<std::size_t>(m.nnz));
  if (m.nnz) {
    iota_kernel<<<grid_for(m.nnz), 256, 0, st>>>(iota.get(), m.nnz);
    RB_LAUNCH_CHECK();
    int end_bit = 1;
    while (end_bit < 31 && (1LL << end_bit) <= m.cols) ++end_bit;
    std::size_t temp_bytes = 0;
    RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, m.ci.get(), keys_sorted.get(),
                                            iota.get(), perm.get(), static_cast<int>(m.nnz), 0,
                                            end_bit, st));
    DevBuf<unsigned char> temp(temp_bytes);
    RB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), temp_bytes, m.ci.get(), keys_sorted.get(),
                                            iota.get(), perm.get(), static_cast<int>(m.nnz), 0,
                                            end_bit, st));
    DevBuf<int32_t> row_of;
    expand_rows(row_of, m, st);
    transpose_fill_kernel<<<grid_for(m.nnz), 256, 0, st>>>(out.ci.get(), out.v.get(), perm.get(),
                                                           row_of.get(), m.v.get(), m.nnz);
    RB_LAUNCH_CHECK();
    // temporaries are freed at scope exit: make sure the stream is done with them
    RB_CUDA(cudaStreamSynchronize(st));
  }
  rowptr_from_sorted_kernel<<<grid_for(static_cast<int64_t>(out.rows) + 1), 256, 0, st>>>(
      out.rp.get(), keys_sorted.get(), m.nnz, out.rows);
  RB_LAUNCH_CHECK();
  RB_CUDA(cudaStreamSynchronize(st));
  if (perm_out) *perm_out = std::move(perm);
}

void gather_values(double* dst, const double* src, const int32_t* perm, int64_t nnz,
                   cudaStream_t st) {
  if (!nnz) return;
  gather_values_kernel<<<grid_for(nnz), 256, 0, st>>>(dst, src, perm, nnz);
  RB_LAUNCH_CHECK();
}

void row_lengths(DevBuf<int32_t>& len, const int32_t* rp1, const int32_t* rp2, int64_t rows,
                 cudaStream_t st) {
  len.alloc(static_cast<std::size_t>(rows));
  if (rows) {
    row_lengths_kernel<<<grid_for(rows), 256, 0, st>>>(len.get(), rp1, rp2, rows);
    RB_LAUNCH_CHECK();
  }
}

void symmetry_gap(const DevCsr& m, const DevCsr& mt, double* gap, double* max_abs,
                  cudaStream_t st) {
  DevBuf<unsigned long long> acc(2);
  acc.zero(st);
  if (m.rows) {
    symmetry_gap_kernel<<<grid_for(m.rows), 256, 0, st>>>(m.view(), mt.view(), m.rows, acc.get(),
                                                          acc.get() + 1);
    RB_LAUNCH_CHECK();
  }
  unsigned long long h[2];
  RB_CUDA(cudaMemcpyAsync(h, acc.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  std::memcpy(gap, &h[0], sizeof(double));
  std::memcpy(max_abs, &h[1], sizeof(double));
}

}  // namespace rb
