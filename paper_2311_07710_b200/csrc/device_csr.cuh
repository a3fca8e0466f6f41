// device_csr.cuh — CSR matrices resident in HBM and their structural setup
// (upload, row stacking, transpose). Structural work is integer-only and
// exact; it replaces the reference's SparseMatrix construction / transpose /
// WorkingProblem::from (sparse.hpp:31-62,102-108; solver.hpp:101-112).
#pragma once

#include <cstdint>

#include "common.cuh"
#include "ops.cuh"

namespace rb {

struct DevCsr {
  int32_t rows = 0, cols = 0;
  int64_t nnz = 0;
  DevBuf<int32_t> rp, ci;
  DevBuf<double> v;
  CsrView view() const { return CsrView{rp.get(), ci.get(), v.get()}; }
  CsrView view(const double* vals) const { return CsrView{rp.get(), ci.get(), vals}; }
};

// Host -> device copies of large pageable arrays through pinned staging: up
// to 8 host threads (RAPDHG_STAGE_THREADS) copy 8 MB chunks into per-thread double buffers (pinned,
// cached across solves, 128 MB at most) and enqueue each chunk's DMA as soon
// as it is copied, so the memcpys run in parallel and overlap the transfers
// (the driver's own pageable path is one serial bounce buffer, ~11 GB/s).
// Copies are complete when the stream is; the destructor waits for them
// before the buffers go back to the cache. RAPDHG_STAGE=0: plain copies.
// Arrays already page-locked (cudaHostAlloc / cudaHostRegister, e.g. torch's
// pin_memory) skip the staging: one direct DMA each.
class HostStager {
 public:
  HostStager();
  ~HostStager();
  HostStager(const HostStager&) = delete;
  HostStager& operator=(const HostStager&) = delete;
  void upload(void* dst, const void* src, std::size_t bytes, cudaStream_t st);

 private:
  static constexpr int kMaxThreads = 16;
  static constexpr std::size_t kChunk = std::size_t{8} << 20;
  bool on_ = true;
  int threads_ = 8;  // RAPDHG_STAGE_THREADS
  cudaStream_t last_ = nullptr;
  void* buf_[2 * kMaxThreads] = {};
  cudaEvent_t ev_[2 * kMaxThreads] = {};
  bool used_[2 * kMaxThreads] = {};  // a DMA out of the buffer was enqueued (ev_ recorded after it)
};

// Host CSR (validated for shape/index ranges by the caller) -> device.
void upload_csr(DevCsr& d, const rapdhg_csr& h, cudaStream_t st, HostStager* sg = nullptr);

// Structural check of an uploaded CSR (the per-row part of
// QuadraticProgram::validate, problem.hpp:40-46): *slot (preset to ~0) gets
// min over bad rows of (row << 2 | kind), kind 1 = row_ptr not monotone (or
// outside [0, nnz]), 2 = column out of range, 3 = columns not strictly
// increasing — within a row the first offending entry decides, as in a
// sequential scan. One warp per row.
constexpr unsigned long long kCsrOk = ~0ull;
void csr_check_async(const DevCsr& m, unsigned long long* slot, cudaStream_t st);

// [top; bottom] row stacking of two CSRs with equal column counts.
void stack_csr(DevCsr& out, const DevCsr& top, const DevCsr& bottom, cudaStream_t st);

// out = transpose(m) with entries of each output row in increasing source-row
// order (a stable sort by column). If perm != nullptr it receives, for every
// output position, the source position (so transposed VALUES of a matrix with
// the same pattern can be produced by a gather).
void transpose_csr(DevCsr& out, const DevCsr& m, DevBuf<int32_t>* perm, cudaStream_t st);

// dst[k] = src[perm[k]]
void gather_values(double* dst, const double* src, const int32_t* perm, int64_t nnz,
                   cudaStream_t st);

// Per-row lengths: len[r] = (rp1[r+1]-rp1[r]) + (rp2 ? rp2[r+1]-rp2[r] : 0).
void row_lengths(DevBuf<int32_t>& len, const int32_t* rp1, const int32_t* rp2, int64_t rows,
                 cudaStream_t st);

// Expanded row index of every nnz (row_of[k] = r for rp[r] <= k < rp[r+1]).
void expand_rows(DevBuf<int32_t>& row_of, const DevCsr& m, cudaStream_t st);

// max |M_ij - M_ji| over the union of patterns (sparse.hpp:119-138) and
// max |M_ij| (sparse.hpp:140-144); needs the transpose of M.
void symmetry_gap(const DevCsr& m, const DevCsr& mt, double* gap, double* max_abs,
                  cudaStream_t st);

}  // namespace rb
