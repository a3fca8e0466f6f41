// colblock.cu — setup of L2-sized column blocks (see colblock.cuh).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "colblock.cuh"

namespace rb {

namespace {

constexpr int kMaxColBlocks = 16;

struct Cuts {
  int32_t c[kMaxColBlocks + 1];
  int nb;
};

__device__ __forceinline__ int lower_col(const int32_t* ci, int b, int e, int32_t key) {
  while (b < e) {  // first position in [b, e) with ci >= key (rows are column-sorted)
    const int mid = (b + e) >> 1;
    if (ci[mid] < key) b = mid + 1;
    else e = mid;
  }
  return b;
}

// cnt[b * rows + r] = entries of row r in block b
__global__ void block_counts_kernel(const int32_t* rp, const int32_t* ci, int32_t rows, Cuts cuts, int32_t* cnt) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  int lo = rp[r];
  const int e = rp[r + 1];
  for (int b = 0; b < cuts.nb; ++b) {
    const int hi = b + 1 == cuts.nb ? e : lower_col(ci, lo, e, cuts.c[b + 1]);
    cnt[static_cast<int64_t>(b) * rows + r] = hi - lo;
    lo = hi;
  }
}

// copy block b's entries of every row (columns and source positions)
__global__ void block_fill_kernel(const int32_t* rp, const int32_t* ci, int32_t rows, const int32_t* brp,
                                  const int32_t* skip, int32_t* bci, int32_t* bpos) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int src = rp[r] + skip[r];
  const int n = brp[r + 1] - brp[r];
  for (int k = 0; k < n; ++k) {
    bci[brp[r] + k] = ci[src + k];
    bpos[brp[r] + k] = src + k;
  }
}

__global__ void add_kernel(int32_t* acc, const int32_t* x, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) acc[i] += x[i];
}

__global__ void gather_vals_kernel(double* dst, const double* src, const int32_t* pos, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[pos[i]];
}

__global__ void locality_kernel(const int32_t* rp, const int32_t* ci, int32_t rows, int32_t ncols,
                                unsigned long long* count) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  unsigned long long c = 0;
  if (r < rows) {
    const double diag = static_cast<double>(r) / rows * ncols, band = ncols / 16.0;
    for (int p = rp[r]; p < rp[r + 1]; ++p) c += fabs(ci[p] - diag) <= band ? 1ull : 0ull;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);  // integer: exact
}

inline unsigned g1(int64_t n) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, 256)); }

}  // namespace

int colblock_count(int64_t ncols) {
  const char* off = std::getenv("RAPDHG_L2BLOCK");
  if (off && std::string(off) == "0") return 1;
  std::size_t blk = kL2BlockBytes;
  if (const char* kb = std::getenv("RAPDHG_L2BLOCK_KB")) blk = std::max<std::size_t>(1, std::atoll(kb)) << 10;
  const std::size_t bytes = static_cast<std::size_t>(ncols) * sizeof(double);
  const int nb = static_cast<int>((bytes + blk - 1) / blk);
  return nb < 2 ? 1 : std::min(nb, kMaxColBlocks);
}

void build_colblocks(ColBlocks& cb, int nb, const int32_t* rp, const int32_t* ci, int32_t rows, int32_t ncols,
                     cudaStream_t st) {
  cb = ColBlocks{};
  if (nb < 2 || rows <= 0) return;
  cb.nb = nb;
  Cuts cuts{};
  cuts.nb = nb;
  for (int b = 0; b <= nb; ++b) cuts.c[b] = static_cast<int32_t>(static_cast<int64_t>(ncols) * b / nb);
  cb.cut.assign(cuts.c, cuts.c + nb + 1);
  DevBuf<int32_t> cnt(static_cast<std::size_t>(nb) * rows);
  block_counts_kernel<<<g1(rows), 256, 0, st>>>(rp, ci, rows, cuts, cnt.get());
  RB_LAUNCH_CHECK();
  // row pointers per block (exclusive scans), and per-row skips (entries of
  // the earlier blocks) to locate each block's sub-run in the source row
  DevBuf<int32_t> skip(rows);
  skip.zero(st);
  std::size_t temp_bytes = 0;
  RB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, cnt.get(), cnt.get(), rows + 1, st));
  DevBuf<unsigned char> temp(temp_bytes);
  cb.blk.resize(nb);
  cb.pos.resize(nb);
  for (int b = 0; b < nb; ++b) {
    DevCsr& m = cb.blk[b];
    m.rows = rows;
    m.cols = ncols;
    m.rp.alloc(rows + 1);
    // scan rows + 1 counts: the (rows)-th input is the next block's first count
    // or past the end, so scan `rows` items and append the total
    RB_CUDA(cub::DeviceScan::ExclusiveSum(temp.get(), temp_bytes, cnt.get() + static_cast<int64_t>(b) * rows,
                                          m.rp.get(), rows, st));
    int32_t last_rp = 0, last_cnt = 0;
    RB_CUDA(cudaMemcpyAsync(&last_rp, m.rp.get() + rows - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaMemcpyAsync(&last_cnt, cnt.get() + static_cast<int64_t>(b) * rows + rows - 1, sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    const int32_t total = last_rp + last_cnt;
    RB_CUDA(cudaMemcpyAsync(m.rp.get() + rows, &total, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    m.nnz = total;
    m.ci.alloc(total);
    m.v.alloc(total);
    cb.pos[b].alloc(total);
    block_fill_kernel<<<g1(rows), 256, 0, st>>>(rp, ci, rows, m.rp.get(), skip.get(), m.ci.get(), cb.pos[b].get());
    RB_LAUNCH_CHECK();
    add_kernel<<<g1(rows), 256, 0, st>>>(skip.get(), cnt.get() + static_cast<int64_t>(b) * rows, rows);
    RB_LAUNCH_CHECK();
    RB_CUDA(cudaStreamSynchronize(st));  // `total` lives on the host stack
  }
}

double pattern_locality(const int32_t* rp, const int32_t* ci, int32_t rows, int32_t ncols, int64_t nnz,
                        cudaStream_t st) {
  if (rows <= 0 || nnz <= 0) return 0.0;
  DevBuf<unsigned long long> cnt(1);
  cnt.zero(st);
  locality_kernel<<<g1(rows), 256, 0, st>>>(rp, ci, rows, ncols, cnt.get());
  RB_LAUNCH_CHECK();
  unsigned long long h = 0;
  RB_CUDA(cudaMemcpyAsync(&h, cnt.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  return static_cast<double>(h) / static_cast<double>(nnz);
}

void fill_colblock_values(ColBlocks& cb, const double* vals, cudaStream_t st) {
  for (int b = 0; b < cb.nb && cb.active(); ++b) {
    DevCsr& m = cb.blk[b];
    if (m.nnz) gather_vals_kernel<<<g1(m.nnz), 256, 0, st>>>(m.v.get(), vals, cb.pos[b].get(), m.nnz);
    RB_LAUNCH_CHECK();
  }
}

void build_colblocked_dual(ColBlockedDual& d, int nb, const int32_t* rp, const int32_t* ci, int32_t rows,
                           int32_t ncols, const double* vals, bool sell, cudaStream_t st) {
  d = ColBlockedDual{};
  if (nb < 2 || rows <= 0) return;
  d.rows = rows;
  build_colblocks(d.cb, nb, rp, ci, rows, ncols, st);
  fill_colblock_values(d.cb, vals, st);
  d.part.alloc(static_cast<std::size_t>(nb - 1) * rows);
  d.sch.resize(nb);
  DevBuf<int32_t> len;
  for (int b = 0; b < nb; ++b) {
    row_lengths(len, d.cb.blk[b].rp.get(), nullptr, rows, st);
    build_schedule(d.sch[b], len.get(), rows, false, st);
  }
  if (sell) {
    d.sell.resize(nb);
    for (int b = 0; b < nb; ++b) {
      const DevCsr& m = d.cb.blk[b];
      build_sell_plan(d.sell[b], m.rp.get(), m.ci.get(), nullptr, nullptr, rows, st);
      fill_sell_values(d.sell[b], m.v.get(), nullptr, st);
    }
  }
  RB_CUDA(cudaStreamSynchronize(st));
}

void build_colblocked_primal(ColBlockedPrimal& p, int nq, int na, const int32_t* rpq, const int32_t* ciq,
                             const double* qvals, const int32_t* rpat, const int32_t* ciat, const double* atvals,
                             int32_t rows, int32_t n, int32_t m, bool sell, cudaStream_t st) {
  p = ColBlockedPrimal{};
  if ((nq < 2 && na < 2) || rows <= 0) return;
  p.on = true;
  p.rows = rows;
  DevBuf<int32_t> len;
  if (nq >= 2) {
    build_colblocks(p.q, nq, rpq, ciq, rows, n, st);
    fill_colblock_values(p.q, qvals, st);
    p.part_q.alloc(static_cast<std::size_t>(nq - 1) * rows);
    p.sch_q.resize(nq - 1);
    for (int b = 0; b + 1 < nq; ++b) {
      row_lengths(len, p.q.blk[b].rp.get(), nullptr, rows, st);
      build_schedule(p.sch_q[b], len.get(), rows, false, st);
    }
  }
  p.at_all_partial = nq >= 2;
  if (na >= 2) {
    build_colblocks(p.at, na, rpat, ciat, rows, m, st);
    fill_colblock_values(p.at, atvals, st);
  }
  const int npa = p.at_all_partial ? std::max(na, 1) : na - 1;
  if (npa > 0) {
    p.part_at.alloc(static_cast<std::size_t>(npa) * rows);
    p.sch_at.resize(npa);
    for (int b = 0; b < npa; ++b) {
      row_lengths(len, na >= 2 ? p.at.blk[b].rp.get() : rpat, nullptr, rows, st);
      build_schedule(p.sch_at[b], len.get(), rows, false, st);
    }
  }
  if (p.at_all_partial) {
    p.zero_rp.alloc(static_cast<std::size_t>(rows) + 1);
    p.zero_rp.zero(st);
  }
  const int32_t* fin_rpq = nq >= 2 ? p.q.blk[nq - 1].rp.get() : rpq;
  const int32_t* fin_rpat = p.at_all_partial ? p.zero_rp.get() : na >= 2 ? p.at.blk[na - 1].rp.get() : rpat;
  row_lengths(len, fin_rpq, fin_rpat, rows, st);
  build_schedule(p.fin, len.get(), rows, false, st);
  if (sell) {
    p.sell_q.resize(p.sch_q.size());
    for (std::size_t b = 0; b < p.sch_q.size(); ++b) {
      const DevCsr& mq = p.q.blk[b];
      build_sell_plan(p.sell_q[b], mq.rp.get(), mq.ci.get(), nullptr, nullptr, rows, st);
      fill_sell_values(p.sell_q[b], mq.v.get(), nullptr, st);
    }
    p.sell_at.resize(p.sch_at.size());
    for (std::size_t b = 0; b < p.sch_at.size(); ++b) {
      if (na >= 2) {
        const DevCsr& ma = p.at.blk[b];
        build_sell_plan(p.sell_at[b], ma.rp.get(), ma.ci.get(), nullptr, nullptr, rows, st);
        fill_sell_values(p.sell_at[b], ma.v.get(), nullptr, st);
      } else {
        build_sell_plan(p.sell_at[b], rpat, ciat, nullptr, nullptr, rows, st);
        fill_sell_values(p.sell_at[b], atvals, nullptr, st);
      }
    }
    const int32_t* fin_ciq = nq >= 2 ? p.q.blk[nq - 1].ci.get() : ciq;
    const double* fin_vq = nq >= 2 ? p.q.blk[nq - 1].v.get() : qvals;
    const int32_t* fin_ciat = na >= 2 && !p.at_all_partial ? p.at.blk[na - 1].ci.get() : ciat;
    const double* fin_vat = na >= 2 && !p.at_all_partial ? p.at.blk[na - 1].v.get() : atvals;
    build_sell_plan(p.sell_fin, fin_rpq, fin_ciq, fin_rpat, fin_ciat, rows, st);
    fill_sell_values(p.sell_fin, fin_vq, fin_vat, st);
  }
  RB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace rb
