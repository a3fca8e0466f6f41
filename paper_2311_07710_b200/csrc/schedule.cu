// schedule.cu — builds the length-binned row schedule consumed by
// rowwise_kernel (rowwise.cuh). Built once per matrix pattern at setup, on
// the device: bin ids from row lengths, a stable radix sort of row indices by
// bin (rows stay in increasing order inside a bin, so epilogue stores stay
// mostly contiguous), and a host-side segment table for the few rows longer
// than kSplitLen.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "rowwise.cuh"

namespace rb {

namespace {

// Counts per bin: a shared-memory histogram per block, then one global
// atomic per (block, bin) — a global atomic per row serialised 2e6 rows on
// the 8 counters (C4: 0.78 ms per schedule). Integer counts: exact.
__global__ void bin_kernel(int32_t* bin, int32_t* idx, const int32_t* len, const int32_t* subset,
                           int64_t rows, int* counts, int epl, int block_min) {
  __shared__ int h[kNumBins];
  if (threadIdx.x < kNumBins) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < rows) {
    const int32_t r = subset ? subset[k] : static_cast<int32_t>(k);
    const int b = bin_of_len(len[r], epl, block_min);
    bin[k] = b;
    idx[k] = r;
    atomicAdd(&h[b], 1);
  }
  __syncthreads();
  if (threadIdx.x < kNumBins && h[threadIdx.x]) atomicAdd(&counts[threadIdx.x], h[threadIdx.x]);
}

constexpr int kWinBucket = 128;  // histogram granularity (columns)

__global__ void col_hist_kernel(const int32_t* cols, int64_t nnz, int* hist) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < nnz) atomicAdd(&hist[cols[k] / kWinBucket], 1);  // integer counts: exact
}

struct WinChoice {
  Window w;
  int64_t covered = 0;
};

WinChoice best_window(const int32_t* cols, int64_t nnz, int32_t ncols, cudaStream_t st) {
  WinChoice best;
  if (nnz <= 0 || ncols <= 0) return best;
  const int nb = static_cast<int>(ceil_div(ncols, kWinBucket));
  DevBuf<int> hist(nb);
  hist.zero(st);
  col_hist_kernel<<<static_cast<unsigned>(ceil_div(nnz, 256)), 256, 0, st>>>(cols, nnz, hist.get());
  RB_LAUNCH_CHECK();
  std::vector<int> h(nb);
  RB_CUDA(cudaMemcpyAsync(h.data(), hist.get(), sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  const int wb = std::min(nb, kWinMax / kWinBucket);
  int64_t sum = 0;
  for (int b = 0; b < wb; ++b) sum += h[b];
  int64_t best_sum = sum;
  int best_b = 0;
  for (int b = wb; b < nb; ++b) {  // sliding window of wb buckets
    sum += h[b] - h[b - wb];
    if (sum > best_sum) best_sum = sum, best_b = b - wb + 1;
  }
  int lo_b = best_b, hi_b = best_b + wb;  // trim empty buckets at both ends
  while (lo_b < hi_b && h[lo_b] == 0) ++lo_b;
  while (hi_b > lo_b && h[hi_b - 1] == 0) --hi_b;
  if (lo_b >= hi_b) return best;
  best.w.lo = lo_b * kWinBucket;
  best.w.len = std::min(hi_b * kWinBucket, ncols) - best.w.lo;
  best.covered = best_sum;
  return best;
}

}  // namespace

int resident_ctas(const void* kernel, int smem_bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(kernel, smem_bytes);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (smem_bytes > 48 * 1024)
    RB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  int n = 0;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kBlock, smem_bytes));
  if (n < 1) n = 1;
  cache.emplace(key, n);
  return n;
}

void choose_windows(Schedule& sch, const int32_t* cols1, int64_t nnz1, int32_t ncols1,
                    const int32_t* cols2, int64_t nnz2, int32_t ncols2, cudaStream_t st) {
  sch.view.win[0] = sch.view.win[1] = Window{};
  const char* env = std::getenv("RAPDHG_WINDOW");
  // Measured on B200 (C2/C3/C4): a window large enough to matter costs more in
  // occupancy (2 CTAs/SM at 80-96 KB) than it saves in L1TEX wavefronts, so
  // windows are opt-in (RAPDHG_WINDOW=auto|force) until a variant wins.
  const std::string mode = env ? env : "off";
  if (mode == "off") return;
  WinChoice c[2] = {best_window(cols1, nnz1, ncols1, st), best_window(cols2, nnz2, ncols2, st)};
  const int64_t nnz[2] = {nnz1, nnz2};
  // staging costs len doubles per resident CTA (~2 per SM at a full window)
  const int64_t grid = std::min<int64_t>(sch.view.total_blocks, 2 * kSMs);
  bool keep[2];
  for (int k = 0; k < 2; ++k) {
    keep[k] = c[k].w.len > 0 &&
              (mode == "force" ||
               (c[k].covered * 4 >= nnz[k] && c[k].covered >= 2 * static_cast<int64_t>(c[k].w.len) * grid));
  }
  if (keep[0] && keep[1] && c[0].w.len + c[1].w.len > kWinMax) {
    if (c[0].covered >= c[1].covered) keep[1] = false;
    else keep[0] = false;
  }
  for (int k = 0; k < 2; ++k)
    if (keep[k]) sch.view.win[k] = c[k].w;
}

SchedParams SchedParams::from_env() {
  SchedParams p;
  if (const char* e = std::getenv("RAPDHG_EPL")) p.epl = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("RAPDHG_BLOCK_MIN")) p.block_min = std::max(32 * p.epl, std::atoi(e));
  if (p.block_min > kSplitLen) p.block_min = kSplitLen;
  return p;
}

void build_schedule(Schedule& sch, const int32_t* d_len, int64_t rows, bool strict,
                    cudaStream_t st, const int32_t* d_subset) {
  if (strict && d_subset) invalid("strict schedules cover all rows");
  sch.rows = rows;
  SchedView& v = sch.view;
  v = SchedView{};
  for (int b = 0; b < kNumBins; ++b) sch.bin_rows[b] = 0;
  if (strict) {
    // one thread per row in natural order: the reference's sequential sums
    v.perm = nullptr;
    const int32_t blocks = static_cast<int32_t>(ceil_div(rows, kBlock));
    v.bins[0] = {0, static_cast<int32_t>(rows), 0, blocks};
    for (int b = 1; b < kNumBins; ++b) v.bins[b] = {static_cast<int32_t>(rows), static_cast<int32_t>(rows), blocks, blocks};
    v.total_blocks = blocks;
    sch.bin_rows[0] = static_cast<int32_t>(rows);
    return;
  }
  const SchedParams sp = SchedParams::from_env();
  DevBuf<int32_t> bins(rows), idx(rows), bins_sorted(rows);
  DevBuf<int> counts(kNumBins);
  counts.zero(st);
  sch.perm.alloc(rows);
  if (rows) {
    bin_kernel<<<static_cast<unsigned>(ceil_div(rows, 256)), 256, 0, st>>>(
        bins.get(), idx.get(), d_len, d_subset, rows, counts.get(), sp.epl, sp.block_min);
    RB_LAUNCH_CHECK();
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, bins.get(), bins_sorted.get(), idx.get(),
                                            sch.perm.get(), static_cast<int>(rows), 0, 3, st));
    DevBuf<unsigned char> temp(tb);
    RB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, bins.get(), bins_sorted.get(),
                                            idx.get(), sch.perm.get(), static_cast<int>(rows), 0,
                                            3, st));
    RB_CUDA(cudaStreamSynchronize(st));
  }
  int h_counts[kNumBins];
  RB_CUDA(cudaMemcpyAsync(h_counts, counts.get(), sizeof(h_counts), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));

  int32_t row = 0, blk = 0;
  int32_t nblk[kNumBins];
  for (int b = 0; b < kNumBins; ++b) {
    const int32_t cnt = h_counts[b];
    sch.bin_rows[b] = cnt;
    if (b < kNumVBins) nblk[b] = static_cast<int32_t>(ceil_div(cnt, kBlock >> b));  // V = 1 << b
    else if (b == kBinBlock) nblk[b] = cnt;
    else nblk[b] = 0;  // split: set below
    v.bins[b] = {row, row + cnt, 0, 0};
    row += cnt;
  }
  // split rows: one block per kSplitLen-long segment
  const int32_t nsplit = h_counts[kBinSplit];
  if (nsplit > 0) {
    std::vector<int32_t> rows_h(nsplit), len_h(nsplit);
    RB_CUDA(cudaMemcpyAsync(rows_h.data(), sch.perm.get() + v.bins[kBinSplit].row_begin,
                            sizeof(int32_t) * nsplit, cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    for (int32_t i = 0; i < nsplit; ++i)
      RB_CUDA(cudaMemcpyAsync(&len_h[i], d_len + rows_h[i], sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> srow, slo, shi, sfirst, scount;
    for (int32_t i = 0; i < nsplit; ++i) {
      const int32_t L = len_h[i];
      const int32_t cnt = static_cast<int32_t>(ceil_div(L, kSplitLen));
      const int32_t first = static_cast<int32_t>(srow.size());
      for (int32_t s = 0; s < cnt; ++s) {
        srow.push_back(rows_h[i]);
        slo.push_back(s * kSplitLen);
        shi.push_back(std::min<int64_t>(L, static_cast<int64_t>(s + 1) * kSplitLen));
        sfirst.push_back(first);
        scount.push_back(cnt);
      }
    }
    const std::size_t nseg = srow.size();
    sch.seg_row.alloc(nseg), sch.seg_lo.alloc(nseg), sch.seg_hi.alloc(nseg);
    sch.seg_first.alloc(nseg), sch.seg_count.alloc(nseg);
    sch.seg_partial.alloc(nseg * kMaxAcc);
    sch.seg_ticket.alloc(nseg);
    sch.seg_ticket.zero(st);
    sch.seg_row.upload(srow.data(), nseg, st);
    sch.seg_lo.upload(slo.data(), nseg, st);
    sch.seg_hi.upload(shi.data(), nseg, st);
    sch.seg_first.upload(sfirst.data(), nseg, st);
    sch.seg_count.upload(scount.data(), nseg, st);
    RB_CUDA(cudaStreamSynchronize(st));
    nblk[kBinSplit] = static_cast<int32_t>(nseg);
  }
  // Heavy bins get the lowest block indices: blocks are dispatched roughly in
  // index order, so the long rows start first and the many light blocks fill
  // the tail instead of the heavy ones forming it.
  for (int b = kNumBins - 1; b >= 0; --b) {
    v.bins[b].blk_begin = blk;
    v.bins[b].blk_end = blk + nblk[b];
    blk += nblk[b];
  }
  v.perm = sch.perm.get();
  v.seg_row = sch.seg_row.get();
  v.seg_lo = sch.seg_lo.get();
  v.seg_hi = sch.seg_hi.get();
  v.seg_first = sch.seg_first.get();
  v.seg_count = sch.seg_count.get();
  v.seg_partial = sch.seg_partial.get();
  v.seg_ticket = sch.seg_ticket.get();
  v.total_blocks = blk;
}

}  // namespace rb
