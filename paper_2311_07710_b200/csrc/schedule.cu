// schedule.cu — builds the length-binned row schedule consumed by
// rowwise_kernel (rowwise.cuh). Built once per matrix pattern at setup, on
// the device: bin ids from row lengths, a stable radix sort of row indices by
// bin (rows stay in increasing order inside a bin, so epilogue stores stay
// mostly contiguous), and a host-side segment table for the few rows longer
// than kSplitLen.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "rowwise.cuh"

namespace rb {

namespace {

__global__ void bin_kernel(int32_t* bin, int32_t* idx, const int32_t* len, int64_t rows,
                           int* counts, int epl, int block_min) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int b = bin_of_len(len[r], epl, block_min);
  bin[r] = b;
  idx[r] = static_cast<int32_t>(r);
  atomicAdd(&counts[b], 1);  // integer counts: exact
}

}  // namespace

SchedParams SchedParams::from_env() {
  SchedParams p;
  if (const char* e = std::getenv("RAPDHG_EPL")) p.epl = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("RAPDHG_BLOCK_MIN")) p.block_min = std::max(32 * p.epl, std::atoi(e));
  if (p.block_min > kSplitLen) p.block_min = kSplitLen;
  return p;
}

void build_schedule(Schedule& sch, const int32_t* d_len, int64_t rows, bool strict,
                    cudaStream_t st) {
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
        bins.get(), idx.get(), d_len, rows, counts.get(), sp.epl, sp.block_min);
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
    for (int32_t i = 0; i < nsplit; ++i) {
      RB_CUDA(cudaMemcpy(&len_h[i], d_len + rows_h[i], sizeof(int32_t), cudaMemcpyDeviceToHost));
    }
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
