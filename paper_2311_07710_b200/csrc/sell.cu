// sell.cu — setup of the sliced-ELL plans (see sell.cuh), all on the device.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>

#include "sell.cuh"

namespace rb {

namespace {

inline unsigned g1(int64_t n) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, 256)); }

int sell_sigma() {
  const char* e = std::getenv("RAPDHG_SELL_SIGMA");
  return e ? std::max(1, std::atoi(e)) : kSellSigma;
}

__global__ void sell_len_kernel(const int32_t* rp1, const int32_t* rp2, int32_t rows, int32_t* len, int32_t* l1,
                                uint32_t* key, int32_t* idx, int sigma, const int32_t* subset = nullptr) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int64_t pr = subset ? subset[r] : r;  // the pattern's row
  const int a = rp1[pr + 1] - rp1[pr];
  const int b = rp2 ? rp2[pr + 1] - rp2[pr] : 0;
  len[r] = a + b;
  l1[r] = a;
  if (key) {
    const int L = min(a + b, 255);
    key[r] = (static_cast<uint32_t>(r / sigma) << 8) | static_cast<uint32_t>(255 - L);  // chunk, longest first
    idx[r] = static_cast<int32_t>(r);
  }
}

// per slot: row (sorted order), its length and split; per slice: its width
__global__ void sell_slots_kernel(const int32_t* order, const int32_t* len_r, const int32_t* l1_r, int32_t rows,
                                  int64_t nslices, int32_t* row, int32_t* len, int32_t* l1, int64_t* width32,
                                  const int32_t* subset) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nslices) return;
  int w = 0;
  for (int lane = 0; lane < 32; ++lane) {
    const int64_t s = (q << 5) + lane;
    int r = 0, L = 0, a = 0;
    if (s < rows) {
      const int k = order[s];  // index into the subset (or the row itself)
      r = subset ? subset[k] : k;
      L = len_r[k];
      a = l1_r[k];
    }
    row[s] = r, len[s] = L, l1[s] = a;
    w = max(w, L);
  }
  width32[q] = static_cast<int64_t>((w + 3) & ~3) << 5;  // whole batches of 4 (the kernel's unroll)
}

// thread per slot: the row's entries, segment 1 then 2, at off[q] + 32 e + lane
__global__ void sell_fill_kernel(const int32_t* rp1, const int32_t* ci1, const int32_t* rp2, const int32_t* ci2,
                                 int64_t nslots, const int64_t* off, const int32_t* row, const int32_t* len,
                                 const int32_t* l1, int32_t* col, int64_t* pos) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= nslots) return;
  const int r = row[s], L = len[s], a = l1[s];
  const int64_t base = off[s >> 5] + (s & 31);
  const int b1 = rp1[r];
  for (int e = 0; e < a; ++e) {
    col[base + 32 * static_cast<int64_t>(e)] = ci1[b1 + e];
    pos[base + 32 * static_cast<int64_t>(e)] = b1 + e;
  }
  if (rp2) {
    const int b2 = rp2[r];
    for (int e = a; e < L; ++e) {
      col[base + 32 * static_cast<int64_t>(e)] = ci2[b2 + e - a];
      pos[base + 32 * static_cast<int64_t>(e)] = kSellSeg2 + b2 + e - a;
    }
  }
}

__global__ void sell_vals_kernel(double* val, const int64_t* pos, int64_t n, const double* v1, const double* v2) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t p = pos[i];
  val[i] = p < 0 ? 0.0 : (p >= kSellSeg2 ? v2[p - kSellSeg2] : v1[p]);
}

}  // namespace

bool sell_enabled() {
  const char* e = std::getenv("RAPDHG_SELL");
  return !(e && e[0] == '0');
}

bool sell_eligible(const int32_t* rp1, const int32_t* rp2, int32_t rows, cudaStream_t st) {
  if (!sell_enabled() || rows <= 0) return false;
  DevBuf<int32_t> len(rows), l1(rows);
  sell_len_kernel<<<g1(rows), 256, 0, st>>>(rp1, rp2, rows, len.get(), l1.get(), nullptr, nullptr, 1);
  RB_LAUNCH_CHECK();
  DevBuf<int32_t> mx(1);
  std::size_t tb = 0;
  RB_CUDA(cub::DeviceReduce::Max(nullptr, tb, len.get(), mx.get(), rows, st));
  DevBuf<unsigned char> tmp(tb);
  RB_CUDA(cub::DeviceReduce::Max(tmp.get(), tb, len.get(), mx.get(), rows, st));
  int32_t h = 0;
  RB_CUDA(cudaMemcpyAsync(&h, mx.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  return h <= kSellMaxLen;
}

void build_sell_plan(SellPlan& plan, const int32_t* rp1, const int32_t* ci1, const int32_t* rp2, const int32_t* ci2,
                     int32_t rows, cudaStream_t st, const int32_t* subset) {
  plan = SellPlan{};
  if (rows <= 0) return;
  DevBuf<int32_t> len(rows), l1(rows), idx(rows), order(rows);
  DevBuf<uint32_t> key(rows), key_s(rows);
  const int sigma = sell_sigma();
  sell_len_kernel<<<g1(rows), 256, 0, st>>>(rp1, rp2, rows, len.get(), l1.get(), key.get(), idx.get(), sigma,
                                            subset);
  RB_LAUNCH_CHECK();
  if (sigma <= 32) {  // index order
    RB_CUDA(cudaMemcpyAsync(order.get(), idx.get(), sizeof(int32_t) * rows, cudaMemcpyDeviceToDevice, st));
  } else {
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.get(), key_s.get(), idx.get(), order.get(), rows, 0, 32,
                                            st));
    DevBuf<unsigned char> tmp(tb);
    RB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, key.get(), key_s.get(), idx.get(), order.get(), rows, 0,
                                            32, st));
  }
  const int64_t nslices = ceil_div(static_cast<int64_t>(rows), 32);
  const int64_t nslots = nslices * 32;
  plan.row.alloc(nslots), plan.len.alloc(nslots), plan.l1.alloc(nslots);
  DevBuf<int64_t> w32(nslices);
  sell_slots_kernel<<<g1(nslices), 256, 0, st>>>(order.get(), len.get(), l1.get(), rows, nslices, plan.row.get(),
                                                 plan.len.get(), plan.l1.get(), w32.get(), subset);
  RB_LAUNCH_CHECK();
  plan.off.alloc(nslices + 1);
  plan.off.zero(st);
  {
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, w32.get(), plan.off.get() + 1, nslices, st));
    DevBuf<unsigned char> tmp(tb);
    RB_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, w32.get(), plan.off.get() + 1, nslices, st));
  }
  int64_t total = 0;
  RB_CUDA(cudaMemcpyAsync(&total, plan.off.get() + nslices, sizeof(total), cudaMemcpyDeviceToHost, st));
  RB_CUDA(cudaStreamSynchronize(st));
  total = std::max<int64_t>(total, 32);
  plan.col.alloc(total), plan.pos.alloc(total), plan.val.alloc(total);
  RB_CUDA(cudaMemsetAsync(plan.col.get(), 0, sizeof(int32_t) * total, st));
  RB_CUDA(cudaMemsetAsync(plan.pos.get(), 0xff, sizeof(int64_t) * total, st));  // -1: padding
  sell_fill_kernel<<<g1(nslots), 256, 0, st>>>(rp1, ci1, rp2, ci2, rows, plan.off.get(), plan.row.get(),
                                               plan.len.get(), plan.l1.get(), plan.col.get(), plan.pos.get());
  RB_LAUNCH_CHECK();
  SellView& v = plan.view;
  v.nslots = rows;
  v.nslices = nslices;
  v.off = plan.off.get();
  v.row = plan.row.get();
  v.len = plan.len.get();
  v.l1 = plan.l1.get();
  v.col = plan.col.get();
  v.val = plan.val.get();
  RB_CUDA(cudaStreamSynchronize(st));
}

void fill_sell_values(SellPlan& plan, const double* v1, const double* v2, cudaStream_t st) {
  if (!plan.active()) return;
  const int64_t n = static_cast<int64_t>(plan.val.size());
  sell_vals_kernel<<<g1(n), 256, 0, st>>>(plan.val.get(), plan.pos.get(), n, v1, v2);
  RB_LAUNCH_CHECK();
}

}  // namespace rb
