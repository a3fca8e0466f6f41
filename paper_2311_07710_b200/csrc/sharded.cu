// sharded.cu — row-sharded multi-GPU rAPDHG; see sharded.hpp for the design.
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>

#include "elementwise.cuh"
#include "sharded.hpp"
#include "terms.cuh"

namespace rb {

namespace {

inline unsigned grid1(int64_t n) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, 256)); }

__global__ void halo_pack_kernel(double* dst, const double* src, const int32_t* idx, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = src[idx[k]];
}
__global__ void halo_unpack_kernel(double* dst, const double* src, const int32_t* idx, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[idx[k]] = src[k];
}
inline unsigned gridn(int64_t n) { return static_cast<unsigned>(std::min<int64_t>(ceil_div(n > 0 ? n : 1, 256), 8 * kSMs)); }
void halo_pack(const HaloSide& h, const double* buf, cudaStream_t st) {
  const int64_t n = h.send_off.back();
  if (n > 0) halo_pack_kernel<<<gridn(n), 256, 0, st>>>(h.send_buf.get(), buf, h.send_idx.get(), n);
  RB_LAUNCH_CHECK();
}
void halo_unpack(const HaloSide& h, double* buf, cudaStream_t st) {
  const int64_t n = h.recv_off.back();
  if (n > 0) halo_unpack_kernel<<<gridn(n), 256, 0, st>>>(buf, h.recv_buf.get(), h.recv_idx.get(), n);
  RB_LAUNCH_CHECK();
}

// flags[ci[k]] = 1 for the entries of rows [r0, r1)
__global__ void halo_mark_kernel(const int32_t* rp, const int32_t* ci, int64_t r0, int64_t r1, uint8_t* flags) {
  const int64_t b = rp[r0], e = rp[r1];
  for (int64_t k = b + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < e;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flags[ci[k]] = 1;
}
// pos[j] = first position in the sorted list with value >= keys[j]
__global__ void lower_bounds_kernel(const int32_t* list, const int32_t* count, const int64_t* keys, int nk,
                                    int64_t* pos) {
  const int j = threadIdx.x;
  if (j >= nk) return;
  int64_t lo = 0, hi = *count;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (list[mid] < keys[j]) lo = mid + 1;
    else hi = mid;
  }
  pos[j] = lo;
}

__global__ void invert_kernel(const uint8_t* a, uint8_t* b, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) b[i] = !a[i];
}

// flag[i] = 1 when row r0 + i of [seg1 | seg2] references a column outside
// [lo1, hi1) (segment 1) or [lo2, hi2) (segment 2): a boundary row
__global__ void boundary_kernel(const int32_t* rp1, const int32_t* ci1, int64_t lo1, int64_t hi1, const int32_t* rp2,
                                const int32_t* ci2, int64_t lo2, int64_t hi2, int64_t r0, int64_t rows,
                                uint8_t* flag) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= rows) return;
  const int64_t r = r0 + i;
  uint8_t b = 0;
  for (int k = rp1[r]; k < rp1[r + 1] && !b; ++k) b = ci1[k] < lo1 || ci1[k] >= hi1;
  if (rp2)
    for (int k = rp2[r]; k < rp2[r + 1] && !b; ++k) b = ci2[k] < lo2 || ci2[k] >= hi2;
  flag[i] = b;
}

// Row-aware variant of halo_mark_kernel: rows with skip[r] set are left out.
__global__ void halo_mark_rows_kernel(const int32_t* rp, const int32_t* ci, int64_t r0, int64_t r1,
                                      const uint8_t* skip, uint8_t* flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = r0 + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < r1; r += warps) {
    if (skip[r]) continue;
    for (int64_t k = rp[r] + lane; k < rp[r + 1]; k += 32) flags[ci[k]] = 1;
  }
}
__global__ void clear_listed_kernel(uint8_t* flags, const int32_t* list, int32_t n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[list[i]] = 0;
}
__global__ void set_listed_kernel(uint8_t* flags, const int32_t* list, int32_t n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[list[i]] = 1;
}

// ---- replicated dense primal rows (ShardedEngine::replicated_step) -------------
// For replicated row idx (row j = rows[idx]): the positions of its Q entries
// with a column in [p0, p1) and of its A' entries with a column in [d0, d1) —
// contiguous, since columns are sorted within a row.
__device__ __forceinline__ int32_t first_at_least(const int32_t* c, int32_t b, int32_t e, int64_t key) {
  while (b < e) {
    const int32_t mid = b + (e - b) / 2;
    if (c[mid] < key) b = mid + 1;
    else e = mid;
  }
  return b;
}
__global__ void rep_ranges_kernel(const int32_t* rows, int32_t nr, const int32_t* qrp, const int32_t* qci, int64_t p0,
                                  int64_t p1, const int32_t* arp, const int32_t* aci, int64_t d0, int64_t d1,
                                  int32_t* qlo, int32_t* qhi, int32_t* alo, int32_t* ahi, int32_t* len) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nr) return;
  const int32_t j = rows[idx];
  const int32_t ql = first_at_least(qci, qrp[j], qrp[j + 1], p0), qh = first_at_least(qci, qrp[j], qrp[j + 1], p1);
  const int32_t al = first_at_least(aci, arp[j], arp[j + 1], d0), ah = first_at_least(aci, arp[j], arp[j + 1], d1);
  qlo[idx] = ql, qhi[idx] = qh, alo[idx] = al, ahi[idx] = ah;
  len[idx] = (qh - ql) + (ah - al);
}

// A shard's partial sums of the replicated rows over its own columns, as a
// rowwise op ("row" r = replicated index): (Q x_md, A' y) restricted to the
// owned primal / dual block, the lanes and unroll of the rowwise engine.
struct RepPartialOp {
  static constexpr bool kStrict = false;
  static constexpr int kWideUnroll = kUnroll;
  static constexpr bool kStageWindows = false;
  using AccT = Acc<2>;
  const int32_t *qlo, *qhi, *alo, *ahi;
  const int32_t* qci;
  const double* qv;
  const int32_t* aci;
  const double* av;
  const double* xmd;
  const double* y;
  double* part;  // 2 per row: (Q part, A' part)
  __device__ __forceinline__ int len(int r) const { return (qhi[r] - qlo[r]) + (ahi[r] - alo[r]); }
  template <int U>
  __device__ __forceinline__ void accumulate(int r, int lo, int hi, int lane, int stride, AccT& acc,
                                             const Gather* g) const {
    const int q0 = qlo[r];
    const int L1 = qhi[r] - q0;
    const int p = lo + lane;
    acc.v[0] = seg_dot<false, U>(qv, qci, g[0], q0, p, hi < L1 ? hi : L1, stride, acc.v[0]);
    acc.v[1] = seg_dot<false, U>(av, aci, g[1], static_cast<int64_t>(alo[r]) - L1, next_pos(p, stride, L1), hi,
                                 stride, acc.v[1]);
  }
  __device__ __forceinline__ const double* gather_src(int slot) const { return slot ? y : xmd; }
  __device__ __forceinline__ void finish(int r, const AccT& acc) const {
    part[2 * r] = acc.v[0];
    part[2 * r + 1] = acc.v[1];
  }
};

// Every shard: the replicated rows' sums from all shards' partials (added in
// shard order: the same bits everywhere), then the primal step's epilogue.
__global__ void rep_finish_kernel(const PrimalStepOp<false> pr, const int32_t* rows, const double* part, int32_t nr,
                                  int parts) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nr) return;
  const int j = rows[idx];
  Acc<2> acc;
  acc.v[0] = 0.0;
  acc.v[1] = 0.0;
  const int64_t stride = 2 * static_cast<int64_t>(nr);
  for (int s = 0; s < parts; ++s) {
    acc.v[0] += part[s * stride + 2 * idx];
    acc.v[1] += part[s * stride + 2 * idx + 1];
  }
  pr.finish(j, acc, pr.prefetch(j));
}
// prologue_kernel / restart_kernel (elementwise.cuh) on the replicated rows
__global__ void rep_prologue_kernel(const int32_t* rows, int32_t nr, const double* x, const double* xp,
                                    const double* xb, double* w, double* xmd, const IterParams* P) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nr) return;
  const int j = rows[idx];
  const IterParams& q = P[0];
  const double xj = x[j];
  w[j] = q.theta * (xj - xp[j]) + xj;
  xmd[j] = q.omib * xb[j] + q.ib * xj;
}
__global__ void rep_restart_kernel(const int32_t* rows, int32_t nr, double* x, double* xp, double* xb, int from_avg) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nr) return;
  const int j = rows[idx];
  const double v = from_avg ? xb[j] : x[j];
  x[j] = v;
  xp[j] = v;
  xb[j] = v;
}

// Boundaries of `parts` contiguous blocks of rows with costs len[r] + 2,
// inner boundaries rounded to multiples of kRedChunk (never decreasing).
std::vector<int32_t> balanced_bounds(const std::vector<int64_t>& cost_prefix, int32_t rows, int parts) {
  std::vector<int32_t> b(parts + 1, 0);
  b[parts] = rows;
  const double total = static_cast<double>(cost_prefix[rows]);
  for (int k = 1; k < parts; ++k) {
    const double target = total * k / parts;
    const auto it = std::lower_bound(cost_prefix.begin(), cost_prefix.end(), static_cast<int64_t>(target));
    int64_t r = std::distance(cost_prefix.begin(), it);
    r = ((r + kRedChunk / 2) / kRedChunk) * kRedChunk;  // align for the chunked reductions
    // never past the last whole chunk: a bound at `rows` would hand the final
    // partial chunk's reduction slot to an empty trailing shard
    r = std::min<int64_t>(std::max<int64_t>(r, b[k - 1]), (rows / kRedChunk) * kRedChunk);
    b[k] = static_cast<int32_t>(r);
  }
  return b;
}

}  // namespace

int64_t replicate_min_len_from_env() {
  const char* e = std::getenv("RAPDHG_REPLICATE_MIN_LEN");
  return e ? std::max<int64_t>(0, std::atoll(e)) : 0;
}

ShardPlan make_shard_plan(const rapdhg_qp& p, int parts, int64_t replicate_min_len) {
  if (parts < 1) invalid("shard plan: parts must be >= 1");
  const int n = p.n, m = p.m_ineq + p.m_eq;
  // primal rows: rows of [Q | A'] (A' row j = column j of A)
  std::vector<int64_t> colcnt(static_cast<std::size_t>(n), 0);
  for (int64_t k = 0; k < p.a_ineq.nnz; ++k) ++colcnt[p.a_ineq.col_idx[k]];
  for (int64_t k = 0; k < p.a_eq.nnz; ++k) ++colcnt[p.a_eq.col_idx[k]];
  ShardPlan plan;
  std::vector<uint8_t> rep(static_cast<std::size_t>(n), 0);
  if (replicate_min_len > 0 && parts > 1)
    for (int j = 0; j < n; ++j)
      if ((p.q.row_ptr[j + 1] - p.q.row_ptr[j]) + colcnt[j] >= replicate_min_len) {
        rep[j] = 1;
        plan.replicated.push_back(j);
      }
  // dual rows: rows of [A_ineq; A_eq]; an entry in a replicated column is
  // summed twice per step (A w here, the replicated rows' partial A'y too)
  auto dual_cost = [&](const rapdhg_csr& a, int i) {
    int64_t c = a.row_ptr[i + 1] - a.row_ptr[i] + 2;
    if (!plan.replicated.empty())
      for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) c += rep[a.col_idx[k]];
    return c;
  };
  std::vector<int64_t> dp(static_cast<std::size_t>(m) + 1, 0);
  for (int i = 0; i < p.m_ineq; ++i) dp[i + 1] = dp[i] + dual_cost(p.a_ineq, i);
  for (int i = 0; i < p.m_eq; ++i) dp[p.m_ineq + i + 1] = dp[p.m_ineq + i] + dual_cost(p.a_eq, i);
  std::vector<int64_t> pp(static_cast<std::size_t>(n) + 1, 0);
  for (int j = 0; j < n; ++j)
    pp[j + 1] = pp[j] + (rep[j] ? 0 : (p.q.row_ptr[j + 1] - p.q.row_ptr[j]) + colcnt[j]) + 2;
  plan.dual = balanced_bounds(dp, m, parts);
  plan.primal = balanced_bounds(pp, n, parts);
  return plan;
}

// ---- transports ----------------------------------------------------------------

namespace {

class EmulatedTransport : public Transport {
 public:
  explicit EmulatedTransport(int parts) : parts_(parts) {}
  void allgatherv(const std::vector<double*>& bufs, const std::vector<int64_t>& b, cudaStream_t st) override {
    for (int k = 0; k < parts_; ++k) {  // owner k's slice into every other shard's copy
      const int64_t len = b[k + 1] - b[k];
      if (len <= 0) continue;
      for (int j = 0; j < parts_; ++j)
        if (j != k)
          RB_CUDA(cudaMemcpyAsync(bufs[j] + b[k], bufs[k] + b[k], sizeof(double) * len, cudaMemcpyDeviceToDevice, st));
    }
  }
  // the NCCL protocol with device copies between the shards' packed buffers
  void halo(const std::vector<double*>& bufs, const std::vector<HaloSide*>& sides, cudaStream_t st) override {
    for (int j = 0; j < parts_; ++j) halo_pack(*sides[j], bufs[j], st);
    for (int i = 0; i < parts_; ++i)
      for (int j = 0; j < parts_; ++j) {
        if (i == j) continue;
        const int64_t cnt = sides[i]->recv_off[j + 1] - sides[i]->recv_off[j];
        if (cnt != sides[j]->send_off[i + 1] - sides[j]->send_off[i])
          throw Error(RAPDHG_E_INTERNAL, "halo lists disagree");
        if (cnt > 0)
          RB_CUDA(cudaMemcpyAsync(sides[i]->recv_buf.get() + sides[i]->recv_off[j],
                                  sides[j]->send_buf.get() + sides[j]->send_off[i], sizeof(double) * cnt,
                                  cudaMemcpyDeviceToDevice, st));
      }
    for (int i = 0; i < parts_; ++i) halo_unpack(*sides[i], bufs[i], st);
  }
  long long allreduce_min(const std::vector<long long*>& vals, cudaStream_t st) override {
    long long best = std::numeric_limits<long long>::max();
    for (long long* v : vals) {
      long long h = 0;
      RB_CUDA(cudaMemcpyAsync(&h, v, sizeof(h), cudaMemcpyDeviceToHost, st));
      RB_CUDA(cudaStreamSynchronize(st));
      best = std::min(best, h);
    }
    return best;
  }

 private:
  int parts_;
};

// libnccl is loaded on first use so the library itself has no NCCL
// dependency (and coexists with whichever libnccl.so.2 torch loaded first).
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    // the NCCL the process already has (e.g. torch's), else RAPDHG_NCCL_LIB
    // (the Python binding points it at the pip NCCL torch ships), else the
    // system one. Loading an older libnccl.so.2 first would make a later
    // `import torch` bind to it and fail on newer symbols.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h)
      if (const char* path = std::getenv("RAPDHG_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) err = std::string("libnccl lacks ") + name;
      return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw Error(RAPDHG_E_CUDA, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(RAPDHG_E_CUDA, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

class NcclTransport : public Transport {
 public:
  NcclTransport(int parts, int rank, const void* id) : parts_(parts), rank_(rank) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().CommInitRank(&comm_, parts, uid, rank), "ncclCommInitRank");
    scratch_.alloc(1);
  }
  ~NcclTransport() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  // allgather-v: every owner broadcasts its slice in place, grouped
  void allgatherv(const std::vector<double*>& bufs, const std::vector<int64_t>& b, cudaStream_t st) override {
    double* buf = bufs.at(0);
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int k = 0; k < parts_; ++k) {
      const int64_t len = b[k + 1] - b[k];
      if (len > 0)
        nccl_check(nccl().Broadcast(buf + b[k], buf + b[k], static_cast<size_t>(len), ncclDouble, k, comm_, st),
                   "ncclBroadcast");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }
  // pack, grouped point-to-point sends/receives with every peer, unpack
  void halo(const std::vector<double*>& bufs, const std::vector<HaloSide*>& sides, cudaStream_t st) override {
    const HaloSide& h = *sides.at(0);
    halo_pack(h, bufs.at(0), st);
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int p = 0; p < parts_; ++p) {
      if (p == rank_) continue;
      const int64_t ns = h.send_off[p + 1] - h.send_off[p], nr = h.recv_off[p + 1] - h.recv_off[p];
      if (ns > 0)
        nccl_check(nccl().Send(h.send_buf.get() + h.send_off[p], static_cast<size_t>(ns), ncclDouble, p, comm_, st),
                   "ncclSend");
      if (nr > 0)
        nccl_check(nccl().Recv(h.recv_buf.get() + h.recv_off[p], static_cast<size_t>(nr), ncclDouble, p, comm_, st),
                   "ncclRecv");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    halo_unpack(h, bufs.at(0), st);
  }
  long long allreduce_min(const std::vector<long long*>& vals, cudaStream_t st) override {
    nccl_check(nccl().AllReduce(vals.at(0), scratch_.get(), 1, ncclInt64, ncclMin, comm_, st), "ncclAllReduce");
    long long h = 0;
    RB_CUDA(cudaMemcpyAsync(&h, scratch_.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    return h;
  }

 private:
  int parts_, rank_;
  ncclComm_t comm_ = nullptr;
  DevBuf<long long> scratch_;
};

// The caller's collectives as host callbacks: every exchange is staged
// through pinned host memory around one callback (test and portability path;
// NCCL is the fast path).
class HostTransport : public Transport {
 public:
  HostTransport(int parts, int rank, const rapdhg_host_transport& t) : parts_(parts), rank_(rank), t_(t) {
    if (!t.allgatherv || !t.alltoallv || !t.allreduce_min) invalid("host transport: null callback");
  }
  bool capturable() const override { return false; }
  void allgatherv(const std::vector<double*>& bufs, const std::vector<int64_t>& b, cudaStream_t st) override {
    double* buf = bufs.at(0);
    const int64_t total = b.back(), lo = b[rank_], hi = b[rank_ + 1];
    double* h = stage(a_, total);
    if (hi > lo) RB_CUDA(cudaMemcpyAsync(h + lo, buf + lo, sizeof(double) * (hi - lo), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    call(t_.allgatherv(t_.ctx, h, b.data(), parts_), "allgatherv");
    if (lo > 0) RB_CUDA(cudaMemcpyAsync(buf, h, sizeof(double) * lo, cudaMemcpyHostToDevice, st));
    if (total > hi)
      RB_CUDA(cudaMemcpyAsync(buf + hi, h + hi, sizeof(double) * (total - hi), cudaMemcpyHostToDevice, st));
    RB_CUDA(cudaStreamSynchronize(st));  // the staging buffer is reused by the next exchange
  }
  void halo(const std::vector<double*>& bufs, const std::vector<HaloSide*>& sides, cudaStream_t st) override {
    const HaloSide& h = *sides.at(0);
    halo_pack(h, bufs.at(0), st);
    const int64_t ns = h.send_off.back(), nr = h.recv_off.back();
    double* hs = stage(a_, ns);
    double* hr = stage(b_, nr);
    if (ns) RB_CUDA(cudaMemcpyAsync(hs, h.send_buf.get(), sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    call(t_.alltoallv(t_.ctx, hs, h.send_off.data(), hr, h.recv_off.data(), parts_), "alltoallv");
    if (nr) RB_CUDA(cudaMemcpyAsync(h.recv_buf.get(), hr, sizeof(double) * nr, cudaMemcpyHostToDevice, st));
    halo_unpack(h, bufs.at(0), st);
    RB_CUDA(cudaStreamSynchronize(st));
  }
  long long allreduce_min(const std::vector<long long*>& vals, cudaStream_t st) override {
    int64_t v = 0;
    RB_CUDA(cudaMemcpyAsync(&v, vals.at(0), sizeof(v), cudaMemcpyDeviceToHost, st));
    RB_CUDA(cudaStreamSynchronize(st));
    call(t_.allreduce_min(t_.ctx, &v), "allreduce_min");
    return v;
  }

 private:
  static void call(int rc, const char* what) {
    if (rc != 0) throw Error(RAPDHG_E_CUDA, std::string("host transport ") + what + " failed (" + std::to_string(rc) + ")");
  }
  static double* stage(PinnedBuf<double>& p, int64_t n) {
    if (static_cast<int64_t>(p.size()) < n) p.alloc(static_cast<std::size_t>(n));
    return p.get();
  }
  int parts_, rank_;
  rapdhg_host_transport t_;
  PinnedBuf<double> a_, b_;
};

}  // namespace

std::unique_ptr<Transport> make_host_transport(int parts, int rank, const rapdhg_host_transport& t) {
  return std::make_unique<HostTransport>(parts, rank, t);
}

// Deterministic data for each exchange kind, checked on arrival.
void host_transport_check(const rapdhg_host_transport& t, int parts, int rank, int64_t len) {
  if (parts < 1 || rank < 0 || rank >= parts || len < 0) invalid("host transport check: bad arguments");
  if (!t.allgatherv || !t.alltoallv || !t.allreduce_min) invalid("host transport: null callback");
  auto fail = [](const std::string& m) { throw Error(RAPDHG_E_INTERNAL, "host transport check: " + m); };
  // allgather-v over uneven slices
  std::vector<int64_t> b(parts + 1, 0);
  for (int k = 0; k < parts; ++k) b[k + 1] = b[k] + len / parts + (k < len % parts ? 1 : 0) + k;
  std::vector<double> buf(static_cast<std::size_t>(b[parts]), std::nan(""));
  auto f = [](int64_t i) { return 1.5 * static_cast<double>(i) + 0.25; };
  for (int64_t i = b[rank]; i < b[rank + 1]; ++i) buf[i] = f(i);
  if (t.allgatherv(t.ctx, buf.data(), b.data(), parts) != 0) fail("allgatherv returned an error");
  for (int64_t i = 0; i < b[parts]; ++i)
    if (buf[i] != f(i)) fail("allgatherv delivered a wrong value at " + std::to_string(i));
  // all-to-all-v: rank r sends cnt(r, p) values g(r, p, k) to p
  auto cnt = [&](int r, int p) { return r == p ? int64_t{0} : (r * 7 + p * 3) % 5 + 1 + len % 3; };
  auto g = [](int r, int p, int64_t k) { return r * 1000.0 + p * 100.0 + static_cast<double>(k) + 0.5; };
  std::vector<int64_t> so(parts + 1, 0), ro(parts + 1, 0);
  for (int p = 0; p < parts; ++p) so[p + 1] = so[p] + cnt(rank, p), ro[p + 1] = ro[p] + cnt(p, rank);
  std::vector<double> send(static_cast<std::size_t>(std::max<int64_t>(so[parts], 1))), recv(
      static_cast<std::size_t>(std::max<int64_t>(ro[parts], 1)), std::nan(""));
  for (int p = 0; p < parts; ++p)
    for (int64_t k = 0; k < cnt(rank, p); ++k) send[so[p] + k] = g(rank, p, k);
  if (t.alltoallv(t.ctx, send.data(), so.data(), recv.data(), ro.data(), parts) != 0)
    fail("alltoallv returned an error");
  for (int p = 0; p < parts; ++p)
    for (int64_t k = 0; k < cnt(p, rank); ++k)
      if (recv[ro[p] + k] != g(p, rank, k)) fail("alltoallv delivered a wrong value from rank " + std::to_string(p));
  // min-reduction
  int64_t v = 100 + 3 * (parts - 1 - rank);
  if (t.allreduce_min(t.ctx, &v) != 0) fail("allreduce_min returned an error");
  if (v != 100) fail("allreduce_min returned " + std::to_string(v));
}

std::unique_ptr<Transport> make_emulated_transport(int parts) {
  return std::make_unique<EmulatedTransport>(parts);
}
std::unique_ptr<Transport> make_nccl_transport(int parts, int rank, const void* id) {
  return std::make_unique<NcclTransport>(parts, rank, id);
}
void nccl_unique_id(void* out) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, sizeof(uid));
}

// ---- the sharded engine -----------------------------------------------------------

struct ShardedEngine::Shard {
  int id = 0;
  int64_t d0 = 0, d1 = 0, p0 = 0, p1 = 0;  // dual / primal row blocks
  Schedule sch_dual, sch_primal;
  // slab plans restricted to the owned rows, built from the GLOBAL window
  // choice so every row is computed as on one GPU; + complement schedules
  SlabPhase dual_ph, primal_ph;
  ColBlockedDual cbd;  // column blocks over the owned rows (same block counts as one GPU)
  ColBlockedPrimal cbp;
  SellPlan sell_dual, sell_primal;  // sliced ELL over the owned rows (plain path)
  // overlap (plain path): rows whose entries are all owned ("interior") run
  // while the exchange of the step's gathered vector is in flight; the
  // others ("boundary") after it. Same per-row arithmetic as one launch.
  Schedule sch_dual_in, sch_dual_bd, sch_primal_in, sch_primal_bd;
  SellPlan sell_dual_in, sell_dual_bd, sell_primal_in, sell_primal_bd;
  // full-length copies; only the owned slice is computed here, the rest is
  // received by the exchanges
  DevBuf<double> X[2], XMD[2], w, xb, y, yb, epx, epy, xu[2], yu[2], ax[2], qx[2], aty[2], best_x, best_y;
  DevBuf<double2> xi, yi;  // interleaved unscaled points for the KKT products
  DevBuf<long long> bad, vote;
  ReduceScratch red;
  DevBuf<double> red_out;
  // replicated dense rows (ShardedEngine::replicated_step): the sub-ranges of
  // their entries on this shard's columns, a schedule over them, the partial
  // sums of all shards, and the step's schedule over the owned rows that are
  // not replicated
  DevBuf<int32_t> rep_qlo, rep_qhi, rep_alo, rep_ahi;
  Schedule sch_rep, sch_primal_step;
  DevBuf<double> rep_part;
  // the distributed norm estimate: the A' rows of the owned block, and the
  // iteration's vectors (full length; freed after the setup)
  Schedule sch_at;
  DevBuf<double> nv, nw, nmv;
};

ShardedEngine::ShardedEngine(const rapdhg_qp& p, const rapdhg_config& cfg, int parts, int rank,
                             std::unique_ptr<Transport> tr, Clock::time_point t0, int64_t replicate_min_len)
    : cfg_(cfg), parts_(parts), tr_(std::move(tr)) {
  if (cfg.strict_parity) invalid("sharded solve: strict_parity needs sequential reductions; use one GPU");
  if (parts < 1) invalid("sharded solve: parts must be >= 1");
  // validation, scaling, norms and the slab window choices; the single-GPU
  // slab phases / column blocks over all rows are not built (each shard
  // builds its own over its rows below)
  {
    const char* e = std::getenv("RAPDHG_SHARD_NORMS");
    shard_norms_ = !(e && e[0] == '0');
  }
  full_ = std::make_unique<Engine>(p, cfg, t0, /*full_plans=*/false, /*norm_a=*/!shard_norms_);
  plan_ = make_shard_plan(p, parts,
                          replicate_min_len > 0 ? replicate_min_len
                                                : (replicate_min_len == 0 ? replicate_min_len_from_env() : 0));
  st_ = full_->st_;
  AllocStreamScope scope(st_);
  DeviceQP& P = *full_->P_;
  const int n = P.n, m = P.m;
  pb_.assign(plan_.primal.begin(), plan_.primal.end());
  db_.assign(plan_.dual.begin(), plan_.dual.end());
  nrep_ = static_cast<int32_t>(plan_.replicated.size());
  if (nrep_) {
    rep_rows_.alloc(nrep_);
    rep_rows_.upload(plan_.replicated.data(), nrep_, st_);
    rep_flag_.alloc(n);
    rep_flag_.zero(st_);
    set_listed_kernel<<<grid1(nrep_), 256, 0, st_>>>(rep_flag_.get(), rep_rows_.get(), nrep_);
    RB_LAUNCH_CHECK();
  }
  for (int s = 0; s < parts; ++s) {
    if (rank >= 0 && s != rank) continue;
    auto sh = std::make_unique<Shard>();
    sh->id = s;
    sh->d0 = db_[s], sh->d1 = db_[s + 1], sh->p0 = pb_[s], sh->p1 = pb_[s + 1];
    DevBuf<int32_t> len;
    row_lengths(len, P.A.rp.get() + sh->d0, nullptr, sh->d1 - sh->d0, st_);
    build_schedule(sh->sch_dual, len.get(), sh->d1 - sh->d0, false, st_);
    if (!full_->dual_choice_.empty() && sh->d1 > sh->d0) {
      build_slab_phase(sh->dual_ph, full_->dual_choice_, 0, P.A.rp.get(), P.A.ci.get(), nullptr, nullptr,
                       static_cast<int32_t>(sh->d0), static_cast<int32_t>(sh->d1), len.get(), st_);
      if (sh->dual_ph.active()) {
        fill_slab_values(sh->dual_ph.plan, full_->asv_, nullptr, st_);
        fill_sell_values(sh->dual_ph.others_sell, full_->asv_, nullptr, st_);
        prepare_slab<PhaseSpmvOp<1>>(sh->dual_ph.plan.view.smem_bytes());  // the distributed norm estimate
        assign_slab_ctas(sh->dual_ph.plan, prepare_slab<DualStepOp<false>>(sh->dual_ph.plan.view.smem_bytes()), st_);
      }
    }
    row_lengths(len, P.Q.rp.get() + sh->p0, P.AT.rp.get() + sh->p0, sh->p1 - sh->p0, st_);
    build_schedule(sh->sch_primal, len.get(), sh->p1 - sh->p0, false, st_);
    if (nrep_ == 0 && !full_->primal_choice_.empty() && sh->p1 > sh->p0) {
      build_slab_phase(sh->primal_ph, full_->primal_choice_, 1, P.Q.rp.get(), P.Q.ci.get(), P.AT.rp.get(),
                       P.AT.ci.get(), static_cast<int32_t>(sh->p0), static_cast<int32_t>(sh->p1), len.get(), st_);
      if (sh->primal_ph.active()) {
        fill_slab_values(sh->primal_ph.plan, full_->qsv_, full_->atsv_, st_);
        fill_sell_values(sh->primal_ph.others_sell, full_->qsv_, full_->atsv_, st_);
        prepare_slab<PhaseSpmvOp<2>>(sh->primal_ph.plan.view.smem_bytes());
        assign_slab_ctas(sh->primal_ph.plan, prepare_slab<PrimalStepOp<false>>(sh->primal_ph.plan.view.smem_bytes()), st_);
      }
    }
    for (int i = 0; i < 2; ++i) {
      sh->X[i].alloc(n), sh->XMD[i].alloc(n), sh->xu[i].alloc(n), sh->yu[i].alloc(m);
      sh->ax[i].alloc(m), sh->qx[i].alloc(n), sh->aty[i].alloc(n);
    }
    sh->w.alloc(n), sh->xb.alloc(n), sh->y.alloc(m), sh->yb.alloc(m), sh->epx.alloc(n), sh->epy.alloc(m);
    sh->xi.alloc(n), sh->yi.alloc(m);
    sh->best_x.alloc(n), sh->best_y.alloc(m);
    sh->bad.alloc(1), sh->vote.alloc(1);
    sh->red.init(std::max<int64_t>(n, m), st_);
    sh->red_out.alloc(64);
    shards_.push_back(std::move(sh));
  }
  params_.alloc(kMaxChunk);
  params_h_.alloc(kMaxChunk);
  red_h_.alloc(64);
  // column blocks for the ops whose slab phase is inactive on EVERY shard —
  // the decision one GPU takes over all rows, so every row is computed as
  // there (a vote across ranks)
  bool dual_any = false, primal_any = false;
  for (auto& sh : shards_) dual_any |= sh->dual_ph.active(), primal_any |= sh->primal_ph.active();
  if (rank >= 0 && parts > 1) {  // one process per shard: vote (min over ranks of "none here")
    auto vote = [&](bool any) {
      std::vector<long long*> v;
      const long long none = any ? 0 : 1;
      for (auto& sh : shards_) {
        RB_CUDA(cudaMemcpyAsync(sh->vote.get(), &none, sizeof(none), cudaMemcpyHostToDevice, st_));
        v.push_back(sh->vote.get());
      }
      return tr_->allreduce_min(v, st_) == 0;
    };
    dual_any = vote(dual_any);
    primal_any = vote(primal_any);
  }
  full_->colblock_counts(dual_any, primal_any);
  for (auto& sh : shards_) {
    if (!sh->dual_ph.active() && sh->d1 > sh->d0)
      build_colblocked_dual(sh->cbd, full_->cb_nb_dual_, P.A.rp.get() + sh->d0, P.A.ci.get(),
                            static_cast<int32_t>(sh->d1 - sh->d0), n, full_->asv_, full_->sell_dual_, st_);
    if (nrep_ == 0 && !sh->primal_ph.active() && sh->p1 > sh->p0)
      build_colblocked_primal(sh->cbp, full_->cb_nq_, full_->cb_na_, P.Q.rp.get() + sh->p0, P.Q.ci.get(), full_->qsv_,
                              P.AT.rp.get() + sh->p0, P.AT.ci.get(), full_->atsv_,
                              static_cast<int32_t>(sh->p1 - sh->p0), n, m, full_->sell_primal_, st_);
    // the plain path: sliced ELL over the shard's rows when one GPU would use it
    if (full_->sell_dual_ && !sh->dual_ph.active() && !sh->cbd.active() && sh->d1 > sh->d0) {
      build_sell_plan(sh->sell_dual, P.A.rp.get() + sh->d0, P.A.ci.get(), nullptr, nullptr,
                      static_cast<int32_t>(sh->d1 - sh->d0), st_);
      fill_sell_values(sh->sell_dual, full_->asv_, nullptr, st_);
    }
    if (nrep_ == 0 && full_->sell_primal_ && !sh->primal_ph.active() && !sh->cbp.active() && sh->p1 > sh->p0) {
      build_sell_plan(sh->sell_primal, P.Q.rp.get() + sh->p0, P.Q.ci.get(), P.AT.rp.get() + sh->p0, P.AT.ci.get(),
                      static_cast<int32_t>(sh->p1 - sh->p0), st_);
      fill_sell_values(sh->sell_primal, full_->qsv_, full_->atsv_, st_);
    }
  }
  build_replicated();
  build_overlap(rank < 0);
  build_halos();
  RB_CUDA(cudaStreamSynchronize(st_));
  if (shard_norms_) {
    full_->norm_a = 1.01 * distributed_norm_a(5000, 1e-4, cfg.seed);  // solver.hpp:286-289
    full_->setup_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
  }
}

namespace {
__global__ void scale_slice_kernel(double* v, const double* w, double s, int64_t lo, int64_t hi) {
  const int64_t i = lo + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < hi) v[i] = w[i] * s;  // v = w; scale(v, 1/nrm) (opnorm.hpp:52-53)
}
}  // namespace

double ShardedEngine::distributed_norm_a(int max_iters, double tol, uint64_t seed) {
  DeviceQP& P = *full_->P_;
  Engine& e = *full_;
  const int n = P.n, m = P.m;
  if (P.A.nnz == 0) return 0.0;
  const int K = norm_slab_step();  // the single-GPU switch step (Engine::norm_a_power)
  for (auto& sh : shards_) {
    sh->nv.alloc(n), sh->nw.alloc(n), sh->nmv.alloc(m);
    if (sh->p1 > sh->p0) {
      DevBuf<int32_t> len;
      row_lengths(len, P.AT.rp.get() + sh->p0, nullptr, sh->p1 - sh->p0, st_);
      build_schedule(sh->sch_at, len.get(), sh->p1 - sh->p0, false, st_);
    }
  }
  RandomStart start = draw_random_start(n, seed);
  std::mt19937_64 rng = start.rng;
  // random_unit (opnorm.hpp:20-30): the draws normalised over all n (every
  // shard holds the whole vector)
  auto random_unit = [&](const std::vector<double>& h) {
    for (auto& sh : shards_) sh->nv.upload(h.data(), n, st_);
    double s[1];
    reduce<1, 0>(true, [&](Shard& sh, int64_t lo) { return SumSq{sh.nv.get() + lo}; }, s);
    const double nrm = std::sqrt(s[0]);
    if (nrm > 0.0)
      for (auto& sh : shards_) {
        scale_slice_kernel<<<grid1(n), 256, 0, st_>>>(sh->nv.get(), sh->nv.get(), 1.0 / nrm, 0, n);
        RB_LAUNCH_CHECK();
      }
  };
  random_unit(start.v);
  double lambda = 0.0;
  bool slab = false;
  for (int it = 0; it < max_iters; ++it) {
    if (!slab && K >= 0 && it >= K) slab = true;  // the switch step (deterministic, as one GPU)
    // mv = A v on the owned dual rows, then everywhere
    for (auto& sh : shards_) {
      if (sh->d1 <= sh->d0) continue;
      const int64_t o = sh->d0;
      if (slab && sh->dual_ph.active()) {
        launches_ += launch_slab_phase(PhaseSpmvOp<1>{CsrView{P.A.rp.get() + o, P.A.ci.get(), e.asv_}, CsrView{},
                                                      sh->nv.get(), sh->nv.get(), sh->nmv.get() + o},
                                       sh->dual_ph, st_);
      } else {
        launch_rowwise(SpmvOp<false>{CsrView{P.A.rp.get() + o, P.A.ci.get(), e.asv_}, sh->nv.get(), sh->nmv.get() + o},
                       sh->sch_dual.view, st_);
        ++launches_;
      }
    }
    exchange([](Shard& sh) { return sh.nmv.get(); }, false);
    // w = A' mv on the owned primal rows (the A' segment of [Q | A'])
    for (auto& sh : shards_) {
      if (sh->p1 <= sh->p0) continue;
      const int64_t o = sh->p0;
      if (slab && sh->primal_ph.active()) {
        launches_ += launch_slab_phase(
            PhaseSpmvOp<2>{CsrView{P.Q.rp.get() + o, P.Q.ci.get(), e.qsv_}, CsrView{P.AT.rp.get() + o, P.AT.ci.get(), e.atsv_},
                           sh->nv.get(), sh->nmv.get(), sh->nw.get() + o},
            sh->primal_ph, st_);
      } else {
        launch_rowwise(SpmvOp<false>{CsrView{P.AT.rp.get() + o, P.AT.ci.get(), e.atsv_}, sh->nmv.get(), sh->nw.get() + o},
                       sh->sch_at.view, st_);
        ++launches_;
      }
    }
    double h[2];
    reduce<2, 0>(true, [&](Shard& sh, int64_t lo) { return DotAndSumSq{sh.nv.get() + lo, sh.nw.get() + lo}; }, h);
    const double lambda_next = h[0];
    const double nrm = std::sqrt(h[1]);
    if (nrm == 0.0) {  // v in the null space: restart from fresh draws (opnorm.hpp:53-57)
      std::vector<double> v(n);
      for (double& x : v) x = 2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0;
      random_unit(v);
      continue;
    }
    if (it > 0 && std::fabs(lambda_next - lambda) <= tol * std::fabs(lambda_next)) {
      lambda = lambda_next;
      break;
    }
    lambda = lambda_next;
    // v = w / ||w|| on the owned slice, then everywhere
    const double inv = 1.0 / nrm;
    for (auto& sh : shards_) {
      if (sh->p1 <= sh->p0) continue;
      scale_slice_kernel<<<grid1(sh->p1 - sh->p0), 256, 0, st_>>>(sh->nv.get(), sh->nw.get(), inv, sh->p0, sh->p1);
      RB_LAUNCH_CHECK();
    }
    exchange([](Shard& sh) { return sh.nv.get(); }, true);
  }
  RB_CUDA(cudaStreamSynchronize(st_));
  for (auto& sh : shards_) sh->nv.reset(), sh->nw.reset(), sh->nmv.reset();
  return std::sqrt(std::max(lambda, 0.0));
}

void ShardedEngine::build_replicated() {
  if (!nrep_) return;
  DeviceQP& P = *full_->P_;
  const thrust::counting_iterator<int32_t> idx(0);
  for (auto& sh : shards_) {
    DevBuf<int32_t> len(nrep_);
    sh->rep_qlo.alloc(nrep_), sh->rep_qhi.alloc(nrep_), sh->rep_alo.alloc(nrep_), sh->rep_ahi.alloc(nrep_);
    rep_ranges_kernel<<<grid1(nrep_), 256, 0, st_>>>(rep_rows_.get(), nrep_, P.Q.rp.get(), P.Q.ci.get(), sh->p0, sh->p1,
                                                     P.AT.rp.get(), P.AT.ci.get(), sh->d0, sh->d1, sh->rep_qlo.get(),
                                                     sh->rep_qhi.get(), sh->rep_alo.get(), sh->rep_ahi.get(), len.get());
    RB_LAUNCH_CHECK();
    build_schedule(sh->sch_rep, len.get(), nrep_, false, st_);
    sh->rep_part.alloc(static_cast<std::size_t>(parts_) * 2 * nrep_);
    sh->rep_part.zero(st_);
    // the step's primal rows: the owned ones that are not replicated
    const int64_t nl = sh->p1 - sh->p0;
    if (nl <= 0) continue;
    DevBuf<uint8_t> keep(nl);
    invert_kernel<<<grid1(nl), 256, 0, st_>>>(rep_flag_.get() + sh->p0, keep.get(), nl);
    RB_LAUNCH_CHECK();
    DevBuf<int32_t> list(nl), cnt(1), plen;
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx, keep.get(), list.get(), cnt.get(), static_cast<int>(nl), st_));
    DevBuf<unsigned char> tmp(tb);
    RB_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, idx, keep.get(), list.get(), cnt.get(), static_cast<int>(nl), st_));
    int32_t k = 0;
    RB_CUDA(cudaMemcpyAsync(&k, cnt.get(), sizeof(k), cudaMemcpyDeviceToHost, st_));
    RB_CUDA(cudaStreamSynchronize(st_));
    row_lengths(plen, P.Q.rp.get() + sh->p0, P.AT.rp.get() + sh->p0, nl, st_);
    if (k) build_schedule(sh->sch_primal_step, plen.get(), k, false, st_, list.get());
    RB_CUDA(cudaStreamSynchronize(st_));
  }
  if (std::getenv("RAPDHG_TRACE"))
    std::fprintf(stderr, "[shard] %d replicated primal rows\n", nrep_);
}

// The replicated rows' part of primal step `it` (after the dual step, before
// the y exchange: each shard's partials need only the y it computed).
void ShardedEngine::replicated_step(int it, int c) {
  DeviceQP& P = *full_->P_;
  const Engine& e = *full_;
  std::vector<double*> bufs;
  for (auto& sh : shards_) {
    RepPartialOp op{sh->rep_qlo.get(), sh->rep_qhi.get(), sh->rep_alo.get(), sh->rep_ahi.get(),
                    P.Q.ci.get(),      e.qsv_,            P.AT.ci.get(),     e.atsv_,
                    sh->XMD[c].get(),  sh->y.get(),       sh->rep_part.get() + static_cast<int64_t>(sh->id) * 2 * nrep_};
    launch_rowwise(op, sh->sch_rep.view, st_);
    ++launches_;
    bufs.push_back(sh->rep_part.get());
  }
  std::vector<int64_t> bounds(parts_ + 1);
  for (int k = 0; k <= parts_; ++k) bounds[k] = static_cast<int64_t>(k) * 2 * nrep_;
  tr_->allgatherv(bufs, bounds, st_);
  for (auto& sh : shards_) {
    const PrimalStepOp<false> pr{CsrView{}, CsrView{}, nullptr, nullptr, sh->X[c].get(), sh->X[c ^ 1].get(),
                                 sh->xb.get(), e.csv_, sh->w.get(), sh->XMD[c ^ 1].get(), params_.get(), it,
                                 sh->bad.get(), e.lsv_, e.hsv_};
    rep_finish_kernel<<<grid1(nrep_), 256, 0, st_>>>(pr, rep_rows_.get(), sh->rep_part.get(), nrep_, parts_);
    RB_LAUNCH_CHECK();
    ++launches_;
  }
}

// Interior / boundary row lists of each shard's plain-path ops (see Shard).
// Global decision: an op overlaps when it is on the plain path everywhere (no
// slab windows, no column blocks) and parts > 1; by default only with a real
// transport (one process per GPU): emulated shards share one GPU, where the
// exchanges are device copies and splitting the launches only costs (C5-L, 4
// emulated shards: 660 against 718 it/s). RAPDHG_OVERLAP=1 / 0 forces it.
void ShardedEngine::build_overlap(bool emulated) {
  const char* env = std::getenv("RAPDHG_OVERLAP");
  const bool want = env ? env[0] == '1' : !emulated;
  if (!want || parts_ < 2) return;
  const Engine& e = *full_;
  DeviceQP& P = *e.P_;
  overlap_dual_ = e.dual_choice_.empty() && e.cb_nb_dual_ <= 1;
  overlap_primal_ = e.primal_choice_.empty() && e.cb_nq_ <= 1 && e.cb_na_ <= 1 && nrep_ == 0;
  if (!overlap_dual_ && !overlap_primal_) return;
  const thrust::counting_iterator<int32_t> idx(0);
  auto split = [&](int64_t rows, const int32_t* rp1, const int32_t* ci1, int64_t lo1, int64_t hi1,
                   const int32_t* rp2, const int32_t* ci2, int64_t lo2, int64_t hi2, int64_t r0, bool sell,
                   const double* v1, const double* v2, Schedule& s_in, Schedule& s_bd, SellPlan& p_in,
                   SellPlan& p_bd) {
    if (rows <= 0) return;
    DevBuf<uint8_t> flag(rows), inv(rows);
    boundary_kernel<<<grid1(rows), 256, 0, st_>>>(rp1, ci1, lo1, hi1, rp2, ci2, lo2, hi2, r0, rows, flag.get());
    invert_kernel<<<grid1(rows), 256, 0, st_>>>(flag.get(), inv.get(), rows);
    RB_LAUNCH_CHECK();
    DevBuf<int32_t> lst_in(rows), lst_bd(rows), cnt(2), len;
    std::size_t tb = 0;
    RB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx, flag.get(), lst_bd.get(), cnt.get(), static_cast<int>(rows),
                                       st_));
    DevBuf<unsigned char> tmp(tb);
    RB_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, idx, inv.get(), lst_in.get(), cnt.get(), static_cast<int>(rows),
                                       st_));
    RB_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, idx, flag.get(), lst_bd.get(), cnt.get() + 1,
                                       static_cast<int>(rows), st_));
    int32_t n[2] = {0, 0};
    RB_CUDA(cudaMemcpyAsync(n, cnt.get(), sizeof(n), cudaMemcpyDeviceToHost, st_));
    RB_CUDA(cudaStreamSynchronize(st_));
    row_lengths(len, rp1 + r0, rp2 ? rp2 + r0 : nullptr, rows, st_);
    if (sell) {
      if (n[0]) build_sell_plan(p_in, rp1 + r0, ci1, rp2 ? rp2 + r0 : nullptr, ci2, n[0], st_, lst_in.get());
      if (n[1]) build_sell_plan(p_bd, rp1 + r0, ci1, rp2 ? rp2 + r0 : nullptr, ci2, n[1], st_, lst_bd.get());
      fill_sell_values(p_in, v1, v2, st_);
      fill_sell_values(p_bd, v1, v2, st_);
    } else {
      if (n[0]) build_schedule(s_in, len.get(), n[0], false, st_, lst_in.get());
      if (n[1]) build_schedule(s_bd, len.get(), n[1], false, st_, lst_bd.get());
    }
    RB_CUDA(cudaStreamSynchronize(st_));
    overlap_rows_[0] += n[0], overlap_rows_[1] += n[1];
  };
  for (auto& sh : shards_) {
    if (overlap_dual_)
      split(sh->d1 - sh->d0, P.A.rp.get(), P.A.ci.get(), sh->p0, sh->p1, nullptr, nullptr, 0, 0, sh->d0,
            e.sell_dual_, e.asv_, nullptr, sh->sch_dual_in, sh->sch_dual_bd, sh->sell_dual_in, sh->sell_dual_bd);
    if (overlap_primal_)
      split(sh->p1 - sh->p0, P.Q.rp.get(), P.Q.ci.get(), sh->p0, sh->p1, P.AT.rp.get(), P.AT.ci.get(), sh->d0,
            sh->d1, sh->p0, e.sell_primal_, e.qsv_, e.atsv_, sh->sch_primal_in, sh->sch_primal_bd,
            sh->sell_primal_in, sh->sell_primal_bd);
  }
  st2_ = own_st2_.create();
  RB_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  RB_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  if (std::getenv("RAPDHG_TRACE"))
    std::fprintf(stderr, "[shard] overlap dual %d primal %d: interior %lld, boundary %lld rows\n", overlap_dual_,
                 overlap_primal_, static_cast<long long>(overlap_rows_[0]), static_cast<long long>(overlap_rows_[1]));
}

// Halo lists of the three per-step exchanges: w (gathered by the dual rows
// through A, owned by the primal blocks), x_md (primal rows through Q) and y
// (primal rows through A', owned by the dual blocks). For every shard p the
// sorted set of indices its rows reference (a flag pass over its entries + a
// select), cut at the owners' bounds; shard s receives its segments from the
// other owners and sends every peer p the segment of p's set that s owns.
void ShardedEngine::build_halos() {
  const char* env = std::getenv("RAPDHG_HALO");
  const std::string mode = env ? env : "auto";
  halo_.clear();
  halo_.resize(3);
  if (mode == "off" || parts_ < 2) return;
  DeviceQP& P = *full_->P_;
  struct Spec {
    const DevCsr* mat;
    const std::vector<int64_t>* rows;    // row blocks of the shards
    const std::vector<int64_t>* owners;  // owner blocks of the gathered vector
    int64_t N;
  };
  const Spec spec[3] = {{&P.A, &db_, &pb_, P.n}, {&P.Q, &pb_, &pb_, P.n}, {&P.AT, &pb_, &db_, P.m}};
  for (int kind = 0; kind < 3; ++kind) {
    const Spec& sp = spec[kind];
    const int64_t N = sp.N;
    if (N <= 0) continue;
    const std::vector<int64_t>& ob = *sp.owners;
    std::vector<DevBuf<int32_t>> L(parts_);
    std::vector<std::vector<int64_t>> off(parts_, std::vector<int64_t>(parts_ + 1, 0));
    DevBuf<uint8_t> flags(N);
    DevBuf<int32_t> cnt(1);
    DevBuf<int64_t> keys(parts_ + 1), pos(parts_ + 1);
    keys.upload(ob.data(), parts_ + 1, st_);
    const thrust::counting_iterator<int32_t> idx(0);
    std::size_t tmp_bytes = 0;
    RB_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, idx, flags.get(), static_cast<int32_t*>(nullptr), cnt.get(),
                                       static_cast<int>(N), st_));
    DevBuf<unsigned char> tmp(tmp_bytes);
    int64_t moved = 0, gathered = 0;
    for (int p = 0; p < parts_; ++p) {
      flags.zero(st_);
      const int64_t r0 = (*sp.rows)[p], r1 = (*sp.rows)[p + 1];
      if (r1 > r0) {
        if (nrep_ && kind != kHaloW)  // primal rows: the replicated ones gather nothing remote
          halo_mark_rows_kernel<<<8 * kSMs, 256, 0, st_>>>(sp.mat->rp.get(), sp.mat->ci.get(), r0, r1,
                                                           rep_flag_.get(), flags.get());
        else
          halo_mark_kernel<<<4 * kSMs, 256, 0, st_>>>(sp.mat->rp.get(), sp.mat->ci.get(), r0, r1, flags.get());
        RB_LAUNCH_CHECK();
      }
      if (nrep_ && kind != kHaloY) {  // w / x_md of the replicated rows are on every shard
        clear_listed_kernel<<<grid1(nrep_), 256, 0, st_>>>(flags.get(), rep_rows_.get(), nrep_);
        RB_LAUNCH_CHECK();
      }
      L[p].alloc(N);
      RB_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tmp_bytes, idx, flags.get(), L[p].get(), cnt.get(),
                                         static_cast<int>(N), st_));
      lower_bounds_kernel<<<1, static_cast<unsigned>((parts_ + 32) / 32 * 32), 0, st_>>>(L[p].get(), cnt.get(), keys.get(),
                                                                                     parts_ + 1, pos.get());
      RB_LAUNCH_CHECK();
      pos.download(off[p].data(), parts_ + 1, st_);
      RB_CUDA(cudaStreamSynchronize(st_));
      for (int j = 0; j < parts_; ++j)
        if (j != p) moved += off[p][j + 1] - off[p][j];
      gathered += N - (ob[p + 1] - ob[p]);
    }
    halo_entries_[kind] = moved;
    halo_on_[kind] = mode == "on" || 2 * moved <= gathered;
    if (!halo_on_[kind]) continue;
    halo_[kind].resize(shards_.size());
    for (std::size_t li = 0; li < shards_.size(); ++li) {
      const int sid = shards_[li]->id;
      HaloSide& h = halo_[kind][li];
      h.recv_off.assign(parts_ + 1, 0);
      h.send_off.assign(parts_ + 1, 0);
      for (int j = 0; j < parts_; ++j) {
        h.recv_off[j + 1] = h.recv_off[j] + (j == sid ? 0 : off[sid][j + 1] - off[sid][j]);
        h.send_off[j + 1] = h.send_off[j] + (j == sid ? 0 : off[j][sid + 1] - off[j][sid]);
      }
      const int64_t nr = h.recv_off[parts_], ns = h.send_off[parts_];
      h.recv_idx.alloc(std::max<int64_t>(nr, 1)), h.recv_buf.alloc(std::max<int64_t>(nr, 1));
      h.send_idx.alloc(std::max<int64_t>(ns, 1)), h.send_buf.alloc(std::max<int64_t>(ns, 1));
      for (int j = 0; j < parts_; ++j) {
        if (j == sid) continue;
        const int64_t cr = h.recv_off[j + 1] - h.recv_off[j], cs = h.send_off[j + 1] - h.send_off[j];
        if (cr > 0)
          RB_CUDA(cudaMemcpyAsync(h.recv_idx.get() + h.recv_off[j], L[sid].get() + off[sid][j], sizeof(int32_t) * cr,
                                  cudaMemcpyDeviceToDevice, st_));
        if (cs > 0)
          RB_CUDA(cudaMemcpyAsync(h.send_idx.get() + h.send_off[j], L[j].get() + off[j][sid], sizeof(int32_t) * cs,
                                  cudaMemcpyDeviceToDevice, st_));
      }
    }
    RB_CUDA(cudaStreamSynchronize(st_));
  }
  if (std::getenv("RAPDHG_TRACE"))
    std::fprintf(stderr, "[shard] halo (w, x_md, y): %s %s %s, entries per exchange %lld %lld %lld\n",
                 halo_on_[0] ? "on" : "off", halo_on_[1] ? "on" : "off", halo_on_[2] ? "on" : "off",
                 static_cast<long long>(halo_entries_[0]), static_cast<long long>(halo_entries_[1]),
                 static_cast<long long>(halo_entries_[2]));
}

void ShardedEngine::step_exchange(double* (*pick)(Shard&), HaloKind kind, cudaStream_t st) {
  if (!halo_on_[kind]) {
    std::vector<double*> bufs;
    for (auto& sh : shards_) bufs.push_back(pick(*sh));
    tr_->allgatherv(bufs, kind != kHaloY ? pb_ : db_, st);
    return;
  }
  std::vector<double*> bufs;
  std::vector<HaloSide*> sides;
  for (std::size_t li = 0; li < shards_.size(); ++li) {
    bufs.push_back(pick(*shards_[li]));
    sides.push_back(&halo_[kind][li]);
  }
  tr_->halo(bufs, sides, st);
}

void ShardedEngine::fork() {
  RB_CUDA(cudaEventRecord(ev_fork_, st_));
  RB_CUDA(cudaStreamWaitEvent(st2_, ev_fork_, 0));
}
void ShardedEngine::join() {
  RB_CUDA(cudaEventRecord(ev_join_, st2_));
  RB_CUDA(cudaStreamWaitEvent(st_, ev_join_, 0));
}

ShardedEngine::~ShardedEngine() {
  if (st_) cudaStreamSynchronize(st_);
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
}

void ShardedEngine::solve(rapdhg_result* out, Clock::time_point t0) {
  AllocStreamScope scope(st_);
  const Engine& e = *full_;
  run_loop(*this, cfg_, LoopScalars{e.norm_q, e.norm_a, e.omega0, e.setup_seconds, e.n_, e.mi_, e.m_ - e.mi_},
           out, t0);
}

void ShardedEngine::exchange(double* (*pick)(Shard&), bool primal_space) {
  std::vector<double*> bufs;
  for (auto& sh : shards_) bufs.push_back(pick(*sh));
  tr_->allgatherv(bufs, primal_space ? pb_ : db_, st_);
}

// One deterministic reduction over the primal (n) or dual (m) index space:
// per-shard chunk partials, allgather-v of the partials, fixed combine.
template <int NS, int NM, class MakeF>
void ShardedEngine::reduce(bool primal_space, const MakeF& make, double* out_host) {
  constexpr int NT = NS + NM;
  const std::vector<int64_t>& b = primal_space ? pb_ : db_;
  const int64_t total = b.back();
  if (total == 0) {
    for (int k = 0; k < NT; ++k) out_host[k] = 0.0;
    return;
  }
  for (auto& sh : shards_) {
    const int64_t lo = b[sh->id], hi = b[sh->id + 1];
    launch_reduce_partials<NS, NM>(make(*sh, lo), hi - lo, lo / kRedChunk, sh->red, st_);
    ++launches_;
  }
  std::vector<int64_t> cb(parts_ + 1);
  // a shard owns the chunks its first row starts; a bound at `total` (only
  // empty trailing shards) owns none
  for (int k = 0; k < parts_; ++k) cb[k] = (b[k] == total ? reduce_chunks(total) : b[k] / kRedChunk) * NT;
  cb[parts_] = reduce_chunks(total) * NT;
  std::vector<double*> bufs;
  for (auto& sh : shards_) bufs.push_back(sh->red.partials.get());
  tr_->allgatherv(bufs, cb, st_);
  Shard& s0 = *shards_[0];
  launch_reduce_combine<NS, NM>(total, s0.red, s0.red_out.get(), st_);
  ++launches_;
  RB_CUDA(cudaMemcpyAsync(red_h_.get(), s0.red_out.get(), sizeof(double) * NT, cudaMemcpyDeviceToHost, st_));
  RB_CUDA(cudaStreamSynchronize(st_));
  for (int k = 0; k < NT; ++k) out_host[k] = red_h_[k];
}

void ShardedEngine::loop_begin() {
  launches_ = 0;
  cur_ = 0;
  RB_CUDA(cudaEventCreate(&ev0_));
  RB_CUDA(cudaEventCreate(&ev1_));
  RB_CUDA(cudaEventRecord(ev0_, st_));
  const long long big = std::numeric_limits<long long>::max();
  for (auto& sh : shards_) {
    for (auto* buf : {&sh->X[0], &sh->X[1], &sh->xb, &sh->epx, &sh->y, &sh->yb, &sh->epy}) buf->zero(st_);
    RB_CUDA(cudaMemcpyAsync(sh->bad.get(), &big, sizeof(big), cudaMemcpyHostToDevice, st_));
  }
  RB_CUDA(cudaStreamSynchronize(st_));
}

void ShardedEngine::body(int len, int cur) {
  DeviceQP& P = *full_->P_;
  const Engine& e = *full_;
  // chunk prologue: w and x_md of the first step on each slice, then exchange
  for (auto& sh : shards_) {
    const int64_t nl = sh->p1 - sh->p0;
    if (nl > 0) {
      prologue_kernel<<<grid1(nl), 256, 0, st_>>>(sh->X[cur].get() + sh->p0, sh->X[cur ^ 1].get() + sh->p0,
                                                  sh->xb.get() + sh->p0, sh->w.get() + sh->p0,
                                                  sh->XMD[cur].get() + sh->p0, params_.get(), static_cast<int>(nl));
      RB_LAUNCH_CHECK();
      ++launches_;
    }
  }
  if (nrep_)
    for (auto& sh : shards_) {
      rep_prologue_kernel<<<grid1(nrep_), 256, 0, st_>>>(rep_rows_.get(), nrep_, sh->X[cur].get(),
                                                         sh->X[cur ^ 1].get(), sh->xb.get(), sh->w.get(),
                                                         sh->XMD[cur].get(), params_.get());
      RB_LAUNCH_CHECK();
      ++launches_;
    }
  // the w / x_md exchange feeding step `it`: on st2_ beside the interior dual
  // rows when the dual overlaps, else in line on st_
  auto exchange_wx = [&](int c_md) {
    cudaStream_t s = overlap_dual_ ? st2_ : st_;
    if (overlap_dual_) fork();
    step_exchange([](Shard& sh) { return sh.w.get(); }, kHaloW, s);
    if (c_md == 0) step_exchange([](Shard& sh) { return sh.XMD[0].get(); }, kHaloX, s);
    else step_exchange([](Shard& sh) { return sh.XMD[1].get(); }, kHaloX, s);
  };
  exchange_wx(cur);
  for (int it = 0; it < len; ++it) {
    const int c = (cur + it) & 1;
    // dual step; part: 0 all rows, 1 interior rows, 2 boundary rows
    auto dual = [&](int part) {
      for (auto& sh : shards_) {
        if (sh->d1 <= sh->d0) continue;
        DualStepOp<false> d{CsrView{P.A.rp.get() + sh->d0, P.A.ci.get(), e.asv_}, sh->w.get(), e.bsv_ + sh->d0,
                            sh->y.get() + sh->d0, sh->yb.get() + sh->d0, e.mi_ - static_cast<int>(sh->d0),
                            params_.get(), it, sh->bad.get()};
        if (part) {
          const SellPlan& sp = part == 1 ? sh->sell_dual_in : sh->sell_dual_bd;
          const Schedule& sc = part == 1 ? sh->sch_dual_in : sh->sch_dual_bd;
          if (sp.active()) launch_sell(d, sp, st_), ++launches_;
          else if (sc.view.total_blocks > 0) launch_rowwise(d, sc.view, st_), ++launches_;
        } else if (sh->dual_ph.active()) {
          launches_ += launch_slab_phase(d, sh->dual_ph, st_);
        } else if (sh->cbd.active()) {
          launches_ += launch_colblocked_dual(d, sh->cbd, st_);
        } else if (sh->sell_dual.active()) {
          launch_sell(d, sh->sell_dual, st_);
          ++launches_;
        } else {
          launch_rowwise(d, sh->sch_dual.view, st_);
          ++launches_;
        }
      }
    };
    auto primal = [&](int part) {
      for (auto& sh : shards_) {
        if (sh->p1 <= sh->p0) continue;
        const int64_t o = sh->p0;
        PrimalStepOp<false> pr{CsrView{P.Q.rp.get() + o, P.Q.ci.get(), e.qsv_},
                               CsrView{P.AT.rp.get() + o, P.AT.ci.get(), e.atsv_},
                               sh->XMD[c].get(), sh->y.get(), sh->X[c].get() + o, sh->X[c ^ 1].get() + o,
                               sh->xb.get() + o, e.csv_ + o, sh->w.get() + o, sh->XMD[c ^ 1].get() + o,
                               params_.get(), it, sh->bad.get(), e.lsv_ ? e.lsv_ + o : nullptr,
                               e.hsv_ ? e.hsv_ + o : nullptr};
        if (part) {
          const SellPlan& sp = part == 1 ? sh->sell_primal_in : sh->sell_primal_bd;
          const Schedule& sc = part == 1 ? sh->sch_primal_in : sh->sch_primal_bd;
          if (sp.active()) launch_sell(pr, sp, st_), ++launches_;
          else if (sc.view.total_blocks > 0) launch_rowwise(pr, sc.view, st_), ++launches_;
        } else if (sh->primal_ph.active()) {
          launches_ += launch_slab_phase(pr, sh->primal_ph, st_);
        } else if (sh->cbp.active()) {
          launches_ += launch_colblocked_primal(pr, sh->cbp, st_);
        } else if (sh->sell_primal.active()) {
          launch_sell(pr, sh->sell_primal, st_);
          ++launches_;
        } else {
          launch_rowwise(pr, (nrep_ ? sh->sch_primal_step : sh->sch_primal).view, st_);
          ++launches_;
        }
      }
    };
    if (overlap_dual_) {  // interior rows beside the w / x_md exchange, then the rest
      dual(1);
      join();
      dual(2);
    } else {
      dual(0);
    }
    if (nrep_) replicated_step(it, c);
    if (overlap_primal_) {  // the y exchange beside the interior primal rows
      fork();
      step_exchange([](Shard& sh) { return sh.y.get(); }, kHaloY, st2_);
      primal(1);
      join();
      primal(2);
    } else {
      step_exchange([](Shard& sh) { return sh.y.get(); }, kHaloY, st_);
      primal(0);
    }
    if (it + 1 < len) exchange_wx(c ^ 1);  // the next step gathers the new w and x_md
  }
}

void ShardedEngine::run_chunk(int len) {
  params_.upload(params_h_.get(), len, st_);
  if (cfg_.use_graphs && tr_->capturable()) {
    const int key = (len << 1) | cur_;
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
      const int64_t before = launches_;
      const cudaGraphExec_t ge = capture_graph(st_, [&] { body(len, cur_); });
      const int64_t per_replay = launches_ - before;
      launches_ = before;
      it = graphs_.emplace(key, ge).first;
      replay_launches_[key] = per_replay;
    }
    RB_CUDA(cudaGraphLaunch(it->second, st_));
    launches_ += replay_launches_[key];
  } else {
    body(len, cur_);
  }
  cur_ ^= (len & 1);
  RB_CUDA(cudaStreamSynchronize(st_));
}

long long ShardedEngine::first_bad() {
  std::vector<long long*> v;
  for (auto& sh : shards_) v.push_back(sh->bad.get());
  return tr_->allreduce_min(v, st_);
}

bool ShardedEngine::any_rank(bool flag) {
  const long long keep_going = flag ? 0 : 1;  // min over ranks == 0: someone stops
  std::vector<long long*> v;
  for (auto& sh : shards_) {
    RB_CUDA(cudaMemcpyAsync(sh->vote.get(), &keep_going, sizeof(keep_going), cudaMemcpyHostToDevice, st_));
    v.push_back(sh->vote.get());
  }
  return tr_->allreduce_min(v, st_) == 0;
}

Cand ShardedEngine::evaluate() {
  DeviceQP& P = *full_->P_;
  const Engine& e = *full_;
  const int n = e.n_, m = e.m_, mi = e.mi_;
  const double* d = e.d_.get();
  for (auto& sh : shards_) {  // unscale the owned slices (scaling.hpp:126-133)
    const int64_t nl = sh->p1 - sh->p0, ml = sh->d1 - sh->d0;
    if (nl > 0)
      unscale_kernel<<<grid1(nl), 256, 0, st_>>>(sh->X[cur_].get() + sh->p0, sh->xb.get() + sh->p0, nullptr, nullptr,
                                                 d + sh->p0, sh->xu[0].get() + sh->p0, sh->xu[1].get() + sh->p0,
                                                 nullptr, nullptr, static_cast<int>(nl), 0);
    if (ml > 0)
      unscale_kernel<<<grid1(ml), 256, 0, st_>>>(nullptr, nullptr, sh->y.get() + sh->d0, sh->yb.get() + sh->d0,
                                                 d + n + sh->d0, nullptr, nullptr, sh->yu[0].get() + sh->d0,
                                                 sh->yu[1].get() + sh->d0, 0, static_cast<int>(ml));
    RB_LAUNCH_CHECK();
    launches_ += 2;
  }
  exchange([](Shard& s) { return s.xu[0].get(); }, true);
  exchange([](Shard& s) { return s.xu[1].get(); }, true);
  exchange([](Shard& s) { return s.yu[0].get(); }, false);
  exchange([](Shard& s) { return s.yu[1].get(); }, false);
  for (auto& sh : shards_) {  // KKT products on the ORIGINAL matrices, owned rows
    interleave_kernel<<<grid1(n), 256, 0, st_>>>(sh->xu[0].get(), sh->xu[1].get(), sh->xi.get(), n);
    interleave_kernel<<<grid1(m), 256, 0, st_>>>(sh->yu[0].get(), sh->yu[1].get(), sh->yi.get(), m);
    RB_LAUNCH_CHECK();
    launches_ += 2;
    if (sh->d1 > sh->d0) {
      KktAxOp<false> ax{CsrView{P.A.rp.get() + sh->d0, P.A.ci.get(), P.A.v.get()}, sh->xi.get(),
                        sh->ax[0].get() + sh->d0, sh->ax[1].get() + sh->d0};
      launch_rowwise(ax, sh->sch_dual.view, st_);
      ++launches_;
    }
    if (sh->p1 > sh->p0) {
      const int64_t o = sh->p0;
      KktQAtyOp<false> qa{CsrView{P.Q.rp.get() + o, P.Q.ci.get(), P.Q.v.get()},
                          CsrView{P.AT.rp.get() + o, P.AT.ci.get(), P.AT.v.get()}, mi, sh->xi.get(),
                          sh->yi.get(), sh->qx[0].get() + o,
                          sh->qx[1].get() + o, sh->aty[0].get() + o, sh->aty[1].get() + o};
      launch_rowwise(qa, sh->sch_primal.view, st_);
      ++launches_;
    }
  }
  double h[16], g[16];
  const double* b = P.b.get();
  const double* c = P.c.get();
  reduce<4, 5>(false, [&](Shard& s, int64_t lo) {
    return KktDualTerms{s.ax[0].get() + lo, s.ax[1].get() + lo, b + lo, s.yu[0].get() + lo, s.yu[1].get() + lo,
                        mi - static_cast<int>(lo)};
  }, h);
  const double* lob = P.lo.size() ? P.lo.get() : nullptr;
  const double* hib = P.hi.size() ? P.hi.get() : nullptr;
  reduce<kKktPrimalSums, kKktPrimalMaxes>(true, [&](Shard& s, int64_t lo) {
    return KktPrimalTerms{s.qx[0].get() + lo, s.qx[1].get() + lo, s.aty[0].get() + lo, s.aty[1].get() + lo,
                          s.xu[0].get() + lo, s.xu[1].get() + lo, c + lo, lob ? lob + lo : nullptr,
                          hib ? hib + lo : nullptr};
  }, g);
  KktRaw r;
  r.by_i[0] = h[0], r.by_e[0] = h[1], r.by_i[1] = h[2], r.by_e[1] = h[3];
  r.viol[0] = h[4], r.viol[1] = h[5], r.ax_inf[0] = h[6], r.ax_inf[1] = h[7], r.b_inf = h[8];
  primal_terms_into(r, g);
  Kkt k2[2];
  finalize_kkt(r, k2);
  Cand cd;
  cd.cur = k2[0];
  cd.avg = k2[1];
  cd.is_avg = !(cd.cur.relkkt() < cd.avg.relkkt());  // ties -> average
  return cd;
}

void ShardedEngine::keep_best(bool avg) {
  const int i = avg ? 1 : 0;
  for (auto& sh : shards_) {
    const int64_t nl = sh->p1 - sh->p0, ml = sh->d1 - sh->d0;
    if (nl > 0)
      RB_CUDA(cudaMemcpyAsync(sh->best_x.get() + sh->p0, sh->xu[i].get() + sh->p0, sizeof(double) * nl,
                              cudaMemcpyDeviceToDevice, st_));
    if (ml > 0)
      RB_CUDA(cudaMemcpyAsync(sh->best_y.get() + sh->d0, sh->yu[i].get() + sh->d0, sizeof(double) * ml,
                              cudaMemcpyDeviceToDevice, st_));
  }
}

void ShardedEngine::restart(bool from_avg, double* dx, double* dy) {
  for (auto& sh : shards_) {  // solver.hpp:442-448 on the owned slices
    const int64_t nl = sh->p1 - sh->p0, ml = sh->d1 - sh->d0;
    if (nl > 0)
      restart_kernel<<<grid1(nl), 256, 0, st_>>>(sh->X[cur_].get() + sh->p0, sh->X[cur_ ^ 1].get() + sh->p0,
                                                 sh->xb.get() + sh->p0, nullptr, nullptr, from_avg ? 1 : 0,
                                                 static_cast<int>(nl), 0);
    if (ml > 0)
      restart_kernel<<<grid1(ml), 256, 0, st_>>>(nullptr, nullptr, nullptr, sh->y.get() + sh->d0,
                                                 sh->yb.get() + sh->d0, from_avg ? 1 : 0, 0, static_cast<int>(ml));
    RB_LAUNCH_CHECK();
    launches_ += 2;
    if (nrep_) {  // the replicated rows' state is every shard's (idempotent on the owner's)
      rep_restart_kernel<<<grid1(nrep_), 256, 0, st_>>>(rep_rows_.get(), nrep_, sh->X[cur_].get(),
                                                        sh->X[cur_ ^ 1].get(), sh->xb.get(), from_avg ? 1 : 0);
      RB_LAUNCH_CHECK();
      ++launches_;
    }
  }
  const int cur = cur_;
  double sx[1], sy[1];
  reduce<1, 0>(true, [&](Shard& s, int64_t lo) { return DistAndAdvance{s.X[cur].get() + lo, s.epx.get() + lo}; }, sx);
  reduce<1, 0>(false, [&](Shard& s, int64_t lo) { return DistAndAdvance{s.y.get() + lo, s.epy.get() + lo}; }, sy);
  *dx = std::sqrt(sx[0]);
  *dy = std::sqrt(sy[0]);
}

void ShardedEngine::download(int src, double* x, double* y) {
  Shard& s0 = *shards_[0];
  const double *xs, *ys;
  if (src == 2) {
    exchange([](Shard& s) { return s.best_x.get(); }, true);
    exchange([](Shard& s) { return s.best_y.get(); }, false);
    xs = s0.best_x.get(), ys = s0.best_y.get();
  } else {  // the unscaled candidates were exchanged by evaluate()
    xs = s0.xu[src].get(), ys = s0.yu[src].get();
  }
  const int64_t n = pb_.back(), m = db_.back();
  if (n) RB_CUDA(cudaMemcpyAsync(x, xs, sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
  if (m) RB_CUDA(cudaMemcpyAsync(y, ys, sizeof(double) * m, cudaMemcpyDeviceToHost, st_));
  RB_CUDA(cudaStreamSynchronize(st_));
}

void ShardedEngine::loop_end(rapdhg_result* out) {
  RB_CUDA(cudaEventRecord(ev1_, st_));
  RB_CUDA(cudaEventSynchronize(ev1_));
  float ms = 0.f;
  RB_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
  cudaEventDestroy(ev0_);
  cudaEventDestroy(ev1_);
  out->loop_seconds = 1e-3 * ms;
  out->kernel_launches = full_->P_->launches + launches_;
}

}  // namespace rb
