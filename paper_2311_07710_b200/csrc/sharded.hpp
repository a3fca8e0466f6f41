// sharded.hpp — row-sharded multi-GPU rAPDHG.
//
// Rank k owns a contiguous block of the dual rows (rows of A = [A_ineq; A_eq])
// and a contiguous block of the primal rows (rows of [Q | A']), balanced by
// nnz and aligned to kRedChunk so the chunked reductions (reduce.cuh) see the
// same chunks as on one GPU. Every rank runs the full setup (validation,
// scaling, norms: identical on every rank), then iterates on its row blocks
// only: shard matrices are zero-copy row views of the set-up matrices.
//
// Per inner step the exchange is one allgather-v of y (after the dual step)
// and one of w and x_md (after the primal step, except on a chunk's last
// step); checks exchange the unscaled points and the reduction partials. Each
// row is computed exactly as on one GPU (same row, same length, same lanes),
// and reductions combine the same chunk partials in the same order, so a
// sharded solve is BIT-IDENTICAL to the single-GPU fast-mode solve.
//
// Transports: Emulated (all shards in one process on one GPU; exchanges are
// D2D copies of the owner's slice into every other shard's buffer — used to
// test the sharded path on a single B200) and NCCL (one process per GPU;
// allgather-v as grouped in-place ncclBroadcast from each owner; libnccl is
// dlopen'ed on first use).
#pragma once

#include <memory>
#include <vector>

#include "engine.hpp"

namespace rb {

struct ShardPlan {
  std::vector<int32_t> dual;        // parts + 1 bounds over [0, m)
  std::vector<int32_t> primal;      // parts + 1 bounds over [0, n)
  std::vector<int32_t> replicated;  // dense primal rows computed on every shard (sorted)
};

// nnz-balanced contiguous blocks; inner bounds are multiples of kRedChunk.
// replicate_min_len > 0: the rows of [Q | A'] with at least that many entries
// are replicated (SURVEY §8(e) "dense-coupling columns"): every shard sums
// their entries on its own columns and the partial sums are exchanged, so
// they cost no primal-block balance and no y exchange (see ShardedEngine).
ShardPlan make_shard_plan(const rapdhg_qp& p, int parts, int64_t replicate_min_len = 0);
// RAPDHG_REPLICATE_MIN_LEN (0 / unset: no replication)
int64_t replicate_min_len_from_env();

// Halo exchange of one gathered vector: per local shard, the
// entries its rows reference that other shards own (recv_idx, grouped by owner,
// ascending) and the owned entries each peer references (send_idx, grouped by
// peer) — every rank derives both from the full patterns it holds, so no
// metadata is exchanged. Values travel packed (send_buf / recv_buf).
struct HaloSide {
  DevBuf<int32_t> recv_idx, send_idx;
  std::vector<int64_t> recv_off, send_off;  // parts + 1 each
  DevBuf<double> recv_buf, send_buf;
};

class Transport {
 public:
  virtual ~Transport() = default;
  // false: the exchanges synchronise with the host (host-staged transport),
  // so the chunk cannot be captured into a CUDA graph
  virtual bool capturable() const { return true; }
  // After the call, bufs[s] holds every entry sides[s]->recv_idx names
  // (from its owner); other non-owned entries are left as they were.
  virtual void halo(const std::vector<double*>& bufs, const std::vector<HaloSide*>& sides, cudaStream_t st) = 0;
  // After the call, bufs[s] (one per LOCAL shard) holds every owner's slice
  // [bounds[k], bounds[k+1]) of the vector (elements of 8 bytes).
  virtual void allgatherv(const std::vector<double*>& bufs, const std::vector<int64_t>& bounds,
                          cudaStream_t st) = 0;
  // Minimum over all shards of one int64 per local shard, returned to host.
  virtual long long allreduce_min(const std::vector<long long*>& vals, cudaStream_t st) = 0;
};

std::unique_ptr<Transport> make_emulated_transport(int parts);
// NCCL communicator for `rank` of `parts` from a 128-byte ncclUniqueId.
std::unique_ptr<Transport> make_nccl_transport(int parts, int rank, const void* unique_id);
void nccl_unique_id(void* out128);
// The caller's collectives as host callbacks (rapdhg_host_transport).
std::unique_ptr<Transport> make_host_transport(int parts, int rank, const rapdhg_host_transport& t);
// Host-only self-check of a host transport's callbacks (rapdhg_host_transport_check).
void host_transport_check(const rapdhg_host_transport& t, int parts, int rank, int64_t len);

class ShardedEngine : public LoopBackend {
 public:
  // rank < 0: emulate all `parts` shards in this process; else own shard `rank`.
  // replicate_min_len: see rapdhg_shard_opts (0: RAPDHG_REPLICATE_MIN_LEN)
  ShardedEngine(const rapdhg_qp& p, const rapdhg_config& cfg, int parts, int rank,
                std::unique_ptr<Transport> tr, Clock::time_point t0, int64_t replicate_min_len = 0);
  ~ShardedEngine() override;
  void solve(rapdhg_result* out, Clock::time_point t0);

  void loop_begin() override;
  IterParams* host_params() override { return params_h_.get(); }
  void run_chunk(int len) override;
  long long first_bad() override;
  Cand evaluate() override;
  void keep_best(bool avg) override;
  void restart(bool from_avg, double* dx, double* dy) override;
  void download(int src, double* x, double* y) override;
  void loop_end(rapdhg_result* out) override;
  bool any_rank(bool flag) override;

  const ShardPlan& plan() const { return plan_; }
  bool halo_on(int kind) const { return halo_on_[kind]; }

 private:
  struct Shard;
  void body(int len, int cur);
  // Replicated dense primal rows (plan_.replicated, nrep_ of them): every
  // shard sums each such row's entries on the columns it owns (Q: its primal
  // block, A': its dual block — the y it has just computed), the 2 * nrep_
  // partial sums of all shards are allgathered and added in shard order, and
  // every shard runs the rows' epilogue, so x, x_bar, w and x_md of those rows
  // are the same bits everywhere and never travel. Deterministic for a given
  // shard count; the sums' association differs from one GPU's (not a parity
  // mode: iterates agree to rounding, see tests/test_gpu_shard.py).
  void build_replicated();
  void replicated_step(int it, int c);
  // estimate_op_norm on A (opnorm.hpp:36-61) over the shards: each step's
  // products on the owned rows (rowwise, then from the same switch step as
  // one GPU the shards' slab phases), allgathers of A v and of the normalised
  // v, and the chunked reduction of (v.w, w.w) — the single-GPU estimate
  // bit for bit (rows, chunks and combine as there), without any rank
  // building plans over all rows or computing all products
  // (RAPDHG_SHARD_NORMS=0: every rank runs the single-GPU estimate)
  double distributed_norm_a(int max_iters, double tol, uint64_t seed);
  bool shard_norms_ = true;
  int32_t nrep_ = 0;
  DevBuf<int32_t> rep_rows_;
  DevBuf<uint8_t> rep_flag_;  // n: 1 on replicated rows
  void exchange(double* (*pick)(Shard&), bool primal_space);  // allgather-v on st_
  // per-step exchanges: the halo of the gathered entries when that moves at
  // most half of an allgather (RAPDHG_HALO=on|off|auto), else the allgather
  enum HaloKind { kHaloW = 0, kHaloX = 1, kHaloY = 2 };
  void build_halos();
  void build_overlap(bool emulated);
  void step_exchange(double* (*pick)(Shard&), HaloKind kind, cudaStream_t st);
  // plain-path overlap (build_overlap): the exchanges on st2_ beside the
  // interior rows on st_
  bool overlap_dual_ = false, overlap_primal_ = false;
  int64_t overlap_rows_[2] = {0, 0};
  OwnedStream own_st2_;
  cudaStream_t st2_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  void fork();  // st2_ waits for st_
  void join();  // st_ waits for st2_
  bool halo_on_[3] = {false, false, false};
  std::vector<std::vector<HaloSide>> halo_;  // [kind][local shard]
  int64_t halo_entries_[3] = {0, 0, 0};      // entries moved per exchange (all shards)
  template <int NS, int NM, class MakeF>
  void reduce(bool primal_space, const MakeF& make, double* out_host);

  rapdhg_config cfg_;
  std::unique_ptr<Engine> full_;  // the set-up problem (matrices, scaling, norms)
  ShardPlan plan_;
  int parts_;
  std::vector<std::unique_ptr<Shard>> shards_;  // local shards
  std::unique_ptr<Transport> tr_;
  cudaStream_t st_ = nullptr;
  int cur_ = 0;
  std::vector<int64_t> pb_, db_;  // primal / dual bounds as int64
  DevBuf<IterParams> params_;
  PinnedBuf<IterParams> params_h_;
  PinnedBuf<double> red_h_;
  ReduceScratch red_;  // partials over the full index space (chunks)
  std::map<int, cudaGraphExec_t> graphs_;
  std::map<int, int64_t> replay_launches_;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  int64_t launches_ = 0;
  SyncBeforeFree sync_{&st_, &st2_};  // last member: runs first on destruction
};

}  // namespace rb
