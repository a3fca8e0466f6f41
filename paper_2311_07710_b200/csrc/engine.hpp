// engine.hpp — host-side driver of the B200 rAPDHG solver.
//
// DeviceQP: the problem resident in HBM (original CSRs, stacked A, its
// transpose, schedules) plus the setup numerics (scaling, power iteration).
// Engine: a DeviceQP after the full solve() setup (solver.hpp:277-300), and the
// iteration loop (solver.hpp:318-471) driven as CUDA-graph chunks of at most
// kMaxChunk iterations with one host synchronisation per chunk.
#pragma once

#include <atomic>
#include <chrono>
#include <future>
#include <map>
#include <memory>
#include <random>
#include <utility>
#include <vector>

#include "device_csr.cuh"
#include "ops.cuh"
#include "reduce.cuh"
#include "rowwise.cuh"
#include "colblock.cuh"
#include "slab.cuh"
#include "sell.cuh"

namespace rb {

constexpr int kMaxChunk = 64;
constexpr int kProfilePeriod = 32;  // profile_kernels: time every 32nd chunk (events between
                                    // the steps cost the programmatic overlap of that chunk)

using Clock = std::chrono::steady_clock;

struct Kkt {
  double r_primal = 0.0, r_dual = 0.0, r_gap = 0.0;
  double relkkt() const {
    double m = r_primal;
    if (m < r_dual) m = r_dual;
    if (m < r_gap) m = r_gap;
    return m;  // std::max({r_primal, r_dual, r_gap}) (kkt.hpp:16)
  }
};

// Raw reduction outputs of one relKKT evaluation of two points (c, a).
struct KktRaw {
  double by_i[2], by_e[2], viol[2], ax_inf[2], b_inf;
  double xqx[2], cx[2], dn[2], qx_inf[2], aty_inf[2], c_inf;
  double bl[2] = {0.0, 0.0}, bu[2] = {0.0, 0.0};  // box_projection: l.max(g,0), u.min(g,0)
};
void finalize_kkt(const KktRaw& r, Kkt out[2]);  // kkt.hpp:54,63,68-69
// the KktPrimalTerms reduction outputs (kKktPrimalSums sums, then maxes) into r
void primal_terms_into(KktRaw& r, const double* g);

// The final point of a solve (x | y_ineq | y_eq in one block): pinned when
// large. result_block_free returns false for pointers it did not hand out.
void* result_block_alloc(std::size_t bytes);
bool result_block_free(void* p);

// The power iterations' random start (opnorm.hpp:20-30): `len` draws of
// mt19937_64(seed), and the generator after them (for the zero-norm restarts).
// Norm Q and norm A both start from mt19937_64(cfg.seed) over n entries, so
// one draw, made on a host thread while the matrices upload, serves both.
struct RandomStart {
  std::vector<double> v;
  std::mt19937_64 rng;
};
RandomStart draw_random_start(int len, uint64_t seed);

class DeviceQP {
 public:
  // check_structure: run the per-row CSR checks of validate_dims on the
  // device after the upload (validate_dims(p, false) ran on the host).
  DeviceQP(const rapdhg_qp& p, bool strict, cudaStream_t st, bool check_structure = false);

  // QuadraticProgram::validate (problem.hpp:40-50): throws invalid_argument.
  // structure = false: shapes and row_ptr endpoints only (the per-row scan is
  // left to the device, see the constructor).
  static void validate_dims(const rapdhg_qp& p, bool structure = true);
  void validate_symmetry();

  // compute_scaling / ruiz_scaling (scaling.hpp:85-106). d: n + m factors
  // (d2 = d[0:n], d1 = d[n:]).
  void compute_scaling(int ruiz_iters, bool full, DevBuf<double>& d);
  // apply_scaling (scaling.hpp:109-123) into value arrays with the original
  // patterns; d as above.
  void scale_values(const double* d, DevBuf<double>& qs, DevBuf<double>& as, DevBuf<double>& ats,
                    DevBuf<double>& cs, DevBuf<double>& bs);
  // estimate_op_norm_symmetric / estimate_op_norm (opnorm.hpp:36-87) on the
  // given values (patterns of Q / A / A').
  // pre: the draws of mt19937_64(seed) over n entries (draw_random_start), or
  // null to draw them here
  // on / rs: run on that stream with that scratch (norm Q beside norm A)
  double op_norm_q(const double* qv, int max_iters, double tol, uint64_t seed, const RandomStart* pre = nullptr,
                   cudaStream_t on = nullptr, ReduceScratch* rs = nullptr);
  double op_norm_a(const double* av, const double* atv, int max_iters, double tol, uint64_t seed,
                   const RandomStart* pre = nullptr);

  // Deterministic reduction to host (strict: sequential).
  template <int NS, int NM, class F>
  void reduce_to_host(const F& f, int64_t n, double* out);

  // Launch helpers for plain products with given values.
  void spmv(const DevCsr& m, const Schedule& s, const double* vals, const double* x, double* y,
            StepGate gate = {}, cudaStream_t on = nullptr);

  cudaStream_t st;
  bool strict;
  int n, mi, me, m;
  DevCsr Q, A, AT;  // original values; A = [A_ineq; A_eq]
  DevBuf<int32_t> at_perm;  // AT position -> A position
  DevBuf<double> c, b;      // original c and stacked b
  DevBuf<double> lo, hi;    // variable bounds (box_projection; empty = none)
  Schedule sch_dual;    // rows of A
  Schedule sch_primal;  // rows of [Q | A']
  Schedule sch_q;       // rows of Q
  Schedule sch_at;      // rows of A'
  ReduceScratch red;
  DevBuf<double> red_out;
  PinnedBuf<double> red_host;
  std::atomic<int64_t> launches{0};  // (norm Q counts from its own host thread)
};

// relKKT of the current iterate and of the average at one check
// (evaluate_candidate, solver.hpp:255-264): the candidate is the smaller,
// ties to the average.
struct Cand {
  Kkt cur, avg;
  bool is_avg = true;
  const Kkt& res() const { return is_avg ? avg : cur; }
};

// Device side of the iteration loop. run_loop() (the host controller:
// chunk planning, checks, restarts — solver.hpp:293-471) drives any backend:
// the single-GPU Engine or the row-sharded ShardedEngine (sharded.cu).
class LoopBackend {
 public:
  virtual ~LoopBackend() = default;
  virtual void loop_begin() = 0;          // zero state (solver.hpp:293), start timers
  virtual IterParams* host_params() = 0;  // kMaxChunk pinned entries
  virtual void run_chunk(int len) = 0;    // len inner steps with host_params()[0..len)
  virtual long long first_bad() = 0;      // first non-finite iteration (sticky), syncs
                                          // (after evaluate(): may reuse its read-back)
  virtual Cand evaluate() = 0;            // unscale + relKKT of current and average
  virtual void keep_best(bool avg) = 0;   // best <- that candidate's unscaled point
  virtual void restart(bool from_avg, double* dx, double* dy) = 0;  // + dist2 for omega
  virtual void download(int src, double* x, double* y) = 0;  // 0 cur, 1 avg, 2 best
  virtual void loop_end(rapdhg_result* out) = 0;  // loop time, launch counts
  // Collective OR of a host decision taken at a check (the time limit): every
  // rank must leave the loop at the same check, or their collectives diverge.
  virtual bool any_rank(bool flag) { return flag; }
};

struct LoopScalars {
  double norm_q, norm_a, omega0, setup_seconds;
  int n, mi, me;
};

void run_loop(LoopBackend& be, const rapdhg_config& cfg, const LoopScalars& sc, rapdhg_result* out,
              Clock::time_point t0);

class ShardedEngine;

// The step at which the fast-mode norm estimate of A moves from the rowwise
// SpMV to the slab phases (RAPDHG_NORM_SLAB_STEP, default kNormSlabStep; -1 =
// never). Shared by Engine::norm_a_power and the sharded solver's distributed
// estimate, which must switch at the same step to produce the same bits.
constexpr int kNormSlabStep = 40;
int norm_slab_step();

class Engine : public LoopBackend {
 public:
  // full_plans = false (the sharded solver's setup): the slab phases over all
  // rows serve the norm estimate only (then dropped: the shards rebuild them
  // over their own rows) and no column blocks are built.
  // own_norm_a = false (the sharded solver with distributed norms): the norm of A
  // is left to the caller (ShardedEngine::distributed_norm_a), and with
  // full_plans = false no slab phases over all rows are built at all.
  Engine(const rapdhg_qp& p, const rapdhg_config& cfg, Clock::time_point t0, bool full_plans = true,
         bool own_norm_a = true);
  ~Engine() override;
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // Runs the iteration loop from the zero start (solver.hpp:293-471) and fills
  // out (library-owned arrays). t0: the clock solve_seconds is measured from.
  void solve(rapdhg_result* out, Clock::time_point t0);

  double setup_seconds = 0.0;
  double norm_q = 0.0, norm_a = 0.0, omega0 = 1.0;
  // algorithmic bytes
  double bytes_iter() const;
  double bytes_dual() const;
  double bytes_primal() const;

  // LoopBackend
  void loop_begin() override;
  IterParams* host_params() override { return params_h_.get(); }
  void run_chunk(int len) override;
  long long first_bad() override;
  Cand evaluate() override;
  void keep_best(bool avg) override;
  void restart(bool from_avg, double* dx, double* dy) override;
  void download(int src, double* x, double* y) override;
  void loop_end(rapdhg_result* out) override;

 private:
  friend class ShardedEngine;
  // the streams outlive every buffer below (declared first, destroyed last)
  OwnedStream own_st_, own_st2_;
  void launch_chunk_body(int len, int cur, bool prof);
  void download_point(const double* xu, const double* yu, double* x, double* y);
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  // fast-mode checks: the primal-side KKT product and its reduction run on a
  // second stream beside the dual side (each alone is latency-bound)
  cudaStream_t st2_ = nullptr;
  cudaEvent_t evf_ = nullptr, evj_ = nullptr;
  ReduceScratch red2_;

  rapdhg_config cfg_;
  std::unique_ptr<DeviceQP> P_;
  cudaStream_t st_ = nullptr;
  int n_, m_, mi_;
  // scaled problem (values share the original patterns)
  DevBuf<double> d_;  // n + m scaling factors (d2 then d1)
  DevBuf<double> qs_, as_, ats_, cs_, bs_;
  const double *qsv_, *asv_, *atsv_, *csv_, *bsv_;
  // box_projection: bounds in the scaled space (l / d2, u / d2) for the
  // primal step's projection; null when absent
  DevBuf<double> los_, his_;
  const double *lsv_ = nullptr, *hsv_ = nullptr;
  // iterate state (scaled)
  DevBuf<double> X_[2], XMD_[2], w_, xb_, y_, yb_, epx_, epy_;
  int cur_ = 0;
  // check workspace (unscaled)
  DevBuf<double> xu_[2], yu_[2], ax_[2], qx_[2], aty_[2], best_x_, best_y_;
  DevBuf<double2> xi_, yi_;  // (current, average) interleaved for the KKT products
  // per-chunk params
  DevBuf<IterParams> params_;
  PinnedBuf<IterParams> params_h_;
  DevBuf<long long> bad_;
  PinnedBuf<long long> bad_h_;
  bool bad_fresh_ = false;  // bad_h_ was read back by the last evaluate()
  // slab-staged gathers (fast mode, slab.cuh): plans + the complement schedules
  void setup_slabs();  // idempotent (the norm estimate may run it first)
  void setup_chunk_kernel();
  int chunk_grid_ = 0;  // > 0: chunks run as one cooperative launch of that grid (persistent.cuh)
  // the plain path's step kernels as programmatic dependent launches
  // (RAPDHG_PDL, as the slab kernels)
  bool plain_pdl_ = pdl_enabled();
  void plan_slabs_async();
  bool slabs_ready_ = false;
  double norm_a_power(int max_iters, double tol, uint64_t seed, const RandomStart* pre);
  std::future<void> plan_future_, plan_future2_;
  std::future<RandomStart> rand_future_;  // the power iterations' start, drawn during the upload
  SlabChoice dual_choice_, primal_choice_;
  SlabPhase dual_ph_, primal_ph_;
  // L2-sized column blocks (colblock.cuh) of the gather-bound ops without a slab plan
  void setup_colblocks();
  // column-block counts of the ops without an active slab phase
  void colblock_counts(bool dual_slab_active, bool primal_slab_active);
  bool full_plans_ = true;
  bool own_norm_a_ = true;  // this object estimates norm A (else the sharded solver does)
  int cb_nb_dual_ = 1, cb_nq_ = 1, cb_na_ = 1;  // block counts (global: shards reuse them)
  // sliced-ELL (sell.cuh) for ops whose rows are all short — decided on the
  // whole matrices (shards reuse the decision); plans of the plain path
  bool sell_dual_ = false, sell_primal_ = false;
  SellPlan sell_dual_plan_, sell_primal_plan_;
  ColBlockedDual cbd_;
  ColBlockedPrimal cbp_;

  std::map<int, cudaGraphExec_t> graphs_;  // key: len, parity, profiled
  std::map<int, int64_t> graph_launches_;
  int64_t chunk_counter_ = 0;
  std::vector<cudaEvent_t> events_;
  // profile_kernels = 2: in-loop step times from the slab kernels' start
  // stamps (no events between the steps, so the programmatic overlap stays)
  bool span_mode_ = false;
  DevBuf<unsigned long long> span_;
  double kernel_ms_[2] = {0, 0};
  int64_t kernel_count_[2] = {0, 0};
  int64_t launches_ = 0;
  SyncBeforeFree sync_{&st_, &st2_};  // last member: runs first on destruction
};

// ---- secondary API helpers (host buffers in/out) ----------------------------
void api_validate(const rapdhg_qp& p);              // problem.hpp:40-50
double api_symmetry_gap(const rapdhg_csr& m);        // sparse.hpp:119-138
void api_spmv(const rapdhg_csr& m, const double* x, double* y, bool transpose, bool strict);
void api_rel_kkt(const rapdhg_qp& p, const double* x, const double* yi, const double* ye,
                 bool strict, Kkt* out);
void api_inner_step(const rapdhg_qp& p, rapdhg_iterate* s, const rapdhg_step_params& sp,
                    int steps, bool strict);
void api_scaling(const rapdhg_qp& p, int ruiz_iters, bool full, double* d1, double* d2,
                 bool strict);
void api_apply_scaling(const rapdhg_qp& p, const double* d1, const double* d2, double* qv,
                       double* aiv, double* aev, double* c, double* bi, double* be);
double api_op_norm(const rapdhg_csr& m, bool symmetric, int max_iters, double tol, uint64_t seed,
                   bool strict);

}  // namespace rb
