// capi.cu — extern "C" entry points declared in include/rapdhg_b200.h.
// Exceptions never cross the boundary: each call returns a code and leaves the
// message in rapdhg_last_error() (thread-local).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <new>
#include <string>

#include "engine.hpp"
#include "rules.hpp"
#include "sharded.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return RAPDHG_OK;
  } catch (const rb::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return RAPDHG_E_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RAPDHG_E_INTERNAL;
  }
}

}  // namespace
extern "C" void rapdhg_result_free(rapdhg_result* r);
namespace {

// Entry points that fill a rapdhg_result: `out` starts zeroed, and on any
// error its partly filled arrays are released again, so a failed call leaves
// nothing to free.
template <typename F>
int result_guard(rapdhg_result* out, F&& f) {
  if (out) std::memset(out, 0, sizeof(*out));
  const int rc = guard(std::forward<F>(f));
  if (rc != RAPDHG_OK && out) rapdhg_result_free(out);
  return rc;
}

void require_device() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();  // clear the sticky "no device" error
    throw rb::Error(RAPDHG_E_NO_DEVICE,
                    "no CUDA device visible: the B200 solver has no CPU fallback");
  }
}

void null_check(const void* p, const char* what) {
  if (!p) rb::invalid(std::string("null argument: ") + what);
}

}  // namespace

// shared with host.cpp
void rb_set_error(const char* msg) { g_err = msg; }

struct rapdhg_session {
  rapdhg_config cfg;
  std::unique_ptr<rb::Engine> engine;
};

extern "C" {

const char* rapdhg_last_error(void) { return g_err.c_str(); }
int rapdhg_abi_version(void) { return RAPDHG_ABI_VERSION; }

int rapdhg_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return count;
}

void rapdhg_config_default(rapdhg_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->algorithm = RAPDHG_ALG_APDHG;
  c->restart = RAPDHG_RESTART_PDQP;
  c->restart_length = 0;
  c->step_rule = RAPDHG_STEP_ADAPTIVE;
  c->primal_weight = RAPDHG_PW_ADAPTIVE;
  c->fixed_primal_weight = 1.0;
  c->tol = 1e-3;
  c->max_iters = 200000;
  c->time_limit_s = std::numeric_limits<double>::infinity();
  c->check_interval = 40;
  c->scaling = 1;
  c->seed = 1;
  c->snapshot_interval = 0;
  c->record_restart_points = 0;
  c->device = 0;
  c->strict_parity = 0;
  c->use_graphs = 1;
  c->profile_kernels = 0;
}

void rapdhg_result_free(rapdhg_result* r) {
  if (!r) return;
  if (!rb::result_block_free(r->x)) {  // one block holds x, y_ineq, y_eq
    std::free(r->x);
    std::free(r->y_ineq);
    std::free(r->y_eq);
  }
  std::free(r->log);
  std::free(r->snapshot_iters);
  std::free(r->snapshot_x);
  std::free(r->snapshot_y);
  std::free(r->restart_x);
  std::free(r->restart_y);
  std::memset(r, 0, sizeof(*r));
}

int rapdhg_solve(const rapdhg_qp* qp, const rapdhg_config* cfg, rapdhg_result* out) {
  const auto t0 = rb::Clock::now();  // solve_seconds counts from entry (solver.hpp:274)
  return result_guard(out, [&] {
    null_check(qp, "qp");
    null_check(cfg, "cfg");
    null_check(out, "out");
    require_device();
    rb::Tracer tr(nullptr);
    {
      rb::Engine e(*qp, *cfg, t0);
      tr.mark("engine setup total");
      e.solve(out, t0);
      tr.mark("solve loop + download");
    }
    tr.mark("engine teardown");
  });
}

int rapdhg_shard_plan(const rapdhg_qp* qp, int32_t parts, int32_t* dual_bounds, int32_t* primal_bounds) {
  return guard([&] {
    null_check(qp, "qp");
    null_check(dual_bounds, "dual_bounds");
    null_check(primal_bounds, "primal_bounds");
    rb::DeviceQP::validate_dims(*qp);
    // the plan the sharded solver uses (RAPDHG_REPLICATE_MIN_LEN included)
    const rb::ShardPlan plan = rb::make_shard_plan(*qp, parts, rb::replicate_min_len_from_env());
    std::copy(plan.dual.begin(), plan.dual.end(), dual_bounds);
    std::copy(plan.primal.begin(), plan.primal.end(), primal_bounds);
  });
}

int rapdhg_host_transport_check(const rapdhg_host_transport* t, int32_t parts, int32_t rank, int64_t len) {
  return guard([&] {
    null_check(t, "transport");
    rb::host_transport_check(*t, parts, rank, len);
  });
}

int rapdhg_nccl_unique_id(uint8_t* out128) {
  return guard([&] {
    null_check(out128, "out");
    rb::nccl_unique_id(out128);
  });
}

}  // extern "C"

namespace {
std::unique_ptr<rb::ShardedEngine> make_sharded(const rapdhg_qp* qp, const rapdhg_config* cfg,
                                                const rapdhg_shard_opts* opts, rb::Clock::time_point t0) {
  null_check(qp, "qp");
  null_check(cfg, "cfg");
  null_check(opts, "opts");
  require_device();
  if (opts->parts < 1) rb::invalid("sharded solve: parts must be >= 1");
  std::unique_ptr<rb::Transport> tr;
  int rank = -1;
  if (opts->emulate) {
    tr = rb::make_emulated_transport(opts->parts);
  } else {
    if (opts->rank < 0 || opts->rank >= opts->parts) rb::invalid("sharded solve: rank out of range");
    RB_CUDA(cudaSetDevice(cfg->device));
    tr = opts->host ? rb::make_host_transport(opts->parts, opts->rank, *opts->host)
                    : rb::make_nccl_transport(opts->parts, opts->rank, opts->nccl_id);
    rank = opts->rank;
  }
  return std::make_unique<rb::ShardedEngine>(*qp, *cfg, opts->parts, rank, std::move(tr), t0,
                                             opts->replicate_min_len);
}
}  // namespace

struct rapdhg_shard_session {
  std::unique_ptr<rb::ShardedEngine> engine;
};

extern "C" {

int rapdhg_solve_sharded(const rapdhg_qp* qp, const rapdhg_config* cfg, const rapdhg_shard_opts* opts,
                         rapdhg_result* out) {
  const auto t0 = rb::Clock::now();
  return result_guard(out, [&] {
    null_check(out, "out");
    auto e = make_sharded(qp, cfg, opts, t0);
    e->solve(out, t0);
  });
}

int rapdhg_shard_session_create(const rapdhg_qp* qp, const rapdhg_config* cfg, const rapdhg_shard_opts* opts,
                                rapdhg_shard_session** out) {
  return guard([&] {
    null_check(out, "out");
    *out = nullptr;
    auto s = std::make_unique<rapdhg_shard_session>();
    s->engine = make_sharded(qp, cfg, opts, rb::Clock::now());
    *out = s.release();
  });
}

int rapdhg_shard_session_solve(rapdhg_shard_session* s, rapdhg_result* out) {
  return result_guard(out, [&] {
    null_check(s, "session");
    null_check(out, "out");
    s->engine->solve(out, rb::Clock::now());
  });
}

void rapdhg_shard_session_destroy(rapdhg_shard_session* s) { delete s; }

int rapdhg_session_create(const rapdhg_qp* qp, const rapdhg_config* cfg, rapdhg_session** out) {
  return guard([&] {
    null_check(qp, "qp");
    null_check(cfg, "cfg");
    null_check(out, "out");
    *out = nullptr;
    require_device();
    auto s = std::make_unique<rapdhg_session>();
    s->cfg = *cfg;
    s->engine = std::make_unique<rb::Engine>(*qp, *cfg, rb::Clock::now());
    *out = s.release();
  });
}

int rapdhg_session_solve(rapdhg_session* s, rapdhg_result* out) {
  return result_guard(out, [&] {
    null_check(s, "session");
    null_check(out, "out");
    s->engine->solve(out, rb::Clock::now());
  });
}

int rapdhg_session_bytes(const rapdhg_session* s, double* b_iter, double* b_dual, double* b_primal) {
  return guard([&] {
    null_check(s, "session");
    if (b_iter) *b_iter = s->engine->bytes_iter();
    if (b_dual) *b_dual = s->engine->bytes_dual();
    if (b_primal) *b_primal = s->engine->bytes_primal();
  });
}

void rapdhg_session_destroy(rapdhg_session* s) { delete s; }

int rapdhg_validate(const rapdhg_qp* qp) {
  return guard([&] {
    null_check(qp, "qp");
    require_device();
    rb::api_validate(*qp);
  });
}

int rapdhg_symmetry_gap(const rapdhg_csr* m, double* out) {
  return guard([&] {
    null_check(m, "m");
    null_check(out, "out");
    require_device();
    *out = rb::api_symmetry_gap(*m);
  });
}

int rapdhg_spmv(const rapdhg_csr* m, const double* x, int64_t x_len, double* y, int32_t strict) {
  return guard([&] {
    null_check(m, "m");
    if (x_len != m->n_cols) rb::invalid("spmv: vector length does not match column count");
    require_device();
    rb::api_spmv(*m, x, y, false, strict != 0);
  });
}

int rapdhg_spmv_t(const rapdhg_csr* m, const double* x, int64_t x_len, double* y, int32_t strict) {
  return guard([&] {
    null_check(m, "m");
    if (x_len != m->n_rows) rb::invalid("spmv_t: vector length does not match row count");
    require_device();
    rb::api_spmv(*m, x, y, true, strict != 0);
  });
}

int rapdhg_inner_step(const rapdhg_qp* p, rapdhg_iterate* s, const rapdhg_step_params* sp,
                      int32_t steps, int32_t strict) {
  return guard([&] {
    null_check(p, "p");
    null_check(s, "state");
    null_check(sp, "params");
    if (steps < 0) rb::invalid("steps must be >= 0");
    require_device();
    rb::api_inner_step(*p, s, *sp, steps, strict != 0);
  });
}

int rapdhg_pdhg_step(const rapdhg_qp* p, rapdhg_iterate* s, double eta, double tau, int32_t strict) {
  const rapdhg_step_params sp{1.0, 1.0, eta, tau};  // solver.hpp:195-198
  return rapdhg_inner_step(p, s, &sp, 1, strict);
}

int rapdhg_rel_kkt(const rapdhg_qp* p, const double* x, const double* y_ineq, const double* y_eq,
                   rapdhg_kkt* out, int32_t strict) {
  return guard([&] {
    null_check(p, "p");
    null_check(out, "out");
    require_device();
    rb::Kkt k;
    rb::api_rel_kkt(*p, x, y_ineq, y_eq, strict != 0, &k);
    *out = {k.r_primal, k.r_dual, k.r_gap};
  });
}

int rapdhg_compute_scaling(const rapdhg_qp* p, double* d1, double* d2, int32_t strict) {
  return guard([&] {
    null_check(p, "p");
    require_device();
    rb::api_scaling(*p, 10, true, d1, d2, strict != 0);
  });
}

int rapdhg_ruiz_scaling(const rapdhg_qp* p, int32_t iterations, double* d1, double* d2,
                        int32_t strict) {
  return guard([&] {
    null_check(p, "p");
    require_device();
    rb::api_scaling(*p, iterations, false, d1, d2, strict != 0);
  });
}

int rapdhg_apply_scaling(const rapdhg_qp* p, const double* d1, const double* d2, double* q_values,
                         double* a_ineq_values, double* a_eq_values, double* c, double* b_ineq,
                         double* b_eq) {
  return guard([&] {
    null_check(p, "p");
    require_device();
    rb::api_apply_scaling(*p, d1, d2, q_values, a_ineq_values, a_eq_values, c, b_ineq, b_eq);
  });
}

int rapdhg_estimate_op_norm(const rapdhg_csr* m, int32_t max_iters, double tol, uint64_t seed,
                            double* out, int32_t strict) {
  return guard([&] {
    null_check(m, "m");
    null_check(out, "out");
    require_device();
    *out = rb::api_op_norm(*m, false, max_iters, tol, seed, strict != 0);
  });
}

int rapdhg_estimate_op_norm_symmetric(const rapdhg_csr* m, int32_t max_iters, double tol,
                                      uint64_t seed, double* out, int32_t strict) {
  return guard([&] {
    null_check(m, "m");
    null_check(out, "out");
    require_device();
    *out = rb::api_op_norm(*m, true, max_iters, tol, seed, strict != 0);
  });
}

int rapdhg_step_schedule_theoretical(int32_t k, int32_t horizon, double norm_q, double norm_a,
                                     rapdhg_step_params* out) {
  return guard([&] { *out = rb::step_schedule_theoretical(k, horizon, norm_q, norm_a); });
}

int rapdhg_pdhg_constant_steps(double norm_q, double norm_a, rapdhg_step_params* out) {
  return guard([&] { *out = rb::pdhg_constant_steps(norm_q, norm_a); });
}

int rapdhg_adaptive_eta(int32_t k, double prev_eta, double norm_q, double norm_a, double omega,
                        double* out) {
  return guard([&] { *out = rb::adaptive_eta(k, prev_eta, norm_q, norm_a, omega); });
}

int rapdhg_primal_weight_update(double dx, double dy, double omega_prev, double* out) {
  return guard([&] { *out = rb::primal_weight_update(dx, dy, omega_prev); });
}

int rapdhg_restart_decision(int32_t policy, double cand, double cand_prev, double start, int64_t k,
                            int64_t total_iters, int64_t fixed_length) {
  if (policy < RAPDHG_RESTART_NONE || policy > RAPDHG_RESTART_PDQP) {
    g_err = "unknown restart policy";
    return RAPDHG_E_INVALID_ARGUMENT;
  }
  return rb::restart_decision(policy, cand, cand_prev, start, k, total_iters, fixed_length) ? 1 : 0;
}

}  // extern "C"
