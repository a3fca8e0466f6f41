/*
 * rapdhg_b200.h — C-ABI of the B200-native rAPDHG (PDQP) solver.
 *
 * Drop-in boundary for the reference C++ solver's iteration path
 * (/root/reference/proj/include/rapdhg/*.hpp). Every entry point below names
 * the reference interface it replaces (file:line, paths relative to
 * proj/include/rapdhg/). Plain pointers and sizes only: no C++ or torch types
 * cross this boundary. All array arguments are HOST memory unless a function
 * name says `_device`; the library uploads, runs the fp64 sm_100a kernels and
 * copies results back.
 *
 * Error behaviour mirrors the reference's exceptions: a function returns
 * RAPDHG_OK (0) or a negative code; the message the reference would have put
 * in its std::invalid_argument / std::out_of_range is available from
 * rapdhg_last_error() (thread-local). Numerical outcomes (iteration limit,
 * NaN) are statuses in the result, not errors — as in solver.hpp:26,372.
 *
 * There is no CPU fallback: without a visible CUDA device every compute entry
 * point returns RAPDHG_E_NO_DEVICE.
 */
#ifndef RAPDHG_B200_H_
#define RAPDHG_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAPDHG_ABI_VERSION 2

/* ---- error codes (return values) ------------------------------------- */
enum {
  RAPDHG_OK = 0,
  RAPDHG_E_INVALID_ARGUMENT = -1, /* std::invalid_argument in the reference */
  RAPDHG_E_OUT_OF_RANGE = -2,     /* std::out_of_range (sparse.hpp:36)     */
  RAPDHG_E_CUDA = -3,             /* CUDA runtime / kernel failure         */
  RAPDHG_E_NO_DEVICE = -4,        /* no CUDA device: there is no fallback  */
  RAPDHG_E_PARSE = -5,            /* QpsParseError (qps.hpp:30)            */
  RAPDHG_E_INTERNAL = -6
};

/* ---- enums: values equal the reference enum order (solver.hpp:22-26) --- */
enum { RAPDHG_ALG_PDHG = 0, RAPDHG_ALG_APDHG = 1 };
enum {
  RAPDHG_RESTART_NONE = 0,
  RAPDHG_RESTART_FIXED = 1,
  RAPDHG_RESTART_HALVING = 2,
  RAPDHG_RESTART_PDQP = 3
};
enum { RAPDHG_STEP_THEORETICAL = 0, RAPDHG_STEP_ADAPTIVE = 1 };
enum { RAPDHG_PW_FIXED = 0, RAPDHG_PW_ADAPTIVE = 1 };
enum {
  RAPDHG_STATUS_OPTIMAL = 0,
  RAPDHG_STATUS_ITERATION_LIMIT = 1,
  RAPDHG_STATUS_TIME_LIMIT = 2,
  RAPDHG_STATUS_NUMERICAL_ERROR = 3
};

/* ---- problem ----------------------------------------------------------- */

/* Compressed sparse row matrix. Replaces rapdhg::SparseMatrix
 * (sparse.hpp:27-170), whose private storage is exactly this triple
 * (sparse.hpp:165-169: int row_start_, int cols_, double values_). Input
 * must be canonical as the reference constructor makes it (sparse.hpp:31-62):
 * columns strictly increasing within a row, no explicit zeros. Use
 * rapdhg_csr_from_triplets() to canonicalize raw triplets. */
typedef struct {
  int32_t n_rows;
  int32_t n_cols;
  int64_t nnz;
  const int32_t* row_ptr; /* n_rows + 1 */
  const int32_t* col_idx; /* nnz */
  const double* values;   /* nnz */
} rapdhg_csr;

/* Canonical convex QP  min ½x'Qx + c'x  s.t. A_ineq x <= b_ineq, A_eq x = b_eq.
 * Replaces rapdhg::QuadraticProgram (problem.hpp:24-56). Sizes are implied
 * as in the reference: n = len(c) (num_vars), m_ineq = len(b_ineq), m_eq =
 * len(b_eq) (problem.hpp:35-38). */
typedef struct {
  int32_t n;
  int32_t m_ineq;
  int32_t m_eq;
  rapdhg_csr q;      /* n x n, symmetric, full (both triangles) storage */
  const double* c;   /* n */
  rapdhg_csr a_ineq; /* m_ineq x n */
  const double* b_ineq;
  rapdhg_csr a_eq;   /* m_eq x n */
  const double* b_eq;
  double obj_offset;
  const char* name;              /* QuadraticProgram::name; NULL = "" */
  const char* const* var_names;  /* n entries (var_names), or NULL = none */
  /* B200 extension, no reference counterpart (the reference turns variable
   * bounds into singleton <= rows: canonicalize, problem.hpp:178-185): bounds
   * l <= x <= u (n each, +-inf allowed; NULL = none) enforced by projecting
   * the primal step, for rapdhg_config.box_projection = 1 only. */
  const double* lower;
  const double* upper;
} rapdhg_qp;

/* ---- options ----------------------------------------------------------- */

/* Mirrors rapdhg::SolverConfig field by field (solver.hpp:38-55) plus the
 * B200 fields at the end. rapdhg_config_default() fills the reference
 * defaults (APDHG, PDQP restart, adaptive step, adaptive omega, tol 1e-3,
 * 200000 iterations, check every 40, scaling on, seed 1). */
typedef struct {
  int32_t algorithm;
  int32_t restart;
  int64_t restart_length;
  int32_t step_rule;
  int32_t primal_weight;
  double fixed_primal_weight;
  double tol;
  int64_t max_iters;
  double time_limit_s; /* +inf = none */
  int32_t check_interval;
  int32_t scaling;
  uint64_t seed;
  int64_t snapshot_interval;
  int32_t record_restart_points;
  /* --- B200 extensions --- */
  int32_t device;        /* CUDA ordinal */
  int32_t strict_parity; /* 1: sequential fp64 sums, no FMA -> bit-exact with
                            the reference; 0: fast deterministic kernels */
  int32_t use_graphs;    /* capture each check interval in a CUDA graph */
  int32_t profile_kernels; /* 1: CUDA events around the two steps of every 32nd chunk;
                             2: in-loop step times from %globaltimer stamps (slab path) */
  int32_t box_projection; /* 1: honour rapdhg_qp.lower / upper by projecting the primal
                             step onto the box (north_star's "primal step with box
                             projection"; fast mode only; no reference counterpart, so
                             not a parity mode); relKKT then uses the bound multipliers */
} rapdhg_config;

void rapdhg_config_default(rapdhg_config* cfg);

/* ---- results ----------------------------------------------------------- */

typedef struct { /* rapdhg::KktResiduals (kkt.hpp:11-17) */
  double r_primal;
  double r_dual;
  double r_gap;
} rapdhg_kkt;

typedef struct { /* rapdhg::LogRecord (solver.hpp:66-74) */
  int64_t iteration;
  double r_primal;
  double r_dual;
  double r_gap;
  double eta;
  double omega;
  int32_t restarted;
} rapdhg_log_record;

/* rapdhg::SolveResult (solver.hpp:76-89). Arrays are allocated by the library
 * and released by rapdhg_result_free(). Every call that fills a result zeroes
 * it first and, when it fails, releases what it had filled: a failed call
 * leaves an all-zero result (nothing to free). snapshots are stored row-major:
 * snapshot s has x at snapshot_x + s*n and y (ineq then eq) at
 * snapshot_y + s*(m_ineq+m_eq); restart points likewise. x, y_ineq and y_eq
 * are consecutive parts of one block (page-locked when large: free it only
 * through rapdhg_result_free, never with free()). */
typedef struct {
  int32_t status;
  int32_t n, m_ineq, m_eq;
  double* x;      /* n       */
  double* y_ineq; /* m_ineq  */
  double* y_eq;   /* m_eq    */
  rapdhg_kkt residuals;
  int64_t iterations;
  int64_t restarts;
  double solve_seconds;
  double norm_q;
  double norm_a;
  int32_t norm_fallback;
  int64_t n_log;
  rapdhg_log_record* log;
  int64_t n_snapshots;
  int64_t* snapshot_iters;
  double* snapshot_x;
  double* snapshot_y;
  int64_t n_restart_points;
  double* restart_x;
  double* restart_y;
  /* --- B200 instrumentation --- */
  double setup_seconds;     /* upload + validate + scaling + norms */
  double loop_seconds;      /* iterations + checks + restarts, device time (the final download excluded) */
  int64_t kernel_launches;  /* library kernels launched by this call */
  /* profile_kernels=1|2: summed time (ms) and sample counts of the two
   * steps (0 = dual step A*w, 1 = primal step [Q|A']) in sampled chunks */
  double kernel_ms[2];
  int64_t kernel_count[2];
} rapdhg_result;

void rapdhg_result_free(rapdhg_result* r);

/* Thread-local message of the last failing call on this thread. */
const char* rapdhg_last_error(void);
int rapdhg_abi_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host). */
int rapdhg_device_count(void);

/* ---- main entry: rapdhg::solve (solver.hpp:272-471) -------------------- */
int rapdhg_solve(const rapdhg_qp* qp, const rapdhg_config* cfg, rapdhg_result* out);

/* Resident-data variant: upload + validate + scaling + norms once
 * (solver.hpp:277-300), then solve repeatedly from the zero start on the
 * HBM-resident problem. Used to time the iteration loop with inputs already
 * in HBM. */
typedef struct rapdhg_session rapdhg_session;
int rapdhg_session_create(const rapdhg_qp* qp, const rapdhg_config* cfg, rapdhg_session** out);
int rapdhg_session_solve(rapdhg_session* s, rapdhg_result* out);
/* Algorithmic bytes of one iteration (SURVEY §8(d) B_iter) and of one launch
 * of each hot kernel, for the roofline. */
int rapdhg_session_bytes(const rapdhg_session* s, double* b_iter, double* b_dual,
                         double* b_primal);
void rapdhg_session_destroy(rapdhg_session* s);

/* ---- row-sharded multi-GPU solve (no reference counterpart:
 * the reference is single-threaded) ------------------------- */

/* nnz-balanced contiguous row blocks for `parts` ranks: dual rows of
 * [A_ineq; A_eq] (dual_bounds, parts+1 entries over [0, m)) and primal rows
 * of [Q | A'] (primal_bounds over [0, n)); inner bounds are multiples of the
 * reduction chunk (2048). Host-only. */
int rapdhg_shard_plan(const rapdhg_qp* qp, int32_t parts, int32_t* dual_bounds,
                      int32_t* primal_bounds);

/* Host-staged transport: the caller's own collectives (MPI, gloo, ...) as
 * callbacks. The library stages each exchange through host memory, so one
 * process per rank works over any process group (and several ranks may share
 * a GPU); NCCL is the fast path. Every callback is collective over all ranks,
 * called in the same order on every rank, and returns 0 on success.
 *  - allgatherv: buf (length bounds[parts]) holds this rank's slice
 *    [bounds[rank], bounds[rank+1]); fill every other rank's slice in place.
 *  - alltoallv: send[send_off[p] .. send_off[p+1]) goes to rank p, which
 *    receives it into its recv[recv_off[me] .. recv_off[me+1]) (offsets have
 *    parts+1 entries; this rank's own segments are empty).
 *  - allreduce_min: *value = min over ranks. */
typedef struct {
  void* ctx;
  int (*allgatherv)(void* ctx, double* buf, const int64_t* bounds, int32_t parts);
  int (*alltoallv)(void* ctx, const double* send, const int64_t* send_off, double* recv,
                   const int64_t* recv_off, int32_t parts);
  int (*allreduce_min)(void* ctx, int64_t* value);
} rapdhg_host_transport;

typedef struct {
  int32_t parts;    /* number of shards */
  int32_t rank;     /* this process's shard (ignored when emulate = 1) */
  int32_t emulate;  /* 1: all shards in this process on cfg->device */
  int32_t pad;
  uint8_t nccl_id[128]; /* ncclUniqueId from rank 0 (emulate = 0, no host transport) */
  const rapdhg_host_transport* host; /* non-NULL (emulate = 0): use these collectives, not NCCL */
  /* > 0: replicate the rows of [Q | A'] with at least this many entries
   * (SURVEY 8(e) dense-coupling columns: every shard computes them from
   * per-shard partial sums; deterministic for a given shard count, within
   * rounding of rapdhg_solve but not bit-identical); 0: the
   * RAPDHG_REPLICATE_MIN_LEN environment variable, else none; < 0: none */
  int64_t replicate_min_len;
} rapdhg_shard_opts;

/* Exercises a host transport's callbacks without a GPU: allgather-v, an
 * all-to-all-v and a min-reduction over `parts` ranks with deterministic
 * per-rank data of about `len` elements, each result checked against its
 * expected value. Collective; returns 0 when every exchange delivered the
 * expected data. */
int rapdhg_host_transport_check(const rapdhg_host_transport* t, int32_t parts, int32_t rank, int64_t len);

/* 128-byte ncclUniqueId for rapdhg_shard_opts.nccl_id (call on rank 0 and
 * broadcast it, e.g. with torch.distributed). */
int rapdhg_nccl_unique_id(uint8_t* out128);

/* Same contract as rapdhg_solve; every rank returns the full result. The
 * result is bit-identical to rapdhg_solve in fast mode unless rows are
 * replicated (opts.replicate_min_len); strict mode is rejected: its
 * sequential reductions do not shard. */
int rapdhg_solve_sharded(const rapdhg_qp* qp, const rapdhg_config* cfg,
                         const rapdhg_shard_opts* opts, rapdhg_result* out);

/* Persistent sharded session: setup and communicator once (an ncclUniqueId
 * bootstraps exactly one communicator), then repeated solves from the zero
 * start. Collective: every rank calls create / solve / destroy together. */
typedef struct rapdhg_shard_session rapdhg_shard_session;
int rapdhg_shard_session_create(const rapdhg_qp* qp, const rapdhg_config* cfg,
                                const rapdhg_shard_opts* opts, rapdhg_shard_session** out);
int rapdhg_shard_session_solve(rapdhg_shard_session* s, rapdhg_result* out);
void rapdhg_shard_session_destroy(rapdhg_shard_session* s);

/* ---- secondary API used by the reference's tests ----------------------- */

/* y = M x (sparse.hpp:79-88) and y = M' x (sparse.hpp:91-100). */
int rapdhg_spmv(const rapdhg_csr* m, const double* x, int64_t x_len, double* y, int32_t strict);
int rapdhg_spmv_t(const rapdhg_csr* m, const double* x, int64_t x_len, double* y, int32_t strict);

/* rapdhg::StepParams (stepsize.hpp:13-18). */
typedef struct {
  double beta;
  double theta;
  double eta;
  double tau;
} rapdhg_step_params;

/* rapdhg::IterateState (solver.hpp:125-143): x, x_prev, x_bar (n) and y,
 * y_bar (m = m_ineq + m_eq, ineq first), updated in place. */
typedef struct {
  double* x;
  double* x_prev;
  double* y;
  double* x_bar;
  double* y_bar;
  int64_t k;
  int64_t n;
} rapdhg_iterate;

/* rapdhg::inner_step(s, p, sp) (solver.hpp:156-191): one unified PDHG/APDHG
 * iteration on the (already scaled, if desired) problem, `steps` times with
 * the same parameters. */
int rapdhg_inner_step(const rapdhg_qp* p, rapdhg_iterate* s, const rapdhg_step_params* sp,
                      int32_t steps, int32_t strict);
/* rapdhg::pdhg_step (solver.hpp:195-203) */
int rapdhg_pdhg_step(const rapdhg_qp* p, rapdhg_iterate* s, double eta, double tau,
                     int32_t strict);

/* rapdhg::rel_kkt (kkt.hpp:28-72). */
int rapdhg_rel_kkt(const rapdhg_qp* p, const double* x, const double* y_ineq,
                   const double* y_eq, rapdhg_kkt* out, int32_t strict);

/* rapdhg::compute_scaling (scaling.hpp:97-106): d1 (m), d2 (n). */
int rapdhg_compute_scaling(const rapdhg_qp* p, double* d1, double* d2, int32_t strict);
/* rapdhg::ruiz_scaling (scaling.hpp:85-92) */
int rapdhg_ruiz_scaling(const rapdhg_qp* p, int32_t iterations, double* d1, double* d2,
                        int32_t strict);
/* rapdhg::apply_scaling (scaling.hpp:109-123): writes the scaled values into
 * caller buffers laid out like the input CSRs (same patterns). */
int rapdhg_apply_scaling(const rapdhg_qp* p, const double* d1, const double* d2,
                         double* q_values, double* a_ineq_values, double* a_eq_values,
                         double* c, double* b_ineq, double* b_eq);

/* rapdhg::estimate_op_norm / _symmetric (opnorm.hpp:36-87) with
 * PowerIterOptions{max_iters, tol, seed} (opnorm.hpp:12-16). */
int rapdhg_estimate_op_norm(const rapdhg_csr* m, int32_t max_iters, double tol, uint64_t seed,
                            double* out, int32_t strict);
int rapdhg_estimate_op_norm_symmetric(const rapdhg_csr* m, int32_t max_iters, double tol,
                                      uint64_t seed, double* out, int32_t strict);

/* rapdhg::unscale_point (scaling.hpp:126-133): x *= d2, y *= d1 (ineq then
 * eq), in place; and its inverse scale_point (scaling.hpp:136-143). Host,
 * elementwise (the solver unscales its checks on the device). */
int rapdhg_unscale_point(const double* d1, const double* d2, int32_t n, int32_t m_ineq, int32_t m_eq,
                         double* x, double* y_ineq, double* y_eq);
int rapdhg_scale_point(const double* d1, const double* d2, int32_t n, int32_t m_ineq, int32_t m_eq,
                       double* x, double* y_ineq, double* y_eq);

/* QuadraticProgram::validate (problem.hpp:40-50): dimensions, then the
 * symmetry test gap <= 1e-12 * max(1, max|Q|) on the device. */
int rapdhg_validate(const rapdhg_qp* qp);
/* SparseMatrix::symmetry_gap (sparse.hpp:119-138): max |M_ij - M_ji| over
 * both patterns, on the device (square matrices only). */
int rapdhg_symmetry_gap(const rapdhg_csr* m, double* out);

/* ---- host scalar rules (stepsize.hpp, solver.hpp:218-235) ------------- */
/* primal_weight_init (stepsize.hpp:73-78): ||c||_2 / ||b||_2 when both
 * exceed 1e-10, else 1 (sequential sums, as vec.hpp:20). */
int rapdhg_primal_weight_init(const double* c, int64_t n, const double* b, int64_t m, double* out);
int rapdhg_step_schedule_theoretical(int32_t k, int32_t horizon, double norm_q, double norm_a,
                                     rapdhg_step_params* out);
int rapdhg_pdhg_constant_steps(double norm_q, double norm_a, rapdhg_step_params* out);
int rapdhg_adaptive_eta(int32_t k, double prev_eta, double norm_q, double norm_a, double omega,
                        double* out);
int rapdhg_primal_weight_update(double delta_x, double delta_y, double omega_prev, double* out);
/* RestartContext (solver.hpp:206-212) flattened. Returns 0/1, or <0 on error. */
int rapdhg_restart_decision(int32_t policy, double relkkt_candidate, double relkkt_candidate_prev,
                            double relkkt_epoch_start, int64_t k, int64_t total_iters,
                            int64_t fixed_length);

/* ---- host utilities ---------------------------------------------------- */

/* Owned CSR / QP containers returned by the generators and converters. */
typedef struct {
  int32_t n_rows, n_cols;
  int64_t nnz;
  int32_t* row_ptr;
  int32_t* col_idx;
  double* values;
} rapdhg_csr_owned;

typedef struct {
  int32_t n, m_ineq, m_eq;
  rapdhg_csr_owned q, a_ineq, a_eq;
  double* c;
  double* b_ineq;
  double* b_eq;
  double obj_offset;
  char* name;        /* malloc'd, or NULL */
  char** var_names;  /* n malloc'd strings, or NULL */
  double* lower;     /* n, or NULL: bounds kept out of the rows (rapdhg_canonicalize_box) */
  double* upper;
} rapdhg_qp_owned;

/* SparseMatrix(n_rows, n_cols, triplets) (sparse.hpp:31-62): sort by
 * (row, col), sum duplicates, drop exact zeros. */
int rapdhg_csr_from_triplets(int32_t n_rows, int32_t n_cols, int64_t nnz, const int32_t* rows,
                             const int32_t* cols, const double* vals, rapdhg_csr_owned* out);
void rapdhg_csr_free(rapdhg_csr_owned* m);
void rapdhg_qp_free(rapdhg_qp_owned* p);
/* Borrowed view of an owned QP, for passing to the compute entry points. */
void rapdhg_qp_view(const rapdhg_qp_owned* p, rapdhg_qp* view);

/* rapdhg::RowType (problem.hpp:72). */
enum { RAPDHG_ROW_EQ = 0, RAPDHG_ROW_LE = 1, RAPDHG_ROW_GE = 2 };

/* rapdhg::RawProblem (problem.hpp:76-92): typed rows, optional ranges and
 * variable bounds, before conversion to the canonical <= / = form. q and a
 * are canonical CSRs (as the reference's SparseMatrix members are). */
typedef struct {
  int32_t n;                 /* num_vars = len(c) */
  int32_t m;                 /* num_rows = len(rhs) */
  rapdhg_csr q;              /* n x n, full (mirrored) */
  const double* c;           /* n */
  double obj_offset;
  rapdhg_csr a;              /* m x n, one row per constraint, original orientation */
  const int32_t* row_types;  /* m: RAPDHG_ROW_* */
  const double* rhs;         /* m */
  const double* range;       /* m, NaN = no RANGES entry; NULL = none at all */
  const double* lower;       /* n, -inf allowed */
  const double* upper;       /* n, +inf allowed */
  const char* name;          /* NULL = "" */
  const char* const* row_names; /* m entries or NULL (labels use "r<i>") */
  const char* const* var_names; /* n entries or NULL (labels use "x<j>") */
} rapdhg_raw_problem;

/* rapdhg::CanonicalMap (problem.hpp:95-99): provenance label of every
 * canonical row ("row:<name>", "row:<name>:ub" / ":lb", "bound:<var>:ub" /
 * ":lb"). Library-owned strings, released by rapdhg_canonical_map_free. */
typedef struct {
  int32_t n_ineq, n_eq;
  char** ineq_labels;
  char** eq_labels;
} rapdhg_canonical_map;

/* rapdhg::canonicalize (problem.hpp:131-198): G rows negated into <= rows,
 * ranged rows split into two <= rows, rows whose interval is a point kept as
 * equalities, finite variable bounds appended as singleton <= rows, then
 * QuadraticProgram::validate (Q symmetric). Errors (std::invalid_argument in
 * the reference) return RAPDHG_E_INVALID_ARGUMENT with the same messages.
 * map may be NULL. Host-only. */
int rapdhg_canonicalize(const rapdhg_raw_problem* raw, rapdhg_qp_owned* out, rapdhg_canonical_map* map);
/* The same, except that variable bounds stay out of the rows: out->lower /
 * out->upper hold them (for box_projection = 1). B200 extension. */
int rapdhg_canonicalize_box(const rapdhg_raw_problem* raw, rapdhg_qp_owned* out, rapdhg_canonical_map* map);
void rapdhg_canonical_map_free(rapdhg_canonical_map* map);

/* QPS (MPS + QUADOBJ/QMATRIX) text or file -> canonical QP: parse_qps
 * (qps.hpp:69-298) then canonicalize (problem.hpp:131-198: G rows negated,
 * ranges split, finite bounds as singleton <= rows, E rows kept). Parse errors
 * return RAPDHG_E_PARSE with the reference's "qps parse error at line N: ..."
 * message. Host-only. */
int rapdhg_parse_qps(const char* text, rapdhg_qp_owned* out);
int rapdhg_parse_qps_file(const char* path, rapdhg_qp_owned* out);
/* The same, also returning canonicalize's CanonicalMap (map may be NULL). */
int rapdhg_parse_qps_map(const char* text, rapdhg_qp_owned* out, rapdhg_canonical_map* map);
int rapdhg_parse_qps_file_map(const char* path, rapdhg_qp_owned* out, rapdhg_canonical_map* map);
/* write_qps (qps.hpp:320-381): *out is malloc'd text, release with rapdhg_free. */
int rapdhg_write_qps(const rapdhg_qp* qp, char** out);
void rapdhg_free(void* p);

/* Synthetic instances of SURVEY §8(d) (no reference generator ships;
 * SPEC.md:417-489 describes the classes). scale multiplies the headline
 * sizes (1.0 = the BASELINE config). Deterministic in seed. */
enum {
  RAPDHG_GEN_RANDOM_QP = 1, /* C1: SPEC.md:431 random QP */
  RAPDHG_GEN_LASSO = 2,     /* C2 */
  RAPDHG_GEN_PORTFOLIO = 3, /* C3: Markowitz factor model */
  RAPDHG_GEN_SVM = 4,       /* C4 */
  RAPDHG_GEN_LARGE = 5,     /* C5: uniform columns */
  RAPDHG_GEN_LARGE_LOCAL = 6 /* C5-L: 95% block-local columns */
};
int rapdhg_generate(int32_t kind, double scale, uint64_t seed, rapdhg_qp_owned* out);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* RAPDHG_B200_H_ */
