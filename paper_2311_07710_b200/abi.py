"""ctypes mirrors of the plain structs in include/rapdhg_b200.h.

Only layouts live here (no library loading), so the product binding
(``paper_2311_07710_b200``) and the test-only oracle binding (``oracle``)
describe the same C-ABI without depending on each other.
"""
import ctypes as C

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P_i32, P_i64, P_f64 = C.POINTER(i32), C.POINTER(i64), C.POINTER(f64)

RAPDHG_OK = 0
E_INVALID_ARGUMENT = -1
E_OUT_OF_RANGE = -2
E_CUDA = -3
E_NO_DEVICE = -4
E_PARSE = -5
E_INTERNAL = -6
ABI_VERSION = 2


class Csr(C.Structure):
    _fields_ = [("n_rows", i32), ("n_cols", i32), ("nnz", i64),
                ("row_ptr", P_i32), ("col_idx", P_i32), ("values", P_f64)]


class Qp(C.Structure):
    _fields_ = [("n", i32), ("m_ineq", i32), ("m_eq", i32),
                ("q", Csr), ("c", P_f64), ("a_ineq", Csr), ("b_ineq", P_f64),
                ("a_eq", Csr), ("b_eq", P_f64), ("obj_offset", f64),
                ("name", C.c_char_p), ("var_names", C.POINTER(C.c_char_p)),
                ("lower", P_f64), ("upper", P_f64)]


class RawProblem(C.Structure):
    _fields_ = [("n", i32), ("m", i32), ("q", Csr), ("c", P_f64), ("obj_offset", f64),
                ("a", Csr), ("row_types", P_i32), ("rhs", P_f64), ("range", P_f64),
                ("lower", P_f64), ("upper", P_f64), ("name", C.c_char_p),
                ("row_names", C.POINTER(C.c_char_p)), ("var_names", C.POINTER(C.c_char_p))]


class CanonicalMap(C.Structure):
    _fields_ = [("n_ineq", i32), ("n_eq", i32), ("ineq_labels", C.POINTER(C.c_char_p)),
                ("eq_labels", C.POINTER(C.c_char_p))]


class Config(C.Structure):
    _fields_ = [("algorithm", i32), ("restart", i32), ("restart_length", i64),
                ("step_rule", i32), ("primal_weight", i32),
                ("fixed_primal_weight", f64), ("tol", f64), ("max_iters", i64),
                ("time_limit_s", f64), ("check_interval", i32), ("scaling", i32),
                ("seed", u64), ("snapshot_interval", i64),
                ("record_restart_points", i32),
                ("device", i32), ("strict_parity", i32), ("use_graphs", i32),
                ("profile_kernels", i32), ("box_projection", i32)]


class Kkt(C.Structure):
    _fields_ = [("r_primal", f64), ("r_dual", f64), ("r_gap", f64)]


class LogRecord(C.Structure):
    _fields_ = [("iteration", i64), ("r_primal", f64), ("r_dual", f64),
                ("r_gap", f64), ("eta", f64), ("omega", f64), ("restarted", i32)]


class Result(C.Structure):
    _fields_ = [("status", i32), ("n", i32), ("m_ineq", i32), ("m_eq", i32),
                ("x", P_f64), ("y_ineq", P_f64), ("y_eq", P_f64),
                ("residuals", Kkt), ("iterations", i64), ("restarts", i64),
                ("solve_seconds", f64), ("norm_q", f64), ("norm_a", f64),
                ("norm_fallback", i32), ("n_log", i64),
                ("log", C.POINTER(LogRecord)), ("n_snapshots", i64),
                ("snapshot_iters", P_i64), ("snapshot_x", P_f64),
                ("snapshot_y", P_f64), ("n_restart_points", i64),
                ("restart_x", P_f64), ("restart_y", P_f64),
                ("setup_seconds", f64), ("loop_seconds", f64),
                ("kernel_launches", i64), ("kernel_ms", f64 * 2),
                ("kernel_count", i64 * 2)]


class StepParams(C.Structure):
    _fields_ = [("beta", f64), ("theta", f64), ("eta", f64), ("tau", f64)]


class Iterate(C.Structure):
    _fields_ = [("x", P_f64), ("x_prev", P_f64), ("y", P_f64), ("x_bar", P_f64),
                ("y_bar", P_f64), ("k", i64), ("n", i64)]


class CsrOwned(C.Structure):
    _fields_ = [("n_rows", i32), ("n_cols", i32), ("nnz", i64),
                ("row_ptr", P_i32), ("col_idx", P_i32), ("values", P_f64)]


class QpOwned(C.Structure):
    _fields_ = [("n", i32), ("m_ineq", i32), ("m_eq", i32),
                ("q", CsrOwned), ("a_ineq", CsrOwned), ("a_eq", CsrOwned),
                ("c", P_f64), ("b_ineq", P_f64), ("b_eq", P_f64),
                ("obj_offset", f64), ("name", C.c_char_p), ("var_names", C.POINTER(C.c_char_p)),
                ("lower", P_f64), ("upper", P_f64)]


ALLGATHERV_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, P_f64, P_i64, i32)
ALLTOALLV_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, P_f64, P_i64, P_f64, P_i64, i32)
ALLREDUCE_MIN_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, P_i64)


class HostTransport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgatherv", ALLGATHERV_CB), ("alltoallv", ALLTOALLV_CB),
                ("allreduce_min", ALLREDUCE_MIN_CB)]


class ShardOpts(C.Structure):
    _fields_ = [("parts", i32), ("rank", i32), ("emulate", i32), ("pad", i32),
                ("nccl_id", C.c_uint8 * 128), ("host", C.POINTER(HostTransport)),
                ("replicate_min_len", C.c_int64)]


def declare(lib, name, restype, *argtypes):
    """Bind a symbol's signature; raises AttributeError if it is missing."""
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn
