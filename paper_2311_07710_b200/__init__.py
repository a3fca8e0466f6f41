"""B200-native rAPDHG (PDQP, arXiv 2311.07710) — Python host mirror.

Mirrors the reference C++ API of /root/reference/proj/include/rapdhg/
(same names, argument meaning and error behaviour) over the C-ABI of
include/rapdhg_b200.h, implemented by the fp64 sm_100a kernels in
``librapdhg_b200.so``:

====================================  =======================================
reference (file:line)                 here
====================================  =======================================
SparseMatrix (sparse.hpp:27-170)      SparseMatrix (canonical CSR, numpy)
QuadraticProgram (problem.hpp:24-56)  QuadraticProgram
SolverConfig (solver.hpp:38-64)       SolverConfig
solve (solver.hpp:272-471)            solve -> SolveResult
inner_step / pdhg_step (:182-203)     inner_step / pdhg_step
rel_kkt (kkt.hpp:28-72)               rel_kkt -> KktResiduals
compute_scaling etc. (scaling.hpp)    compute_scaling, ruiz_scaling,
                                      apply_scaling, unscale_point
estimate_op_norm(_symmetric)          estimate_op_norm(_symmetric)
stepsize.hpp scalar rules             step_schedule_theoretical, ...
====================================  =======================================

Errors: std::invalid_argument -> InvalidArgument (a ValueError),
std::out_of_range -> IndexError, no CUDA device -> NoDeviceError. There is no
CPU fallback: compute calls raise NoDeviceError on a host without a GPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import weakref
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
# RAPDHG_LIB selects an alternative build of the same library (A/B kernel variants)
LIB_PATH = os.environ.get("RAPDHG_LIB") or os.path.join(_HERE, "librapdhg_b200.so")


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference."""


class NoDeviceError(RuntimeError):
    """No CUDA device visible: the solver has no CPU fallback."""


class CudaError(RuntimeError):
    pass


class QpsParseError(RuntimeError):
    pass


_lib = None


def _point_at_pip_nccl():
    """The sharded solver dlopens NCCL on first use: prefer the pip NCCL that
    torch ships (RAPDHG_NCCL_LIB), so a later `import torch` finds the NCCL it
    was built against already loaded, not an older system libnccl.so.2."""
    if os.environ.get("RAPDHG_NCCL_LIB"):
        return
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["RAPDHG_NCCL_LIB"] = cand
            return


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2311_07710_b200` "
            "(or __graft_entry__.build()); there is no fallback implementation")
    lib = C.CDLL(LIB_PATH)
    _point_at_pip_nccl()
    d = abi.declare
    P = C.POINTER
    d(lib, "rapdhg_last_error", C.c_char_p)
    d(lib, "rapdhg_abi_version", C.c_int)
    d(lib, "rapdhg_device_count", C.c_int)
    d(lib, "rapdhg_config_default", None, P(abi.Config))
    d(lib, "rapdhg_result_free", None, P(abi.Result))
    d(lib, "rapdhg_solve", C.c_int, P(abi.Qp), P(abi.Config), P(abi.Result))
    d(lib, "rapdhg_session_create", C.c_int, P(abi.Qp), P(abi.Config), P(C.c_void_p))
    d(lib, "rapdhg_session_solve", C.c_int, C.c_void_p, P(abi.Result))
    d(lib, "rapdhg_session_bytes", C.c_int, C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_double))
    d(lib, "rapdhg_session_destroy", None, C.c_void_p)
    d(lib, "rapdhg_spmv", C.c_int, P(abi.Csr), abi.P_f64, C.c_int64, abi.P_f64, C.c_int32)
    d(lib, "rapdhg_spmv_t", C.c_int, P(abi.Csr), abi.P_f64, C.c_int64, abi.P_f64, C.c_int32)
    d(lib, "rapdhg_inner_step", C.c_int, P(abi.Qp), P(abi.Iterate), P(abi.StepParams), C.c_int32, C.c_int32)
    d(lib, "rapdhg_pdhg_step", C.c_int, P(abi.Qp), P(abi.Iterate), C.c_double, C.c_double, C.c_int32)
    d(lib, "rapdhg_rel_kkt", C.c_int, P(abi.Qp), abi.P_f64, abi.P_f64, abi.P_f64, P(abi.Kkt), C.c_int32)
    d(lib, "rapdhg_compute_scaling", C.c_int, P(abi.Qp), abi.P_f64, abi.P_f64, C.c_int32)
    d(lib, "rapdhg_ruiz_scaling", C.c_int, P(abi.Qp), C.c_int32, abi.P_f64, abi.P_f64, C.c_int32)
    d(lib, "rapdhg_apply_scaling", C.c_int, P(abi.Qp), abi.P_f64, abi.P_f64, abi.P_f64, abi.P_f64,
      abi.P_f64, abi.P_f64, abi.P_f64, abi.P_f64)
    d(lib, "rapdhg_estimate_op_norm", C.c_int, P(abi.Csr), C.c_int32, C.c_double, C.c_uint64,
      abi.P_f64, C.c_int32)
    d(lib, "rapdhg_estimate_op_norm_symmetric", C.c_int, P(abi.Csr), C.c_int32, C.c_double,
      C.c_uint64, abi.P_f64, C.c_int32)
    d(lib, "rapdhg_step_schedule_theoretical", C.c_int, C.c_int32, C.c_int32, C.c_double,
      C.c_double, P(abi.StepParams))
    d(lib, "rapdhg_pdhg_constant_steps", C.c_int, C.c_double, C.c_double, P(abi.StepParams))
    d(lib, "rapdhg_adaptive_eta", C.c_int, C.c_int32, C.c_double, C.c_double, C.c_double,
      C.c_double, abi.P_f64)
    d(lib, "rapdhg_primal_weight_update", C.c_int, C.c_double, C.c_double, C.c_double, abi.P_f64)
    d(lib, "rapdhg_restart_decision", C.c_int, C.c_int32, C.c_double, C.c_double, C.c_double,
      C.c_int64, C.c_int64, C.c_int64)
    d(lib, "rapdhg_csr_from_triplets", C.c_int, C.c_int32, C.c_int32, C.c_int64, abi.P_i32,
      abi.P_i32, abi.P_f64, P(abi.CsrOwned))
    d(lib, "rapdhg_csr_free", None, P(abi.CsrOwned))
    d(lib, "rapdhg_qp_free", None, P(abi.QpOwned))
    d(lib, "rapdhg_qp_view", None, P(abi.QpOwned), P(abi.Qp))
    d(lib, "rapdhg_generate", C.c_int, C.c_int32, C.c_double, C.c_uint64, P(abi.QpOwned))
    d(lib, "rapdhg_shard_plan", C.c_int, P(abi.Qp), C.c_int32, abi.P_i32, abi.P_i32)
    d(lib, "rapdhg_parse_qps", C.c_int, C.c_char_p, P(abi.QpOwned))
    d(lib, "rapdhg_parse_qps_file", C.c_int, C.c_char_p, P(abi.QpOwned))
    d(lib, "rapdhg_write_qps", C.c_int, P(abi.Qp), P(C.c_void_p))
    d(lib, "rapdhg_free", None, C.c_void_p)
    d(lib, "rapdhg_nccl_unique_id", C.c_int, P(C.c_uint8))
    d(lib, "rapdhg_solve_sharded", C.c_int, P(abi.Qp), P(abi.Config), P(abi.ShardOpts), P(abi.Result))
    d(lib, "rapdhg_shard_session_create", C.c_int, P(abi.Qp), P(abi.Config), P(abi.ShardOpts), P(C.c_void_p))
    d(lib, "rapdhg_shard_session_solve", C.c_int, C.c_void_p, P(abi.Result))
    d(lib, "rapdhg_shard_session_destroy", None, C.c_void_p)
    d(lib, "rapdhg_host_transport_check", C.c_int, P(abi.HostTransport), C.c_int32, C.c_int32, C.c_int64)
    d(lib, "rapdhg_canonicalize", C.c_int, P(abi.RawProblem), P(abi.QpOwned), P(abi.CanonicalMap))
    d(lib, "rapdhg_canonical_map_free", None, P(abi.CanonicalMap))
    d(lib, "rapdhg_canonicalize_box", C.c_int, P(abi.RawProblem), P(abi.QpOwned), P(abi.CanonicalMap))
    d(lib, "rapdhg_parse_qps_map", C.c_int, C.c_char_p, P(abi.QpOwned), P(abi.CanonicalMap))
    d(lib, "rapdhg_parse_qps_file_map", C.c_int, C.c_char_p, P(abi.QpOwned), P(abi.CanonicalMap))
    d(lib, "rapdhg_unscale_point", C.c_int, abi.P_f64, abi.P_f64, C.c_int32, C.c_int32, C.c_int32,
      abi.P_f64, abi.P_f64, abi.P_f64)
    d(lib, "rapdhg_scale_point", C.c_int, abi.P_f64, abi.P_f64, C.c_int32, C.c_int32, C.c_int32,
      abi.P_f64, abi.P_f64, abi.P_f64)
    d(lib, "rapdhg_validate", C.c_int, P(abi.Qp))
    d(lib, "rapdhg_symmetry_gap", C.c_int, P(abi.Csr), abi.P_f64)
    d(lib, "rapdhg_primal_weight_init", C.c_int, abi.P_f64, C.c_int64, abi.P_f64, C.c_int64, abi.P_f64)
    if lib.rapdhg_abi_version() != abi.ABI_VERSION:
        raise ImportError("librapdhg_b200.so ABI version mismatch")
    _lib = lib
    return lib


def lib():
    """The loaded C-ABI library (ctypes.CDLL)."""
    return _load()


def _check(rc: int):
    if rc >= 0:
        return rc
    msg = _load().rapdhg_last_error().decode()
    if rc == abi.E_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == abi.E_OUT_OF_RANGE:
        raise IndexError(msg)
    if rc == abi.E_NO_DEVICE:
        raise NoDeviceError(msg)
    if rc == abi.E_CUDA:
        raise CudaError(msg)
    if rc == abi.E_PARSE:
        raise QpsParseError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    return _load().rapdhg_device_count()


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _pf(a: np.ndarray):
    return a.ctypes.data_as(abi.P_f64)


def _pi(a: np.ndarray):
    return a.ctypes.data_as(abi.P_i32)


# --------------------------------------------------------------------------
# model types
# --------------------------------------------------------------------------

class SparseMatrix:
    """Canonical CSR: rows sorted, no duplicates, no explicit zeros
    (sparse.hpp:27-62). Storage: int32 row_ptr/col_idx, fp64 values."""

    def __init__(self, n_rows: int, n_cols: int, triplets: Sequence[Tuple[int, int, float]] = ()):
        if triplets is None:
            triplets = ()
        t = list(triplets)
        r = _i32([e[0] for e in t]) if t else np.zeros(0, np.int32)
        c = _i32([e[1] for e in t]) if t else np.zeros(0, np.int32)
        v = _f64([e[2] for e in t]) if t else np.zeros(0, np.float64)
        self._from_coo(int(n_rows), int(n_cols), r, c, v)

    def _from_coo(self, n_rows, n_cols, r, c, v):
        out = abi.CsrOwned()
        L = _load()
        _check(L.rapdhg_csr_from_triplets(n_rows, n_cols, len(v), _pi(r), _pi(c), _pf(v), C.byref(out)))
        try:
            self.n_rows, self.n_cols = n_rows, n_cols
            nnz = int(out.nnz)
            self.row_ptr = np.ctypeslib.as_array(out.row_ptr, (n_rows + 1,)).copy()
            self.col_idx = (np.ctypeslib.as_array(out.col_idx, (nnz,)).copy() if nnz else np.zeros(0, np.int32))
            self.values = (np.ctypeslib.as_array(out.values, (nnz,)).copy() if nnz else np.zeros(0, np.float64))
        finally:
            L.rapdhg_csr_free(C.byref(out))

    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, vals) -> "SparseMatrix":
        m = cls.__new__(cls)
        m._from_coo(int(n_rows), int(n_cols), _i32(rows), _i32(cols), _f64(vals))
        return m

    @classmethod
    def from_csr(cls, n_rows, n_cols, row_ptr, col_idx, values) -> "SparseMatrix":
        """Adopt arrays that are already canonical (not re-checked here; the
        solver validates ordering and ranges)."""
        m = cls.__new__(cls)
        m.n_rows, m.n_cols = int(n_rows), int(n_cols)
        m.row_ptr, m.col_idx, m.values = _i32(row_ptr), _i32(col_idx), _f64(values)
        return m

    @classmethod
    def identity(cls, n: int) -> "SparseMatrix":
        return cls.from_csr(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    @classmethod
    def zero(cls, n_rows: int, n_cols: int) -> "SparseMatrix":
        return cls.from_csr(n_rows, n_cols, np.zeros(n_rows + 1), np.zeros(0), np.zeros(0))

    def rows(self) -> int:
        return self.n_rows

    def cols(self) -> int:
        return self.n_cols

    def nnz(self) -> int:
        return int(len(self.values))

    def empty(self) -> bool:
        return self.nnz() == 0

    def _csr(self) -> abi.Csr:
        return abi.Csr(self.n_rows, self.n_cols, self.nnz(), _pi(self.row_ptr), _pi(self.col_idx),
                       _pf(self.values))

    def multiply(self, x, strict: bool = False) -> np.ndarray:
        """y = M x on the GPU (sparse.hpp:79-88)."""
        x = _f64(x)
        y = np.empty(self.n_rows, np.float64)
        m = self._csr()
        _check(_load().rapdhg_spmv(C.byref(m), _pf(x), len(x), _pf(y), int(strict)))
        return y

    def multiply_transpose(self, x, strict: bool = False) -> np.ndarray:
        """y = M' x on the GPU (sparse.hpp:91-100)."""
        x = _f64(x)
        y = np.empty(self.n_cols, np.float64)
        m = self._csr()
        _check(_load().rapdhg_spmv_t(C.byref(m), _pf(x), len(x), _pf(y), int(strict)))
        return y

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for r in range(self.n_rows):
            s, e = self.row_ptr[r], self.row_ptr[r + 1]
            d[r, self.col_idx[s:e]] = self.values[s:e]
        return d


def spmv(m: SparseMatrix, x, strict: bool = False) -> np.ndarray:
    return m.multiply(x, strict)


def spmv_t(m: SparseMatrix, x, strict: bool = False) -> np.ndarray:
    return m.multiply_transpose(x, strict)


@dataclass
class QuadraticProgram:
    """min ½x'Qx + c'x + obj_offset  s.t. A_ineq x <= b_ineq, A_eq x = b_eq
    (problem.hpp:24-56)."""
    q: SparseMatrix
    c: np.ndarray
    a_ineq: SparseMatrix
    b_ineq: np.ndarray
    a_eq: SparseMatrix
    b_eq: np.ndarray
    name: str = ""
    obj_offset: float = 0.0
    var_names: List[str] = field(default_factory=list)
    # B200 extension (box_projection): l <= x <= u, None = none
    lower: Optional[np.ndarray] = None
    upper: Optional[np.ndarray] = None

    def num_vars(self) -> int:
        return len(self.c)

    def num_ineq(self) -> int:
        return len(self.b_ineq)

    def num_eq(self) -> int:
        return len(self.b_eq)

    def num_rows(self) -> int:
        return self.num_ineq() + self.num_eq()

    def objective(self, x) -> float:
        """½x'Qx + c'x + obj_offset, evaluated on the host (reporting only)."""
        x = _f64(x)
        q = self.q
        rows = np.repeat(np.arange(q.n_rows), np.diff(q.row_ptr))
        qx = np.bincount(rows, weights=q.values * x[q.col_idx], minlength=q.n_rows)
        return 0.5 * float(x @ qx) + float(self.c @ x) + self.obj_offset

    def validate(self) -> None:
        """QuadraticProgram::validate (problem.hpp:40-50) on the GPU: raises
        InvalidArgument with the reference's messages."""
        qp = self._struct()
        _check(_load().rapdhg_validate(C.byref(qp)))

    def _struct(self) -> abi.Qp:
        self.c, self.b_ineq, self.b_eq = _f64(self.c), _f64(self.b_ineq), _f64(self.b_eq)
        names = None
        if self.var_names:  # kept alive with the struct (it refers to them)
            names = (C.c_char_p * len(self.var_names))(*[v.encode() for v in self.var_names])
        lo = _f64(self.lower) if self.lower is not None else None
        hi = _f64(self.upper) if self.upper is not None else None
        if (lo is not None and len(lo) != len(self.c)) or (hi is not None and len(hi) != len(self.c)):
            raise InvalidArgument("bounds must have num_vars entries")
        s = abi.Qp(len(self.c), len(self.b_ineq), len(self.b_eq), self.q._csr(), _pf(self.c),
                   self.a_ineq._csr(), _pf(self.b_ineq), self.a_eq._csr(), _pf(self.b_eq),
                   float(self.obj_offset), (self.name or "").encode(),
                   C.cast(names, C.POINTER(C.c_char_p)) if names is not None else None,
                   _pf(lo) if lo is not None else None, _pf(hi) if hi is not None else None)
        s._keep = (names, lo, hi)
        return s


@dataclass
class PrimalDualPoint:
    x: np.ndarray
    y_ineq: np.ndarray
    y_eq: np.ndarray

    @staticmethod
    def zeros(p: QuadraticProgram) -> "PrimalDualPoint":
        return PrimalDualPoint(np.zeros(p.num_vars()), np.zeros(p.num_ineq()), np.zeros(p.num_eq()))


class Algorithm(enum.IntEnum):
    kPdhg = 0
    kApdhg = 1


class RestartPolicy(enum.IntEnum):
    kNone = 0
    kFixed = 1
    kAdaptiveHalving = 2
    kPdqpAdaptive = 3


class StepRule(enum.IntEnum):
    kTheoretical = 0
    kAdaptive = 1


class PrimalWeightMode(enum.IntEnum):
    kFixed = 0
    kAdaptive = 1


class SolveStatus(enum.IntEnum):
    kOptimal = 0
    kIterationLimit = 1
    kTimeLimit = 2
    kNumericalError = 3


def to_string(s: SolveStatus) -> str:
    return {0: "optimal", 1: "iteration_limit", 2: "time_limit", 3: "numerical_error"}.get(int(s), "unknown")


@dataclass
class SolverConfig:
    """solver.hpp:38-55 plus the B200 fields."""
    algorithm: Algorithm = Algorithm.kApdhg
    restart: RestartPolicy = RestartPolicy.kPdqpAdaptive
    restart_length: int = 0
    step_rule: StepRule = StepRule.kAdaptive
    primal_weight: PrimalWeightMode = PrimalWeightMode.kAdaptive
    fixed_primal_weight: float = 1.0
    tol: float = 1e-3
    max_iters: int = 200000
    time_limit_s: float = math.inf
    check_interval: int = 40
    scaling: bool = True
    seed: int = 1
    snapshot_interval: int = 0
    record_restart_points: bool = False
    # B200
    device: int = 0
    strict_parity: bool = False
    use_graphs: bool = True
    profile_kernels: int = 0  # 1: CUDA events around the steps of sampled chunks; 2: in-loop step stamps
    box_projection: bool = False  # B200 extension: honour QuadraticProgram.lower / upper by projection

    def _struct(self) -> abi.Config:
        c = abi.Config()
        c.algorithm, c.restart = int(self.algorithm), int(self.restart)
        c.restart_length, c.step_rule = int(self.restart_length), int(self.step_rule)
        c.primal_weight, c.fixed_primal_weight = int(self.primal_weight), float(self.fixed_primal_weight)
        c.tol, c.max_iters, c.time_limit_s = float(self.tol), int(self.max_iters), float(self.time_limit_s)
        c.check_interval, c.scaling, c.seed = int(self.check_interval), int(bool(self.scaling)), int(self.seed)
        c.snapshot_interval = int(self.snapshot_interval)
        c.record_restart_points = int(bool(self.record_restart_points))
        c.device, c.strict_parity = int(self.device), int(bool(self.strict_parity))
        c.use_graphs, c.profile_kernels = int(bool(self.use_graphs)), int(self.profile_kernels)
        c.box_projection = int(bool(self.box_projection))
        return c


@dataclass
class KktResiduals:
    r_primal: float = 0.0
    r_dual: float = 0.0
    r_gap: float = 0.0

    def relkkt(self) -> float:
        return max(self.r_primal, self.r_dual, self.r_gap)


@dataclass
class LogRecord:
    iteration: int
    r_primal: float
    r_dual: float
    r_gap: float
    eta: float
    omega: float
    restarted: bool


@dataclass
class SolveResult:
    status: SolveStatus
    point: PrimalDualPoint
    residuals: KktResiduals
    iterations: int
    restarts: int
    solve_seconds: float
    norm_q: float
    norm_a: float
    norm_fallback: bool
    log: List[LogRecord]
    snapshots: List[Tuple[int, PrimalDualPoint]]
    restart_points: List[PrimalDualPoint]
    # B200 instrumentation
    setup_seconds: float = 0.0
    loop_seconds: float = 0.0
    kernel_launches: int = 0
    kernel_ms: Tuple[float, float] = (0.0, 0.0)
    kernel_count: Tuple[int, int] = (0, 0)


def _arr(p, n) -> np.ndarray:
    if n <= 0:
        return np.zeros(0, np.float64)
    return np.ctypeslib.as_array(p, (n,)).copy()


class _ResultBlock:
    """Owns a C result whose final point (x | y_ineq | y_eq, one block that is
    page-locked when large) numpy views share without a copy; the block goes
    back to the library when the last view is gone."""

    def __init__(self, r: abi.Result):
        self.r = r
        weakref.finalize(self, _free_result, r)

    def view(self, ptr, n) -> np.ndarray:
        if n <= 0:
            return np.zeros(0, np.float64)
        buf = (C.c_double * n).from_address(C.cast(ptr, C.c_void_p).value)
        buf._owner = self  # the numpy view keeps buf, buf keeps the block
        return np.frombuffer(buf, dtype=np.float64)


def _free_result(r):
    _load().rapdhg_result_free(C.byref(r))


def take_result(r: abi.Result) -> SolveResult:
    """result_from_struct, taking ownership of `r`: the point arrays are views
    of the library's result block (no copy); the rest is copied and the C
    arrays are released with the block."""
    try:
        res = result_from_struct(r, point=False)
    except BaseException:
        _free_result(r)
        raise
    blk = _ResultBlock(r)
    res.point = PrimalDualPoint(blk.view(r.x, r.n), blk.view(r.y_ineq, r.m_ineq), blk.view(r.y_eq, r.m_eq))
    return res


def result_from_struct(r: abi.Result, point: bool = True) -> SolveResult:
    """Convert (and copy out of) a C result struct; the caller frees it."""
    n, mi, me = r.n, r.m_ineq, r.m_eq
    m = mi + me
    point = PrimalDualPoint(_arr(r.x, n), _arr(r.y_ineq, mi), _arr(r.y_eq, me)) if point else None
    log = [LogRecord(int(L.iteration), L.r_primal, L.r_dual, L.r_gap, L.eta, L.omega, bool(L.restarted))
           for L in (r.log[i] for i in range(r.n_log))]
    snaps = []
    for s in range(r.n_snapshots):
        xs = np.ctypeslib.as_array(r.snapshot_x, ((s + 1) * n + 1,))[s * n:(s + 1) * n].copy() if n else np.zeros(0)
        ys = np.ctypeslib.as_array(r.snapshot_y, ((s + 1) * m + 1,))[s * m:(s + 1) * m].copy() if m else np.zeros(0)
        snaps.append((int(r.snapshot_iters[s]), PrimalDualPoint(xs, ys[:mi], ys[mi:])))
    rps = []
    for s in range(r.n_restart_points):
        xs = np.ctypeslib.as_array(r.restart_x, ((s + 1) * n + 1,))[s * n:(s + 1) * n].copy() if n else np.zeros(0)
        ys = np.ctypeslib.as_array(r.restart_y, ((s + 1) * m + 1,))[s * m:(s + 1) * m].copy() if m else np.zeros(0)
        rps.append(PrimalDualPoint(xs, ys[:mi], ys[mi:]))
    return SolveResult(SolveStatus(r.status), point,
                       KktResiduals(r.residuals.r_primal, r.residuals.r_dual, r.residuals.r_gap),
                       int(r.iterations), int(r.restarts), r.solve_seconds, r.norm_q, r.norm_a,
                       bool(r.norm_fallback), log, snaps, rps, r.setup_seconds, r.loop_seconds,
                       int(r.kernel_launches), (r.kernel_ms[0], r.kernel_ms[1]),
                       (int(r.kernel_count[0]), int(r.kernel_count[1])))


# --------------------------------------------------------------------------
# solver entry points
# --------------------------------------------------------------------------

def solve(original: QuadraticProgram, cfg: Optional[SolverConfig] = None) -> SolveResult:
    """rapdhg::solve (solver.hpp:272-471) on the GPU."""
    cfg = cfg or SolverConfig()
    L = _load()
    qp = original._struct()
    cs = cfg._struct()
    out = abi.Result()
    _check(L.rapdhg_solve(C.byref(qp), C.byref(cs), C.byref(out)))  # a failed call leaves nothing to free
    return take_result(out)


def shard_plan(p: QuadraticProgram, parts: int) -> Tuple[np.ndarray, np.ndarray]:
    """(dual_bounds, primal_bounds): nnz-balanced contiguous row blocks of the
    row-sharded solver (host computation, works without a GPU)."""
    db, pb = np.zeros(parts + 1, np.int32), np.zeros(parts + 1, np.int32)
    qp = p._struct()
    _check(_load().rapdhg_shard_plan(C.byref(qp), int(parts), _pi(db), _pi(pb)))
    return db, pb


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for a multi-process sharded solve (rank 0)."""
    buf = (C.c_uint8 * 128)()
    _check(_load().rapdhg_nccl_unique_id(buf))
    return bytes(buf)


class ProcessGroupTransport:
    """rapdhg_host_transport over a torch.distributed process group (e.g.
    gloo): the sharded solver's exchanges staged through host memory and done
    with the group's collectives — one process per rank on any backend (and
    several ranks may share a GPU). NCCL (nccl_id) is the fast path."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.errors = []
        self._cbs = (abi.ALLGATHERV_CB(self._allgatherv), abi.ALLTOALLV_CB(self._alltoallv),
                     abi.ALLREDUCE_MIN_CB(self._allreduce_min))
        self.struct = abi.HostTransport(None, *self._cbs)

    def _gather_padded(self, local: np.ndarray):
        """all_gather of variable-length float64 arrays."""
        torch, dist = self.torch, self.dist
        n = torch.tensor([len(local)], dtype=torch.int64)
        ns = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        L = max(max(int(x.item()) for x in ns), 1)
        mine = torch.zeros(L, dtype=torch.float64)
        mine[:len(local)] = torch.from_numpy(np.ascontiguousarray(local))
        out = [torch.empty(L, dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(out, mine, group=self.group)
        return [o[:int(k.item())].numpy() for o, k in zip(out, ns)]

    def _guard(self, f):
        try:
            f()
            return 0
        except Exception as e:  # reported by the library as a failed exchange
            self.errors.append(e)
            return 1

    def _allgatherv(self, ctx, buf, bounds, parts):
        def run():
            b = np.ctypeslib.as_array(bounds, (parts + 1,)).copy()
            total = int(b[-1])
            if total == 0:
                self._gather_padded(np.zeros(0))
                return
            arr = np.ctypeslib.as_array(buf, (total,))
            got = self._gather_padded(arr[b[self.rank]:b[self.rank + 1]])
            for k in range(parts):
                if k != self.rank:
                    arr[b[k]:b[k + 1]] = got[k]
        return self._guard(run)

    def _alltoallv(self, ctx, send, send_off, recv, recv_off, parts):
        def run():
            so = np.ctypeslib.as_array(send_off, (parts + 1,)).copy()
            ro = np.ctypeslib.as_array(recv_off, (parts + 1,)).copy()
            sbuf = np.ctypeslib.as_array(send, (int(so[-1]),)).copy() if so[-1] else np.zeros(0)
            # every rank's packed send buffer and offsets; take this rank's segments
            bufs = self._gather_padded(sbuf)
            offs = self._gather_padded(so.astype(np.float64))
            if ro[-1]:
                rbuf = np.ctypeslib.as_array(recv, (int(ro[-1]),))
                for p in range(parts):
                    if p != self.rank:
                        o = offs[p].astype(np.int64)
                        seg = bufs[p][o[self.rank]:o[self.rank + 1]]
                        if len(seg) != ro[p + 1] - ro[p]:
                            raise RuntimeError("alltoallv: segment sizes disagree")
                        rbuf[ro[p]:ro[p + 1]] = seg
        return self._guard(run)

    def _allreduce_min(self, ctx, value):
        def run():
            t = self.torch.tensor([int(value[0])], dtype=self.torch.int64)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
            value[0] = int(t.item())
        return self._guard(run)

    def check(self, length: int = 1000) -> None:
        """rapdhg_host_transport_check: the library drives these callbacks
        (collective; raises on a wrong delivery)."""
        _check(_load().rapdhg_host_transport_check(C.byref(self.struct), self.world, self.rank, int(length)))


def _shard_opts(parts, emulate, rank, nccl_id, transport=None, replicate_min_len=0) -> abi.ShardOpts:
    opts = abi.ShardOpts()
    opts.parts, opts.rank, opts.emulate = int(parts), int(rank), int(bool(emulate))
    opts.replicate_min_len = int(replicate_min_len or 0)
    if nccl_id is not None:
        C.memmove(opts.nccl_id, nccl_id, 128)
    if transport is not None:
        opts.parts, opts.rank, opts.emulate = transport.world, transport.rank, 0
        opts.host = C.pointer(transport.struct)
    return opts


class ShardSession:
    """Persistent row-sharded solver: setup and (NCCL) communicator once, then
    repeated solves. Collective across ranks when emulate=False."""

    def __init__(self, original: QuadraticProgram, cfg: Optional[SolverConfig] = None, parts: int = 2,
                 emulate: bool = True, rank: int = 0, nccl_id: Optional[bytes] = None,
                 transport: Optional[ProcessGroupTransport] = None, replicate_min_len: int = 0):
        self.cfg = cfg or SolverConfig()
        self._transport = transport  # its callbacks must outlive the session
        h = C.c_void_p()
        qp, cs = original._struct(), self.cfg._struct()
        opts = _shard_opts(parts, emulate, rank, nccl_id, transport, replicate_min_len)
        _check(_load().rapdhg_shard_session_create(C.byref(qp), C.byref(cs), C.byref(opts), C.byref(h)))
        self._h = h

    def solve(self) -> SolveResult:
        L = _load()
        out = abi.Result()
        _check(L.rapdhg_shard_session_solve(self._h, C.byref(out)))
        return take_result(out)

    def close(self):
        if getattr(self, "_h", None):
            _load().rapdhg_shard_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_sharded(original: QuadraticProgram, cfg: Optional[SolverConfig] = None, parts: int = 2,
                  emulate: bool = True, rank: int = 0, nccl_id: Optional[bytes] = None,
                  transport: Optional[ProcessGroupTransport] = None, replicate_min_len: int = 0) -> SolveResult:
    """Row-sharded solve. emulate=True runs all `parts` shards in
    this process on cfg.device (exchanges as device copies); emulate=False is
    one process per GPU, shard `rank`, NCCL communicator from `nccl_id`
    (nccl_unique_id() on rank 0, broadcast by the caller), or the host-staged
    collectives of `transport` (a ProcessGroupTransport: parts and rank come
    from its group). Bit-identical to solve() in fast mode. replicate_min_len
    > 0: rows of [Q | A'] with at least that many entries are replicated
    (rapdhg_shard_opts.replicate_min_len; within rounding of solve(), not
    bit-identical); 0: RAPDHG_REPLICATE_MIN_LEN, else none; < 0: none."""
    cfg = cfg or SolverConfig()
    opts = _shard_opts(parts, emulate, rank, nccl_id, transport, replicate_min_len)
    qp, cs, out = original._struct(), cfg._struct(), abi.Result()
    L = _load()
    _check(L.rapdhg_solve_sharded(C.byref(qp), C.byref(cs), C.byref(opts), C.byref(out)))
    return take_result(out)


class Session:
    """Problem uploaded and preprocessed once (validate, scaling, norms), then
    solved from the zero start as often as wanted on HBM-resident data."""

    def __init__(self, original: QuadraticProgram, cfg: Optional[SolverConfig] = None):
        self.cfg = cfg or SolverConfig()
        self._qp = original
        L = _load()
        h = C.c_void_p()
        qp = original._struct()
        cs = self.cfg._struct()
        _check(L.rapdhg_session_create(C.byref(qp), C.byref(cs), C.byref(h)))
        self._h = h

    def solve(self) -> SolveResult:
        L = _load()
        out = abi.Result()
        _check(L.rapdhg_session_solve(self._h, C.byref(out)))
        return take_result(out)

    def bytes(self) -> Tuple[float, float, float]:
        """(B_iter, bytes of one dual-step launch, bytes of one primal-step launch)."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        _check(_load().rapdhg_session_bytes(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def close(self):
        if getattr(self, "_h", None):
            _load().rapdhg_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class StepParams:
    beta: float = 1.0
    theta: float = 1.0
    eta: float = 0.0
    tau: float = 0.0


@dataclass
class IterateState:
    """solver.hpp:125-143; y stacks [y_ineq | y_eq]."""
    x: np.ndarray
    x_prev: np.ndarray
    y: np.ndarray
    x_bar: np.ndarray
    y_bar: np.ndarray
    k: int = 0
    n: int = 0

    @staticmethod
    def zeros(num_vars: int, num_rows: int) -> "IterateState":
        return IterateState(np.zeros(num_vars), np.zeros(num_vars), np.zeros(num_rows),
                            np.zeros(num_vars), np.zeros(num_rows))

    def copy(self) -> "IterateState":
        return IterateState(self.x.copy(), self.x_prev.copy(), self.y.copy(), self.x_bar.copy(),
                            self.y_bar.copy(), self.k, self.n)


def inner_step(s: IterateState, p: QuadraticProgram, sp: StepParams, steps: int = 1,
               strict: bool = False) -> IterateState:
    """rapdhg::inner_step(s, p, sp) (solver.hpp:156-191), `steps` times."""
    o = s.copy()
    for name in ("x", "x_prev", "y", "x_bar", "y_bar"):
        setattr(o, name, _f64(getattr(o, name)).copy())
    it = abi.Iterate(_pf(o.x), _pf(o.x_prev), _pf(o.y), _pf(o.x_bar), _pf(o.y_bar), o.k, o.n)
    qp = p._struct()
    spc = abi.StepParams(sp.beta, sp.theta, sp.eta, sp.tau)
    _check(_load().rapdhg_inner_step(C.byref(qp), C.byref(it), C.byref(spc), int(steps), int(strict)))
    o.k, o.n = int(it.k), int(it.n)
    return o


def pdhg_step(s: IterateState, p: QuadraticProgram, eta: float, tau: float,
              strict: bool = False) -> IterateState:
    """rapdhg::pdhg_step (solver.hpp:195-203): beta = theta = 1."""
    return inner_step(s, p, StepParams(1.0, 1.0, eta, tau), 1, strict)


def rel_kkt(p: QuadraticProgram, z: PrimalDualPoint, strict: bool = False) -> KktResiduals:
    """rapdhg::rel_kkt (kkt.hpp:28-72) on the GPU."""
    x, yi, ye = _f64(z.x), _f64(z.y_ineq), _f64(z.y_eq)
    out = abi.Kkt()
    qp = p._struct()
    _check(_load().rapdhg_rel_kkt(C.byref(qp), _pf(x), _pf(yi), _pf(ye), C.byref(out), int(strict)))
    return KktResiduals(out.r_primal, out.r_dual, out.r_gap)


@dataclass
class ScalingInfo:
    d1: np.ndarray  # m dual factors
    d2: np.ndarray  # n primal factors

    @staticmethod
    def identity(p: QuadraticProgram) -> "ScalingInfo":
        return ScalingInfo(np.ones(p.num_rows()), np.ones(p.num_vars()))


def compute_scaling(p: QuadraticProgram, strict: bool = False) -> ScalingInfo:
    """scaling.hpp:97-106 on the GPU."""
    d1, d2 = np.empty(p.num_rows()), np.empty(p.num_vars())
    qp = p._struct()
    _check(_load().rapdhg_compute_scaling(C.byref(qp), _pf(d1), _pf(d2), int(strict)))
    return ScalingInfo(d1, d2)


def ruiz_scaling(p: QuadraticProgram, iterations: int, strict: bool = False) -> ScalingInfo:
    """scaling.hpp:85-92 on the GPU."""
    d1, d2 = np.empty(p.num_rows()), np.empty(p.num_vars())
    qp = p._struct()
    _check(_load().rapdhg_ruiz_scaling(C.byref(qp), int(iterations), _pf(d1), _pf(d2), int(strict)))
    return ScalingInfo(d1, d2)


def apply_scaling(p: QuadraticProgram, s: ScalingInfo) -> QuadraticProgram:
    """scaling.hpp:109-123 on the GPU (patterns kept)."""
    if len(s.d2) != p.num_vars() or len(s.d1) != p.num_rows():
        raise InvalidArgument("apply_scaling: dimension mismatch")
    qv, aiv, aev = np.empty(p.q.nnz()), np.empty(p.a_ineq.nnz()), np.empty(p.a_eq.nnz())
    c, bi, be = np.empty(p.num_vars()), np.empty(p.num_ineq()), np.empty(p.num_eq())
    d1, d2 = _f64(s.d1), _f64(s.d2)
    qp = p._struct()
    _check(_load().rapdhg_apply_scaling(C.byref(qp), _pf(d1), _pf(d2), _pf(qv), _pf(aiv), _pf(aev),
                                        _pf(c), _pf(bi), _pf(be)))
    mk = lambda m, v: SparseMatrix.from_csr(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, v)
    return QuadraticProgram(mk(p.q, qv), c, mk(p.a_ineq, aiv), bi, mk(p.a_eq, aev), be, p.name,
                            p.obj_offset, list(p.var_names))


def _point_op(fn, z: PrimalDualPoint, s: ScalingInfo) -> PrimalDualPoint:
    o = PrimalDualPoint(_f64(z.x).copy(), _f64(z.y_ineq).copy(), _f64(z.y_eq).copy())
    d1, d2 = _f64(s.d1), _f64(s.d2)
    if len(d2) != len(o.x) or len(d1) != len(o.y_ineq) + len(o.y_eq):
        raise InvalidArgument("scaling factors do not match the point")
    _check(fn(_pf(d1), _pf(d2), len(o.x), len(o.y_ineq), len(o.y_eq), _pf(o.x), _pf(o.y_ineq), _pf(o.y_eq)))
    return o


def unscale_point(z: PrimalDualPoint, s: ScalingInfo) -> PrimalDualPoint:
    """unscale_point (scaling.hpp:126-133): x = D2 x~, y = D1 y~ (C-ABI, host)."""
    return _point_op(_load().rapdhg_unscale_point, z, s)


def scale_point(z: PrimalDualPoint, s: ScalingInfo) -> PrimalDualPoint:
    """scale_point (scaling.hpp:136-143), the inverse (C-ABI, host)."""
    return _point_op(_load().rapdhg_scale_point, z, s)


def symmetry_gap(m: "SparseMatrix") -> float:
    """SparseMatrix::symmetry_gap (sparse.hpp:119-138) on the GPU."""
    out = C.c_double()
    cm = m._csr()
    _check(_load().rapdhg_symmetry_gap(C.byref(cm), C.byref(out)))
    return out.value


@dataclass
class PowerIterOptions:
    max_iters: int = 5000
    tol: float = 1e-4
    seed: int = 20240601


def estimate_op_norm(m: SparseMatrix, opts: Optional[PowerIterOptions] = None,
                     strict: bool = False) -> float:
    """opnorm.hpp:36-61 on the GPU."""
    o = opts or PowerIterOptions()
    out = C.c_double()
    cm = m._csr()
    _check(_load().rapdhg_estimate_op_norm(C.byref(cm), o.max_iters, o.tol, o.seed, C.byref(out), int(strict)))
    return out.value


def estimate_op_norm_symmetric(m: SparseMatrix, opts: Optional[PowerIterOptions] = None,
                               strict: bool = False) -> float:
    """opnorm.hpp:64-87 on the GPU."""
    o = opts or PowerIterOptions()
    out = C.c_double()
    cm = m._csr()
    _check(_load().rapdhg_estimate_op_norm_symmetric(C.byref(cm), o.max_iters, o.tol, o.seed,
                                                     C.byref(out), int(strict)))
    return out.value


# --- scalar rules (host code of the library; stepsize.hpp) -------------------

def step_schedule_theoretical(k: int, horizon: int, norm_q: float, norm_a: float) -> StepParams:
    o = abi.StepParams()
    _check(_load().rapdhg_step_schedule_theoretical(k, horizon, norm_q, norm_a, C.byref(o)))
    return StepParams(o.beta, o.theta, o.eta, o.tau)


def pdhg_constant_steps(norm_q: float, norm_a: float) -> StepParams:
    o = abi.StepParams()
    _check(_load().rapdhg_pdhg_constant_steps(norm_q, norm_a, C.byref(o)))
    return StepParams(o.beta, o.theta, o.eta, o.tau)


def adaptive_eta(k: int, prev_eta: float, norm_q: float, norm_a: float, omega: float) -> float:
    o = C.c_double()
    _check(_load().rapdhg_adaptive_eta(k, prev_eta, norm_q, norm_a, omega, C.byref(o)))
    return o.value


def primal_weight_init(c, b) -> float:
    """stepsize.hpp:73-78 (C-ABI, host norms in sequential order)."""
    c, b = _f64(c), _f64(b)
    out = C.c_double()
    _check(_load().rapdhg_primal_weight_init(_pf(c), len(c), _pf(b), len(b), C.byref(out)))
    return out.value


def primal_weight_update(delta_x: float, delta_y: float, omega_prev: float) -> float:
    o = C.c_double()
    _check(_load().rapdhg_primal_weight_update(delta_x, delta_y, omega_prev, C.byref(o)))
    return o.value


@dataclass
class RestartContext:
    relkkt_candidate: float = 0.0
    relkkt_candidate_prev: float = 0.0
    relkkt_epoch_start: float = 0.0
    k: int = 0
    total_iters: int = 0


def restart_decision(policy: RestartPolicy, ctx: RestartContext, fixed_length: int = 0) -> bool:
    rc = _check(_load().rapdhg_restart_decision(int(policy), ctx.relkkt_candidate,
                                                ctx.relkkt_candidate_prev, ctx.relkkt_epoch_start,
                                                ctx.k, ctx.total_iters, fixed_length))
    return bool(rc)


# --- QPS I/O (qps.hpp + canonicalize, problem.hpp:131-198) -------------------

def parse_qps(text: str) -> QuadraticProgram:
    """parse_qps + canonicalize of QPS text (host; raises QpsParseError or
    InvalidArgument with the reference's messages)."""
    L = _load()
    o = abi.QpOwned()
    _check(L.rapdhg_parse_qps(text.encode(), C.byref(o)))
    try:
        return qp_from_owned(o)
    finally:
        L.rapdhg_qp_free(C.byref(o))


class RowType(enum.IntEnum):
    """problem.hpp:72"""
    kEq = 0
    kLe = 1
    kGe = 2


@dataclass
class RawProblem:
    """problem.hpp:76-92: typed rows, optional ranges (NaN = none) and variable
    bounds (+-inf allowed), before canonicalize."""
    q: SparseMatrix
    c: np.ndarray
    a: SparseMatrix
    row_types: Sequence[int]
    rhs: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    range: Optional[np.ndarray] = None
    obj_offset: float = 0.0
    name: str = ""
    row_names: List[str] = field(default_factory=list)
    var_names: List[str] = field(default_factory=list)

    def num_vars(self) -> int:
        return len(self.c)

    def num_rows(self) -> int:
        return len(self.rhs)


@dataclass
class CanonicalMap:
    """problem.hpp:95-99"""
    ineq_labels: List[str]
    eq_labels: List[str]


def _names(v):
    return (C.c_char_p * len(v))(*[x.encode() for x in v]) if v else None


def _map_from(m: abi.CanonicalMap) -> CanonicalMap:
    return CanonicalMap([m.ineq_labels[i].decode() for i in range(m.n_ineq)],
                        [m.eq_labels[i].decode() for i in range(m.n_eq)])


def canonicalize(raw: RawProblem, keep_bounds: bool = False) -> Tuple[QuadraticProgram, CanonicalMap]:
    """canonicalize (problem.hpp:131-198) through the C-ABI (host): returns
    CanonicalProblem{qp, map} as a pair. keep_bounds (B200 extension, for
    SolverConfig.box_projection): variable bounds stay in qp.lower / qp.upper
    instead of becoming singleton rows."""
    L = _load()
    n, m = raw.num_vars(), raw.num_rows()
    c, rhs = _f64(raw.c), _f64(raw.rhs)
    lo, up = _f64(raw.lower), _f64(raw.upper)
    rng = _f64(raw.range) if raw.range is not None else None
    rt = _i32(raw.row_types)
    if len(rt) != m or len(lo) != n or len(up) != n or (rng is not None and len(rng) != m):
        raise InvalidArgument("RawProblem: array lengths do not match num_vars / num_rows")
    rn, vn = _names(raw.row_names), _names(raw.var_names)
    st = abi.RawProblem(n, m, raw.q._csr(), _pf(c), float(raw.obj_offset), raw.a._csr(),
                        rt.ctypes.data_as(abi.P_i32), _pf(rhs), _pf(rng) if rng is not None else None,
                        _pf(lo), _pf(up), raw.name.encode(),
                        C.cast(rn, C.POINTER(C.c_char_p)) if rn is not None else None,
                        C.cast(vn, C.POINTER(C.c_char_p)) if vn is not None else None)
    o, mp = abi.QpOwned(), abi.CanonicalMap()
    fn = L.rapdhg_canonicalize_box if keep_bounds else L.rapdhg_canonicalize
    _check(fn(C.byref(st), C.byref(o), C.byref(mp)))
    try:
        return qp_from_owned(o), _map_from(mp)
    finally:
        L.rapdhg_qp_free(C.byref(o))
        L.rapdhg_canonical_map_free(C.byref(mp))


def parse_qps_with_map(text: str) -> Tuple[QuadraticProgram, CanonicalMap]:
    """parse_qps + canonicalize, returning the CanonicalMap too."""
    L = _load()
    o, mp = abi.QpOwned(), abi.CanonicalMap()
    _check(L.rapdhg_parse_qps_map(text.encode(), C.byref(o), C.byref(mp)))
    try:
        return qp_from_owned(o), _map_from(mp)
    finally:
        L.rapdhg_qp_free(C.byref(o))
        L.rapdhg_canonical_map_free(C.byref(mp))


def read_qps(path: str) -> QuadraticProgram:
    """parse_qps_file (qps.hpp:300) + canonicalize."""
    L = _load()
    o = abi.QpOwned()
    _check(L.rapdhg_parse_qps_file(os.fsencode(path), C.byref(o)))
    try:
        return qp_from_owned(o)
    finally:
        L.rapdhg_qp_free(C.byref(o))


def write_qps(p: QuadraticProgram) -> str:
    """write_qps (qps.hpp:320-381) of a canonical problem."""
    L = _load()
    ptr = C.c_void_p()
    qp = p._struct()
    _check(L.rapdhg_write_qps(C.byref(qp), C.byref(ptr)))
    try:
        return C.string_at(ptr).decode()
    finally:
        L.rapdhg_free(ptr)


# --- synthetic instances --------------------------------------

class Gen(enum.IntEnum):
    RANDOM_QP = 1
    LASSO = 2
    PORTFOLIO = 3
    SVM = 4
    LARGE = 5
    LARGE_LOCAL = 6


def qp_from_owned(o: abi.QpOwned, name: str = "") -> QuadraticProgram:
    def csr(m):
        nnz = int(m.nnz)
        rp = np.ctypeslib.as_array(m.row_ptr, (m.n_rows + 1,)).copy()
        ci = np.ctypeslib.as_array(m.col_idx, (nnz,)).copy() if nnz else np.zeros(0, np.int32)
        v = np.ctypeslib.as_array(m.values, (nnz,)).copy() if nnz else np.zeros(0)
        return SparseMatrix.from_csr(m.n_rows, m.n_cols, rp, ci, v)
    if o.name:
        name = o.name.decode()
    var_names = [o.var_names[j].decode() for j in range(o.n)] if o.var_names else []
    return QuadraticProgram(csr(o.q), _arr(o.c, o.n), csr(o.a_ineq), _arr(o.b_ineq, o.m_ineq),
                            csr(o.a_eq), _arr(o.b_eq, o.m_eq), name, o.obj_offset, var_names,
                            _arr(o.lower, o.n) if o.lower else None, _arr(o.upper, o.n) if o.upper else None)


def bounds_from_rows(p: QuadraticProgram) -> QuadraticProgram:
    """Inverse of canonicalize's bound rows (problem.hpp:178-185), for
    SolverConfig.box_projection (B200 extension): every singleton row
    a x_j <= b of the inequality block becomes the bound x_j <= b / a (a > 0)
    or x_j >= b / a (a < 0), the tightest one per variable; the other rows stay
    in order. Host-side, O(nnz)."""
    A, n = p.a_ineq, p.num_vars()
    lens = np.diff(A.row_ptr)
    single = np.flatnonzero(lens == 1)
    single = single[A.values[A.row_ptr[single]] != 0]  # 0 x_j <= b stays a row
    lo = np.full(n, -np.inf) if p.lower is None else _f64(p.lower).copy()
    hi = np.full(n, np.inf) if p.upper is None else _f64(p.upper).copy()
    j = A.col_idx[A.row_ptr[single]]
    a = A.values[A.row_ptr[single]]
    v = _f64(p.b_ineq)[single] / a
    np.minimum.at(hi, j[a > 0], v[a > 0])
    np.maximum.at(lo, j[a < 0], v[a < 0])
    keep = np.ones(A.rows(), bool)
    keep[single] = False
    kept = np.flatnonzero(keep)
    starts, kl = A.row_ptr[:-1][kept], lens[kept]
    idx = np.repeat(starts - np.concatenate([[0], np.cumsum(kl)[:-1]]), kl) + np.arange(int(kl.sum()))
    a2 = SparseMatrix.from_csr(len(kept), n, np.concatenate([[0], np.cumsum(kl)]).astype(np.int32),
                               A.col_idx[idx], A.values[idx])
    return QuadraticProgram(p.q, p.c, a2, _f64(p.b_ineq)[kept], p.a_eq, p.b_eq, p.name, p.obj_offset,
                            list(p.var_names), lo if np.isfinite(lo).any() else None,
                            hi if np.isfinite(hi).any() else None)


def generate(kind: Gen, scale: float = 1.0, seed: int = 1) -> QuadraticProgram:
    """Deterministic synthetic QP of SURVEY §8(d) (C1..C5), host C++."""
    L = _load()
    o = abi.QpOwned()
    _check(L.rapdhg_generate(int(kind), float(scale), int(seed), C.byref(o)))
    try:
        return qp_from_owned(o, f"{Gen(kind).name.lower()}-{scale:g}-{seed}")
    finally:
        L.rapdhg_qp_free(C.byref(o))


__all__ = [
    "SparseMatrix", "QuadraticProgram", "PrimalDualPoint", "SolverConfig", "SolveResult",
    "SolveStatus", "Algorithm", "RestartPolicy", "StepRule", "PrimalWeightMode", "KktResiduals",
    "LogRecord", "IterateState", "StepParams", "ScalingInfo", "PowerIterOptions", "RestartContext",
    "Session", "Gen", "solve", "solve_sharded", "ShardSession", "ProcessGroupTransport", "shard_plan", "nccl_unique_id", "inner_step", "pdhg_step", "rel_kkt", "compute_scaling",
    "ruiz_scaling", "apply_scaling", "unscale_point", "scale_point", "estimate_op_norm",
    "estimate_op_norm_symmetric", "step_schedule_theoretical", "pdhg_constant_steps",
    "adaptive_eta", "primal_weight_init", "primal_weight_update", "restart_decision", "generate",
    "RowType", "RawProblem", "CanonicalMap", "canonicalize", "bounds_from_rows", "parse_qps_with_map", "symmetry_gap",
    "spmv", "spmv_t", "to_string", "parse_qps", "read_qps", "write_qps", "device_count", "lib", "InvalidArgument", "NoDeviceError",
    "CudaError", "QpsParseError",
]
