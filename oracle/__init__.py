"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.

Two CPU implementations of the reference path behind one Python surface:

* ``REF``  — the reference's own headers compiled unmodified into
  ``oracle/_ref/libref_rapdhg.so`` (oracle/Makefile, oracle/ref_capi.cpp);
* ``PORT`` — the plain-C restatement ``oracle/rapdhg_oracle.c`` built into
  ``oracle/_build/liboracle.so``, pinned bit-for-bit to REF and to the SPEC
  known answers by tests/test_oracle.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference /
cpu_baseline legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2311_07710_b200 import abi
import paper_2311_07710_b200 as rb

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libref_rapdhg.so")
PORT_PATH = os.path.join(HERE, "_build", "liboracle.so")


def build(quiet: bool = True) -> None:
    """Compile the checkers (the reference one only where its headers exist)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class OracleError(RuntimeError):
    pass


def _pf(a):
    return a.ctypes.data_as(abi.P_f64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class CpuSolver:
    """ctypes binding of one checker library (prefix ``ref_`` or ``orc_``)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise OracleError(f"{path} not built (run `make -C oracle`)")
        self.path, self.prefix = path, prefix
        L = self.lib = C.CDLL(path)
        P = C.POINTER
        d = lambda name, res, *args: abi.declare(L, prefix + name, res, *args)
        d("last_error", C.c_char_p)
        d("solve", C.c_int, P(abi.Qp), P(abi.Config), P(abi.Result))
        d("result_free", None, P(abi.Result))
        d("spmv", C.c_int, P(abi.Csr), abi.P_f64, C.c_int64, abi.P_f64)
        d("spmv_t", C.c_int, P(abi.Csr), abi.P_f64, C.c_int64, abi.P_f64)
        d("inner_step", C.c_int, P(abi.Qp), P(abi.Iterate), P(abi.StepParams), C.c_int32)
        d("rel_kkt", C.c_int, P(abi.Qp), abi.P_f64, abi.P_f64, abi.P_f64, P(abi.Kkt))
        d("compute_scaling", C.c_int, P(abi.Qp), abi.P_f64, abi.P_f64)
        d("ruiz_scaling", C.c_int, P(abi.Qp), C.c_int32, abi.P_f64, abi.P_f64)
        d("estimate_op_norm", C.c_int, P(abi.Csr), C.c_int32, C.c_double, C.c_uint64, abi.P_f64)
        d("estimate_op_norm_symmetric", C.c_int, P(abi.Csr), C.c_int32, C.c_double, C.c_uint64, abi.P_f64)
        d("step_schedule_theoretical", C.c_int, C.c_int32, C.c_int32, C.c_double, C.c_double, P(abi.StepParams))
        d("pdhg_constant_steps", C.c_int, C.c_double, C.c_double, P(abi.StepParams))
        d("adaptive_eta", C.c_int, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, abi.P_f64)
        d("primal_weight_init", C.c_int, abi.P_f64, C.c_int64, abi.P_f64, C.c_int64, abi.P_f64)
        d("primal_weight_update", C.c_int, C.c_double, C.c_double, C.c_double, abi.P_f64)
        d("restart_decision", C.c_int, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int64,
          C.c_int64, C.c_int64)
        d("symmetry_gap", C.c_int, P(abi.Csr), abi.P_f64)
        if prefix == "ref_":
            d("apply_scaling", C.c_int, P(abi.Qp), abi.P_f64, abi.P_f64, abi.P_f64, abi.P_f64,
              abi.P_f64, abi.P_f64, abi.P_f64, abi.P_f64, abi.P_i64)
            d("parse_qps_canonical", C.c_int, C.c_char_p, P(abi.QpOwned))
            d("parse_qps_map", C.c_int, C.c_char_p, P(abi.QpOwned), P(abi.CanonicalMap))
            d("canonicalize", C.c_int, P(abi.RawProblem), P(abi.QpOwned), P(abi.CanonicalMap))
            d("canonical_map_free", None, P(abi.CanonicalMap))
            d("qp_free", None, P(abi.QpOwned))
            d("write_qps", C.c_int, P(abi.Qp), P(C.c_void_p))
            d("free", None, C.c_void_p)
        else:
            d("apply_scaling", C.c_int, P(abi.Qp), abi.P_f64, abi.P_f64, abi.P_f64, abi.P_f64,
              abi.P_f64, abi.P_f64, abi.P_f64, abi.P_f64)

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc < 0:
            msg = self._fn("last_error")().decode()
            if rc == abi.E_INVALID_ARGUMENT:
                raise rb.InvalidArgument(msg)
            if rc == abi.E_OUT_OF_RANGE:
                raise IndexError(msg)
            raise OracleError(msg)
        return rc

    # -- entry points ---------------------------------------------------------
    def solve(self, p: rb.QuadraticProgram, cfg: rb.SolverConfig) -> rb.SolveResult:
        out = abi.Result()
        qp, cs = p._struct(), cfg._struct()
        self._check(self._fn("solve")(C.byref(qp), C.byref(cs), C.byref(out)))
        try:
            return rb.result_from_struct(out)
        finally:
            self._fn("result_free")(C.byref(out))

    def spmv(self, m: rb.SparseMatrix, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(m.n_rows)
        cm = m._csr()
        self._check(self._fn("spmv")(C.byref(cm), _pf(x), len(x), _pf(y)))
        return y

    def spmv_t(self, m: rb.SparseMatrix, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(m.n_cols)
        cm = m._csr()
        self._check(self._fn("spmv_t")(C.byref(cm), _pf(x), len(x), _pf(y)))
        return y

    def inner_step(self, s: rb.IterateState, p: rb.QuadraticProgram, sp: rb.StepParams,
                   steps: int = 1) -> rb.IterateState:
        o = s.copy()
        for name in ("x", "x_prev", "y", "x_bar", "y_bar"):
            setattr(o, name, _f64(getattr(o, name)).copy())
        it = abi.Iterate(_pf(o.x), _pf(o.x_prev), _pf(o.y), _pf(o.x_bar), _pf(o.y_bar), o.k, o.n)
        qp = p._struct()
        spc = abi.StepParams(sp.beta, sp.theta, sp.eta, sp.tau)
        self._check(self._fn("inner_step")(C.byref(qp), C.byref(it), C.byref(spc), int(steps)))
        o.k, o.n = int(it.k), int(it.n)
        return o

    def rel_kkt(self, p: rb.QuadraticProgram, z: rb.PrimalDualPoint) -> rb.KktResiduals:
        x, yi, ye = _f64(z.x), _f64(z.y_ineq), _f64(z.y_eq)
        out = abi.Kkt()
        qp = p._struct()
        self._check(self._fn("rel_kkt")(C.byref(qp), _pf(x), _pf(yi), _pf(ye), C.byref(out)))
        return rb.KktResiduals(out.r_primal, out.r_dual, out.r_gap)

    def compute_scaling(self, p: rb.QuadraticProgram) -> rb.ScalingInfo:
        d1, d2 = np.empty(p.num_rows()), np.empty(p.num_vars())
        qp = p._struct()
        self._check(self._fn("compute_scaling")(C.byref(qp), _pf(d1), _pf(d2)))
        return rb.ScalingInfo(d1, d2)

    def ruiz_scaling(self, p: rb.QuadraticProgram, iters: int) -> rb.ScalingInfo:
        d1, d2 = np.empty(p.num_rows()), np.empty(p.num_vars())
        qp = p._struct()
        self._check(self._fn("ruiz_scaling")(C.byref(qp), int(iters), _pf(d1), _pf(d2)))
        return rb.ScalingInfo(d1, d2)

    def apply_scaling(self, p: rb.QuadraticProgram, s: rb.ScalingInfo):
        """Scaled (q, a_ineq, a_eq values, c, b_ineq, b_eq)."""
        qv, aiv, aev = np.empty(p.q.nnz()), np.empty(p.a_ineq.nnz()), np.empty(p.a_eq.nnz())
        c, bi, be = np.empty(p.num_vars()), np.empty(p.num_ineq()), np.empty(p.num_eq())
        d1, d2 = _f64(s.d1), _f64(s.d2)
        qp = p._struct()
        args = [C.byref(qp), _pf(d1), _pf(d2), _pf(qv), _pf(aiv), _pf(aev), _pf(c), _pf(bi), _pf(be)]
        if self.prefix == "ref_":
            dropped = C.c_int64()
            args.append(C.byref(dropped))
        self._check(self._fn("apply_scaling")(*args))
        return qv, aiv, aev, c, bi, be

    def estimate_op_norm(self, m: rb.SparseMatrix, max_iters=5000, tol=1e-4, seed=20240601) -> float:
        out = C.c_double()
        cm = m._csr()
        self._check(self._fn("estimate_op_norm")(C.byref(cm), max_iters, tol, seed, C.byref(out)))
        return out.value

    def estimate_op_norm_symmetric(self, m: rb.SparseMatrix, max_iters=5000, tol=1e-4,
                                   seed=20240601) -> float:
        out = C.c_double()
        cm = m._csr()
        self._check(self._fn("estimate_op_norm_symmetric")(C.byref(cm), max_iters, tol, seed, C.byref(out)))
        return out.value

    def step_schedule_theoretical(self, k, horizon, nq, na) -> rb.StepParams:
        o = abi.StepParams()
        self._check(self._fn("step_schedule_theoretical")(k, horizon, nq, na, C.byref(o)))
        return rb.StepParams(o.beta, o.theta, o.eta, o.tau)

    def pdhg_constant_steps(self, nq, na) -> rb.StepParams:
        o = abi.StepParams()
        self._check(self._fn("pdhg_constant_steps")(nq, na, C.byref(o)))
        return rb.StepParams(o.beta, o.theta, o.eta, o.tau)

    def adaptive_eta(self, k, prev, nq, na, omega) -> float:
        o = C.c_double()
        self._check(self._fn("adaptive_eta")(k, prev, nq, na, omega, C.byref(o)))
        return o.value

    def primal_weight_init(self, c, b) -> float:
        c, b = _f64(c), _f64(b)
        o = C.c_double()
        self._check(self._fn("primal_weight_init")(_pf(c), len(c), _pf(b), len(b), C.byref(o)))
        return o.value

    def primal_weight_update(self, dx, dy, w) -> float:
        o = C.c_double()
        self._check(self._fn("primal_weight_update")(dx, dy, w, C.byref(o)))
        return o.value

    def restart_decision(self, policy, ctx: rb.RestartContext, fixed_length=0) -> bool:
        return bool(self._check(self._fn("restart_decision")(
            int(policy), ctx.relkkt_candidate, ctx.relkkt_candidate_prev, ctx.relkkt_epoch_start,
            ctx.k, ctx.total_iters, fixed_length)))

    def symmetry_gap(self, m: rb.SparseMatrix) -> float:
        o = C.c_double()
        cm = m._csr()
        self._check(self._fn("symmetry_gap")(C.byref(cm), C.byref(o)))
        return o.value

    def write_qps(self, p: rb.QuadraticProgram) -> str:
        """qps.hpp write_qps_string (reference build only)."""
        ptr = C.c_void_p()
        qp = p._struct()
        self._check(self._fn("write_qps")(C.byref(qp), C.byref(ptr)))
        try:
            return C.string_at(ptr).decode()
        finally:
            self._fn("free")(ptr)

    def parse_qps(self, text: str) -> rb.QuadraticProgram:
        """qps.hpp parse + problem.hpp canonicalize (reference build only)."""
        o = abi.QpOwned()
        self._check(self._fn("parse_qps_canonical")(text.encode(), C.byref(o)))
        try:
            return rb.qp_from_owned(o)
        finally:
            self._fn("qp_free")(C.byref(o))

    def _canonical(self, call):
        o, mp = abi.QpOwned(), abi.CanonicalMap()
        self._check(call(o, mp))
        try:
            return rb.qp_from_owned(o), rb._map_from(mp)
        finally:
            self._fn("qp_free")(C.byref(o))
            self._fn("canonical_map_free")(C.byref(mp))

    def parse_qps_with_map(self, text: str):
        """parse_qps + canonicalize -> (qp, CanonicalMap) (reference build only)."""
        return self._canonical(lambda o, mp: self._fn("parse_qps_map")(text.encode(), C.byref(o), C.byref(mp)))

    def canonicalize(self, raw: rb.RawProblem):
        """problem.hpp canonicalize of a RawProblem (reference build only)."""
        n, m = raw.num_vars(), raw.num_rows()
        c, rhs, lo, up = _f64(raw.c), _f64(raw.rhs), _f64(raw.lower), _f64(raw.upper)
        rng = _f64(raw.range) if raw.range is not None else None
        rt = np.ascontiguousarray(raw.row_types, dtype=np.int32)
        rn, vn = rb._names(raw.row_names), rb._names(raw.var_names)
        st = abi.RawProblem(n, m, raw.q._csr(), _pf(c), float(raw.obj_offset), raw.a._csr(),
                            rt.ctypes.data_as(abi.P_i32), _pf(rhs), _pf(rng) if rng is not None else None,
                            _pf(lo), _pf(up), raw.name.encode(),
                            C.cast(rn, C.POINTER(C.c_char_p)) if rn is not None else None,
                            C.cast(vn, C.POINTER(C.c_char_p)) if vn is not None else None)
        return self._canonical(lambda o, mp: self._fn("canonicalize")(C.byref(st), C.byref(o), C.byref(mp)))


_cache = {}


def ref() -> CpuSolver:
    """The reference itself (compiled from /root/reference headers)."""
    if "ref" not in _cache:
        _cache["ref"] = CpuSolver(REF_PATH, "ref_")
    return _cache["ref"]


def port() -> CpuSolver:
    """The plain-C restatement."""
    if "port" not in _cache:
        _cache["port"] = CpuSolver(PORT_PATH, "orc_")
    return _cache["port"]


def have_ref() -> bool:
    return os.path.exists(REF_PATH)
