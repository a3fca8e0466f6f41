"""CPU: the C-ABI library builds, loads, exports every declared symbol, has
no CPU fallback, and its host-side code (CSR canonicalization, scalar rules,
generators) matches the reference."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import oracle
import paper_2311_07710_b200 as rb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rapdhg_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rapdhg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(rb.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert rb.lib().rapdhg_abi_version() == 2


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {rb.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    if rb.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    M = rb.SparseMatrix.identity(3)
    with pytest.raises(rb.NoDeviceError):
        M.multiply([1.0, 2.0, 3.0])
    from instances import one_d
    with pytest.raises(rb.NoDeviceError):
        rb.solve(one_d(), rb.SolverConfig())
    with pytest.raises(rb.NoDeviceError):
        one_d().validate()
    with pytest.raises(rb.NoDeviceError):
        rb.symmetry_gap(M)


def test_csr_from_triplets_semantics():
    # sparse.hpp:31-62: sort, sum duplicates, drop exact zeros, range check
    M = rb.SparseMatrix(2, 3, [(1, 2, 1.0), (0, 1, 2.0), (1, 2, 2.0), (0, 0, 1.0), (0, 0, -1.0)])
    assert list(M.row_ptr) == [0, 1, 2]
    assert list(M.col_idx) == [1, 2] and list(M.values) == [2.0, 3.0]
    with pytest.raises(IndexError, match="out of range"):
        rb.SparseMatrix(2, 2, [(2, 0, 1.0)])
    if oracle.have_ref():
        g = np.random.default_rng(0)
        r, c, v = g.integers(0, 30, 400), g.integers(0, 20, 400), g.standard_normal(400)
        mine = rb.SparseMatrix.from_coo(30, 20, r, c, v)
        ref = oracle.ref()
        x = g.standard_normal(20)
        assert np.allclose(ref.spmv(mine, x), mine.to_dense() @ x)


def test_scalar_rules_match_reference():
    oracle.build()
    O = oracle.ref() if oracle.have_ref() else oracle.port()
    for k in range(0, 50, 3):
        for prev in (0.0, 0.2, 1.3):
            for om in (0.5, 1.0, 4.0):
                assert rb.adaptive_eta(k, prev, 1.7, 0.9, om) == O.adaptive_eta(k, prev, 1.7, 0.9, om)
    for K in (1, 10, 160):
        for k in range(0, K, max(1, K // 7)):
            a, b = rb.step_schedule_theoretical(k, K, 2.0, 0.5), O.step_schedule_theoretical(k, K, 2.0, 0.5)
            assert a == b
    assert rb.step_schedule_theoretical(0, 10, 2.0, 0.0) == O.step_schedule_theoretical(0, 10, 2.0, 0.0)
    assert rb.pdhg_constant_steps(2.0, 1.0) == O.pdhg_constant_steps(2.0, 1.0)
    assert rb.pdhg_constant_steps(2.0, 0.0) == O.pdhg_constant_steps(2.0, 0.0)
    for dx, dy, w in ((1, 4, 1), (0, 1, 2), (2, 2, 2), (3.5, 1e-3, 0.7)):
        assert rb.primal_weight_update(dx, dy, w) == O.primal_weight_update(dx, dy, w)
    for pol in rb.RestartPolicy:
        for ctx in (rb.RestartContext(0.1, 0.05, 1.0, 10, 100), rb.RestartContext(0.7, 0.6, 1.0, 10, 100),
                    rb.RestartContext(0.9, 0.6, 1.0, 40, 100), rb.RestartContext(0.5, math.inf, 1.0, 3, 10)):
            assert rb.restart_decision(pol, ctx, 10) == O.restart_decision(pol, ctx, 10)
    with pytest.raises(rb.InvalidArgument, match="omega must be positive"):
        rb.adaptive_eta(0, 0.0, 1.0, 1.0, 0.0)
    with pytest.raises(rb.InvalidArgument, match="k out of range"):
        rb.step_schedule_theoretical(10, 10, 1.0, 1.0)


@pytest.mark.parametrize("kind,scale", [(rb.Gen.RANDOM_QP, 0.2), (rb.Gen.LASSO, 0.01), (rb.Gen.PORTFOLIO, 0.002),
                                        (rb.Gen.SVM, 0.001), (rb.Gen.LARGE, 1e-5), (rb.Gen.LARGE_LOCAL, 1e-5)])
def test_generators_deterministic_and_canonical(kind, scale):
    a, b = rb.generate(kind, scale, 5), rb.generate(kind, scale, 5)
    for m1, m2 in ((a.q, b.q), (a.a_ineq, b.a_ineq), (a.a_eq, b.a_eq)):
        assert np.array_equal(m1.row_ptr, m2.row_ptr) and np.array_equal(m1.values, m2.values)
        for r in range(m1.n_rows):
            cols = m1.col_idx[m1.row_ptr[r]:m1.row_ptr[r + 1]]
            assert np.all(np.diff(cols) > 0)
        assert np.all(m1.values != 0)
    assert np.array_equal(a.c, b.c) and np.array_equal(a.b_ineq, b.b_ineq)
    Q = a.q.to_dense() if a.num_vars() < 3000 else None
    if Q is not None:
        assert np.array_equal(Q, Q.T)
        assert np.linalg.eigvalsh(Q).min() > -1e-9


def test_generator_sizes_match_survey():
    """C2 Lasso headline sizes: n = m = 210,000, nnz(A) ~ 1.041e7."""
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    nf, ns = 5000, 500
    assert p.num_vars() == 2 * nf + ns and p.num_rows() == 2 * nf + ns
    assert p.num_eq() == ns and p.num_ineq() == 2 * nf


def test_point_scaling_and_primal_weight_init_match_reference():
    """unscale_point / scale_point (scaling.hpp:126-143) and primal_weight_init
    (stepsize.hpp:73-78) through the C-ABI: the reference's arithmetic."""
    g = np.random.default_rng(3)
    n, mi, me = 50, 20, 7
    s = rb.ScalingInfo(g.uniform(0.1, 3, mi + me), g.uniform(0.1, 3, n))
    z = rb.PrimalDualPoint(g.standard_normal(n), g.random(mi), g.standard_normal(me))
    u = rb.unscale_point(z, s)
    assert np.array_equal(u.x, z.x * s.d2) and np.array_equal(u.y_ineq, z.y_ineq * s.d1[:mi])
    assert np.array_equal(u.y_eq, z.y_eq * s.d1[mi:])
    back = rb.scale_point(u, s)
    assert np.allclose(back.x, z.x, rtol=1e-14) and np.allclose(back.y_eq, z.y_eq, rtol=1e-14)
    with pytest.raises(rb.InvalidArgument):
        rb.unscale_point(z, rb.ScalingInfo(s.d1[:-1], s.d2))
    ref = oracle.ref() if oracle.have_ref() else oracle.port()
    for c, b in ((g.standard_normal(40), g.standard_normal(9)), (np.zeros(3), np.ones(2)), ([-2.0], [0.5])):
        assert rb.primal_weight_init(c, b) == ref.primal_weight_init(c, b)
    assert rb.primal_weight_init([-2.0], [0.5]) == 4.0
