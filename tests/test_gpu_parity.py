"""GPU parity: the sm_100a kernels through the C-ABI against the oracle.

strict mode (sequential fp64, no FMA) must be BIT-IDENTICAL to the reference
(oracle.ref() where built, else the pinned C port oracle.port(), plus the
golden fixtures made from the reference). Fast mode must match within the
north-star tolerances: iterates at a fixed iteration count within 1e-9
relative, final objective / KKT within 1e-6.
"""
import math
import os

import numpy as np
import pytest

import oracle
import paper_2311_07710_b200 as rb
from instances import csr_from_dense, long_row_qp, one_d, random_qp, random_sparse
from test_oracle import CONFIGS, assert_results_identical, golden_config, golden_problem

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def O():
    oracle.build()
    return oracle.ref() if oracle.have_ref() else oracle.port()


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = max(np.max(np.abs(b)) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b)) / den) if a.size else 0.0


def test_library_is_native_and_device_present():
    assert rb.device_count() >= 1


# ---- SpMV ---------------------------------------------------------------------

@pytest.mark.parametrize("shape,long_rows", [((50, 40), 0), ((300, 2000), 3), ((7, 40000), 2), ((1, 1), 0)])
def test_spmv_strict_bit_exact(O, shape, long_rows):
    M = random_sparse(3, *shape, dens=0.05, long_rows=long_rows)
    g = np.random.default_rng(1)
    x = g.standard_normal(M.n_cols)
    v = g.standard_normal(M.n_rows) * (g.random(M.n_rows) < 0.8)
    assert np.array_equal(M.multiply(x, strict=True), O.spmv(M, x))
    assert np.array_equal(M.multiply_transpose(v, strict=True), O.spmv_t(M, v))


@pytest.mark.parametrize("shape,long_rows", [((300, 2000), 3), ((7, 40000), 2), ((5000, 300), 0)])
def test_spmv_fast_close(O, shape, long_rows):
    M = random_sparse(4, *shape, dens=0.05, long_rows=long_rows)
    g = np.random.default_rng(2)
    x = g.standard_normal(M.n_cols)
    v = g.standard_normal(M.n_rows)
    assert rel_err(M.multiply(x), O.spmv(M, x)) < 1e-13
    assert rel_err(M.multiply_transpose(v), O.spmv_t(M, v)) < 1e-13
    # deterministic: identical on repeat
    assert np.array_equal(M.multiply(x), M.multiply(x))


def test_spmv_spec_examples():
    M = csr_from_dense([[1, 2], [3, 4]])
    assert list(M.multiply([1, -1])) == [-1.0, -1.0]
    assert list(M.multiply_transpose([1, 0])) == [1.0, 2.0]
    assert list(rb.SparseMatrix.zero(2, 3).multiply_transpose([1, 1])) == [0, 0, 0]
    with pytest.raises(rb.InvalidArgument, match="vector length"):
        M.multiply([1.0, 2.0, 3.0])


# ---- inner step / kkt / scaling / norms ------------------------------------------

@pytest.mark.parametrize("strict", [True, False])
def test_inner_step(O, strict):
    p = random_qp(5, n=60, mi=25, me=8)
    g = np.random.default_rng(0)
    s = rb.IterateState(g.standard_normal(60), g.standard_normal(60), np.abs(g.standard_normal(p.num_rows())),
                        g.standard_normal(60), np.abs(g.standard_normal(p.num_rows())), 3, 1)
    for sp in (rb.StepParams(2.5, 0.75, 0.01, 0.02), rb.StepParams(1.0, 1.0, 0.05, 0.05)):
        a, b = rb.inner_step(s, p, sp, 7, strict=strict), O.inner_step(s, p, sp, 7)
        for name in ("x", "x_prev", "y", "x_bar", "y_bar"):
            if strict:
                assert np.array_equal(getattr(a, name), getattr(b, name)), name
            else:
                assert rel_err(getattr(a, name), getattr(b, name)) < 1e-12, name
        assert a.k == b.k == 10
    # SPEC.md:244 single step from 0 on the 1-D instance
    s1 = rb.inner_step(rb.IterateState.zeros(1, 1), one_d(), rb.StepParams(1.0, 0.0, 1 / 24, 1 / 20), strict=strict)
    assert math.isclose(s1.x[0], 1 / 12) and s1.y[0] == 0.0 and math.isclose(s1.x_bar[0], 1 / 12)


@pytest.mark.parametrize("strict", [True, False])
def test_rel_kkt(O, strict):
    for seed in (1, 2):
        p = random_qp(seed, n=70, mi=30, me=9, zero_q=seed == 2)
        g = np.random.default_rng(seed)
        z = rb.PrimalDualPoint(g.standard_normal(70), g.random(p.num_ineq()), g.standard_normal(p.num_eq()))
        a, b = rb.rel_kkt(p, z, strict=strict), O.rel_kkt(p, z)
        if strict:
            assert (a.r_primal, a.r_dual, a.r_gap) == (b.r_primal, b.r_dual, b.r_gap)
        else:
            assert abs(a.r_primal - b.r_primal) < 1e-12 and abs(a.r_dual - b.r_dual) < 1e-12
            assert abs(a.r_gap - b.r_gap) < 1e-10
    k = rb.rel_kkt(one_d(), rb.PrimalDualPoint.zeros(one_d()), strict=strict)
    assert k.r_primal == 0.0 and math.isclose(k.r_dual, 2 / 3) and k.r_gap == 0.0
    with pytest.raises(rb.InvalidArgument, match="negative inequality dual"):
        rb.rel_kkt(one_d(), rb.PrimalDualPoint(np.zeros(1), np.array([-1.0]), np.zeros(0)))


@pytest.mark.parametrize("strict", [True, False])
def test_scaling(O, strict):
    p = random_qp(3, n=90, mi=40, me=10)
    a, b = rb.compute_scaling(p, strict=strict), O.compute_scaling(p)
    if strict:
        assert np.array_equal(a.d1, b.d1) and np.array_equal(a.d2, b.d2)
    else:
        assert rel_err(a.d1, b.d1) < 1e-12 and rel_err(a.d2, b.d2) < 1e-12
    a, b = rb.ruiz_scaling(p, 4, strict=strict), O.ruiz_scaling(p, 4)
    assert np.array_equal(a.d1, b.d1) and np.array_equal(a.d2, b.d2)  # max-abs: order-free, always exact
    sc = rb.apply_scaling(p, b)
    ref_vals = O.apply_scaling(p, b)
    for got, want in zip((sc.q.values, sc.a_ineq.values, sc.a_eq.values, sc.c, sc.b_ineq, sc.b_eq), ref_vals):
        assert np.array_equal(got, want)


@pytest.mark.parametrize("strict", [True, False])
def test_op_norms(O, strict):
    p = random_qp(4, n=80, mi=35, me=7)
    for seed in (1, 20240601):
        opts = rb.PowerIterOptions(seed=seed)
        a = rb.estimate_op_norm_symmetric(p.q, opts, strict=strict)
        b = O.estimate_op_norm_symmetric(p.q, seed=seed)
        assert a == b if strict else abs(a - b) <= 1e-6 * b
        a = rb.estimate_op_norm(p.a_ineq, opts, strict=strict)
        b = O.estimate_op_norm(p.a_ineq, seed=seed)
        assert a == b if strict else abs(a - b) <= 1e-6 * b
    assert abs(rb.estimate_op_norm(csr_from_dense([[0, 2], [0, 0]])) - 2) < 1e-3
    assert rb.estimate_op_norm(rb.SparseMatrix.zero(3, 3)) == 0.0


# ---- full solve ----------------------------------------------------------------------

@pytest.mark.parametrize("cfg_name", sorted(CONFIGS))
@pytest.mark.parametrize("seed", [1, 2])
def test_solve_strict_bit_exact(O, seed, cfg_name):
    """The whole trajectory (log, restarts, snapshots, restart points, final
    point) equals the reference's bit for bit."""
    p = random_qp(seed, n=40, mi=20, me=6, zero_q=(seed == 2 and cfg_name == "default"))
    cfg = rb.SolverConfig(tol=1e-7, max_iters=1500, record_restart_points=True, strict_parity=True,
                          **CONFIGS[cfg_name])
    assert_results_identical(rb.solve(p, cfg), O.solve(p, cfg))


def test_solve_strict_c1_bit_exact(O):
    p = rb.generate(rb.Gen.RANDOM_QP, 1.0, 1)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=2000, snapshot_interval=40, record_restart_points=True,
                          strict_parity=True)
    assert_results_identical(rb.solve(p, cfg), O.solve(p, cfg))


def test_golden_fixtures_strict():
    g = np.load(os.path.join(HERE, "golden", "golden.npz"))
    for case in sorted({k.split("__")[0] for k in g.files}):
        p = golden_problem(g, case)
        r = rb.solve(p, rb.SolverConfig(strict_parity=True, **golden_config(g, case)))
        assert r.iterations == int(g[f"{case}__iterations"]), case
        assert np.array_equal(r.point.x, g[f"{case}__x"]), case
        assert np.array_equal(np.concatenate([r.point.y_ineq, r.point.y_eq]), g[f"{case}__y"]), case
        log = np.array([[L.iteration, L.r_primal, L.r_dual, L.r_gap, L.eta, L.omega, L.restarted] for L in r.log])
        assert np.array_equal(log, g[f"{case}__log"]), case


def _fast_vs_ref(O, p, cfg_kw, max_iters):
    """Fast mode: snapshots (unscaled averages every 40 iterations) within 1e-9
    relative of the reference while the restart decisions agree."""
    cfg = rb.SolverConfig(max_iters=max_iters, snapshot_interval=40, **cfg_kw)
    a = rb.solve(p, cfg)
    b = O.solve(p, cfg)
    agree = 0
    for (ta, za), (tb, zb), la, lb in zip(a.snapshots, b.snapshots, a.log[1:], b.log[1:]):
        assert ta == tb
        if la.restarted != lb.restarted:
            break
        assert rel_err(za.x, zb.x) <= 1e-9, ta
        assert rel_err(np.concatenate([za.y_ineq, za.y_eq]), np.concatenate([zb.y_ineq, zb.y_eq])) <= 1e-9, ta
        agree += 1
    return a, b, agree


@pytest.mark.parametrize("seed", [1, 3])
def test_solve_fast_iterates_within_1e9(O, seed):
    p = random_qp(seed, n=120, mi=50, me=15)
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 800)
    assert agree >= 5
    assert a.norm_q == pytest.approx(b.norm_q, rel=1e-9) and a.norm_a == pytest.approx(b.norm_a, rel=1e-9)


def test_solve_fast_c1_final_within_1e6(O):
    p = rb.generate(rb.Gen.RANDOM_QP, 1.0, 1)
    cfg = rb.SolverConfig(tol=1e-6)
    a, b = rb.solve(p, cfg), O.solve(p, cfg)
    assert a.status == b.status == rb.SolveStatus.kOptimal
    assert abs(p.objective(a.point.x) - p.objective(b.point.x)) <= 1e-6 * max(1.0, abs(p.objective(b.point.x)))
    assert a.residuals.relkkt() <= 1e-6
    assert rel_err(a.point.x, b.point.x) < 1e-4


def test_solve_fast_long_rows(O):
    """Split and block bins (a 40000-nnz row, 3000-nnz rows, singletons)."""
    p = long_row_qp()
    cfg = rb.SolverConfig(tol=1e-12, max_iters=200, snapshot_interval=40)
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 200)
    assert agree >= 3


def test_solve_deterministic():
    p = random_qp(8, n=200, mi=80, me=20)
    cfg = rb.SolverConfig(tol=1e-8, max_iters=3000)
    a, b = rb.solve(p, cfg), rb.solve(p, cfg)
    assert_results_identical(a, b)


def test_solve_edge_cases(O):
    p = one_d()
    r = rb.solve(p, rb.SolverConfig(tol=1e-9))
    assert r.status == rb.SolveStatus.kOptimal
    assert abs(r.point.x[0] - 0.5) < 1e-6 and abs(r.point.y_ineq[0] - 1.0) < 1e-6
    r = rb.solve(p, rb.SolverConfig(max_iters=0))
    assert r.status == rb.SolveStatus.kIterationLimit and r.iterations == 0
    # optimal at iteration 0 (Q=0, c=0, A=[1], b=1)
    q0 = rb.QuadraticProgram(rb.SparseMatrix.zero(1, 1), np.zeros(1), csr_from_dense([[1.0]]), np.ones(1),
                             rb.SparseMatrix.zero(0, 1), np.zeros(0))
    r = rb.solve(q0, rb.SolverConfig())
    assert r.status == rb.SolveStatus.kOptimal and r.iterations == 0
    # equality-only and unconstrained problems
    p2 = random_qp(9, n=30, mi=0, me=10, bounds=False)
    assert_results_identical(rb.solve(p2, rb.SolverConfig(tol=1e-8, strict_parity=True, max_iters=4000)),
                             O.solve(p2, rb.SolverConfig(tol=1e-8, max_iters=4000)))
    p3 = random_qp(10, n=25, mi=0, me=0, bounds=False)
    assert_results_identical(rb.solve(p3, rb.SolverConfig(tol=1e-8, strict_parity=True, max_iters=4000)),
                             O.solve(p3, rb.SolverConfig(tol=1e-8, max_iters=4000)))
    # errors as the reference raises them
    bad = one_d()
    bad.q = csr_from_dense([[2.0, 1.0], [0.0, 1.0]])
    bad.c = np.array([-2.0, 0.0])
    bad.a_ineq = csr_from_dense([[1.0, 0.0]])
    bad.a_eq = rb.SparseMatrix.zero(0, 2)
    with pytest.raises(rb.InvalidArgument, match="Q is not symmetric"):
        rb.solve(bad, rb.SolverConfig())
    with pytest.raises(rb.InvalidArgument, match="check_interval"):
        rb.solve(p, rb.SolverConfig(check_interval=0))
    dim = one_d()
    dim.b_ineq = np.array([0.5, 1.0])
    with pytest.raises(rb.InvalidArgument, match="inequality block dimension mismatch"):
        rb.solve(dim, rb.SolverConfig())
    # per-row CSR structure (checked on the device after the upload, the
    # first offending row as a sequential scan meets it; problem.hpp:40-46)
    def with_a(rp, ci, v, n_rows=3):
        q = random_qp(11, n=6, mi=3, me=0, bounds=False)
        q.a_ineq = rb.SparseMatrix.from_csr(n_rows, 6, rp, ci, v)
        q.b_ineq = np.zeros(n_rows)
        return q
    with pytest.raises(rb.InvalidArgument, match="strictly increasing"):
        rb.solve(with_a([0, 2, 4, 5], [0, 3, 2, 2, 1], [1.0] * 5), rb.SolverConfig())
    with pytest.raises(IndexError, match="out of range"):
        rb.solve(with_a([0, 2, 4, 5], [0, 3, 2, 6, 1], [1.0] * 5), rb.SolverConfig())
    with pytest.raises(rb.InvalidArgument, match="not monotone"):
        rb.solve(with_a([0, 3, 2, 5], [0, 3, 5, 2, 4], [1.0] * 5), rb.SolverConfig())
    # first row wins: an order error in row 0 before a range error in row 2
    with pytest.raises(rb.InvalidArgument, match="strictly increasing"):
        rb.solve(with_a([0, 2, 4, 5], [3, 1, 2, 4, 9], [1.0] * 5), rb.SolverConfig())


def test_numerical_error_status(O):
    """A non-finite iterate stops the solve with kNumericalError at the first
    bad iteration and returns the best checked candidate (solver.hpp:372-373)."""
    p = random_qp(6, n=30, mi=10, me=3)
    p.c = p.c.copy()
    p.c[0] = 1e308
    cfg = rb.SolverConfig(tol=1e-9, max_iters=500, scaling=False)
    a = rb.solve(p, rb.SolverConfig(tol=1e-9, max_iters=500, scaling=False, strict_parity=True))
    b = O.solve(p, cfg)
    assert a.status == b.status == rb.SolveStatus.kNumericalError
    assert a.iterations == b.iterations
    assert np.array_equal(a.point.x, b.point.x)


def test_session_reuse_and_bytes():
    p = rb.generate(rb.Gen.LASSO, 0.02, 2)
    s = rb.Session(p, rb.SolverConfig(tol=1e-4, max_iters=400))
    r1, r2 = s.solve(), s.solve()
    assert_results_identical(r1, r2)
    b_iter, b_dual, b_primal = s.bytes()
    assert b_iter > 0 and b_dual > 0 and b_primal > 0
    s.close()


def test_profile_events_and_no_graph_mode_agree():
    p = random_qp(12, n=150, mi=60, me=10)
    base = rb.solve(p, rb.SolverConfig(tol=1e-8, max_iters=600))
    prof = rb.solve(p, rb.SolverConfig(tol=1e-8, max_iters=600, profile_kernels=True))
    nograph = rb.solve(p, rb.SolverConfig(tol=1e-8, max_iters=600, use_graphs=False))
    assert_results_identical(base, prof)
    assert_results_identical(base, nograph)
    assert prof.kernel_count[0] > 0 and prof.kernel_ms[1] > 0


def test_reference_side_adapter_drop_in():
    """oracle/_ref/adapter_check: rapdhg::solve (the reference) vs
    rapdhg_b200::solve (include/rapdhg_b200_adapter.hpp) on the same
    reference-typed problems — strict bit-identical, fast within tolerance."""
    exe = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "adapter_check")
    if not os.path.exists(exe):
        pytest.skip("adapter_check not built (needs the reference headers at build time)")
    import subprocess
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("bit-identical") == 3


@pytest.fixture
def force_windows(monkeypatch):
    monkeypatch.setenv("RAPDHG_WINDOW", "force")
    yield


def test_staged_windows_strict_bit_exact(O, force_windows):
    """Shared-memory gather windows forced on every schedule: strict mode must
    still be bit-identical (a window only changes where a value is read from)."""
    for seed in (1, 2):
        p = random_qp(seed, n=40, mi=20, me=6)
        cfg = rb.SolverConfig(tol=1e-7, max_iters=1500, record_restart_points=True, strict_parity=True)
        assert_results_identical(rb.solve(p, cfg), O.solve(p, cfg))


def test_staged_windows_fast(O, force_windows, monkeypatch):
    p = rb.generate(rb.Gen.LASSO, 0.02, 2)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=400, snapshot_interval=40)
    a = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_WINDOW", "off")
    b = rb.solve(p, cfg)
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb
        assert np.array_equal(za.x, zb.x), "windows must not change fast-mode results either"
    a2, _, agree = _fast_vs_ref(O, long_row_qp(), dict(tol=1e-12), 160)
    assert agree >= 2


def test_concurrent_solves_are_independent():
    """concurrent solves on independent data are allowed — two
    host threads solving at once (each solve has its own stream, plan threads,
    staging buffers) give exactly the sequential results."""
    import threading
    probs = [rb.generate(rb.Gen.LASSO, 0.05, 2), random_qp(41, n=3000, mi=1200, me=300, dens=0.004, q_rank=800)]
    cfgs = [rb.SolverConfig(tol=1e-6, max_iters=3000), rb.SolverConfig(tol=1e-7, max_iters=2000, strict_parity=True)]
    seq = [rb.solve(p, c) for p, c in zip(probs, cfgs)]
    out = [None, None]
    errs = []

    def run(i):
        try:
            for _ in range(2):
                out[i] = rb.solve(probs[i], cfgs[i])
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for a, b in zip(out, seq):
        assert_results_identical(a, b)


def test_solves_capture_beside_legacy_stream_work():
    """every solve captures its chunk graphs on its own stream. With
    a blocking stream, any legacy-stream operation of the process during a
    capture (another thread's torch kernels on the default stream, a pool
    allocation) invalidates it. The solver's streams are non-blocking and its
    allocations are ordered on them, so fresh sessions (each capturing anew)
    next to a thread hammering the legacy stream still give the sequential
    results. (A device-wide synchronisation — cudaDeviceSynchronize, i.e.
    torch.cuda.synchronize() — from another thread cannot coexist with any
    stream capture in the process, the library's or torch's own, so the noise
    thread synchronises its stream only.)"""
    import threading

    import torch

    p = random_qp(43, n=2000, mi=800, me=200, dens=0.004, q_rank=500)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=1500)
    want = rb.solve(p, cfg)
    stop = threading.Event()
    errs = []

    def legacy_noise():
        try:
            a = torch.randn(512, 512, device="cuda:0")
            while not stop.is_set():
                b = a @ a  # default (legacy) stream kernels and allocator traffic
                a = b / b.norm()
                torch.cuda.current_stream().synchronize()  # not a device-wide sync (see doc)
        except Exception as e:
            errs.append(e)

    def solves(out):
        try:
            for _ in range(6):
                s = rb.Session(p, cfg)
                out.append(s.solve())
                s.close()
        except Exception as e:
            errs.append(e)

    outs = [[], []]
    noise = threading.Thread(target=legacy_noise)
    th = [threading.Thread(target=solves, args=(o,)) for o in outs]
    noise.start()
    for t in th:
        t.start()
    for t in th:
        t.join()
    stop.set()
    noise.join()
    assert not errs, errs
    for o in outs:
        assert len(o) == 6
        for r in o:
            assert_results_identical(r, want)


def _partial_q_qp(seed, n=400, frac=0.3, explicit_zero=False):
    """A QP whose Q lives on a fraction of the variables (like C2's / C4's
    features), so the norm estimate of Q runs on the compacted index set;
    explicit_zero adds a stored 0 outside that set (pattern-asymmetric)."""
    p = random_qp(seed, n=n, mi=150, me=20, dens=0.05)
    g = np.random.default_rng(seed + 7)
    k = int(frac * n)
    idx = np.sort(g.choice(n, k, replace=False))
    M = g.standard_normal((k // 2, k)) * (g.random((k // 2, k)) < 0.2)
    Qk = M.T @ M + 1e-2 * np.eye(k)
    Q = np.zeros((n, n))
    Q[np.ix_(idx, idx)] = 0.5 * (Qk + Qk.T)
    rows, cols = np.nonzero(Q)
    rows, cols, vv = list(rows), list(cols), list(Q[rows, cols])
    if explicit_zero:  # a stored zero in a row the rest of Q never touches
        out = np.setdiff1d(np.arange(n), idx)
        rows.append(int(out[0])), cols.append(int(idx[0])), vv.append(0.0)
    order = np.lexsort((np.array(cols), np.array(rows)))  # CSR by hand: from_coo drops stored zeros
    rows, cols, vv = np.array(rows)[order], np.array(cols)[order], np.array(vv)[order]
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))])
    q = rb.SparseMatrix.from_csr(n, n, rp, cols, vv)
    return rb.QuadraticProgram(q, p.c, p.a_ineq, p.b_ineq, p.a_eq, p.b_eq)


@pytest.mark.parametrize("seed,explicit_zero", [(1, False), (2, True), (3, False)])
def test_compacted_norm_q_matches_reference(O, seed, explicit_zero):
    """Fast mode's norm of Q on the compacted index set (Q touches < half of
    the variables): the reference's estimate within 1e-9, same trajectory."""
    p = _partial_q_qp(seed, explicit_zero=explicit_zero)
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 400)
    assert a.norm_q == pytest.approx(b.norm_q, rel=1e-9) and a.norm_a == pytest.approx(b.norm_a, rel=1e-9)
    assert agree >= 3


@pytest.mark.parametrize("seed", [1, 2])
def test_persistent_chunks_bit_identical(seed, monkeypatch):
    """Small problems run a chunk as one cooperative launch (persistent.cuh):
    the same rowwise tiles as the per-step kernels, so the whole solve is the
    graph-replayed one bit for bit, with one launch per chunk."""
    p = random_qp(seed, n=600, mi=250, me=40, dens=0.05)
    cfg = rb.SolverConfig(tol=1e-10, max_iters=3000, snapshot_interval=100, record_restart_points=True)
    monkeypatch.setenv("RAPDHG_PERSISTENT", "0")
    a = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_PERSISTENT", "1")
    b = rb.solve(p, cfg)
    assert_results_identical(b, a)
    assert b.kernel_launches < a.kernel_launches
    with_box = rb.QuadraticProgram(p.q, p.c, p.a_ineq, p.b_ineq, p.a_eq, p.b_eq,
                                   lower=-np.ones(p.num_vars()), upper=np.ones(p.num_vars()))
    bc = rb.SolverConfig(tol=1e-9, max_iters=2000, box_projection=True)
    monkeypatch.setenv("RAPDHG_PERSISTENT", "0")
    c = rb.solve(with_box, bc)
    monkeypatch.setenv("RAPDHG_PERSISTENT", "1")
    assert_results_identical(rb.solve(with_box, bc), c)
