"""CPU: pin the oracle before trusting it.

* PORT (the C restatement) == REF (the reference compiled unmodified from
  /root/reference) bit for bit on seeded instances and every config variant;
* both reproduce the SPEC.md known answers (adaptive_eta
  uses the code's 0.410071, not the SPEC's mis-evaluated 0.40985);
* both reproduce the committed golden fixtures (tests/golden/).
"""
import math
import os

import numpy as np
import pytest

import oracle
import paper_2311_07710_b200 as rb
from instances import csr_from_dense, one_d, random_qp

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def impls():
    out = [oracle.port()]
    if oracle.have_ref():
        out.append(oracle.ref())
    return out


@pytest.mark.parametrize("which", ["port", "ref"])
def test_spec_known_answers(which):
    if which == "ref" and not oracle.have_ref():
        pytest.skip("reference build absent")
    o = oracle.port() if which == "port" else oracle.ref()
    M = csr_from_dense([[1, 2], [3, 4]])
    assert list(o.spmv(M, [1, -1])) == [-1.0, -1.0]
    assert list(o.spmv_t(M, [1, 0])) == [1.0, 2.0]
    assert list(o.spmv(rb.SparseMatrix.identity(3), [1, 2, 3])) == [1, 2, 3]
    assert list(o.spmv_t(rb.SparseMatrix.zero(2, 3), [1, 1])) == [0, 0, 0]
    D = csr_from_dense([[3, 0], [0, 1]])
    assert abs(o.estimate_op_norm_symmetric(D) - 3) < 1e-3
    assert abs(o.estimate_op_norm(D) - 3) < 1e-3
    assert abs(o.estimate_op_norm(csr_from_dense([[0, 2], [0, 0]])) - 2) < 1e-3
    assert o.estimate_op_norm(rb.SparseMatrix.zero(3, 3)) == 0.0
    sp = o.step_schedule_theoretical(0, 10, 2.0, 1.0)
    assert (sp.beta, sp.theta) == (1.0, 0.0)
    assert math.isclose(sp.eta, 1 / 24) and math.isclose(sp.tau, 1 / 20)
    sp = o.step_schedule_theoretical(9, 10, 2.0, 1.0)
    assert (sp.beta, sp.theta) == (5.5, 0.9)
    assert math.isclose(sp.eta, 10 / 24) and math.isclose(sp.tau, 0.5)
    # adaptive_eta: the code's value 1.98/(2+sqrt(8)) (SPEC arithmetic is wrong)
    assert math.isclose(o.adaptive_eta(0, 0.0, 2.0, 1.0, 1.0), 1.98 / (2 + math.sqrt(8)), rel_tol=1e-15)
    assert math.isclose(o.adaptive_eta(0, 0.0, 2.0, 1.0, 1.0), 0.410071, abs_tol=5e-7)
    assert o.adaptive_eta(1, 0.4, 0.0, 1.0, 1.0) == 0.8
    assert o.primal_weight_init([-2.0], [0.5]) == 4.0
    assert o.primal_weight_init([-2.0], [0.0]) == 1.0
    assert math.isclose(o.primal_weight_update(1, 4, 1), 4 ** 0.2, rel_tol=1e-15)
    assert o.primal_weight_update(0.0, 4, 3.0) == 3.0
    assert math.isclose(o.primal_weight_update(2, 2, 2.0), math.exp(0.8 * math.log(2)), rel_tol=1e-15)
    ctx = rb.RestartContext(0.1, math.inf, 1.0, 5, 100)
    assert o.restart_decision(rb.RestartPolicy.kPdqpAdaptive, ctx)
    assert o.restart_decision(rb.RestartPolicy.kPdqpAdaptive, rb.RestartContext(0.5, 0.4, 1.0, 5, 100))
    assert not o.restart_decision(rb.RestartPolicy.kAdaptiveHalving, rb.RestartContext(0.51, 0, 1.0, 5, 100))
    assert o.restart_decision(rb.RestartPolicy.kFixed, rb.RestartContext(k=10), 10)
    # inner step from 0 on the 1-D instance
    p = one_d()
    s = rb.IterateState.zeros(1, 1)
    s1 = o.inner_step(s, p, rb.StepParams(1.0, 0.0, 1 / 24, 1 / 20))
    assert math.isclose(s1.x[0], 1 / 12) and s1.y[0] == 0.0 and math.isclose(s1.x_bar[0], 1 / 12)
    assert s1.x_prev[0] == 0.0 and s1.k == 1
    # fixed point
    s = rb.IterateState(np.array([0.5]), np.array([0.5]), np.array([1.0]), np.array([0.5]), np.array([1.0]))
    s1 = o.inner_step(s, p, rb.StepParams(1.0, 0.0, 1 / 24, 1 / 20))
    assert s1.x[0] == 0.5 and s1.y[0] == 1.0
    # relKKT(0,0) on 1-D = (0, 2/3, 0)
    k = o.rel_kkt(p, rb.PrimalDualPoint.zeros(p))
    assert k.r_primal == 0.0 and math.isclose(k.r_dual, 2 / 3) and k.r_gap == 0.0
    with pytest.raises(rb.InvalidArgument):
        o.rel_kkt(p, rb.PrimalDualPoint(np.zeros(1), np.array([-1.0]), np.zeros(0)))
    # acceptance 1: the 1-D instance solves to 1e-9
    r = o.solve(p, rb.SolverConfig(tol=1e-9))
    assert r.status == rb.SolveStatus.kOptimal
    assert abs(r.point.x[0] - 0.5) < 1e-6 and abs(r.point.y_ineq[0] - 1.0) < 1e-6
    # max_iters = 0 -> iteration_limit at the initial point
    r = o.solve(p, rb.SolverConfig(max_iters=0))
    assert r.status == rb.SolveStatus.kIterationLimit and r.iterations == 0
    # config validation messages (solver.hpp:57-63)
    with pytest.raises(rb.InvalidArgument, match="tol must be positive"):
        o.solve(p, rb.SolverConfig(tol=0.0))
    with pytest.raises(rb.InvalidArgument, match="restart_length"):
        o.solve(p, rb.SolverConfig(restart=rb.RestartPolicy.kFixed))


def test_port_rejects_asymmetric_q():
    p = one_d()
    p.q = csr_from_dense([[2.0, 1.0], [0.0, 1.0]])
    p.c = np.array([-2.0, 0.0])
    p.a_ineq = csr_from_dense([[1.0, 0.0]])
    p.a_eq = rb.SparseMatrix.zero(0, 2)
    for o in impls():
        with pytest.raises(rb.InvalidArgument, match="Q is not symmetric"):
            o.solve(p, rb.SolverConfig())


CONFIGS = {
    "default": dict(),
    "pdhg_adaptive": dict(algorithm=rb.Algorithm.kPdhg),
    "halving": dict(restart=rb.RestartPolicy.kAdaptiveHalving),
    "fixed_theoretical": dict(restart=rb.RestartPolicy.kFixed, restart_length=64,
                              step_rule=rb.StepRule.kTheoretical),
    "pdqp_theoretical": dict(step_rule=rb.StepRule.kTheoretical),
    "pdhg_theoretical_none": dict(algorithm=rb.Algorithm.kPdhg, restart=rb.RestartPolicy.kNone,
                                  step_rule=rb.StepRule.kTheoretical),
    "no_scaling_fixed_w": dict(scaling=False, primal_weight=rb.PrimalWeightMode.kFixed,
                               fixed_primal_weight=2.0),
    "check7_snap": dict(check_interval=7, snapshot_interval=21),
}


def assert_results_identical(a: rb.SolveResult, b: rb.SolveResult):
    assert a.status == b.status and a.iterations == b.iterations and a.restarts == b.restarts
    assert np.array_equal(a.point.x, b.point.x)
    assert np.array_equal(a.point.y_ineq, b.point.y_ineq) and np.array_equal(a.point.y_eq, b.point.y_eq)
    assert (a.residuals.r_primal, a.residuals.r_dual, a.residuals.r_gap) == (
        b.residuals.r_primal, b.residuals.r_dual, b.residuals.r_gap)
    assert a.norm_q == b.norm_q and a.norm_a == b.norm_a
    assert len(a.log) == len(b.log)
    for la, lb in zip(a.log, b.log):
        assert la == lb
    assert len(a.snapshots) == len(b.snapshots)
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb and np.array_equal(za.x, zb.x) and np.array_equal(za.y_ineq, zb.y_ineq)
    assert len(a.restart_points) == len(b.restart_points)
    for za, zb in zip(a.restart_points, b.restart_points):
        assert np.array_equal(za.x, zb.x) and np.array_equal(za.y_eq, zb.y_eq)


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build absent")
@pytest.mark.parametrize("cfg_name", sorted(CONFIGS))
@pytest.mark.parametrize("seed", [1, 2])
def test_port_matches_reference_solve(seed, cfg_name):
    p = random_qp(seed, n=40, mi=20, me=6, zero_q=(seed == 2 and cfg_name == "default"))
    cfg = rb.SolverConfig(tol=1e-7, max_iters=1500, record_restart_points=True, **CONFIGS[cfg_name])
    assert_results_identical(oracle.port().solve(p, cfg), oracle.ref().solve(p, cfg))


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build absent")
def test_port_matches_reference_c1():
    p = rb.generate(rb.Gen.RANDOM_QP, 1.0, 1)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=2000, snapshot_interval=40, record_restart_points=True)
    assert_results_identical(oracle.port().solve(p, cfg), oracle.ref().solve(p, cfg))


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build absent")
def test_port_matches_reference_kernels():
    p = random_qp(5, n=50, mi=25, me=8)
    P, R = oracle.port(), oracle.ref()
    g = np.random.default_rng(0)
    x = g.standard_normal(50)
    for M in (p.q, p.a_ineq, p.a_eq):
        assert np.array_equal(P.spmv(M, x[:M.n_cols]), R.spmv(M, x[:M.n_cols]))
        v = g.standard_normal(M.n_rows) * (g.random(M.n_rows) < 0.7)
        assert np.array_equal(P.spmv_t(M, v), R.spmv_t(M, v))
    s1, s2 = P.compute_scaling(p), R.compute_scaling(p)
    assert np.array_equal(s1.d1, s2.d1) and np.array_equal(s1.d2, s2.d2)
    s1, s2 = P.ruiz_scaling(p, 3), R.ruiz_scaling(p, 3)
    assert np.array_equal(s1.d1, s2.d1) and np.array_equal(s1.d2, s2.d2)
    for a, b in zip(P.apply_scaling(p, s2), R.apply_scaling(p, s2)):
        assert np.array_equal(a, b)
    for seed in (1, 20240601):
        assert P.estimate_op_norm(p.a_ineq, seed=seed) == R.estimate_op_norm(p.a_ineq, seed=seed)
        assert P.estimate_op_norm_symmetric(p.q, seed=seed) == R.estimate_op_norm_symmetric(p.q, seed=seed)
    z = rb.PrimalDualPoint(g.standard_normal(50), g.random(p.num_ineq()), g.standard_normal(p.num_eq()))
    assert P.rel_kkt(p, z) == R.rel_kkt(p, z)
    s = rb.IterateState(g.standard_normal(50), g.standard_normal(50), np.abs(g.standard_normal(p.num_rows())),
                        g.standard_normal(50), np.abs(g.standard_normal(p.num_rows())), 3, 1)
    for sp in (rb.StepParams(2.5, 0.75, 0.01, 0.02), rb.StepParams(1.0, 1.0, 0.05, 0.05)):
        a, b = P.inner_step(s, p, sp, 5), R.inner_step(s, p, sp, 5)
        for name in ("x", "x_prev", "y", "x_bar", "y_bar"):
            assert np.array_equal(getattr(a, name), getattr(b, name)), name
        assert a.k == b.k == 8
    for k in range(0, 30, 7):
        for prev in (0.0, 0.3):
            assert P.adaptive_eta(k, prev, 1.3, 0.7, 2.0) == R.adaptive_eta(k, prev, 1.3, 0.7, 2.0)
    assert P.symmetry_gap(p.q) == R.symmetry_gap(p.q) == 0.0
    asym = rb.SparseMatrix.from_coo(3, 3, [0, 1, 2, 2], [1, 0, 0, 2], [1.0, 1.5, -2.0, 4.0])
    assert P.symmetry_gap(asym) == R.symmetry_gap(asym) == 2.0


def test_golden_fixtures():
    """The committed fixtures (made by tests/golden/make_golden.py from the
    reference build) are reproduced by every available CPU implementation."""
    path = os.path.join(HERE, "golden", "golden.npz")
    g = np.load(path, allow_pickle=False)
    for case in sorted({k.split("__")[0] for k in g.files}):
        p = golden_problem(g, case)
        cfg = rb.SolverConfig(**golden_config(g, case))
        for o in impls():
            r = o.solve(p, cfg)
            assert r.iterations == int(g[f"{case}__iterations"])
            assert np.array_equal(r.point.x, g[f"{case}__x"])
            assert np.array_equal(np.concatenate([r.point.y_ineq, r.point.y_eq]), g[f"{case}__y"])
            assert np.array_equal(np.array([[L.iteration, L.r_primal, L.r_dual, L.r_gap, L.eta, L.omega,
                                             L.restarted] for L in r.log]), g[f"{case}__log"])


def golden_problem(g, case) -> rb.QuadraticProgram:
    def m(name):
        sh = g[f"{case}__{name}_shape"]
        return rb.SparseMatrix.from_csr(int(sh[0]), int(sh[1]), g[f"{case}__{name}_rp"],
                                        g[f"{case}__{name}_ci"], g[f"{case}__{name}_v"])
    return rb.QuadraticProgram(m("q"), g[f"{case}__c"], m("ai"), g[f"{case}__bi"], m("ae"), g[f"{case}__be"])


def golden_config(g, case) -> dict:
    keys = ["tol", "max_iters", "check_interval"]
    vals = g[f"{case}__cfg"]
    d = dict(zip(keys, vals))
    d["max_iters"] = int(d["max_iters"])
    d["check_interval"] = int(d["check_interval"])
    return d
