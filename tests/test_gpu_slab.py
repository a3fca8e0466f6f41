"""GPU: slab-staged gathers (csrc/slab.cuh). Forced on at test sizes
(RAPDHG_SLAB=force) they must keep the fast-mode contract against the
reference, agree with the unstaged kernels, keep the sharded solve
bit-identical, and trigger by themselves on the full C2 Lasso."""
import numpy as np
import pytest

import oracle
import paper_2311_07710_b200 as rb
from instances import long_row_qp, random_qp
from test_gpu_parity import _fast_vs_ref, rel_err
from test_oracle import assert_results_identical

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def O():
    oracle.build()
    return oracle.ref() if oracle.have_ref() else oracle.port()


@pytest.mark.parametrize("resident", ["1", "0"])
@pytest.mark.parametrize("seed", [1, 3])
def test_slab_forced_fast_vs_reference(O, seed, resident, monkeypatch):
    """Both slab modes: resident (every window staged at once, W rows finish
    in the slab kernel) and windowed (per-window partials + finish pass)."""
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    monkeypatch.setenv("RAPDHG_SLAB_RESIDENT", resident)
    p = random_qp(seed, n=300, mi=120, me=30, dens=0.2)
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 600)
    assert agree >= 5


def test_slab_forced_matches_unstaged(monkeypatch):
    p = random_qp(5, n=500, mi=200, me=50, dens=0.15)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=400, snapshot_interval=40)
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    a = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_SLAB", "off")
    b = rb.solve(p, cfg)
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb and rel_err(za.x, zb.x) < 1e-10
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    c = rb.solve(p, cfg)
    assert_results_identical(a, c)  # deterministic


def test_slab_long_rows(O, monkeypatch):
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    a, b, agree = _fast_vs_ref(O, long_row_qp(), dict(tol=1e-12), 160)
    assert agree >= 2


@pytest.mark.parametrize("resident", ["1", "0"])
@pytest.mark.parametrize("parts", [2, 3])
def test_slab_sharded_bit_identical(parts, resident, monkeypatch):
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    monkeypatch.setenv("RAPDHG_SLAB_RESIDENT", resident)
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=2000, snapshot_interval=80)
    assert_results_identical(rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg))


def test_slab_auto_on_c2(monkeypatch):
    """The full C2 Lasso gets slab plans by itself; iterates stay within the
    fast-mode tolerance of the unstaged kernels at a fixed iteration count."""
    p = rb.generate(rb.Gen.LASSO, 1.0, 2)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=200, snapshot_interval=40)
    a = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_SLAB", "off")
    b = rb.solve(p, cfg)
    same = True
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb and rel_err(za.x, zb.x) < 1e-9
        same = same and np.array_equal(za.x, zb.x)
    assert not same  # a different summation order ran: the slab tiles


@pytest.mark.parametrize("mode", ["slab", "colblock"])
def test_forced_paths_edge_problems(O, mode, monkeypatch):
    """Equality-only and unconstrained problems (m = 0: no dual rows, an empty
    A') through the forced slab / column-block paths, against the reference."""
    if mode == "slab":
        monkeypatch.setenv("RAPDHG_SLAB", "force")
    else:
        monkeypatch.setenv("RAPDHG_SLAB", "off")
        monkeypatch.setenv("RAPDHG_L2BLOCK_KB", "1")
    for seed, mi, me in [(9, 0, 10), (10, 0, 0), (12, 40, 0)]:
        p = random_qp(seed, n=300, mi=mi, me=me, bounds=False)
        cfg = rb.SolverConfig(tol=1e-8, max_iters=4000)
        a, b = rb.solve(p, cfg), O.solve(p, cfg)
        assert a.status == b.status
        assert abs(a.iterations - b.iterations) <= 2 * cfg.check_interval
        assert rel_err(a.point.x, b.point.x) < 1e-5


def test_forced_slab_numerical_error(O, monkeypatch):
    """A non-finite iterate under the slab path stops at the reference's
    first bad iteration (the NaN flag sits in the finish epilogue)."""
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    p = random_qp(6, n=300, mi=100, me=30)
    p.c = p.c.copy()
    p.c[0] = 1e308
    cfg = rb.SolverConfig(tol=1e-9, max_iters=500, scaling=False)
    a, b = rb.solve(p, cfg), O.solve(p, cfg)
    assert a.status == b.status == rb.SolveStatus.kNumericalError
    assert a.iterations == b.iterations


def test_slab_many_windows(monkeypatch):
    """More than 64 windows per op (the window table lives in device memory;
    the finish pass sums the partials of 8 windows per warp per round)."""
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    monkeypatch.setenv("RAPDHG_SLAB_WIDTH", "128")
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    assert p.num_vars() // 128 > 64
    cfg = rb.SolverConfig(tol=1e-12, max_iters=400, snapshot_interval=40)
    a = rb.solve(p, cfg)
    assert_results_identical(a, rb.solve(p, cfg))  # deterministic
    assert_results_identical(rb.solve_sharded(p, cfg, 2), a)  # shard-invariant
    monkeypatch.setenv("RAPDHG_SLAB", "off")
    b = rb.solve(p, cfg)
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb and rel_err(za.x, zb.x) < 1e-10 and rel_err(za.y_eq, zb.y_eq) < 1e-10


def test_inloop_step_stamps(monkeypatch):
    """profile_kernels=2 times the slab steps in-loop (no events between the
    steps) and leaves the iterates unchanged."""
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = dict(tol=1e-9, max_iters=800, snapshot_interval=80)
    a = rb.solve(p, rb.SolverConfig(**cfg))
    b = rb.solve(p, rb.SolverConfig(profile_kernels=2, **cfg))
    assert_results_identical(a, b)
    assert b.kernel_count[0] > 0 and b.kernel_count[1] > 0
    assert 0.0 < b.kernel_ms[0] / b.kernel_count[0] < 10.0 and 0.0 < b.kernel_ms[1] / b.kernel_count[1] < 10.0


def test_pdl_schedule_matches_serialised(monkeypatch):
    """The finish kernel's rows without partials read vectors written two
    grids earlier while the slab kernel between them still runs (programmatic
    dependent launches; slab.cuh). Over a 2000-iteration C2-size solve that
    schedule must give bit-identical results to fully serialised launches
    (RAPDHG_PDL=0), and repeat bit for bit."""
    p = rb.generate(rb.Gen.LASSO, 0.5, 2)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=2000, snapshot_interval=400, record_restart_points=True)
    s = rb.Session(p, cfg)
    a = s.solve()
    a2 = s.solve()
    s.close()
    monkeypatch.setenv("RAPDHG_PDL", "0")
    b = rb.solve(p, cfg)
    assert_results_identical(a, a2)
    assert_results_identical(a, b)


@pytest.mark.parametrize("kind, scale, seed", [(rb.Gen.PORTFOLIO, 0.2, 3), (rb.Gen.SVM, 0.1, 4)])
def test_finish_block_order_does_not_change_results(kind, scale, seed, monkeypatch):
    """The finish grid runs its W-row blocks first when they fit two per SM
    (C3's dual) and last otherwise (slab.cuh launch_slab_phase); forcing
    either order (RAPDHG_FINISH_WFIRST) gives bit-identical solves, with and
    without programmatic dependent launches."""
    p = rb.generate(kind, scale, seed)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=400, snapshot_interval=80, record_restart_points=True)
    base = rb.solve(p, cfg)
    for pdl in ("1", "0"):
        monkeypatch.setenv("RAPDHG_PDL", pdl)
        for wfirst in ("0", "1"):
            monkeypatch.setenv("RAPDHG_FINISH_WFIRST", wfirst)
            assert_results_identical(rb.solve(p, cfg), base)


def test_resident_plan_on_c4_svm_dual(monkeypatch):
    """The C4 dual (5 windows over the 1e4 feature columns) qualifies for a
    resident plan (opt-in, RAPDHG_SLAB_RESIDENT=1); at 1/10 scale both modes
    stay within 1e-12 of each other over 200 iterations, and resident repeats
    bit for bit."""
    p = rb.generate(rb.Gen.SVM, 0.1, 4)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=200, snapshot_interval=40)
    monkeypatch.setenv("RAPDHG_SLAB_RESIDENT", "1")
    a = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_SLAB_RESIDENT", "0")
    b = rb.solve(p, cfg)
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb and rel_err(za.x, zb.x) < 1e-12 and rel_err(za.y_ineq, zb.y_ineq) < 1e-12
    monkeypatch.setenv("RAPDHG_SLAB_RESIDENT", "1")
    assert_results_identical(a, rb.solve(p, cfg))


@pytest.mark.parametrize("resident", ["0", "1"])
def test_norm_estimate_switches_to_slab_phases(resident, monkeypatch):
    """The norm estimate of A (opnorm.hpp:36-61) runs its first
    RAPDHG_NORM_SLAB_STEP steps on the rowwise SpMV and the rest on the step's
    slab phases (PhaseSpmvOp): the same estimate up to rounding, deterministic,
    and the sharded setup (which runs the same code on the full matrices)
    gets the same bits."""
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    monkeypatch.setenv("RAPDHG_SLAB_RESIDENT", resident)
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=300, snapshot_interval=60)
    monkeypatch.setenv("RAPDHG_NORM_SLAB_STEP", "-1")
    rowwise = rb.solve(p, cfg)
    for step in ("0", "8", "24"):
        monkeypatch.setenv("RAPDHG_NORM_SLAB_STEP", step)
        a = rb.solve(p, cfg)
        assert a.norm_q == rowwise.norm_q
        assert a.norm_a == pytest.approx(rowwise.norm_a, rel=1e-12)
        assert_results_identical(a, rb.solve(p, cfg))  # deterministic
        for parts in (2, 3):
            assert_results_identical(rb.solve_sharded(p, cfg, parts), a)
