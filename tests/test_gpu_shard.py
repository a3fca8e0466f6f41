"""GPU: the row-sharded solver is bit-identical to the
single-GPU fast solve. Ranks are emulated in one process on the single B200
available (exchanges become device copies of each owner's slice), and the
NCCL transport is exercised with one rank."""
import numpy as np
import pytest

import paper_2311_07710_b200 as rb
from instances import random_qp
from test_oracle import assert_results_identical

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_emulated_shards_bit_identical_lasso(parts):
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=4000, snapshot_interval=80, record_restart_points=True)
    assert_results_identical(rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg))


@pytest.mark.parametrize("parts", [2, 4])
def test_emulated_shards_bit_identical_random(parts):
    p = random_qp(21, n=9000, mi=5000, me=800, dens=0.0015, q_rank=3000)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=1500, snapshot_interval=40, record_restart_points=True)
    a, b = rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg)
    assert_results_identical(a, b)
    db, pb = rb.shard_plan(p, parts)
    assert (np.diff(db) > 0).sum() >= 2 and (np.diff(pb) > 0).sum() >= 2  # really split


@pytest.mark.parametrize("parts", [3, 8])
def test_emulated_shards_unaligned_tail(parts):
    """row counts whose balanced bounds would land past the last
    whole reduction chunk (m = 3500 over 8 parts): the partial chunk must stay
    with a non-empty shard, so the KKT sums and restart distances agree."""
    p = random_qp(41, n=3000, mi=1200, me=300, dens=0.02)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=1200, snapshot_interval=40, record_restart_points=True)
    assert_results_identical(rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg))


def test_emulated_shards_other_configs():
    p = rb.generate(rb.Gen.SVM, 0.004, 4)
    for kw in (dict(restart=rb.RestartPolicy.kAdaptiveHalving),
               dict(step_rule=rb.StepRule.kTheoretical, check_interval=25),
               dict(scaling=False, primal_weight=rb.PrimalWeightMode.kFixed)):
        cfg = rb.SolverConfig(tol=1e-5, max_iters=600, **kw)
        assert_results_identical(rb.solve_sharded(p, cfg, 3), rb.solve(p, cfg))


def test_nccl_transport_single_rank():
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=2000)
    uid = rb.nccl_unique_id()
    assert len(uid) == 128
    a = rb.solve_sharded(p, cfg, parts=1, emulate=False, rank=0, nccl_id=uid)
    assert_results_identical(a, rb.solve(p, cfg))


def test_sharded_rejects_strict():
    p = rb.generate(rb.Gen.LASSO, 0.02, 2)
    with pytest.raises(rb.InvalidArgument, match="strict_parity"):
        rb.solve_sharded(p, rb.SolverConfig(strict_parity=True), 2)


def test_shard_session_repeated_solves():
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=2000)
    base = rb.solve(p, cfg)
    s = rb.ShardSession(p, cfg, parts=3)
    for _ in range(2):
        assert_results_identical(s.solve(), base)
    s.close()
    # one NCCL communicator, several solves
    s = rb.ShardSession(p, cfg, parts=1, emulate=False, rank=0, nccl_id=rb.nccl_unique_id())
    for _ in range(2):
        assert_results_identical(s.solve(), base)
    s.close()


@pytest.mark.parametrize("parts", [2, 3, 8])
@pytest.mark.parametrize("kind", ["lasso", "random", "large_local"])
def test_emulated_halo_exchange_bit_identical(parts, kind, monkeypatch):
    """Per-step exchanges as halos (only the entries each shard's rows
    reference, packed and sent owner-to-peer, the NCCL protocol with device
    copies): still bit-identical to the single-GPU solve."""
    monkeypatch.setenv("RAPDHG_HALO", "on")
    if kind == "lasso":
        p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    elif kind == "random":
        p = random_qp(21, n=9000, mi=5000, me=800, dens=0.0015, q_rank=3000)
    else:  # block-local columns: the case halos are for
        p = rb.generate(rb.Gen.LARGE_LOCAL, 0.002, 5)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=800, snapshot_interval=80, record_restart_points=True)
    assert_results_identical(rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg))
    monkeypatch.setenv("RAPDHG_HALO", "auto")
    assert_results_identical(rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg))


@pytest.mark.parametrize("parts", [2, 4])
@pytest.mark.parametrize("halo", ["on", "off"])
def test_overlapped_exchanges_bit_identical(parts, halo, monkeypatch):
    """Plain-path ops split their rows into interior (all entries owned) and
    boundary rows; the exchanges run on a second stream beside the interior
    rows (graph-captured with a fork / join). Bit-identical to one GPU and to
    the serialised schedule (RAPDHG_OVERLAP=0), halos and allgathers alike."""
    monkeypatch.setenv("RAPDHG_HALO", halo)
    monkeypatch.setenv("RAPDHG_OVERLAP", "1")  # (emulated shards default to the serial schedule)
    p = rb.generate(rb.Gen.LARGE_LOCAL, 0.002, 5)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=800, snapshot_interval=80, record_restart_points=True)
    a = rb.solve_sharded(p, cfg, parts)
    assert_results_identical(a, rb.solve(p, cfg))
    monkeypatch.setenv("RAPDHG_OVERLAP", "0")
    assert_results_identical(a, rb.solve_sharded(p, cfg, parts))


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if a.size else 0.0


def _close_trajectories(a, b, tol=1e-9):
    """Same decisions; iterates within `tol` (the replicated rows' sums are
    associated per shard, so the two runs differ by rounding only)."""
    assert a.status == b.status and a.iterations == b.iterations and a.restarts == b.restarts
    assert [L.restarted for L in a.log] == [L.restarted for L in b.log]
    assert len(a.snapshots) == len(b.snapshots) > 0
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb
        assert _rel(za.x, zb.x) <= tol and _rel(np.concatenate([za.y_ineq, za.y_eq]),
                                                 np.concatenate([zb.y_ineq, zb.y_eq])) <= tol
    assert a.norm_q == b.norm_q and a.norm_a == b.norm_a  # the setup is not sharded


@pytest.mark.parametrize("parts", [2, 3, 4, 8])
@pytest.mark.parametrize("halo", ["auto", "off"])
def test_replicated_dense_rows_svm(parts, halo, monkeypatch):
    """SURVEY §8(e) dense-coupling columns: with RAPDHG_REPLICATE_MIN_LEN the
    SVM's feature rows of [Q | A'] are computed on every shard from per-shard
    partial sums (no y exchange for them): deterministic, and the trajectory of
    one GPU up to rounding."""
    p = rb.generate(rb.Gen.SVM, 0.01, 4)  # 100 feature rows of ~4000 entries
    cfg = rb.SolverConfig(tol=1e-8, max_iters=600, snapshot_interval=40)
    one = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_HALO", halo)
    monkeypatch.setenv("RAPDHG_REPLICATE_MIN_LEN", "100")
    a = rb.solve_sharded(p, cfg, parts)
    assert_results_identical(a, rb.solve_sharded(p, cfg, parts))  # deterministic
    _close_trajectories(a, one)
    # the option overrides the environment: -1 off (bit-identical again), > 0 on
    assert_results_identical(rb.solve_sharded(p, cfg, parts, replicate_min_len=-1), one)
    monkeypatch.delenv("RAPDHG_REPLICATE_MIN_LEN")
    assert_results_identical(rb.solve_sharded(p, cfg, parts, replicate_min_len=100), a)


def test_replicated_rows_other_patterns(monkeypatch):
    """Replication on patterns whose long rows also have Q entries (Lasso) and
    on a random QP, with box bounds, restarts and the time-to-tolerance path."""
    monkeypatch.setenv("RAPDHG_REPLICATE_MIN_LEN", "60")
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = rb.SolverConfig(tol=1e-7, max_iters=3000, snapshot_interval=200)
    a, one = rb.solve_sharded(p, cfg, 3), rb.solve(p, cfg)
    assert a.status == one.status == rb.SolveStatus.kOptimal
    assert abs(p.objective(a.point.x) - p.objective(one.point.x)) <= 1e-6 * max(1.0, abs(p.objective(one.point.x)))
    q = random_qp(22, n=3000, mi=1500, me=200, dens=0.004, q_rank=800)
    lens = np.diff(q.q.row_ptr) + np.bincount(np.concatenate([q.a_ineq.col_idx, q.a_eq.col_idx]), minlength=3000)
    monkeypatch.setenv("RAPDHG_REPLICATE_MIN_LEN", str(int(np.percentile(lens, 90))))
    cfg = rb.SolverConfig(tol=1e-9, max_iters=800, snapshot_interval=40)
    _close_trajectories(rb.solve_sharded(q, cfg, 4), rb.solve(q, cfg))


def test_sharded_setup_norms_both_ways(monkeypatch):
    """The norm estimate of A over the shards (default) and on every rank alone
    (RAPDHG_SHARD_NORMS=0) give the same bits as one GPU, the slab switch
    included."""
    monkeypatch.setenv("RAPDHG_SLAB", "force")
    monkeypatch.setenv("RAPDHG_NORM_SLAB_STEP", "8")
    p = rb.generate(rb.Gen.LASSO, 0.05, 2)
    cfg = rb.SolverConfig(tol=1e-7, max_iters=600, snapshot_interval=100)
    one = rb.solve(p, cfg)
    for flag in ("1", "0"):
        monkeypatch.setenv("RAPDHG_SHARD_NORMS", flag)
        for parts in (2, 4):
            r = rb.solve_sharded(p, cfg, parts)
            assert r.norm_a == one.norm_a and r.norm_q == one.norm_q
            assert_results_identical(r, one)


def test_box_sharded_with_replicated_rows():
    """Box projection and replicated dense rows together (C4's box form, small):
    deterministic, one GPU's trajectory within rounding."""
    p = rb.bounds_from_rows(rb.generate(rb.Gen.SVM, 0.01, 4))
    cfg = rb.SolverConfig(tol=1e-8, max_iters=600, snapshot_interval=40, box_projection=True)
    one = rb.solve(p, cfg)
    a = rb.solve_sharded(p, cfg, 4, replicate_min_len=100)
    assert_results_identical(a, rb.solve_sharded(p, cfg, 4, replicate_min_len=100))
    _close_trajectories(a, one)
