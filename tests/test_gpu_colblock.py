"""GPU: L2-sized column blocking (csrc/colblock.cuh). Forced on at test sizes
(RAPDHG_L2BLOCK_KB small, slabs off) it must keep the fast-mode contract
against the reference, agree with the unblocked kernels and stay
deterministic."""
import numpy as np
import pytest

import oracle
import paper_2311_07710_b200 as rb
from instances import random_qp
from test_gpu_parity import _fast_vs_ref, rel_err
from test_oracle import assert_results_identical

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def O():
    oracle.build()
    return oracle.ref() if oracle.have_ref() else oracle.port()


@pytest.fixture
def blocked(monkeypatch):
    monkeypatch.setenv("RAPDHG_SLAB", "off")
    monkeypatch.setenv("RAPDHG_L2BLOCK_KB", "1")  # 128 columns per block


@pytest.mark.parametrize("seed", [1, 4])
def test_colblock_fast_vs_reference(O, seed, blocked):
    p = random_qp(seed, n=600, mi=300, me=60, dens=0.1)
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 600)
    assert agree >= 5


def test_colblock_matches_unblocked(blocked, monkeypatch):
    p = rb.generate(rb.Gen.LASSO, 0.05, 3)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=400, snapshot_interval=40)
    a = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_L2BLOCK", "0")
    b = rb.solve(p, cfg)
    same = True
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb and rel_err(za.x, zb.x) < 1e-10
        same = same and np.array_equal(za.x, zb.x)
    assert not same  # the blocked summation order ran
    monkeypatch.delenv("RAPDHG_L2BLOCK")
    assert_results_identical(a, rb.solve(p, cfg))  # deterministic


def test_colblock_qp_with_q(O, blocked):
    # Q and A' both blocked (primal partials on both accumulators)
    p = random_qp(7, n=800, mi=500, me=100, dens=0.08)
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 400)
    assert agree >= 4


def test_colblock_q_only(O, monkeypatch):
    # n*8 over the block size, m*8 under it: A'y becomes a single partial pass
    monkeypatch.setenv("RAPDHG_SLAB", "off")
    monkeypatch.setenv("RAPDHG_L2BLOCK_KB", "4")
    p = random_qp(11, n=900, mi=300, me=60, dens=0.08)
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 400)
    assert agree >= 4


@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("kb", ["1", "4"])
def test_colblock_sharded_bit_identical(parts, kb, monkeypatch):
    monkeypatch.setenv("RAPDHG_SLAB", "off")
    monkeypatch.setenv("RAPDHG_L2BLOCK_KB", kb)
    p = random_qp(13, n=900, mi=300, me=60, dens=0.08)
    cfg = rb.SolverConfig(tol=1e-8, max_iters=600, snapshot_interval=80)
    assert_results_identical(rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg))
