"""GPU: the sliced-ELL path (csrc/sell.cuh) for ops whose rows are all short
— the plain path of C5-L / C1-like problems, the column-block passes of C5-U
and the shards. It must keep the fast-mode contract against the reference,
agree with rowwise_kernel, stay deterministic and keep the sharded solve
bit-identical to one GPU."""
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


def test_sell_plain_path_vs_reference(O):
    p = random_qp(31, n=3000, mi=1200, me=300, dens=0.003, q_rank=200)  # rows well under 64 entries
    a, b, agree = _fast_vs_ref(O, p, dict(tol=1e-12), 600)
    assert agree >= 5


@pytest.mark.parametrize("kind,blocks", [(rb.Gen.LARGE_LOCAL, None), (rb.Gen.LARGE, "64")])
def test_sell_matches_rowwise(kind, blocks, monkeypatch):
    """C5-L (plain path) and C5-U with forced 64 KB column blocks (SELL partial
    passes): both engines within 1e-12, SELL repeatable bit for bit."""
    if blocks:
        monkeypatch.setenv("RAPDHG_L2BLOCK_KB", blocks)
    p = rb.generate(kind, 0.002, 5)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=200, snapshot_interval=40)
    a = rb.solve(p, cfg)
    monkeypatch.setenv("RAPDHG_SELL", "0")
    b = rb.solve(p, cfg)
    for (ta, za), (tb, zb) in zip(a.snapshots, b.snapshots):
        assert ta == tb and rel_err(za.x, zb.x) < 1e-12 and rel_err(za.y_ineq, zb.y_ineq) < 1e-12
    monkeypatch.setenv("RAPDHG_SELL", "1")
    assert_results_identical(a, rb.solve(p, cfg))


@pytest.mark.parametrize("parts", [2, 3])
def test_sell_sharded_bit_identical(parts):
    p = rb.generate(rb.Gen.LARGE_LOCAL, 0.002, 5)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=600, snapshot_interval=40, record_restart_points=True)
    assert_results_identical(rb.solve_sharded(p, cfg, parts), rb.solve(p, cfg))
