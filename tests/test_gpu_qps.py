"""GPU: end-to-end from QPS text — SPEC.md:116/517 fixture solves to objective
-0.75 at x = 0.5, and matches the reference solve of the same parsed problem."""
import pytest

import oracle
import paper_2311_07710_b200 as rb
from test_oracle import assert_results_identical
from test_qps import ONE_D, RICH

pytestmark = pytest.mark.gpu


def test_one_d_fixture_objective():
    p = rb.parse_qps(ONE_D)
    r = rb.solve(p, rb.SolverConfig(tol=1e-9))
    assert r.status == rb.SolveStatus.kOptimal
    assert abs(r.point.x[0] - 0.5) < 1e-6
    assert abs(p.objective(r.point.x) + 0.75) < 1e-6


def test_qps_problems_strict_match_reference():
    O = oracle.ref() if oracle.have_ref() else oracle.port()
    for text in (ONE_D, RICH):
        p = rb.parse_qps(text)
        cfg = rb.SolverConfig(tol=1e-8, max_iters=5000, strict_parity=True)
        assert_results_identical(rb.solve(p, cfg), O.solve(p, cfg))
