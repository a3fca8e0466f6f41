"""GPU: box projection (the north star's "primal step with box projection"),
an opt-in B200 extension with no reference counterpart — the reference turns
variable bounds into singleton <= rows (canonicalize, problem.hpp:178-185), so
this is not a parity mode. The same bounded problem solved both ways must
reach the same optimum; the box form keeps every iterate inside the bounds,
reports relKKT with the bound multipliers, shards bit-identically and rejects
the combinations that have no meaning."""
import numpy as np
import pytest

import paper_2311_07710_b200 as rb
from instances import random_qp
from test_oracle import assert_results_identical

pytestmark = pytest.mark.gpu


def bounded_raw(seed, n=150, mi=60, me=10, inf_frac=0.3):
    """A feasible convex QP: random_qp's Q, c and row patterns, right-hand
    sides moved so that x = 0 satisfies the rows, and box bounds around 0
    (some infinite)."""
    base = random_qp(seed, n=n, mi=mi, me=me, bounds=False)
    g = np.random.default_rng(seed + 100)
    lo = -g.uniform(0.2, 1.5, n)
    hi = g.uniform(0.2, 1.5, n)
    lo[g.random(n) < inf_frac] = -np.inf
    hi[g.random(n) < inf_frac] = np.inf
    A = rb.SparseMatrix.from_csr(mi + me, n, np.concatenate([base.a_ineq.row_ptr, base.a_ineq.row_ptr[-1] + base.a_eq.row_ptr[1:]]),
                                 np.concatenate([base.a_ineq.col_idx, base.a_eq.col_idx]),
                                 np.concatenate([base.a_ineq.values, base.a_eq.values]))
    # shift the rows so that x = 0 (inside every box) satisfies them strictly / exactly
    b_i = np.abs(base.b_ineq) + 1.0
    b_e = np.zeros(me)
    rows = [int(rb.RowType.kLe)] * mi + [int(rb.RowType.kEq)] * me
    return rb.RawProblem(q=base.q, c=base.c, a=A, row_types=rows, rhs=np.concatenate([b_i, b_e]), lower=lo, upper=hi)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_box_form_reaches_the_rows_form_optimum(seed):
    raw = bounded_raw(seed)
    rows, _ = rb.canonicalize(raw)
    box, _ = rb.canonicalize(raw, keep_bounds=True)
    assert box.num_ineq() < rows.num_ineq() and box.lower is not None
    a = rb.solve(rows, rb.SolverConfig(tol=1e-8, max_iters=200000))
    b = rb.solve(box, rb.SolverConfig(tol=1e-8, max_iters=200000, box_projection=True, snapshot_interval=64))
    assert a.status == b.status == rb.SolveStatus.kOptimal
    assert b.residuals.relkkt() <= 1e-8
    oa, ob = rows.objective(a.point.x), box.objective(b.point.x)
    assert abs(oa - ob) <= 1e-6 * max(1.0, abs(oa)), (oa, ob)
    assert np.max(np.abs(a.point.x - b.point.x)) <= 1e-4 * max(1.0, np.max(np.abs(a.point.x)))
    # inside the box up to a few ulps: the averages are convex combinations of
    # projected iterates, rounded, then unscaled (measured: <= 8e-16 relative)
    lo, hi = box.lower, box.upper
    for x in [b.point.x] + [z.x for _, z in b.snapshots]:
        assert np.all(x >= lo - 2e-15 * np.abs(lo)) and np.all(x <= hi + 2e-15 * np.abs(hi))


def test_box_projection_on_active_bounds():
    """Bounds that bind: min 1/2 |x|^2 - 3 1'x on [0, 1]^n has x* = 1 (all upper
    bounds active, multipliers 2); one slack row (sum x <= 100)."""
    n = 40
    q = rb.SparseMatrix.identity(n)
    a = rb.SparseMatrix.from_csr(1, n, np.array([0, n]), np.arange(n), np.ones(n))
    p = rb.QuadraticProgram(q, -3.0 * np.ones(n), a, np.array([100.0]),
                            rb.SparseMatrix.zero(0, n), np.zeros(0), lower=np.zeros(n), upper=np.ones(n))
    r = rb.solve(p, rb.SolverConfig(tol=1e-9, box_projection=True))
    assert r.status == rb.SolveStatus.kOptimal
    assert np.allclose(r.point.x, 1.0, atol=1e-8)
    assert r.residuals.r_dual <= 1e-9 and r.residuals.r_gap <= 1e-9  # the bound multipliers close the gap


@pytest.mark.parametrize("parts", [2, 3])
def test_box_sharded_bit_identical(parts):
    raw = bounded_raw(5, n=400, mi=150, me=20)
    box, _ = rb.canonicalize(raw, keep_bounds=True)
    cfg = rb.SolverConfig(tol=1e-7, max_iters=4000, snapshot_interval=40, box_projection=True)
    assert_results_identical(rb.solve_sharded(box, cfg, parts), rb.solve(box, cfg))


def test_box_rules():
    raw = bounded_raw(7, n=30, mi=10, me=2)
    box, _ = rb.canonicalize(raw, keep_bounds=True)
    with pytest.raises(rb.InvalidArgument, match="need box_projection"):
        rb.solve(box, rb.SolverConfig())
    with pytest.raises(rb.InvalidArgument, match="strict_parity = 0"):
        rb.solve(box, rb.SolverConfig(box_projection=True, strict_parity=True))
    bad = rb.QuadraticProgram(box.q, box.c, box.a_ineq, box.b_ineq, box.a_eq, box.b_eq,
                              lower=np.ones(30), upper=np.zeros(30))
    with pytest.raises(rb.InvalidArgument, match="infeasible bounds"):
        rb.solve(bad, rb.SolverConfig(box_projection=True))
    # no bounds: box_projection changes nothing (the reference's form, bit for bit)
    rows, _ = rb.canonicalize(raw)
    cfg = rb.SolverConfig(tol=1e-6, max_iters=3000)
    assert_results_identical(rb.solve(rows, cfg), rb.solve(rows, rb.SolverConfig(tol=1e-6, max_iters=3000,
                                                                                  box_projection=True)))
