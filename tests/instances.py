"""Shared test instances (numpy-built, deterministic)."""
import numpy as np

import paper_2311_07710_b200 as rb


def csr_from_dense(d):
    d = np.asarray(d, dtype=float)
    r, c = np.nonzero(d)
    return rb.SparseMatrix.from_coo(d.shape[0], d.shape[1], r, c, d[r, c])


def one_d():
    """SPEC.md:244 instance: min x^2 - 2x s.t. x <= 0.5 (x* = 0.5, y* = 1)."""
    return rb.QuadraticProgram(csr_from_dense([[2.0]]), np.array([-2.0]), csr_from_dense([[1.0]]),
                               np.array([0.5]), rb.SparseMatrix.zero(0, 1), np.zeros(0))


def random_qp(seed, n=60, mi=30, me=10, dens=0.1, q_rank=None, bounds=True, zero_q=False):
    """Random convex QP with inequality, equality and bound rows."""
    g = np.random.default_rng(seed)
    if zero_q:
        q = rb.SparseMatrix.zero(n, n)
    else:
        k = q_rank or max(1, n // 2)
        P = g.standard_normal((k, n)) * (g.random((k, n)) < dens)
        Q = P.T @ P + 1e-2 * np.eye(n)
        Q = 0.5 * (Q + Q.T)
        q = csr_from_dense(Q)
    x0 = g.standard_normal(n)
    Ai = g.standard_normal((mi, n)) * (g.random((mi, n)) < dens)
    bi = Ai @ x0 + g.random(mi)
    if bounds:  # finite bounds as singleton <= rows, like canonicalize (problem.hpp:180-185)
        nb = n // 3
        idx = g.choice(n, nb, replace=False)
        B = np.zeros((nb, n))
        B[np.arange(nb), idx] = 1.0
        Ai = np.vstack([Ai, B, -B])
        bi = np.concatenate([bi, x0[idx] + 1.0 + g.random(nb), -(x0[idx] - 1.0 - g.random(nb))])
    Ae = g.standard_normal((me, n)) * (g.random((me, n)) < dens)
    be = Ae @ x0
    c = g.standard_normal(n)
    return rb.QuadraticProgram(q, c, csr_from_dense(Ai), bi, csr_from_dense(Ae), be)


def long_row_qp(seed=7, n=40000):
    """A budget-style dense row (n nnz > split threshold) next to singleton
    rows: exercises the split / block bins of the fast schedule."""
    g = np.random.default_rng(seed)
    d = 1.0 + g.random(n)
    q = rb.SparseMatrix.from_csr(n, n, np.arange(n + 1), np.arange(n), d)
    # eq: sum x = 1 ; ineq: -x <= 0 ; plus 50 medium rows (~3000 nnz)
    rows, cols, vals = [], [], []
    for r in range(50):
        cc = np.unique(g.integers(0, n, 3000))
        rows += [r] * len(cc)
        cols += list(cc)
        vals += list(g.standard_normal(len(cc)))
    rows += list(50 + np.arange(n))
    cols += list(np.arange(n))
    vals += [-1.0] * n
    ai = rb.SparseMatrix.from_coo(50 + n, n, rows, cols, vals)
    bi = np.concatenate([g.random(50) + 1.0, np.zeros(n)])
    ae = rb.SparseMatrix.from_coo(1, n, np.zeros(n, int), np.arange(n), np.ones(n))
    return rb.QuadraticProgram(q, -g.standard_normal(n), ai, bi, ae, np.array([1.0]))


def random_sparse(seed, rows, cols, dens=0.05, long_rows=0, empty_rows=True):
    g = np.random.default_rng(seed)
    r_, c_, v_ = [], [], []
    for r in range(rows):
        if empty_rows and r % 7 == 3:
            continue
        k = g.binomial(cols, dens)
        if r < long_rows:
            k = cols
        cc = g.choice(cols, size=min(k, cols), replace=False)
        r_ += [r] * len(cc)
        c_ += list(cc)
        v_ += list(g.standard_normal(len(cc)))
    return rb.SparseMatrix.from_coo(rows, cols, r_, c_, v_)
