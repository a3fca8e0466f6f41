"""CPU: the row-sharding plan and the exchange protocol of the sharded solver
(SURVEY §8(e)), across 2 real processes over torch.distributed/gloo.

The GPU path (sharded.cu) runs per inner step: dual step on owned dual rows ->
allgather-v(y) -> primal step on owned primal rows -> allgather-v(w, x_md).
Here the same protocol runs in numpy on 2 gloo ranks, using the library's own
plan (rapdhg_shard_plan), and must reproduce the unsharded iteration bit for
bit — checking that the plan covers every row exactly once and that the
exchanges deliver everything the next phase gathers."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2311_07710_b200 as rb
from instances import random_qp


def test_plan_properties():
    for kind, scale in ((rb.Gen.LASSO, 0.05), (rb.Gen.SVM, 0.01), (rb.Gen.LARGE, 2e-3), (rb.Gen.PORTFOLIO, 0.01)):
        p = rb.generate(kind, scale, 3)
        n, m = p.num_vars(), p.num_rows()
        for parts in (1, 2, 3, 4, 8):
            db, pb = rb.shard_plan(p, parts)
            assert db[0] == 0 and db[-1] == m and pb[0] == 0 and pb[-1] == n
            assert np.all(np.diff(db) >= 0) and np.all(np.diff(pb) >= 0)
            # reduction chunks: inner bounds are multiples of 2048, never the
            # unaligned end (that would give the last partial chunk to an empty shard)
            assert np.all(db[1:-1] % 2048 == 0) and np.all(pb[1:-1] % 2048 == 0)
    # m = 1500 rows, 8 parts -> every inner bound at 0 or 0 (the
    # whole partial chunk stays with the last, non-empty shard)
    p = random_qp(41, n=3000, mi=1200, me=300)
    db, pb = rb.shard_plan(p, 8)
    assert np.all(db[1:-1] % 2048 == 0) and np.all(pb[1:-1] % 2048 == 0)
    assert db[-2] < db[-1] and pb[-2] < pb[-1]
    # balance on a large enough instance (block size granularity: 2048 rows)
    p = rb.generate(rb.Gen.LARGE, 1e-2, 3)  # n = 1e5, m = 5e4
    db, pb = rb.shard_plan(p, 4)
    a = sp.vstack([csr(p.a_ineq), csr(p.a_eq)]).tocsr()
    cost = np.diff(a.indptr) + 2
    blocks = [cost[db[k]:db[k + 1]].sum() for k in range(4)]
    assert max(blocks) <= 1.5 * cost.sum() / 4


def csr(m: rb.SparseMatrix):
    return sp.csr_matrix((m.values, m.col_idx, m.row_ptr), shape=(m.n_rows, m.n_cols))


def step_full(Q, A, AT, b, c, mi, s, prm):
    x, xp, y, xb, yb = s
    th, ib, omib, eta, tau = prm
    w = th * (x - xp) + x
    y = y + tau * (A @ w - b)
    y[:mi] = np.maximum(y[:mi], 0.0)
    yb = omib * yb + ib * y
    xmd = omib * xb + ib * x
    xn = x - eta * ((Q @ xmd + c) + AT @ y)
    xb = omib * xb + ib * xn
    return [xn, x, y, xb, yb]


def _worker(rank, world, port, q, halo=False):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = random_qp(31, n=5000, mi=3000, me=400, dens=0.002, q_rank=1500)
    Q, A = csr(p.q), sp.vstack([csr(p.a_ineq), csr(p.a_eq)]).tocsr()
    AT, b, c, mi = A.T.tocsr(), np.concatenate([p.b_ineq, p.b_eq]), p.c, p.num_ineq()
    db, pb = rb.shard_plan(p, world)
    d0, d1, p0, p1 = db[rank], db[rank + 1], pb[rank], pb[rank + 1]

    def allgatherv(vec, lo, hi):  # every rank receives every owner's slice
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, vec[lo:hi].copy()))
        out = vec.copy()
        for l_, h_, v in parts:
            out[l_:h_] = v
        return out

    def needed(M, r0, r1):  # sorted columns the rows [r0, r1) of M reference
        return np.unique(M.indices[M.indptr[r0]:M.indptr[r1]])

    def halo_x(vec, M, rows, owners):
        """Halo protocol of sharded.cu (world 2): send the peer the entries of
        its reference set this rank owns, receive the owned-by-peer entries of
        this rank's set; every other non-owned entry stays stale."""
        peer = 1 - rank
        mine = needed(M, rows[rank], rows[rank + 1])
        theirs = needed(M, rows[peer], rows[peer + 1])
        send = theirs[(theirs >= owners[rank]) & (theirs < owners[rank + 1])]
        recv = mine[(mine >= owners[peer]) & (mine < owners[peer + 1])]
        out = vec.copy()
        rb_ = torch.zeros(len(recv), dtype=torch.float64)
        reqs = [dist.isend(torch.from_numpy(vec[send].copy()), peer), dist.irecv(rb_, peer)]
        for r_ in reqs:
            r_.wait()
        out[recv] = rb_.numpy()
        return out

    n, m = p.num_vars(), p.num_rows()
    g = np.random.default_rng(5)
    state = [g.standard_normal(n) * 0.1, np.zeros(n), np.abs(g.standard_normal(m)) * 0.1, np.zeros(n), np.zeros(m)]
    ref = [v.copy() for v in state]
    x, xp, y, xb, yb = [v.copy() for v in state]
    for k in range(12):
        prm = (k / (k + 1), 2.0 / (k + 2), 1 - 2.0 / (k + 2), 0.01, 0.02)
        th, ib, omib, eta, tau = prm
        ref = step_full(Q, A, AT, b, c, mi, ref, prm)
        # primal-owned slices of w and x_md, then exchange (prologue / previous step);
        # halo mode: non-owned entries start as NaN, so any use of an entry the
        # lists missed poisons the result
        w, xmd = np.full(n, np.nan if halo else 0.0), np.full(n, np.nan if halo else 0.0)
        w[p0:p1] = th * (x[p0:p1] - xp[p0:p1]) + x[p0:p1]
        xmd[p0:p1] = omib * xb[p0:p1] + ib * x[p0:p1]
        if halo:
            w, xmd = halo_x(w, A, db, pb), halo_x(xmd, Q, pb, pb)
        else:
            w, xmd = allgatherv(w, p0, p1), allgatherv(xmd, p0, p1)
        # dual step on owned dual rows, exchange y
        yn = y.copy()
        yn[d0:d1] = y[d0:d1] + tau * (A[d0:d1] @ w - b[d0:d1])
        lo, hi = d0, min(d1, mi)
        if hi > lo:
            yn[lo:hi] = np.maximum(yn[lo:hi], 0.0)
        yb[d0:d1] = omib * yb[d0:d1] + ib * yn[d0:d1]
        if halo:
            ys = np.full(m, np.nan)
            ys[d0:d1] = yn[d0:d1]
            y_used = halo_x(ys, AT, pb, db)
        else:
            y_used = allgatherv(yn, d0, d1)
        y = allgatherv(yn, d0, d1)  # the full y for the comparison (checks allgather it too)
        # primal step on owned primal rows
        xn = x.copy()
        xn[p0:p1] = x[p0:p1] - eta * ((Q[p0:p1] @ xmd + c[p0:p1]) + AT[p0:p1] @ y_used)
        xb[p0:p1] = omib * xb[p0:p1] + ib * xn[p0:p1]
        xp, x = x, xn
    x, xb = allgatherv(x, p0, p1), allgatherv(xb, p0, p1)
    yb = allgatherv(yb, d0, d1)
    ok = all(np.array_equal(a, b_) for a, b_ in zip([x, y, xb, yb], [ref[0], ref[2], ref[3], ref[4]]))
    q.put((rank, ok, int(d1 - d0), int(p1 - p0)))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("halo", [False, True])
def test_two_rank_gloo_protocol_matches_unsharded(halo):
    torch_mp = pytest.importorskip("torch.multiprocessing")
    ctx = torch_mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, halo)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    res.sort()
    assert all(ok for _, ok, _, _ in res), res
    assert all(nd > 0 and np_ > 0 for _, _, nd, np_ in res), res  # both ranks own rows


def test_host_structure_validation_messages():
    """The host-side per-row CSR scan (used where no device is involved, e.g.
    the shard plan) reports what the device scan does: the first offending row
    of a sequential scan, with the reference's messages (problem.hpp:40-46)."""
    def with_a(rp, ci):
        q = random_qp(11, n=6, mi=3, me=0, bounds=False)
        q.a_ineq = rb.SparseMatrix.from_csr(3, 6, rp, ci, [1.0] * len(ci))
        q.b_ineq = np.zeros(3)
        return q
    with pytest.raises(rb.InvalidArgument, match="strictly increasing"):
        rb.shard_plan(with_a([0, 2, 4, 5], [0, 3, 2, 2, 1]), 2)
    with pytest.raises(IndexError, match="out of range"):
        rb.shard_plan(with_a([0, 2, 4, 5], [0, 3, 2, 6, 1]), 2)
    with pytest.raises(rb.InvalidArgument, match="not monotone"):
        rb.shard_plan(with_a([0, 3, 2, 5], [0, 3, 5, 2, 4]), 2)
    with pytest.raises(rb.InvalidArgument, match="strictly increasing"):
        rb.shard_plan(with_a([0, 2, 4, 5], [3, 1, 2, 4, 9]), 2)


def test_plan_with_replicated_dense_rows(monkeypatch):
    """RAPDHG_REPLICATE_MIN_LEN: the replicated rows of [Q | A'] (the SVM's
    feature rows) cost nothing in the primal balance, so the primal blocks
    split the other rows evenly; dual entries in replicated columns count
    twice."""
    import paper_2311_07710_b200 as rb

    p = rb.generate(rb.Gen.SVM, 0.01, 4)  # 100 feature rows of ~4000 entries, 10000 slack rows of 2
    cc = np.bincount(p.a_ineq.col_idx, minlength=p.num_vars()) + np.diff(p.q.row_ptr)
    rep = cc >= 100
    assert rep.sum() == 100
    parts = 4
    _, pb0 = rb.shard_plan(p, parts)
    monkeypatch.setenv("RAPDHG_REPLICATE_MIN_LEN", "100")
    db, pb = rb.shard_plan(p, parts)
    assert pb[0] == 0 and pb[-1] == p.num_vars() and np.all(np.diff(pb) >= 0) and np.all(pb[1:-1] % 2048 == 0)
    assert not np.array_equal(pb, pb0)
    # non-replicated primal work per block, within one reduction chunk of even
    cost = np.where(rep, 0, cc) + 2
    per = [cost[pb[k]:pb[k + 1]].sum() for k in range(parts)]
    assert max(per) - min(per) <= 2 * 2048 * (cost.max() + 0)
