"""TEST / REFERENCE-ARM INFRASTRUCTURE — numpy restatement of the counter-based
synthetic generators (paper_2311_07710_b200/csrc/crng.h, host.cpp gen_svm).

The reference ships no generators, so the instances are
builder-defined. The B200 library builds them in C++ (host) or CUDA (device);
this module rebuilds the SAME arrays bit for bit with numpy only, so that
``bench.py --impl reference`` can feed the reference solver without loading
any of the repository's native libraries. tests/test_generators.py pins it to
the library's generator.

Every draw is a pure function of (seed, tag, index) through splitmix64 mixing;
uniforms are 53-bit; normals are Irwin-Hall sums of 12 uniforms added in order
(only IEEE-exact operations, so numpy, C++ and CUDA agree).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

M1 = np.uint64(0x9E3779B97F4A7C15)
M2 = np.uint64(0xBF58476D1CE4E5B9)
M3 = np.uint64(0x94D049BB133111EB)
P = np.uint64(0x100000001B3)
K_SVM_COL, K_SVM_VAL = 8, 9  # crng.h Tag


def mix64(x):
    """splitmix64 finaliser (crng.h mix64), elementwise on uint64 arrays."""
    with np.errstate(over="ignore"):
        x = x + M1
        x = (x ^ (x >> np.uint64(30))) * M2
        x = (x ^ (x >> np.uint64(27))) * M3
        return x ^ (x >> np.uint64(31))


def _tag_key(seed: int, tag: int):
    return mix64(np.array([(seed ^ (tag << 56)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]


def uniform(seed: int, tag: int, i, k):
    """crng.h uniform(seed, tag, i, k) in [0, 1) for arrays i (uint64), k."""
    with np.errstate(over="ignore"):
        h = mix64(_tag_key(seed, tag) ^ mix64(i.astype(np.uint64) * P + np.asarray(k, dtype=np.uint64)))
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, tag: int, i, k):
    """crng.h normal: sum of uniforms 12k .. 12k+11, in order, minus 6."""
    k = np.asarray(k, dtype=np.uint64)
    s = np.zeros(np.broadcast(i, k).shape)
    for t in range(12):
        s = s + uniform(seed, tag, i, np.uint64(12) * k + np.uint64(t))
    return s - 6.0


def _svm_rows(seed, r0, r1, ns, nf, per_row):
    """Merged (column, value) entries of sample rows [r0, r1) (host.cpp svm_row),
    returned as (counts, cols, vals) without the t entries."""
    r = np.arange(r0, r1, dtype=np.uint64)[:, None]
    k = np.arange(per_row, dtype=np.uint64)[None, :]
    col = (uniform(seed, K_SVM_COL, r, k) * float(nf)).astype(np.uint64).astype(np.int64)
    label = np.where(np.arange(r0, r1) < ns // 2, 1.0, -1.0)[:, None]
    sd = np.sqrt(1.0 / nf)
    val = label * (label / float(nf) + sd * normal(seed, K_SVM_VAL, r, k))
    rows = np.broadcast_to(np.arange(r1 - r0)[:, None], col.shape)
    order = np.lexsort((np.broadcast_to(k, col.shape).ravel(), col.ravel(), rows.ravel()))
    rr, cc, vv = rows.ravel()[order], col.ravel()[order], val.ravel()[order]
    start = np.ones(len(cc), dtype=bool)
    start[1:] = (rr[1:] != rr[:-1]) | (cc[1:] != cc[:-1])
    # duplicates merged left to right, like the C loop (x = x + next)
    idx = np.flatnonzero(start)
    summed = vv[idx].copy()
    j = idx + 1
    alive = (j < len(cc)) & ~np.r_[start, True][np.minimum(j, len(cc))]
    while alive.any():
        summed[alive] = summed[alive] + vv[j[alive]]
        j = j + 1
        nxt = np.r_[start, True][np.minimum(j, len(cc))]
        alive = alive & (j < len(cc)) & ~nxt
    keep = summed != 0.0
    mr, mc, mv = rr[idx][keep], cc[idx][keep], summed[keep]
    return np.bincount(mr, minlength=r1 - r0), mc, mv


def svm(scale: float = 1.0, seed: int = 4, threads: int | None = None):
    """C4 SVM (host.cpp gen_svm) as plain arrays:
    dict(n, m_ineq, m_eq, q=(rp, ci, v), a_ineq=(rp, ci, v), a_eq=(rp, ci, v), c, b_ineq, b_eq)."""
    ns = max(2, int(round(1000000 * scale)))
    nf = max(2, int(round(10000 * scale)))
    per_row = min(50, nf)
    n, m = nf + ns, 2 * ns
    step = 20000
    ranges = [(a, min(a + step, ns)) for a in range(0, ns, step)]
    threads = threads or min(16, os.cpu_count() or 1)
    with ThreadPoolExecutor(threads) as ex:  # numpy releases the GIL in the ufuncs
        parts = list(ex.map(lambda ab: _svm_rows(seed, ab[0], ab[1], ns, nf, per_row), ranges))
    cnt = np.concatenate([p[0] for p in parts]) + 1  # + the t entry
    top_rp = np.zeros(ns + 1, dtype=np.int64)
    np.cumsum(cnt, out=top_rp[1:])
    nnz_top = int(top_rp[-1])
    ci = np.empty(nnz_top + ns, dtype=np.int32)
    v = np.empty(nnz_top + ns)
    t_pos = top_rp[1:] - 1
    body = np.ones(nnz_top, dtype=bool)
    body[t_pos] = False
    ci[:nnz_top][body] = np.concatenate([p[1] for p in parts])
    v[:nnz_top][body] = np.concatenate([p[2] for p in parts])
    ci[t_pos] = nf + np.arange(ns)
    v[t_pos] = -1.0
    ci[nnz_top:] = nf + np.arange(ns)
    v[nnz_top:] = -1.0
    a_rp = np.concatenate([top_rp, nnz_top + np.arange(1, ns + 1)]).astype(np.int32)
    q_rp = np.concatenate([np.arange(nf + 1), np.full(ns, nf)]).astype(np.int32)
    c = np.zeros(n)
    c[nf:] = 0.5
    b = np.zeros(m)
    b[:ns] = -1.0
    return dict(n=n, m_ineq=m, m_eq=0,
                q=(q_rp, np.arange(nf, dtype=np.int32), np.full(nf, 2.0)),
                a_ineq=(a_rp, ci, v),
                a_eq=(np.zeros(1, dtype=np.int32), np.zeros(0, dtype=np.int32), np.zeros(0)),
                c=c, b_ineq=b, b_eq=np.zeros(0))


def as_qp(d):
    """The arrays of svm() as a rapdhg QuadraticProgram (pure Python: the
    package's model types load no native library until a solve is called)."""
    import paper_2311_07710_b200 as rb

    n, mi, me = d["n"], d["m_ineq"], d["m_eq"]
    return rb.QuadraticProgram(q=rb.SparseMatrix.from_csr(n, n, *d["q"]), c=d["c"],
                               a_ineq=rb.SparseMatrix.from_csr(mi, n, *d["a_ineq"]), b_ineq=d["b_ineq"],
                               a_eq=rb.SparseMatrix.from_csr(me, n, *d["a_eq"]), b_eq=d["b_eq"])
