"""Per-iteration exchange volume of the row-sharded solver for
an instance and shard count, from the library's shard plan: for each of the
three per-step exchanges (w gathered by the dual rows through A, x_md by the
primal rows through Q, y by the primal rows through A'), the entries each
shard references but does not own (halo), against an allgather. Host only.

    python scripts/exchange_volume.py svm 1.0 8"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb  # noqa: E402

GEN = {"svm": rb.Gen.SVM, "lasso": rb.Gen.LASSO, "large": rb.Gen.LARGE, "large_local": rb.Gen.LARGE_LOCAL,
       "portfolio": rb.Gen.PORTFOLIO}


def remote_refs(rp, ci, row_bounds, col_bounds, ncols):
    tot = 0
    for k in range(len(row_bounds) - 1):
        r0, r1 = row_bounds[k], row_bounds[k + 1]
        cols = np.unique(ci[rp[r0]:rp[r1]])
        own = (cols >= col_bounds[k]) & (cols < col_bounds[k + 1])
        tot += int((~own).sum())
    return tot


kind, scale, parts = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
p = rb.generate(GEN[kind], scale, {"svm": 4, "lasso": 2, "portfolio": 3}.get(kind, 5))
db, pb = rb.shard_plan(p, parts)
n, m = p.num_vars(), p.num_rows()
import scipy.sparse as sp  # noqa: E402

A = sp.vstack([sp.csr_matrix((p.a_ineq.values, p.a_ineq.col_idx, p.a_ineq.row_ptr), shape=(p.num_ineq(), n)),
               sp.csr_matrix((p.a_eq.values, p.a_eq.col_idx, p.a_eq.row_ptr), shape=(p.num_eq(), n))]).tocsr()
AT = A.T.tocsr()
Q = sp.csr_matrix((p.q.values, p.q.col_idx, p.q.row_ptr), shape=(n, n))
w = remote_refs(A.indptr, A.indices, db, pb, n)
x = remote_refs(Q.indptr, Q.indices, pb, pb, n)
y = remote_refs(AT.indptr, AT.indices, pb, db, m)
ag = (parts - 1) * (2 * n + m)  # allgather: every rank receives the others' slices of w, x_md, y
print(f"{kind} scale {scale} P={parts}: n={n} m={m}")
print(f"  halo entries per iteration (all ranks): w {w}, x_md {x}, y {y} -> {8 * (w + x + y) / 1e6:.1f} MB")
print(f"  allgather entries per iteration (all ranks): {ag} -> {8 * ag / 1e6:.1f} MB")
