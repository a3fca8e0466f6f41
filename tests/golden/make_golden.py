"""Generate tests/golden/golden.npz from the REFERENCE itself.

Runs the reference solver (compiled unmodified from /root/reference by
oracle/Makefile into oracle/_ref/) on small seeded instances and stores the
instances, configs and outputs (solution, iteration count, full check log).
The GPU box has no /root/reference: these fixtures let the strict GPU mode be
checked against reference outputs there too.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.dirname(HERE)]

import oracle  # noqa: E402
import paper_2311_07710_b200 as rb  # noqa: E402
from instances import one_d, random_qp  # noqa: E402

CASES = {
    "oned": (one_d, dict(tol=1e-9, max_iters=200000, check_interval=40)),
    "c1s": (lambda: rb.generate(rb.Gen.RANDOM_QP, 0.3, 3), dict(tol=1e-6, max_iters=20000, check_interval=40)),
    "rqp11": (lambda: random_qp(11, n=80, mi=30, me=12), dict(tol=1e-6, max_iters=20000, check_interval=40)),
    "rqp12lp": (lambda: random_qp(12, n=50, mi=40, me=5, zero_q=True), dict(tol=1e-5, max_iters=20000, check_interval=25)),
}


def main():
    oracle.build()
    ref = oracle.ref()
    out = {}
    for case, (mk, cfgd) in CASES.items():
        p = mk()
        r = ref.solve(p, rb.SolverConfig(**cfgd))
        for name, m in (("q", p.q), ("ai", p.a_ineq), ("ae", p.a_eq)):
            out[f"{case}__{name}_shape"] = np.array([m.n_rows, m.n_cols])
            out[f"{case}__{name}_rp"], out[f"{case}__{name}_ci"], out[f"{case}__{name}_v"] = m.row_ptr, m.col_idx, m.values
        out[f"{case}__c"], out[f"{case}__bi"], out[f"{case}__be"] = p.c, p.b_ineq, p.b_eq
        out[f"{case}__cfg"] = np.array([cfgd["tol"], cfgd["max_iters"], cfgd["check_interval"]], dtype=float)
        out[f"{case}__iterations"] = np.array(r.iterations)
        out[f"{case}__x"] = r.point.x
        out[f"{case}__y"] = np.concatenate([r.point.y_ineq, r.point.y_eq])
        out[f"{case}__log"] = np.array([[L.iteration, L.r_primal, L.r_dual, L.r_gap, L.eta, L.omega, L.restarted]
                                        for L in r.log])
        print(case, rb.to_string(r.status), r.iterations, r.restarts, p.num_vars(), p.num_rows())
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)


if __name__ == "__main__":
    main()
