"""Generate tests/golden/scale_c2_1e6.npz: the REFERENCE's full solve of the
bench-size C2 Lasso (n = m = 210,000, nnz(A) = 1.04e7, seed 2)
to relKKT 1e-6 — about 3-4 minutes of CPU, too long for the GPU test step,
so its summary is stored here and tests/test_gpu_scale_parity.py compares the
GPU's own full solve against it.

Stored: status, iterations, restarts, residuals, norms, objective, the check
log, and the solution at 4096 fixed indices of x and of y (plus the full-vector
norms), so the fixture stays small.

    python tests/golden/make_scale_golden.py
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.dirname(HERE)]

import oracle  # noqa: E402
import paper_2311_07710_b200 as rb  # noqa: E402

SAMPLE = 4096


def sample_idx(length, salt):
    return np.sort(np.random.default_rng(salt).choice(length, size=min(SAMPLE, length), replace=False))


def main():
    oracle.build()
    ref = oracle.ref()
    p = rb.generate(rb.Gen.LASSO, 1.0, 2)
    t = time.perf_counter()
    r = ref.solve(p, rb.SolverConfig(tol=1e-6))
    wall = time.perf_counter() - t
    y = np.concatenate([r.point.y_ineq, r.point.y_eq])
    ix, iy = sample_idx(len(r.point.x), 1), sample_idx(len(y), 2)
    out = dict(status=np.array(int(r.status)), iterations=np.array(r.iterations), restarts=np.array(r.restarts),
               residuals=np.array([r.residuals.r_primal, r.residuals.r_dual, r.residuals.r_gap]),
               norms=np.array([r.norm_q, r.norm_a]), objective=np.array(p.objective(r.point.x)),
               log=np.array([[L.iteration, L.r_primal, L.r_dual, L.r_gap, L.eta, L.omega, L.restarted]
                             for L in r.log]),
               x_idx=ix, x_val=r.point.x[ix], y_idx=iy, y_val=y[iy],
               x_norm=np.array([np.linalg.norm(r.point.x), np.max(np.abs(r.point.x))]),
               y_norm=np.array([np.linalg.norm(y), np.max(np.abs(y))]),
               shape=np.array([p.num_vars(), p.num_ineq(), p.num_eq(), p.a_ineq.nnz() + p.a_eq.nnz()]),
               wall_s=np.array(wall))
    np.savez_compressed(os.path.join(HERE, "scale_c2_1e6.npz"), **out)
    print(rb.to_string(r.status), r.iterations, r.restarts, r.residuals.relkkt(), f"{wall:.1f} s")


if __name__ == "__main__":
    main()
