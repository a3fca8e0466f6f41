"""Box projection (B200 extension) on the benchmark instances whose bounds the
reference form carries as singleton rows: C3 portfolio (x >= 0) and C4 SVM
(hinge slacks t >= 0). Each is solved to relKKT 1e-6 twice on one GPU — the
reference form (bounds as rows) and bounds_from_rows(...) with box_projection
— and the line reports rows, iterations, loop it/s and the objectives.

    python scripts/box_configs.py > profiles/r02_box_configs.jsonl
"""
import json
import sys

sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb  # noqa: E402

CASES = [("c3", rb.Gen.PORTFOLIO, 3), ("c4", rb.Gen.SVM, 4)]

for name, kind, seed in CASES:
    p = rb.generate(kind, 1.0, seed)
    b = rb.bounds_from_rows(p)
    out = {"config": name, "n": p.num_vars()}
    for form, q, box in (("rows", p, False), ("box", b, True)):
        cfg = rb.SolverConfig(tol=1e-6, max_iters=100000, box_projection=box)
        rb.solve(q, cfg)  # warm (module load, pool)
        r = rb.solve(q, cfg)
        out[form] = {"m": q.num_rows(), "nnz_a": q.a_ineq.nnz() + q.a_eq.nnz(), "status": r.status.name,
                     "iterations": r.iterations, "restarts": r.restarts,
                     "loop_it_s": round(r.iterations / r.loop_seconds, 1), "loop_s": round(r.loop_seconds, 4),
                     "setup_s": round(r.setup_seconds, 4), "relkkt": r.residuals.relkkt(),
                     "objective": q.objective(r.point.x)}
    print(json.dumps(out), flush=True)
