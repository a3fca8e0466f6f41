# setup / solve seconds of C2, C3, C4 solves to 1e-6 (pinned inputs; median of 5 after one warm-up)
# under the RAPDHG_NORM_SLAB_STEP the caller sets; one JSON line per config
import json, statistics, sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
from bench import pinned_qp
for name, kind, seed in (("C2", rb.Gen.LASSO, 2), ("C3", rb.Gen.PORTFOLIO, 3), ("C4", rb.Gen.SVM, 4)):
    p = pinned_qp(rb.generate(kind, 1.0, seed))
    rs = [rb.solve(p, rb.SolverConfig(tol=1e-6)) for _ in range(6)][1:]
    print(json.dumps({"K": int(sys.argv[1]), "config": name, "iterations": rs[0].iterations, "norm_a": rs[0].norm_a,
                      "setup_s": statistics.median(r.setup_seconds for r in rs),
                      "solve_s": statistics.median(r.solve_seconds for r in rs)}), flush=True)
