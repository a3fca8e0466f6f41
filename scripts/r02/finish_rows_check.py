# bit-identity of RAPDHG_FINISH_ROWS=2 against 1 on small C3 / C4 / C2 solves (env read per launch)
import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2311_07710_b200 as rb
from test_oracle import assert_results_identical
for kind, scale, seed in ((rb.Gen.PORTFOLIO, 0.2, 3), (rb.Gen.SVM, 0.1, 4), (rb.Gen.LASSO, 0.3, 2)):
    p = rb.generate(kind, scale, seed)
    cfg = rb.SolverConfig(tol=1e-12, max_iters=400, snapshot_interval=80, record_restart_points=True)
    os.environ["RAPDHG_FINISH_ROWS"] = "1"
    a = rb.solve(p, cfg)
    os.environ["RAPDHG_FINISH_ROWS"] = "2"
    b = rb.solve(p, cfg)
    assert_results_identical(a, b)
    print("identical", kind, flush=True)
