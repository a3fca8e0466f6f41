import os, sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
rb.solve(p, cfg)
os.environ["RAPDHG_TRACE"] = "host"
for i in range(3):
    r = rb.solve(p, cfg)
    print(i, "setup %.3f" % r.setup_seconds, file=sys.stderr, flush=True)
