import sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
out = []
for i in range(8):
    t = time.perf_counter()
    r = rb.solve(p, cfg)
    out.append("%.3f/%.3f" % (r.setup_seconds, time.perf_counter() - t))
print(" ".join(out), flush=True)
