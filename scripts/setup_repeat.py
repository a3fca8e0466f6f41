"""setup_seconds / loop_seconds of consecutive solves (no tracing)."""
import sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
for i in range(4):
    t = time.perf_counter()
    r = rb.solve(p, cfg)
    print(i, "wall %.3f setup %.3f loop %.3f" % (time.perf_counter() - t, r.setup_seconds, r.loop_seconds), flush=True)
s = rb.Session(p, rb.SolverConfig(tol=1e-6, max_iters=20000, profile_kernels=True))
s.solve(); s.close()
for i in range(2):
    t = time.perf_counter()
    r = rb.solve(p, cfg)
    print("after session", i, "wall %.3f setup %.3f loop %.3f" % (time.perf_counter() - t, r.setup_seconds, r.loop_seconds), flush=True)
