"""Setup time of 12 consecutive C2 solves in one process (outlier hunt)."""
import sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
out = []
for k in range(12):
    t = time.perf_counter()
    r = rb.solve(p, cfg)
    out.append((round(1e3 * r.setup_seconds, 1), round(1e3 * (time.perf_counter() - t), 1)))
print(out, flush=True)
