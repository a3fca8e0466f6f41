"""Setup phase breakdown (RAPDHG_TRACE) of one solve, after a warm-up solve."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
kind = rb.Gen[sys.argv[1]] if len(sys.argv) > 1 else rb.Gen.LASSO
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
p = rb.generate(kind, scale, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
r = rb.solve(p, cfg)
os.environ["RAPDHG_TRACE"] = "1"
t = time.perf_counter()
r = rb.solve(p, cfg)
print("wall", time.perf_counter() - t, "setup", r.setup_seconds, "loop", r.loop_seconds, "its", r.iterations, flush=True)
