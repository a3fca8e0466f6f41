"""Loop time per iteration with checks every 40 vs every 1000 (C2, fixed iterations)."""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
for ci in (40, 1000, 40, 1000):
    s = rb.Session(p, rb.SolverConfig(tol=1e-14, max_iters=3000, check_interval=ci))
    s.solve()
    r = s.solve()
    print(f"check_interval {ci}: {1e6 * r.loop_seconds / r.iterations:.2f} us/iteration ({r.iterations} its)", flush=True)
    s.close()
