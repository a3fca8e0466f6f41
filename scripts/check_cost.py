"""Loop time per iteration with checks every 40 vs every 1000 at fixed
iteration counts. python scripts/check_cost.py [lasso|svm] (default lasso)."""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
kind, seed, its = {"lasso": (rb.Gen.LASSO, 2, 3000), "svm": (rb.Gen.SVM, 4, 400)}[sys.argv[1] if len(sys.argv) > 1 else "lasso"]
p = rb.generate(kind, 1.0, seed)
for ci in (40, 1000, 40, 1000):
    s = rb.Session(p, rb.SolverConfig(tol=1e-14, max_iters=its, check_interval=ci))
    s.solve()
    r = s.solve()
    print(f"check_interval {ci}: {1e6 * r.loop_seconds / r.iterations:.2f} us/iteration ({r.iterations} its)", flush=True)
    s.close()
