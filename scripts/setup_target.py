"""ncu target: one solve with a single iteration (the launches are the
setup's). python scripts/setup_target.py [lasso|svm|portfolio] (default lasso)."""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
kind, seed = {"lasso": (rb.Gen.LASSO, 2), "svm": (rb.Gen.SVM, 4), "portfolio": (rb.Gen.PORTFOLIO, 3)}[
    sys.argv[1] if len(sys.argv) > 1 else "lasso"]
p = rb.generate(kind, 1.0, seed)
rb.solve(p, rb.SolverConfig(tol=1e-6, max_iters=1))
