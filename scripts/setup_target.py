"""ncu target: one C2 solve with a single iteration (the launches are the setup's)."""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
rb.solve(p, rb.SolverConfig(tol=1e-6, max_iters=1))
