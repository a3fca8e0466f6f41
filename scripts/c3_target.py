"""ncu target: C3 portfolio, a short resident solve (steps + checks)."""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.PORTFOLIO, 1.0, 3)
s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=120))
s.solve()
s.solve()
