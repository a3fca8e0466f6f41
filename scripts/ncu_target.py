"""Short C2 run for ncu: a few hundred iterations of the resident solve."""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 120
strict = len(sys.argv) > 2 and sys.argv[2] == "strict"
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
s = rb.Session(p, rb.SolverConfig(tol=1e-6, max_iters=iters, strict_parity=strict))
r = s.solve()
print("iterations", r.iterations, "loop_s", r.loop_seconds)
