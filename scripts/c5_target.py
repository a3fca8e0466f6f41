"""C5 (LARGE) resident solve for ncu: a few iterations."""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
kind = rb.Gen[sys.argv[1]] if len(sys.argv) > 1 else rb.Gen.LARGE
p = rb.generate(kind, 1.0, 5)
s = rb.Session(p, rb.SolverConfig(tol=1e-9, max_iters=40))
r = s.solve()
print("iterations", r.iterations, "loop_s", r.loop_seconds)
