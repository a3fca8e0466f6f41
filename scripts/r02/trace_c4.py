# C4 solves to 1e-6 from pinned host arrays (bench.py's e2e inputs); run with RAPDHG_TRACE=1
import sys; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
from bench import pinned_qp
p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
for _ in range(3):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print("solve", r.iterations, repr(r.norm_a), r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
