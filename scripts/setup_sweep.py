"""Median setup time of C4 solves from pinned host arrays (2 warm solves,
then 10 timed). python scripts/setup_sweep.py LABEL"""
import statistics
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb  # noqa: E402
from bench import pinned_qp  # noqa: E402

p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
cfg = rb.SolverConfig(tol=1e-6)
rb.solve(p, cfg)
rb.solve(p, cfg)
rs = [rb.solve(p, cfg) for _ in range(10)]
s = [r.setup_seconds for r in rs]
print(sys.argv[1] if len(sys.argv) > 1 else "", "setup ms median %.1f min %.1f max %.1f" %
      (1e3 * statistics.median(s), 1e3 * min(s), 1e3 * max(s)),
      "solve ms median %.1f" % (1e3 * statistics.median(r.solve_seconds for r in rs)), flush=True)
