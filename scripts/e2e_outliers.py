"""Repeated C4 solves from pinned host arrays, as the bench's e2e leg runs
them (the previous result alive during the next solve), with per-phase
host timestamps (RAPDHG_TRACE=host) to find what an occasional slow solve
spends its time on."""
import sys
import time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb  # noqa: E402
from bench import pinned_qp  # noqa: E402

p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
cfg = rb.SolverConfig(tol=1e-6)
for _ in range(3):
    rb.solve(p, cfg)
res = None
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    t = time.perf_counter()
    res = rb.solve(p, cfg)
    print(f"solve {k}: wall {time.perf_counter() - t:.4f} setup {res.setup_seconds:.4f} loop {res.loop_seconds:.4f}",
          file=sys.stderr, flush=True)
