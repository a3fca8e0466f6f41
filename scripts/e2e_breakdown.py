"""Where does the end-to-end solve time go? (Python wall vs C-ABI timers)."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb

p = rb.generate(rb.Gen.LASSO, 1.0, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
rb.solve(p, rb.SolverConfig(tol=1e-6, max_iters=40))  # context warm-up
for i in range(2):
    t = time.perf_counter()
    r = rb.solve(p, cfg)
    w = time.perf_counter() - t
    print(f"wall {w:.3f}s  solve_seconds {r.solve_seconds:.3f}  setup {r.setup_seconds:.3f}  loop {r.loop_seconds:.3f}  it {r.iterations}", flush=True)
