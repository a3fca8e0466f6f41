export PYTHONUNBUFFERED=1
RAPDHG_TRACE_MODE=host timeout 300 python - <<'PY' 2>&1 | tail -40
import os, sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
r = rb.solve(p, cfg)
os.environ["RAPDHG_TRACE"] = "host"
for k in range(2):
    t = time.perf_counter()
    r = rb.solve(p, cfg)
    print("wall", time.perf_counter() - t, "setup", r.setup_seconds, "loop", r.loop_seconds, flush=True)
PY
