export PYTHONUNBUFFERED=1
for st in 1 0; do
echo "== RAPDHG_STAGE=$st"
RAPDHG_STAGE=$st timeout 300 python - <<'PY' 2>&1 | grep -E "upload|setup total|wall"
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
done
timeout 300 python scripts/e2e_parts.py 2>&1 | tail -3
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
