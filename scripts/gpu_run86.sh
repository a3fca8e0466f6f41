export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python - <<'PY'
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
for name, kind, seed in (("C1", rb.Gen.RANDOM_QP, 1), ("C2", rb.Gen.LASSO, 2), ("C3", rb.Gen.PORTFOLIO, 3), ("C4", rb.Gen.SVM, 4), ("C5L", rb.Gen.LARGE_LOCAL, 5)):
    p = rb.generate(kind, 1.0, seed)
    s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=400, profile_kernels=2))
    s.solve(); r = s.solve(); s.close()
    print(name, round(r.iterations / r.loop_seconds), [round(1e3 * r.kernel_ms[i] / r.kernel_count[i], 1) if r.kernel_count[i] else None for i in range(2)], flush=True)
PY
