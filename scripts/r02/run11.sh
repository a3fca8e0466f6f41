# round 2 call 11: setup timings (C2, C4, C5-U) after the planner/SELL changes
export PYTHONUNBUFFERED=1
for w in svm lasso large; do
RAPDHG_TRACE=1 timeout 300 python - $w <<'PY' > gpurun_out/r02_11_trace_$w.log 2>&1
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
kind = {"svm": (rb.Gen.SVM, 4), "lasso": (rb.Gen.LASSO, 2), "large": (rb.Gen.LARGE, 5)}[sys.argv[1]]
p = rb.generate(kind[0], 1.0, kind[1])
for _ in range(3):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6, max_iters=400))
    print("solve", r.iterations, round(r.solve_seconds, 4), round(r.setup_seconds, 4), round(r.loop_seconds, 4), flush=True)
PY
echo "== $w"; grep -E "^solve|engine setup|norm A|norm Q|slab plans|upload, stack|scaling  |sell|colblock" gpurun_out/r02_11_trace_$w.log | tail -12
done
