# round 2 call 12: C4 setup variance after the planner-thread change; slab window width sweep
export PYTHONUNBUFFERED=1
RAPDHG_TRACE=1 timeout 300 python - <<'PY' > gpurun_out/r02_12_trace_svm.log 2>&1
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.SVM, 1.0, 4)
for _ in range(6):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print("solve", r.iterations, round(r.solve_seconds, 4), round(r.setup_seconds, 4), round(r.loop_seconds, 4), flush=True)
PY
grep -E "^solve|norm A" gpurun_out/r02_12_trace_svm.log
for env in "RAPDHG_SLAB_WIDTH=2048" "RAPDHG_SLAB_WIDTH=4096" "RAPDHG_SLAB_WIDTH=1024"; do
env $env timeout 300 python - <<'PY'
import json, os, sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
tag = [k + "=" + v for k, v in os.environ.items() if k.startswith("RAPDHG_SLAB")]
for name, kind, seed in (("C2", rb.Gen.LASSO, 2), ("C3", rb.Gen.PORTFOLIO, 3), ("C4", rb.Gen.SVM, 4)):
    p = rb.generate(kind, 1.0, seed)
    s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=400, profile_kernels=2))
    s.solve(); r = s.solve(); s.close()
    ks = [round(1e3 * r.kernel_ms[i] / r.kernel_count[i], 1) if r.kernel_count[i] else None for i in range(2)]
    print(json.dumps({"env": tag, "config": name, "it_per_s": round(r.iterations / r.loop_seconds, 1), "inloop_us": ks}), flush=True)
PY
done
