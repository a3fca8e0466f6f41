# round 2 call 6: host layout planner (slab_layout.cpp + device fills); C5 lanes-per-row experiment
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q -k "slab or shard or parity and not scale" > gpurun_out/r02_06_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_06_tests.log
RAPDHG_TRACE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.SVM, 1.0, 4)
for _ in range(3):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print('solve', r.iterations, r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
" > gpurun_out/r02_06_setup_trace.log 2>&1; echo "trace rc=$?"; grep -E "solve |layout|counts|upload \+ fill|slab plan|joined|norm A|engine setup" gpurun_out/r02_06_setup_trace.log | tail -16
for epl in 16 8 4 2; do
RAPDHG_EPL=$epl timeout 300 python - <<'PY'
import json, os, sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
for name, kind in (("C5-U", rb.Gen.LARGE), ("C5-L", rb.Gen.LARGE_LOCAL)):
    p = rb.generate(kind, 1.0, 5)
    s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=200))
    s.solve(); r = s.solve(); bi, _, _ = s.bytes(); s.close()
    print(json.dumps({"epl": os.environ["RAPDHG_EPL"], "config": name, "it_per_s": r.iterations / r.loop_seconds,
                      "iter_GBs": bi * r.iterations / r.loop_seconds / 1e9}), flush=True)
PY
done
