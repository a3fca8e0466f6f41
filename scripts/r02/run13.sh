# round 2 call 13: C4 setup variance — pool reservation / no pool
export PYTHONUNBUFFERED=1
for env in "X=1"; do
echo "== $env"
env $env RAPDHG_TRACE=1 timeout 300 python - <<'PY' > gpurun_out/r02_13_trace.log 2>&1
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.SVM, 1.0, 4)
for _ in range(10):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print("solve", r.iterations, round(r.solve_seconds, 4), round(r.setup_seconds, 4), round(r.loop_seconds, 4), flush=True)
PY
grep -E "^solve|upload \+ fill|norm A" gpurun_out/r02_13_trace.log | awk '{printf "%s ", $0} /^solve/{print ""}'
done
