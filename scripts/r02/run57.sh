# round 2 call 57: e2e outliers — 10 C4 solves from pinned arrays with host-only trace marks, then the bench's e2e leg shape
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
cat > /tmp/t10.py <<'PY'
import sys, time; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
from bench import pinned_qp
p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
for i in range(10):
    t = time.perf_counter(); r = rb.solve(p, rb.SolverConfig(tol=1e-6)); w = time.perf_counter() - t
    print("solve", i, round(w, 4), round(r.setup_seconds, 4), round(r.loop_seconds, 4), flush=True)
PY
RAPDHG_TRACE=host timeout 300 python /tmp/t10.py > gpurun_out/r02_57_trace.log 2>&1
grep "^solve" gpurun_out/r02_57_trace.log
