# round 2 call 31: power-iteration random start drawn beside the upload: GPU suite incl. scale parity, C4 setup trace
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_31_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_31_tests.log
cat > /tmp/trace_pinned.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
from bench import pinned_qp
p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
for _ in range(4):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print("solve", r.iterations, repr(r.norm_q), repr(r.norm_a), r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
PY
RAPDHG_TRACE=1 timeout 300 python /tmp/trace_pinned.py > gpurun_out/r02_31_trace.log 2>&1; echo "trace rc=$?"; grep -E "norm|setup total|^solve" gpurun_out/r02_31_trace.log | tail -8
