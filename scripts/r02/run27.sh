# round 2 call 27: C4 setup trace (synced marks) from pinned inputs, for profiles/r02_c4_setup_trace.log
export PYTHONUNBUFFERED=1
cat > /tmp/trace_pinned.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
from bench import pinned_qp
p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
for _ in range(3):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print("solve", r.iterations, repr(r.norm_a), r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
PY
RAPDHG_TRACE=1 timeout 300 python /tmp/trace_pinned.py > gpurun_out/r02_27_setup_trace.log 2>&1; echo "trace rc=$?"; tail -5 gpurun_out/r02_27_setup_trace.log
