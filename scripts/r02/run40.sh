# round 2 call 40: norm Q beside norm A (own thread and stream), no graphs in the power batches — full GPU suite, C4 setup sweep
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_40_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_40_tests.log
cat > /tmp/sweep.py <<'PY'
import sys, statistics; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
from bench import pinned_qp
p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
rb.solve(p, rb.SolverConfig(tol=1e-6)); rb.solve(p, rb.SolverConfig(tol=1e-6))
s = [rb.solve(p, rb.SolverConfig(tol=1e-6)).setup_seconds for _ in range(8)]
print(sys.argv[1], "setup ms median %.1f min %.1f max %.1f" % (1e3 * statistics.median(s), 1e3 * min(s), 1e3 * max(s)), flush=True)
PY
timeout 300 python /tmp/sweep.py head; timeout 300 python /tmp/sweep.py head
