# round 2 call 24: C4 setup trace (synced marks) with the slab-phase norm estimate
cat > /tmp/trace_pinned.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
from bench import pinned_qp
p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
for _ in range(3):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
print('solve', r.iterations, repr(r.norm_a), r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
PY
RAPDHG_TRACE=1 timeout 300 python /tmp/trace_pinned.py 2>&1 | tail -36
