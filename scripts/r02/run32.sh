# round 2 call 32: norm-A switch step sweep (setup time of C4 from pinned inputs, 6 solves each)
export PYTHONUNBUFFERED=1
cat > /tmp/sweep.py <<'PY'
import sys, statistics; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
from bench import pinned_qp
p = pinned_qp(rb.generate(rb.Gen.SVM, 1.0, 4))
rb.solve(p, rb.SolverConfig(tol=1e-6)); rb.solve(p, rb.SolverConfig(tol=1e-6))
s = [rb.solve(p, rb.SolverConfig(tol=1e-6)).setup_seconds for _ in range(6)]
print(sys.argv[1], "setup ms median %.1f min %.1f max %.1f" % (1e3 * statistics.median(s), 1e3 * min(s), 1e3 * max(s)), flush=True)
PY
for k in 72 96 120 -1; do RAPDHG_NORM_SLAB_STEP=$k timeout 300 python /tmp/sweep.py $k; done
