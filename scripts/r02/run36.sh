# round 2 call 36: persistent cooperative chunks for small problems — tests, C1 rates
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not scale_parity" > gpurun_out/r02_36_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_36_tests.log
for m in 0 1; do RAPDHG_PERSISTENT=$m timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.RANDOM_QP, 1.0, 1)
s = rb.Session(p, rb.SolverConfig(tol=1e-6)); s.solve(); r = s.solve()
q = rb.solve(p, rb.SolverConfig(tol=1e-6))
print('persistent', '$m', 'loop it/s %.0f' % (r.iterations / r.loop_seconds), 'solve s %.4f' % q.solve_seconds, 'launches', r.kernel_launches)
"; done
