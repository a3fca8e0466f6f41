# round 2 call 17: power iteration with device-side stop (no overshoot): op-norm tests, C4 setup trace
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -k "norm or parity or shard or box" > gpurun_out/r02_17_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_17_tests.log
RAPDHG_TRACE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
for kind, seed in ((rb.Gen.SVM, 4), (rb.Gen.LASSO, 2)):
    p = rb.generate(kind, 1.0, seed)
    for _ in range(2):
        r = rb.solve(p, rb.SolverConfig(tol=1e-6))
        print('solve', kind, r.iterations, r.norm_q, r.norm_a, r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
" > gpurun_out/r02_17_setup_trace.log 2>&1; echo "trace rc=$?"; grep -E "norm|power|setup total|^solve" gpurun_out/r02_17_setup_trace.log
