# round 2 call 19: norm Q beside norm A (two streams): op-norm, parity, shard tests; setup trace
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -k "norm or parity or shard or box or host_transport" > gpurun_out/r02_19_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_19_tests.log
RAPDHG_TRACE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
for kind, seed in ((rb.Gen.SVM, 4), (rb.Gen.LASSO, 2)):
    p = rb.generate(kind, 1.0, seed)
    for _ in range(2):
        r = rb.solve(p, rb.SolverConfig(tol=1e-6))
        print('solve', kind, r.iterations, r.norm_q, r.norm_a, r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
" > gpurun_out/r02_19_setup_trace.log 2>&1; echo "trace rc=$?"; grep -E "norm|power|setup total|^solve" gpurun_out/r02_19_setup_trace.log
