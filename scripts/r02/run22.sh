# round 2 call 22: norm estimate on the slab phases after step 72: tests, C4/C2 setup traces, bench
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_shard.py tests/test_gpu_parity.py tests/test_host_transport.py -x -q > gpurun_out/r02_22_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_22_tests.log
cat > /tmp/trace_pinned.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
from bench import pinned_qp
for kind, seed in ((rb.Gen.SVM, 4), (rb.Gen.LASSO, 2), (rb.Gen.PORTFOLIO, 3)):
    p = pinned_qp(rb.generate(kind, 1.0, seed))
    for _ in range(2):
        r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print('solve', kind, r.iterations, repr(r.norm_a), r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
PY
for k in 72 -1; do echo "== RAPDHG_NORM_SLAB_STEP=$k"; RAPDHG_NORM_SLAB_STEP=$k RAPDHG_TRACE=host timeout 300 python /tmp/trace_pinned.py 2>&1 | grep -E "norm A|setup total|^solve|slab plan:"; done
timeout 600 python bench.py > gpurun_out/r02_22_bench.json 2> gpurun_out/r02_22_bench.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.loads(open('gpurun_out/r02_22_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['e2e']['wall_s_each'], d['time_to_tol_s'])
PY
