export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q 2>&1 | tail -5
RAPDHG_TRACE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
for kind, sc in ((rb.Gen.LARGE_LOCAL, 0.05), (rb.Gen.LARGE, 0.05), (rb.Gen.LASSO, 0.2)):
    p = rb.generate(kind, sc, 5)
    r = rb.solve_sharded(p, rb.SolverConfig(tol=1e-6, max_iters=200), 8)
    print(kind.name, p.num_vars(), r.iterations)
" 2>&1 | grep -E "halo|^LARGE|^LASSO"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
