# persistent chunk kernel: slab tests first (bounded), then timing
export PYTHONUNBUFFERED=1
RAPDHG_TRACE=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 0.05, 2)
r = rb.solve(p, rb.SolverConfig(tol=1e-6, max_iters=2000))
print('small', r.status, r.iterations)
" 2>&1 | grep -v "^\[trace\]" | tail -5
timeout 600 python -m pytest tests/test_gpu_slab.py -x -q 2>&1 | tail -5
timeout 300 python scripts/check_cost.py
timeout 300 env RAPDHG_SLAB_CHUNK=0 python scripts/check_cost.py
