export PYTHONUNBUFFERED=1
for w in 2048 16384; do echo "== width $w"; RAPDHG_SLAB_WIDTH=$w RAPDHG_TRACE=1 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.SVM, 1.0, 2)
s = rb.Session(p, rb.SolverConfig(tol=1e-9, max_iters=10)); s.solve()
" 2>&1 | grep -E "^\[slab\]" ; done
