# round 2 call 37: plain-path step kernels as programmatic dependent launches — tests, C1 / C5-L / random rates
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not scale_parity" > gpurun_out/r02_37_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_37_tests.log
for pdl in 0 1; do RAPDHG_PDL=$pdl timeout 600 python -c "
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2311_07710_b200 as rb
from instances import random_qp
for name, p, its in (('C1', rb.generate(rb.Gen.RANDOM_QP, 1.0, 1), 2000), ('random 9000', random_qp(21, n=9000, mi=5000, me=800, dens=0.0015, q_rank=3000), 2000),
                     ('C5-L', rb.generate(rb.Gen.LARGE_LOCAL, 1.0, 5), 200)):
    s = rb.Session(p, rb.SolverConfig(tol=1e-14, max_iters=its)); s.solve(); r = s.solve(); s.close()
    print('pdl', '$pdl', name, 'loop it/s %.0f' % (r.iterations / r.loop_seconds), flush=True)
"; done
