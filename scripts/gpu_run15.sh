timeout 900 python -m pytest tests/test_gpu_slab.py -x -q > gpurun_out/pytest_slab15.log 2>&1; echo "slab pytest rc=$?"; tail -25 gpurun_out/pytest_slab15.log
for s in auto off; do echo "== slab $s"; RAPDHG_SLAB=$s python scripts/sweep_sched.py LASSO 1.0 800; RAPDHG_SLAB=$s python scripts/sweep_sched.py SVM 1.0 300; RAPDHG_SLAB=$s python scripts/sweep_sched.py PORTFOLIO 1.0 300; done 2>&1 | cut -c1-330
python scripts/e2e_breakdown.py 2>&1 | tail -2
