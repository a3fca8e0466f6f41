timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu3.log
for e in 2 4 8 16 32; do RAPDHG_EPL=$e python scripts/sweep_sched.py LASSO 1.0 800; done > gpurun_out/sweep3.log 2>&1
cat gpurun_out/sweep3.log
RAPDHG_TRACE=1 python scripts/explore_c2.py LASSO 1.0 1e-6 20000 > gpurun_out/trace3.log 2>&1; cat gpurun_out/trace3.log | head -30
