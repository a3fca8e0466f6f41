export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_slab.py -x -q --timeout 150 > gpurun_out/pytest_slab16.log 2>&1; echo "slab pytest rc=$?"; tail -25 gpurun_out/pytest_slab16.log
for s in auto off; do echo "== slab $s"; for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_SLAB=$s timeout 150 python scripts/sweep_sched.py $k; done; done 2>&1 | cut -c1-330
