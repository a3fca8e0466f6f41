export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py -x -q --timeout 200 2>&1 | tail -1
for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-220; done
for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_SLAB=off timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-220; done
