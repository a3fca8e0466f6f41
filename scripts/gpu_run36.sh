export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300" "RANDOM_QP 1.0 2000" "LARGE 0.5 120"; do timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-220; done
for k in "LASSO 1.0 800" "LARGE 0.5 120"; do RAPDHG_SLAB=off timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-220; done
