export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
for k in "LARGE 1.0 200" "LASSO 1.0 800"; do timeout 600 python scripts/sweep_sched.py $k 2>&1 | grep -E "^\{" | cut -c1-200; done
