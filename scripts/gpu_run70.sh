export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for k in LARGE LARGE_LOCAL RANDOM_QP; do echo "== $k"; timeout 600 python scripts/sweep_sched.py $k 1.0 200 2>&1 | grep -E "^\{" | cut -c1-200; done
timeout 300 python scripts/check_cost.py
