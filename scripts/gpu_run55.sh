# one sync per check: GPU tests, check cost, short bench
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python scripts/check_cost.py
timeout 600 python bench.py --steps 3 --warmup 3 2>/dev/null | tail -1 | cut -c1-400
