export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_slab.py -x -q 2>&1 | tail -3
for r in 1 2; do echo "== early"; timeout 300 python scripts/check_cost.py 2>&1 | head -2; echo "== grid wait"; RAPDHG_SLAB_EARLY=0 timeout 300 python scripts/check_cost.py 2>&1 | head -2; done
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
