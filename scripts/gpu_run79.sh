export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py -x -q 2>&1 | tail -5
for r in 1 2; do timeout 300 python scripts/check_cost.py 2>&1 | head -2; done
echo "== kkt rowwise"; RAPDHG_KKT_SLAB=0 timeout 300 python scripts/check_cost.py 2>&1 | head -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
