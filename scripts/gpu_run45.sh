export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_shard.py -x -q --timeout 300 2>&1 | tail -1
for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_TRACE=1 timeout 200 python scripts/sweep_sched.py $k 2>&1 | grep -E "^\[slab\]|^\{" | cut -c1-200; done
for j in 0 1; do for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_SLAB_JAGGED=$j timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-160; done; done
