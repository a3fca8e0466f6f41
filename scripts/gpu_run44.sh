export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_shard.py tests/test_gpu_colblock.py -x -q --timeout 300 2>&1 | tail -1
python scripts/setup_trace.py LASSO 1.0 2>&1 | grep -E "slab|chunks|arrays|setup total|wall"
for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-200; done
for t in 2048 3072 3584; do echo "t=$t"; RAPDHG_SLAB_TILE=$t timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-200; done
