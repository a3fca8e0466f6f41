export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_shard.py -x -q --timeout 200 2>&1 | tail -2
for s in auto off; do echo "== slab $s"; for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_SLAB=$s timeout 150 python scripts/sweep_sched.py $k; done; done 2>&1 | cut -c1-250
echo "== C2 variants"
for w in 2048 4096; do for t in 2048 3584; do echo "w=$w t=$t"; RAPDHG_SLAB_WIDTH=$w RAPDHG_SLAB_TILE=$t timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-200; done; done
