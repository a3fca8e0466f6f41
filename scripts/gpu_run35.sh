export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_shard.py -x -q --timeout 200 2>&1 | tail -1
RAPDHG_LIB=paper_2311_07710_b200/librapdhg_b200_prof.so timeout 200 python scripts/sweep_sched.py LASSO 1.0 200 2>&1 | grep -v "^  \.\.\." | cut -c1-200 | head -12
for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-220; done
for t in 1536 2048 3072; do echo "t=$t"; RAPDHG_SLAB_TILE=$t timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-200; done
