export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_slab.py -x -q --timeout 150 > gpurun_out/pytest_slab21.log 2>&1; echo "slab pytest rc=$?"; tail -5 gpurun_out/pytest_slab21.log
for s in auto off; do echo "== slab $s"; for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_SLAB=$s timeout 150 python scripts/sweep_sched.py $k; done; done 2>&1 | cut -c1-330
echo "== C2 variants"
for f in 1 0; do for w in 2048 4096; do for t in 4096 8192 12288; do echo "fuse=$f w=$w t=$t"; RAPDHG_SLAB_FUSE=$f RAPDHG_SLAB_WIDTH=$w RAPDHG_SLAB_TILE=$t timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-250; done; done; done
for v in 4 16; do echo "V=$v"; RAPDHG_SLAB_V=$v timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-250; done
