export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_slab.py -x -q --timeout 150 > gpurun_out/pytest_slab26.log 2>&1; echo "slab pytest rc=$?"; tail -5 gpurun_out/pytest_slab26.log
RAPDHG_LIB=paper_2311_07710_b200/librapdhg_b200_prof.so timeout 200 python scripts/sweep_sched.py LASSO 1.0 200 2>&1 | cut -c1-250
for s in auto off; do echo "== slab $s"; for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_SLAB=$s timeout 150 python scripts/sweep_sched.py $k; done; done 2>&1 | cut -c1-330
echo "== C2 variants"
for w in 2048 4096; do for t in 2048 3584 5120; do echo "w=$w t=$t"; RAPDHG_SLAB_WIDTH=$w RAPDHG_SLAB_TILE=$t timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-250; done; done
for v in 2 8; do echo "V=$v"; RAPDHG_SLAB_V=$v timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-250; done
