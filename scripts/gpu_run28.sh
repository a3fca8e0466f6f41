export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_slab.py -x -q --timeout 150 2>&1 | tail -3
RAPDHG_LIB=paper_2311_07710_b200/librapdhg_b200_prof.so timeout 200 python scripts/sweep_sched.py LASSO 1.0 200 2>&1 | grep -v "^  \.\.\." | cut -c1-200 | head -12
for s in auto off; do echo "== slab $s"; for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300"; do RAPDHG_SLAB=$s timeout 150 python scripts/sweep_sched.py $k; done; done 2>&1 | cut -c1-250
echo "== C2 variants"
for w in 2048 4096; do for t in 2048 3584 5120; do echo "w=$w t=$t"; RAPDHG_SLAB_WIDTH=$w RAPDHG_SLAB_TILE=$t timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-200; done; done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel|SlabFinish" -s 6 -c 4 -o gpurun_out/prof_slab28 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full28.log 2>&1; echo "ncu full rc=$?"
