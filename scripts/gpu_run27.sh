export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_slab.py -x -q --timeout 150 2>&1 | tail -2
timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-250
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"slab_kernel|rowwise_kernel" -s 200 -c 40 --csv \
    --log-file gpurun_out/launches27.csv python scripts/ncu_target.py 120 > gpurun_out/ncu_l27.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel|SlabFinish" -s 6 -c 4 -o gpurun_out/prof_slab27 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full27.log 2>&1; echo "ncu full rc=$?"
