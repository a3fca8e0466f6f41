export PYTHONUNBUFFERED=1
for k in "LARGE 1.0 200" "LARGE_LOCAL 1.0 200"; do RAPDHG_TRACE=1 timeout 600 python scripts/sweep_sched.py $k 2>&1 | grep -E "^\[slab\]|^\{" | cut -c1-260; done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"DualStepOp|PrimalStepOp" -c 2 -o gpurun_out/prof_c5 \
    python scripts/c5_target.py LARGE > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"
