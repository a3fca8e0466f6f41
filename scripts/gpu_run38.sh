export PYTHONUNBUFFERED=1
for k in "LARGE 1.0 200" "LARGE_LOCAL 1.0 200"; do timeout 600 python scripts/sweep_sched.py $k 2>&1 | grep -E "^\{" | cut -c1-260; done
for k in "LARGE 1.0 200"; do RAPDHG_L2PIN=0 timeout 600 python scripts/sweep_sched.py $k 2>&1 | grep -E "^\{" | cut -c1-260; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 2>&1 | tail -1
ncu --set full --clock-control none --kernel-name-base demangled \
    -k regex:"DualStepOp|PrimalStepOp" -c 2 -o gpurun_out/prof_c5_pin \
    python scripts/c5_target.py LARGE > gpurun_out/ncu_c5pin.log 2>&1; echo "ncu rc=$?"
