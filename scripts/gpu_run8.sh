python scripts/ncu_target.py 120 > gpurun_out/target_plain8.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"PrimalStepOp|DualStepOp" -s 12 -c 2 -o gpurun_out/prof_r01b \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full8.log 2>&1
echo "ncu rc=$?"
