export PYTHONUNBUFFERED=1
RAPDHG_L2BLOCK_KB=49152 ncu --set full --clock-control none --kernel-name-base demangled \
    -k regex:"DualStepOp|PrimalStepOp|SpmvOp" -s 2 -c 6 -o gpurun_out/prof_c5_blk \
    python scripts/c5_target.py LARGE > gpurun_out/ncu_c5blk.log 2>&1; echo "ncu rc=$?"
