export PYTHONUNBUFFERED=1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel" -s 4 -c 2 -o gpurun_out/prof_slab24 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full24.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full24.log
