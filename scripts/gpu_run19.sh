export PYTHONUNBUFFERED=1
python scripts/ncu_target.py 120 > gpurun_out/target_plain19.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel|rowwise_kernel" -s 20 -c 4 -o gpurun_out/prof_slab19 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full19.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full19.log
