export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest34.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest34.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench34.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench34.log | cut -c1-1500
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench34_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file gpurun_out/launches34.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch34.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel|SlabFinish|rowwise_kernel<PrimalStepOp|KktQAtyOp|KktAxOp" -s 8 -c 6 -o gpurun_out/prof_r01_slab \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full34.log 2>&1
echo "ncu full rc=$?"
