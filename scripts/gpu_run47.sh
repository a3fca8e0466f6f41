export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 > gpurun_out/bench47.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench47.log | cut -c1-3000
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench47_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file gpurun_out/launches47.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch47.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel|slab_finish" -s 4 -c 4 -o gpurun_out/prof_r01_slab2 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full47.log 2>&1
echo "ncu full rc=$?"
