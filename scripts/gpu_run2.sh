set -x
python bench.py --steps 2 --warmup 1 > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python scripts/ncu_target.py 120 > gpurun_out/target_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"PrimalStepOp|DualStepOp|KktQAtyOp|KktAxOp" -s 12 -c 6 -o gpurun_out/prof_r01 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
