# round 2 call 2: GPU suite (incl. the at-scale parity module), smoke, the C4 bench (both arms),
# ncu launch list of the bench and a --set full capture of the C4 step kernels
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q -rA -k "not scale_parity" > gpurun_out/r02_02_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_02_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q -s > gpurun_out/r02_02_scale.log 2>&1; echo "scale rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/r02_02_scale.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_02_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02_02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_02_bench.json 2> gpurun_out/r02_02_bench.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/r02_02_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r02_02_bench_ref.json 2> gpurun_out/r02_02_bench_ref.err; echo "ref rc=$?"; tail -c 1500 gpurun_out/r02_02_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_02_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02_02_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"DualStepOp|PrimalStepOp" -s 4 -c 8 -o gpurun_out/r02_02_c4_full python scripts/ncu_target.py svm 80 > gpurun_out/r02_02_ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/r02_02_ncu_full.log
