# round 2, first call: GPU suite at HEAD, C4 (svm) bench with the round-1 bench.py, per-config throughput
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_01_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_01_tests.log
timeout 600 python bench.py --workload svm --seed 4 --steps 5 --warmup 3 --no-cpu-baseline --max-iters 2000 > gpurun_out/r02_01_bench_svm.json 2> gpurun_out/r02_01_bench_svm.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_01_bench_svm.json
timeout 900 bash scripts/gpu_configs.sh
