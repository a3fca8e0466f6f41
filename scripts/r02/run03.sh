# round 2 call 3: device SVM generator fix; GPU suite, at-scale parity, bench (both arms), C4 setup trace,
# ncu launch list + --set full of the C4 step kernels
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 -k "not scale_parity" > gpurun_out/r02_03_tests.log 2>&1; echo "tests rc=$?"; tail -22 gpurun_out/r02_03_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q -s --durations=0 > gpurun_out/r02_03_scale.log 2>&1; echo "scale rc=$?"; grep -E "worst|passed|failed|Error|s call" gpurun_out/r02_03_scale.log | tail -20
timeout 600 python bench.py > gpurun_out/r02_03_bench.json 2> gpurun_out/r02_03_bench.err; echo "bench rc=$?"; tail -c 3500 gpurun_out/r02_03_bench.json
RAPDHG_TRACE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.SVM, 1.0, 4)
for _ in range(2):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
    print('solve', r.iterations, r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
" > gpurun_out/r02_03_setup_trace.log 2>&1; echo "trace rc=$?"; tail -45 gpurun_out/r02_03_setup_trace.log
timeout 900 python bench.py --impl reference > gpurun_out/r02_03_bench_ref.json 2> gpurun_out/r02_03_bench_ref.err; echo "ref rc=$?"; tail -c 1200 gpurun_out/r02_03_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02_03_launches.csv python scripts/ncu_target.py svm 200 > gpurun_out/r02_03_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"DualStepOp|PrimalStepOp" -s 4 -c 8 -o gpurun_out/r02_03_c4_full python scripts/ncu_target.py svm 80 > gpurun_out/r02_03_ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/r02_03_ncu_full.log
