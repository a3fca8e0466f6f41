# round 2 call 4: resident slab plans (C4 dual) — GPU suite, smoke, bench, configs, C4 ncu
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 -k "not scale_parity" > gpurun_out/r02_04_tests.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/r02_04_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q -s > gpurun_out/r02_04_scale.log 2>&1; echo "scale rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/r02_04_scale.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_04_bench.json 2> gpurun_out/r02_04_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r02_04_bench.json')); r=d['roofline']
print('value', d['value'], 'e2e', d['e2e']['value'], 'inloop', r['inloop']['avg_step_ms'], r['inloop']['achieved_GBs'], 'iter frac', r['iteration']['frac_of_measured'], 'clk', d['clocks'])"
timeout 900 python scripts/gpu_configs.py > gpurun_out/r02_04_configs.jsonl 2> gpurun_out/r02_04_configs.err; cat gpurun_out/r02_04_configs.jsonl
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"DualStepOp|PrimalStepOp" -s 4 -c 4 -o gpurun_out/r02_04_c4_full python scripts/ncu_target.py svm 80 > gpurun_out/r02_04_ncu_full.log 2>&1; echo "ncu full rc=$?"
