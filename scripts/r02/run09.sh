# round 2 call 9: short rows without partials (slab finish "others") via SELL — suite, parity, configs
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not scale_parity" > gpurun_out/r02_09_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/r02_09_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q -s > gpurun_out/r02_09_scale.log 2>&1; echo "scale rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/r02_09_scale.log | tail -8
timeout 600 python scripts/gpu_configs.py > gpurun_out/r02_09_configs.jsonl 2> gpurun_out/r02_09_configs.err; cat gpurun_out/r02_09_configs.jsonl; tail -3 gpurun_out/r02_09_configs.err
RAPDHG_SELL=0 timeout 600 python scripts/gpu_configs.py > gpurun_out/r02_09_configs_nosell.jsonl 2>&1; cat gpurun_out/r02_09_configs_nosell.jsonl | cut -c1-200
