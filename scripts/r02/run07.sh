# round 2 call 7: sliced-ELL (SELL) short-row path — GPU suite, parity at scale, configs, C5 ncu
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not scale_parity" > gpurun_out/r02_07_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r02_07_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q -s > gpurun_out/r02_07_scale.log 2>&1; echo "scale rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/r02_07_scale.log | tail -8
timeout 600 python scripts/gpu_configs.py > gpurun_out/r02_07_configs.jsonl 2> gpurun_out/r02_07_configs.err; cat gpurun_out/r02_07_configs.jsonl; tail -3 gpurun_out/r02_07_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 2000 --csv --log-file gpurun_out/r02_07_c5u_launches.csv python scripts/ncu_target.py large 80 > /dev/null 2>&1; echo "c5u launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 30 -o gpurun_out/r02_07_c5u_full python scripts/ncu_target.py large 2 > gpurun_out/r02_07_c5u.log 2>&1; echo "c5u full rc=$?"
