# round 2 call 23: full GPU suite incl. at-scale parity after the slab-phase norm estimate
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not scale_parity" > gpurun_out/r02_23_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_23_tests.log
timeout 1800 python -m pytest tests/test_gpu_scale_parity.py -x -q -s --durations=0 > gpurun_out/r02_23_scale.log 2>&1; echo "scale rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/r02_23_scale.log | tail -12
