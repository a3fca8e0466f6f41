# slab windows in device memory (up to 1024 per op): tests, then C2/C3/C4 timings
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_colblock.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for k in LASSO PORTFOLIO SVM; do echo "== $k"; RAPDHG_TRACE=1 timeout 600 python scripts/sweep_sched.py $k 1.0 200 2>&1 | grep -E "^\[slab\] seg|^\{" ; done
