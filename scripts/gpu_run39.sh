export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_colblock.py tests/test_gpu_parity.py -x -q --timeout 300 2>&1 | tail -2
for k in "LARGE 1.0 200" "LARGE_LOCAL 1.0 200"; do timeout 600 python scripts/sweep_sched.py $k 2>&1 | grep -E "^\{" | cut -c1-260; done
for mb in 16384 49152; do RAPDHG_L2BLOCK_KB=$mb timeout 600 python scripts/sweep_sched.py LARGE 1.0 200 2>&1 | grep -E "^\{" | cut -c1-260; done
RAPDHG_L2BLOCK=0 timeout 600 python scripts/sweep_sched.py LARGE 1.0 200 2>&1 | grep -E "^\{" | cut -c1-260
