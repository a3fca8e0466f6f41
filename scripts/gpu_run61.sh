export PYTHONUNBUFFERED=1
RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -v "^\[slab\]"
timeout 300 python scripts/e2e_parts.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_slab.py tests/test_gpu_colblock.py -x -q 2>&1 | tail -2
