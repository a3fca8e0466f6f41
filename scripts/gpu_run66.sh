export PYTHONUNBUFFERED=1
RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -E "^\[rapdhg\]|^wall" | tail -34
timeout 300 python scripts/e2e_parts.py 2>&1 | tail -3
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
