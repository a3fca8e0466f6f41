export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -E "validate|upload|setup total|^wall" | tail -6
timeout 300 python scripts/e2e_parts.py 2>&1 | tail -3
