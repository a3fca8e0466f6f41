export PYTHONUNBUFFERED=1
timeout 300 python scripts/e2e_parts.py 2>&1 | tail -4
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -E "upload|setup total|wall|scaling|norm"
