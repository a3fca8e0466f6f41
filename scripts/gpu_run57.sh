export PYTHONUNBUFFERED=1
timeout 300 python scripts/setup_trace.py 2>&1 | tail -45
timeout 300 python scripts/e2e_parts.py 2>&1 | tail -4
