python scripts/e2e_trace.py 2>&1
