export PYTHONUNBUFFERED=1
RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -E "^\[rapdhg\]     |slab plan|joined|setup total|^wall" | tail -30
