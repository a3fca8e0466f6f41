export PYTHONUNBUFFERED=1
for w in off auto force; do echo "== RAPDHG_WINDOW=$w"; RAPDHG_WINDOW=$w RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -E "norm A|setup total|^wall" | tail -3; done
