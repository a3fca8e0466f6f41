export PYTHONUNBUFFERED=1
for t in 4 8 16; do echo "== plan threads $t"; RAPDHG_PLAN_THREADS=$t RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -E "tiles|tile arrays|counts|upload \+ fill|slab plan|joined|setup total|^wall" | tail -14; done
