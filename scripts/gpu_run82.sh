export PYTHONUNBUFFERED=1
for o in "" natural sorted; do echo "== order '$o'"; env ${o:+RAPDHG_SLAB_ORDER=$o} RAPDHG_TRACE=1 timeout 300 python scripts/check_cost.py 2>&1 | grep -E "padded|check_interval" | head -4; done
