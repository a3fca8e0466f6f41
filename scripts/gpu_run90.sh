export PYTHONUNBUFFERED=1
echo "== default"; timeout 600 python scripts/setup_repeat10.py
echo "== reserve 4 GB"; RAPDHG_POOL_RESERVE_MB=4096 timeout 600 python scripts/setup_repeat10.py
echo "== default again"; timeout 600 python scripts/setup_repeat10.py
