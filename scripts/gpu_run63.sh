export PYTHONUNBUFFERED=1
nproc; lscpu | grep -E "Model name|Socket|Thread|NUMA node\(s\)"
for t in 4 8 12 16; do echo "== threads $t"; RAPDHG_STAGE_THREADS=$t RAPDHG_TRACE=host timeout 300 python scripts/setup_trace.py 2>&1 | grep -E "upload \+ stack|setup total|^wall"; done
