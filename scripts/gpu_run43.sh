export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
python scripts/setup_trace.py LASSO 1.0 2>&1 | tail -18
python bench.py --steps 5 --warmup 3 > gpurun_out/bench43.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench43.log | cut -c1-1200
