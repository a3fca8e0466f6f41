export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 > gpurun_out/bench75.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench75.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['time_to_tol_s'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks'])"
