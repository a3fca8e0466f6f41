export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench76.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench76.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value']); print(json.dumps(d['roofline'], indent=1))"
