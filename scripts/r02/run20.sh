# round 2 call 20: pinned result blocks + zero-copy Python views: GPU suite (minus scale parity), bench
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not scale_parity" > gpurun_out/r02_20_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_20_tests.log
timeout 600 python bench.py > gpurun_out/r02_20_bench.json 2> gpurun_out/r02_20_bench.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.loads(open('gpurun_out/r02_20_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['e2e']['wall_s_each'], d['time_to_tol_s'])
PY
