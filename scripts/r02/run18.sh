# round 2 call 18: C4 setup knobs for the power iteration (windows, bins), pinned-input e2e bench
export PYTHONUNBUFFERED=1
cat > /tmp/trace_c4.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.SVM, 1.0, 4)
for _ in range(2):
    r = rb.solve(p, rb.SolverConfig(tol=1e-6))
print('solve', r.iterations, r.norm_a, r.solve_seconds, r.setup_seconds, r.loop_seconds, flush=True)
PY
for env in "X=1" "RAPDHG_WINDOW=force" "RAPDHG_EPL=2" "RAPDHG_EPL=4" "RAPDHG_EPL=8"; do
  echo "== $env"
  env $env RAPDHG_TRACE=host timeout 300 python /tmp/trace_c4.py 2>&1 | grep -E "norm A|norm Q|upload \+ stack|setup total|^solve" | tail -5
done
timeout 600 python bench.py > gpurun_out/r02_18_bench.json 2> gpurun_out/r02_18_bench.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.loads(open('gpurun_out/r02_18_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['e2e']['wall_s_each'], d['time_to_tol_s'])
PY
