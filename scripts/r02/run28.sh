# round 2 call 28: replicated dense rows (sharded): tests, C4 exchange volume at 8 emulated shards
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_shard.py tests/test_host_transport.py -x -q > gpurun_out/r02_28_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_28_tests.log
cat > /tmp/rep_c4.py <<'PY'
import sys, time; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.SVM, 1.0, 4)
cfg = rb.SolverConfig(tol=1e-6)
one = rb.solve(p, cfg)
for parts in (2, 4, 8):
    r = rb.solve_sharded(p, cfg, parts)
    print("parts", parts, r.status.name, r.iterations, r.restarts, "objective rel diff",
          abs(p.objective(r.point.x) - p.objective(one.point.x)) / abs(p.objective(one.point.x)), flush=True)
PY
for L in 0 1000; do echo "== RAPDHG_REPLICATE_MIN_LEN=$L"; RAPDHG_REPLICATE_MIN_LEN=$L RAPDHG_TRACE=host timeout 600 python /tmp/rep_c4.py 2>&1 | grep -E "\[shard\]|^parts"; done
