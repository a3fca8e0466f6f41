# round 2 call 10: SELL for the slab finish's short rows (rebuilt); C4/C3/C2 slab order and tile-size sweep
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not scale_parity" > gpurun_out/r02_10_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/r02_10_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q -s > gpurun_out/r02_10_scale.log 2>&1; echo "scale rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/r02_10_scale.log | tail -8
timeout 600 python scripts/gpu_configs.py > gpurun_out/r02_10_configs.jsonl 2> gpurun_out/r02_10_configs.err; cat gpurun_out/r02_10_configs.jsonl | cut -c1-330
for env in "RAPDHG_SELL=0" "RAPDHG_SLAB_ORDER=sorted" "RAPDHG_SLAB_TILE=2048" "RAPDHG_SLAB_TILE=4096"; do
env $env timeout 300 python - <<'PY'
import json, os, sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
tag = [k + "=" + v for k, v in os.environ.items() if k in ("RAPDHG_SELL", "RAPDHG_SLAB_ORDER", "RAPDHG_SLAB_TILE")]
for name, kind, seed in (("C2", rb.Gen.LASSO, 2), ("C3", rb.Gen.PORTFOLIO, 3), ("C4", rb.Gen.SVM, 4)):
    p = rb.generate(kind, 1.0, seed)
    s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=400, profile_kernels=2))
    s.solve(); r = s.solve(); bi, _, _ = s.bytes(); s.close()
    ks = [round(1e3 * r.kernel_ms[i] / r.kernel_count[i], 1) if r.kernel_count[i] else None for i in range(2)]
    print(json.dumps({"env": tag, "config": name, "it_per_s": round(r.iterations / r.loop_seconds, 1), "inloop_us": ks}), flush=True)
PY
done
