# round 2 call 15: counter-based C2/C3 generators (device = host), parity at scale with the new instances
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r02_15_tests.log 2>&1; echo "tests rc=$?"; tail -9 gpurun_out/r02_15_tests.log
grep -E "worst" gpurun_out/r02_15_tests.log
timeout 600 python scripts/gpu_configs.py > gpurun_out/r02_15_configs.jsonl 2> gpurun_out/r02_15_configs.err; cut -c1-300 gpurun_out/r02_15_configs.jsonl
timeout 300 python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
for kind in (rb.Gen.LASSO, rb.Gen.PORTFOLIO, rb.Gen.SVM, rb.Gen.LARGE):
    rb.generate(kind, 0.01, 1)
    t = time.time(); p = rb.generate(kind, 1.0, 2); print(kind.name, "generate", round(time.time() - t, 3), "s", flush=True)
PY
