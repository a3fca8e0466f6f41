# round 2 call 45: norm-A switch at step 40 (default) + parallel order allocation: C4 trace, K sweep, slab/shard tests
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
RAPDHG_TRACE=1 timeout 300 python scripts/r02/trace_c4.py > gpurun_out/r02_45_setup_trace.log 2>&1; echo "trace rc=$?"
grep -E "joined|norms|setup total|^solve|slab plan: |layout \(host\)" gpurun_out/r02_45_setup_trace.log | tail -9
for K in 40 32; do RAPDHG_NORM_SLAB_STEP=$K timeout 600 python scripts/r02/setup_k.py $K; done > gpurun_out/r02_45_k.jsonl 2> gpurun_out/r02_45_k.err
cat gpurun_out/r02_45_k.jsonl
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_shard.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02_45_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02_45_tests.log
