# round 2 call 16: overlapped exchanges (sharded plain path) + emulated sharded timing
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -k "shard or host_transport or sell" > gpurun_out/r02_16_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/r02_16_tests.log
for ov in 1 0; do RAPDHG_OVERLAP=$ov RAPDHG_TRACE=host timeout 300 python bench.py --workload large_local --shard-emulate 4 --steps 3 --warmup 1 --max-iters 400 --tol 1e-12 --e2e-steps 1 2> gpurun_out/r02_16_emu_$ov.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap', $ov, 'value', round(d['value'],1), 'launches', d['gpu_launches'])"; grep -E "overlap|halo" gpurun_out/r02_16_emu_$ov.err | head -3; done
