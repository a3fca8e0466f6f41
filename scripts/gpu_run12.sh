timeout 900 python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/pytest_shard12.log 2>&1; echo "shard pytest rc=$?"; tail -30 gpurun_out/pytest_shard12.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu12.log 2>&1; echo "all gpu pytest rc=$?"; tail -3 gpurun_out/pytest_gpu12.log
