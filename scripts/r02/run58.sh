# round 2 call 58: column-block passes as programmatic dependent launches — colblock/parity tests + C5 configs
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_colblock.py tests/test_gpu_sell.py -q -x 2>&1 | tail -1
for i in 1 2; do timeout 900 python scripts/gpu_configs.py C5-U 2>&1 | cut -c1-200; done | tee gpurun_out/r02_58_c5.log
RAPDHG_PDL=0 timeout 900 python scripts/gpu_configs.py C5-U 2>&1 | cut -c1-200 | tee -a gpurun_out/r02_58_c5.log
