# round 2 call 53: W-row blocks first by default (when they fit two per SM): slab tests + C2-C4 configs
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_slab.py -q -x 2>&1 | tail -2
timeout 600 python scripts/gpu_configs.py C2 C3 C4 2>&1 | cut -c1-300 | tee gpurun_out/r02_53_configs.log
