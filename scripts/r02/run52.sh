# round 2 call 52: finish-grid block order (W-row blocks first: 0 / 1 / auto) on C2-C4, plus the slab tests under each
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
for WF in 0 1 a 0; do
  echo "WFIRST=$WF"; RAPDHG_FINISH_WFIRST=$WF timeout 600 python scripts/gpu_configs.py C2 C3 C4 2>&1 | cut -c1-300
done > gpurun_out/r02_52_wfirst.log
cat gpurun_out/r02_52_wfirst.log
RAPDHG_FINISH_WFIRST=1 timeout 900 python -m pytest tests/test_gpu_slab.py -q -x 2>&1 | tail -1
