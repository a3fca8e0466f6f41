# round 2 call 55: C3 slab plan shapes (trace) and its step kernels after the W-first finish (launch list, full)
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
RAPDHG_TRACE=1 timeout 300 python scripts/ncu_target.py portfolio 40 2>&1 | grep -E "^\[slab\]" | head
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_55_c3_launches.csv python scripts/ncu_target.py portfolio 80 > /dev/null 2>&1; echo "launches rc=$?"
python scripts/summarize_ncu.py launches gpurun_out/r02_55_c3_launches.csv gpurun_out/r02_55_c3_shares.json | head -40
