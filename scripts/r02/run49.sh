# round 2 call 49: rowwise gather windows (RAPDHG_WINDOW=auto) for the norm estimate's rowwise steps (C4)
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
for W in off auto; do for K in -1 40; do
  echo "WINDOW=$W K=$K"
  RAPDHG_WINDOW=$W RAPDHG_NORM_SLAB_STEP=$K RAPDHG_TRACE=1 timeout 300 python scripts/r02/trace_c4.py 2>&1 | grep -E "norms|setup total|^solve" | tail -3
done; done > gpurun_out/r02_49_window.log
cat gpurun_out/r02_49_window.log
