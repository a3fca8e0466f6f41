# round 2 call 44: C4 norm-A cost against the switch step (all rowwise, early, default)
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
for K in -1 0 8 40 72; do
  echo "K=$K"
  RAPDHG_NORM_SLAB_STEP=$K RAPDHG_TRACE=1 timeout 300 python scripts/r02/trace_c4.py 2>&1 | grep -E "norms|setup total|^solve|slab plan: |power iteration" | tail -7
done > gpurun_out/r02_44_k_trace.log
cat gpurun_out/r02_44_k_trace.log
