# round 2 call 43: host slab layout without re-sorts / zero fills (metadata written into pinned
# staging): C4 setup trace, then setup time against the norm-A switch step on C2-C4
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > gpurun_out/r02_43_build.log 2>&1 || { echo build failed; tail gpurun_out/r02_43_build.log; exit 1; }
RAPDHG_TRACE=1 timeout 300 python scripts/r02/trace_c4.py > gpurun_out/r02_43_setup_trace.log 2>&1; echo "trace rc=$?"
for K in 72 56 40 24; do
  RAPDHG_NORM_SLAB_STEP=$K timeout 600 python scripts/r02/setup_k.py $K >> gpurun_out/r02_43_k.jsonl 2>> gpurun_out/r02_43_k.err
done
cat gpurun_out/r02_43_k.jsonl
