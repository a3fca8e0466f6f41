# round 2 call 51: slab CTAs per SM (2 by occupancy vs 1) and tile stages (3 / 5 / 6) on C2-C4
export PYTHONUNBUFFERED=1
for ST in 3 5 6; do
  rm -rf /tmp/objst; make -C paper_2311_07710_b200 -j8 OBJDIR=/tmp/objst NVEXTRA=-DRB_SLAB_STAGES=$ST > /dev/null 2>&1 || { echo build failed; exit 1; }
  for C in 0 1; do
    [ $ST != 3 ] && [ $C = 0 ] && continue
    echo "STAGES=$ST CTAS=$C"; RAPDHG_SLAB_CTAS=$C timeout 600 python scripts/gpu_configs.py C2 C3 C4 2>&1 | cut -c1-300
  done
done > gpurun_out/r02_51_stages.log
echo "STAGES=3 CTAS=0 (again)" >> gpurun_out/r02_51_stages.log
rm -rf /tmp/objst; make -C paper_2311_07710_b200 -j8 OBJDIR=/tmp/objst > /dev/null 2>&1
timeout 600 python scripts/gpu_configs.py C2 C3 C4 2>&1 | cut -c1-300 >> gpurun_out/r02_51_stages.log
cat gpurun_out/r02_51_stages.log
