# round 2 call 47: slab finish kernel occupancy (min blocks per SM 1 / 4 / 5) on C2-C5
export PYTHONUNBUFFERED=1
for MB in 1 5 4; do
  rm -rf /tmp/objmb; make -C paper_2311_07710_b200 -j8 OBJDIR=/tmp/objmb NVEXTRA=-DRB_FINISH_MINB=$MB > /dev/null 2>&1 || { echo build failed; exit 1; }
  echo "MINB=$MB"; timeout 600 python scripts/gpu_configs.py 2>&1 | cut -c1-330 | grep -v "C1 "
done > gpurun_out/r02_47_minb.log
cat gpurun_out/r02_47_minb.log
rm -rf /tmp/objmb; make -C paper_2311_07710_b200 -j8 OBJDIR=/tmp/objmb > /dev/null 2>&1
