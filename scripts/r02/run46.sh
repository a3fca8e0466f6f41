# round 2 call 46: C3 portfolio step kernels — launch list of a 80-iteration solve + --set full of the step kernels
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
: timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_46_c3_launches.csv python scripts/ncu_target.py portfolio 80 > gpurun_out/r02_46_launch.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k regex:"slab.*StepOp" -s 8 -c 8 -o gpurun_out/r02_46_c3_full -f \
  python scripts/ncu_target.py portfolio 80 > gpurun_out/r02_46_full.log 2>&1; echo "full rc=$?"
python scripts/summarize_ncu.py full gpurun_out/r02_46_c3_full.ncu-rep gpurun_out/r02_46_c3_full.json 2>&1 | head -80
