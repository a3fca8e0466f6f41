# round 2 call 59: refresh of the C3 and C5-U kernel profiles at HEAD (SELL passes, W-first finish)
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k regex:"slab.*StepOp" -s 8 -c 4 -o gpurun_out/r02_59_c3_full -f \
  python scripts/ncu_target.py portfolio 80 > gpurun_out/r02_59_c3.log 2>&1; echo "c3 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 12 \
  -o gpurun_out/r02_59_c5u_full -f python scripts/ncu_target.py large 2 > gpurun_out/r02_59_c5u.log 2>&1; echo "c5u full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 2000 --csv \
  --log-file gpurun_out/r02_59_c5u_launches.csv python scripts/ncu_target.py large 80 > /dev/null 2>&1; echo "c5u launches rc=$?"
