# round 2 call 5: loop-only ncu captures — C5-U (column blocks) and C4 (slab) step kernels, C4 launch list
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 40 -o gpurun_out/r02_05_c5u_full python scripts/ncu_target.py large 2 > gpurun_out/r02_05_c5u.log 2>&1; echo "c5u rc=$?"; tail -2 gpurun_out/r02_05_c5u.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 2000 --csv --log-file gpurun_out/r02_05_c4_launches.csv python scripts/ncu_target.py svm 160 > gpurun_out/r02_05_c4_launch.log 2>&1; echo "c4 launches rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 2000 --csv --log-file gpurun_out/r02_05_c5u_launches.csv python scripts/ncu_target.py large 80 > gpurun_out/r02_05_c5u_launch.log 2>&1; echo "c5u launches rc=$?"
timeout 600 python scripts/gpu_configs.py > gpurun_out/r02_05_configs.jsonl 2> gpurun_out/r02_05_configs.err; cat gpurun_out/r02_05_configs.jsonl
