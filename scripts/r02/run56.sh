# round 2 call 56: two W rows per finish thread (RAPDHG_FINISH_ROWS=2) — bit identity and C2-C4 throughput
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python scripts/r02/finish_rows_check.py 2>&1 | tail -4
for R in 1 2 1 2; do
  echo "ROWS=$R"; RAPDHG_FINISH_ROWS=$R timeout 600 python scripts/gpu_configs.py C2 C3 C4 2>&1 | cut -c1-300
done > gpurun_out/r02_56_rows.log
cat gpurun_out/r02_56_rows.log
