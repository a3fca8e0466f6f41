timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu5.log
echo "== U8"
for e in 8 16 32; do RAPDHG_EPL=$e python scripts/sweep_sched.py LASSO 1.0 800; done 2>&1
python scripts/e2e_breakdown.py 2>&1 | tail -2
make -C paper_2311_07710_b200 clean > /dev/null; make -C paper_2311_07710_b200 -j8 NVEXTRA=-DRB_UNROLL_WIDE=4 > /dev/null 2>&1
echo "== U4"
for e in 8 16 32; do RAPDHG_EPL=$e python scripts/sweep_sched.py LASSO 1.0 800; done 2>&1
python scripts/e2e_breakdown.py 2>&1 | tail -2
