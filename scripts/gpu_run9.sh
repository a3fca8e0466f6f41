timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu9.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu9.log
echo "== pipelined"
python scripts/sweep_sched.py LASSO 1.0 800; python scripts/sweep_sched.py SVM 1.0 300; python scripts/sweep_sched.py PORTFOLIO 1.0 300
python scripts/e2e_breakdown.py 2>&1 | tail -1
make -C paper_2311_07710_b200 clean > /dev/null; make -C paper_2311_07710_b200 -j8 NVEXTRA=-DRB_PIPELINE=0 > /dev/null 2>&1
echo "== not pipelined"
python scripts/sweep_sched.py LASSO 1.0 800; python scripts/sweep_sched.py SVM 1.0 300; python scripts/sweep_sched.py PORTFOLIO 1.0 300
python scripts/e2e_breakdown.py 2>&1 | tail -1
