timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu10.log
for w in auto off; do echo "== window $w"; RAPDHG_WINDOW=$w python scripts/sweep_sched.py LASSO 1.0 800; RAPDHG_WINDOW=$w python scripts/sweep_sched.py SVM 1.0 300; RAPDHG_WINDOW=$w python scripts/sweep_sched.py PORTFOLIO 1.0 300; done 2>&1
python scripts/e2e_breakdown.py 2>&1 | tail -1
make -C paper_2311_07710_b200 clean > /dev/null; make -C paper_2311_07710_b200 -j8 NVEXTRA=-DRB_DUAL_UNROLL=4 > /dev/null 2>&1
echo "== dual unroll 4"; python scripts/sweep_sched.py LASSO 1.0 800; python scripts/sweep_sched.py SVM 1.0 300
