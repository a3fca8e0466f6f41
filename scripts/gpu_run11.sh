timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu11.log
for v in default variants/lib_dual_u4.so; do
  if [ $v = default ]; then unset RAPDHG_LIB; else export RAPDHG_LIB=$PWD/paper_2311_07710_b200/$v; fi
  echo "== $v"; python scripts/sweep_sched.py LASSO 1.0 800; python scripts/sweep_sched.py SVM 1.0 300; python scripts/sweep_sched.py PORTFOLIO 1.0 300
done 2>&1
unset RAPDHG_LIB
RAPDHG_WINDOW=auto python scripts/sweep_sched.py SVM 1.0 300
