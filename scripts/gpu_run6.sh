timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu6.log
for e in 8 16 32; do RAPDHG_EPL=$e python scripts/sweep_sched.py LASSO 1.0 800; done 2>&1
python scripts/e2e_breakdown.py 2>&1 | tail -2
for k in RANDOM_QP:1.0 PORTFOLIO:1.0 SVM:1.0 LARGE:1.0; do python scripts/sweep_sched.py ${k%%:*} ${k##*:} 400; done 2>&1
