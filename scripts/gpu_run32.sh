export PYTHONUNBUFFERED=1
for k in "LASSO 1.0 800" "SVM 1.0 300" "PORTFOLIO 1.0 300" "LARGE 1.0 100" "RANDOM_QP 1.0 800"; do RAPDHG_TRACE=1 timeout 200 python scripts/sweep_sched.py $k 2>&1 | grep -E "^\[slab\]|^\{" | cut -c1-220; done
for k in "SVM 1.0 300" "PORTFOLIO 1.0 300" "LARGE 1.0 100"; do RAPDHG_SLAB=off timeout 200 python scripts/sweep_sched.py $k 2>&1 | cut -c1-220; done
RAPDHG_SLAB_MIN_WINDOWS=1 timeout 150 python scripts/sweep_sched.py LASSO 1.0 800 | cut -c1-220
RAPDHG_LIB=paper_2311_07710_b200/librapdhg_b200_prof.so timeout 200 python scripts/sweep_sched.py LASSO 1.0 200 2>&1 | grep -v "^  \.\.\." | cut -c1-200 | head -12
