export PYTHONUNBUFFERED=1
RAPDHG_LIB=paper_2311_07710_b200/librapdhg_b200_prof.so timeout 200 python scripts/sweep_sched.py LASSO 1.0 200 2>&1 | cut -c1-250
RAPDHG_LIB=paper_2311_07710_b200/librapdhg_b200_prof.so RAPDHG_SLAB_V=2 timeout 200 python scripts/sweep_sched.py LASSO 1.0 200 2>&1 | cut -c1-250
