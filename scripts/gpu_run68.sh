export PYTHONUNBUFFERED=1
for k in PORTFOLIO SVM LARGE LARGE_LOCAL; do echo "== $k"; s=1.0; RAPDHG_TRACE=1 timeout 600 python scripts/sweep_sched.py $k $s 200 2>&1 | grep -E "^\[slab\]|^\{" ; done
