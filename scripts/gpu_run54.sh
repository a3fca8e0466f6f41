# dynamic tile tail: parity tests, then C2 timing per RAPDHG_SLAB_DYN
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_colblock.py -x -q 2>&1 | tail -5
run() { echo "== $1 $2"; for r in 1 2; do timeout 300 env $2 python scripts/sweep_sched.py LASSO 1.0 800; done; }
for d in 0 10 15 25 40; do run dyn$d "RAPDHG_SLAB_DYN=$d"; done
cd paper_2311_07710_b200
make -s OBJDIR=/tmp/b_ncf LIBOUT=/tmp/lib_ncf.so NVEXTRA="-DRB_DBG_NOCOMP -DRB_DBG_NOFINW -DRB_DBG_NOOTHERS" -j8 > /tmp/b.log 2>&1
cd ..
for d in 0 15 30; do run ncf_dyn$d "RAPDHG_LIB=/tmp/lib_ncf.so RAPDHG_SLAB_DYN=$d"; done
for d in 0 15; do echo "== SVM dyn$d"; RAPDHG_SLAB_DYN=$d timeout 300 python scripts/sweep_sched.py SVM 1.0 200; done
