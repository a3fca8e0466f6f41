# streaming floor of the slab kernels: window drains and per-kernel ramp (timing-only builds)
export PYTHONUNBUFFERED=1
cd paper_2311_07710_b200
declare -A V=( [nocompfin]="-DRB_DBG_NOCOMP -DRB_DBG_NOFINW -DRB_DBG_NOOTHERS" \
               [nodrain]="-DRB_DBG_NOCOMP -DRB_DBG_NOFINW -DRB_DBG_NOOTHERS -DRB_DBG_NODRAIN" \
               [nodrain_full]="-DRB_DBG_NODRAIN" )
for k in "${!V[@]}"; do
  make -s OBJDIR=/tmp/b_$k LIBOUT=/tmp/lib_$k.so NVEXTRA="${V[$k]}" -j4 > /tmp/build_$k.log 2>&1 &
done
wait
cd ..
run() { echo "== $1 $2"; for r in 1 2; do timeout 300 env $2 python scripts/sweep_sched.py LASSO 1.0 800; done; }
for k in nocompfin nodrain nodrain_full; do run $k "RAPDHG_LIB=/tmp/lib_$k.so"; done
run nocompfin_grid1 "RAPDHG_LIB=/tmp/lib_nocompfin.so RAPDHG_SLAB_TILE=2048"
