# in-loop cost decomposition of the slab phases (timing-only debug builds)
export PYTHONUNBUFFERED=1
cd paper_2311_07710_b200
declare -A V=( [nocomp]="-DRB_DBG_NOCOMP" [nofinw]="-DRB_DBG_NOFINW" [noothers]="-DRB_DBG_NOOTHERS" \
               [nofin]="-DRB_DBG_NOFINW -DRB_DBG_NOOTHERS" [nocompfin]="-DRB_DBG_NOCOMP -DRB_DBG_NOFINW -DRB_DBG_NOOTHERS" )
for k in "${!V[@]}"; do
  make -s OBJDIR=/tmp/b_$k LIBOUT=/tmp/lib_$k.so NVEXTRA="${V[$k]}" -j4 > /tmp/build_$k.log 2>&1 &
done
wait
cd ..
run() { echo "== $1 $2"; for r in 1 2; do timeout 300 env $2 python scripts/sweep_sched.py LASSO 1.0 800; done; }
run base ""
for k in nocomp nofinw noothers nofin nocompfin; do run $k "RAPDHG_LIB=/tmp/lib_$k.so"; done
