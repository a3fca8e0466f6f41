# slab consumer variants: build on the box, per-phase C2 timings for each
export PYTHONUNBUFFERED=1
cd paper_2311_07710_b200
declare -A V=( [c12]="-DRB_SLAB_CONSUMERS=12" [u8]="-DRB_SLAB_UNROLL=8" [acc2]="-DRB_SLAB_ACC2" \
               [u8acc2]="-DRB_SLAB_UNROLL=8 -DRB_SLAB_ACC2" [c16]="-DRB_SLAB_CONSUMERS=16" [s4]="-DRB_SLAB_STAGES=4" )
for k in "${!V[@]}"; do
  make -s OBJDIR=/tmp/b_$k LIBOUT=/tmp/lib_$k.so NVEXTRA="${V[$k]}" -j4 > /tmp/build_$k.log 2>&1 &
done
wait
cd ..
ls -la /tmp/lib_*.so
run() { echo "== $1 $2"; for r in 1 2; do timeout 300 env $2 python scripts/sweep_sched.py LASSO 1.0 800; done; }
run base ""
for k in c12 u8 acc2 u8acc2 c16 s4; do run $k "RAPDHG_LIB=/tmp/lib_$k.so"; done
run tile2048 "RAPDHG_SLAB_TILE=2048"
run tile1536 "RAPDHG_SLAB_TILE=1536"
run s4tile2048 "RAPDHG_LIB=/tmp/lib_s4.so RAPDHG_SLAB_TILE=2048"
for k in c12 u8acc2; do echo "== SVM $k"; timeout 300 env RAPDHG_LIB=/tmp/lib_$k.so python scripts/sweep_sched.py SVM 1.0 200; done
echo "== SVM base"; timeout 300 python scripts/sweep_sched.py SVM 1.0 200
