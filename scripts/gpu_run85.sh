# finish-kernel occupancy (min blocks per SM in the launch bounds)
export PYTHONUNBUFFERED=1
cd paper_2311_07710_b200
for mb in 6 8; do make -s OBJDIR=/tmp/b_mb$mb LIBOUT=/tmp/lib_mb$mb.so NVEXTRA="-DRB_FINISH_MINB=$mb" -j4 > /tmp/bmb$mb.log 2>&1 & done; wait
cd ..
cuobjdump -res-usage /tmp/lib_mb8.so 2>/dev/null | grep -A1 "slab_finish_kernel" | grep -o "REG:[0-9]*\|LOCAL:[0-9]*" | head -8
for lib in paper_2311_07710_b200/librapdhg_b200.so /tmp/lib_mb6.so /tmp/lib_mb8.so; do echo "== $lib"
RAPDHG_LIB=$lib timeout 600 python - <<'PY'
import json, sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
for name, kind, seed in (("C2", rb.Gen.LASSO, 2), ("C3", rb.Gen.PORTFOLIO, 3), ("C4", rb.Gen.SVM, 4)):
    p = rb.generate(kind, 1.0, seed)
    s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=400, profile_kernels=2))
    s.solve(); r = s.solve(); s.close()
    print(name, round(r.iterations / r.loop_seconds), [round(1e3 * r.kernel_ms[i] / r.kernel_count[i], 1) for i in range(2)], flush=True)
PY
done
