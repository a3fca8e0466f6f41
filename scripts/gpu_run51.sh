# per-CTA slab timeline (RB_SLAB_PROFILE build made on the box)
export PYTHONUNBUFFERED=1
make -s -C paper_2311_07710_b200 OBJDIR=/tmp/b_prof LIBOUT=/tmp/lib_prof.so NVEXTRA="-DRB_SLAB_PROFILE" -j8 > /tmp/bp.log 2>&1 || { tail /tmp/bp.log; exit 1; }
for k in 1 2; do
RAPDHG_LIB=/tmp/lib_prof.so python - <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
s = rb.Session(p, rb.SolverConfig(tol=1e-9, max_iters=400))
s.solve(); r = s.solve(); print("it/s", r.iterations / r.loop_seconds)
del s
PY
done
