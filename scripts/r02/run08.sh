# round 2 call 8: SELL in index order (and sigma sweep) on C5 / C1
export PYTHONUNBUFFERED=1
for sig in 32 256; do for sell in 1 0; do
RAPDHG_SELL=$sell RAPDHG_SELL_SIGMA=$sig timeout 300 python - <<'PY'
import json, os, sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
for name, kind, scale, seed in (("C5-U", rb.Gen.LARGE, 1.0, 5), ("C5-L", rb.Gen.LARGE_LOCAL, 1.0, 5), ("C1", rb.Gen.RANDOM_QP, 1.0, 1)):
    p = rb.generate(kind, scale, seed)
    s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=400 if name == "C1" else 200))
    s.solve(); r = s.solve(); bi, _, _ = s.bytes(); s.close()
    print(json.dumps({"sell": os.environ["RAPDHG_SELL"], "sigma": os.environ["RAPDHG_SELL_SIGMA"], "config": name,
                      "it_per_s": round(r.iterations / r.loop_seconds, 1),
                      "iter_GBs": round(bi * r.iterations / r.loop_seconds / 1e9, 1)}), flush=True)
PY
done; done
