"""Per-kernel timing of the C2 (or other) resident solve under the current
schedule env (RAPDHG_EPL / RAPDHG_BLOCK_MIN). One JSON line."""
import json, os, sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb

kind = rb.Gen[sys.argv[1]] if len(sys.argv) > 1 else rb.Gen.LASSO
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 800
p = rb.generate(kind, scale, 2)
s = rb.Session(p, rb.SolverConfig(tol=1e-9, max_iters=iters, profile_kernels=True))
s.solve()
r = s.solve()
bi, bd, bp = s.bytes()
dual = r.kernel_ms[0] / r.kernel_count[0]
prim = r.kernel_ms[1] / r.kernel_count[1]
print(json.dumps({"kind": kind.name, "scale": scale, "epl": os.environ.get("RAPDHG_EPL", "8"),
                  "block_min": os.environ.get("RAPDHG_BLOCK_MIN", "4096"),
                  "it_per_s": r.iterations / r.loop_seconds, "dual_ms": dual, "primal_ms": prim,
                  "dual_GBs": bd / dual / 1e6, "primal_GBs": bp / prim / 1e6,
                  "iter_GBs": bi * r.iterations / r.loop_seconds / 1e9}), flush=True)
