"""The reference beside the B200 on the other SURVEY §8(d) configs (BASELINE.md
§3: "setup plus a fixed 50-200-iteration loop on the reference beside the
GPU"): per config, on the same instance and the same host, the reference's
own solve() (oracle/_ref, single thread) with max_iters = 0 (setup) and with
a fixed iteration count, and the library's solve from host arrays with the
same settings. C4 is bench.py's workload (profiles/r02_bench_c4*.json); C5 is
run at scale 0.1 (1e7 nnz: the reference's setup at 1e8 nnz takes minutes).

    python scripts/reference_configs.py > profiles/r02_reference_configs.jsonl
"""
import json
import sys
import time

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2311_07710_b200 as rb  # noqa: E402

oracle.build()
O = oracle.ref() if oracle.have_ref() else oracle.port()
kind = "reference" if oracle.have_ref() else "port"
CASES = [("C1 random QP", rb.Gen.RANDOM_QP, 1.0, 1, None), ("C2 lasso", rb.Gen.LASSO, 1.0, 2, 200),
         ("C3 portfolio", rb.Gen.PORTFOLIO, 1.0, 3, 100), ("C5-U large (scale 0.1)", rb.Gen.LARGE, 0.1, 5, 100),
         ("C5-L large local (scale 0.1)", rb.Gen.LARGE_LOCAL, 0.1, 5, 100)]
for name, gen, scale, seed, iters in CASES:
    p = rb.generate(gen, scale, seed)
    cfg = rb.SolverConfig(tol=1e-6) if iters is None else rb.SolverConfig(tol=1e-14, max_iters=iters)
    # the library: one warm solve, then the timed one (from host arrays: setup included)
    rb.solve(p, cfg)
    g = rb.solve(p, cfg)
    # the reference: setup only, then the same solve
    t = time.perf_counter()
    O.solve(p, rb.SolverConfig(max_iters=0))
    setup = time.perf_counter() - t
    t = time.perf_counter()
    r = O.solve(p, cfg)
    full = time.perf_counter() - t
    line = {"config": name, "n": p.num_vars(), "m": p.num_rows(), "nnz_A": p.a_ineq.nnz() + p.a_eq.nnz(),
            "nnz_Q": p.q.nnz(), "iterations": r.iterations, "same_iterations": r.iterations == g.iterations,
            "reference": {"kind": kind, "setup_s": setup, "solve_s": full,
                          "loop_it_s": r.iterations / max(full - setup, 1e-9)},
            "b200": {"setup_s": g.setup_seconds, "solve_s": g.solve_seconds,
                     "loop_it_s": g.iterations / max(g.loop_seconds, 1e-12)}}
    line["speedup_solve"] = full / g.solve_seconds
    line["speedup_loop"] = line["b200"]["loop_it_s"] / line["reference"]["loop_it_s"]
    print(json.dumps(line), flush=True)
