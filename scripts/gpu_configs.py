"""Per-config throughput on one B200 (fast mode, 400-iteration resident solves,
in-loop step stamps): one JSON line per SURVEY §8(d) config."""
import json
import sys

sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb  # noqa: E402

for name, kind, scale, seed in (("C1 random QP", rb.Gen.RANDOM_QP, 1.0, 1), ("C2 lasso", rb.Gen.LASSO, 1.0, 2),
                                ("C3 portfolio", rb.Gen.PORTFOLIO, 1.0, 3), ("C4 svm", rb.Gen.SVM, 1.0, 4),
                                ("C5-U large", rb.Gen.LARGE, 1.0, 5), ("C5-L large local", rb.Gen.LARGE_LOCAL, 1.0, 5)):
    if len(sys.argv) > 1 and name.split()[0] not in sys.argv[1:]:  # e.g. gpu_configs.py C2 C4
        continue
    p = rb.generate(kind, scale, seed)
    s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=400, profile_kernels=2))
    s.solve()
    r = s.solve()
    bi, bd, bp = s.bytes()
    s.close()
    ks = [r.kernel_ms[i] / r.kernel_count[i] if r.kernel_count[i] else None for i in range(2)]
    print(json.dumps({"config": name, "n": p.num_vars(), "m": p.num_rows(), "nnz_A": p.a_ineq.nnz() + p.a_eq.nnz(),
                      "nnz_Q": p.q.nnz(), "it_per_s": r.iterations / r.loop_seconds,
                      "B_iter_MB": bi / 1e6, "iter_GBs": bi * r.iterations / r.loop_seconds / 1e9,
                      "inloop_step_us": [None if k is None else 1e3 * k for k in ks],
                      "inloop_step_GBs": [None if k is None else b / (k * 1e-3) / 1e9 for k, b in zip(ks, (bd, bp))],
                      "setup_s": r.setup_seconds}), flush=True)
