"""Quick look at a workload on the GPU: iterations, restarts and timing."""
import sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb

kind = rb.Gen[sys.argv[1]] if len(sys.argv) > 1 else rb.Gen.LASSO
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
maxit = int(sys.argv[4]) if len(sys.argv) > 4 else 20000
t = time.time(); p = rb.generate(kind, scale, 2); print("gen", round(time.time() - t, 2), "s", p.num_vars(), p.num_rows(), p.q.nnz(), p.a_ineq.nnz() + p.a_eq.nnz(), flush=True)
for strict in (False,):
    r = rb.solve(p, rb.SolverConfig(tol=tol, max_iters=maxit, strict_parity=strict, profile_kernels=True))
    print(f"strict={strict} {rb.to_string(r.status)} it={r.iterations} restarts={r.restarts} relkkt={r.residuals.relkkt():.3e} "
          f"solve={r.solve_seconds:.3f}s setup={r.setup_seconds:.3f}s loop={r.loop_seconds:.3f}s it/s={r.iterations / max(r.loop_seconds, 1e-9):.0f} "
          f"dual_ms={r.kernel_ms[0] / max(r.kernel_count[0], 1):.4f} primal_ms={r.kernel_ms[1] / max(r.kernel_count[1], 1):.4f} launches={r.kernel_launches}", flush=True)
    for L in r.log[:: max(1, len(r.log) // 15)]:
        print("  ", L.iteration, f"{L.r_primal:.2e} {L.r_dual:.2e} {L.r_gap:.2e} eta={L.eta:.3e} w={L.omega:.3e} R={int(L.restarted)}")
