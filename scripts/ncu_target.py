"""A short resident solve to run under ncu: python scripts/ncu_target.py
[workload] [iterations] [strict]. workload: svm (C4, default), lasso (C2),
portfolio (C3), large / large_local (C5), random_qp (C1).

The setup (Session) runs outside the CUDA profiler range; only the solve's
kernels are inside it, so `ncu --profile-from-start off` captures the loop
(iteration and check kernels) without the setup's power iterations."""
import ctypes
import sys

sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb  # noqa: E402

GEN = {"random_qp": (rb.Gen.RANDOM_QP, 1), "lasso": (rb.Gen.LASSO, 2), "portfolio": (rb.Gen.PORTFOLIO, 3),
       "svm": (rb.Gen.SVM, 4), "large": (rb.Gen.LARGE, 5), "large_local": (rb.Gen.LARGE_LOCAL, 5)}
kind, seed = GEN[sys.argv[1] if len(sys.argv) > 1 else "svm"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 120
strict = len(sys.argv) > 3 and sys.argv[3] == "strict"
p = rb.generate(kind, 1.0, seed)
s = rb.Session(p, rb.SolverConfig(tol=1e-12, max_iters=iters, strict_parity=strict))
try:
    cudart = ctypes.CDLL("libcudart.so")
except OSError:
    import glob
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = ctypes.CDLL(cands[0]) if cands else None
if cudart:
    cudart.cudaProfilerStart()
r = s.solve()
if cudart:
    cudart.cudaProfilerStop()
print("iterations", r.iterations, "loop_s", r.loop_seconds)
