"""Where an end-to-end rb.solve spends its wall time (C2)."""
import sys, time
sys.path.insert(0, ".")
import ctypes as C
import paper_2311_07710_b200 as rb
from paper_2311_07710_b200 import abi
p = rb.generate(rb.Gen.LASSO, 1.0, 2)
cfg = rb.SolverConfig(tol=1e-6, max_iters=20000)
rb.solve(p, cfg)
for _ in range(3):
    t0 = time.perf_counter()
    q = p._struct()
    c = cfg._struct()
    t1 = time.perf_counter()
    res = abi.Result()
    L = rb.lib()
    rc = L.rapdhg_solve(C.byref(q), C.byref(c), C.byref(res))
    t2 = time.perf_counter()
    r = rb.result_from_struct(res)
    L.rapdhg_result_free(C.byref(res))
    t3 = time.perf_counter()
    print("struct %.1f ms | C solve %.1f ms (setup %.1f loop %.1f) | result %.1f ms" % (
        1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * r.setup_seconds, 1e3 * r.loop_seconds, 1e3 * (t3 - t2)), flush=True)
