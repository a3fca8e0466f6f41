"""Trace the end-to-end call: Python-side phases + RAPDHG_TRACE engine phases."""
import ctypes as C, os, sys, time
sys.path.insert(0, ".")
os.environ["RAPDHG_TRACE"] = "1"
import paper_2311_07710_b200 as rb
from paper_2311_07710_b200 import abi

p = rb.generate(rb.Gen.LASSO, 1.0, 2)
L = rb.lib()
for i in range(4):
    cfg = rb.SolverConfig(tol=1e-6, max_iters=20000 if i else 40)
    t0 = time.perf_counter()
    qp = p._struct(); cs = cfg._struct(); out = abi.Result()
    t1 = time.perf_counter()
    rc = L.rapdhg_solve(C.byref(qp), C.byref(cs), C.byref(out))
    t2 = time.perf_counter()
    r = rb.result_from_struct(out)
    t3 = time.perf_counter()
    L.rapdhg_result_free(C.byref(out))
    t4 = time.perf_counter()
    print(f"call {i}: struct {1e3*(t1-t0):.1f} ms | C call {1e3*(t2-t1):.1f} ms (solve_seconds {1e3*r.solve_seconds:.1f}, setup {1e3*r.setup_seconds:.1f}, loop {1e3*r.loop_seconds:.1f}) | convert {1e3*(t3-t2):.1f} ms | free {1e3*(t4-t3):.1f} ms", flush=True)
