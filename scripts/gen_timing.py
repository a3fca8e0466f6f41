"""Device vs host C5 generation time."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb
for dev in ("1", "0"):
    os.environ["RAPDHG_GEN_DEVICE"] = dev
    for scale in (0.1, 1.0):
        if dev == "0" and scale == 1.0:
            continue
        t = time.perf_counter()
        p = rb.generate(rb.Gen.LARGE, scale, 5)
        print(f"device={dev} scale={scale}: {time.perf_counter() - t:.2f} s, nnz(A)={p.a_ineq.nnz()} nnz(Q)={p.q.nnz()}", flush=True)
