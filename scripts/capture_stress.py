"""Concurrent sessions next to a thread using torch's legacy stream (the
test_solves_capture_beside_legacy_stream_work scenario), repeated; prints
every error in full."""
import sys
import threading
sys.path[:0] = [".", "tests"]
import torch  # noqa: E402
import paper_2311_07710_b200 as rb  # noqa: E402
from instances import random_qp  # noqa: E402

p = random_qp(43, n=2000, mi=800, me=200, dens=0.004, q_rank=500)
cfg = rb.SolverConfig(tol=1e-6, max_iters=1500)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    stop, errs = threading.Event(), []

    def noise():
        try:
            a = torch.randn(512, 512, device="cuda:0")
            while not stop.is_set():
                b = a @ a
                a = b / b.norm()
                torch.cuda.current_stream().synchronize()  # not a device-wide sync (see doc)
        except Exception as e:
            errs.append(("torch", repr(e)))

    def solves():
        try:
            for _ in range(6):
                s = rb.Session(p, cfg)
                s.solve()
                s.close()
        except Exception as e:
            errs.append(("rb", repr(e)))

    nt = threading.Thread(target=noise)
    th = [threading.Thread(target=solves) for _ in range(2)]
    nt.start()
    for t in th:
        t.start()
    for t in th:
        t.join()
    stop.set()
    nt.join()
    print("rep", rep, "errors:", errs, flush=True)
