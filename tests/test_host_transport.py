"""The sharded solver's host-staged transport (rapdhg_host_transport) over
real torch.distributed process groups.

CPU (gloo, 2 and 3 processes): the LIBRARY drives the Python callbacks of
ProcessGroupTransport (rapdhg_host_transport_check: allgather-v over uneven
slices, all-to-all-v, min-reduction, every delivery checked on arrival).

GPU (gloo, 2 processes sharing cuda:0): ShardedEngine itself runs one shard
per process, its exchanges going through the transport (allgather-v of y / w /
x_md or packed halos, reduction partials, first-bad vote), and the result is
bit-identical to the single-GPU solve — the multi-process library path that
the NCCL transport takes on a multi-GPU node, exercised on the one GPU a box
has (the ranks' kernels never wait on each other on the device: every
exchange completes on the host)."""
import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    sys.path[:0] = [os.path.dirname(HERE), HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _check_worker(rank, world, port, q):
    try:
        dist = _init(rank, world, port)
        import paper_2311_07710_b200 as rb

        t = rb.ProcessGroupTransport()
        for length in (0, 1, 37, 5000):
            t.check(length)
        q.put((rank, "ok", ""))
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        q.put((rank, "error", repr(e)))


def _solve_worker(rank, world, port, q, halo):
    try:
        os.environ["RAPDHG_HALO"] = "on" if halo else "off"
        dist = _init(rank, world, port)
        import paper_2311_07710_b200 as rb
        from test_oracle import assert_results_identical

        p = rb.generate(rb.Gen.LASSO, 0.05, 2)
        cfg = rb.SolverConfig(tol=1e-6, max_iters=1500, snapshot_interval=80, record_restart_points=True)
        t = rb.ProcessGroupTransport()
        got = rb.solve_sharded(p, cfg, transport=t)
        s = rb.ShardSession(p, cfg, transport=t)  # persistent session, two solves
        again = [s.solve(), s.solve()]
        s.close()
        want = rb.solve(p, cfg)
        assert_results_identical(got, want)
        for r in again:
            assert_results_identical(r, want)
        assert not t.errors, t.errors
        q.put((rank, "ok", f"{got.iterations} it"))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e)))


def _run(target, world, *args, timeout=300):
    torch_mp = pytest.importorskip("torch.multiprocessing")
    ctx = torch_mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q, *args)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=timeout) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert all(status == "ok" for _, status, _ in res), res
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_library_drives_process_group_callbacks(world):
    _run(_check_worker, world)


@pytest.mark.gpu
@pytest.mark.parametrize("halo", [False, True])
def test_two_process_sharded_solve_bit_identical(halo):
    _run(_solve_worker, 2, halo, timeout=600)


def _replicated_worker(rank, world, port, q):
    try:
        os.environ["RAPDHG_REPLICATE_MIN_LEN"] = "100"
        dist = _init(rank, world, port)
        import paper_2311_07710_b200 as rb
        from test_oracle import assert_results_identical

        p = rb.generate(rb.Gen.SVM, 0.01, 4)
        cfg = rb.SolverConfig(tol=1e-8, max_iters=600, snapshot_interval=40)
        got = rb.solve_sharded(p, cfg, transport=rb.ProcessGroupTransport())
        # the same shard count emulated in one process: the same bits
        assert_results_identical(got, rb.solve_sharded(p, cfg, world))
        q.put((rank, "ok", f"{got.iterations} it"))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e)))


@pytest.mark.gpu
def test_two_process_replicated_rows_match_emulated():
    """Replicated dense rows (RAPDHG_REPLICATE_MIN_LEN) through the host
    transport: the partial sums' allgather runs over the process group, and
    the result is the emulated run's with the same shard count, bit for bit."""
    _run(_replicated_worker, 2, timeout=600)
