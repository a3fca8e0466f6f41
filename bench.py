#!/usr/bin/env python
"""bench.py — rAPDHG iteration throughput on B200 (BASELINE.json metric).

Workload (BASELINE configs[1]): synthetic Lasso QP, 1e5
features x 1e4 samples -> n = m = 210,000, nnz(A) ~ 1.04e7, solved with the
reference's default SolverConfig except tol (1e-6).

A "step" is one full rAPDHG solve (zero start -> relKKT <= tol, capped at
--max-iters) on the HBM-resident, preprocessed problem (rapdhg_session_solve):
`value` = iterations / device time of the loop (CUDA events on the solver's
stream), summed over ranks. `e2e` is the same metric through the public C-ABI
entry rapdhg_solve() from HOST arrays: upload, validation, scaling, norm
estimation, the loop and the download of the solution all inside the timed
region. N > 1 GPUs run independent replicas ("replicas only": C2 does not
shard), scaling "weak".

--impl reference times the reference's own CPU solver (oracle/_ref, compiled
unmodified from /root/reference) on the same instance: a step is a bounded
solve of --ref-iters iterations; value = iterations / loop seconds (setup
subtracted), single thread (the reference is single-threaded by design,
SPEC.md:327).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402



# BASELINE.json's metric, verbatim (both arms): the value is rAPDHG iterations
# per second of the solve loop; time-to-1e-6 and the HBM roofline ride along
METRIC = "rAPDHG iters/sec and time-to-1e-6 KKT; SpMV HBM GB/s vs roofline"

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="lasso", choices=["lasso", "random_qp", "portfolio", "svm", "large"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--max-iters", type=int, default=20000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-iters", type=int, default=160)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strict", action="store_true", help="bit-exact strict mode")
    ap.add_argument("--shard", action="store_true",
                    help="row-shard ONE instance across the torchrun ranks (NCCL) instead of replicas")
    ap.add_argument("--shard-emulate", type=int, default=0,
                    help="run this many shards in one process (single-GPU functional check)")
    return ap.parse_args()


GEN = {"lasso": 2, "random_qp": 1, "portfolio": 3, "svm": 4, "large": 5}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def ncu_traffic(dom):
    """DRAM bytes (read + write) per launch of the dominant step's kernels (its
    slab kernel + finish kernel) from the committed `ncu --set full` capture of
    this code (profiles/r01_slab_ncu_full.json, values in MB), or None."""
    path = os.path.join(ROOT, "profiles", "r01_slab_ncu_full.json")
    try:
        with open(path) as f:
            rows = json.load(f)
    except (OSError, ValueError):
        return None
    op = ["DualStepOp", "PrimalStepOp"][dom]
    hit = [r for r in rows if op in r.get("Kernel Name", "")]
    if not hit:
        return None
    return 1e6 * sum(float(r["dram__bytes_read.sum"]) + float(r["dram__bytes_write.sum"]) for r in hit)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def qp_bytes(p):
    b = 0
    for m in (p.q, p.a_ineq, p.a_eq):
        b += m.row_ptr.nbytes + m.col_idx.nbytes + m.values.nbytes
    return b + p.c.nbytes + p.b_ineq.nbytes + p.b_eq.nbytes


def make_instance(args):
    import paper_2311_07710_b200 as rb

    t = time.perf_counter()
    p = rb.generate(GEN[args.workload], args.scale, args.seed)
    return p, time.perf_counter() - t


def workload_desc(args, p):
    return {"workload": f"{args.workload} (SURVEY C2)" if args.workload == "lasso" else args.workload,
            "n": p.num_vars(), "m": p.num_rows(), "m_eq": p.num_eq(),
            "nnz_A": p.a_ineq.nnz() + p.a_eq.nnz(), "nnz_Q": p.q.nnz(), "scale": args.scale,
            "seed": args.seed, "tol": args.tol, "max_iters": args.max_iters,
            "solver_config": "reference SolverConfig defaults (APDHG, PDQP restart, adaptive step, "
                             "adaptive omega, Ruiz+l2+PC scaling, check every 40) except tol",
            "l2_policy": "inputs larger than L2: each iteration streams A, A' and Q "
                         "(>= 250 MB) through the 126 MB L2"}


def reference_solver():
    import oracle

    oracle.build()
    if oracle.have_ref():
        return oracle.ref(), "reference"
    return oracle.port(), "port"


def reference_setup_seconds(O, p, reps=2):
    """Median wall time of the reference's solve() with max_iters = 0: its
    setup (validate, scaling, norms, first candidate; solver.hpp:277-341)."""
    import paper_2311_07710_b200 as rb

    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.solve(p, rb.SolverConfig(max_iters=0))
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def reference_sample(O, p, iters, setup):
    """One bounded reference solve; loop time = wall - setup (median)."""
    import paper_2311_07710_b200 as rb

    t0 = time.perf_counter()
    r = O.solve(p, rb.SolverConfig(tol=1e-12, max_iters=iters))
    return r.iterations, max(time.perf_counter() - t0 - setup, 1e-9)


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    p, _ = make_instance(args)
    desc = workload_desc(args, p)
    O, kind = reference_solver()
    setup = reference_setup_seconds(O, p)
    for _ in range(min(args.warmup, 1)):  # CPU: one warm-up sample is enough
        reference_sample(O, p, args.ref_iters, setup)
    its = loop = 0.0
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        i, l_ = reference_sample(O, p, args.ref_iters, setup)
        its += i
        loop += l_
    wall = time.perf_counter() - t_wall
    v = its / loop
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iter/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": desc,
        "cpu_baseline": {"value": v, "unit": "iter/s", "cores": 1, "kind": kind,
                         "sample": f"C2, {args.ref_iters} iterations per step, the reference's setup "
                                   f"({setup:.2f} s, median of 2 setup-only solves) subtracted, single thread"},
        "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, p, desc, rank, world, local, dist, barrier, allmax):
    """Strong scaling: ONE instance row-sharded over the ranks:
    NCCL allgather-v of y, w, x_md between the dual and primal steps. A step is
    one full sharded solve; value = iterations / max-over-ranks loop time.
    --shard-emulate P runs P shards in one process (single-GPU functional run)."""
    import paper_2311_07710_b200 as rb

    cfg = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local)

    def fresh_kw():  # an ncclUniqueId bootstraps exactly one communicator
        if args.shard_emulate:
            return dict(parts=args.shard_emulate, emulate=True)
        uid = rb.nccl_unique_id() if rank == 0 else None
        if dist:
            obj = [uid]
            dist[1].broadcast_object_list(obj, src=0)
            uid = obj[0]
        return dict(parts=world, emulate=False, rank=rank, nccl_id=uid)

    kw = fresh_kw()
    parts = kw["parts"]
    sess = rb.ShardSession(p, cfg, **kw)
    for _ in range(args.warmup):
        sess.solve()
    barrier()
    its, loop_s = 0, 0.0
    for _ in range(args.steps):
        r = sess.solve()
        its += r.iterations
        loop_s += r.loop_seconds
    sess.close()
    # e2e: setup + communicator + solve from host arrays, per step
    wall, e2e_its = 0.0, 0
    for _ in range(max(args.e2e_steps, 1)):
        kw = fresh_kw()
        barrier()
        t = time.perf_counter()
        r2 = rb.solve_sharded(p, cfg, **kw)
        wall += time.perf_counter() - t
        e2e_its += r2.iterations
    barrier()
    t_max = allmax(loop_s)
    wall = allmax(wall)
    if rank == 0:
        line = {"metric": "rAPDHG iters/sec (row-sharded, one instance)", "value": its / t_max, "unit": "iter/s",
                "n_gpus": world, "shards": parts, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": desc,
                "iterations_per_step": its / args.steps, "status": rb.to_string(r.status),
                "e2e": {"value": e2e_its / wall, "unit": "iter/s", "h2d_bytes_per_step": qp_bytes(p),
                        "d2h_bytes_per_step": 8 * (p.num_vars() + p.num_rows())},
                "gpu_launches": r.kernel_launches}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        tdist.init_process_group(backend)
        dist = (torch, tdist, backend)

    def barrier():
        if dist:
            dist[1].barrier()

    def allmax(x):
        if not dist:
            return x
        torch, tdist, backend = dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if dist:
            dist[1].destroy_process_group()
        return

    import paper_2311_07710_b200 as rb

    p, gen_s = make_instance(args)
    desc = workload_desc(args, p)
    if args.shard or args.shard_emulate:
        run_sharded(args, p, desc, rank, world, local, dist, barrier, allmax)
        if dist:
            dist[1].destroy_process_group()
        return
    cfg = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local, profile_kernels=True,
                          strict_parity=args.strict)
    sess = rb.Session(p, cfg)
    b_iter, b_dual, b_primal = sess.bytes()
    for _ in range(max(args.warmup, 0)):
        sess.solve()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    its = 0
    loop_s = 0.0
    kms = [0.0, 0.0]
    kcnt = [0, 0]
    launches = 0
    statuses = []
    relkkt = []
    for _ in range(args.steps):
        r = sess.solve()
        its += r.iterations
        loop_s += r.loop_seconds
        kms[0] += r.kernel_ms[0]
        kms[1] += r.kernel_ms[1]
        kcnt[0] += r.kernel_count[0]
        kcnt[1] += r.kernel_count[1]
        launches += r.kernel_launches
        statuses.append(rb.to_string(r.status))
        relkkt.append(r.residuals.relkkt())
    barrier()
    clk = clocks.stop()
    t_max = allmax(loop_s)
    value = world * its / t_max
    ms_per_step = 1e3 * t_max / args.steps

    # roofline of the dominant kernel (CUDA events around every launch)
    peak, peak_kind = peaks()
    k_avg = [kms[i] / kcnt[i] if kcnt[i] else float("nan") for i in range(2)]
    dom = 1 if kms[1] >= kms[0] else 0
    k_bytes = [b_dual, b_primal][dom]
    achieved = k_bytes / (k_avg[dom] * 1e-3) / 1e9
    it_rate_dev = its / loop_s
    roof = {"bound": "hbm", "kernel": ["dual_step(A*w+projection)", "primal_step([Q|A']*[x_md;y]+update)"][dom],
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)", "traffic": ncu_traffic(dom),
            "traffic_source": "profiles/r01_slab_ncu_full.json (slab + finish kernel of the step, one ncu --set full "
                              "capture; tiles carry 16-bit window offsets, so DRAM bytes < algorithmic bytes)",
            "bytes_per_launch": k_bytes, "avg_launch_ms": k_avg[dom],
            "share_of_loop": k_avg[dom] * 1e-3 * its / loop_s,  # sampled launches x all iterations
            "iteration": {"B_iter": b_iter, "achieved_GBs": b_iter * it_rate_dev / 1e9,
                          "frac_of_measured": b_iter * it_rate_dev / 1e9 / peak,
                          "frac_of_8TBs": b_iter * it_rate_dev / 8e12},
            "other_kernel": {"name": ["dual_step", "primal_step"][1 - dom], "avg_launch_ms": k_avg[1 - dom],
                             "bytes_per_launch": [b_dual, b_primal][1 - dom],
                             "achieved_GBs": [b_dual, b_primal][1 - dom] / (k_avg[1 - dom] * 1e-3) / 1e9}}
    # the same steps timed in-loop (untimed extra solve, profile_kernels=2):
    # each slab kernel stamps %globaltimer when its inputs are complete, a step
    # lasts until the next step's stamp — no events between the steps, so the
    # programmatic overlap of the step boundaries is kept
    scfg = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local, profile_kernels=2,
                           strict_parity=args.strict)
    rs = None
    if not args.strict:
        ss = rb.Session(p, scfg)
        rs = ss.solve()
        ss.close()
    if rs is not None and rs.kernel_count[dom] > 0:
        span = rs.kernel_ms[dom] / rs.kernel_count[dom]
        roof["inloop"] = {"avg_step_ms": span, "achieved": k_bytes / (span * 1e-3) / 1e9,
                          "frac": k_bytes / (span * 1e-3) / 1e9 / peak, "samples": rs.kernel_count[dom],
                          "method": "%globaltimer stamp of the step's slab kernel once its inputs are complete "
                                    "(min over CTAs) to the next step's stamp, every 32nd chunk of one untimed solve"}
    sess.close()

    # e2e through the public C-ABI from host arrays
    e2e_its = 0
    e2e_wall = 0.0
    e2e_res = None
    ecfg = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local, strict_parity=args.strict)
    rb.solve(p, ecfg)  # warm-up (untimed), like the device-timed arm
    e2e_each = []
    for _ in range(args.e2e_steps):
        t = time.perf_counter()
        e2e_res = rb.solve(p, ecfg)
        e2e_each.append(time.perf_counter() - t)
        e2e_wall += e2e_each[-1]
        e2e_its += e2e_res.iterations
    e2e_wall = allmax(e2e_wall)
    h2d = qp_bytes(p)
    d2h = 8 * (p.num_vars() + p.num_rows()) + 52 * len(e2e_res.log)
    t4 = rb.solve(p, rb.SolverConfig(tol=1e-4, max_iters=args.max_iters, device=local))

    line = {
        "metric": METRIC,
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": desc,
        "iterations_per_step": its / args.steps, "status": statuses[-1], "final_relkkt": relkkt[-1],
        "time_to_tol_s": {"1e-6": e2e_res.solve_seconds if args.tol == 1e-6 else None,
                          "1e-4": t4.solve_seconds, "iters_1e-6": e2e_res.iterations, "iters_1e-4": t4.iterations,
                          "setup_s": e2e_res.setup_seconds},
        "e2e": {"value": world * e2e_its / e2e_wall, "unit": "iter/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "wall_s_per_step": e2e_wall / max(args.e2e_steps, 1),
                "wall_s_each": [round(w, 4) for w in e2e_each]},
        "roofline": roof, "gpu_launches": launches, "clocks": clk,
        "mode": "strict (bit-exact)" if args.strict else "fast (deterministic)",
        "generator_s": gen_s,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        O, kind = reference_solver()
        s_ = reference_setup_seconds(O, p)
        i, l_ = reference_sample(O, p, args.ref_iters, s_)
        line["cpu_baseline"] = {"value": i / l_, "unit": "iter/s", "cores": 1, "kind": kind,
                                "setup_s": s_,
                                "sample": f"C2, {i} iterations, the reference's setup ({s_:.2f} s, median of "
                                          f"2 setup-only solves) subtracted, single thread"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist[1].destroy_process_group()


if __name__ == "__main__":
    main()
