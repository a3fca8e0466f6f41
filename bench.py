#!/usr/bin/env python
"""bench.py — rAPDHG iteration throughput on B200 (BASELINE.json metric).

Workload (BASELINE configs[3], the largest single-GPU
configuration): synthetic sparse SVM QP, 1e6 samples x 1e4 features ->
n = 1,010,000, m = 2,000,000, nnz(A) ~ 5.2e7, solved to relKKT 1e-6 with the
reference's default SolverConfig otherwise. --workload lasso|portfolio|large|
large_local|random_qp selects the other SURVEY configs (parity-test cases).

A "step" is one full rAPDHG solve (zero start -> relKKT <= tol, capped at
--max-iters) on the HBM-resident, preprocessed problem (rapdhg_session_solve):
`value` = iterations / device time of the loops (CUDA events on the solver's
stream), summed over ranks. `e2e` is the same metric through the public C-ABI
entry rapdhg_solve() from HOST arrays: upload, validation, scaling, norm
estimation, the loop and the download of the solution all inside the timed
region. N > 1 GPUs (torchrun) row-shard ONE instance (NCCL,
strong scaling); --replicas runs N independent solves instead.

--impl reference times the reference's own CPU solver (oracle/_ref, the
reference's headers compiled unmodified) on the same instance, built by the
numpy restatement of the generator (oracle/synth.py) so that none of the
repository's native code is loaded: one setup-only solve (max_iters = 0) and
one full solve to tol; value = iterations / (full - setup) wall seconds,
single thread (the reference is single-threaded by design).
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="svm",
                    choices=["svm", "lasso", "random_qp", "portfolio", "large", "large_local"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=None, help="default: the SURVEY seed of the workload")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--max-iters", type=int, default=20000)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-steps", type=int, default=20, help="reference inner steps timed for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strict", action="store_true", help="bit-exact strict mode")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent solves per rank instead of one row-sharded instance")
    ap.add_argument("--replicate-min-len", type=int, default=None,
                    help="sharded runs: replicate the rows of [Q | A'] with at least this many entries "
                         "(default: 1000 for svm — its feature rows — else none; -1 none)")
    ap.add_argument("--shard-emulate", type=int, default=0,
                    help="run this many shards in one process (single-GPU functional check)")
    a = ap.parse_args()
    if a.seed is None:
        a.seed = SEED[a.workload]
    return a


GEN = {"random_qp": 1, "lasso": 2, "portfolio": 3, "svm": 4, "large": 5, "large_local": 6}
SEED = {"random_qp": 1, "lasso": 2, "portfolio": 3, "svm": 4, "large": 5, "large_local": 5}
NAME = {"random_qp": "C1 random QP (BASELINE configs[0])", "lasso": "C2 Lasso (BASELINE configs[1])",
        "portfolio": "C3 Markowitz portfolio (BASELINE configs[2])",
        "svm": "C4 sparse SVM (BASELINE configs[3])", "large": "C5-U large random QP (BASELINE configs[4])",
        "large_local": "C5-L large random QP, block-local columns (BASELINE configs[4])"}


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


def ncu_traffic(workload, dom):
    """DRAM bytes (read + write) per launch of the dominant step's kernels
    from the committed `ncu --set full` capture of this code for the workload
    (profiles/r02_<workload>_ncu_full.json, scripts/summarize_ncu.py format:
    values in MB), or None."""
    path = os.path.join(ROOT, "profiles", f"r02_{workload}_ncu_full.json")
    try:
        with open(path) as f:
            rows = json.load(f)
    except (OSError, ValueError):
        return None, None
    op = ["DualStepOp", "PrimalStepOp"][dom]
    hit = [r for r in rows if op in r.get("Kernel Name", "")]
    if not hit:
        return None, None
    # one step = one launch of each distinct kernel of that op (slab + finish,
    # or the column-block passes); the capture may hold several steps
    per = {}
    for r in hit:
        per.setdefault(r["Kernel Name"], []).append(
            1e6 * (float(r["dram__bytes_read.sum"]) + float(r["dram__bytes_write.sum"])))
    return sum(float(np.mean(v)) for v in per.values()), os.path.relpath(path, ROOT)


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


def pinned_qp(p):
    """The e2e leg's inputs: the instance's arrays copied once (untimed) into
    page-locked host memory, the contract's "pinned host memory" — the library
    then DMAs them directly instead of staging pageable arrays."""
    try:
        import torch
        if not torch.cuda.is_available():
            return p
    except ImportError:
        return p
    import copy

    def pin(a):
        t = torch.empty(a.shape, dtype=getattr(torch, a.dtype.name), pin_memory=True)
        out = t.numpy()
        out[...] = a
        return out

    q = copy.copy(p)
    for name in ("q", "a_ineq", "a_eq"):
        m = copy.copy(getattr(p, name))
        m.row_ptr, m.col_idx, m.values = pin(m.row_ptr), pin(m.col_idx), pin(m.values)
        setattr(q, name, m)
    q.c, q.b_ineq, q.b_eq = pin(p.c), pin(p.b_ineq), pin(p.b_eq)
    return q


def make_instance(args):
    import paper_2311_07710_b200 as rb

    t = time.perf_counter()
    p = rb.generate(GEN[args.workload], args.scale, args.seed)
    return p, time.perf_counter() - t


def workload_desc(args, p):
    return {"workload": NAME[args.workload] + ("" if args.scale == 1.0 else f" at scale {args.scale:g}"),
            "n": p.num_vars(), "m": p.num_rows(), "m_eq": p.num_eq(),
            "nnz_A": p.a_ineq.nnz() + p.a_eq.nnz(), "nnz_Q": p.q.nnz(), "scale": args.scale,
            "seed": args.seed, "tol": args.tol, "max_iters": args.max_iters,
            "solver_config": "reference SolverConfig defaults (APDHG, PDQP restart, adaptive step, "
                             "adaptive omega, Ruiz+l2+PC scaling, check every 40) except tol",
            "l2_policy": "inputs larger than L2: each iteration streams A, A' and Q "
                         f"({(12 * (2 * (p.a_ineq.nnz() + p.a_eq.nnz()) + p.q.nnz())) / 1e6:.0f} MB) "
                         "through the 126 MB L2; no flush between steps"}


def host_info():
    """Host provenance for the CPU numbers."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model,
            "compiler_flags": "g++ -O2 -std=c++20 -ffp-contract=off (no -march), oracle/Makefile"}


def reference_solver():
    import oracle

    oracle.build()
    if oracle.have_ref():
        return oracle.ref(), "reference"
    return oracle.port(), "port"


def run_reference_arm(args, rank, world):
    """The reference's own solve() on the same instance, built without any of
    the repository's native code (numpy generator for C4, else the package's
    generator is unavoidable and the line says so)."""
    if rank != 0:
        return
    import paper_2311_07710_b200 as rb

    t = time.perf_counter()
    if args.workload == "svm":
        from oracle import synth

        p = synth.as_qp(synth.svm(args.scale, args.seed))
        gen = "oracle/synth.py (numpy restatement of the counter-based generator; no repository .so loaded)"
    else:
        p, _ = make_instance(args)
        gen = "paper_2311_07710_b200 host generator (loads the repository library for generation only)"
    gen_s = time.perf_counter() - t
    desc = workload_desc(args, p)
    O, kind = reference_solver()
    # setup: solve() with max_iters = 0 (validate, scaling, norms, first
    # candidate; solver.hpp:277-341); then one full solve to tol
    t = time.perf_counter()
    O.solve(p, rb.SolverConfig(max_iters=0))
    setup = time.perf_counter() - t
    t = time.perf_counter()
    r = O.solve(p, rb.SolverConfig(tol=args.tol, max_iters=args.max_iters))
    full = time.perf_counter() - t
    loop = max(full - setup, 1e-9)
    v = r.iterations / loop
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iter/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * loop / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 and not args.replicas else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": desc,
        "iterations": r.iterations, "status": rb.to_string(r.status), "final_relkkt": r.residuals.relkkt(),
        "time_to_tol_s": {f"{args.tol:g}": r.solve_seconds, "setup_s": setup},
        "cpu_baseline": {"value": v, "unit": "iter/s", "cores": 1, "kind": kind, **host_info(),
                         "sample": f"one full reference solve to relKKT {args.tol:g} ({r.iterations} iterations, "
                                   f"{full:.1f} s wall) minus one setup-only solve ({setup:.1f} s); the loop "
                                   f"time is split evenly over --steps {args.steps} for ms_per_step; single "
                                   f"thread (SPEC.md:327)"},
        "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "generator": gen, "generator_s": gen_s,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(p, args):
    """The reference's inner step (inner_step_inplace, solver.hpp:156-180, on
    WorkingProblem::from of this instance) timed on the host: one call with 0
    steps (conversion + stacking) and one with --cpu-steps; a bounded sample
    (~10-30 s) of the same per-iteration work the GPU arm times."""
    import paper_2311_07710_b200 as rb

    O, kind = reference_solver()
    s = rb.IterateState.zeros(p.num_vars(), p.num_rows())
    sp = rb.StepParams(1.0, 0.0, 1e-3, 1e-3)
    t = time.perf_counter()
    O.inner_step(s, p, sp, 0)
    t0 = time.perf_counter() - t
    t = time.perf_counter()
    O.inner_step(s, p, sp, args.cpu_steps)
    t1 = time.perf_counter() - t
    per = max(t1 - t0, 1e-9) / args.cpu_steps
    return {"value": 1.0 / per, "unit": "iter/s", "cores": 1, "kind": kind, **host_info(),
            "sample": f"{args.cpu_steps} reference inner steps (inner_step_inplace: A*w, Q*x_md, A'*y and the "
                      f"vector updates) on this instance, minus the 0-step call's conversion "
                      f"({t0:.1f} s); excludes the 40-iteration checks; single thread"}


def run_sharded(args, p, desc, rank, world, local, dist, barrier, allmax):
    """Strong scaling: ONE instance row-sharded over the ranks.
    A step is one full sharded solve; value = iterations / max-over-ranks loop
    time. --shard-emulate P runs P shards in one process (single-GPU check)."""
    import paper_2311_07710_b200 as rb

    cfg = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local)

    rep = args.replicate_min_len
    if rep is None:  # C4's 1e4 dense feature rows (SURVEY §8(e) dense-coupling columns)
        rep = 1000 if args.workload == "svm" else -1

    def fresh_kw():  # an ncclUniqueId bootstraps exactly one communicator
        if args.shard_emulate:
            return dict(parts=args.shard_emulate, emulate=True, replicate_min_len=rep)
        uid = rb.nccl_unique_id() if rank == 0 else None
        if dist:
            obj = [uid]
            dist[1].broadcast_object_list(obj, src=0)
            uid = obj[0]
        return dict(parts=world, emulate=False, rank=rank, nccl_id=uid, replicate_min_len=rep)

    kw = fresh_kw()
    parts = kw["parts"]
    sess = rb.ShardSession(p, cfg, **kw)
    for _ in range(max(args.warmup, 0)):
        sess.solve()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    its, loop_s, launches = 0, 0.0, 0
    for _ in range(args.steps):
        r = sess.solve()
        its += r.iterations
        loop_s += r.loop_seconds
        launches += r.kernel_launches
    barrier()
    clk = clocks.stop()
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
        line = {"metric": METRIC, "value": its / t_max, "unit": "iter/s",
                "n_gpus": world, "shards": parts, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {**desc, "parallelism": (f"row-sharded over {parts} shards (NCCL)"
                                                   if not args.shard_emulate else f"{parts} emulated shards on one GPU")
                           + (f", rows of [Q | A'] with >= {rep} entries replicated" if rep > 0 else "")},
                "iterations_per_step": its / args.steps, "status": rb.to_string(r.status),
                "e2e": {"value": e2e_its / wall, "unit": "iter/s", "h2d_bytes_per_step": qp_bytes(p),
                        "d2h_bytes_per_step": 8 * (p.num_vars() + p.num_rows())},
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if args.impl == "reference":  # rank 0 alone; no process group, no GPU
        run_reference_arm(args, rank, world)
        return
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

    import paper_2311_07710_b200 as rb

    p, gen_s = make_instance(args)
    desc = workload_desc(args, p)
    if (world > 1 and not args.replicas) or args.shard_emulate:
        run_sharded(args, p, desc, rank, world, local, dist, barrier, allmax)
        if dist:
            dist[1].destroy_process_group()
        return
    cfg = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local, strict_parity=args.strict)
    sess = rb.Session(p, cfg)
    b_iter, b_dual, b_primal = sess.bytes()
    for _ in range(max(args.warmup, 0)):
        sess.solve()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    its, loop_s, launches = 0, 0.0, 0
    statuses, relkkt = [], []
    for _ in range(args.steps):
        r = sess.solve()
        its += r.iterations
        loop_s += r.loop_seconds
        launches += r.kernel_launches
        statuses.append(rb.to_string(r.status))
        relkkt.append(r.residuals.relkkt())
    barrier()
    clk = clocks.stop()
    sess.close()
    t_max = allmax(loop_s)
    value = world * its / t_max
    ms_per_step = 1e3 * t_max / args.steps

    # ---- roofline of the dominant kernel (untimed profiling solves) --------
    # in-loop (primary): profile_kernels=2 — each step's slab kernel stamps
    # %globaltimer once its inputs are complete (min over CTAs) and a step
    # lasts until the next step's stamp, in the first chunk of every solve; no
    # events between the steps, so the programmatic overlap is kept.
    # events (secondary): profile_kernels=1 — CUDA events around each step of
    # the first chunk (breaks the overlap of the step boundaries).
    peak, peak_kind = peaks()
    k_ms = {}
    for mode in (2, 1):
        pc = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local, profile_kernels=mode,
                             strict_parity=args.strict)
        ps = rb.Session(p, pc)
        ms, cnt = [0.0, 0.0], [0, 0]
        for _ in range(max(args.steps // 2, 4)):
            rr = ps.solve()
            for i in range(2):
                ms[i] += rr.kernel_ms[i]
                cnt[i] += rr.kernel_count[i]
        ps.close()
        k_ms[mode] = [ms[i] / cnt[i] if cnt[i] else float("nan") for i in range(2)], cnt
    inloop_ok = all(c > 0 for c in k_ms[2][1])
    src = 2 if inloop_ok else 1
    step_ms = k_ms[src][0]
    dom = 1 if step_ms[1] >= step_ms[0] else 0
    k_bytes = [b_dual, b_primal]
    names = ["dual_step (A~w + projection, y and y_bar updates)",
             "primal_step ([Q~|A~'] [x_md; y] + x, x_bar, w, x_md updates)"]
    achieved = k_bytes[dom] / (step_ms[dom] * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args.workload, dom)
    it_rate_dev = its / loop_s
    roof = {"bound": "hbm", "kernel": names[dom], "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_source": traffic_src and f"{traffic_src} (DRAM read + write of the step's kernels, one "
                                              f"ncu --set full capture)",
            "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
            "bytes_per_launch": k_bytes[dom], "avg_step_ms": step_ms[dom],
            "timing": "in-loop %globaltimer stamps (first chunk of each of several untimed solves)"
                      if src == 2 else "CUDA events around each step of the first chunk (untimed solves)",
            "share_of_loop": step_ms[dom] * 1e-3 * its / loop_s,
            "events": {"avg_step_ms": k_ms[1][0], "samples": k_ms[1][1],
                       "achieved_GBs": [k_bytes[i] / (k_ms[1][0][i] * 1e-3) / 1e9 for i in range(2)]},
            "inloop": {"avg_step_ms": k_ms[2][0], "samples": k_ms[2][1],
                       "achieved_GBs": [k_bytes[i] / (k_ms[2][0][i] * 1e-3) / 1e9 for i in range(2)]
                       if inloop_ok else None},
            "iteration": {"B_iter": b_iter, "achieved_GBs": b_iter * it_rate_dev / 1e9,
                          "frac_of_measured": b_iter * it_rate_dev / 1e9 / peak,
                          "frac_of_8TBs": b_iter * it_rate_dev / 8e12},
            "other_kernel": {"name": names[1 - dom], "avg_step_ms": step_ms[1 - dom],
                             "bytes_per_launch": k_bytes[1 - dom],
                             "achieved_GBs": k_bytes[1 - dom] / (step_ms[1 - dom] * 1e-3) / 1e9}}

    # ---- e2e through the public C-ABI from host arrays ----------------------
    ecfg = rb.SolverConfig(tol=args.tol, max_iters=args.max_iters, device=local, strict_parity=args.strict)
    ph = pinned_qp(p)
    for _ in range(max(1, args.warmup)):  # W untimed warm-up solves, like the device-timed arm
        rb.solve(ph, ecfg)
    e2e_its, e2e_each, e2e_res = 0, [], None
    for _ in range(max(args.e2e_steps, 1)):
        t = time.perf_counter()
        e2e_res = rb.solve(ph, ecfg)
        e2e_each.append(time.perf_counter() - t)
        e2e_its += e2e_res.iterations
    e2e_wall = allmax(sum(e2e_each))
    h2d = qp_bytes(p)
    d2h = 8 * (p.num_vars() + p.num_rows()) + 52 * len(e2e_res.log)
    t4 = rb.solve(p, rb.SolverConfig(tol=1e-4, max_iters=args.max_iters, device=local))

    line = {
        "metric": METRIC,
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {**desc, "parallelism": "single GPU" if world == 1 else f"{world} independent replicas"},
        "iterations_per_step": its / args.steps, "status": statuses[-1], "final_relkkt": relkkt[-1],
        "time_to_tol_s": {f"{args.tol:g}": e2e_res.solve_seconds, "1e-4": t4.solve_seconds,
                          f"iters_{args.tol:g}": e2e_res.iterations, "iters_1e-4": t4.iterations,
                          "setup_s": e2e_res.setup_seconds,
                          "note": "solve_seconds of rapdhg_solve from host arrays (the reference's "
                                  "definition: from solve() entry, setup included)"},
        "e2e": {"value": world * e2e_its / e2e_wall, "unit": "iter/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "wall_s_per_step": e2e_wall / len(e2e_each),
                "wall_s_each": [round(w, 4) for w in e2e_each],
                "path": "rapdhg_solve (C-ABI) from pinned host arrays: upload, validation, scaling, norms, loop, "
                        "download"},
        "roofline": roof, "gpu_launches": launches, "clocks": clk,
        "mode": "strict (bit-exact)" if args.strict else "fast (deterministic)",
        "generator_s": gen_s,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(p, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist[1].destroy_process_group()


if __name__ == "__main__":
    main()
