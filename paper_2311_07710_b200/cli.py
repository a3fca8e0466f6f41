"""bench_cli over the B200 solver.

    python -m paper_2311_07710_b200.cli solve    FILE.qps [flags] [--out sol.json] [--log checks.csv]
    python -m paper_2311_07710_b200.cli bench    DIR [flags] [--out table.csv]
    python -m paper_2311_07710_b200.cli generate CLASS SCALE SEED OUT.qps
    python -m paper_2311_07710_b200.cli sgm10    V1 V2 ... [--limit L]

Exit codes (cli_solve): 0 optimal, 2 iteration/time limit, 3 parse error or
unreadable input, 4 numerical error. Flags mirror SPEC's DESIGN DECISIONS:
--tol, --algorithm {pdhg,apdhg}, --restart {none,fixed=K,halving,adaptive},
--step {theoretical,adaptive}, --scaling {on,off}, --max-iters, --time-limit,
--check-interval, --seed; defaults are §6 PDQP (apdhg, adaptive restart,
adaptive step, scaling on) with tol 1e-3 (the paper's low-accuracy headline).
Bench tables are deterministic apart from the seconds column: rows in sorted
file order, footer rows with the solved count and SGM10 of iterations
(unsolved clamped to 200000, §5) and of seconds (clamped to 3600, §6.1).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys
import time
from typing import List, Optional, Sequence

from . import (Algorithm, Gen, QpsParseError, RestartPolicy, SolveStatus, SolverConfig, StepRule, generate,
               read_qps, solve, to_string, write_qps)

ITER_LIMIT = 200000.0  # §5: unsolved instances count as 200000 iterations
TIME_LIMIT = 3600.0    # §6.1: ... and as 3600 s


def sgm10(values: Sequence[float], limit: Optional[float] = None) -> float:
    """Shifted geometric mean, shift 10 (SPEC sgm10): exp(mean(log(v + 10))) - 10.
    Entries above `limit` are clamped to it (unsolved instances are encoded as
    the limit by the caller)."""
    vals = [float(v) for v in values]
    if not vals:
        raise ValueError("sgm10 of an empty list")
    if any(v < 0 for v in vals):
        raise ValueError("sgm10 needs values >= 0")
    if limit is not None:
        vals = [min(v, limit) for v in vals]
    return math.exp(sum(math.log(v + 10.0) for v in vals) / len(vals)) - 10.0


def _restart(text: str):
    if text == "none":
        return RestartPolicy.kNone, 0
    if text == "halving":
        return RestartPolicy.kAdaptiveHalving, 0
    if text == "adaptive":
        return RestartPolicy.kPdqpAdaptive, 0
    if text.startswith("fixed="):
        return RestartPolicy.kFixed, int(text.split("=", 1)[1])
    raise argparse.ArgumentTypeError(f"unknown restart policy {text!r}")


def add_solver_flags(ap: argparse.ArgumentParser) -> None:
    ap.add_argument("--tol", type=float, default=1e-3)
    ap.add_argument("--algorithm", choices=["pdhg", "apdhg"], default="apdhg")
    ap.add_argument("--restart", default="adaptive", help="none | fixed=K | halving | adaptive")
    ap.add_argument("--step", choices=["theoretical", "adaptive"], default="adaptive")
    ap.add_argument("--scaling", choices=["on", "off"], default="on")
    ap.add_argument("--max-iters", type=int, default=200000)
    ap.add_argument("--time-limit", type=float, default=math.inf)
    ap.add_argument("--check-interval", type=int, default=40)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--strict", action="store_true", help="bit-exact reference arithmetic")


def config_from_args(a) -> SolverConfig:
    policy, length = _restart(a.restart)
    return SolverConfig(algorithm=Algorithm.kApdhg if a.algorithm == "apdhg" else Algorithm.kPdhg,
                        restart=policy, restart_length=length,
                        step_rule=StepRule.kAdaptive if a.step == "adaptive" else StepRule.kTheoretical,
                        tol=a.tol, max_iters=a.max_iters, time_limit_s=a.time_limit,
                        check_interval=a.check_interval, scaling=a.scaling == "on", seed=a.seed,
                        device=a.device, strict_parity=a.strict)


def config_id(a) -> str:
    return (f"{a.algorithm}-{a.restart}-{a.step}-scaling_{a.scaling}-tol{a.tol:g}"
            + ("-strict" if a.strict else ""))


def exit_code(status: SolveStatus) -> int:
    return {SolveStatus.kOptimal: 0, SolveStatus.kIterationLimit: 2, SolveStatus.kTimeLimit: 2,
            SolveStatus.kNumericalError: 4}[SolveStatus(status)]


def _write_atomic(path: str, text: str) -> None:
    tmp = f"{path}.tmp{os.getpid()}"
    with open(tmp, "w") as f:
        f.write(text)
    os.replace(tmp, path)


def cmd_solve(a) -> int:
    try:
        p = read_qps(a.file)
    except (OSError, QpsParseError) as e:
        print(f"error: {a.file}: {e}", file=sys.stderr)
        return 3
    t = time.perf_counter()
    r = solve(p, config_from_args(a))
    secs = time.perf_counter() - t
    sol = {"status": to_string(r.status), "objective": p.objective(r.point.x),
           "x": [float(v) for v in r.point.x],
           "y": [float(v) for v in r.point.y_ineq] + [float(v) for v in r.point.y_eq],  # stacked [ineq; eq]
           "relkkt": {"primal": r.residuals.r_primal, "dual": r.residuals.r_dual, "gap": r.residuals.r_gap},
           "iterations": r.iterations, "restarts": r.restarts, "seconds": secs}
    text = json.dumps(sol)
    if a.out:
        _write_atomic(a.out, text + "\n")
    else:
        print(text)
    if a.log:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(["iter", "r_primal", "r_dual", "r_gap", "eta", "omega", "restarted"])
        for rec in r.log:
            w.writerow([rec.iteration, repr(rec.r_primal), repr(rec.r_dual), repr(rec.r_gap), repr(rec.eta),
                        repr(rec.omega), int(rec.restarted)])
        _write_atomic(a.log, buf.getvalue())
    return exit_code(r.status)


QPS_SUFFIXES = (".qps", ".mps", ".QPS", ".MPS", ".sif", ".SIF")


def bench_rows(directory: str, a) -> List[list]:
    files = sorted(f for f in os.listdir(directory) if f.endswith(QPS_SUFFIXES))
    if not files:
        raise ValueError(f"{directory}: no QPS files")
    cfg, cid = config_from_args(a), config_id(a)
    rows = []
    for f in files:
        name = os.path.splitext(f)[0]
        try:
            p = read_qps(os.path.join(directory, f))
        except (OSError, QpsParseError):
            rows.append([name, cid, "parse_failure", "", "", "", "", ""])
            continue
        t = time.perf_counter()
        r = solve(p, cfg)
        secs = time.perf_counter() - t
        rows.append([name, cid, to_string(r.status), r.iterations, f"{secs:.6f}", repr(r.residuals.r_primal),
                     repr(r.residuals.r_dual), repr(r.residuals.r_gap)])
    return rows


def bench_table(rows: List[list]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["instance", "config", "status", "iterations", "seconds", "r_primal", "r_dual", "r_gap"])
    for r in rows:
        w.writerow(r)
    solved = [r for r in rows if r[2] == "optimal"]
    its = [float(r[3]) if r[2] == "optimal" else ITER_LIMIT for r in rows]
    secs = [float(r[4]) if r[2] == "optimal" else TIME_LIMIT for r in rows]
    cid = rows[0][1] if rows else ""
    w.writerow(["#solved", cid, len(solved), "", "", "", "", ""])
    w.writerow(["#sgm10_iterations", cid, repr(sgm10(its, ITER_LIMIT)), "", "", "", "", ""])
    w.writerow(["#sgm10_seconds", cid, "", "", repr(sgm10(secs, TIME_LIMIT)), "", "", ""])
    return buf.getvalue()


def cmd_bench(a) -> int:
    try:
        rows = bench_rows(a.dir, a)
    except (OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    text = bench_table(rows)
    if a.out:
        _write_atomic(a.out, text)
    else:
        sys.stdout.write(text)
    return 0


GEN_CLASSES = {"random_qp": Gen.RANDOM_QP, "lasso": Gen.LASSO, "portfolio": Gen.PORTFOLIO, "svm": Gen.SVM,
               "large": Gen.LARGE, "large_local": Gen.LARGE_LOCAL}


def cmd_generate(a) -> int:
    kind = GEN_CLASSES.get(a.cls)
    if kind is None:
        print(f"error: unknown class {a.cls!r} (one of {', '.join(sorted(GEN_CLASSES))})", file=sys.stderr)
        return 3
    try:
        p = generate(kind, a.scale, a.seed)
    except Exception as e:  # invalid spec
        print(f"error: {e}", file=sys.stderr)
        return 3
    _write_atomic(a.out, write_qps(p))
    meta = {"class": a.cls, "scale": a.scale, "seed": a.seed, "n": p.num_vars(), "m_ineq": p.num_ineq(),
            "m_eq": p.num_eq(), "nnz_q": p.q.nnz(), "nnz_a": p.a_ineq.nnz() + p.a_eq.nnz(), "known_optimum": None}
    _write_atomic(os.path.splitext(a.out)[0] + ".json", json.dumps(meta, indent=1) + "\n")
    return 0


def cmd_sgm10(a) -> int:
    print(repr(sgm10(a.values, a.limit)))
    return 0


def main(argv: Optional[Sequence[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2311_07710_b200.cli", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve")
    s.add_argument("file")
    add_solver_flags(s)
    s.add_argument("--out")
    s.add_argument("--log")
    b = sub.add_parser("bench")
    b.add_argument("dir")
    add_solver_flags(b)
    b.add_argument("--out")
    g = sub.add_parser("generate")
    g.add_argument("cls")
    g.add_argument("scale", type=float)
    g.add_argument("seed", type=int)
    g.add_argument("out")
    m = sub.add_parser("sgm10")
    m.add_argument("values", type=float, nargs="+")
    m.add_argument("--limit", type=float)
    a = ap.parse_args(argv)
    return {"solve": cmd_solve, "bench": cmd_bench, "generate": cmd_generate, "sgm10": cmd_sgm10}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
