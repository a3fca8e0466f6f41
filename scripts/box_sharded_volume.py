"""C4 in its box form (bounds_from_rows: the 1e6 bound rows t >= 0 become
bounds) row-sharded with its feature rows replicated: the exchanges left per
iteration (RAPDHG_TRACE prints the halo entry counts), against the reference
form. python scripts/box_sharded_volume.py [parts]"""
import sys
sys.path.insert(0, ".")
import paper_2311_07710_b200 as rb  # noqa: E402

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = rb.generate(rb.Gen.SVM, 1.0, 4)
b = rb.bounds_from_rows(p)
for name, q, cfg in (("rows form", p, rb.SolverConfig(tol=1e-6)),
                     ("box form", b, rb.SolverConfig(tol=1e-6, box_projection=True))):
    one = rb.solve(q, cfg)
    r = rb.solve_sharded(q, cfg, parts, replicate_min_len=1000)
    print(f"{name}: m = {q.num_rows()}, {parts} shards: {r.status.name} {r.iterations} it "
          f"(one GPU {one.iterations}), objective rel diff "
          f"{abs(q.objective(r.point.x) - q.objective(one.point.x)) / abs(q.objective(one.point.x)):.1e}", flush=True)
