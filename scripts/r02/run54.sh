# round 2 call 54: final validation at HEAD — GPU suite, smoke, bench (both arms), configs, ncu (C4 launch list + full)
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/r02_54_tests.log 2>&1; echo "tests rc=$?"; tail -9 gpurun_out/r02_54_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02_54_bench.json 2> gpurun_out/r02_54_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r02_54_bench.json')); r=d['roofline']
print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['e2e']['wall_s_each'], 'frac', round(r['frac'],3), 'inloop', r['inloop']['avg_step_ms'], 'iter', round(r['iteration']['frac_of_measured'],3), 'ttt', d['time_to_tol_s'], 'cpu', round(d['cpu_baseline']['value'],2), d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/r02_54_bench_ref.json 2> gpurun_out/r02_54_bench_ref.err; echo "ref rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r02_54_bench_ref.json')); print('ref value', d['value'], d['time_to_tol_s'], d['status'], d['iterations'])"
timeout 600 python scripts/gpu_configs.py > gpurun_out/r02_54_configs.jsonl 2> gpurun_out/r02_54_configs.err; cut -c1-260 gpurun_out/r02_54_configs.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 2000 --csv --log-file gpurun_out/r02_54_c4_launches.csv python scripts/ncu_target.py svm 160 > /dev/null 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"DualStepOp|PrimalStepOp" -s 4 -c 4 -o gpurun_out/r02_54_c4_full python scripts/ncu_target.py svm 40 > gpurun_out/r02_54_ncu_full.log 2>&1; echo "ncu full rc=$?"
