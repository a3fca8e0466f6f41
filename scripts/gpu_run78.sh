# round-end refresh: ncu full of the slab kernels, bench, launch list, reference arm, smoke, tests
export PYTHONUNBUFFERED=1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel|slab_finish" -s 4 -c 4 -o gpurun_out/prof_r01_slab5 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full78.log 2>&1
echo "ncu full rc=$?"
python bench.py --steps 5 --warmup 3 > gpurun_out/bench78.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench78.log | cut -c1-600
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench78_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file gpurun_out/launches78.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch78.log 2>&1
echo "launch list rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench78_ref.log 2>&1; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
