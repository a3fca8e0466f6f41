export PYTHONUNBUFFERED=1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench62.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench62.log | cut -c1-3000
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench62_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file gpurun_out/launches62.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch62.log 2>&1
echo "launch list rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench62_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench62_ref.log | cut -c1-600
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
