set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench13.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench13.log | cut -c1-400
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench13_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file gpurun_out/launches_r01_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch13.log 2>&1
echo "launch list rc=$?"
python scripts/ncu_target.py 120 > gpurun_out/target_plain13.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"PrimalStepOp|DualStepOp|KktQAtyOp|KktAxOp" -s 12 -c 4 -o gpurun_out/prof_r01_final \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full13.log 2>&1
echo "ncu full rc=$?"
python bench.py --shard-emulate 4 --workload large --scale 0.1 --steps 2 --warmup 1 --max-iters 400 > gpurun_out/bench_shard_emu.log 2>&1; echo "shard emu rc=$?"; tail -1 gpurun_out/bench_shard_emu.log | cut -c1-300
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --shard --steps 2 --warmup 1 > gpurun_out/bench_shard_nccl1.log 2>&1; echo "shard nccl rc=$?"; tail -1 gpurun_out/bench_shard_nccl1.log | cut -c1-300
for k in RANDOM_QP:1.0 PORTFOLIO:1.0 SVM:1.0 LARGE:1.0; do python scripts/sweep_sched.py ${k%%:*} ${k##*:} 400; done > gpurun_out/sweep13.log 2>&1; cat gpurun_out/sweep13.log | cut -c1-250
