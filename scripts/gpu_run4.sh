for e in 8 16; do for b in 256 512 1024 2048; do RAPDHG_EPL=$e RAPDHG_BLOCK_MIN=$b python scripts/sweep_sched.py LASSO 1.0 800; done; done > gpurun_out/sweep4.log 2>&1
cat gpurun_out/sweep4.log
RAPDHG_TRACE=1 RAPDHG_EPL=16 python scripts/e2e_breakdown.py 2>&1 | tail -28
