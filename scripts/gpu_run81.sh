# C5: column-block size sweep (per-phase times)
export PYTHONUNBUFFERED=1
for kb in 16384 24576 32768 49152 65536; do echo "== block $kb KB"; RAPDHG_L2BLOCK_KB=$kb timeout 600 python scripts/sweep_sched.py LARGE 1.0 120 2>&1 | grep "^{" | cut -c1-260; done
echo "== LARGE_LOCAL default"; timeout 600 python scripts/sweep_sched.py LARGE_LOCAL 1.0 120 2>&1 | grep "^{" | cut -c1-260
