export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -3
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"slab_kernel|slab_finish" -s 4 -c 4 -o gpurun_out/prof_r01_slab3 \
    python scripts/ncu_target.py 120 > gpurun_out/ncu_full49.log 2>&1
echo "ncu full rc=$?"
