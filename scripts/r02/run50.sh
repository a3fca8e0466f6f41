# round 2 call 50: flakiness check — the GPU suite three times back to back, plus smoke
export PYTHONUNBUFFERED=1
make -C paper_2311_07710_b200 -j8 > /dev/null 2>&1 || { echo build failed; exit 1; }
for i in 1 2 3; do
  timeout 1200 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02_50_tests_$i.log 2>&1; echo "run $i rc=$?"; tail -1 gpurun_out/r02_50_tests_$i.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
