# A/B: windows in device memory (working tree) vs the previous commit's slab files
export PYTHONUNBUFFERED=1
rm -rf /tmp/ab && mkdir -p /tmp/ab && cp -r paper_2311_07710_b200 /tmp/ab/pkg && cp -r include /tmp/ab/include && cp ab_old/* /tmp/ab/pkg/csrc/
make -s -C /tmp/ab/pkg OBJDIR=/tmp/ab/obj LIBOUT=/tmp/ab/lib_old.so -j8 > /tmp/ab/build.log 2>&1 || tail /tmp/ab/build.log
for r in 1 2 3; do
echo "== new"; timeout 300 python scripts/check_cost.py 2>&1 | head -2
echo "== old"; RAPDHG_LIB=/tmp/ab/lib_old.so timeout 300 python scripts/check_cost.py 2>&1 | head -2
done
