"""Summarise an ncu launch-list CSV (gpu__time_duration) by kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[h + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0][:90]
        tot[name] += float(r[vi].replace(",", "")) / 1e3; cnt[name] += 1
all_us = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    print(f"{v:10.1f} us {cnt[k]:6d}x  {k}")
print(f"total {all_us:.1f} us over {sum(cnt.values())} launches")
