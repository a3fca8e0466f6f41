"""Top SASS lines by warp-stall samples for kernel #k of an ncu report (with
the 14 preceding instructions of the top few)."""
import csv, subprocess, sys
rep, k = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kk, seq = 0, []
for r in rows:
    if r and r[0] == "Kernel Name":
        kk += 1
        if kk == k: print(r[1][:100])
        continue
    if kk == k and len(r) > 3 and r[0].startswith("0x"):
        try: seq.append((r[0][-5:], r[1].strip()[:90], int(r[2])))
        except ValueError: pass
T = sum(n for _, _, n in seq)
print("total samples", T)
top = sorted(range(len(seq)), key=lambda i: -seq[i][2])[:14]
for i in top: print(seq[i][2], seq[i][0], seq[i][1])
for i in top[:3]:
    print("--- context of", seq[i][0])
    for a, s, n in seq[max(0, i - 12):i + 2]: print("  ", a, n, s)
