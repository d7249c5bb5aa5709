"""Top SASS instructions of an ncu report by warp-stall samples, with shared
memory excess wavefronts:  python tools/sass_hot.py rep.ncu-rep [N] [kernel-regex]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
S = h.index("Warp Stall Sampling (All Samples)")
X = h.index("L1 Wavefronts Shared Excessive")
data = [r for r in rows[2:] if len(r) > S and r[S] not in ("", "0")]
tot = sum(float(r[S]) for r in data)
ex = sum(float(r[X] or 0) for r in rows[2:] if len(r) > X)
print(f"total samples {tot:.0f}, shared excessive wavefronts {ex:.0f}")
for r in sorted(data, key=lambda r: -float(r[S]))[:top]:
    print(f"{float(r[S]) / tot:6.1%} {r[0]:>6s} {r[1][:70]:70s} xs={r[X]}")
