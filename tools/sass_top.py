"""Top SASS instructions by warp-stall samples in an ncu report (with --import-source):
python tools/sass_top.py rep.ncu-rep [N] [context]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = list(csv.reader(out.splitlines()))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[start]
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
data = [r for r in rows[start + 1:] if len(r) > si]
tot = sum(int(r[si]) for r in data if r[si].isdigit())
top = sorted([(int(r[si]), j) for j, r in enumerate(data) if r[si].isdigit()], reverse=True)[:top_n]
print("total samples", tot)
for s, j in top:
    print(f"{100 * s / tot:5.1f}%  #{j}  {data[j][src][:100]}")
    for k in range(max(0, j - ctx), j):
        print(f"          #{k}  {data[k][src][:100]}  [{data[k][si]}]")
