"""Per-stage breakdown of an ncu launch list (last pipeline step)."""
import csv
import sys

path = sys.argv[1]
first = sys.argv[2] if len(sys.argv) > 2 else "hashed_keygen"
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
idx = [i for i, d in enumerate(data) if first in d["Kernel Name"]]
last = data[idx[-1]:] if idx else data
tot = 0.0
for d in last:
    v = float(d["Metric Value"]) / 1000
    tot += v
    print(f"{v:9.1f} us  {d['Grid Size']:>16s}  {d['Kernel Name'][:80]}")
print(f"total {tot:.1f} us over {len(last)} launches")
