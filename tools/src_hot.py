"""Per-CUDA-source-line warp-stall breakdown of an ncu report (first file in
the source page):  python tools/src_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(io.StringIO(out)))
agg, src, cur = {}, {}, None
h = None
for r in rows:
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < len(h) - 5:
        continue
    if r[0]:
        cur = int(r[0])
        src[cur] = r[1]
        continue  # the line's own row repeats the sum of its SASS rows
    a = agg.setdefault(cur, {})
    for i, name in enumerate(h):
        if name.startswith("stall_") and "Not Issued" not in name:
            v = r[i]
            a[name] = a.get(name, 0.0) + (float(v) if v not in ("", "-") else 0.0)
tot = sum(sum(a.values()) for a in agg.values())
print(f"total samples {tot:.0f}")
for line, a in sorted(agg.items(), key=lambda t: -sum(t[1].values()))[:top]:
    s = sum(a.values())
    tops = sorted(a.items(), key=lambda t: -t[1])[:3]
    why = " ".join(f"{k[6:]}={v / s:.0%}" for k, v in tops)
    print(f"{s / tot:6.1%} L{line:<4d} {src[line].strip()[:70]:70s} {why}")
