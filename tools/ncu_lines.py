"""Aggregate warp-stall samples of a .ncu-rep by CUDA source line (cuda,sass page)."""
import csv, subprocess, sys, collections
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.Counter()
src = {}
fname = None
cur = None
idx = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        idx = r.index("Warp Stall Sampling (All Samples)")
        continue
    if idx is None or len(r) <= idx:
        continue
    if r[0]:  # a CUDA line row
        cur = (fname, r[0])
        src[cur] = r[1][:90]
    try:
        v = float(r[idx] or 0)
    except ValueError:
        continue
    if cur and not r[0]:
        agg[cur] += v
tot = sum(agg.values()) or 1
for k, v in agg.most_common(top):
    print(f"{100*v/tot:5.1f}% {k[0]}:{k[1]:>4} {src.get(k,'')}")
