"""Top stall-sampled SASS instructions of a .ncu-rep (with preceding context)."""
import csv, subprocess, sys
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
i = hdr.index('Warp Stall Sampling (All Samples)')
data = []
for k, r in enumerate(rows[2:]):
    try: data.append((float(r[i] or 0), k, r[1][:70]))
    except Exception: pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for d in sorted(data, reverse=True)[:top]:
    k = d[1]
    ctx = ' | '.join(rows[2 + j][1][:34] for j in range(max(0, k - 2), k))
    print(f'{100*d[0]/tot:5.1f}% #{k:5d} {d[2]:70s} <- {ctx}')
