"""Per CUDA source line of one file in a .ncu-rep: warp-stall samples split by reason, executed
instructions and excess shared-memory wavefronts.   python tools/ncu_stalls.py rep.ncu-rep file.cu [lo hi]"""
import csv, subprocess, sys, collections
path, fname = sys.argv[1], sys.argv[2]
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10 ** 9)
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, hdr, cur = None, None, None
agg = collections.defaultdict(collections.Counter)
src = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Name" or r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or cur_file != fname or len(r) < len(hdr):
        continue
    if r[0]:
        cur = int(r[0]); src[cur] = r[1][:80]
        continue
    if cur is None or not (lo <= cur <= hi):
        continue
    d = dict(zip(hdr[2:], r[2:]))
    def f(k):
        try: return float(d.get(k, 0) or 0)
        except ValueError: return 0.0
    a = agg[cur]
    a["samples"] += f("Warp Stall Sampling (All Samples)")
    a["inst"] += f("Instructions Executed")
    a["smem_excess"] += f("L1 Wavefronts Shared Excessive")
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            a[k[6:]] += f(k)
tot = sum(a["samples"] for a in agg.values()) or 1
for ln in sorted(agg):
    a = agg[ln]
    if a["samples"] < 0.002 * tot and a["smem_excess"] == 0:
        continue
    reasons = sorted(((v, k) for k, v in a.items() if k not in ("samples", "inst", "smem_excess") and v > 0), reverse=True)[:3]
    rs = " ".join(f"{k}:{v/max(a['samples'],1)*100:.0f}%" for v, k in reasons)
    print(f"{ln:5d} {a['samples']/tot*100:5.1f}% inst {a['inst']:9.0f} xs {a['smem_excess']:7.0f} {rs:40s} {src.get(ln,'')}")
