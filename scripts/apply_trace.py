"""Parse apply_mma_kernel phase stamps (NUGPR_APPLY_DBG=16 printf lines 'T cta sm k t')."""
import sys, collections
rows = collections.defaultdict(dict)
sms = {}
for ln in open(sys.argv[1]):
    p = ln.split()
    if len(p) == 5 and p[0] == "T":
        c, sm, k, t = int(p[1]), int(p[2]), int(p[3]), int(p[4])
        rows[c][k] = t; sms[c] = sm
# keep the last launch only: group by launch via start time clusters
starts = sorted(r[0] for r in rows.values())
t0 = min(starts)
tend = max(max(r.values()) for r in rows.values())
print(f"ctas {len(rows)} span {(tend - t0)/1e3:.1f} us; start spread {(max(starts)-t0)/1e3:.1f} us")
conv, comp, epi = [], [], []
for c, r in rows.items():
    ks = sorted(r)
    for q in range((len(ks) - 1) // 3):
        a, b, cc, d = r[3*q], r[3*q+1], r[3*q+2], r[3*q+3]
        conv.append(b - a); comp.append(cc - b); epi.append(d - cc)
import statistics as S
for name, v in (("convert", conv), ("stream+mma", comp), ("epilogue", epi)):
    print(f"{name:11s} mean {S.mean(v)/1e3:6.2f} us  max {max(v)/1e3:6.2f} us  n={len(v)}")
ends = sorted(max(r.values()) - t0 for r in rows.values())
print("CTA end times (us) p10/p50/p90/max:", [round(ends[int(f*(len(ends)-1))]/1e3, 1) for f in (0.1, 0.5, 0.9, 1.0)])
