"""Per-step kernel shares from an ncu launch list (--metrics gpu__time_duration.sum --csv)
of `bench.py`: our kernels only (namespace stg / dm), steps delimited by the ingestion's
first kernel. Usage: python tools/launch_summary.py launches.csv [steps_to_average]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
k, v = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[k], float(r[v])) for r in rows[hi + 1:] if len(r) > v]
ours = [(n, t) for n, t in ks if "stg::" in n or "dm::" in n]
starts = [i for i, (n, _) in enumerate(ours) if "edit_check_kernel" in n or "edit_bucket_kernel" in n]
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sel = starts[-nsteps:]
steps = [ours[a:b] for a, b in zip(sel, sel[1:] + [len(ours)])]
agg = collections.defaultdict(float)
cnt = collections.defaultdict(int)
for st in steps:
    for n, t in st:
        key = n.split("(")[0].replace("void ", "").replace("stg::", "")
        agg[key] += t / len(steps)
        cnt[key] += 1
tot = sum(agg.values())
print(f"steps averaged: {len(steps)}; our kernels per step: {sum(len(s) for s in steps) / len(steps):.0f}; "
      f"serialized device time per step (ncu, cold caches): {tot / 1e6:.3f} ms")
for n, t in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{t / 1e3:9.1f} us/step {100 * t / tot:5.1f}%  x{cnt[n] / len(steps):4.1f}  {n}")
