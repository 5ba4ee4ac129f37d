"""Per-kernel times of the last step in STG_KLOG outputs, side by side: python tools/klog_summary.py a.txt b.txt ..."""
import re
import sys


def last_step(path):
    rows, cur = [], []
    for line in open(path):
        if line.startswith("klog"):
            m = re.match(r"klog cls=\s*(\d+)\s+(.*?)\s+([\d.]+) us  @", line)
            if m:
                cur.append((int(m.group(1)), re.sub(r"\d{4,}", "N", m.group(2).strip()), float(m.group(3))))
        elif line.startswith("step"):
            rows, cur = cur, []
    return rows


cols = [last_step(p) for p in sys.argv[1:]]
n = min(len(c) for c in cols)
tot = [0.0] * len(cols)
for i in range(n):
    tag = cols[0][i][1]
    if tag.startswith("eig D") or not tag:
        continue
    vals = [c[i][2] for c in cols]
    if cols[0][i][0] in (0, 1, 13, 14):
        for j, v in enumerate(vals):
            tot[j] += v
    print(f"{cols[0][i][0]:3d} {tag:34s} " + " ".join(f"{v:9.1f}" for v in vals))
print("DMMA classes total (us): " + " ".join(f"{v:9.1f}" for v in tot))
