#!/bin/bash
# Per-kernel durations of the device eigensolver (ncu launch list over tools/eig_bench.py).
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/eig_bench.py 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
k, v, g = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
for r in rows[hi + 1:]:
    if len(r) > v: print(f'{r[k][:24]:26s} {r[g]:12s} {float(r[v]) / 1e3:9.1f} us')
"
