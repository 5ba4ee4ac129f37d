"""Prints the last step's STG_KLOG timeline (start offset, duration, gap to
the previous end) from a profile_step.py log."""
import re
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith("klog")]
groups, cur = [], []
for l in lines:
    m = re.match(r"klog cls=(\d+) (.*?)\s+([\d.]+) us  @\s*([\d.]+) us", l)
    cls, tag, dur, off = int(m.group(1)), m.group(2).strip(), float(m.group(3)), float(m.group(4))
    if off == 0.0 and cur:
        groups.append(cur)
        cur = []
    cur.append((off, dur, cls, tag))
groups.append(cur)
end = 0.0
for off, dur, cls, tag in sorted(groups[-1]):
    print(f"{off:8.1f} {dur:8.1f} gap {off - end:7.1f}  cls{cls:2d} {tag}")
    end = max(end, off + dur)
print("span", end)
