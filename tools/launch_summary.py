"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list."""
import csv, sys
from collections import defaultdict

path, cmd = sys.argv[1], " ".join(sys.argv[2:])
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    k = r[ki].split("(")[0]
    tot[k] += float(r[vi].replace(",", ""))
    cnt[k] += 1
unit = rows[1][hdr.index("Metric Unit")] if "Metric Unit" in hdr else "?"
s = sum(tot.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)")
print(f"command: {cmd}")
print("note: covers the whole bench process (setup, refill and untimed drain included), "
      "not only the timed steps")
print(f"{'kernel':40s} {'launches':>9s} {'total_' + unit:>14s}   share")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} {cnt[k]:9d} {tot[k]:14.1f} {100 * tot[k] / s:6.1f}%")
