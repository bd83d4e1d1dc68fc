"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: launch_summary.py launches.csv [title]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
    tot[r[ki]] += v
    cnt[r[ki]] += 1
all_us = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:70]:70s} launches={cnt[k]:3d} mean={v / cnt[k]:9.3f} us  share={100 * v / all_us:5.1f}%")
