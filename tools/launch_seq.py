"""Print an ncu launch-list CSV (gpu__time_duration.sum) as a sequence and
per-kernel totals.  usage: python tools/launch_seq.py <csv> [--seq]"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
seq = []
for r in rows[1:]:
    name = re.sub(r"\(.*", "", re.sub(r"ftt::<unnamed>::", "", r[ki]))
    seq.append((name[:60], float(r[vi].replace(",", "")) / 1e3, r[gi], r[bi]))
if "--seq" in sys.argv:
    for n, us, g, b in seq:
        print(f"{us:8.1f} {g:>14} {b:>12} {n}")
agg = defaultdict(lambda: [0, 0.0])
for n, us, _, _ in seq:
    agg[n][0] += 1
    agg[n][1] += us
print(f"{len(seq)} launches, {sum(x[1] for x in seq):.1f} us")
for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{us:9.1f} us {c:4d} {n}")
