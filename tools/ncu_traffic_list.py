"""Per-launch time / DRAM bytes from an `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv` log.
usage: python tools/ncu_traffic_list.py <csv> [min_us]"""
import csv
import re
import sys
from collections import OrderedDict

U = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
     "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
idi, gi = hdr.index("ID"), hdr.index("Grid Size")
L = OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[idi], {"name": re.sub(r"\(.*", "", re.sub(r"ftt::<unnamed>::", "", r[ki]))[:45],
                              "grid": r[gi]})
    d[r[mi]] = float(r[vi].replace(",", "")) * U.get(r[ui], 1)
lim = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
tot = 0.0
for d in L.values():
    t = d.get("gpu__time_duration.sum", 0.0)
    tot += t
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    if t >= lim:
        print(f"{t:9.1f}us {b / 1e6:9.1f}MB {b / t / 1e3 if t else 0:7.0f}GB/s {d['grid']:>14} {d['name']}")
print(f"total {tot:.1f} us, {len(L)} launches")
