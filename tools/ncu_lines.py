"""Per-CUDA-source-line instructions and warp-stall samples from
`ncu -i rep --page source --csv --print-source cuda,sass`.

usage: ncu -i r.ncu-rep --page source --csv --print-source cuda,sass -k K --launch-count 1 > s.csv
       python tools/ncu_lines.py s.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = [r for r in rows if "Instructions Executed" in r][0]
ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg = collections.defaultdict(lambda: [0.0, 0.0])
fname, cur = "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]), r[1].strip()[:90])
        try:
            agg[cur][0] += float(r[si])
            agg[cur][1] += float(r[ii])
        except ValueError:
            pass
tot = sum(v[1] for v in agg.values())
stot = sum(v[0] for v in agg.values()) or 1
print(f"total warp instructions {tot:.0f}, stall samples {stot:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / stot:5.1f}% {v[1]:10.0f}  {k[0]}:{k[1]}  {k[2]}")
