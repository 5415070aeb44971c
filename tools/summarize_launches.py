"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, total time and share (cold-cache, serialised times:
compare shares, not absolutes).

usage: python tools/summarize_launches.py launches.csv [top_n]
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append(d)
    return out


def to_us(value, unit):
    v = float(value.replace(",", ""))
    unit = unit.strip().lower()
    if unit in ("ns", "nsecond"):
        return v / 1e3
    if unit in ("ms", "msecond"):
        return v * 1e3
    if unit in ("s", "second"):
        return v * 1e6
    return v


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    data = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("ftt::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += to_us(d["Metric Value"], d["Metric Unit"])
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | avg us | share |")
    print("|---|---:|---:|---:|---:|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| `{k}` | {n} | {us:.1f} | {us / n:.1f} | {100 * us / tot:.1f}% |")
    print(f"\n{len(data)} launches, {tot:.1f} us total (serialised under ncu)")


if __name__ == "__main__":
    main()
