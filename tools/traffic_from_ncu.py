"""Per-kernel-class DRAM traffic from an ncu metrics capture.

usage: python tools/traffic_from_ncu.py traffic_c5.csv [--json out.json] [--md out.md]

Input: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` of one warm decomposition (tools/profile_step.py).
Output: per class (the ftt_profile tags bench.py reports) the launches, the
summed DRAM bytes and the bytes per launch, which bench.py quotes as
roofline.traffic next to its algorithmic bytes per launch.
"""
import collections
import csv
import json
import sys

CLASSES = [
    ("sort", ("k_onesweep", "k_part_scatter")),
    ("hist", ("k_keys_hist", "k_hist", "k_distinct_hash", "k_linearize")),
    ("segment", ("k_compact", "k_count", "k_emit", "k_scan_counts", "k_count_changes", "k_distinct_",
                 "k_part_count", "k_sel_count", "k_group_count")),
    ("sweep", ("k_sweep",)),
    ("scatter", ("k_pivot_scatter", "k_side_core", "k_scatter_", "k_sp_entries", "k_sp_gather",
                 "k_sc_pos", "k_sc_iptr", "k_pack_cores",
                 "k_gather_i32", "k_sp_bitmap", "k_lower_bounds", "k_scan_blocks", "k_scan_fix",
                 "k_seg_counts")),
    ("gemm", ("k_dgemm", "k_splitk_reduce", "k_sum_partials", "k_spmm_", "k_sp_resid", "k_sc_",
              "k_seg_reduce", "k_sp_sum", "k_resid_", "k_gram_", "k_sp_on_dd")),
    ("qr_panel", ("k_panel", "k_larft", "k_extract_v")),
    ("jacobi", ("k_jacobi", "k_svd_small", "k_svd_wy", "k_tsqr", "k_qr_root", "k_chol")),
    ("entries", ("k_entries", "k_mitm", "k_half_", "k_seg_", "k_left_vec", "k_right_vec",
                 "k_inner_struct", "k_sum_fixed")),
]

UNIT = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
        "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def classify(name):
    for ns in ("<unnamed>::", "unnamed>::", "(anonymous namespace)::", "ftt::"):
        name = name.replace(ns, "")
    short = name.split("(")[0].split("::")[-1]
    short = short.replace("void ", "").split("<")[0].strip()
    for cls, prefixes in CLASSES:
        if any(short.startswith(p) for p in prefixes):
            return cls, short
    return "other", short


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        rec = launches.setdefault(key, {"name": d["Kernel Name"]})
        v = float(d["Metric Value"].replace(",", ""))
        rec[d["Metric Name"]] = v * UNIT.get(d["Metric Unit"].strip().lower(), 1.0)
    return list(launches.values())


def main():
    path = sys.argv[1]
    out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    out_md = sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None
    # --total KEY: also record the capture's summed DRAM bytes under KEY
    # (e.g. index_path: one select_p + fibers + sweeps pass, for bench.py's
    # index leg); --merge: update an existing json instead of replacing it
    total_key = sys.argv[sys.argv.index("--total") + 1] if "--total" in sys.argv else None
    agg = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    kern = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    for rec in load(path):
        cls, short = classify(rec["name"])
        by = rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0)
        for tgt in (agg[cls], kern[(cls, short)]):
            tgt["launches"] += 1
            tgt["us"] += rec.get("gpu__time_duration.sum", 0.0)
            tgt["dram_bytes"] += by
    tot_us = sum(v["us"] for v in agg.values()) or 1.0
    lines = ["| class | kernel | launches | total us | share | DRAM MB | DRAM GB/s |",
             "|---|---|---:|---:|---:|---:|---:|"]
    for (cls, short), v in sorted(kern.items(), key=lambda kv: -kv[1]["us"]):
        gbs = v["dram_bytes"] / (v["us"] * 1e-6) / 1e9 if v["us"] else 0.0
        lines.append(f"| {cls} | `{short}` | {v['launches']} | {v['us']:.1f} | "
                     f"{100 * v['us'] / tot_us:.1f}% | {v['dram_bytes'] / 1e6:.1f} | {gbs:.0f} |")
    text = "\n".join(lines)
    print(text)
    res = {}
    for cls, v in agg.items():
        if v["launches"]:
            res[cls] = v["dram_bytes"] / v["launches"]
    ss = [agg[c] for c in ("sort", "hist", "segment") if agg[c]["launches"]]
    if ss:
        res["sort+hist+segment"] = sum(v["dram_bytes"] for v in ss) / sum(v["launches"] for v in ss)
    if total_key:
        res = {total_key: sum(v["dram_bytes"] for v in agg.values()),
               total_key + "_us": tot_us}
    if out_json:
        old = {}
        if "--merge" in sys.argv:
            try:
                old = json.load(open(out_json))
            except Exception:  # noqa: BLE001
                old = {}
        old.update({k: round(v, 1) for k, v in res.items()})
        with open(out_json, "w") as fh:
            json.dump(old, fh, indent=1)
    if out_md:
        with open(out_md, "w") as fh:
            fh.write(text + "\n")


if __name__ == "__main__":
    main()
