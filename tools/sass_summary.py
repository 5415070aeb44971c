"""Instruction-class counts of the hot kernels' SASS (static, per kernel),
from `cuobjdump -sass` of the built library: evidence of which hardware
paths a kernel uses (DMMA = fp64 tensor pipe, UBLKCP = TMA bulk copy,
LDGSTS = cp.async, ATOMS = shared atomics, MATCH = warp match.any, ...).

usage: python tools/sass_summary.py [lib.so] > profiles/r02/sass_summary.md
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1908_02721_b200/libfasttt_b200.so"
HOT = ["k_onesweep_tma", "k_onesweep", "k_sel_count", "k_keys_hist_lin", "k_hist_hashmod",
       "k_emit", "k_sweep_mark", "k_dgemm", "k_jacobi_persistent", "k_tsqr_level",
       "k_jacobi_qr", "k_sp_on_dd", "k_gram_dd", "k_spmm_seg", "k_spmm_rows", "k_inner_struct"]
CLASSES = ["DMMA", "DFMA", "DADD", "DMUL", "UBLKCP", "UTMALDG", "SYNCS", "LDGSTS", "LDG", "STG",
           "LDS", "STS", "ATOMS", "ATOMG", "RED", "SHFL", "MATCH", "BAR", "MUFU"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
    if m:
        funcs[cur][m.group(1)] += 1


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


names = list(funcs)
pretty = dict(zip(names, demangle(names)))
print("| kernel | instrs | " + " | ".join(CLASSES) + " |")
print("|---|---:|" + "---:|" * len(CLASSES))
for h in HOT:
    for n in names:
        p = pretty[n].replace("(anonymous namespace)::", "").replace("ftt::", "")
        short = re.sub(r"^void ", "", re.sub(r"\(.*", "", p)).split("::")[-1]
        if not short.startswith(h + "<") and short != h:
            continue
        c = funcs[n]
        tot = sum(c.values())
        row = [str(sum(v for k, v in c.items() if k == cls or k.startswith(cls)))
               for cls in CLASSES]
        tmpl = re.search(r"<(.*)>", short)
        label = h + (f"<{tmpl.group(1)[:40]}>" if tmpl else "")
        print(f"| `{label}` | {tot} | " + " | ".join(row) + " |")
