#!/bin/bash
# A/B of library builds on the GPU box (run from the repo root):
#   bash tools/ab_libs.sh <tag> "<configs>" lib1.so lib2.so ...  -> gpurun_out/<tag>/
# Each library (FTT_LIB) runs the bench line of each config, no CPU legs.
set -u
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
for lib in "$@"; do
  name=$(basename $lib .so)
  for c in $CFGS; do
    st=10; [ "$c" = 3 ] && st=2
    FTT_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline \
      > $OUT/${name}_c$c.json 2> $OUT/${name}_c$c.err
  done
done
python - "$OUT" <<'PY'
import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/*.json")):
    try:
        d = json.load(open(f))
        print(f, round(d["ms_per_step"], 3), "e2e", d.get("e2e") and d["e2e"].get("ms_per_step"),
              d.get("result", {}).get("ranks"))
    except Exception as e:
        print(f, "unreadable", e)
PY
