#!/bin/bash
# One build->measure iteration on the GPU box (run from the repo root):
#   bash tools/gpu_iter.sh <tag> [configs]   -> gpurun_out/<tag>/
# GPU parity tests, the default bench line, per-config bench lines and the
# ncu launch list of one warm config-2 decomposition.
set -u
TAG=${1:-it}
CFGS=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
python tools/profile_step.py 2 > $OUT/ps2.log 2>&1 &&
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launch_c2.csv python tools/profile_step.py 2 > $OUT/ncu2.log 2>&1
tail -2 $OUT/pytest_gpu.log
python - "$OUT" <<'PY'
import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/bench*.json")):
    try:
        d = json.load(open(f))
        print(f, round(d["ms_per_step"], 3), "e2e", d.get("e2e") and round(d["e2e"]["ms_per_step"], 3),
              d.get("stages_ms"))
    except Exception as e:
        print(f, "unreadable", e)
PY
