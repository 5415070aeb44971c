#!/bin/bash
# Bench line per BASELINE config (device + e2e), for DESIGN.md's status table.
OUT=${1:-gpurun_out/cfgs}
mkdir -p $OUT
for c in 1 2 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-index-leg > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-index-leg > $OUT/bench_c3.json 2> $OUT/bench_c3.err
