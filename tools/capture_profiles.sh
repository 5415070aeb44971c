#!/bin/bash
# Profiling session for one round (run on the GPU box from the repo root):
#   bash tools/capture_profiles.sh r01
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
TAG=${1:-r01}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
NCU="ncu --clock-control none"

# 1. the bench line itself (default = config 2, plus the config-5 index leg)
#    and the reference arm
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err

# 2. launch list of the bench command (per-launch times, cold-cache, serialised)
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-index-leg > $OUT/bench_small.json 2>&1 &&
  $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-index-leg > $OUT/ncu_bench.log 2>&1

# 3. per-launch DRAM traffic of one warm decomposition per config
#    (ncu cannot replay the cooperative launch of clustered Jacobi pairs, so
#    these captures run the Jacobi with one CTA per pair: FTT_JCLUSTER=1)
export FTT_JCLUSTER=1
for c in 2 5 1 4; do
  python tools/profile_step.py $c > $OUT/step_c$c.log 2>&1 &&
    $NCU --profile-from-start off \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --csv --log-file $OUT/traffic_c$c.csv python tools/profile_step.py $c > $OUT/ncu_traffic_c$c.log 2>&1
done

# 4. full captures of the top kernels (source-mapped)
python tools/profile_step.py 5 > /dev/null 2>&1 &&
  $NCU --profile-from-start off --set full --import-source on \
    -k regex:"k_onesweep|k_keys_hist|k_part_scatter|k_part_count" -c 4 -o $OUT/full_c5_sort -f \
    python tools/profile_step.py 5 > $OUT/ncu_full_c5_sort.log 2>&1
python tools/profile_step.py 5 > /dev/null 2>&1 &&
  $NCU --profile-from-start off --set full --import-source on \
    -k regex:"k_sp_resid_off|k_spmm_seg|k_spmm_rows" -c 3 -o $OUT/full_c5_sparse -f \
    python tools/profile_step.py 5 > $OUT/ncu_full_c5_sparse.log 2>&1
python tools/profile_step.py 2 > /dev/null 2>&1 &&
  $NCU --profile-from-start off --set full --import-source on \
    -k regex:"k_tsqr_level|k_dgemm|k_jacobi_small|k_chol_inv" -c 8 -o $OUT/full_c2 -f \
    python tools/profile_step.py 2 > $OUT/ncu_full_c2.log 2>&1
for f in $OUT/*.ncu-rep; do
  [ -f "$f" ] || continue
  ncu -i "$f" --page details > "${f%.ncu-rep}.details.txt" 2>&1
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}.raw.csv" 2>&1
done
ls -la $OUT
