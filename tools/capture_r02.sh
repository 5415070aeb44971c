#!/bin/bash
# Round-2 profiling session (run on the GPU box from the repo root):
#   bash tools/capture_r02.sh
# Every ncu command runs only after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/prof_r02
mkdir -p $OUT/configs
NCU="ncu --clock-control none"

# 1. the bench line (config 5) and the reference arm, then configs 1-4
python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err
for c in 1 2 4; do
  python bench.py --config $c --no-index-leg > $OUT/configs/bench_c$c.json 2> $OUT/configs/bench_c$c.err
done
python bench.py --config 3 --steps 3 --warmup 3 --no-index-leg > $OUT/configs/bench_c3.json 2> $OUT/configs/bench_c3.err

# 2. launch list of the bench command (cold, serialised per-launch times)
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-index-leg > $OUT/bench_small.json 2>&1 &&
  $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_bench_c5.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-index-leg > $OUT/ncu_bench.log 2>&1

# 3. per-launch time + DRAM bytes: one warm decomposition per config, and the
#    config-5 index pass alone (FTT_JCLUSTER=1: ncu cannot replay clustered
#    cooperative Jacobi launches)
export FTT_JCLUSTER=1
for c in 5 2 4; do
  python tools/profile_step.py $c > $OUT/step_c$c.log 2>&1 &&
    $NCU --profile-from-start off \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --csv --log-file $OUT/traffic_c$c.csv python tools/profile_step.py $c > $OUT/ncu_traffic_c$c.log 2>&1
done
python tools/profile_index.py 5 > $OUT/index_c5.log 2>&1 &&
  $NCU --profile-from-start off \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --csv --log-file $OUT/traffic_index_c5.csv python tools/profile_index.py 5 > $OUT/ncu_index_c5.log 2>&1
unset FTT_JCLUSTER

# 4. full captures of the top kernels (source-mapped)
python tools/profile_index.py 5 > /dev/null 2>&1 &&
  $NCU --profile-from-start off --set full --import-source on \
    -k regex:"k_sel_count|k_onesweep|k_keys_hist_lin|k_compact1|k_sweep_gather_mark|k_hist_hashmod" -c 10 -o $OUT/full_c5_index -f \
    python tools/profile_index.py 5 > $OUT/ncu_full_c5_index.log 2>&1
python tools/profile_step.py 5 > /dev/null 2>&1 &&
  $NCU --profile-from-start off --set full --import-source on \
    -k regex:"k_tsqr_wy|k_svd_wy|k_sp_on_dd|k_spmm_seg|k_spmm_rows|k_dgemm|k_sc_w|k_sc_ysum|k_sc_qta|k_sc_resid|k_resid_cols" -c 14 -o $OUT/full_c5_round -f \
    python tools/profile_step.py 5 > $OUT/ncu_full_c5_round.log 2>&1
for f in $OUT/*.ncu-rep; do
  [ -f "$f" ] || continue
  ncu -i "$f" --page details > "${f%.ncu-rep}.details.txt" 2>&1
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}.raw.csv" 2>&1
done
ls -la $OUT
