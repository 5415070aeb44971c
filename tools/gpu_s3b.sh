set -u
OUT=gpurun_out/s3b; mkdir -p $OUT
export FTT_JCLUSTER=1
python tools/profile_step.py 5 > $OUT/step_c5.log 2>&1 &&
  ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --csv --log-file $OUT/traffic_c5.csv python tools/profile_step.py 5 > $OUT/ncu_c5.log 2>&1
unset FTT_JCLUSTER
timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --no-index-leg --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
