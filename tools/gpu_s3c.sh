set -u
OUT=gpurun_out/s3c; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_conformance.py -q -x > $OUT/conf.log 2>&1; echo "rc=$?" >> $OUT/conf.log
timeout 300 python tools/e2e_split.py 5 5 > $OUT/e2e_split.log 2>&1
