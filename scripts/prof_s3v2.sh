#!/usr/bin/env bash
# A/B of the CTA-pair Step-3 kernel (FTK_S3V2=1) against k_step3_tc at c5 shapes, after scripts/s23_check.py.  Usage: scripts/prof_s3v2.sh TAG
set -u
TAG=${1:-r2r}
OUT=gpurun_out
timeout 150 python scripts/s23_check.py > $OUT/s23_check_${TAG}.log 2>&1; echo "check rc $?"; cat $OUT/s23_check_${TAG}.log
ARGS="--config c5 --images 2048 --templates 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for V in 0 1; do
  FTK_S3V2=$V timeout 150 python bench.py $ARGS > $OUT/ab_s3v2_${V}_${TAG}.json 2> $OUT/ab_s3v2_${V}_${TAG}.err || { echo "bench failed"; tail -5 $OUT/ab_s3v2_${V}_${TAG}.err; }
  python -c "
import json; d=json.load(open('$OUT/ab_s3v2_${V}_${TAG}.json')); print('S3V2=$V', '%.3e'%d['value'], {k: round(v,2) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
echo done
