#!/usr/bin/env bash
# ncu --set full of one k_step3_tc launch at c5 per-pair shapes (reduced job).  Usage: scripts/prof_s3.sh TAG [kernel-regex]
set -u
TAG=${1:-x}
K=${2:-k_step3_tc}
OUT=gpurun_out
mkdir -p $OUT
ARGS="--config c5 --images 1024 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > $OUT/plain_s3_${TAG}.json 2> $OUT/plain_s3_${TAG}.err || { tail -20 $OUT/plain_s3_${TAG}.err; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o $OUT/prof_${K}_${TAG} python bench.py $ARGS > $OUT/ncu_${K}_${TAG}.log 2>&1
echo done
