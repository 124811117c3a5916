#!/usr/bin/env bash
# ncu --set full of one launch of each named kernel at c5 per-pair shapes (reduced job).
# Usage: scripts/prof_k.sh TAG kernel [kernel...]
set -u
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
ARGS="--config c5 --images 1024 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > $OUT/plain_${TAG}.json 2> $OUT/plain_${TAG}.err || { tail -20 $OUT/plain_${TAG}.err; exit 1; }
for K in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 0 -c 1 \
      -o $OUT/prof_${K}_${TAG} python bench.py $ARGS > $OUT/ncu_${K}_${TAG}.log 2>&1
done
echo done
