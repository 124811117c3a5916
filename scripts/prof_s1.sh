#!/usr/bin/env bash
# ncu --set full of one k_step1_tc launch at c5 shapes (2048 x 64 reduced job).  Usage: scripts/prof_s1.sh TAG
set -u
TAG=${1:-r2q}
OUT=gpurun_out
ARGS1="--config c5 --images 2048 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 120 python bench.py $ARGS1 > $OUT/plain_s1_${TAG}.json 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_step1_tc" -s 1 -c 1 -o $OUT/prof_s1_${TAG} python bench.py $ARGS1 > $OUT/ncu_s1_${TAG}.log 2>&1
echo "ncu rc $?"
