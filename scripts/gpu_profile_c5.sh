#!/usr/bin/env bash
# ncu evidence at c5 per-pair shapes on a reduced job (2048 images x 128 templates), one launch per kernel.
set -u
TAG=${1:-r1}
OUT=gpurun_out
ARGS="--config c5 --images 2048 --templates 128 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > $OUT/plain_c5s_${TAG}.json 2> $OUT/plain_c5s_${TAG}.err || { tail -20 $OUT/plain_c5s_${TAG}.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $OUT/launches_c5s_${TAG}.csv \
    python bench.py $ARGS > $OUT/ncu_launch_c5s_${TAG}.log 2>&1
for K in ${KERNELS:-k_step3_tc k_step1_tc k_step2_tc}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o $OUT/prof_${K}_c5s_${TAG} python bench.py $ARGS > $OUT/ncu_full_${K}_c5s_${TAG}.log 2>&1
done
echo done
