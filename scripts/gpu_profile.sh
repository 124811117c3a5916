#!/usr/bin/env bash
# Run under gpurun: plain bench (must exit 0) -> launch list -> one full ncu capture of the top kernels.
# Usage: scripts/gpu_profile.sh <config> <tag>
set -u
CFG=${1:-c3}
TAG=${2:-r1}
OUT=gpurun_out
mkdir -p $OUT
ARGS="--config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > $OUT/plain_${CFG}_${TAG}.json 2> $OUT/plain_${CFG}_${TAG}.err || { tail -20 $OUT/plain_${CFG}_${TAG}.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $OUT/launches_${CFG}_${TAG}.csv \
    python bench.py $ARGS > $OUT/ncu_launch_${CFG}_${TAG}.log 2>&1
for K in k_step3_tc k_step1_tc k_step2_tc; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o $OUT/prof_${K}_${CFG}_${TAG} python bench.py $ARGS > $OUT/ncu_full_${K}_${CFG}_${TAG}.log 2>&1
done
echo done
