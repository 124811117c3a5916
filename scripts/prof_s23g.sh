#!/usr/bin/env bash
set -u
TAG=${1:-r2i}
OUT=gpurun_out
ARGS1="--config c5 --images 512 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS1 > $OUT/plain_s23_${TAG}.json 2>&1 && \
ncu --section SpeedOfLight --section SchedulerStats --section WarpStateStats --section ComputeWorkloadAnalysis \
    --section MemoryWorkloadAnalysis --section LaunchStats --section Occupancy --clock-control none -k regex:k_step23 -s 1 -c 1 \
    -o $OUT/prof_s23hw_${TAG} python bench.py $ARGS1 > $OUT/ncu_s23hw_${TAG}.log 2>&1
echo "ncu rc $?"
grep -E "ERROR|LaunchFailed" $OUT/ncu_s23hw_${TAG}.log | head -3
echo done
