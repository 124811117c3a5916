#!/usr/bin/env bash
set -u
TAG=${1:-r2b}
OUT=gpurun_out
ARGS="--config c5 --images 2048 --templates 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > $OUT/ab_fused_${TAG}.json 2> $OUT/ab_fused_${TAG}.err || { tail -20 $OUT/ab_fused_${TAG}.err; exit 1; }
python -c "
import json; d=json.load(open('$OUT/ab_fused_${TAG}.json')); print('fused', '%.3e'%d['value'], d['kernel_ms'], d['clocks'])"
ARGS1="--config c5 --images 512 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS1 > $OUT/plain_s23_${TAG}.json 2>&1 && \
ncu --replay-mode application --section SpeedOfLight --section WarpStateStats --section SchedulerStats --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section SourceCounters --import-source on --clock-control none -k regex:k_step23 -s 1 -c 1 \
    -o $OUT/prof_s23_${TAG} python bench.py $ARGS1 > $OUT/ncu_s23_${TAG}.log 2>&1
echo "ncu rc $?"
FTK_DIAG=1 python -c "from paper_1905_12317_b200 import build as b; b.build(force=True)" > $OUT/diag_build.log 2>&1
FTK_S23_TRACE=1 python bench.py --config c5 --images 2048 --templates 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/trace_${TAG}.json 2> $OUT/trace_${TAG}.err
grep s23trace $OUT/trace_${TAG}.err | tail -4
echo done
