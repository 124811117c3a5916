#!/usr/bin/env bash
set -u
TAG=${1:-r2e}
OUT=gpurun_out
ARGS1="--config c5 --images 512 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS1 > $OUT/plain_s23_${TAG}.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $OUT/launches_${TAG}.csv python bench.py $ARGS1 > $OUT/ncu_launch_${TAG}.log 2>&1
echo "ncu launch rc $?"
FTK_DIAG=1 python -c "from paper_1905_12317_b200 import build as b; b.build(force=True)" > $OUT/diag_build.log 2>&1
FTK_S23_TRACE=1 python bench.py --config c5 --images 2048 --templates 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/trace_${TAG}.json 2> $OUT/trace_${TAG}.err
grep s23trace $OUT/trace_${TAG}.err | tail -2
echo done
