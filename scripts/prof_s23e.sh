#!/usr/bin/env bash
set -u
TAG=${1:-r2f}
OUT=gpurun_out
FTK_DIAG=1 python -c "from paper_1905_12317_b200 import build as b; b.build(force=True)" > $OUT/diag_build.log 2>&1
FTK_S23_TRACE=1 python bench.py --config c5 --images 2048 --templates 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/trace_${TAG}.json 2> $OUT/trace_${TAG}.err
grep s23trace $OUT/trace_${TAG}.err | tail -2
echo done
