#!/usr/bin/env bash
set -u
TAG=${1:-r2o}
OUT=gpurun_out
FTK_DIAG=1 python -c "from paper_1905_12317_b200 import build as b; b.build(force=True)" > $OUT/diag_build.log 2>&1
for DBG in 0 8 16 24; do
  FTK_S23_DBG=$DBG FTK_S23_TRACE=1 timeout 120 python bench.py --config c5 --images 2048 --templates 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/trace_${TAG}_$DBG.json 2> $OUT/trace_${TAG}_$DBG.err
  echo "dbg $DBG"; grep s23trace $OUT/trace_${TAG}_$DBG.err | tail -2 | head -1
done
echo done
