#!/usr/bin/env bash
set -u
TAG=${1:-r2m}
OUT=gpurun_out
timeout 120 python scripts/s23_check.py > $OUT/s23_check_${TAG}.log 2>&1; echo "check rc $?"; cat $OUT/s23_check_${TAG}.log
ARGS="--config c5 --images 2048 --templates 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 120 python bench.py $ARGS > $OUT/ab_fused_${TAG}.json 2> $OUT/ab_fused_${TAG}.err || { echo "bench failed"; tail -5 $OUT/ab_fused_${TAG}.err; exit 1; }
python -c "
import json; d=json.load(open('$OUT/ab_fused_${TAG}.json')); print('fused', '%.3e'%d['value'], d['kernel_ms'], d['clocks'])"
FTK_DIAG=1 python -c "from paper_1905_12317_b200 import build as b; b.build(force=True)" > $OUT/diag_build.log 2>&1
for DBG in 0 2; do
  FTK_S23_DBG=$DBG FTK_S23_TRACE=1 timeout 120 python bench.py --config c5 --images 2048 --templates 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/trace_${TAG}_$DBG.json 2> $OUT/trace_${TAG}_$DBG.err
  grep s23trace $OUT/trace_${TAG}_$DBG.err | tail -2 | head -1
done
echo done
