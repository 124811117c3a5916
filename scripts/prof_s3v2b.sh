#!/usr/bin/env bash
set -u
TAG=${1:-r2s}
OUT=gpurun_out
FTK_DIAG=1 python -c "from paper_1905_12317_b200 import build as b; b.build(force=True)" > $OUT/diag_build.log 2>&1
ARGS="--config c5 --images 2048 --templates 128 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for DBG in 0 8 2; do
  FTK_S23_DBG=$DBG timeout 150 python bench.py $ARGS > $OUT/s3v2dbg_${DBG}_${TAG}.json 2> $OUT/s3v2dbg_${DBG}_${TAG}.err || { echo "bench failed"; tail -3 $OUT/s3v2dbg_${DBG}_${TAG}.err; }
  python -c "
import json; d=json.load(open('$OUT/s3v2dbg_${DBG}_${TAG}.json')); print('dbg $DBG', {k: round(v,2) for k,v in d['kernel_ms'].items()})"
done
FTK_S23_TRACE=1 timeout 150 python bench.py --config c5 --images 2048 --templates 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/trace_s3v2_${TAG}.json 2> $OUT/trace_s3v2_${TAG}.err
grep s23trace $OUT/trace_s3v2_${TAG}.err | tail -2
echo done
