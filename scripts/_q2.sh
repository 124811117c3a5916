#!/usr/bin/env bash
set -u
cp scripts/_ab/diag.so paper_1905_12317_b200/libftk.so
for E in 0.001 0.0001; do
  echo "== eps $E"
  FTK_S1_TRACE=1 timeout 300 python bench.py --config c3 --eps $E --images 1024 --templates 128 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -i "s1trace" | tail -3
done
