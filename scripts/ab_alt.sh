#!/usr/bin/env bash
# Alternating A/B runs of two environment settings (ENV_A / ENV_B) at c5 shapes; per-kernel times and clocks.
set -u
A="--config c5 --images 2048 --templates 256 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  env $ENV_A timeout 300 python bench.py $A > gpurun_out/alt_A$i.json 2> gpurun_out/alt_A$i.err
  env $ENV_B timeout 300 python bench.py $A > gpurun_out/alt_B$i.json 2> gpurun_out/alt_B$i.err
done
python scripts/summ.py gpurun_out/alt_A*.json gpurun_out/alt_B*.json
grep -o '"sm_mhz": [0-9.]*' gpurun_out/alt_*.json
