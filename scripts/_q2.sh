#!/usr/bin/env bash
set -u
for E in 0.01 0.001 0.0001 0.00001; do
  timeout 300 python bench.py --config c3 --eps $E --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/eps_$E.json 2>&1
done
python scripts/summ.py gpurun_out/eps_*.json
python -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/eps_*.json')):
    d=json.load(open(f)); print(f, d['config']['H_plus'], d['kernel_ms'])
"
