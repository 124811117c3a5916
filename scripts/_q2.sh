#!/usr/bin/env bash
set -u
r() { N=$1; shift; timeout 300 python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/q2_$N.json 2>&1; }
r e3_ws24 --eps 0.001 --workspace-gb 24
r e3_ws19 --eps 0.001 --workspace-gb 19
r e3_ws12 --eps 0.001 --workspace-gb 12
r e4_ws24 --eps 0.0001 --workspace-gb 24
r e4_ws48 --eps 0.0001 --workspace-gb 48
r e4_ws12 --eps 0.0001 --workspace-gb 12
python -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/q2_*.json')):
    try:
        d=json.load(open(f)); print(f, d['config']['H_plus'], round(d['kernel_ms']['step1'],1), round(d['kernel_ms']['step2'],1))
    except Exception as e: print(f, 'ERR', open(f).read()[-300:])
"
