#!/usr/bin/env bash
# usage: /tmp/run_bench.sh tag configs...
TAG=$1; shift
for C in "$@"; do
  python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_${C}_${TAG}.json 2> gpurun_out/b_${C}_${TAG}.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/b_${C}_${TAG}.json")); print("$C", "%.3e"%d["value"], round(d["ms_per_step"],1), {k: round(v,1) for k,v in d["kernel_ms"].items()}, "frac", round(d["roofline"]["frac"],3), d["clocks"]["reasons"])
except Exception as e:
    print("$C FAILED", e); print(open("gpurun_out/b_${C}_${TAG}.err").read()[-600:])
PY
done
