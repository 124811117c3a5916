#!/usr/bin/env bash
# Quick benches without tests.  Usage: scripts/quick.sh TAG [configs...]  (c5s = reduced c5)
set -u
TAG=$1; shift
mkdir -p gpurun_out
for C in "$@"; do
  if [ "$C" = c5s ]; then A="--config c5 --images 2048 --templates 256"; else A="--config $C"; fi
  timeout 300 python bench.py $A --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_$C.json 2> gpurun_out/${TAG}_$C.err; echo $C rc=$?
done
python scripts/summ.py gpurun_out/${TAG}_*.json
