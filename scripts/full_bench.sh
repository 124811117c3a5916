#!/usr/bin/env bash
# Full default bench (c5, N=1) -> gpurun_out/${TAG}_bench.json, then the ncu launch list of a reduced
# run.  Usage: scripts/full_bench.sh TAG
set -u
TAG=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
python scripts/summ.py gpurun_out/${TAG}_bench.json
A="--config c5 --images 2048 --templates 256 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
python bench.py $A > gpurun_out/${TAG}_plain_launch.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py $A > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo ncu rc=$?
