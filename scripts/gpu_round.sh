#!/usr/bin/env bash
# One GPU round-trip: parity tests, then quick benches.  Usage: scripts/gpu_round.sh TAG [configs...]
set -u
TAG=${1:-x}; shift
CFGS=${@:-c3 c4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -15 gpurun_out/${TAG}_pytest.log
for C in $CFGS; do timeout 300 python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_$C.json 2> gpurun_out/${TAG}_$C.err; echo $C rc=$?; done
timeout 400 python bench.py --config c5 --images 2048 --templates 256 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c5s.json 2> gpurun_out/${TAG}_c5s.err; echo c5s rc=$?
python scripts/summ.py gpurun_out/${TAG}_*.json
