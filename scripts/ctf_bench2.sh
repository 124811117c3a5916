#!/usr/bin/env bash
set -u
TAG=${1:-ctfw}
mkdir -p gpurun_out
run() { N=$1; shift; timeout 600 python bench.py "$@" --steps 2 --warmup 3 > gpurun_out/${TAG}_$N.json 2> gpurun_out/${TAG}_$N.err; echo $N rc=$?; }
run c3_ctf4 --config c3 --ctf-defoci 8000,15000,22000,30000
run c3_ctf4_simt --config c3 --ctf-defoci 8000,15000,22000,30000 --engine simt --images 256 --templates 256
run c3_ctf4_tc_s --config c3 --ctf-defoci 8000,15000,22000,30000 --images 256 --templates 256
run c5_ctf2 --config c5 --ctf-defoci 10000,20000 --images 2048 --templates 256
python scripts/summ.py gpurun_out/${TAG}_*.json
