#!/usr/bin/env bash
# CTF-parameterized kernel benches (NEXT-4): c3 x 2 defoci, c2 x 4 defoci, c5 x 1 defocus, plus the plain
# configs for comparison.  Usage: scripts/ctf_bench.sh TAG
set -u
TAG=${1:-ctf}
mkdir -p gpurun_out
run() { N=$1; shift; timeout 600 python bench.py "$@" --steps 3 --warmup 3 > gpurun_out/${TAG}_$N.json 2> gpurun_out/${TAG}_$N.err; echo $N rc=$?; }
run c3_plain --config c3 --no-e2e --no-cpu-baseline
run c3_ctf2 --config c3 --ctf-defoci 10000,20000
run c2_plain --config c2 --no-e2e --no-cpu-baseline
run c2_ctf4 --config c2 --ctf-defoci 8000,15000,22000,30000
run c5_ctf1 --config c5 --ctf-defoci 15000
python scripts/summ.py gpurun_out/${TAG}_*.json
