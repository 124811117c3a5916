#!/usr/bin/env bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over scripts/sanitize_case.py on one GPU.
# Logs: gpurun_out/san_<tool>.log
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --version > gpurun_out/san_version.log 2>&1
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $T --print-limit 50 --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/san_$T.log 2>&1
  echo "$T rc=$?" | tee -a gpurun_out/san_$T.log
done
