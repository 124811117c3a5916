#!/usr/bin/env bash
# (needs both .so files under abtmp/, which is not tracked)
# Alternating A/B of two prebuilt libftk.so files (abtmp/$LIB_A, abtmp/$LIB_B) at c5 shapes (kernel ms per step).
set -u
A="--config c5 --images 2048 --templates 256 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  for L in $LIB_A $LIB_B; do
    cp abtmp/$L paper_1905_12317_b200/libftk.so
    timeout 300 python bench.py $A > gpurun_out/ablib_${L}_$i.json 2> gpurun_out/ablib_${L}_$i.err
  done
done
python scripts/summ.py gpurun_out/ablib_*.json
