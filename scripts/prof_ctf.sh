#!/usr/bin/env bash
# ncu --set full of one Step-1 launch, c3 plain vs c3 x 2 defoci (CTF kernel).  Usage: scripts/prof_ctf.sh TAG
set -u
TAG=$1
OUT=gpurun_out
mkdir -p $OUT
A="--config c3 --images 1024 --templates 256 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $A > $OUT/${TAG}_plain.json 2>&1 && python bench.py $A --ctf-defoci 10000,20000 > $OUT/${TAG}_ctf.json 2>&1 || exit 1
FTK_VERBOSE=1 python bench.py $A --ctf-defoci 10000,20000 2>&1 | grep -i "block\|shape" | head -5
for V in plain ctf; do
  X=""; [ $V = ctf ] && X="--ctf-defoci 10000,20000"
  ncu --set full --clock-control none -k regex:k_step1 -s 0 -c 1 -o $OUT/${TAG}_s1_$V python bench.py $A $X > $OUT/${TAG}_ncu_$V.log 2>&1
done
echo done
