#!/usr/bin/env bash
# Fused Step 2+3 A/B on a reduced c5 job (2048 images x 128 templates) + one ncu capture of k_step23.
set -u
TAG=${1:-r2}
OUT=gpurun_out
ARGS="--config c5 --images 2048 --templates 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
FTK_S23=0 python bench.py $ARGS > $OUT/ab_sep_${TAG}.json 2> $OUT/ab_sep_${TAG}.err || { tail -20 $OUT/ab_sep_${TAG}.err; exit 1; }
python bench.py $ARGS > $OUT/ab_fused_${TAG}.json 2> $OUT/ab_fused_${TAG}.err || { tail -20 $OUT/ab_fused_${TAG}.err; exit 1; }
python - <<PY
import json
for t in ("sep", "fused"):
    d = json.load(open("$OUT/ab_%s_${TAG}.json" % t))
    print(t, "value %.3e" % d["value"], "ms/step %.1f" % d["ms_per_step"], {k: round(v, 2) for k, v in d["kernel_ms"].items()}, d["clocks"])
PY
ARGS1="--config c5 --images 512 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS1 > $OUT/plain_s23_${TAG}.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step23 -s 1 -c 1 \
    -o $OUT/prof_s23_${TAG} python bench.py $ARGS1 > $OUT/ncu_s23_${TAG}.log 2>&1
echo done
