#!/usr/bin/env bash
# A/B of Step 2: CUDA-core k_step2_fft vs tensor-core k_step2_tc (plus timing-only variants) at c5 shapes.
set -u
A="--config c5 --images 2048 --templates 128 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
FTK_S2TC=0 timeout 300 python bench.py $A > gpurun_out/ab_fft.json 2> gpurun_out/ab_fft.err
FTK_S2TC=1 timeout 300 python bench.py $A > gpurun_out/ab_tc.json 2> gpurun_out/ab_tc.err
for D in ${DBGS:-}; do FTK_S2TC=1 FTK_S2TC_DBG=$D timeout 300 python bench.py $A > gpurun_out/ab_tc_d$D.json 2> gpurun_out/ab_tc_d$D.err; done
python scripts/summ.py gpurun_out/ab_*.json
timeout 200 python scripts/s2tc_check.py 2>&1 | tail -4
if [ -n "${NCU:-}" ]; then
FTK_S2TC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step2_tc -s 0 -c 1 -o gpurun_out/prof_s2tc_$NCU python bench.py --config c5 --images 1024 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_s2tc.log 2>&1; echo ncu rc=$?
fi
