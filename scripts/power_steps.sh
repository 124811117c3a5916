#!/usr/bin/env bash
# Board power and SM clock while one step's kernel runs alone (FTK_ONLY_STEP=1|2|3; results are garbage) vs the
# whole step, c5 shapes, one B200: energy per pair of each kernel = power x time / pairs.
set -u
A="--config c5 --images 2048 --templates 512 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
for S in ${STEPS:-0 1 2 3}; do
  FTK_ONLY_STEP=$S timeout 300 python bench.py $A > gpurun_out/pw_$S.json 2> gpurun_out/pw_$S.err
  FTK_S2TC=0 FTK_ONLY_STEP=$S timeout 300 python bench.py $A > gpurun_out/pw_fft_$S.json 2> gpurun_out/pw_fft_$S.err
done
python - <<'PY'
import json
for tag in ["", "fft_"]:
    for S in range(4):
        try:
            d = json.load(open(f"gpurun_out/pw_{tag}{S}.json"))
        except Exception as e:
            print(tag, S, "failed", e); continue
        c = d["clocks"]; k = d["kernel_ms"]
        print(f"{tag or 'tc_'}step{S}: ms/step {d['ms_per_step']:.1f} kernels {[round(k[x],1) for x in ('step1','step2','step3')]} "
              f"power {c.get('power_w')} W clock {c.get('sm_mhz')} MHz cap {c.get('power_cap_frac')}")
PY
