"""Summarise bench.py JSON lines: value, ms/step, per-kernel ms, roofline fraction, clock reasons.
Usage: python scripts/summ.py gpurun_out/*.json (used by full_bench.sh / gpu_round.sh / ctf_bench.sh)."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f.split("/")[-1], "%.3e" % d["value"], "ms/step %.1f" % d["ms_per_step"],
          {k: round(v, 1) for k, v in d["kernel_ms"].items()}, "frac %.3f" % r["frac"], r["kernel"],
          "issued %.0f" % (r.get("tensor_issued_tflops") or 0), d["clocks"].get("reasons"))
