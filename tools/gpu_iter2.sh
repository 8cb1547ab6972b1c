#!/bin/bash
# Iteration call: GPU tests (subset via PYT), smoke, bench (no reference arm).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYT:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -n 15 gpurun_out/pytest_gpu.log | cut -c1-300; tail -2 gpurun_out/smoke.log
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").readline())
    print("step ms", round(d["ms_per_step"], 4), "frac", round(d["roofline"]["frac"], 3), "step frac", round(d["roofline"]["step"]["frac"], 3))
    for k, v in d["phases"].items(): print(" ", k, v["kernel"], round(v["us"], 1), "us", round(v["frac"], 3))
    print(" fused", d.get("fused_one_gpu"))
    print(" c4", d.get("decode_c4"))
    print(" lane8", {k: (round(v["ms_per_step"], 4), round(v["frac"], 3)) for k, v in (d.get("lane8") or {}).items()})
    print(" c5", {k: (round(v["quantize_us"], 1), round(v["frac_quantize"], 3), round(v["dequantize_us"], 1), round(v["frac_dequantize"], 3)) for k, v in d["codec_c5"].items()})
except Exception as e:
    print("bench parse failed", e)
PY
tail -n 3 gpurun_out/bench.err
